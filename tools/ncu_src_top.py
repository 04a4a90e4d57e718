"""Top stall-sampled SASS instructions from an `ncu --page source --csv` export:
python tools/ncu_src_top.py src.csv[.gz] [n]"""
import csv
import gzip
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
op = gzip.open if path.endswith(".gz") else open
with op(path, "rt") as fh:
    rows = list(csv.reader(fh))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
ex = sum(int(r[ix["Instructions Executed"]] or 0) for r in body)
print(f"samples {tot}, warp instructions executed {ex}")
top = sorted(body, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:n]
for r in top:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{s:6d} {100 * s / max(tot, 1):5.1f}%  ex={r[ix['Instructions Executed']]:>7s}  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:90]}")
