"""Brief of one `ncu --page details --csv` + `--page source --csv` pair:
python tools/ncu_brief.py details.csv [source.csv] — key launch/throughput
metrics and the SASS lines holding the most warp-stall samples."""
import csv
import sys

WANT = ["Duration", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Executed Instructions",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block", "Block Size",
        "Grid Size", "L2 Hit Rate", "Mem Busy"]


def details(path):
    rows = list(csv.reader(open(path)))
    ix = {k: i for i, k in enumerate(rows[0])}
    first = rows[1][ix["ID"]] if len(rows) > 1 else None
    for r in rows[1:]:
        if r[ix["ID"]] == first and r[ix["Metric Name"]] in WANT:
            print(f"  {r[ix['Metric Name']]:36s} {r[ix['Metric Value']]} {r[ix['Metric Unit']]}")


def source(path, frac=0.015):
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1], None, []]
            blocks.append(cur)
        elif r and r[0] == "Address" and cur is not None:
            cur[1] = r
        elif cur and cur[1] and len(r) == len(cur[1]):
            cur[2].append(r)
    if not blocks:
        return
    _, hdr, data = blocks[0]
    ix = {h: i for i, h in enumerate(hdr)}
    k, ex = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"]
    tot = sum(float(r[k] or 0) for r in data) or 1.0
    for n, r in enumerate(data):
        if float(r[k] or 0) / tot > frac:
            print(f"  {n:5d} {float(r[k] or 0) / tot * 100:5.1f}% ex={r[ex]:>9s} {r[ix['Source']].strip()[:72]}")


if __name__ == "__main__":
    details(sys.argv[1])
    if len(sys.argv) > 2:
        source(sys.argv[2])
