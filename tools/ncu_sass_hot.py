"""Hot SASS lines of an `ncu --page source --csv --print-source sass` export:
python tools/ncu_sass_hot.py file.csv [top]  (stall samples, executed counts,
dominant stall reasons per line)."""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    k, ex = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"]
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    f = lambda v: float(v or 0)  # noqa: E731
    tot = sum(f(r[k]) for r in data)
    print(f"samples {tot:.0f}  warp-instructions executed {sum(f(r[ex]) for r in data):.0f}")
    agg = {s: sum(f(r[ix[s]]) for r in data) for s in stalls}
    print("stall mix:", ", ".join(f"{s[6:]}={v / tot * 100:.1f}%" for s, v in
                                  sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
    for r in sorted(data, key=lambda r: -f(r[k]))[:top]:
        why = sorted(((f(r[ix[s]]), s[6:]) for s in stalls), reverse=True)[:2]
        print(f"{r[ix['Address']][-5:]} {f(r[k]) / tot * 100:5.1f}% ex={r[ex]:>8s} "
              f"{r[ix['Source']].strip()[:60]:60s} {why[0][1]}:{why[0][0]:.0f} {why[1][1]}:{why[1][0]:.0f}")


if __name__ == "__main__":
    main()
