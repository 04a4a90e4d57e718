"""Summarise an `ncu --page raw --csv` export per launch and per kernel:
python tools/ncu_summary.py raw.csv [--launches] [--json out.json]

Per kernel: launches, summed duration, DRAM read/write bytes per launch,
achieved DRAM GB/s (bytes / duration), DRAM %-of-peak, L2 hit rate.  With
--json, writes {kernel: dram bytes per launch} (the bench's roofline
`traffic`, keyed like the library's profiler names)."""
import collections
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
         "usecond": 1, "nsecond": 1e-3, "msecond": 1e3, "%": 1}


def _pivot_long(rows):
    """`ncu --metrics ... --csv` long format (one row per metric) -> raw-page
    layout (header row, unit row, one row per launch)."""
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    launches, order, units = {}, [], {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        lid = r[ix["ID"]]
        if lid not in launches:
            launches[lid] = {"Kernel Name": r[ix["Kernel Name"]], "Grid Size": r[ix["Grid Size"]],
                             "Block Size": r[ix["Block Size"]]}
            order.append(lid)
        launches[lid][r[ix["Metric Name"]]] = r[ix["Metric Value"]]
        units[r[ix["Metric Name"]]] = r[ix["Metric Unit"]]
    cols = ["Kernel Name", "Grid Size", "Block Size"] + sorted(units)
    out = [cols, [units.get(c, "") for c in cols]]
    for lid in order:
        out.append([launches[lid].get(c, "") for c in cols])
    return out


def load(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    if "Metric Name" in rows[0]:
        rows = _pivot_long(rows)
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def get(r, k):
        try:
            return float(r[ix[k]].replace(",", "")) * SCALE.get(units[ix[k]], 1)
        except (KeyError, ValueError):
            return float("nan")

    out = []
    for r in data:
        nm = r[ix["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").replace("sfft::", "")
        out.append({"kernel": nm.strip(), "grid": r[ix.get("Grid Size", 0)],
                    "block": r[ix.get("Block Size", 0)],
                    "us": get(r, "gpu__time_duration.sum"),
                    "rd": get(r, "dram__bytes_read.sum"), "wr": get(r, "dram__bytes_write.sum"),
                    "dram_pct": get(r, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                    "l2_hit": get(r, "lts__t_sector_hit_rate.pct"),
                    "sm_pct": get(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed")})
    return out


def main():
    path = sys.argv[1]
    launches = load(path)
    if "--launches" in sys.argv:
        for i, l in enumerate(launches):
            gbs = (l["rd"] + l["wr"]) / (l["us"] * 1e3)
            print(f"{i:3d} {l['kernel']:22s} grid={l['grid']:>14s} {l['us']:8.1f} us "
                  f"rd={l['rd'] / 1e6:8.2f} MB wr={l['wr'] / 1e6:7.2f} MB {gbs:7.0f} GB/s "
                  f"dram%={l['dram_pct']:5.1f} l2hit={l['l2_hit']:5.1f}")
    agg = collections.defaultdict(list)
    for l in launches:
        agg[l["kernel"]].append(l)
    tot = sum(l["us"] for l in launches)
    print(f"{len(launches)} launches, {tot:.0f} us serialised (cold cache, ncu replay)")
    print(f"{'kernel':22s} {'n':>3s} {'us':>8s} {'share':>6s} {'rd MB/l':>8s} {'wr MB/l':>8s} "
          f"{'GB/s':>7s} {'dram%':>6s} {'l2hit':>6s}")
    traffic = {}
    for nm, ls in sorted(agg.items(), key=lambda kv: -sum(l["us"] for l in kv[1])):
        us = sum(l["us"] for l in ls)
        rd = sum(l["rd"] for l in ls)
        wr = sum(l["wr"] for l in ls)
        traffic[nm] = (rd + wr) / len(ls)
        print(f"{nm:22s} {len(ls):3d} {us:8.1f} {us / tot * 100:5.1f}% {rd / len(ls) / 1e6:8.2f} "
              f"{wr / len(ls) / 1e6:8.2f} {(rd + wr) / (us * 1e3):7.0f} "
              f"{sum(l['dram_pct'] for l in ls) / len(ls):6.1f} "
              f"{sum(l['l2_hit'] for l in ls) / len(ls):6.1f}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(traffic, fh, indent=1)


if __name__ == "__main__":
    main()
