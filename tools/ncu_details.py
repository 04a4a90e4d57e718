"""Key ncu --page details metrics per launch: python tools/ncu_details.py details.csv[.gz] [kernel-regex] [metric-regex] [rules]"""
import csv
import gzip
import re
import sys

path = sys.argv[1]
kre = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
mre = re.compile(sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] else
                 r"^(Duration|DRAM Throughput|Memory Throughput|Achieved Occupancy|Registers Per Thread|"
                 r"Issue Slots Busy|Executed Ipc Active|L1/TEX Hit Rate|L2 Hit Rate|Theoretical Occupancy|"
                 r"Dynamic Shared Memory Per Block|Waves Per SM|"
                 r"Compute \(SM\) Throughput|One or More Eligible|No Eligible|"
                 r"Avg. Active Threads Per Warp|Warp Cycles Per Issued Instruction|Executed Instructions)$")
op = gzip.open if path.endswith(".gz") else open
rows = {}
with op(path, "rt") as fh:
    for r in csv.DictReader(fh):
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
        if not kre.search(name):
            continue
        key = (int(r["ID"]), name, r["Grid Size"], r["Block Size"])
        if mre.search(r["Metric Name"]):
            rows.setdefault(key, []).append(f'{r["Metric Name"]}={r["Metric Value"]}{r["Metric Unit"]}')
        if r.get("Rule Type") in ("OPT", "WRN") and r.get("Rule Description") and len(sys.argv) > 4:
            rows.setdefault(key, []).append("  ! " + r["Rule Description"][:300])
for k in sorted(rows):
    print(k)
    print("    " + "; ".join(dict.fromkeys(rows[k])))
