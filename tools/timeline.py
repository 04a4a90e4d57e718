"""GPU timeline of one workload's transforms from a CUPTI kernel trace
(torch.profiler): busy vs idle time per transform and the largest gaps.
python tools/timeline.py [fp32|fp64] [reps] [c3|c1|c2|c3sfft|c5]"""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
work = sys.argv[3] if len(sys.argv) > 3 else "c3"
if work == "c1":
    sig = P.planted_image(256, 10, 1)
    x = torch.from_numpy(sig.x).cuda()
    def call():
        return P.sfft2d_arrays(x, P.SfftConfig(n=256, k=10), 2, precision=prec)
elif work == "c3sfft":
    x = torch.from_numpy(P.sparse_image(4096, 100, 7, snr_db=20.0).x).cuda()
    def call():
        return P.sfft2d_arrays(x, P.SfftConfig(n=4096, k=100), 12, precision=prec)
elif work == "c2":
    x = torch.from_numpy(P.sparse_image(1024, 50, 7, snr_db=30.0).x).cuda()
    def call():
        return P.atsfft2d_arrays(x, P.TunerConfig(), 8, 11, precision=prec)
elif work.startswith("c5"):
    k5 = int(work[2:] or 64) if len(work) > 2 else 64
    x = P.device_sparse_image(16384, k5, 5, snr_db=15.0, cluster_frac=0.2, cluster_side=64).x
    def call():
        return P.atsfft2d_arrays(x, P.TunerConfig(), 8, 6, precision=prec)
else:
    x = torch.from_numpy(P.sparse_image(4096, 100, 7, snr_db=20.0).x).cuda()
    def call():
        return P.atsfft2d_arrays(x, P.TunerConfig(), 8, 11, precision=prec)
for _ in range(3):
    call()
torch.cuda.synchronize()
import time  # noqa: E402
t0w = time.perf_counter()
for _ in range(reps):
    call()
torch.cuda.synchronize()
_wall = (time.perf_counter() - t0w) / reps
print(f"{work} {prec}: host wall {_wall * 1e3:.3f} ms per transform (no profiler)")
_out = call()
try:
    print(f"state: passes {len(_out[1].history)}, detected_k {_out[1].detected_k}, b_estimate "
          f"{_out[1].b_estimate}, candidates {getattr(_out[1], 'n_candidates', None)}")
except Exception:  # noqa: BLE001 - SFFT calls return no state
    pass
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        call()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
ks = sorted((e for e in ev if e.get("cat") == "kernel"), key=lambda e: e["ts"])
mem = [e for e in ev if e.get("cat") in ("gpu_memcpy", "gpu_memset")]
t0, t1 = ks[0]["ts"], max(e["ts"] + e["dur"] for e in ks)
busy, end, gaps = 0.0, t0, []
for e in ks:
    s, d = e["ts"], e["dur"]
    if s > end:
        gaps.append((s - end, e["name"][:40]))
    busy += max(0.0, s + d - max(s, end))
    end = max(end, s + d)
span = t1 - t0
print(f"{len(ks) / reps:.0f} kernels/transform, span {span / reps:.1f} us/transform, "
      f"busy {busy / reps:.1f} us ({busy / span * 100:.1f}%), idle {(span - busy) / reps:.1f} us, "
      f"memcpy/memset ops {len(mem) / reps:.0f}/transform")
import collections  # noqa: E402
agg = collections.defaultdict(lambda: [0, 0.0])
for e in ks:
    nm = e["name"].split("(")[0].split("<")[0].replace("void ", "").replace("sfft::", "")
    agg[nm][0] += 1
    agg[nm][1] += e["dur"]
print("per-kernel time per transform (warm pipeline, CUPTI):")
for nm, (cnt, dur) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {nm:24s} {cnt / reps:5.1f} launches {dur / reps:8.1f} us  ({dur / busy * 100:4.1f}% of busy)")
gaps.sort(reverse=True)
big = [g for g in gaps if g[0] > 2.0]
print(f"gaps > 2 us: {len(big) / reps:.1f}/transform totalling {sum(g for g, _ in big) / reps:.1f} us")
for g, nm in gaps[:6]:
    print(f"  {g:7.1f} us before {nm}")
# gaps by the position of the following kernel inside a transform (the last
# transform's sequence; memsets/memcpys in between count as idle)
per = len(ks) // reps
seq = ks[-per:]
print("idle before each kernel of the last transform (> 1 us):")
prev_end = None
for i, e in enumerate(seq):
    nm = e["name"].split("(")[0].split("<")[0].replace("void ", "").replace("sfft::", "")
    if prev_end is not None and e["ts"] - prev_end > 1.0:
        print(f"  [{i:2d}] {e['ts'] - prev_end:6.1f} us before {nm}")
    prev_end = max(prev_end or 0, e["ts"] + e["dur"])
