"""Kernel timeline of c4 transforms (1024^2, bench.c4_image): python tools/c4_timeline.py [n]"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_1908_02461_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
xs = [torch.from_numpy(bench.c4_image(i)).cuda() for i in range(n)]
cfg = P.TunerConfig()
for i in range(n):
    P.atsfft2d_arrays(xs[i], cfg, 8, 1 + i, precision="fp32")
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    _, st = P.atsfft2d_arrays(xs[i], cfg, 8, 1 + i, precision="fp32")
torch.cuda.synchronize()
print(f"serial {(time.perf_counter() - t0) / n * 1e6:.0f} us per c4 transform")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(n):
        P.atsfft2d_arrays(xs[i], cfg, 8, 1 + i, precision="fp32")
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
ks = [e for e in ev if e.get("cat") == "kernel"]
import collections  # noqa: E402
agg = collections.defaultdict(lambda: [0, 0.0])
for e in ks:
    nm = e["name"].split("(")[0].split("<")[0].replace("void ", "").replace("sfft::", "")
    agg[nm][0] += 1
    agg[nm][1] += e["dur"]
for nm, (cnt, dur) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {nm:24s} {cnt / n:5.1f} launches {dur / n:8.1f} us per transform")
