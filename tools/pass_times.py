"""Per-pass host timings + per-kernel profile of c3 ATSFFT: python tools/pass_times.py [fp32|fp64]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402
from paper_1908_02461_b200 import _native  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
img = P.sparse_image(4096, 100, 7, snr_db=20.0)
x = torch.from_numpy(img.x).cuda()
for _ in range(3):
    out, st = P.atsfft2d(x, P.TunerConfig(), 8, 11, precision=prec)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    out, st = P.atsfft2d(x, P.TunerConfig(), 8, 11, precision=prec)
e1.record()
torch.cuda.synchronize()
print(f"ms/transform {e0.elapsed_time(e1) / 10:.3f}")
import time
t0 = time.perf_counter()
out, st = P.atsfft2d(x, P.TunerConfig(), 8, 11, precision=prec)
t_py = (time.perf_counter() - t0) * 1e6
ctx0 = _native.context()
print(f"python call {t_py:.0f} us, native call {ctx0.last_call_us:.0f} us, "
      f"of which blocked in sync {ctx0.lib.sfft2d_ctx_sync_us(ctx0.handle):.0f} us")
print("passes (B, count, host_us):")
for (b, c, _), us in zip(st.history, st.pass_us):
    print(f"  B={b:5d} count={c:7d} {us:8.1f} us")
ctx = _native.context()
ctx.set_profiling(True)
P.atsfft2d(x, P.TunerConfig(), 8, 11, precision=prec)
rep = ctx.profile_report()
ctx.set_profiling(False)
tot = sum(v[1] for v in rep.values())
print(f"kernel total {tot * 1e3:.1f} us in {sum(v[0] for v in rep.values())} launches")
for k, (n, ms, by) in sorted(rep.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:28s} {n:4d} {ms * 1e3:9.1f} us  {by / ms / 1e6 if ms else 0:8.1f} GB/s")
