"""Repeatability of the in-flight throughput: python tools/stress_conc.py [conc] [reps]
(c3 fp32, 48 transforms per rep; prints every rep so hiccups show)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402

conc = int(sys.argv[1]) if len(sys.argv) > 1 else 6
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
imgs = [torch.from_numpy(P.sparse_image(4096, 100, 7 + i, snr_db=20.0).x).cuda() for i in range(8)]
xs = [imgs[i % 8] for i in range(48)]
from paper_1908_02461_b200 import batch as PB  # noqa: E402
for j in range(8):
    PB.warm_workers(lambda j=j: P.atsfft2d_arrays(imgs[j], P.TunerConfig(), 8, 11, precision="fp32"), conc)
P.atsfft2d_batch(xs, P.TunerConfig(), 8, [11] * len(xs), concurrency=conc, precision="fp32", arrays=True)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.atsfft2d_batch(xs, P.TunerConfig(), 8, [11] * len(xs), concurrency=conc, precision="fp32",
                     arrays=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"rep {r}: {len(xs) / dt:8.1f} transforms/s", flush=True)
