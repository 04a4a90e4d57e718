"""Throughput of c3 ATSFFT vs in-flight concurrency: python tools/concurrency.py [fp32|fp64]."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
imgs = [torch.from_numpy(P.sparse_image(4096, 100, 7 + i, snr_db=20.0).x).cuda() for i in range(8)]
from paper_1908_02461_b200 import batch as PB  # noqa: E402
for conc in (1, 2, 3, 4, 6, 8):
    xs = [imgs[i % 8] for i in range(48)]
    for j in range(8):
        PB.warm_workers(lambda j=j: P.atsfft2d_arrays(imgs[j], P.TunerConfig(), 8, 11, precision=prec), conc)
    P.atsfft2d_batch(xs, P.TunerConfig(), 8, [11] * len(xs), concurrency=conc,
                     precision=prec, arrays=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.atsfft2d_batch(xs, P.TunerConfig(), 8, [11] * len(xs), concurrency=conc, precision=prec,
                     arrays=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"concurrency {conc}: {len(xs) / dt:8.1f} transforms/s ({dt / len(xs) * 1e3:.3f} ms each)")
