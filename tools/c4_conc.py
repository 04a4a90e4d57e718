"""c4 batched throughput vs in-flight concurrency: python tools/c4_conc.py [images]
(device-generated c4 images, bench.c4_params seeds)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1908_02461_b200 as P  # noqa: E402
from paper_1908_02461_b200.signals import device_sparse_image  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
xs = []
for i in range(n):
    seed, k = bench.c4_params(i)
    xs.append(device_sparse_image(1024, k, seed, snr_db=25.0, magnitude="loguniform").x)
seeds = [1 + i for i in range(n)]
for conc in (4, 6, 8, 12, 16, 24):
    P.atsfft2d_batch(xs, P.TunerConfig(), 8, seeds, concurrency=conc, precision="fp32", arrays=True)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        t0 = time.perf_counter()
        P.atsfft2d_batch(xs, P.TunerConfig(), 8, seeds, concurrency=conc, precision="fp32", arrays=True)
        torch.cuda.synchronize()
        best = max(best, n / (time.perf_counter() - t0))
    print(f"c4 concurrency {conc:2d}: {best:8.1f} images/s", flush=True)
