"""Profile the Python-side overhead of atsfft2d_arrays on a c3 image."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402

img = P.sparse_image(4096, 100, 7, snr_db=20.0)
x = torch.from_numpy(img.x).cuda()
cfg = P.TunerConfig()
for _ in range(5):
    P.atsfft2d_arrays(x, cfg, 8, 11, precision="fp32")
pr = cProfile.Profile()
pr.enable()
for _ in range(100):
    P.atsfft2d_arrays(x, cfg, 8, 11, precision="fp32")
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
