"""Run a few c3 ATSFFT transforms (for ncu captures): python tools/run_one.py [fp32|fp64] [reps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
img = P.sparse_image(4096, 100, 7, snr_db=20.0)
x = torch.from_numpy(img.x).cuda()
for _ in range(reps):
    out, st = P.atsfft2d(x, P.TunerConfig(), 8, 11, precision=prec)
torch.cuda.synchronize()
print("ok", len(out), st.detected_k)
