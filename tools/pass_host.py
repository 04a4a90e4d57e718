"""Host wall time of each tuner pass of one c3 transform (state.pass_us,
from the native controller) + the tail: python tools/pass_host.py [fp32|fp64]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402
from paper_1908_02461_b200 import _native  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
x = torch.from_numpy(P.sparse_image(4096, 100, 7, snr_db=20.0).x).cuda()
ctx = _native.context(0)
rows = []
for it in range(25):
    (ij, v), st = P.atsfft2d_arrays(x, P.TunerConfig(), 8, 11, precision=prec)
    if it >= 5:
        rows.append(list(st.pass_us) + [ctx.last_call_us - sum(st.pass_us)])
a = np.median(np.array(rows), axis=0)
bs = [b for b, _, _ in st.history]
print("pass  B      host us (median of 20)")
for i, b in enumerate(bs):
    print(f"{i:4d} {b:5d} {a[i]:8.1f}")
print(f"tail (votes, estimation, output) {a[-1]:8.1f}")
print(f"native call total {np.median([sum(r) for r in rows]):.1f} us")
