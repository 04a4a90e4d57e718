"""Per-stage host time of one c3 atsfft2d_arrays call (mirrors tuner._run_ats):
python tools/py_stages.py [fp32|fp64]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402
from paper_1908_02461_b200 import _native  # noqa: E402
from paper_1908_02461_b200._tensors import as_device_image  # noqa: E402
from paper_1908_02461_b200.engine import _fetch, _stream  # noqa: E402
from paper_1908_02461_b200.tuner import _state  # noqa: E402

prec_s = sys.argv[1] if len(sys.argv) > 1 else "fp32"
img0 = P.sparse_image(4096, 100, 7, snr_db=20.0)
x = torch.from_numpy(img0.x).cuda()
cfg = P.TunerConfig()
for _ in range(5):
    P.atsfft2d_arrays(x, cfg, 8, 11, precision=prec_s)
torch.cuda.synchronize()
names = ["as_device_image", "precision_code", "default_rng", "bitgen ptr", "context", "ensure_tables",
         "cfg._c + structs", "cuda.device enter", "_stream", "native call", "_state", "_fetch",
         "cuda.device exit"]
acc = np.zeros(len(names))
R = 200
t_all = time.perf_counter()
for _ in range(R):
    t = [time.perf_counter()]
    img = as_device_image(x, None, upload=False); t.append(time.perf_counter())
    prec = _native.precision_code(prec_s); t.append(time.perf_counter())
    gen = np.random.default_rng(11); t.append(time.perf_counter())
    bitgen = gen.bit_generator.ctypes.bit_generator.value; t.append(time.perf_counter())
    ctx = _native.context(img.device); t.append(time.perf_counter())
    ctx.ensure_tables(img.n, cfg.window_delta_pass, cfg.window_delta_stop); t.append(time.perf_counter())
    ccfg = cfg._c(); sc = _native.TunerStateC(); res = _native.ResultC(); t.append(time.perf_counter())
    dm = torch.cuda.device(img.device); dm.__enter__(); t.append(time.perf_counter())
    st = _stream(torch, img.device); t.append(time.perf_counter())
    rc = ctx.lib.sfft2d_atsfft_bitgen(ctx.handle, img.tensor.data_ptr(), img.dtype_code, 0, img.n,
                                      ctypes.byref(ccfg), 8, bitgen, prec, st, ctypes.byref(res),
                                      ctypes.byref(sc)); t.append(time.perf_counter())
    ctx.check(rc)
    state = _state(sc); t.append(time.perf_counter())
    ij, vals = _fetch(ctx, res, st, prec); t.append(time.perf_counter())
    dm.__exit__(None, None, None); t.append(time.perf_counter())
    acc += np.diff(t)
tot = (time.perf_counter() - t_all) / R * 1e6
print(f"{prec_s}: {tot:.0f} us per call (sum of stages {acc.sum() / R * 1e6:.0f})")
for nm, v in zip(names, acc / R * 1e6):
    print(f"  {nm:20s} {v:8.1f} us")
ctx.set_profiling(False)
t0 = time.perf_counter()
for _ in range(R):
    P.atsfft2d_arrays(x, cfg, 8, 11, precision=prec_s)
print(f"public atsfft2d_arrays: {(time.perf_counter() - t0) / R * 1e6:.0f} us per call")
