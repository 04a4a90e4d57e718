"""Cost of each Python step of atsfft2d_arrays on the GPU box (us per call)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402
from paper_1908_02461_b200 import _native, engine, tuner  # noqa: E402
from paper_1908_02461_b200._tensors import as_device_image  # noqa: E402

x = torch.from_numpy(P.sparse_image(1024, 50, 7, snr_db=30.0).x).cuda()
cfg = P.TunerConfig()
for _ in range(5):
    P.atsfft2d_arrays(x, cfg, 8, 11, precision="fp32")
torch.cuda.synchronize()


def t(name, fn, n=2000):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{name:32s} {(time.perf_counter() - t0) / n * 1e6:8.2f} us")


ctx = _native.context(0)
t("as_device_image", lambda: as_device_image(x, None, upload=False))
t("_generator(11)", lambda: tuner._generator(11))
t("context()", lambda: _native.context(0))
t("ensure_tables", lambda: ctx.ensure_tables(1024, cfg.window_delta_pass, cfg.window_delta_stop))
t("cfg._c()", lambda: cfg._c())
t("TunerStateC()", lambda: _native.TunerStateC())
t("ResultC()", lambda: _native.ResultC())


def dev():
    with torch.cuda.device(0):
        pass


t("torch.cuda.device ctx", dev)
t("_stream", lambda: engine._stream(torch, 0))
t("data_ptr", lambda: x.data_ptr())
sc = _native.TunerStateC()
t("_state(sc)", lambda: tuner._state(sc))
res = _native.ResultC()
t("_fetch (count 0)", lambda: engine._fetch(ctx, res, 0, _native.FP32))
tot = []
nat = []
for _ in range(200):
    t0 = time.perf_counter()
    P.atsfft2d_arrays(x, cfg, 8, 11, precision="fp32")
    tot.append((time.perf_counter() - t0) * 1e6)
    nat.append(ctx.last_call_us)
print(f"c2 total {np.median(tot):.1f} us, native {np.median(nat):.1f} us, python {np.median(tot) - np.median(nat):.1f} us")

# step timestamps through a replica of tuner._run_ats (same calls)
import ctypes  # noqa: E402
from paper_1908_02461_b200.engine import _fetch, _stream  # noqa: E402


def replica(marks):
    T = time.perf_counter
    marks.append(T())
    img = as_device_image(x, None, upload=False)
    n = img.n
    prec = _native.precision_code("fp32")
    gen, bitgen, snapshot = tuner._generator(11)
    c = _native.context(img.device)
    c.ensure_tables(n, cfg.window_delta_pass, cfg.window_delta_stop)
    ccfg = cfg._c()
    sc = _native.TunerStateC()
    r = _native.ResultC()
    marks.append(T())
    with torch.cuda.device(img.device):
        st = _stream(torch, img.device)
        ptr, on_host = img.tensor.data_ptr(), 0
        marks.append(T())
        rc = c.lib.sfft2d_atsfft_bitgen(c.handle, ptr, img.dtype_code, on_host, n, ctypes.byref(ccfg),
                                        8, bitgen, prec, st, ctypes.byref(r), ctypes.byref(sc))
        marks.append(T())
        c.check(rc)
        c.last_launches = int(r.gpu_launches)
        state = tuner._state(sc)
        ij, vals = _fetch(c, r, st, prec)
        marks.append(T())
    marks.append(T())
    return (ij, vals), state


acc = np.zeros(5)
for i in range(300):
    m = []
    replica(m)
    if i >= 50:
        acc += np.diff(m)
acc /= 250
print("replica steps (us): setup %.1f | device ctx+stream %.1f | native call %.1f | state+fetch %.1f | exit %.1f"
      % tuple(acc * 1e6))
