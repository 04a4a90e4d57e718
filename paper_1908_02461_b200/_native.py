"""ctypes binding of ``libsfft2d_b200.so`` (the C ABI in ``include/sfft2d_b200.h``).

There is no CPU fallback: if the library or a CUDA device is missing, every
transform raises ``RuntimeError`` naming what is missing.  One context per CUDA
device holds the device workspace and the registered window/twiddle tables
(the device-side counterpart of the reference's ``WindowCache``,
``hashing.py:249-261``).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsfft2d_b200.so")

OK, ERR_VALUE, ERR_CONFIG, ERR_CUDA, ERR_NOMEM, ERR_UNSUPPORTED, ERR_STATE = 0, -1, -2, -3, -4, -5, -6
C64, C128 = 0, 1
FP32, FP64 = 0, 1
MAX_HISTORY = 256
ABI_VERSION = 3   # include/sfft2d_b200.h SFFT2D_ABI_VERSION

EXPORTS = (
    "sfft2d_abi_version", "sfft2d_ctx_create", "sfft2d_ctx_destroy", "sfft2d_ctx_last_error",
    "sfft2d_ctx_set_tables", "sfft2d_sfft", "sfft2d_atsfft", "sfft2d_detect_sparsity",
    "sfft2d_fetch_result", "sfft2d_fetch_votes", "sfft2d_binned_spectrum", "sfft2d_fft2d",
    "sfft2d_local_maxima", "sfft2d_top_bins", "sfft2d_ctx_set_profiling",
    "sfft2d_ctx_profile_report", "sfft2d_atsfft_bitgen", "sfft2d_detect_sparsity_bitgen",
    "sfft2d_ctx_sync_us", "sfft2d_sfft_votes", "sfft2d_sfft_from_votes",
    "sfft2d_estimate_loops", "sfft2d_median_select", "sfft2d_generate",
    "sfft2d_ctx_set_workspace", "sfft2d_ctx_workspace_size", "sfft2d_sfft_draw_perms",
    "sfft2d_sfft_bitgen",
)


class Perm(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in
                ("sigma1", "sigma2", "tau1", "tau2", "sigma1_inv", "sigma2_inv")]


class SfftCfg(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("k", ctypes.c_int32), ("loops", ctypes.c_int32),
                ("d_factor", ctypes.c_int32), ("vote_threshold", ctypes.c_int32),
                ("b_bins", ctypes.c_int32), ("window_delta_pass", ctypes.c_double),
                ("window_delta_stop", ctypes.c_double), ("gain_floor", ctypes.c_double),
                ("prune_rel", ctypes.c_double)]


class TunerCfg(ctypes.Structure):
    _fields_ = [("b0", ctypes.c_int32), ("max_tuning_iters", ctypes.c_int32),
                ("eps1", ctypes.c_double), ("eps2", ctypes.c_double), ("delta1", ctypes.c_double),
                ("delta2", ctypes.c_double), ("mag_floor", ctypes.c_double),
                ("window_delta_pass", ctypes.c_double), ("window_delta_stop", ctypes.c_double),
                ("gain_floor", ctypes.c_double), ("prune_rel", ctypes.c_double)]


class TunerStateC(ctypes.Structure):
    _fields_ = [("passes", ctypes.c_int32),
                ("hist_bins", ctypes.c_int32 * MAX_HISTORY),
                ("hist_count", ctypes.c_int64 * MAX_HISTORY),
                ("hist_ratio", ctypes.c_double * MAX_HISTORY),
                ("hist_has_ratio", ctypes.c_int32 * MAX_HISTORY),
                ("hist_us", ctypes.c_double * MAX_HISTORY),
                ("converged", ctypes.c_int32), ("detected_k", ctypes.c_int64),
                ("b_detect", ctypes.c_int32), ("b_estimate", ctypes.c_int32),
                ("vote_passes", ctypes.c_int32), ("perms_used", ctypes.c_int32),
                ("n_votes", ctypes.c_int64), ("n_candidates", ctypes.c_int64),
                ("perms_drawn", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class ResultC(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("ordered_by_magnitude", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("n_candidates", ctypes.c_int64),
                ("perms_used", ctypes.c_int32), ("gpu_launches", ctypes.c_int32)]


_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and declare every exported signature."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"native library {path} is missing: build it with `python -c "
                f"'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        P = ctypes.POINTER
        sig = {
            "sfft2d_abi_version": ([], i32),
            "sfft2d_ctx_create": ([i32, P(vp)], i32),
            "sfft2d_ctx_destroy": ([vp], None),
            "sfft2d_ctx_last_error": ([vp], ctypes.c_char_p),
            "sfft2d_ctx_set_tables": ([vp, i32, dbl, dbl, vp, vp, vp], i32),
            "sfft2d_sfft": ([vp, vp, i32, i32, P(SfftCfg), P(Perm), i32, vp, P(ResultC)], i32),
            "sfft2d_atsfft": ([vp, vp, i32, i32, i32, P(TunerCfg), i32, P(Perm), i32, i32, vp,
                               P(ResultC), P(TunerStateC)], i32),
            "sfft2d_detect_sparsity": ([vp, vp, i32, i32, i32, P(TunerCfg), P(Perm), i32, i32, vp,
                                        P(TunerStateC)], i32),
            "sfft2d_atsfft_bitgen": ([vp, vp, i32, i32, i32, P(TunerCfg), i32, vp, i32, vp,
                                      P(ResultC), P(TunerStateC)], i32),
            "sfft2d_detect_sparsity_bitgen": ([vp, vp, i32, i32, i32, P(TunerCfg), vp, i32, vp,
                                               P(TunerStateC)], i32),
            "sfft2d_fetch_result": ([vp, vp, vp, i32, vp], i32),
            "sfft2d_fetch_votes": ([vp, vp, vp, i32, vp], i32),
            "sfft2d_binned_spectrum": ([vp, vp, i32, i32, i32, P(Perm), i32, dbl, dbl, i32, vp, vp],
                                       i32),
            "sfft2d_fft2d": ([vp, vp, i32, i32, i32, i32, vp], i32),
            "sfft2d_local_maxima": ([vp, vp, i32, dbl, i32, P(i64), vp, i64, vp], i32),
            "sfft2d_top_bins": ([vp, vp, i32, i32, i64, i32, vp, vp], i32),
            "sfft2d_ctx_set_profiling": ([vp, i32], i32),
            "sfft2d_ctx_sync_us": ([vp], dbl),
            "sfft2d_sfft_votes": ([vp, vp, i32, i32, P(SfftCfg), P(Perm), i32, i32, vp, vp], i32),
            "sfft2d_sfft_from_votes": ([vp, vp, i32, i32, P(SfftCfg), vp, P(Perm), i32, vp,
                                        P(ResultC)], i32),
            "sfft2d_ctx_profile_report": ([vp, ctypes.c_char_p, i64], i64),
            "sfft2d_estimate_loops": ([vp, vp, i32, i32, i32, i32, dbl, dbl, dbl, vp, i64, P(Perm),
                                       i32, i32, vp, vp, vp], i32),
            "sfft2d_median_select": ([vp, i32, vp, i64, vp, vp, i32, i64, dbl, i32, vp,
                                      P(ResultC)], i32),
            "sfft2d_ctx_set_workspace": ([vp, vp, i64], i32),
            "sfft2d_sfft_draw_perms": ([vp, i32, i32, P(Perm)], i32),
            "sfft2d_sfft_bitgen": ([vp, vp, i32, i32, P(SfftCfg), vp, i32, vp, P(ResultC)], i32),
            "sfft2d_ctx_workspace_size": ([vp, P(i64), P(i64)], i32),
            "sfft2d_generate": ([vp, i32, i64, vp, vp, vp, dbl, ctypes.c_uint64, i32, vp, vp],
                                i32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.sfft2d_abi_version() != ABI_VERSION:
            raise RuntimeError(f"{path} has ABI version {lib.sfft2d_abi_version()}, this package "
                               f"expects {ABI_VERSION}: rebuild it (g.build())")
        _lib = lib
        return lib


def _torch():
    import torch
    return torch


class StatusError(RuntimeError):
    pass


class Context:
    """Per-device native context (workspace + registered tables)."""

    def __init__(self, device: int):
        self.lib = load_library()
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device is available: the sm_100a path has no CPU fallback")
        self.device = device
        with torch.cuda.device(device):
            h = ctypes.c_void_p()
            rc = self.lib.sfft2d_ctx_create(device, ctypes.byref(h))
            if rc != OK:
                raise RuntimeError(f"sfft2d_ctx_create failed with status {rc}")
        self.handle = h
        self._tables: set = set()
        self.last_launches = 0
        self._lock = threading.Lock()

    def error(self) -> str:
        msg = self.lib.sfft2d_ctx_last_error(self.handle)
        return msg.decode() if msg else ""

    def check(self, rc: int):
        if rc == OK:
            return
        msg = self.error()
        if rc == ERR_VALUE:
            raise ValueError(msg)
        if rc == ERR_CONFIG:
            from .engine import ConfigurationError
            raise ConfigurationError(msg)
        raise StatusError(f"sfft2d status {rc}: {msg}")

    def set_profiling(self, enable: bool):
        self.check(self.lib.sfft2d_ctx_set_profiling(self.handle, 1 if enable else 0))

    def profile_report(self) -> dict:
        """{kernel: (launches, total_ms, total_algorithmic_bytes)} since enabling."""
        buf = ctypes.create_string_buffer(1 << 20)
        n = self.lib.sfft2d_ctx_profile_report(self.handle, buf, len(buf))
        if n < 0:
            self.check(int(n))
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms, by = line.split()
            out[name] = (int(cnt), float(ms), float(by))
        return out

    def workspace_size(self) -> tuple:
        """(bytes in use, high-water mark) of this context's device workspace."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self.check(self.lib.sfft2d_ctx_workspace_size(self.handle, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def use_workspace(self, buf) -> None:
        """Run every later call of this context inside the caller-owned device
        buffer `buf` (a CUDA uint8 tensor, kept alive here); None returns to
        the context's own pool."""
        if buf is None:
            self.check(self.lib.sfft2d_ctx_set_workspace(self.handle, None, 0))
            self._ws_buf = None
            return
        if not buf.is_cuda or not buf.is_contiguous():
            raise ValueError("workspace must be a contiguous CUDA tensor")
        self.check(self.lib.sfft2d_ctx_set_workspace(self.handle, buf.data_ptr(),
                                                     buf.numel() * buf.element_size()))
        self._ws_buf = buf

    def ensure_tables(self, n: int, delta_pass: float, delta_stop: float):
        key = (n, float(delta_pass), float(delta_stop))
        if key in self._tables:
            return
        from .hashing import host_tables
        space, freq, tw = host_tables(n, delta_pass, delta_stop)
        self.check(self.lib.sfft2d_ctx_set_tables(
            self.handle, n, float(delta_pass), float(delta_stop),
            space.ctypes.data, freq.ctypes.data, tw.ctypes.data))
        self._tables.add(key)


_contexts: dict = {}
_ctx_lock = threading.Lock()


def context(device=None) -> Context:
    """The calling thread's context on `device`: a context (workspace, streams,
    tables) must not be shared by concurrent host threads, so each thread gets
    its own — this is what lets independent transforms run concurrently."""
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device is available: the sm_100a path has no CPU fallback")
    if device is None:
        device = torch.cuda.current_device()
    key = (int(device), threading.get_ident())
    ctx = _contexts.get(key)
    if ctx is None:
        with _ctx_lock:
            ctx = _contexts.get(key)
            if ctx is None:
                ctx = Context(int(device))
                _contexts[key] = ctx
    return ctx


def perm_array(perms) -> ctypes.Array:
    arr = (Perm * max(len(perms), 1))()
    for i, p in enumerate(perms):
        arr[i] = Perm(p.sigma1, p.sigma2, p.tau1, p.tau2, p.sigma1_inv, p.sigma2_inv)
    return arr


def precision_code(precision) -> int:
    if precision in ("fp64", "float64", FP64, np.float64):
        return FP64
    if precision in ("fp32", "float32", FP32, np.float32):
        return FP32
    raise ValueError(f"unknown precision {precision!r} (use 'fp64' or 'fp32')")
