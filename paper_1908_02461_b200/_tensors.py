"""Input marshalling for the native path: numpy arrays or CUDA tensors in,
validated exactly like ``corefft.as_complex_matrix`` (corefft.py:38-51)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native


@dataclass
class DeviceImage:
    tensor: object          # torch tensor on the GPU (or None when passed as host pointer)
    host: np.ndarray | None  # contiguous host array (numpy input)
    n: int
    dtype_code: int
    device: int
    from_numpy: bool


def _check_square_pow2(shape):
    if len(shape) != 2 or shape[0] != shape[1]:
        raise ValueError(f"expected a square matrix, got shape {tuple(shape)}")
    n = int(shape[0])
    if not (n >= 1 and (n & (n - 1)) == 0):
        raise ValueError(f"side {n} is not a power of 2")
    return n


def host_image(x) -> tuple[np.ndarray, int]:
    """Contiguous complex64/complex128 host array + its dtype code.  Other
    numeric inputs are upcast to complex128 like the reference."""
    a = np.asarray(x)
    if a.dtype == np.complex64:
        code = _native.C64
    elif a.dtype == np.complex128:
        code = _native.C128
    else:
        a = a.astype(np.complex128)
        code = _native.C128
    _check_square_pow2(a.shape)
    return np.ascontiguousarray(a), code


def is_torch_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def as_device_image(x, device=None, *, upload: bool = True) -> DeviceImage:
    torch = _native._torch()
    if is_torch_tensor(x):
        if not x.is_cuda:
            return as_device_image(x.detach().cpu().numpy(), device, upload=upload)
        if x.dtype == torch.complex64:
            code = _native.C64
        elif x.dtype == torch.complex128:
            code = _native.C128
        else:
            x = x.to(torch.complex128)
            code = _native.C128
        n = _check_square_pow2(tuple(x.shape))
        return DeviceImage(x.contiguous(), None, n, code, x.device.index, False)
    a, code = host_image(x)
    n = a.shape[0]
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    t = torch.from_numpy(a).to(f"cuda:{int(device)}") if upload else None
    return DeviceImage(t, a, n, code, int(device), True)


def to_numpy_complex(t) -> np.ndarray:
    return t.detach().cpu().numpy()
