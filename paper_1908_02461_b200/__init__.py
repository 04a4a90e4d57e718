"""B200-native 2D sparse FFT with adaptive sparsity detection (ATSFFT,
arXiv 1908.02461) — a drop-in for the reference ``sfft2d`` package's hot path.

Public surface mirrors ``/root/reference/pkg/src/sfft2d/__init__.py``: the
fixed-sparsity transform ``sfft2d`` (Algorithm 1), the sparsity-detecting
``atsfft2d`` (Algorithm 2), ``detect_sparsity``, ``count_local_maxima``, the
hash front end (``binned_spectrum``, permutations, flat windows, coordinate
maps) and their configuration/state types.  Every transform runs on the GPU
through ``libsfft2d_b200.so`` (C ABI: ``include/sfft2d_b200.h``); there is no
CPU fallback.  ``precision="fp64"`` (default) reproduces the reference's
float64 arithmetic; ``precision="fp32"`` is the fast path.
"""

__version__ = "0.1.0"

from .batch import atsfft2d_batch, sfft2d_batch
from .engine import (ConfigurationError, SfftConfig, default_bins, estimate_once, median_combine,
                     seek_location_once, sfft2d, sfft2d_arrays, vote_and_select)
from .hashing import (BinGrid, FlatWindow, PermutationParams, WindowCache, all_pass_window,
                      binned_spectrum, build_flat_window, draw_permutation, hash_coord,
                      identity_permutation, mod_inverse, offset_coord, unhash_bin)
from .signals import (device_sparse_image, error_metric, load_signal, planted_image, save_signal,
                      sparse_image)
from .tuner import (TunerConfig, TunerState, atsfft2d, atsfft2d_arrays, count_local_maxima,
                    detect_sparsity, update_bins)

__all__ = [
    "__version__", "ConfigurationError", "SfftConfig", "default_bins", "sfft2d", "sfft2d_arrays",
    "BinGrid", "FlatWindow", "PermutationParams", "WindowCache", "all_pass_window",
    "binned_spectrum", "build_flat_window", "draw_permutation", "hash_coord",
    "identity_permutation", "mod_inverse", "offset_coord", "unhash_bin", "error_metric",
    "planted_image", "sparse_image", "TunerConfig", "TunerState", "atsfft2d", "atsfft2d_arrays",
    "count_local_maxima", "detect_sparsity", "update_bins", "atsfft2d_batch", "sfft2d_batch",
    "seek_location_once", "vote_and_select", "estimate_once", "median_combine", "save_signal",
    "load_signal", "device_sparse_image",
]
