"""Batched / concurrent transforms on one GPU (BASELINE.json config c4: many
independent images).

ATSFFT is a chain of small sequential tuner passes, so one transform cannot
fill 148 SMs.  Independent images are therefore run `concurrency` at a time,
each on its own host thread with its own native context (workspace + CUDA
streams); ctypes releases the GIL for the duration of the native call, so the
latency-bound passes of one image overlap the bandwidth-bound passes of
another.  Results are exactly those of calling ``atsfft2d`` on each image.
"""

from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor

from . import _native
from .engine import SfftConfig, sfft2d, sfft2d_arrays
from .tuner import TunerConfig, atsfft2d, atsfft2d_arrays

__all__ = ["atsfft2d_batch", "sfft2d_batch", "warm_workers"]

_pools: dict = {}


def _pool(workers: int) -> ThreadPoolExecutor:
    pool = _pools.get(workers)
    if pool is None:
        pool = ThreadPoolExecutor(max_workers=workers, thread_name_prefix="sfft2d")
        _pools[workers] = pool
    return pool


_local = threading.local()


def _worker_stream(torch, device):
    """This worker thread's own CUDA stream on `device` (the legacy default
    stream every thread would otherwise share serialises the batch)."""
    streams = getattr(_local, "streams", None)
    if streams is None:
        streams = _local.streams = {}
    s = streams.get(device)
    if s is None:
        s = streams[device] = torch.cuda.Stream(device=device)
    return s


def _run(fn, n_items, concurrency, device):
    """Run fn(i) for every item, `concurrency` at a time, each worker on its
    own stream ordered after the caller's current stream."""
    if concurrency <= 1 or n_items <= 1:
        return [fn(i) for i in range(n_items)]
    torch = _native._torch()
    if not torch.cuda.is_available():
        return list(_pool(concurrency).map(fn, range(n_items)))
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    ready = torch.cuda.current_stream(dev).record_event()

    def one(i):
        s = _worker_stream(torch, dev)
        s.wait_event(ready)
        with torch.cuda.stream(s):
            return fn(i)

    return list(_pool(concurrency).map(one, range(n_items)))


def warm_workers(fn, concurrency: int, device=None) -> None:
    """Run fn() once on EVERY worker thread of the `concurrency` pool (a barrier
    makes the pool start all of them), so each thread's native context, pinned
    result buffer and workspace exist before a timed or latency-sensitive batch:
    creating them later (cudaHostAlloc, table uploads) synchronises the device
    and stalls every transform in flight."""
    if concurrency <= 1:
        fn()
        return
    barrier = threading.Barrier(concurrency)
    torch = _native._torch()
    dev = None
    if torch.cuda.is_available():
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)

    def one(_):
        barrier.wait()
        if dev is None:
            return fn()
        s = _worker_stream(torch, dev)
        with torch.cuda.stream(s):
            return fn()

    list(_pool(concurrency).map(one, range(concurrency)))


def _shared_generators(rngs) -> bool:
    """True when one numpy Generator object is passed for several items: the
    native controller draws straight from its bit generator, so those items
    must run one after another in input order (as sequential calls would)."""
    import numpy as np
    seen = set()
    for r in rngs:
        if isinstance(r, np.random.Generator):
            if id(r) in seen:
                return True
            seen.add(id(r))
    return False


def atsfft2d_batch(xs, cfg: TunerConfig, est_loops: int, rngs, *, concurrency: int = 4,
                   precision: str = "fp64", device=None, arrays: bool = False):
    """``atsfft2d`` over a batch: ``xs`` images, ``rngs`` one seed/Generator per
    image.  Returns a list of ``(spectrum, TunerState)`` in input order
    (``((coords, values), state)`` with ``arrays=True``)."""
    if len(xs) != len(rngs):
        raise ValueError("need one rng per image")
    fn = atsfft2d_arrays if arrays else atsfft2d
    if _shared_generators(rngs):
        concurrency = 1

    def one(i):
        return fn(xs[i], cfg, est_loops, rngs[i], precision=precision, device=device)

    return _run(one, len(xs), concurrency, device)


def sfft2d_batch(xs, cfg: SfftConfig, rngs, *, concurrency: int = 4, precision: str = "fp64",
                 device=None, arrays: bool = False):
    """``sfft2d`` over a batch of images (one rng per image), input order kept."""
    if len(xs) != len(rngs):
        raise ValueError("need one rng per image")
    fn = sfft2d_arrays if arrays else sfft2d
    if _shared_generators(rngs):
        concurrency = 1

    def one(i):
        return fn(xs[i], cfg, rngs[i], precision=precision, device=device)

    return _run(one, len(xs), concurrency, device)
