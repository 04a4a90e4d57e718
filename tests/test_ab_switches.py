"""The A/B switches of the native library select alternative
code paths, never different results: each is run in a fresh process (the
library reads them once) on cases that exercise its path, and the output must
equal the reference golden like the default path's does."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

# switch -> golden cases whose path it changes
SWITCHES = {
    "SFFT2D_NO_PASSCONV": ["c2_ats"],             # B = N/2 pass by fold + FFT
    "SFFT2D_NO_CONV": ["c4b_00"],                 # estimation at B < N by folds
    "SFFT2D_OLD_MLFOLD": ["c3_sfft", "c1_sfft"],  # multi-loop fold k_fold
    "SFFT2D_NO_PASS_PIPE": ["c2_ats"],            # post-fold work on the main stream
    "SFFT2D_OLD_VOTE_LAZY": ["c2_ats"],           # one-pass-at-a-time lazy votes
    "SFFT2D_NO_SPEC": ["c2_ats"],                 # no speculative next-pass folds
    "SFFT2D_NO_EARLY_VOTES": ["c2_ats"],          # one vote tally at the end
    "SFFT2D_NO_SMALL_BITMAP": ["c2_ats"],         # small-pass vote bitmaps by k_vote_bitmap
    "SFFT2D_OLD_LMAX_WIN": ["c2_ats"],            # k_lmax_win (natural-column lanes, per-warp atomics)
    "SFFT2D_NO_EARLY_EST": ["c3_sfft", "c1_sfft"],  # estimation folds after the candidate count
    "SFFT2D_SYNC_ALIVE": ["c3_sfft", "c1_sfft"],    # alive count read before the top-k cut
    "SFFT2D_NO_FUSED_CUT": ["c3_sfft", "c1_sfft", "c4b_00"],  # K7 tail by the general kernels
    "SFFT2D_NO_TOPK_LIST": ["c3_sfft", "c1_sfft"],  # location top-k by the bitmask kernels
    "SFFT2D_OLD_PASSCONV": ["c2_ats"],            # fixed 4-row (2 in fp64) tiles for the B = N/2 pass
    "SFFT2D_FP64_FACTORED": ["c3_ats"],           # fp64 dense FFT without a stored x_hat (no k_pass_conv)
    "SFFT2D_NO_FUSED_TAIL": ["c2_ats"],           # dense estimate + selection by the general kernels
}

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
import paper_1908_02461_b200 as P
from tests.conftest import golden, fixture_input
out = {}
for name in %(cases)r:
    g = golden(name)
    x = fixture_input(g)
    if name.endswith("_sfft"):
        n, k, loops, b, thr, seed = (int(v) for v in g["cfg"])
        cfg = P.SfftConfig(n=n, k=k, loops=loops, b_bins=b, vote_threshold=thr)
        got = P.sfft2d(x, cfg, seed, precision="fp64")
    else:
        t = g["tuner"]
        tc = P.TunerConfig(b0=int(t[0]), eps1=float(t[1]), eps2=float(t[2]), delta1=float(t[3]),
                           delta2=float(t[4]), max_tuning_iters=None if t[5] < 0 else int(t[5]),
                           mag_floor=float(t[6]))
        got, st = P.atsfft2d(x, tc, int(g["est_loops"]), int(g["seed"]), precision="fp64")
    ref = dict(zip(map(tuple, g["coords"].tolist()), g["vals"].tolist()))
    vmax = max([abs(v) for v in ref.values()] or [1.0])
    worst = max([abs(got[key] - v) / max(abs(v), 1e-3 * vmax) for key, v in ref.items() if key in got] or [0.0])
    out[name] = {"same_support": set(got) == set(ref), "worst": worst}
print(json.dumps(out))
"""


@pytest.mark.parametrize("switch", sorted(SWITCHES))
def test_switch_keeps_results(switch):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, **{switch: "1"})
    code = SCRIPT % {"root": ROOT, "cases": SWITCHES[switch]}
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for name, v in res.items():
        assert v["same_support"], (switch, name)
        assert v["worst"] <= 1e-10, (switch, name, v["worst"])
