"""Golden vectors for adaptive density control: runs the reference's own
densify_and_prune / reset_opacity (gsmesh/train/densify.py:46-101, Adam row
surgery adam.py:44-60) on fp32-quantised inputs and stores inputs and
outputs in tests/golden/densify.npz.

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden_densify.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from gsmesh.config import TrainConfig  # noqa: E402
from gsmesh.train.adam import Adam  # noqa: E402
from gsmesh.train.densify import DensifyState, densify_and_prune, reset_opacity  # noqa: E402


def q32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    rng = np.random.default_rng(7)
    n = 3000
    params = {
        "centers": q32(rng.normal(0, 1, (n, 3))),
        "rotations": q32(rng.normal(0, 1, (n, 4))),
        "log_scales": q32(rng.uniform(-6.0, -2.0, (n, 3))),
        "logit_opacities": q32(rng.uniform(-7.0, 2.0, n)),
        "colors_dc": q32(rng.uniform(-1, 1, (n, 3))),
        "colors_rest": q32(rng.uniform(-0.2, 0.2, (n, 3, 3))),
    }
    cfg = TrainConfig()
    extent = 1.7
    opt = Adam({k: v.copy() for k, v in params.items()}, {k: 1e-3 for k in params})
    for k in params:  # non-zero moments, to check their row surgery
        opt.m[k] = q32(rng.normal(0, 1e-3, params[k].shape))
        opt.v[k] = q32(rng.uniform(0, 1e-6, params[k].shape))
    state = DensifyState.zeros(n)
    state.grad_accum = q32(rng.uniform(0, 6e-4, n) * rng.integers(0, 2, n))
    state.denom = rng.integers(0, 3, n).astype(np.float64)
    inputs = {f"in_{k}": v for k, v in params.items()}
    inputs.update({f"in_m_{k}": opt.m[k].copy() for k in params})
    inputs.update({f"in_v_{k}": opt.v[k].copy() for k in params})
    inputs["in_accum"], inputs["in_denom"] = state.grad_accum.copy(), state.denom.copy()
    split_seed = 123
    stats = densify_and_prune(opt.params, opt, state, extent, cfg, np.random.default_rng(split_seed))
    out = {f"out_{k}": v for k, v in opt.params.items()}
    out.update({f"out_m_{k}": opt.m[k] for k in params})
    out.update({f"out_v_{k}": opt.v[k] for k in params})
    reset_opacity(opt)
    out["reset_logits"] = opt.params["logit_opacities"].copy()
    np.savez_compressed(os.path.join(HERE, "densify.npz"), extent=extent, split_seed=split_seed,
                        stats=np.array([stats["cloned"], stats["split"], stats["pruned"], stats["n_after"]]),
                        **inputs, **out)
    print("densify.npz", stats)


if __name__ == "__main__":
    main()
