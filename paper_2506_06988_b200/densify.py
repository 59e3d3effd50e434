"""Adaptive density control on the device -- drop-in for
gsmesh/train/densify.py (DensifyState :20-43, densify_and_prune :46-94,
reset_opacity :97-101) and the Adam row surgery it drives (adam.py:44-60).

Every step runs in libhgs.so (csrc/densify.cu): the per-Gaussian decisions
reproduce the reference's fp64 arithmetic, the row surgery is a stream
compaction writing the new flat parameter buffer and both Adam moments in
one pass (hgs_densify_plan / hgs_densify_apply), the statistic update and the
opacity reset are one kernel each.  The split samples come from the caller's
numpy ``Generator`` exactly as the reference draws them
(``rng.normal(0, 1, (2 n_split, 3))``, uploaded once), so a run seeded like
the reference splits into the same positions, and every data-parallel rank
(same seed, all-reduced statistics) performs the identical surgery.
"""

from __future__ import annotations

import ctypes
from typing import Dict, Tuple

import numpy as np
import torch

from . import _lib
from .adam import Adam
from .scene import GROUPS, GaussianSet


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


class DensifyState:
    """Per-Gaussian screen-gradient accumulators (densify.py:20-43), fp64 on
    the device.  ``update`` takes the batch sums of one step: the summed
    per-view gradient norms and the number of views each row was visible in
    (for a one-view step exactly the reference's masked update)."""

    def __init__(self, n: int, device):
        self.grad_accum = torch.zeros(n, dtype=torch.float64, device=device)
        self.denom = torch.zeros(n, dtype=torch.float64, device=device)

    @staticmethod
    def zeros(n: int, device) -> "DensifyState":
        return DensifyState(n, device)

    def update(self, visible_count: torch.Tensor, grad_norm_sum: torch.Tensor, scale: float = 1.0) -> None:
        """Where a row was visible: grad_accum += scale * grad_norm_sum,
        denom += visible_count (densify.py:31-33 for a batch of views)."""
        n = self.grad_accum.numel()
        vc = visible_count[:n].float().contiguous()
        ns = grad_norm_sum[:n].float().contiguous()
        _lib.call("hgs_densify_accumulate", _lib.ptr(vc), _lib.ptr(ns), float(scale), n, _lib.ptr(self.grad_accum),
                  _lib.ptr(self.denom), _stream(self.grad_accum.device))

    def average(self) -> torch.Tensor:
        seen = self.denom > 0
        return torch.where(seen, self.grad_accum / torch.where(seen, self.denom, torch.ones_like(self.denom)),
                           torch.zeros_like(self.grad_accum))

    def reset(self, n: int) -> None:
        dev = self.grad_accum.device
        self.grad_accum = torch.zeros(n, dtype=torch.float64, device=dev)
        self.denom = torch.zeros(n, dtype=torch.float64, device=dev)


def _moments(opt: Adam, which: Dict[str, torch.Tensor], gs: GaussianSet) -> _lib.HGSGaussians:
    s = _lib.HGSGaussians()
    s.centers, s.rotations = _lib.ptr(which["centers"]), _lib.ptr(which["rotations"])
    s.log_scales, s.logits = _lib.ptr(which["log_scales"]), _lib.ptr(which["logit_opacities"])
    s.colors_dc = _lib.ptr(which["colors_dc"])
    s.colors_rest = _lib.ptr(which["colors_rest"]) if gs.sh_degree else None
    s.n = len(gs)
    return s


def rebind(opt: Adam, gs: GaussianSet, m: Dict[str, torch.Tensor], v: Dict[str, torch.Tensor]) -> None:
    """Point the optimiser at the groups of ``gs`` (new row count) with
    moments ``m``, ``v`` (same shapes), keeping its step count and lrs."""
    opt.params = {k: gs.group(k) for k in opt.params}
    opt.m = {k: m[k] for k in opt.params}
    opt.v = {k: v[k] for k in opt.params}


def densify_and_prune(gs: GaussianSet, opt: Adam, state: DensifyState, extent: float, config,
                      rng: np.random.Generator) -> Tuple[GaussianSet, dict]:
    """One density-control step (densify.py:46-94): clone small hot
    Gaussians, split large hot ones (2 samples each), then drop the split
    originals and every Gaussian whose opacity is below the prune threshold.
    Returns the new GaussianSet (the optimiser is rebound to it)."""
    groups = [g for g in GROUPS if g in gs.layout]
    if set(opt.params) != set(groups):
        raise ValueError(f"optimiser groups {sorted(opt.params)} != Gaussian groups {groups}")
    dev = gs.device
    n0 = len(gs)
    nbytes = _lib.load().hgs_densify_scratch_bytes(n0)
    scratch = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
    counts = (ctypes.c_int64 * 7)()
    _lib.call("hgs_densify_plan", ctypes.byref(gs.struct()), _lib.ptr(state.grad_accum), _lib.ptr(state.denom),
              float(config.densify_grad_threshold), float(config.percent_dense * extent),
              float(config.opacity_prune_threshold), _lib.ptr(scratch), scratch.numel(), counts, _stream(dev))
    n_clone, n_split, n_pruned, n_after = (int(counts[i]) for i in range(4))
    normals = None
    if n_split:  # the reference draws only when some row splits (densify.py:64-66)
        normals = torch.as_tensor(rng.normal(0.0, 1.0, (2 * n_split, 3)), dtype=torch.float64).to(dev)
    new_gs = GaussianSet.allocate(n_after, gs.sh_degree, dev)
    new_m = GaussianSet.allocate(n_after, gs.sh_degree, dev)
    new_v = GaussianSet.allocate(n_after, gs.sh_degree, dev)
    state.grad_accum = torch.empty(n_after, dtype=torch.float64, device=dev)  # zeroed by the kernel (state.reset)
    state.denom = torch.empty(n_after, dtype=torch.float64, device=dev)
    _lib.call("hgs_densify_apply", ctypes.byref(gs.struct()), ctypes.byref(_moments(opt, opt.m, gs)),
              ctypes.byref(_moments(opt, opt.v, gs)), _lib.ptr(normals), _lib.ptr(scratch),
              ctypes.byref(new_gs.buf()), ctypes.byref(new_m.buf()), ctypes.byref(new_v.buf()),
              _lib.ptr(state.grad_accum), _lib.ptr(state.denom), _stream(dev))
    rebind(opt, new_gs, {k: new_m.group(k) for k in groups}, {k: new_v.group(k) for k in groups})
    stats = {"cloned": n_clone, "split": n_split, "pruned": n_pruned, "n_after": n_after}
    return new_gs, stats


def reset_opacity(gs: GaussianSet, opt: Adam = None, ceiling: float = 0.01) -> None:
    """densify.py:97-101: activated opacities clamped to <= ceiling (in
    place), their Adam moments cleared."""
    m = opt.m.get("logit_opacities") if opt is not None else None
    v = opt.v.get("logit_opacities") if opt is not None else None
    _lib.call("hgs_reset_opacity", _lib.ptr(gs.logit_opacities), _lib.ptr(m), _lib.ptr(v), len(gs), float(ceiling),
              _stream(gs.device))
