"""Adaptive density control on the device -- drop-in for
gsmesh/train/densify.py (DensifyState :20-43, densify_and_prune :46-94,
reset_opacity :97-101) and the Adam row surgery it drives (adam.py:44-60).

Runs every ``densify_interval`` iterations, not per frame: the row surgery
is device gather / concatenate over the flat parameter and moment buffers
(PyTorch as plumbing); the per-Gaussian decisions reproduce the
reference's fp64 arithmetic.  The split samples come from the caller's
numpy ``Generator`` exactly as the reference draws them
(``rng.normal(0, 1, (2 n_split, 3))``), so a run seeded like the reference
splits into the same positions, and every data-parallel rank (same seed,
all-reduced statistics) performs the identical surgery.
"""

from __future__ import annotations

import math
from typing import Dict, Optional, Tuple

import numpy as np
import torch

from .adam import Adam
from .scene import GaussianSet


def inverse_sigmoid(x: torch.Tensor) -> torch.Tensor:
    """densify.py:15-16."""
    return torch.log(x / (1.0 - x))


def quaternions_to_rotations(q: torch.Tensor) -> torch.Tensor:
    """scene.py:126-141 in fp64: (N, 4) (w, x, y, z), normalised -> (N, 3, 3)."""
    q = q.double()
    qn = q / torch.linalg.norm(q, dim=-1, keepdim=True)
    w, x, y, z = qn.unbind(-1)
    r = torch.empty(q.shape[:-1] + (3, 3), dtype=torch.float64, device=q.device)
    r[..., 0, 0] = 1 - 2 * (y * y + z * z)
    r[..., 0, 1] = 2 * (x * y - w * z)
    r[..., 0, 2] = 2 * (x * z + w * y)
    r[..., 1, 0] = 2 * (x * y + w * z)
    r[..., 1, 1] = 1 - 2 * (x * x + z * z)
    r[..., 1, 2] = 2 * (y * z - w * x)
    r[..., 2, 0] = 2 * (x * z - w * y)
    r[..., 2, 1] = 2 * (y * z + w * x)
    r[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return r


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

    def update(self, visible_count: torch.Tensor, grad_norm_sum: torch.Tensor) -> None:
        n = self.grad_accum.numel()
        vis = visible_count[:n].double()
        seen = vis > 0
        self.grad_accum += torch.where(seen, grad_norm_sum[:n].double(), torch.zeros_like(vis))
        self.denom += vis

    def average(self) -> torch.Tensor:
        seen = self.denom > 0
        return torch.where(seen, self.grad_accum / torch.where(seen, self.denom, torch.ones_like(self.denom)),
                           torch.zeros_like(self.grad_accum))

    def reset(self, n: int) -> None:
        dev = self.grad_accum.device
        self.grad_accum = torch.zeros(n, dtype=torch.float64, device=dev)
        self.denom = torch.zeros(n, dtype=torch.float64, device=dev)


def _rows(gs: GaussianSet) -> Dict[str, torch.Tensor]:
    return {k: gs.group(k) for k in gs.layout}


def rebuild(gs: GaussianSet, rows: Dict[str, torch.Tensor]) -> GaussianSet:
    """A GaussianSet (same device, same groups) holding ``rows``."""
    return GaussianSet(rows["centers"], rows["rotations"], rows["log_scales"], rows["logit_opacities"],
                       rows["colors_dc"], rows.get("colors_rest"), device=gs.device)


def rebind(opt: Adam, gs: GaussianSet, m: Dict[str, torch.Tensor], v: Dict[str, torch.Tensor]) -> None:
    """Point the optimiser at the groups of ``gs`` (new row count) with
    moments ``m``, ``v`` (same shapes), keeping its step count and lrs."""
    opt.params = {k: gs.group(k) for k in opt.params}
    opt.m = {k: m[k].contiguous() for k in opt.params}
    opt.v = {k: v[k].contiguous() for k in opt.params}


def densify_and_prune(gs: GaussianSet, opt: Adam, state: DensifyState, extent: float, config,
                      rng: np.random.Generator) -> Tuple[GaussianSet, dict]:
    """One density-control step (densify.py:46-94): clone small hot
    Gaussians, split large hot ones (2 samples each), then drop the split
    originals and every Gaussian whose opacity is below the prune threshold.
    Returns the new GaussianSet (the optimiser is rebound to it)."""
    dev = gs.device
    n0 = len(gs)
    avg = state.average()
    scales = torch.exp(gs.log_scales.double()).max(dim=1).values
    hot = avg > config.densify_grad_threshold
    small = scales <= config.percent_dense * extent
    clone_mask = hot & small
    split_mask = hot & ~small
    n_clone, n_split = int(clone_mask.sum()), int(split_mask.sum())
    stats = {"cloned": n_clone, "split": n_split}

    rows = _rows(gs)
    names = list(rows)
    new_p = {k: [rows[k]] for k in names}
    new_m = {k: [opt.m[k]] if k in opt.m else [] for k in names}
    new_v = {k: [opt.v[k]] if k in opt.v else [] for k in names}

    def append(block: Dict[str, torch.Tensor]):
        for k in names:
            new_p[k].append(block[k])
            if k in opt.m:
                new_m[k].append(torch.zeros_like(block[k]))
                new_v[k].append(torch.zeros_like(block[k]))

    if n_clone:
        append({k: rows[k][clone_mask].clone() for k in names})
    if n_split:
        reps = 2
        stds = torch.repeat_interleave(torch.exp(rows["log_scales"][split_mask].double()), reps, dim=0)
        samples = torch.as_tensor(rng.normal(0.0, 1.0, tuple(stds.shape)), dtype=torch.float64, device=dev) * stds
        rots = torch.repeat_interleave(quaternions_to_rotations(rows["rotations"][split_mask]), reps, dim=0)
        block = {k: torch.repeat_interleave(rows[k][split_mask], reps, dim=0) for k in names}
        block["centers"] = (torch.einsum("nij,nj->ni", rots, samples) + block["centers"].double()).float()
        block["log_scales"] = (block["log_scales"].double() - math.log(1.6)).float()
        append(block)

    cat_p = {k: torch.cat(new_p[k]) for k in names}
    n_now = len(cat_p["centers"])
    keep = torch.ones(n_now, dtype=torch.bool, device=dev)
    keep[:n0][split_mask] = False
    alpha = torch.sigmoid(cat_p["logit_opacities"].double())
    low = alpha < config.opacity_prune_threshold
    stats["pruned"] = int((low & keep).sum())
    keep &= ~low
    out_p = {k: cat_p[k][keep] for k in names}
    out_m = {k: torch.cat(new_m[k])[keep] for k in names if k in opt.m}
    out_v = {k: torch.cat(new_v[k])[keep] for k in names if k in opt.v}
    new_gs = rebuild(gs, out_p)
    rebind(opt, new_gs, out_m, out_v)
    state.reset(len(new_gs))
    stats["n_after"] = len(new_gs)
    return new_gs, stats


def reset_opacity(gs: GaussianSet, opt: Optional[Adam] = None, ceiling: float = 0.01) -> None:
    """densify.py:97-101: activated opacities clamped to <= ceiling (in
    place), their Adam moments cleared."""
    lg = gs.logit_opacities
    alpha = torch.sigmoid(lg.double())
    lg.copy_(inverse_sigmoid(torch.clamp(alpha, max=ceiling)).float())
    if opt is not None and "logit_opacities" in opt.m:
        opt.m["logit_opacities"].zero_()
        opt.v["logit_opacities"].zero_()
