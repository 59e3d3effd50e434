"""rasterize_backward (gsmesh/splat/render.py:124-182) on the device.

blend backward (K5, hgs_blend_backward) accumulates per-Gaussian screen
gradients (N x 9 fp64); the chain rule (K6, hgs_project_backward) maps them
to parameter gradients laid out exactly like GaussianSet.params, so a
training step can accumulate many views into one flat buffer that Adam and
the NCCL all-reduce consume directly.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np
import torch

from . import _lib
from .scene import GaussianSet, camera_tensor
from .splat import GaussianGrads, RenderCtx, _c_f64_3, _stream_ptr


class GradBuffer:
    """Flat fp32 gradient buffer with the parameter layout of a GaussianSet."""

    def __init__(self, gs: GaussianSet, flat: Optional[torch.Tensor] = None,
                 densify_norm: Optional[torch.Tensor] = None, visible_count: Optional[torch.Tensor] = None):
        self.gs = gs
        self.flat = flat if flat is not None else torch.zeros_like(gs.params)
        assert self.flat.numel() == gs.params.numel() and self.flat.dtype == torch.float32
        self.densify_norm = densify_norm if densify_norm is not None else torch.zeros(
            max(len(gs), 1), dtype=torch.float32, device=gs.device)
        self.visible = torch.zeros(max(len(gs), 1), dtype=torch.uint8, device=gs.device)
        self.visible_count = visible_count  # optional: views in which each row was visible

    def group(self, name: str) -> Optional[torch.Tensor]:
        if name not in self.gs.layout:
            return None
        off, size = self.gs.layout[name]
        v = self.flat[off:off + size]
        n = len(self.gs)
        if name == "logit_opacities":
            return v
        if name == "colors_rest":
            return v.view(n, 3, 3)
        return v.view(n, -1)

    def zero_(self):
        self.flat.zero_()
        self.densify_norm.zero_()
        self.visible.zero_()
        if self.visible_count is not None:
            self.visible_count.zero_()

    def struct(self) -> _lib.HGSGaussianGrads:
        s = _lib.HGSGaussianGrads()
        base = self.flat.data_ptr()
        elt = self.flat.element_size()
        for name, field in (("centers", "centers"), ("rotations", "rotations"), ("log_scales", "log_scales"),
                            ("logit_opacities", "logits"), ("colors_dc", "colors_dc"), ("colors_rest", "colors_rest")):
            if name in self.gs.layout:
                setattr(s, field, base + self.gs.layout[name][0] * elt)
        s.densify_norm = self.densify_norm.data_ptr()
        s.visible = self.visible.data_ptr()
        s.visible_count = self.visible_count.data_ptr() if self.visible_count is not None else None
        return s


def screen_backward(ctx: RenderCtx, grad_color: torch.Tensor, grad_t: Optional[torch.Tensor],
                    screen: torch.Tensor, mesh_grad: Optional[torch.Tensor] = None, accumulate_mesh: bool = False):
    """K5: add the per-Gaussian screen gradients of one view into ``screen``."""
    cam = ctx.camera
    w, h = int(cam.width), int(cam.height)
    dev = ctx.gaussians.device
    ml = ctx.mesh.struct() if ctx.mesh is not None else _lib.HGSMeshLayer()
    _lib.call("hgs_blend_backward", ctypes.byref(ctx.proj.struct()), ctypes.byref(ctx.tiles.struct()), w, h,
              ctypes.byref(ml), _c_f64_3(np.asarray(ctx.background, dtype=np.float64)), _lib.ptr(ctx.final_t),
              _lib.ptr(ctx.last_consumed), _lib.ptr(grad_color), _lib.ptr(grad_t), _lib.ptr(screen),
              _lib.ptr(mesh_grad), int(accumulate_mesh), _stream_ptr(dev))


def chain_backward(ctx: RenderCtx, screen: torch.Tensor, out: GradBuffer, scale: float = 1.0, accumulate: bool = False):
    """K6: parameter gradients (+ densify norm, visibility) from screen grads."""
    dev = ctx.gaussians.device
    cam_dev = ctx.cam_dev if ctx.cam_dev is not None else camera_tensor(ctx.camera, dev)
    ps = ctx.proj.struct()
    _lib.call("hgs_project_backward", _lib.ptr(cam_dev), ctypes.byref(ctx.gaussians.struct()), ctypes.byref(ps),
              _lib.ptr(screen), ctypes.byref(out.struct()), float(scale), int(accumulate), _stream_ptr(dev))


def _as_dev(a, dev, shape, name) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, dtype=np.float64))
    if tuple(t.shape) != shape:
        raise ValueError(f"{name} shape {tuple(t.shape)} != {shape}")
    return t.to(device=dev, dtype=torch.float32).contiguous()


def rasterize_backward(ctx: RenderCtx, grad_color, grad_transmittance=None) -> GaussianGrads:
    """Analytic gradients of sum(grad_color * pixel) (+ sum(grad_T * T))
    for all parameters (splat/render.py:124-182)."""
    gs = ctx.gaussians
    dev = gs.device
    h, w = int(ctx.camera.height), int(ctx.camera.width)
    gc = _as_dev(grad_color, dev, (h, w, 3), "grad_color")
    gt = None if grad_transmittance is None else _as_dev(grad_transmittance, dev, (h, w), "grad_transmittance")
    n = len(gs)
    screen = torch.zeros(max(n, 1) * 9, dtype=torch.float64, device=dev)
    mesh_grad = torch.empty(h, w, 3, dtype=torch.float32, device=dev) if ctx.mesh is not None else None
    if n:
        screen_backward(ctx, gc, gt, screen, mesh_grad)
    elif mesh_grad is not None:
        mesh_grad.copy_(gc * (ctx.final_t * (ctx.mesh.triangle_id >= 0)).float()[..., None])
    out = GradBuffer(gs)
    if n:
        chain_backward(ctx, screen, out)
    return GaussianGrads(centers=out.group("centers"), rotations=out.group("rotations"),
                         log_scales=out.group("log_scales"), logit_opacities=out.group("logit_opacities"),
                         colors_dc=out.group("colors_dc"), colors_rest=out.group("colors_rest"),
                         densify_norm=out.densify_norm[:n], visible=out.visible[:n].bool(), mesh_color=mesh_grad)
