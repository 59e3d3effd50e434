"""Training losses on the device -- drop-in for gsmesh/train/losses.py:
transmittance_mask (:79-91), texture_loss_active (:134-136) and
composite_loss (:139-174: L1 + D-SSIM + texture loss), one fused pass
(hgs_composite_loss) with all reductions on the device."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .splat import SCRATCH, _stream_ptr

MASK_VARIANTS = {"sigmoid": 0, "identity_t": 1, "constant_one": 2, "constant_zero": 3}


def gaussian_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    """losses.py:27-30 (same numpy expression)."""
    x = np.arange(size) - size // 2
    w = np.exp(-(x ** 2) / (2 * sigma ** 2))
    return w / w.sum()


_WIN = (ctypes.c_double * 11)(*gaussian_window().tolist())


def transmittance_mask(t, k: float = 20.0, variant: str = "sigmoid") -> torch.Tensor:
    """losses.py:79-91."""
    if variant not in MASK_VARIANTS:
        raise ValueError(f"unknown transmittance mask variant {variant!r}")
    tt = t if isinstance(t, torch.Tensor) else torch.as_tensor(np.asarray(t, dtype=np.float64))
    if not tt.is_cuda:
        tt = tt.cuda()
    tt = tt.float().contiguous()
    out = torch.empty_like(tt)
    _lib.call("hgs_transmittance_mask", _lib.ptr(tt), tt.numel(), float(k), MASK_VARIANTS[variant], _lib.ptr(out),
              _stream_ptr(tt.device))
    return out


def texture_loss_active(iteration: int, config, has_mesh: bool) -> bool:
    """losses.py:134-136."""
    return has_mesh and config.texture_weight > 0.0 and config.warmup_iters < iteration < config.densify_until_iter


@dataclass
class LossBreakdown:
    """losses.py:119-131; values live on the device until read."""

    scalars: torch.Tensor  # fp64[6]: l1, dssim, l_c, l_t, total, mean_T_on_mesh

    def _v(self, i):
        return float(self.scalars[i].item())

    l1 = property(lambda self: self._v(0))
    dssim = property(lambda self: self._v(1))
    l_c = property(lambda self: self._v(2))
    l_t = property(lambda self: self._v(3))
    total = property(lambda self: self._v(4))
    mean_t_on_mesh = property(lambda self: self._v(5))

    def to_dict(self) -> dict:
        v = self.scalars.tolist()
        return {"l1": v[0], "dssim": v[1], "l_c": v[2], "l_t": v[3], "total": v[4], "mean_T_on_mesh": v[5]}


def _dev_img(a, dev, dtype=torch.float32):
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
    return t.to(device=dev, dtype=dtype).contiguous()


def composite_loss(i_gt, i_h, i_m, covered, t, iteration: int, config, grad_scale: float = 1.0,
                   out: Optional[dict] = None):
    """losses.py:139-174 -> (LossBreakdown, grad_ih, grad_im | None, grad_t).

    ``covered`` may be a bool mask or a triangle-id map (>= 0 covered)."""
    dev = i_h.device if isinstance(i_h, torch.Tensor) and i_h.is_cuda else torch.device("cuda", torch.cuda.current_device())
    ih = _dev_img(i_h, dev)
    gt = _dev_img(i_gt, dev)
    h, w = ih.shape[:2]
    if tuple(gt.shape) != tuple(ih.shape) or ih.shape[2:] != (3,):
        raise ValueError(f"image shapes differ: {tuple(gt.shape)} vs {tuple(ih.shape)}")
    tt = _dev_img(t, dev)
    lam = config.dssim_weight
    if getattr(config, "zero_dssim_after_densify", False) and iteration >= config.densify_until_iter:
        lam = 0.0
    has_mesh = i_m is not None and covered is not None
    tri = None
    im = None
    if has_mesh:
        cv = covered if isinstance(covered, torch.Tensor) else torch.as_tensor(np.asarray(covered))
        cv = cv.to(dev)
        tri = (torch.where(cv, 0, -1) if cv.dtype == torch.bool else cv).to(torch.int32).contiguous()
        im = _dev_img(i_m, dev)
    active = texture_loss_active(iteration, config, has_mesh)
    if config.mask_variant not in MASK_VARIANTS:
        raise ValueError(f"unknown transmittance mask variant {config.mask_variant!r}")
    o = out or {}
    grad_ih = o.get("grad_ih") if o.get("grad_ih") is not None else torch.empty(h, w, 3, dtype=torch.float32, device=dev)
    grad_im = None
    if active:
        grad_im = o.get("grad_im") if o.get("grad_im") is not None else torch.empty(h, w, 3, dtype=torch.float32, device=dev)
    grad_t = o.get("grad_t") if o.get("grad_t") is not None else torch.empty(h, w, dtype=torch.float32, device=dev)
    scalars = o.get("scalars") if o.get("scalars") is not None else torch.empty(6, dtype=torch.float64, device=dev)
    nbytes = _lib.load().hgs_loss_scratch_bytes(h, w)
    scratch = SCRATCH.get("loss", nbytes, dev)
    _lib.call("hgs_composite_loss", _lib.ptr(gt), _lib.ptr(ih), _lib.ptr(im), _lib.ptr(tri), _lib.ptr(tt), h, w,
              float(lam), int(active), float(config.texture_weight), float(config.mask_sharpness),
              MASK_VARIANTS[config.mask_variant], _WIN, float(grad_scale), _lib.ptr(grad_ih), _lib.ptr(grad_im),
              _lib.ptr(grad_t), _lib.ptr(scalars), _lib.ptr(scratch), scratch.numel(), _stream_ptr(dev))
    return LossBreakdown(scalars), grad_ih, grad_im, grad_t


# ---- the reference's individual loss terms (losses.py:41-116), each a
# configuration of the fused composite kernel (same arithmetic) -------------

class _TermConfig:
    def __init__(self, lam=0.0, texture_weight=0.0, k=20.0, variant="sigmoid"):
        self.dssim_weight = lam
        self.zero_dssim_after_densify = False
        self.warmup_iters = 0
        self.densify_until_iter = 2  # iteration 1 is inside the texture window
        self.texture_weight = texture_weight
        self.mask_sharpness = k
        self.mask_variant = variant


def l1_loss(pred, target):
    """losses.py:41-44 -> (mean |pred - target|, sign(pred - target) / size)."""
    bd, g, _, _ = composite_loss(target, pred, None, None, _zeros_t(pred), 1, _TermConfig(lam=0.0))
    return bd.l1, g


def dssim(pred, target):
    """losses.py:73-76 -> ((1 - SSIM) / 2, its gradient w.r.t. pred)."""
    bd, g, _, _ = composite_loss(target, pred, None, None, _zeros_t(pred), 1, _TermConfig(lam=1.0))
    return bd.dssim, g


def ssim(pred, target):
    """losses.py:47-70 -> (mean SSIM, its gradient w.r.t. pred): 11-tap
    sigma 1.5 zero-padded separable window, fp64."""
    v, g = dssim(pred, target)
    return 1.0 - 2.0 * v, g * -2.0


def texture_loss(i_gt, i_m, covered, t, k: float = 20.0, variant: str = "sigmoid"):
    """losses.py:103-116 -> (L_t, grad w.r.t. I_m, grad w.r.t. T); uncovered
    pixels contribute nothing, the mean is over covered pixels."""
    bd, _, g_im, g_t = composite_loss(i_gt, i_gt, i_m, covered, t, 1,
                                      _TermConfig(texture_weight=1.0, k=k, variant=variant))
    return bd.l_t, g_im, g_t


def _zeros_t(img):
    shp = tuple(img.shape[:2])
    dev = img.device if isinstance(img, torch.Tensor) and img.is_cuda else torch.device("cuda", torch.cuda.current_device())
    return torch.zeros(shp, dtype=torch.float32, device=dev)
