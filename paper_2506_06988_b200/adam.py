"""Adam with per-group learning rates over device tensors -- drop-in for
gsmesh/train/adam.py (Adam :16-42, exponential_lr :63-73).  One fused
launch updates every group (hgs_adam_step); quaternion renormalisation
(loop.py:139-140) and texture clamping (loop.py:144-145) are fused as group
modes."""

from __future__ import annotations

import math
from typing import Dict, Iterable, Optional

import torch

from . import _lib
from .splat import _stream_ptr

MODE_PLAIN, MODE_RENORM4, MODE_CLAMP01 = 0, 1, 2


class Adam:
    def __init__(self, params: Dict[str, torch.Tensor], lrs: Dict[str, float], beta1: float = 0.9,
                 beta2: float = 0.999, eps: float = 1e-15):
        self.params = params
        self.lrs = dict(lrs)
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.step_count = 0
        self.m = {k: torch.zeros_like(v) for k, v in params.items()}
        self.v = {k: torch.zeros_like(v) for k, v in params.items()}

    def step(self, grads: Dict[str, Optional[torch.Tensor]], renorm: Iterable[str] = (), clamp: Iterable[str] = (),
             grad_scale: float = 1.0) -> None:
        """adam.py:28-42 (+ fused renorm / clamp groups)."""
        self.step_count += 1
        renorm, clamp = set(renorm), set(clamp)
        groups = []
        for name, g in grads.items():
            if g is None:
                continue
            p = self.params[name]
            if tuple(g.shape) != tuple(p.shape):
                raise ValueError(f"gradient shape {tuple(g.shape)} != parameter {tuple(p.shape)} for {name}")
            for t in (p, g, self.m[name], self.v[name]):
                if t.dtype != torch.float32 or not t.is_contiguous() or not t.is_cuda:
                    raise ValueError(f"{name}: Adam state must be contiguous fp32 CUDA tensors")
            gr = _lib.HGSAdamGroup()
            gr.param, gr.m, gr.v, gr.grad = p.data_ptr(), self.m[name].data_ptr(), self.v[name].data_ptr(), g.data_ptr()
            gr.n = p.numel()
            gr.lr = float(self.lrs[name])
            gr.mode = MODE_RENORM4 if name in renorm else (MODE_CLAMP01 if name in clamp else MODE_PLAIN)
            groups.append(gr)
        if not groups:
            return
        dev = next(iter(self.params.values())).device
        for i in range(0, len(groups), _lib.HGS_MAX_ADAM_GROUPS):
            chunk = groups[i:i + _lib.HGS_MAX_ADAM_GROUPS]
            arr = (_lib.HGSAdamGroup * len(chunk))(*chunk)
            _lib.call("hgs_adam_step", arr, len(chunk), self.step_count, self.beta1, self.beta2, self.eps,
                      float(grad_scale), _stream_ptr(dev))


def exponential_lr(initial: float, final: float, max_steps: int):
    """Log-linear interpolation from initial to final (adam.py:63-73)."""
    if initial <= 0 or final <= 0:
        raise ValueError("learning rates must be positive")
    ln_i, ln_f = math.log(initial), math.log(final)

    def lr_at(step: int) -> float:
        t = min(max(step / max_steps, 0.0), 1.0)
        return math.exp(ln_i * (1.0 - t) + ln_f * t)

    return lr_at
