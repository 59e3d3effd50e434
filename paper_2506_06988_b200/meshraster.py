"""Textured-mesh rasterization on the device -- the drop-in for
gsmesh.meshraster (meshraster.py:119-203):

    rasterize_fragments(mesh, cam) -> MeshFragmentBuffer   meshraster.py:119-136
    sample_texture(texture, uv, valid)                     meshraster.py:158-166
    texture_backward(fragments, grad_image, texture_shape) meshraster.py:169-184
    raster_mesh(mesh, cam)                                 meshraster.py:187-193
    mesh_layer(mesh, cam, fragments=None) -> MeshLayer     meshraster.py:196-203

Triangle ids and coverage are bit-identical to the reference z-buffer;
depth, barycentrics and uv are computed with the reference's fp64
arithmetic.  The texture is fp32 (Ht, Wt, 3).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib
from .scene import Camera, TexturedMesh, camera_tensor, default_device
from .splat import SCRATCH, MeshLayer, _stream_ptr


@dataclass
class MeshFragmentBuffer:
    """Per-pixel rasterization state for one camera (meshraster.py:25-42):
    triangle_id (H,W) int32 (-1 uncovered), bary (H,W,3) fp64, depth (H,W)
    fp64 (+inf uncovered), uv (H,W,2) fp64."""

    triangle_id: torch.Tensor
    bary: Optional[torch.Tensor]
    depth: torch.Tensor
    uv: torch.Tensor

    @property
    def valid(self) -> torch.Tensor:
        return self.triangle_id >= 0


def rasterize_fragments(mesh, cam, with_bary: bool = True) -> MeshFragmentBuffer:
    """Z-buffered rasterization of the mesh geometry (meshraster.py:119-136)."""
    mesh = TexturedMesh.from_any(mesh)
    cam = Camera.from_any(cam)
    dev = mesh.device
    h, w = int(cam.height), int(cam.width)
    tri = torch.empty(h, w, dtype=torch.int32, device=dev)
    depth = torch.empty(h, w, dtype=torch.float64, device=dev)
    bary = torch.empty(h, w, 3, dtype=torch.float64, device=dev) if with_bary else None
    uv = torch.empty(h, w, 2, dtype=torch.float64, device=dev)
    out = _lib.HGSFragments()
    out.triangle_id, out.depth, out.bary, out.uv = _lib.ptr(tri), _lib.ptr(depth), _lib.ptr(bary), _lib.ptr(uv)
    cam_dev = camera_tensor(cam, dev)
    ms = mesh.struct()
    nbytes = _lib.load().hgs_raster_scratch_bytes(ms.n_vertices, ms.n_faces, w, h)
    scratch = SCRATCH.get("raster", nbytes, dev)
    _lib.call("hgs_rasterize_fragments", _lib.ptr(cam_dev), w, h, ctypes.byref(ms), ctypes.byref(out),
              _lib.ptr(scratch), scratch.numel(), _stream_ptr(dev))
    return MeshFragmentBuffer(tri, bary, depth, uv)


def _as_dev(a, dev, dtype):
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.asarray(a), device=dev).to(dtype).contiguous()


def sample_texture(texture, uv, valid) -> torch.Tensor:
    """Bilinear texture lookup; invalid pixels come back black (meshraster.py:158-166).

    ``valid`` may be a bool mask or the triangle-id map (>= 0 is valid)."""
    dev = texture.device if isinstance(texture, torch.Tensor) and texture.is_cuda else default_device()
    tex = _as_dev(texture, dev, torch.float32)
    if tex.ndim != 3 or tex.shape[2] != 3:
        raise ValueError("texture must be (H, W, 3)")
    uvt = _as_dev(uv, dev, torch.float64)
    shp = tuple(uvt.shape[:-1])
    v = _as_dev(valid, dev, torch.int32) if not (isinstance(valid, torch.Tensor) and valid.dtype == torch.int32) else valid
    if v.dtype != torch.int32:
        v = v.to(torch.int32)
    if valid is not None and (isinstance(valid, np.ndarray) and valid.dtype == bool or
                              isinstance(valid, torch.Tensor) and valid.dtype == torch.bool):
        v = torch.where(_as_dev(valid, dev, torch.bool), 0, -1).to(torch.int32)
    if tuple(v.shape) != shp:
        raise ValueError(f"valid shape {tuple(v.shape)} does not match uv {shp}")
    out = torch.empty(shp + (3,), dtype=torch.float32, device=dev)
    npix = int(np.prod(shp)) if shp else 1
    _lib.call("hgs_sample_texture", _lib.ptr(tex), tex.shape[0], tex.shape[1], _lib.ptr(uvt), _lib.ptr(v.contiguous()),
              npix, _lib.ptr(out), _stream_ptr(dev))
    return out


def texture_backward(fragments: MeshFragmentBuffer, grad_image, texture_shape: Tuple[int, int],
                     out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Adjoint of sample_texture (meshraster.py:169-184); adds into ``out``
    when given (the training step accumulates over views)."""
    th, tw = int(texture_shape[0]), int(texture_shape[1])
    dev = fragments.triangle_id.device
    g = _as_dev(grad_image, dev, torch.float32)
    if tuple(g.shape[:2]) != tuple(fragments.triangle_id.shape):
        raise ValueError(f"grad image shape {tuple(g.shape)} does not match fragments {tuple(fragments.triangle_id.shape)}")
    if out is None:
        out = torch.zeros(th, tw, 3, dtype=torch.float32, device=dev)
    npix = fragments.triangle_id.numel()
    _lib.call("hgs_texture_backward", _lib.ptr(fragments.uv), _lib.ptr(fragments.triangle_id), _lib.ptr(g), npix, th, tw,
              _lib.ptr(out), _stream_ptr(dev))
    return out


def raster_mesh(mesh, cam):
    """Full mesh render -> (color, depth, triangle_id, fragments) (meshraster.py:187-193)."""
    mesh = TexturedMesh.from_any(mesh)
    if mesh.uvs is None or mesh.texture is None:
        raise ValueError("raster_mesh needs a mesh with UVs and texture")
    frags = rasterize_fragments(mesh, cam)
    color = sample_texture(mesh.texture, frags.uv, frags.triangle_id)
    return color, frags.depth, frags.triangle_id, frags


def mesh_layer(mesh, cam, fragments: Optional[MeshFragmentBuffer] = None) -> MeshLayer:
    """MeshLayer for hybrid compositing; cached fragments skip re-rasterization
    (meshraster.py:196-203)."""
    mesh = TexturedMesh.from_any(mesh)
    if fragments is None:
        fragments = rasterize_fragments(mesh, cam, with_bary=False)
    color = sample_texture(mesh.texture, fragments.uv, fragments.triangle_id)
    return MeshLayer(color=color, depth=fragments.depth, triangle_id=fragments.triangle_id)


def init_texture(mesh, images, cameras, iters: int = 500, mode: str = "optimized", lr: float = 0.05,
                 warn=print) -> TexturedMesh:
    """Texture initialisation (meshraster.py:206-245): constant 0.5, or
    ``iters`` Adam steps (lr, texture clamped to [0, 1] after each) on the
    coverage-normalised masked MSE between the mesh render and the target
    images, views averaged.  Texels no view covers keep 0.5.  Everything
    runs on the device: fragments once per camera, then per step the
    bilinear fetch, masked difference, bilinear adjoint (accumulated over
    views) and the fused Adam + clamp."""
    from .adam import Adam
    mesh = TexturedMesh.from_any(mesh)
    if mesh.uvs is None:
        raise ValueError("init_texture needs a mesh with UVs")
    if mode not in ("constant", "optimized"):
        raise ValueError(f"unknown texture init mode {mode!r}")
    dev = mesh.device
    tex0 = mesh.texture if mesh.texture is not None else torch.zeros(1, 1, 3, device=dev)
    out = TexturedMesh(mesh.vertices.clone(), mesh.triangles.clone(), mesh.uvs.clone(),
                       torch.full_like(tex0, 0.5, dtype=torch.float32), device=dev)
    if mode == "constant" or iters <= 0:
        return out
    if len(images) != len(cameras):
        raise ValueError("images/cameras count mismatch")
    frags = [rasterize_fragments(out, cam, with_bary=False) for cam in cameras]
    covered = [f.triangle_id >= 0 for f in frags]
    n_cov = [int(c.sum().item()) for c in covered]
    if sum(n_cov) == 0:
        warn("init_texture: no camera sees the mesh; falling back to constant 0.5")
        return out
    targets = [_as_dev(im, dev, torch.float32) for im in images]
    th, tw = int(out.texture.shape[0]), int(out.texture.shape[1])
    opt = Adam({"texture": out.texture}, {"texture": lr})
    grad = torch.zeros_like(out.texture)
    for _ in range(iters):
        grad.zero_()
        for img, fr, cov, nc in zip(targets, frags, covered, n_cov):
            if nc == 0:
                continue
            pred = sample_texture(out.texture, fr.uv, fr.triangle_id)
            diff = torch.where(cov[..., None], pred - img, torch.zeros_like(pred))
            texture_backward(fr, diff * (2.0 / nc), (th, tw), out=grad)
        opt.step({"texture": grad}, clamp=("texture",), grad_scale=1.0 / len(cameras))
    return out
