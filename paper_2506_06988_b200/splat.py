"""Differentiable tile-based Gaussian splatting over an optional opaque mesh
layer -- the drop-in for gsmesh.splat (splat/__init__.py:3-31).

Operator API (same names, argument meaning and error behaviour as the
reference):
    project(gs, cam)                                   splat/project.py:70-140
    build_tiles(proj, width, height, tile_px=16)       splat/tiles.py:35-69
    rasterize_forward(proj, tiles, w, h, background, mesh=None, bg_color)
                                                       splat/render.py:74-109
    render(gs, cam, background, mesh, tile_px)         splat/render.py:112-121
    rasterize_backward(ctx, grad_color, grad_transmittance=None)
                                                       splat/render.py:124-182
Inputs may be this package's device types or any object with the
reference's attribute names (numpy float64 arrays are uploaded as fp32).
Outputs are CUDA tensors.  Every compute step runs in libhgs.so.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Union

import numpy as np
import torch

from . import _lib
from .scene import (Camera, GaussianSet, RenderOutputs, camera_tensor, default_device)

# splat/project.py:19-27, tiles.py:16
COV_FLOOR = 0.3
ALPHA_CLAMP = 0.99
SIGMA_SKIP = 1.0 / 255.0
SUPPORT_MAHAL2 = 9.0
EARLY_STOP_T = 1e-4
FRUSTUM_LIMIT = 1.3
SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
TILE_PX = 16
REC_BYTES = 80
MASK_VARIANTS = {"sigmoid": 0, "identity_t": 1, "constant_one": 2, "constant_zero": 3}


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


@dataclass
class MeshLayer:
    """Opaque, depth-fixed background from the mesh rasterizer (MeshLayer,
    splat/render.py:26-41).  color (H,W,3) fp32, depth (H,W) fp64 (+inf where
    uncovered), triangle_id (H,W) int32 (-1 where uncovered)."""

    color: torch.Tensor
    depth: torch.Tensor
    triangle_id: torch.Tensor

    def __post_init__(self):
        dev = None
        for v in (self.color, self.depth, self.triangle_id):
            if isinstance(v, torch.Tensor) and v.is_cuda:
                dev = v.device
        dev = dev or default_device()
        self.color = torch.as_tensor(np.asarray(self.color) if not isinstance(self.color, torch.Tensor) else self.color,
                                     device=dev).float().contiguous()
        self.depth = torch.as_tensor(np.asarray(self.depth) if not isinstance(self.depth, torch.Tensor) else self.depth,
                                     device=dev).double().contiguous()
        tid = self.triangle_id
        self.triangle_id = torch.as_tensor(np.asarray(tid) if not isinstance(tid, torch.Tensor) else tid,
                                           device=dev).to(torch.int32).contiguous()

    @property
    def valid(self) -> torch.Tensor:
        return self.triangle_id >= 0

    def struct(self) -> _lib.HGSMeshLayer:
        s = _lib.HGSMeshLayer()
        s.color, s.depth, s.triangle_id = _lib.ptr(self.color), _lib.ptr(self.depth), _lib.ptr(self.triangle_id)
        return s


class ProjectedGaussians:
    """Screen-space Gaussians that survived culling (ProjectedGaussians,
    splat/project.py:30-53): compacted fp64 views (kept, mean2d, depth,
    cov2d, conic, alpha, color, radius, t_cam, color_pre, view_dir,
    view_dist) over the device state indexed by original row (rec, count,
    rect) that build_tiles / rasterize_forward consume."""

    def __init__(self, n, rec, count, rect, extras=None, width=None, height=None, tile_px=TILE_PX, cull=None,
                 sort_keys=None, tile_diff=None):
        self.sort_keys, self.tile_diff = sort_keys, tile_diff
        # count may be longer than n (buffers are allocated with >= 1 row so
        # their device pointers are never NULL); the API view is count[:n]
        self._count_buf = count
        self.n, self.rec, self.count, self.rect, self.cull = n, rec, count[:n], rect, cull
        self._extras = extras
        self._compact = None
        self.width, self.height, self.tile_px = width, height, tile_px

    def struct(self) -> _lib.HGSProjected:
        s = _lib.HGSProjected()
        s.rec, s.count, s.rect = _lib.ptr(self.rec), _lib.ptr(self._count_buf), _lib.ptr(self.rect)
        s.cull = _lib.ptr(self.cull)
        s.sort_keys, s.tile_diff = _lib.ptr(self.sort_keys), _lib.ptr(self.tile_diff)
        return s

    def _fields(self):
        if self._compact is None:
            alive = self.count > 0
            kept = torch.nonzero(alive).reshape(-1)
            rec = self.rec.view(torch.float64)[:self.n * 10].view(self.n, 10)[kept]
            conic = rec[:, 2:5].clone()
            conic[:, 1] *= 0.5  # the record stores 2 * conic_xy (exact)
            f = {"kept": kept, "mean2d": rec[:, 0:2].contiguous(), "conic": conic,
                 "alpha": rec[:, 6].contiguous(), "depth": rec[:, 5].contiguous(), "color": rec[:, 7:10].contiguous()}
            ex = self._extras or {}
            for k in ("cov2d", "radius", "t_cam", "color_pre", "view_dir", "view_dist"):
                f[k] = ex[k][kept] if ex.get(k) is not None else None
            self._compact = f
        return self._compact

    def __len__(self):
        return int(self._fields()["kept"].numel())

    def __getattr__(self, name):
        if name in ("kept", "mean2d", "depth", "cov2d", "conic", "alpha", "color", "radius", "t_cam", "color_pre",
                    "view_dir", "view_dist"):
            return self._fields()[name]
        raise AttributeError(name)


class TileBins:
    """CSR tile layout (TileBins, splat/tiles.py:19-32).  ``entries`` are
    row indices into the ProjectedGaussians arrays (as in the reference);
    ``entries_orig`` are the original Gaussian rows the kernels consume."""

    def __init__(self, tile_starts, entries_orig, tiles_x, tiles_y, tile_px, proj: Optional[ProjectedGaussians] = None,
                 k: Optional[int] = None, counters: Optional[torch.Tensor] = None, capacity: Optional[int] = None,
                 ready: Optional[torch.Tensor] = None):
        self.tile_starts = tile_starts
        # the binning -> blend ready queue of these bins (hgs_tiles.ready)
        self.ready = ready
        # the binning counters (M, K, overflow flag, ...) travel with the bins:
        # every consumer kernel returns early on an overflowed buffer instead
        # of reading entries past the capacity
        self.counters = counters
        self.capacity = capacity
        self.entries_orig = entries_orig
        self.tiles_x, self.tiles_y, self.tile_px = tiles_x, tiles_y, tile_px
        self._proj = proj
        self._k = k
        self._entries = None

    @property
    def k(self) -> int:
        if self._k is None:
            self._k = int(self.tile_starts[-1].item())
        return self._k

    @property
    def entries(self) -> torch.Tensor:
        if self._entries is None:
            k = self.k
            orig = self.entries_orig[:k].long()
            if self._proj is not None:
                alive = (self._proj.count > 0).to(torch.int64)
                row = torch.cumsum(alive, 0) - 1
                self._entries = row[orig].to(torch.int32)
            else:
                self._entries = orig.to(torch.int32)
        return self._entries

    def tile_list(self, tx: int, ty: int) -> torch.Tensor:
        t = ty * self.tiles_x + tx
        s, e = int(self.tile_starts[t]), int(self.tile_starts[t + 1])
        return self.entries[s:e]

    def struct(self, counters=None, capacity=None) -> _lib.HGSTiles:
        s = _lib.HGSTiles()
        s.tiles_x, s.tiles_y, s.tile_px = self.tiles_x, self.tiles_y, self.tile_px
        if capacity is None:
            capacity = self.capacity if self.capacity is not None else len(self.entries_orig)
        s.capacity = capacity
        s.entries, s.tile_starts = _lib.ptr(self.entries_orig), _lib.ptr(self.tile_starts)
        s.counters = _lib.ptr(counters if counters is not None else self.counters)
        s.ready = _lib.ptr(self.ready) if self.ready is not None else None
        return s


@dataclass
class RenderCtx:
    """State retained from a forward pass for the matching backward pass
    (RenderCtx, splat/render.py:44-55)."""

    gaussians: GaussianSet
    camera: Camera
    proj: ProjectedGaussians
    tiles: TileBins
    mesh: Optional[MeshLayer]
    background: np.ndarray
    final_t: torch.Tensor          # (H, W) fp64
    last_consumed: torch.Tensor    # (H, W) int32, global entry index
    cam_dev: Optional[torch.Tensor] = None


@dataclass
class GaussianGrads:
    """Gradients for every GaussianSet parameter (full-length; culled rows
    carry zeros) plus the incoming mesh-layer colour gradient
    (GaussianGrads, splat/render.py:58-71).  Device fp32 tensors."""

    centers: torch.Tensor
    rotations: torch.Tensor
    log_scales: torch.Tensor
    logit_opacities: torch.Tensor
    colors_dc: torch.Tensor
    colors_rest: Optional[torch.Tensor]
    densify_norm: torch.Tensor
    visible: torch.Tensor
    mesh_color: Optional[torch.Tensor]


# --------------------------------------------------------------------------
# workspace
# --------------------------------------------------------------------------

class _Scratch:
    """Grow-only device scratch buffers shared by calls on one device and
    stream (keyed by the current stream: calls enqueued on different streams
    never share a buffer, calls on one stream are ordered by it)."""

    def __init__(self):
        self.bufs = {}

    def get(self, name: str, nbytes: int, device, zeroed: bool = False) -> torch.Tensor:
        """zeroed: allocated as zeros (buffers whose users keep them zero at
        rest, e.g. the exact-walk queue of hgs_blend_forward)."""
        device = torch.device(device)
        sid = torch.cuda.current_stream(device).cuda_stream if device.type == "cuda" else 0
        key = (name, device, sid)
        b = self.bufs.get(key)
        if b is None or b.numel() < nbytes:
            n = (max(int(nbytes * 1.25), 256) + 255) // 256 * 256
            b = (torch.zeros if zeroed else torch.empty)(n, dtype=torch.uint8, device=device)
            self.bufs[key] = b
        return b


SCRATCH = _Scratch()


def _upload_camera(cam, device) -> torch.Tensor:
    return camera_tensor(cam, device)


def _bg3(background) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(background, dtype=np.float64).reshape(3))


def _c_f64_3(bg: np.ndarray):
    return (ctypes_c_double * 3)(*[float(x) for x in bg])


import ctypes  # noqa: E402

ctypes_c_double = ctypes.c_double


# --------------------------------------------------------------------------
# operators
# --------------------------------------------------------------------------

def _preprocess(gs: GaussianSet, cam, cam_dev, tile_px: int, extras: bool) -> ProjectedGaussians:
    dev = gs.device
    n = len(gs)
    rec = torch.empty(max(n, 1) * REC_BYTES, dtype=torch.uint8, device=dev)
    count = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    rect = torch.zeros(max(n, 1) * 4, dtype=torch.int16, device=dev)
    cull = torch.empty(max(n, 1) * 12, dtype=torch.float32, device=dev)
    sort_keys = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    tx = (int(cam.width) + tile_px - 1) // tile_px
    ty = (int(cam.height) + tile_px - 1) // tile_px
    tile_diff = torch.empty(16 * (tx + 1) * (ty + 1), dtype=torch.int32, device=dev)
    ex = None
    ps = _lib.HGSProjected()
    ps.rec, ps.count, ps.rect, ps.cull = _lib.ptr(rec), _lib.ptr(count), _lib.ptr(rect), _lib.ptr(cull)
    ps.sort_keys, ps.tile_diff = _lib.ptr(sort_keys), _lib.ptr(tile_diff)
    if extras:
        f64 = dict(dtype=torch.float64, device=dev)
        ex = {"cov2d": torch.zeros(n, 3, **f64), "radius": torch.zeros(n, **f64), "t_cam": torch.zeros(n, 3, **f64),
              "color_pre": torch.zeros(n, 3, **f64)}
        if gs.sh_degree:
            ex["view_dir"] = torch.zeros(n, 3, **f64)
            ex["view_dist"] = torch.zeros(n, **f64)
        for k, v in ex.items():
            setattr(ps, k, _lib.ptr(v))
    _lib.call("hgs_preprocess", _lib.ptr(cam_dev), int(cam.width), int(cam.height), ctypes.byref(gs.struct()),
              int(tile_px), ctypes.byref(ps), _stream_ptr(dev))
    return ProjectedGaussians(n, rec, count, rect, ex, int(cam.width), int(cam.height), tile_px, cull, sort_keys,
                              tile_diff)


def project(gs, cam) -> ProjectedGaussians:
    """splat/project.py:70-140 (plus the per-row tile counts of tiles.py:45-50)."""
    gs = GaussianSet.from_any(gs)
    cam = Camera.from_any(cam)
    cam_dev = _upload_camera(cam, gs.device)
    return _preprocess(gs, cam, cam_dev, TILE_PX, extras=True)


def _tiles_core(proj: ProjectedGaussians, width: int, height: int, tile_px: int, capacity: Optional[int]):
    """Runs hgs_build_tiles.  capacity=None sizes the entry buffer exactly
    (one device->host read of K); otherwise uses the given capacity and
    reports overflow in counters[2]."""
    dev = proj.rec.device
    tx = (width + tile_px - 1) // tile_px
    ty = (height + tile_px - 1) // tile_px
    if capacity is None:
        capacity = int(proj.count.sum().item()) if proj.n else 0
    cap = max(int(capacity), 1)
    tile_starts = torch.empty(tx * ty + 1, dtype=torch.int64, device=dev)
    entries = torch.empty(cap, dtype=torch.int32, device=dev)
    counters = torch.zeros(4, dtype=torch.int64, device=dev)
    ready = torch.zeros(_lib.READY_INTS, dtype=torch.int32, device=dev)
    nbytes = _lib.load().hgs_tiles_scratch_bytes(proj.n, cap, tx * ty)
    scratch = SCRATCH.get("tiles", nbytes, dev)
    ts = _lib.HGSTiles()
    ts.tiles_x, ts.tiles_y, ts.tile_px, ts.capacity = tx, ty, tile_px, cap
    ts.entries, ts.tile_starts, ts.counters = _lib.ptr(entries), _lib.ptr(tile_starts), _lib.ptr(counters)
    ts.scratch, ts.scratch_bytes = _lib.ptr(scratch), scratch.numel()
    ts.ready = _lib.ptr(ready)
    _lib.call("hgs_build_tiles", ctypes.byref(proj.struct()), proj.n, ctypes.byref(ts), _stream_ptr(dev))
    return TileBins(tile_starts, entries, tx, ty, tile_px, proj, counters=counters, capacity=cap, ready=ready), counters


def build_tiles(proj: ProjectedGaussians, width: int, height: int, tile_px: int = TILE_PX) -> TileBins:
    """splat/tiles.py:35-69."""
    if tile_px != TILE_PX:
        raise ValueError("only tile_px == 16 is implemented on the B200 path")
    tiles, _ = _tiles_core(proj, width, height, tile_px, None)
    return tiles


def _blend(proj, tiles: TileBins, width, height, mesh: Optional[MeshLayer], bg: np.ndarray, mask=None,
           stats=None, want_state=True):
    dev = proj.rec.device
    if mesh is not None:
        for name, t, shp in (("color", mesh.color, (height, width, 3)), ("depth", mesh.depth, (height, width)),
                             ("triangle_id", mesh.triangle_id, (height, width))):
            if tuple(t.shape) != shp:
                raise ValueError(f"mesh {name} shape {tuple(t.shape)} != {shp}")
    color = torch.empty(height, width, 3, dtype=torch.float32, device=dev)
    depth = torch.empty(height, width, dtype=torch.float32, device=dev)
    trans = torch.empty(height, width, dtype=torch.float32, device=dev)
    final_t = torch.empty(height, width, dtype=torch.float64, device=dev) if want_state else None
    last = torch.empty(height, width, dtype=torch.int32, device=dev) if want_state else None
    out = _lib.HGSBlendOut()
    out.color, out.depth, out.transmittance = _lib.ptr(color), _lib.ptr(depth), _lib.ptr(trans)
    out.final_t, out.last = _lib.ptr(final_t), _lib.ptr(last)
    variant, k = (0, 20.0)
    mask_t = None
    if mask is not None:
        variant, k = MASK_VARIANTS[mask[0]], float(mask[1])
        mask_t = torch.empty(height, width, dtype=torch.float32, device=dev)
        out.mask = _lib.ptr(mask_t)
    out.stats = _lib.ptr(stats)
    fixup = SCRATCH.get("fixup", 4 * (height * width + 4), dev, zeroed=True)
    out.fixup = _lib.ptr(fixup)
    ml = mesh.struct() if mesh is not None else _lib.HGSMeshLayer()
    _lib.call("hgs_blend_forward", ctypes.byref(proj.struct()), ctypes.byref(tiles.struct()), int(width), int(height),
              ctypes.byref(ml), _c_f64_3(bg), variant, k, ctypes.byref(out), _stream_ptr(dev))
    return color, depth, trans, final_t, last, mask_t


def rasterize_forward(proj: ProjectedGaussians, tiles: TileBins, width: int, height: int,
                      background: Union[np.ndarray, MeshLayer, tuple], mesh: Optional[MeshLayer] = None,
                      bg_color=(0.0, 0.0, 0.0)):
    """splat/render.py:74-109 -> (RenderOutputs, final_t, last_consumed)."""
    if isinstance(background, MeshLayer):
        mesh = background
        bg = _bg3(bg_color)
    else:
        bg = _bg3(background)
    color, depth, trans, final_t, last, _ = _blend(proj, tiles, width, height, mesh, bg)
    out = RenderOutputs(color=color, depth=depth, transmittance=trans,
                        triangle_id=mesh.triangle_id.clone() if mesh is not None else None)
    return out, final_t, last


def render(gs, cam, background=(0.0, 0.0, 0.0), mesh: Optional[MeshLayer] = None, tile_px: int = TILE_PX):
    """Project, bin and blend (splat/render.py:112-121) -> (RenderOutputs, RenderCtx)."""
    if tile_px != TILE_PX:
        raise ValueError("only tile_px == 16 is implemented on the B200 path")
    gs = GaussianSet.from_any(gs)
    cam = Camera.from_any(cam)
    if mesh is not None and not isinstance(mesh, MeshLayer):
        mesh = MeshLayer(mesh.color, mesh.depth, mesh.triangle_id)
    cam_dev = _upload_camera(cam, gs.device)
    proj = _preprocess(gs, cam, cam_dev, tile_px, extras=False)
    tiles, _ = _tiles_core(proj, int(cam.width), int(cam.height), tile_px, None)
    bg = _bg3(background)
    out, final_t, last = rasterize_forward(proj, tiles, int(cam.width), int(cam.height), bg, mesh=mesh)
    ctx = RenderCtx(gs, cam, proj, tiles, mesh, bg, final_t, last, cam_dev)
    return out, ctx


def render_depth(gs, cam, tile_px: int = TILE_PX) -> torch.Tensor:
    """(H, W) fp64 median-style depth map for surface extraction, NaN where
    the accumulated opacity never exceeds 0.5 (splat/render.py:316-324,
    depth_kernel splat/kernels.py:163-202)."""
    if tile_px != TILE_PX:
        raise ValueError("only tile_px == 16 is implemented on the B200 path")
    gs = GaussianSet.from_any(gs)
    cam = Camera.from_any(cam)
    w, h = int(cam.width), int(cam.height)
    proj = _preprocess(gs, cam, _upload_camera(cam, gs.device), tile_px, extras=False)
    tiles, counters = _tiles_core(proj, w, h, tile_px, None)
    out = torch.empty(h, w, dtype=torch.float64, device=gs.device)
    _lib.call("hgs_render_depth", ctypes.byref(proj.struct()), ctypes.byref(tiles.struct(counters)), w, h,
              _lib.ptr(out), _stream_ptr(gs.device))
    return out


def rasterize_backward(ctx: RenderCtx, grad_color, grad_transmittance=None) -> GaussianGrads:
    """splat/render.py:124-182: analytic gradients of sum(grad_color * pixel)
    (+ sum(grad_transmittance * T)) for all parameters."""
    from .backward import rasterize_backward as _bw
    return _bw(ctx, grad_color, grad_transmittance)
