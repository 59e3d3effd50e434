"""Python face of the CPU oracle (oracle/gsmesh_oracle.c).

TEST INFRASTRUCTURE ONLY: the parity checker and the CPU baseline.  Imported
only by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``).  The product package never imports this module.

Every function mirrors one reference function (file:line in /root/reference,
``pkg/src/gsmesh``) and works on float64 numpy arrays.  Scene objects are
duck-typed: anything with the reference's attribute names (``centers``,
``rotations``, ``log_scales``, ``logit_opacities``, ``colors_dc``,
``colors_rest``; camera ``fx fy cx cy width height world_to_camera near far``)
is accepted, including the reference's own dataclasses.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

# reference constants (splat/project.py:19-27, tiles.py:16, losses.py:21-24)
SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
FRUSTUM_LIMIT = 1.3
TILE_PX = 16
SUPPORT_MAHAL2 = 9.0
ALPHA_CLAMP = 0.99
SIGMA_SKIP = 1.0 / 255.0
EARLY_STOP_T = 1e-4
MASK_VARIANTS = {"sigmoid": 0, "identity_t": 1, "constant_one": 2, "constant_zero": 3}


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.or_tile_counts.restype = ctypes.c_int64
        _lib.or_ssim.restype = ctypes.c_double
        _lib.or_texture_loss.restype = ctypes.c_double
        _lib.or_l1.restype = ctypes.c_double
        _lib.or_max_threads.restype = ctypes.c_int
    return _lib


def max_threads() -> int:
    return int(lib().or_max_threads())


class _Cam(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("width", ctypes.c_int64), ("height", ctypes.c_int64),
                ("R", ctypes.c_double * 9), ("T", ctypes.c_double * 3), ("near", ctypes.c_double),
                ("far", ctypes.c_double), ("center", ctypes.c_double * 3), ("limx", ctypes.c_double),
                ("limy", ctypes.c_double)]


def camera_struct(cam) -> _Cam:
    W = np.asarray(cam.world_to_camera, dtype=np.float64)
    R = np.ascontiguousarray(W[:3, :3])
    t = np.ascontiguousarray(W[:3, 3])
    c = _Cam()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    c.R[:] = list(R.reshape(-1))
    c.T[:] = list(t)
    c.near, c.far = float(cam.near), float(cam.far)
    c.center[:] = list(-R.T @ t)  # Camera.center() (scene.py:190-192)
    c.limx = FRUSTUM_LIMIT * (cam.width / (2.0 * cam.fx))  # project.py:97-98
    c.limy = FRUSTUM_LIMIT * (cam.height / (2.0 * cam.fy))
    return c


def _p(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


@dataclass
class Projected:
    """ProjectedGaussians (splat/project.py:30-53)."""
    kept: np.ndarray
    mean2d: np.ndarray
    depth: np.ndarray
    cov2d: np.ndarray
    conic: np.ndarray
    alpha: np.ndarray
    color: np.ndarray
    radius: np.ndarray
    t_cam: np.ndarray
    color_pre: np.ndarray
    view_dir: Optional[np.ndarray]
    view_dist: Optional[np.ndarray]

    def __len__(self):
        return len(self.kept)


def project(gs, cam, nthreads: int = 0) -> Projected:
    """splat/project.py:70-140."""
    centers = _f64(gs.centers).reshape(-1, 3)
    n = len(centers)
    rot = _f64(gs.rotations).reshape(-1, 4)
    ls = _f64(gs.log_scales).reshape(-1, 3)
    lg = _f64(gs.logit_opacities).reshape(-1)
    dc = _f64(gs.colors_dc).reshape(-1, 3)
    rest = None if getattr(gs, "colors_rest", None) is None else _f64(gs.colors_rest).reshape(-1, 3, 3)
    alive = np.zeros(n, np.uint8)
    mean2d = np.zeros((n, 2)); depth = np.zeros(n); cov2d = np.zeros((n, 3)); conic = np.zeros((n, 3))
    alpha = np.zeros(n); color = np.zeros((n, 3)); radius = np.zeros(n); t_cam = np.zeros((n, 3))
    color_pre = np.zeros((n, 3))
    vdir = np.zeros((n, 3)) if rest is not None else None
    vdist = np.zeros(n) if rest is not None else None
    c = camera_struct(cam)
    if n:
        lib().or_project(ctypes.byref(c), ctypes.c_int64(n), _p(centers), _p(rot), _p(ls), _p(lg), _p(dc), _p(rest),
                         _p(alive), _p(mean2d), _p(depth), _p(cov2d), _p(conic), _p(alpha), _p(color), _p(radius),
                         _p(t_cam), _p(color_pre), _p(vdir), _p(vdist), ctypes.c_int(nthreads))
    kept = np.nonzero(alive)[0].astype(np.int64)
    return Projected(kept, mean2d[kept], depth[kept], cov2d[kept], conic[kept], alpha[kept], color[kept],
                     radius[kept], t_cam[kept], color_pre[kept],
                     None if vdir is None else vdir[kept], None if vdist is None else vdist[kept])


@dataclass
class Tiles:
    """TileBins (splat/tiles.py:19-32)."""
    tile_starts: np.ndarray
    entries: np.ndarray
    tiles_x: int
    tiles_y: int
    tile_px: int

    def tile_list(self, tx, ty):
        t = ty * self.tiles_x + tx
        return self.entries[self.tile_starts[t]:self.tile_starts[t + 1]]


def tile_counts(proj: Projected, width: int, height: int, tile_px: int = TILE_PX, nthreads: int = 0):
    """Per-row tile counts (tiles.py:45-50)."""
    m = len(proj)
    counts = np.zeros(m, np.int64)
    if m:
        lib().or_tile_counts(ctypes.c_int64(m), _p(_f64(proj.mean2d)), _p(_f64(proj.radius)), ctypes.c_int64(width),
                             ctypes.c_int64(height), ctypes.c_int64(tile_px), _p(counts), ctypes.c_int(nthreads))
    return counts


def build_tiles(proj: Projected, width: int, height: int, tile_px: int = TILE_PX, nthreads: int = 0) -> Tiles:
    """splat/tiles.py:35-69."""
    tx = (width + tile_px - 1) // tile_px
    ty = (height + tile_px - 1) // tile_px
    m = len(proj)
    if m == 0:
        return Tiles(np.zeros(tx * ty + 1, np.int64), np.zeros(0, np.int32), tx, ty, tile_px)
    mean2d, radius = _f64(proj.mean2d), _f64(proj.radius)
    counts = np.zeros(m, np.int64)
    k = lib().or_tile_counts(ctypes.c_int64(m), _p(mean2d), _p(radius), ctypes.c_int64(width),
                             ctypes.c_int64(height), ctypes.c_int64(tile_px), _p(counts), ctypes.c_int(nthreads))
    starts = np.zeros(tx * ty + 1, np.int64)
    entries = np.zeros(k, np.int32)
    lib().or_build_tiles(ctypes.c_int64(m), _p(mean2d), _p(radius), _p(_f64(proj.depth)),
                         _p(np.ascontiguousarray(proj.kept, dtype=np.int64)), ctypes.c_int64(width),
                         ctypes.c_int64(height), ctypes.c_int64(tile_px), _p(starts), _p(entries),
                         ctypes.c_int(nthreads))
    return Tiles(starts, entries, tx, ty, tile_px)


@dataclass
class Mesh:
    """MeshLayer (splat/render.py:26-41)."""
    color: np.ndarray
    depth: np.ndarray
    triangle_id: np.ndarray

    @property
    def valid(self):
        return self.triangle_id >= 0


def rasterize_forward(proj: Projected, tiles: Tiles, width: int, height: int, bg=(0.0, 0.0, 0.0),
                      mesh=None, nthreads: int = 0):
    """splat/render.py:74-109 -> (color, depth, T, last)."""
    bg = _f64(bg).reshape(3)
    out_color = np.zeros((height, width, 3))
    out_t = np.ones((height, width))
    out_depth = np.full((height, width), np.nan)
    out_last = np.full((height, width), -1, np.int32)
    has_mesh = mesh is not None
    mc = _f64(mesh.color) if has_mesh else np.zeros((1, 1, 3))
    md = _f64(mesh.depth) if has_mesh else np.zeros((1, 1))
    mv = np.ascontiguousarray(np.asarray(mesh.triangle_id) >= 0, dtype=np.uint8) if has_mesh else np.zeros((1, 1), np.uint8)
    lib().or_forward(_p(tiles.tile_starts), _p(tiles.entries), ctypes.c_int64(tiles.tiles_x),
                     ctypes.c_int64(tiles.tiles_y), ctypes.c_int64(tiles.tile_px), ctypes.c_int64(width),
                     ctypes.c_int64(height), _p(_f64(proj.mean2d)), _p(_f64(proj.conic)), _p(_f64(proj.alpha)),
                     _p(_f64(proj.color)), _p(_f64(proj.depth)), ctypes.c_int(int(has_mesh)), _p(mc), _p(md),
                     _p(mv), _p(bg), _p(out_color), _p(out_t), _p(out_depth), _p(out_last), ctypes.c_int(nthreads))
    return out_color, out_depth, out_t, out_last


@dataclass
class Grads:
    """GaussianGrads (splat/render.py:58-71)."""
    centers: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    logit_opacities: np.ndarray
    colors_dc: np.ndarray
    colors_rest: Optional[np.ndarray]
    densify_norm: np.ndarray
    visible: np.ndarray
    mesh_color: Optional[np.ndarray]


def rasterize_backward(gs, cam, proj: Projected, tiles: Tiles, mesh, bg, final_t, last, grad_color,
                       grad_transmittance=None, nthreads: int = 0) -> Grads:
    """splat/render.py:124-182 (+ _chain_to_parameters :185-287)."""
    h, w = int(cam.height), int(cam.width)
    grad_color = _f64(grad_color)
    if grad_color.shape != (h, w, 3):
        raise ValueError(f"grad_color shape {grad_color.shape} != {(h, w, 3)}")
    if grad_transmittance is None:
        grad_transmittance = np.zeros((h, w))
    grad_transmittance = _f64(grad_transmittance)
    if grad_transmittance.shape != (h, w):
        raise ValueError(f"grad_transmittance shape {grad_transmittance.shape} != {(h, w)}")
    bg = _f64(bg).reshape(3)
    k = len(tiles.entries)
    entry_grads = np.zeros((max(k, 1), 9))
    has_mesh = mesh is not None
    mc = _f64(mesh.color) if has_mesh else np.zeros((1, 1, 3))
    mv = np.ascontiguousarray(np.asarray(mesh.triangle_id) >= 0, dtype=np.uint8) if has_mesh else np.zeros((1, 1), np.uint8)
    L = lib()
    L.or_backward_entries(_p(tiles.tile_starts), _p(tiles.entries), ctypes.c_int64(tiles.tiles_x),
                          ctypes.c_int64(tiles.tiles_y), ctypes.c_int64(tiles.tile_px), ctypes.c_int64(w),
                          ctypes.c_int64(h), _p(_f64(proj.mean2d)), _p(_f64(proj.conic)), _p(_f64(proj.alpha)),
                          _p(_f64(proj.color)), ctypes.c_int(int(has_mesh)), _p(mc), _p(mv), _p(bg),
                          _p(_f64(final_t)), _p(np.ascontiguousarray(last, dtype=np.int32)), _p(grad_color),
                          _p(grad_transmittance), _p(entry_grads), ctypes.c_int(nthreads))
    m = len(proj)
    per_gauss = np.zeros((max(m, 1), 9))
    if k:
        L.or_reduce_entries(ctypes.c_int64(k), _p(tiles.entries), _p(entry_grads), _p(per_gauss))
    n = len(np.asarray(gs.centers))
    rest = None if getattr(gs, "colors_rest", None) is None else _f64(gs.colors_rest).reshape(-1, 3, 3)
    out = Grads(np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3)), np.zeros(n), np.zeros((n, 3)),
                None if rest is None else np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n, bool), None)
    if m:
        c = camera_struct(cam)
        L.or_chain(ctypes.byref(c), ctypes.c_int64(m), _p(np.ascontiguousarray(proj.kept, dtype=np.int64)),
                   _p(per_gauss), _p(_f64(gs.rotations)), _p(_f64(gs.log_scales)), _p(rest), _p(_f64(proj.alpha)),
                   _p(_f64(proj.t_cam)), _p(_f64(proj.color_pre)), _p(None if proj.view_dir is None else _f64(proj.view_dir)),
                   _p(None if proj.view_dist is None else _f64(proj.view_dist)), _p(out.centers), _p(out.rotations),
                   _p(out.log_scales), _p(out.logit_opacities), _p(out.colors_dc), _p(out.colors_rest),
                   _p(out.densify_norm), ctypes.c_int(nthreads))
        out.visible[proj.kept] = True
    if has_mesh:
        out.mesh_color = grad_color * (_f64(final_t) * (np.asarray(mesh.triangle_id) >= 0))[..., None]
    return out


def render(gs, cam, background=(0.0, 0.0, 0.0), mesh=None, tile_px: int = TILE_PX, nthreads: int = 0):
    """splat/render.py:112-121 -> (color, depth, T, ctx dict)."""
    proj = project(gs, cam, nthreads)
    tiles = build_tiles(proj, int(cam.width), int(cam.height), tile_px, nthreads)
    color, depth, t, last = rasterize_forward(proj, tiles, int(cam.width), int(cam.height), background, mesh, nthreads)
    ctx = dict(gs=gs, cam=cam, proj=proj, tiles=tiles, mesh=mesh, bg=_f64(background).reshape(3), final_t=t, last=last)
    return color, depth, t, ctx


def backward(ctx, grad_color, grad_transmittance=None, nthreads: int = 0) -> Grads:
    return rasterize_backward(ctx["gs"], ctx["cam"], ctx["proj"], ctx["tiles"], ctx["mesh"], ctx["bg"],
                              ctx["final_t"], ctx["last"], grad_color, grad_transmittance, nthreads)


@dataclass
class Fragments:
    """MeshFragmentBuffer (meshraster.py:25-42)."""
    triangle_id: np.ndarray
    bary: np.ndarray
    depth: np.ndarray
    uv: np.ndarray

    @property
    def valid(self):
        return self.triangle_id >= 0


def rasterize_fragments(vertices, triangles, uvs, cam, nthreads: int = 0) -> Fragments:
    """meshraster.py:119-136 (+ _raster_kernel :45-116)."""
    h, w = int(cam.height), int(cam.width)
    tri = np.full((h, w), -1, np.int32)
    depth = np.full((h, w), np.inf)
    bary = np.zeros((h, w, 3))
    uv = np.zeros((h, w, 2))
    v = _f64(vertices).reshape(-1, 3)
    f = np.ascontiguousarray(np.asarray(triangles).reshape(-1, 3), dtype=np.int64)
    if len(f):
        c = camera_struct(cam)
        vs = np.zeros((len(v), 2)); zs = np.zeros(len(v))
        L = lib()
        L.or_mesh_project(ctypes.byref(c), ctypes.c_int64(len(v)), _p(v), _p(vs), _p(zs))
        has_uv = uvs is not None
        u = _f64(uvs) if has_uv else np.zeros((len(f), 3, 2))
        L.or_raster(_p(vs), _p(zs), ctypes.c_int64(len(f)), _p(f), _p(u), ctypes.c_int(int(has_uv)), ctypes.c_int64(w),
                    ctypes.c_int64(h), ctypes.c_double(float(cam.near)), _p(tri), _p(depth), _p(bary), _p(uv),
                    ctypes.c_int(nthreads))
    return Fragments(tri, bary, depth, uv)


def sample_texture(texture, uv, valid, nthreads: int = 0) -> np.ndarray:
    """meshraster.py:158-166."""
    tex = _f64(texture)
    th, tw = tex.shape[:2]
    uvf = _f64(uv)
    shp = uvf.shape[:-1]
    out = np.zeros(shp + (3,))
    vm = np.ascontiguousarray(valid, dtype=np.uint8)
    lib().or_sample_texture(_p(tex), ctypes.c_int64(th), ctypes.c_int64(tw), ctypes.c_int64(int(np.prod(shp))),
                            _p(uvf), _p(vm), _p(out), ctypes.c_int(nthreads))
    return out


def texture_backward(frags: Fragments, grad_image, texture_shape) -> np.ndarray:
    """meshraster.py:169-184."""
    th, tw = texture_shape
    valid = frags.valid
    g = _f64(grad_image)
    if g.shape[:2] != valid.shape:
        raise ValueError(f"grad image shape {g.shape} does not match fragments {valid.shape}")
    out = np.zeros((th, tw, 3))
    lib().or_texture_backward(ctypes.c_int64(th), ctypes.c_int64(tw), ctypes.c_int64(valid.size), _p(_f64(frags.uv)),
                              _p(np.ascontiguousarray(valid, dtype=np.uint8)), _p(g), _p(out))
    return out


def gaussian_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    """losses.py:27-30 (same numpy expression)."""
    x = np.arange(size) - size // 2
    w = np.exp(-(x ** 2) / (2 * sigma ** 2))
    return w / w.sum()


def l1_loss(pred, target):
    """losses.py:41-44."""
    p, t = _f64(pred), _f64(target)
    g = np.zeros_like(p)
    v = lib().or_l1(ctypes.c_int64(p.size), _p(p), _p(t), _p(g))
    return float(v), g


def ssim(pred, target, nthreads: int = 0):
    """losses.py:47-70 -> (mean SSIM, grad wrt pred)."""
    x, y = _f64(pred), _f64(target)
    h, w, c = x.shape
    g = np.zeros_like(x)
    win = _f64(gaussian_window())
    v = lib().or_ssim(_p(x), _p(y), ctypes.c_int64(h), ctypes.c_int64(w), ctypes.c_int64(c), _p(win), _p(g),
                      ctypes.c_int(nthreads))
    return float(v), g


def dssim(pred, target, nthreads: int = 0):
    """losses.py:73-76."""
    s, g = ssim(pred, target, nthreads)
    return (1.0 - s) / 2.0, -0.5 * g


def transmittance_mask(t, k: float = 20.0, variant: str = "sigmoid") -> np.ndarray:
    """losses.py:79-91."""
    if variant not in MASK_VARIANTS:
        raise ValueError(f"unknown transmittance mask variant {variant!r}")
    tt = _f64(t)
    out = np.zeros_like(tt)
    lib().or_transmittance_mask(ctypes.c_int64(tt.size), _p(tt), ctypes.c_double(k), ctypes.c_int(MASK_VARIANTS[variant]),
                                _p(out))
    return out


def texture_loss(i_gt, i_m, covered, t, k: float = 20.0, variant: str = "sigmoid"):
    """losses.py:103-116 -> (L_t, grad_im, grad_t)."""
    gt, im, tt = _f64(i_gt), _f64(i_m), _f64(t)
    cov = np.ascontiguousarray(covered, dtype=np.uint8)
    gim = np.zeros_like(im)
    gtt = np.zeros_like(tt)
    v = lib().or_texture_loss(ctypes.c_int64(tt.size), _p(gt), _p(im), _p(cov), _p(tt), ctypes.c_double(k),
                              ctypes.c_int(MASK_VARIANTS[variant]), _p(gim), _p(gtt))
    return float(v), gim, gtt


def texture_loss_active(iteration: int, cfg, has_mesh: bool) -> bool:
    """losses.py:134-136."""
    return has_mesh and cfg.texture_weight > 0.0 and cfg.warmup_iters < iteration < cfg.densify_until_iter


def composite_loss(i_gt, i_h, i_m, covered, t, iteration: int, cfg, nthreads: int = 0):
    """losses.py:139-174 -> (dict breakdown, grad_ih, grad_im | None, grad_t)."""
    lam = cfg.dssim_weight
    if getattr(cfg, "zero_dssim_after_densify", False) and iteration >= cfg.densify_until_iter:
        lam = 0.0
    v_l1, g_l1 = l1_loss(i_h, i_gt)
    v_ds, g_ds = dssim(i_h, i_gt, nthreads)
    l_c = (1.0 - lam) * v_l1 + lam * v_ds
    grad_ih = (1.0 - lam) * g_l1 + lam * g_ds
    has_mesh = i_m is not None and covered is not None
    t = _f64(t)
    mean_t = float(t[covered].mean()) if (has_mesh and np.any(covered)) else float("nan")
    l_t = 0.0
    grad_im = None
    grad_t = np.zeros_like(t)
    if texture_loss_active(iteration, cfg, has_mesh):
        l_t, g_im, g_t = texture_loss(i_gt, i_m, covered, t, k=cfg.mask_sharpness, variant=cfg.mask_variant)
        grad_im = cfg.texture_weight * g_im
        grad_t = cfg.texture_weight * g_t
        total = l_c + cfg.texture_weight * l_t
    else:
        total = l_c
    bd = dict(l1=v_l1, dssim=v_ds, l_c=l_c, l_t=l_t, total=total, mean_T_on_mesh=mean_t)
    return bd, grad_ih, grad_im, grad_t


def adam_step(p, m, v, g, lr, step, beta1=0.9, beta2=0.999, eps=1e-15):
    """train/adam.py:28-42 for one group, in place on float64 arrays."""
    for a in (p, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    gg = _f64(g)
    lib().or_adam(ctypes.c_int64(p.size), _p(p), _p(m), _p(v), _p(gg), ctypes.c_double(lr), ctypes.c_double(beta1),
                  ctypes.c_double(beta2), ctypes.c_double(eps), ctypes.c_int64(step))


def render_depth(gs, cam, tile_px: int = TILE_PX) -> np.ndarray:
    """splat/render.py:316-324 with depth_kernel (splat/kernels.py:163-202)
    restated as a pure-Python loop (small cases only): per pixel, the depth
    of the entry at which 1 - T first exceeds 0.5, NaN where it never does."""
    import math
    p = project(gs, cam)
    w, h = int(cam.width), int(cam.height)
    t = build_tiles(p, w, h, tile_px)
    out = np.full((h, w), np.nan)
    mean2d, conic, alpha, depth = p.mean2d, p.conic, p.alpha, p.depth
    for ty in range(t.tiles_y):
        for tx in range(t.tiles_x):
            k0 = int(t.tile_starts[ty * t.tiles_x + tx])
            k1 = int(t.tile_starts[ty * t.tiles_x + tx + 1])
            for py in range(ty * tile_px, min(ty * tile_px + tile_px, h)):
                for px in range(tx * tile_px, min(tx * tile_px + tile_px, w)):
                    fx, fy = px + 0.5, py + 0.5
                    trans = 1.0
                    for k in range(k0, k1):
                        i = int(t.entries[k])
                        dx, dy = fx - mean2d[i, 0], fy - mean2d[i, 1]
                        m = conic[i, 0] * dx * dx + 2.0 * conic[i, 1] * dx * dy + conic[i, 2] * dy * dy
                        if m > SUPPORT_MAHAL2 or m < 0.0:
                            continue
                        sig = min(alpha[i] * math.exp(-0.5 * m), ALPHA_CLAMP)
                        if sig < SIGMA_SKIP:
                            continue
                        test_t = trans * (1.0 - sig)
                        if test_t < EARLY_STOP_T:
                            break
                        trans = test_t
                        if 1.0 - trans > 0.5:
                            out[py, px] = depth[i]
                            break
    return out


def init_texture(vertices, triangles, uvs, texture, images, cameras, iters: int = 500, lr: float = 0.05) -> np.ndarray:
    """meshraster.py:206-245, mode "optimized": texture starts at 0.5, then
    ``iters`` fp64 Adam steps on the coverage-normalised masked MSE averaged
    over the views, clamped to [0, 1] after each step.  Returns the texture."""
    tex = np.full(np.asarray(texture).shape, 0.5)
    frags = [rasterize_fragments(vertices, triangles, uvs, c) for c in cameras]
    n_cov = [int(f.valid.sum()) for f in frags]
    if sum(n_cov) == 0:
        return tex
    m, v = np.zeros_like(tex), np.zeros_like(tex)
    th, tw = tex.shape[:2]
    for step in range(1, iters + 1):
        grad = np.zeros_like(tex)
        for img, fr, cov in zip(images, frags, n_cov):
            if cov == 0:
                continue
            pred = sample_texture(tex, fr.uv, fr.valid)
            diff = np.zeros_like(pred)
            diff[fr.valid] = pred[fr.valid] - np.asarray(img, dtype=np.float64)[fr.valid]
            grad += texture_backward(fr, 2.0 * diff / cov, (th, tw))
        adam_step(tex, m, v, grad / len(cameras), lr, step)
        np.clip(tex, 0.0, 1.0, out=tex)
    return tex
