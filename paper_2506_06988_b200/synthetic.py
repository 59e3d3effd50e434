"""Seeded synthetic scenes for the BASELINE.json configs (numpy, host side).

SURVEY.md §8(d) generator: pinhole camera fx=fy=0.8 W with a non-identity
pose; Gaussians sampled inside the view frustum (pixel uniform, depth
uniform, back-projected), quaternions N(0,1)^4, log-scales U(-5.5,-3.5),
logits U(-4,0), dc U(-1,1); a textured mesh behind/among them.  Every
parameter is fp32-quantised (float32 values held in float64 arrays) so the
device path and the CPU oracle consume identical inputs.

Configs (BASELINE.json "configs"):
  c1  10k Gaussians + 2k-tri textured wall, 256x256
  c2  100k Gaussians + 20k-tri textured wall, 640x480
  c3  1M Gaussians + 200k-tri textured box room (2048^2 atlas), 1200x680
  c4  c3 scene, 64 training views on a ring inside the room
  c5  5M Gaussians + 1M-tri room, 1920x1080
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np


def q32(a) -> np.ndarray:
    """fp32-quantise, keep float64 dtype (the reference's in-memory type)."""
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


@dataclass
class HostGaussians:
    centers: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    logit_opacities: np.ndarray
    colors_dc: np.ndarray
    colors_rest: Optional[np.ndarray] = None

    def __len__(self):
        return len(self.centers)


@dataclass
class HostCamera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    world_to_camera: np.ndarray
    near: float = 0.05
    far: float = 100.0

    @property
    def rotation(self):
        return self.world_to_camera[:3, :3]

    @property
    def translation(self):
        return self.world_to_camera[:3, 3]

    def center(self):
        return -self.rotation.T @ self.translation


@dataclass
class HostMesh:
    vertices: np.ndarray
    triangles: np.ndarray
    uvs: Optional[np.ndarray] = None
    texture: Optional[np.ndarray] = None

    @property
    def n_faces(self):
        return len(self.triangles)


@dataclass
class Scene:
    name: str
    gaussians: HostGaussians
    cameras: List[HostCamera]
    mesh: Optional[HostMesh]
    meta: dict = field(default_factory=dict)


def look_at(eye, target, up=(0.0, -1.0, 0.0), width=64, height=64, f=None, near=0.05, far=100.0) -> HostCamera:
    """Camera at eye looking at target (camera +z forward, y down)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    upv = np.asarray(up, dtype=np.float64)
    right = np.cross(upv, fwd)
    if np.linalg.norm(right) < 1e-8:
        right = np.cross(np.array([0.0, 0.0, 1.0]), fwd)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    w2c = np.eye(4)
    w2c[:3, :3] = R
    w2c[:3, 3] = -R @ eye
    f = 0.8 * width if f is None else f
    return HostCamera(f, f, width / 2.0, height / 2.0, width, height, w2c, near, far)


def frustum_gaussians(rng, n, cam: HostCamera, z_range=(1.5, 9.0), log_scale=(-5.5, -3.5), logit=(-4.0, 0.0),
                      sh_degree=0) -> HostGaussians:
    u = rng.uniform(0, cam.width, n)
    v = rng.uniform(0, cam.height, n)
    z = rng.uniform(*z_range, n)
    pc = np.stack([(u - cam.cx) / cam.fx * z, (v - cam.cy) / cam.fy * z, z], axis=1)
    R, t = cam.rotation, cam.translation
    pw = (pc - t) @ R  # R^T (pc - t)
    rest = q32(rng.normal(size=(n, 3, 3)) * 0.2) if sh_degree else None
    return HostGaussians(q32(pw), q32(rng.normal(size=(n, 4))), q32(rng.uniform(*log_scale, (n, 3))),
                         q32(rng.uniform(*logit, n)), q32(rng.uniform(-1.0, 1.0, (n, 3))), rest)


def grid_quad(p0, ex, ey, nx, ny, uv0=(0.0, 0.0), uv1=(1.0, 1.0)):
    """Quad p0 + s ex + t ey subdivided into nx*ny cells (2 tris each) with
    per-corner UVs spanning [uv0, uv1]."""
    s = np.linspace(0.0, 1.0, nx + 1)
    t = np.linspace(0.0, 1.0, ny + 1)
    S, T = np.meshgrid(s, t)
    verts = np.asarray(p0)[None, None] + S[..., None] * np.asarray(ex) + T[..., None] * np.asarray(ey)
    verts = verts.reshape(-1, 3)
    uv = np.stack([uv0[0] + S * (uv1[0] - uv0[0]), uv0[1] + T * (uv1[1] - uv0[1])], -1).reshape(-1, 2)
    idx = np.arange((nx + 1) * (ny + 1)).reshape(ny + 1, nx + 1)
    a, b, c, d = idx[:-1, :-1], idx[:-1, 1:], idx[1:, 1:], idx[1:, :-1]
    tris = np.concatenate([np.stack([a, b, c], -1).reshape(-1, 3), np.stack([a, c, d], -1).reshape(-1, 3)])
    return verts, tris.astype(np.int32), uv[tris]


def wall_mesh(rng, cam: HostCamera, n_tris: int, tex_size: int, depth=6.0) -> HostMesh:
    """Tilted textured wall filling the view at camera depth ~depth (+0.1 x)."""
    cells = max(1, n_tris // 2)
    nx = int(np.ceil(np.sqrt(cells * cam.width / cam.height)))
    ny = max(1, cells // nx)
    half_w = 0.75 * depth * cam.width / cam.fx
    half_h = 0.75 * depth * cam.height / cam.fy
    p0c = np.array([-half_w, -half_h, depth - 0.1 * half_w])
    exc = np.array([2 * half_w, 0.0, 0.2 * half_w])
    eyc = np.array([0.0, 2 * half_h, 0.0])
    v, f, uv = grid_quad(p0c, exc, eyc, nx, ny)
    R, t = cam.rotation, cam.translation
    vw = (v - t) @ R
    tex = q32(rng.uniform(0.0, 1.0, (tex_size, tex_size, 3)))
    return HostMesh(q32(vw), f, q32(uv), tex)


def room_mesh(rng, n_tris: int, tex_size: int, size=(8.0, 3.0, 8.0)) -> HostMesh:
    """Axis-aligned box room (floor, ceiling, 4 walls) centred at the origin,
    subdivided to ~n_tris triangles, UVs packed into a 3x2 atlas."""
    sx, sy, sz = size
    hx, hy, hz = sx / 2, sy / 2, sz / 2
    faces = [  # (p0, ex, ey) with y pointing down (camera convention)
        ((-hx, hy, -hz), (sx, 0, 0), (0, 0, sz)),    # floor (y = +hy)
        ((-hx, -hy, -hz), (sx, 0, 0), (0, 0, sz)),   # ceiling
        ((-hx, -hy, hz), (sx, 0, 0), (0, sy, 0)),    # +z wall
        ((-hx, -hy, -hz), (sx, 0, 0), (0, sy, 0)),   # -z wall
        ((hx, -hy, -hz), (0, 0, sz), (0, sy, 0)),    # +x wall
        ((-hx, -hy, -hz), (0, 0, sz), (0, sy, 0)),   # -x wall
    ]
    areas = [np.linalg.norm(np.cross(ex, ey)) for _, ex, ey in faces]
    tot = sum(areas)
    V, F, U = [], [], []
    base = 0
    for k, ((p0, ex, ey), a) in enumerate(zip(faces, areas)):
        cells = max(1, int(round(n_tris / 2 * a / tot)))
        lx, ly = np.linalg.norm(ex), np.linalg.norm(ey)
        nx = max(1, int(round(np.sqrt(cells * lx / ly))))
        ny = max(1, cells // nx)
        ax, ay = k % 3, k // 3
        uv0 = (ax / 3.0 + 0.002, ay / 2.0 + 0.002)
        uv1 = ((ax + 1) / 3.0 - 0.002, (ay + 1) / 2.0 - 0.002)
        v, f, uv = grid_quad(p0, ex, ey, nx, ny, uv0, uv1)
        V.append(v)
        F.append(f + base)
        U.append(uv)
        base += len(v)
    tex = q32(rng.uniform(0.0, 1.0, (tex_size, tex_size, 3)))
    return HostMesh(q32(np.concatenate(V)), np.concatenate(F).astype(np.int32), q32(np.concatenate(U)), tex)


def room_camera(width, height, yaw=0.6, pitch=0.12, eye=(0.3, -0.2, -0.4), near=0.05, far=100.0) -> HostCamera:
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.array([np.sin(yaw) * np.cos(pitch), np.sin(pitch), np.cos(yaw) * np.cos(pitch)])
    return look_at(eye, eye + fwd, width=width, height=height, near=near, far=far)


def ring_cameras(n_views, width, height, radius=1.0, seed=0) -> List[HostCamera]:
    rng = np.random.default_rng(seed)
    cams = []
    for i in range(n_views):
        a = 2 * np.pi * i / n_views + rng.uniform(-0.05, 0.05)
        eye = (radius * np.cos(a), rng.uniform(-0.3, 0.3), radius * np.sin(a))
        cams.append(room_camera(width, height, yaw=a + np.pi / 2 + rng.uniform(-0.2, 0.2),
                                pitch=rng.uniform(-0.15, 0.15), eye=eye))
    return cams


def room_gaussians(rng, n, size=(8.0, 3.0, 8.0), log_scale=(-5.0, -3.0), logit=(-4.0, 0.0), sh_degree=0):
    hx, hy, hz = size[0] / 2 * 0.95, size[1] / 2 * 0.95, size[2] / 2 * 0.95
    c = np.stack([rng.uniform(-hx, hx, n), rng.uniform(-hy, hy, n), rng.uniform(-hz, hz, n)], 1)
    rest = q32(rng.normal(size=(n, 3, 3)) * 0.2) if sh_degree else None
    return HostGaussians(q32(c), q32(rng.normal(size=(n, 4))), q32(rng.uniform(*log_scale, (n, 3))),
                         q32(rng.uniform(*logit, n)), q32(rng.uniform(-1.0, 1.0, (n, 3))), rest)


def make_config(name: str, seed: int = 0, sh_degree: int = 0, n_views: int = 64) -> Scene:
    rng = np.random.default_rng(seed)
    if name in ("c1", "c2"):
        w, h, n, f, ts = (256, 256, 10_000, 2_000, 256) if name == "c1" else (640, 480, 100_000, 20_000, 1024)
        cam = look_at((0.4, -0.3, -0.2), (0.9, 0.1, 6.0), width=w, height=h)
        gs = frustum_gaussians(rng, n, cam, sh_degree=sh_degree)
        mesh = wall_mesh(rng, cam, f, ts)
        return Scene(name, gs, [cam], mesh, {"width": w, "height": h})
    if name in ("c3", "c4", "c5"):
        w, h, n, f, ts = (1200, 680, 1_000_000, 200_000, 2048) if name != "c5" else (1920, 1080, 5_000_000, 1_000_000, 2048)
        mesh = room_mesh(rng, f, ts)
        if name == "c4":
            gs = room_gaussians(rng, n, sh_degree=sh_degree)
            cams = ring_cameras(n_views, w, h, seed=seed)
        else:
            cam = room_camera(w, h)
            # Gaussians fill the view frustum out to (and partly behind) the walls
            gs = frustum_gaussians(rng, n, cam, z_range=(0.8, 7.0), sh_degree=sh_degree)
            cams = [cam]
        return Scene(name, gs, cams, mesh, {"width": w, "height": h})
    raise ValueError(f"unknown config {name!r}")


def small_scene(seed=0, n=300, width=96, height=80, n_tris=120, tex=32, sh_degree=0, with_mesh=True) -> Scene:
    """Tiny general-pose scene for golden vectors and CPU tests."""
    rng = np.random.default_rng(seed)
    cam = look_at((0.3, -0.2, -0.1), (0.6, 0.1, 5.0), width=width, height=height)
    gs = frustum_gaussians(rng, n, cam, z_range=(1.5, 8.0), log_scale=(-4.0, -2.5), logit=(-3.0, 1.0),
                           sh_degree=sh_degree)
    mesh = wall_mesh(rng, cam, n_tris, tex, depth=5.0) if with_mesh else None
    return Scene("small", gs, [cam], mesh, {"width": width, "height": height})
