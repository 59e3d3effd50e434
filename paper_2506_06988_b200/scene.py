"""Scene data model on the device: Gaussian sets, cameras, textured meshes.

Mirrors gsmesh/scene.py (GaussianSet :37-123, Camera :144-203,
TexturedMesh :206-274, RenderOutputs :277-291) with the same conventions:
camera looks down +z, y down, pixel (iy, ix) sampled at (ix+0.5, iy+0.5),
quaternions (w, x, y, z), colours linear RGB.

Differences by design (B200 layout):
  * Gaussian parameters live in ONE flat fp32 device buffer (``params``) with
    per-group views, so gradients, Adam moments and the NCCL all-reduce are a
    single contiguous buffer each.  Group offsets are 64-float aligned.
  * The Camera is host-side fp64 (like the reference) and is uploaded as a
    256-byte ``hgs_camera`` struct per use.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib

ROTATION_REJECT_TOL = 1e-4
FRUSTUM_LIMIT = 1.3
GROUPS = ("centers", "rotations", "log_scales", "logit_opacities", "colors_dc", "colors_rest")
GROUP_WIDTH = {"centers": 3, "rotations": 4, "log_scales": 3, "logit_opacities": 1, "colors_dc": 3, "colors_rest": 9}


class SceneError(ValueError):
    """Raised for invalid scene data (scene.py:26-27)."""


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2506_06988_b200 needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _as_tensor(a, device, dtype=torch.float32) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype)
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device=device).to(dtype)


def group_layout(n: int, sh_degree: int):
    """Offsets (in floats) of each parameter group inside the flat buffer."""
    off = 0
    layout = {}
    for g in GROUPS:
        if g == "colors_rest" and sh_degree == 0:
            continue
        layout[g] = (off, n * GROUP_WIDTH[g])
        off += (n * GROUP_WIDTH[g] + 63) // 64 * 64
    return layout, off


class GaussianSet:
    """Optimizable Gaussian primitives (GaussianSet, scene.py:37-123) in one
    flat fp32 device buffer."""

    def __init__(self, centers, rotations, log_scales, logit_opacities, colors_dc, colors_rest=None, device=None):
        device = torch.device(device) if device is not None else default_device()
        c = np.asarray(centers.detach().cpu() if isinstance(centers, torch.Tensor) else centers)
        if c.ndim != 2 or c.shape[1:] != (3,):
            raise SceneError(f"centers: expected shape (N, 3), got {c.shape}")
        n = len(c)
        shapes = {"rotations": (rotations, (4,)), "log_scales": (log_scales, (3,)), "colors_dc": (colors_dc, (3,))}
        for name, (arr, tail) in shapes.items():
            a = arr if isinstance(arr, torch.Tensor) else np.asarray(arr)
            if a.ndim != 2 or tuple(a.shape[1:]) != tail:
                raise SceneError(f"{name}: expected shape (N, {', '.join(map(str, tail))}), got {tuple(a.shape)}")
            if len(a) != n:
                raise SceneError(f"{name} has length {len(a)}, centers has {n}")
        lg = logit_opacities.reshape(-1) if isinstance(logit_opacities, torch.Tensor) else np.asarray(logit_opacities).reshape(-1)
        if len(lg) != n:
            raise SceneError(f"logit_opacities has length {len(lg)}, centers has {n}")
        sh = 0
        if colors_rest is not None:
            r = colors_rest if isinstance(colors_rest, torch.Tensor) else np.asarray(colors_rest)
            if tuple(r.shape) != (n, 3, 3):
                raise SceneError(f"colors_rest: expected shape ({n}, 3, 3), got {tuple(r.shape)}")
            sh = 1
        self.n = n
        self.sh_degree = sh
        self.layout, total = group_layout(n, sh)
        self.params = torch.zeros(max(total, 64), dtype=torch.float32, device=device)
        src = {"centers": centers, "rotations": rotations, "log_scales": log_scales,
               "logit_opacities": lg, "colors_dc": colors_dc, "colors_rest": colors_rest}
        for g, (off, size) in self.layout.items():
            if size:
                self.params[off:off + size].copy_(_as_tensor(src[g], device).reshape(-1))

    # group views ---------------------------------------------------------
    def group(self, name: str) -> Optional[torch.Tensor]:
        if name not in self.layout:
            return None
        off, size = self.layout[name]
        v = self.params[off:off + size]
        w = GROUP_WIDTH[name]
        if name == "logit_opacities":
            return v
        if name == "colors_rest":
            return v.view(self.n, 3, 3)
        return v.view(self.n, w)

    centers = property(lambda self: self.group("centers"))
    rotations = property(lambda self: self.group("rotations"))
    log_scales = property(lambda self: self.group("log_scales"))
    logit_opacities = property(lambda self: self.group("logit_opacities"))
    colors_dc = property(lambda self: self.group("colors_dc"))
    colors_rest = property(lambda self: self.group("colors_rest"))

    @property
    def device(self) -> torch.device:
        return self.params.device

    def __len__(self) -> int:
        return self.n

    def opacities(self) -> torch.Tensor:
        return torch.sigmoid(self.logit_opacities.double())

    def scales(self) -> torch.Tensor:
        return torch.exp(self.log_scales.double())

    def normalize_rotations(self) -> None:
        """In-place renormalisation (scene.py:87-92)."""
        q = self.rotations
        norms = torch.linalg.norm(q.double(), dim=1, keepdim=True)
        if bool((norms == 0).any()):
            raise SceneError("zero-norm quaternion cannot be normalized")
        q.copy_((q.double() / norms).float())

    def select(self, idx) -> "GaussianSet":
        if isinstance(idx, np.ndarray):
            idx = torch.as_tensor(idx, device=self.device)
        rest = None if self.colors_rest is None else self.colors_rest[idx]
        return GaussianSet(self.centers[idx], self.rotations[idx], self.log_scales[idx],
                           self.logit_opacities[idx], self.colors_dc[idx], rest, device=self.device)

    def copy(self) -> "GaussianSet":
        out = GaussianSet.__new__(GaussianSet)
        out.n, out.sh_degree, out.layout = self.n, self.sh_degree, dict(self.layout)
        out.params = self.params.clone()
        return out

    def struct(self) -> _lib.HGSGaussians:
        s = _lib.HGSGaussians()
        s.centers = _lib.ptr(self.centers)
        s.rotations = _lib.ptr(self.rotations)
        s.log_scales = _lib.ptr(self.log_scales)
        s.logits = _lib.ptr(self.logit_opacities)
        s.colors_dc = _lib.ptr(self.colors_dc)
        s.colors_rest = _lib.ptr(self.colors_rest) if self.sh_degree else None
        s.n = self.n
        return s

    @staticmethod
    def allocate(n: int, sh_degree: int, device) -> "GaussianSet":
        """Uninitialised rows (filled by a device kernel, e.g. density control)."""
        out = GaussianSet.__new__(GaussianSet)
        out.n, out.sh_degree = int(n), int(sh_degree)
        out.layout, total = group_layout(out.n, out.sh_degree)
        out.params = torch.empty(max(total, 64), dtype=torch.float32, device=device)
        return out

    def buf(self) -> _lib.HGSGaussianBuf:
        s = _lib.HGSGaussianBuf()
        s.centers, s.rotations = _lib.ptr(self.centers), _lib.ptr(self.rotations)
        s.log_scales, s.logits = _lib.ptr(self.log_scales), _lib.ptr(self.logit_opacities)
        s.colors_dc = _lib.ptr(self.colors_dc)
        s.colors_rest = _lib.ptr(self.colors_rest) if self.sh_degree else None
        s.n = self.n
        return s

    @staticmethod
    def empty(sh_degree: int = 0, device=None) -> "GaussianSet":
        rest = np.zeros((0, 3, 3)) if sh_degree >= 1 else None
        return GaussianSet(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros((0,)), np.zeros((0, 3)),
                           rest, device=device)

    @staticmethod
    def from_any(gs, device=None) -> "GaussianSet":
        """Accept this class, or any object with the reference's attribute
        names (e.g. gsmesh.scene.GaussianSet with float64 numpy arrays)."""
        if isinstance(gs, GaussianSet):
            return gs
        return GaussianSet(gs.centers, gs.rotations, gs.log_scales, gs.logit_opacities, gs.colors_dc,
                           getattr(gs, "colors_rest", None), device=device)

    def numpy(self) -> dict:
        return {g: (None if self.group(g) is None else self.group(g).detach().cpu().numpy().astype(np.float64))
                for g in GROUPS}


@dataclass(frozen=True)
class Camera:
    """Pinhole camera (Camera, scene.py:144-203); host-side fp64 with the
    reference's validation and SVD repair of the rotation block."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    world_to_camera: np.ndarray
    near: float = 0.01
    far: float = 100.0

    def __post_init__(self):
        W = np.asarray(self.world_to_camera, dtype=np.float64)
        if W.shape != (4, 4):
            raise SceneError(f"world_to_camera must be 4x4, got {W.shape}")
        R = W[:3, :3]
        defect = float(np.abs(R @ R.T - np.eye(3)).max())
        if defect > ROTATION_REJECT_TOL:
            raise SceneError(f"rotation block not orthonormal (defect {defect:.3g} > {ROTATION_REJECT_TOL:g})")
        if defect > 1e-12:
            U, _, Vt = np.linalg.svd(R)
            W = W.copy()
            W[:3, :3] = U @ Vt
        W = np.array(W)
        W.setflags(write=False)
        object.__setattr__(self, "world_to_camera", W)
        if not (0.0 < self.near < self.far):
            raise SceneError(f"need 0 < near < far, got near={self.near}, far={self.far}")
        if self.width <= 0 or self.height <= 0:
            raise SceneError("image dimensions must be positive")

    @property
    def rotation(self) -> np.ndarray:
        return self.world_to_camera[:3, :3]

    @property
    def translation(self) -> np.ndarray:
        return self.world_to_camera[:3, 3]

    def center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation

    @staticmethod
    def from_any(cam) -> "Camera":
        if isinstance(cam, Camera):
            return cam
        return Camera(cam.fx, cam.fy, cam.cx, cam.cy, int(cam.width), int(cam.height),
                      np.asarray(cam.world_to_camera), cam.near, cam.far)


def camera_extent(cameras) -> float:
    """scene.py:314-322: 1.1 x the largest distance of a camera centre from
    their mean."""
    if not cameras:
        raise SceneError("camera_extent needs at least one camera")
    centers = np.stack([Camera.from_any(c).center() for c in cameras])
    mean = centers.mean(axis=0)
    return 1.1 * float(np.linalg.norm(centers - mean, axis=1).max())


def camera_struct(cam) -> _lib.HGSCamera:
    """hgs_camera with the derived fields computed like the reference."""
    W = np.asarray(cam.world_to_camera, dtype=np.float64)
    R = np.ascontiguousarray(W[:3, :3])
    t = np.ascontiguousarray(W[:3, 3])
    c = _lib.HGSCamera()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    c.R[:] = [float(x) for x in R.reshape(-1)]
    c.T[:] = [float(x) for x in t]
    c.near, c.far = float(cam.near), float(cam.far)
    c.center[:] = [float(x) for x in (-R.T @ t)]  # scene.py:190-192
    c.limx = FRUSTUM_LIMIT * (cam.width / (2.0 * cam.fx))  # project.py:97-98
    c.limy = FRUSTUM_LIMIT * (cam.height / (2.0 * cam.fy))
    return c


CAMERA_BYTES = 256


def camera_tensor(cam, device, out: Optional[torch.Tensor] = None, pinned: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Upload the camera struct to a device byte tensor (H2D of 256 B)."""
    s = camera_struct(cam)
    raw = bytes(s).ljust(CAMERA_BYTES, b"\0")
    host = pinned if pinned is not None else torch.empty(CAMERA_BYTES, dtype=torch.uint8)
    host.numpy()[:] = np.frombuffer(raw, dtype=np.uint8)
    if out is None:
        out = torch.empty(CAMERA_BYTES, dtype=torch.uint8, device=device)
    out.copy_(host, non_blocking=pinned is not None)
    return out


class TexturedMesh:
    """Indexed triangle mesh with optional per-corner UVs and texture
    (TexturedMesh, scene.py:206-274), device-resident: vertices fp32 (V,3),
    triangles int32 (F,3), uvs fp32 (F,3,2), texture fp32 (Ht,Wt,3)."""

    def __init__(self, vertices, triangles, uvs=None, texture=None, device=None):
        device = torch.device(device) if device is not None else default_device()
        v = _as_tensor(vertices, device).reshape(-1, 3).contiguous()
        f = _as_tensor(triangles, device, torch.int32).reshape(-1, 3).contiguous()
        if len(f) and (int(f.min()) < 0 or int(f.max()) >= len(v)):
            raise SceneError("triangle index out of range")
        if (uvs is None) != (texture is None):
            raise SceneError("uvs and texture must be present together")
        self.vertices, self.triangles = v, f
        self.uvs = self.texture = None
        if uvs is not None:
            u = _as_tensor(uvs, device)
            if tuple(u.shape) != (len(f), 3, 2):
                raise SceneError(f"uvs must be (F, 3, 2), got {tuple(u.shape)}")
            t = _as_tensor(texture, device)
            if t.ndim != 3 or t.shape[2] != 3:
                raise SceneError("texture must be (H, W, 3)")
            self.uvs, self.texture = u.contiguous(), t.contiguous()

    @property
    def n_faces(self) -> int:
        return len(self.triangles)

    @property
    def device(self):
        return self.vertices.device

    def struct(self) -> _lib.HGSMesh:
        s = _lib.HGSMesh()
        s.vertices = _lib.ptr(self.vertices)
        s.triangles = _lib.ptr(self.triangles)
        s.uvs = _lib.ptr(self.uvs)
        s.n_vertices = len(self.vertices)
        s.n_faces = len(self.triangles)
        return s

    def copy(self) -> "TexturedMesh":
        out = TexturedMesh.__new__(TexturedMesh)
        out.vertices, out.triangles = self.vertices.clone(), self.triangles.clone()
        out.uvs = None if self.uvs is None else self.uvs.clone()
        out.texture = None if self.texture is None else self.texture.clone()
        return out

    @staticmethod
    def from_any(mesh, device=None) -> "TexturedMesh":
        if isinstance(mesh, TexturedMesh):
            return mesh
        return TexturedMesh(mesh.vertices, mesh.triangles, getattr(mesh, "uvs", None), getattr(mesh, "texture", None),
                            device=device)


@dataclass
class RenderOutputs:
    """Per-pixel render results (RenderOutputs, scene.py:277-291), device tensors."""

    color: torch.Tensor
    depth: torch.Tensor
    transmittance: torch.Tensor
    triangle_id: Optional[torch.Tensor] = None

    def numpy(self) -> dict:
        return {k: (None if v is None else v.detach().cpu().numpy()) for k, v in self.__dict__.items()}
