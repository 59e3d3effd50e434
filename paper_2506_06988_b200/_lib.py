"""ctypes binding of libhgs.so (the C ABI declared in include/hgs.h).

The library is built in-tree (``paper_2506_06988_b200/libhgs.so``) by
``build()`` / ``__graft_entry__.build()``.  There is no fallback: if the
library or a CUDA device is missing, every operator raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HGS_LIB") or os.path.join(_HERE, "libhgs.so")  # HGS_LIB: A/B builds (tools/)
CSRC = os.path.join(_HERE, "csrc")

HGS_OK = 0
HGS_ERR_INVALID = 1
HGS_ERR_CUDA = 2

_lock = threading.Lock()
_lib = None

c_void_p = ctypes.c_void_p
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f32 = ctypes.c_float
c_f64 = ctypes.c_double


class HGSCamera(ctypes.Structure):
    _fields_ = [("fx", c_f64), ("fy", c_f64), ("cx", c_f64), ("cy", c_f64), ("width", c_i64), ("height", c_i64),
                ("R", c_f64 * 9), ("T", c_f64 * 3), ("near", c_f64), ("far", c_f64), ("center", c_f64 * 3),
                ("limx", c_f64), ("limy", c_f64)]


class HGSGaussians(ctypes.Structure):
    _fields_ = [("centers", c_void_p), ("rotations", c_void_p), ("log_scales", c_void_p), ("logits", c_void_p),
                ("colors_dc", c_void_p), ("colors_rest", c_void_p), ("n", c_i64)]


class HGSGaussianBuf(ctypes.Structure):
    _fields_ = [("centers", c_void_p), ("rotations", c_void_p), ("log_scales", c_void_p), ("logits", c_void_p),
                ("colors_dc", c_void_p), ("colors_rest", c_void_p), ("n", c_i64)]


class HGSGaussianGrads(ctypes.Structure):
    _fields_ = [("centers", c_void_p), ("rotations", c_void_p), ("log_scales", c_void_p), ("logits", c_void_p),
                ("colors_dc", c_void_p), ("colors_rest", c_void_p), ("densify_norm", c_void_p),
                ("visible", c_void_p), ("visible_count", c_void_p)]


class HGSProjected(ctypes.Structure):
    _fields_ = [("rec", c_void_p), ("count", c_void_p), ("rect", c_void_p), ("cov2d", c_void_p),
                ("radius", c_void_p), ("t_cam", c_void_p), ("color_pre", c_void_p), ("view_dir", c_void_p),
                ("view_dist", c_void_p), ("cull", c_void_p), ("sort_keys", c_void_p), ("tile_diff", c_void_p)]


class HGSTiles(ctypes.Structure):
    _fields_ = [("tiles_x", c_i32), ("tiles_y", c_i32), ("tile_px", c_i32), ("flags", c_i32),
                ("capacity", c_i64), ("entries", c_void_p), ("tile_starts", c_void_p), ("counters", c_void_p),
                ("scratch", c_void_p), ("scratch_bytes", ctypes.c_size_t), ("ready", c_void_p),
                ("join_event", c_void_p), ("coarse_rows", c_void_p), ("coarse_rects", c_void_p),
                ("coarse_starts", c_void_p), ("coarse_prog", c_void_p)]

TILES_BLEND_ONLY = 1  # HGS_TILES_BLEND_ONLY

READY_INTS = 2 + 2048  # HGS_READY_INTS


class HGSMeshLayer(ctypes.Structure):
    _fields_ = [("color", c_void_p), ("depth", c_void_p), ("triangle_id", c_void_p)]


class HGSBlendOut(ctypes.Structure):
    _fields_ = [("color", c_void_p), ("depth", c_void_p), ("transmittance", c_void_p), ("final_t", c_void_p),
                ("last", c_void_p), ("mask", c_void_p), ("stats", c_void_p), ("fixup", c_void_p)]


class HGSMesh(ctypes.Structure):
    _fields_ = [("vertices", c_void_p), ("triangles", c_void_p), ("uvs", c_void_p), ("n_vertices", c_i64),
                ("n_faces", c_i64)]


class HGSFragments(ctypes.Structure):
    _fields_ = [("triangle_id", c_void_p), ("depth", c_void_p), ("bary", c_void_p), ("uv", c_void_p)]


class HGSAdamGroup(ctypes.Structure):
    _fields_ = [("param", c_void_p), ("m", c_void_p), ("v", c_void_p), ("grad", c_void_p), ("n", c_i64),
                ("lr", c_f32), ("mode", c_i32)]


HGS_MAX_ADAM_GROUPS = 8

# name -> (restype, argtypes); must match include/hgs.h
_P = ctypes.POINTER
SIGNATURES = {
    "hgs_last_error": (ctypes.c_char_p, []),
    "hgs_abi_version": (ctypes.c_int, []),
    "hgs_device_info": (ctypes.c_int, [_P(c_i32), _P(c_i32), _P(c_i32)]),
    "hgs_kernel_launches": (c_i64, []),
    "hgs_graph_instantiate": (ctypes.c_int, [c_void_p, c_i32, _P(c_void_p)]),
    "hgs_graph_launch": (ctypes.c_int, [c_void_p, c_void_p]),
    "hgs_graph_exec_destroy": (ctypes.c_int, [c_void_p]),
    "hgs_preprocess": (ctypes.c_int, [c_void_p, c_i32, c_i32, _P(HGSGaussians), c_i32, _P(HGSProjected), c_void_p]),
    "hgs_tiles_scratch_bytes": (ctypes.c_size_t, [c_i64, c_i64, c_i32]),
    "hgs_build_tiles": (ctypes.c_int, [_P(HGSProjected), c_i64, _P(HGSTiles), c_void_p]),
    "hgs_blend_forward": (ctypes.c_int, [_P(HGSProjected), _P(HGSTiles), c_i32, c_i32, _P(HGSMeshLayer),
                                         _P(c_f64), c_i32, c_f64, _P(HGSBlendOut), c_void_p]),
    "hgs_render_depth": (ctypes.c_int, [_P(HGSProjected), _P(HGSTiles), c_i32, c_i32, c_void_p, c_void_p]),
    "hgs_blend_backward": (ctypes.c_int, [_P(HGSProjected), _P(HGSTiles), c_i32, c_i32, _P(HGSMeshLayer), _P(c_f64),
                                          c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i32,
                                          c_void_p]),
    "hgs_project_backward": (ctypes.c_int, [c_void_p, _P(HGSGaussians), _P(HGSProjected), c_void_p,
                                            _P(HGSGaussianGrads), c_f32, c_i32, c_void_p]),
    "hgs_raster_scratch_bytes": (ctypes.c_size_t, [c_i64, c_i64, c_i32, c_i32]),
    "hgs_rasterize_fragments": (ctypes.c_int, [c_void_p, c_i32, c_i32, _P(HGSMesh), _P(HGSFragments), c_void_p,
                                               ctypes.c_size_t, c_void_p]),
    "hgs_sample_texture": (ctypes.c_int, [c_void_p, c_i32, c_i32, c_void_p, c_void_p, c_i64, c_void_p, c_void_p]),
    "hgs_texture_backward": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_i32, c_i32, c_void_p, c_void_p]),
    "hgs_texture_backward_fixed": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_i32, c_i32, c_void_p,
                                                  c_void_p]),
    "hgs_fixed_to_float": (ctypes.c_int, [c_void_p, c_i64, c_void_p, c_i32, c_void_p]),
    "hgs_transmittance_mask": (ctypes.c_int, [c_void_p, c_i64, c_f64, c_i32, c_void_p, c_void_p]),
    "hgs_loss_scratch_bytes": (ctypes.c_size_t, [c_i32, c_i32]),
    "hgs_composite_loss": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_f64,
                                          c_i32, c_f64, c_f64, c_i32, _P(c_f64), c_f64, c_void_p, c_void_p,
                                          c_void_p, c_void_p, c_void_p, ctypes.c_size_t, c_void_p]),
    "hgs_adam_step": (ctypes.c_int, [_P(HGSAdamGroup), c_i32, c_i64, c_f32, c_f32, c_f32, c_f32, c_void_p]),
    "hgs_densify_scratch_bytes": (ctypes.c_size_t, [c_i64]),
    "hgs_densify_plan": (ctypes.c_int, [_P(HGSGaussians), c_void_p, c_void_p, c_f64, c_f64, c_f64, c_void_p,
                                        ctypes.c_size_t, _P(c_i64), c_void_p]),
    "hgs_densify_apply": (ctypes.c_int, [_P(HGSGaussians), _P(HGSGaussians), _P(HGSGaussians), c_void_p, c_void_p,
                                         _P(HGSGaussianBuf), _P(HGSGaussianBuf), _P(HGSGaussianBuf), c_void_p, c_void_p,
                                         c_void_p]),
    "hgs_densify_accumulate": (ctypes.c_int, [c_void_p, c_void_p, c_f64, c_i64, c_void_p, c_void_p, c_void_p]),
    "hgs_reset_opacity": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_f64, c_void_p]),
}


class HGSError(RuntimeError):
    pass


def build(verbose: bool = False) -> str:
    """Compile libhgs.so for sm_100a with nvcc (csrc/Makefile)."""
    jobs = str(max(1, min(8, os.cpu_count() or 1)))
    res = subprocess.run(["make", "-s", "-j", jobs, "-C", CSRC], capture_output=not verbose, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"building libhgs.so failed:\n{res.stdout}\n{res.stderr}")
    return LIB_PATH


def load():
    """Load libhgs.so and bind every exported symbol (raises if absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue  # reported by missing_symbols(); calling it raises AttributeError
            fn.restype = res
            fn.argtypes = args
        if lib.hgs_abi_version() != 1:
            raise RuntimeError("libhgs.so ABI version mismatch")
        _lib = lib
        return lib


def missing_symbols() -> list:
    lib = load()
    return [n for n in SIGNATURES if getattr(lib, n, None) is None]


def check(status: int, what: str = "") -> None:
    if status == HGS_OK:
        return
    msg = load().hgs_last_error().decode(errors="replace")
    if status == HGS_ERR_INVALID:
        raise ValueError(f"{what}: {msg}" if what else msg)
    raise HGSError(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()
