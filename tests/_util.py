"""Shared test helpers: golden fixture loading and host-scene conversion."""

import os

import numpy as np

from paper_2506_06988_b200 import synthetic as syn

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def golden_scene(d):
    f64 = lambda k: d[k].astype(np.float64)  # noqa: E731
    gs = syn.HostGaussians(f64("g_centers"), f64("g_rotations"), f64("g_log_scales"), f64("g_logits"), f64("g_dc"),
                           f64("g_rest") if "g_rest" in d else None)
    fx, fy, cx, cy, w, h, near, far = d["cam_intr"]
    cam = syn.HostCamera(fx, fy, cx, cy, int(w), int(h), d["cam_w2c"], near, far)
    mesh = None
    if "m_vertices" in d:
        mesh = syn.HostMesh(f64("m_vertices"), d["m_triangles"], f64("m_uvs"), f64("m_texture"))
    return gs, cam, mesh


def assert_close(a, b, atol, rtol=0.0, what=""):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, f"{what}: shape {a.shape} != {b.shape}"
    nan_a, nan_b = np.isnan(a), np.isnan(b)
    assert np.array_equal(nan_a, nan_b), f"{what}: NaN pattern differs ({(nan_a != nan_b).sum()} elements)"
    inf_a, inf_b = np.isinf(a), np.isinf(b)
    assert np.array_equal(inf_a, inf_b), f"{what}: inf pattern differs"
    m = ~(nan_a | inf_a)
    if m.any():
        err = np.abs(a[m] - b[m])
        tol = atol + rtol * np.abs(b[m])
        bad = err > tol
        assert not bad.any(), f"{what}: {bad.sum()} / {m.sum()} elements off, max err {err.max():.3e}"


def grad_close(a, b, atol=1e-4, scale_tol=1e-4, what=""):
    """Gradient parity: absolute 1e-4 and scale-normalised
    |a-b| / max(1, |b|) <= 1e-4."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, f"{what}: shape {a.shape} != {b.shape}"
    err = np.abs(a - b)
    assert err.max(initial=0.0) <= atol, f"{what}: max abs err {err.max():.3e}"
    norm = err / np.maximum(1.0, np.abs(b))
    assert norm.max(initial=0.0) <= scale_tol, f"{what}: max normalised err {norm.max():.3e}"
