"""Golden files for the on-disk formats, written by the reference's own
gsmesh.fileio / train.loop writers (tests/golden/io/):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden_io.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from gsmesh import fileio  # noqa: E402
from gsmesh.scene import Camera, GaussianSet, TexturedMesh  # noqa: E402
from gsmesh.train.adam import Adam  # noqa: E402
from gsmesh.train.loop import _save_optimizer_state  # noqa: E402


def q32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(5)
    n = 40
    gs = GaussianSet(q32(rng.normal(0, 1, (n, 3))), q32(rng.normal(0, 1, (n, 4))), q32(rng.uniform(-5, -2, (n, 3))),
                     q32(rng.uniform(-3, 2, n)), q32(rng.uniform(-1, 1, (n, 3))), q32(rng.uniform(-.2, .2, (n, 3, 3))))
    fileio.save_gaussians(gs, os.path.join(OUT, "gaussians_sh1.ply"))
    verts = q32(rng.uniform(-1, 1, (12, 3)))
    tris = rng.integers(0, 12, (10, 3)).astype(np.int32)
    uvs = q32(rng.uniform(0, 1, (10, 3, 2)))
    tex = np.round(rng.uniform(0, 1, (8, 6, 3)) * 255) / 255
    fileio.save_mesh(TexturedMesh(verts, tris, uvs, tex), os.path.join(OUT, "mesh.obj"))
    m2 = fileio.load_mesh(os.path.join(OUT, "mesh.obj"))
    np.savez(os.path.join(OUT, "mesh_loaded.npz"), vertices=m2.vertices, triangles=m2.triangles, uvs=m2.uvs,
             texture=m2.texture)
    R = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    W = np.eye(4)
    W[:3, :3] = R
    W[:3, 3] = [0.1, -0.2, 2.0]
    fileio.save_cameras([Camera(120.0, 121.0, 64.0, 48.0, 128, 96, W, 0.05, 50.0)], os.path.join(OUT, "cameras.json"))
    params = {"centers": q32(rng.normal(0, 1, (n, 3))), "logit_opacities": q32(rng.normal(0, 1, n)),
              "colors_rest": q32(rng.normal(0, 1, (n, 3, 3)))}
    opt = Adam({k: v.copy() for k, v in params.items()}, {k: 1e-3 for k in params})
    for k in params:
        opt.m[k] = q32(rng.normal(0, 1e-3, params[k].shape))
        opt.v[k] = q32(rng.uniform(0, 1e-6, params[k].shape))
    opt.step_count = 17
    _save_optimizer_state(opt, os.path.join(OUT, "optimizer_state.bin"))
    print(sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
