"""Golden vectors for the Stage-1 consumers, produced by the
REFERENCE: render_depth (splat/render.py:316-324, depth_kernel
kernels.py:163-202) and init_texture (meshraster.py:206-245).  Build
container only:

    PYTHONPATH=/root/reference/pkg/src:/root/repo NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_golden_stage1.py

Writes tests/golden/stage1.npz (inputs fp32-quantised, outputs fp64)."""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import pack_inputs, ref_cam, ref_gs  # noqa: E402  (sets up the reference path)

from gsmesh.meshraster import init_texture  # noqa: E402
from gsmesh.scene import TexturedMesh  # noqa: E402
from gsmesh.splat import render_depth  # noqa: E402

from paper_2506_06988_b200 import synthetic as syn  # noqa: E402


def main():
    d = {}
    # render_depth: a sparse and a dense scene (same camera)
    for tag, n in (("sparse", 300), ("dense", 3000)):
        sc = syn.small_scene(seed=3, n=n)
        gs, cam = ref_gs(sc.gaussians), ref_cam(sc.cameras[0])
        dd = {}
        pack_inputs(dd, sc.gaussians, sc.cameras[0], None)
        for k, v in dd.items():
            d[f"{tag}_{k}"] = v
        d[f"{tag}_depth"] = render_depth(gs, cam)
    # init_texture: 5 Adam steps over two views of the small wall
    sc = syn.small_scene(seed=4)
    cams = [sc.cameras[0], syn.look_at((0.8, 0.1, -0.3), (0.4, 0.0, 5.0), width=96, height=80)]
    m = sc.mesh
    rng = np.random.default_rng(11)
    imgs = [rng.uniform(0, 1, (c.height, c.width, 3)).astype(np.float32).astype(np.float64) for c in cams]
    mesh = TexturedMesh(m.vertices.astype(np.float64), m.triangles, m.uvs.astype(np.float64),
                        m.texture.astype(np.float64))
    out = init_texture(mesh, imgs, [ref_cam(c) for c in cams], iters=5, mode="optimized", lr=0.05)
    d["it_vertices"] = m.vertices.astype(np.float32)
    d["it_triangles"] = m.triangles.astype(np.int32)
    d["it_uvs"] = m.uvs.astype(np.float32)
    d["it_texture_in"] = m.texture.astype(np.float32)
    for i, c in enumerate(cams):
        d[f"it_cam{i}_intr"] = np.array([c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.near, c.far])
        d[f"it_cam{i}_w2c"] = np.asarray(c.world_to_camera)
        d[f"it_img{i}"] = imgs[i].astype(np.float32)
    d["it_texture_out"] = out.texture
    np.savez_compressed(os.path.join(HERE, "stage1.npz"), **d)
    print({k: v.shape for k, v in d.items() if k.endswith("depth") or k.startswith("it_texture")},
          "finite depth px:", [int(np.isfinite(d[f"{t}_depth"]).sum()) for t in ("sparse", "dense")])


if __name__ == "__main__":
    main()
