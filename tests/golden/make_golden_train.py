"""Golden trajectory of the reference's own per-iteration driver
(gsmesh/train/loop.py:147-255) on a tiny hybrid scene, with densification,
opacity reset and the texture window all active:

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden_train.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from gsmesh.config import TrainConfig  # noqa: E402
from gsmesh.scene import Camera, GaussianSet, TexturedMesh  # noqa: E402
from gsmesh.train.loop import train  # noqa: E402

from paper_2506_06988_b200 import synthetic as syn  # noqa: E402

CFG = dict(max_iters=12, warmup_iters=2, densify_until_iter=10, densify_from_iter=4, densify_interval=4,
           opacity_reset_interval=8, log_every=3, densify_grad_threshold=2e-5, seed=3)


def main():
    sc = syn.small_scene(seed=4, n=400, width=96, height=80, n_tris=120, tex=32)
    h = sc.gaussians
    gs = GaussianSet(h.centers, h.rotations, h.log_scales, h.logit_opacities, h.colors_dc, h.colors_rest)
    c0 = sc.cameras[0]
    cams = []
    for dx in (0.0, 0.05):
        w2c = np.asarray(c0.world_to_camera, dtype=np.float64).copy()
        w2c[0, 3] += dx
        cams.append(Camera(c0.fx, c0.fy, c0.cx, c0.cy, c0.width, c0.height, w2c, c0.near, c0.far))
    m = sc.mesh
    mesh = TexturedMesh(m.vertices, m.triangles, m.uvs, m.texture)
    rng = np.random.default_rng(11)
    images = [syn.q32(rng.uniform(0, 1, (80, 96, 3))) for _ in cams]
    cfg = TrainConfig.desk_scale(**CFG)
    res = train(cams, images, cfg, mesh=mesh, init=gs)
    out = {"images": np.stack(images), "cam_w2c": np.stack([np.asarray(c.world_to_camera) for c in cams]),
           "metrics_iter": np.array([r["iter"] for r in res.metrics[:-1]]),
           "metrics_n": np.array([r["n_gaussians"] for r in res.metrics[:-1]]),
           "metrics_total": np.array([r["total"] for r in res.metrics[:-1]]),
           "metrics_l1": np.array([r["l1"] for r in res.metrics[:-1]]),
           "final_mean_t": res.metrics[-1]["mean_T_on_mesh"], "final_n": res.metrics[-1]["n_gaussians"],
           "out_centers": res.gaussians.centers, "out_logits": res.gaussians.logit_opacities,
           "out_texture": res.mesh.texture}
    np.savez_compressed(os.path.join(HERE, "train_small.npz"), **out)
    print([(r["iter"], r["n_gaussians"], round(r.get("total", float("nan")), 6)) for r in res.metrics])


if __name__ == "__main__":
    main()
