"""The reference's per-iteration driver (loop.train) on the device vs the
reference's own trajectory (tests/golden/train_small.npz, written by
tests/golden/make_golden_train.py): same view order, densification events
and Gaussian counts, losses within 1e-4 relative; checkpoints in the
reference's layout."""

import os

import numpy as np
import pytest
import torch

from _util import load_golden

pytestmark = pytest.mark.gpu


def _setup():
    import paper_2506_06988_b200 as hgs
    from paper_2506_06988_b200 import synthetic as syn
    from paper_2506_06988_b200.config import TrainConfig
    d = load_golden("train_small")
    sc = syn.small_scene(seed=4, n=400, width=96, height=80, n_tris=120, tex=32)
    c0 = sc.cameras[0]
    cams = [hgs.Camera(c0.fx, c0.fy, c0.cx, c0.cy, c0.width, c0.height, w, c0.near, c0.far) for w in d["cam_w2c"]]
    cfg = TrainConfig.desk_scale(max_iters=12, warmup_iters=2, densify_until_iter=10, densify_from_iter=4,
                                 densify_interval=4, opacity_reset_interval=8, log_every=3,
                                 densify_grad_threshold=2e-5, seed=3)
    return d, hgs.GaussianSet.from_any(sc.gaussians), hgs.TexturedMesh.from_any(sc.mesh), cams, cfg


def test_train_driver_matches_reference_trajectory(cuda_device, tmp_path):
    from paper_2506_06988_b200 import fileio
    from paper_2506_06988_b200.loop import train
    d, gs, mesh, cams, cfg = _setup()
    res = train(cams, list(d["images"]), cfg, mesh=mesh, init=gs, out_dir=tmp_path)
    got_iter = [r["iter"] for r in res.metrics[:-1]]
    got_n = [r["n_gaussians"] for r in res.metrics[:-1]]
    assert got_iter == list(d["metrics_iter"])
    assert got_n == list(d["metrics_n"]), (got_n, list(d["metrics_n"]))
    tot = np.array([r["total"] for r in res.metrics[:-1]])
    assert np.allclose(tot, d["metrics_total"], rtol=1e-4, atol=1e-6), (tot, d["metrics_total"])
    assert res.final["n_gaussians"] == int(d["final_n"])
    assert abs(res.final["mean_T_on_mesh"] - float(d["final_mean_t"])) < 1e-4
    c = res.gaussians.centers.detach().cpu().numpy().astype(np.float64)
    assert c.shape == d["out_centers"].shape
    assert np.abs(c - d["out_centers"]).max() < 1e-3  # a few lr-sized Adam steps apart at most
    tex = res.mesh.texture.detach().cpu().numpy().astype(np.float64)
    assert np.abs(tex - d["out_texture"]).max() < 1e-3
    for f in ("gaussians.ply", "mesh.obj", "mesh.mtl", "mesh_texture.png", "config.json", "metrics.jsonl",
              "optimizer_state.bin"):
        assert (tmp_path / f).exists(), f
    g2 = fileio.load_gaussians(tmp_path / "gaussians.ply")
    assert len(g2) == res.final["n_gaussians"]
    st = fileio.load_optimizer_state(tmp_path / "optimizer_state.bin")
    assert st["step"] == 12
