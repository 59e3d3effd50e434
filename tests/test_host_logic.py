"""Host-side logic of the device package that runs without a GPU: camera
validation and derived fields, configuration, view sharding, and the
no-fallback contract."""

import numpy as np
import pytest
import torch

from paper_2506_06988_b200 import scene
from paper_2506_06988_b200.config import ConfigError, TrainConfig
from paper_2506_06988_b200.train import shard_views


def test_camera_validation_matches_reference_rules():
    with pytest.raises(scene.SceneError):
        scene.Camera(1, 1, 0, 0, 4, 4, np.eye(3))
    bad = np.eye(4)
    bad[0, 0] = 1.01
    with pytest.raises(scene.SceneError):
        scene.Camera(1, 1, 0, 0, 4, 4, bad)
    with pytest.raises(scene.SceneError):
        scene.Camera(1, 1, 0, 0, 4, 4, np.eye(4), near=1.0, far=0.5)
    with pytest.raises(scene.SceneError):
        scene.Camera(1, 1, 0, 0, 0, 4, np.eye(4))
    # small defects are repaired by SVD (scene.py:170-174)
    w = np.eye(4)
    w[0, 1] = 5e-5
    c = scene.Camera(1, 1, 0, 0, 4, 4, w)
    R = c.rotation
    assert np.abs(R @ R.T - np.eye(3)).max() < 1e-12


def test_camera_struct_derived_fields():
    th = 0.3
    w2c = np.eye(4)
    w2c[:3, :3] = [[np.cos(th), 0, np.sin(th)], [0, 1, 0], [-np.sin(th), 0, np.cos(th)]]
    w2c[:3, 3] = [0.1, -0.2, 0.3]
    c = scene.Camera(100.0, 90.0, 50.0, 40.0, 100, 80, w2c, 0.05, 50.0)
    s = scene.camera_struct(c)
    R, t = c.rotation, c.translation
    assert np.array_equal(np.array(s.center[:]), -R.T @ t)
    assert s.limx == 1.3 * (100 / (2.0 * 100.0)) and s.limy == 1.3 * (80 / (2.0 * 90.0))
    assert (s.width, s.height) == (100, 80)


def test_config_validation():
    TrainConfig()
    with pytest.raises(ConfigError):
        TrainConfig(warmup_iters=10, densify_until_iter=5)
    with pytest.raises(ConfigError):
        TrainConfig(mask_variant="bogus")
    d = TrainConfig.desk_scale()
    assert d.max_iters == 3000 and d.warmup_iters == 300


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (10, 4), (3, 8)])
def test_shard_views_partitions_the_batch(n, world):
    parts = [shard_views(n, r, world) for r in range(world)]
    flat = [v for p in parts for v in p]
    assert flat == list(range(n))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        scene.GaussianSet(np.zeros((1, 3)), np.array([[1.0, 0, 0, 0]]), np.zeros((1, 3)), np.zeros(1),
                          np.zeros((1, 3)))
