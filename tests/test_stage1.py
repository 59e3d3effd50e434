"""Stage-1 consumers: render_depth / depth_kernel
(splat/render.py:316-324, kernels.py:163-202) and init_texture
(meshraster.py:206-245).  The oracle restatements are pinned against the
reference's own outputs (tests/golden/stage1.npz, make_golden_stage1.py);
the device path is checked against the same goldens.  Depth values are
copied, not computed, so the depth map must match bit for bit (NaN where
the reference has NaN); the texture after 5 fp32 Adam steps within 1e-5."""

import numpy as np
import pytest
import torch

from _util import golden_scene, load_golden
from oracle import oracle as orc

from paper_2506_06988_b200 import synthetic as syn


def _scene(d, tag):
    sub = {k[len(tag) + 1:]: v for k, v in d.items() if k.startswith(tag + "_")}
    gs, cam, _ = golden_scene(sub)
    return gs, cam


def _it_inputs(d):
    cams = []
    for i in range(2):
        fx, fy, cx, cy, w, h, near, far = d[f"it_cam{i}_intr"]
        cams.append(syn.HostCamera(fx, fy, cx, cy, int(w), int(h), d[f"it_cam{i}_w2c"], near, far))
    imgs = [d[f"it_img{i}"].astype(np.float64) for i in range(2)]
    return cams, imgs


def _same_depth(a, b):
    return np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])


@pytest.mark.parametrize("tag", ["sparse", "dense"])
def test_oracle_render_depth_matches_reference(tag):
    d = load_golden("stage1")
    gs, cam = _scene(d, tag)
    assert _same_depth(orc.render_depth(gs, cam), d[f"{tag}_depth"])


def test_oracle_init_texture_matches_reference():
    d = load_golden("stage1")
    cams, imgs = _it_inputs(d)
    tex = orc.init_texture(d["it_vertices"].astype(np.float64), d["it_triangles"], d["it_uvs"].astype(np.float64),
                           d["it_texture_in"], imgs, cams, iters=5, lr=0.05)
    assert np.abs(tex - d["it_texture_out"]).max() < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["sparse", "dense"])
def test_render_depth_matches_reference(tag, cuda_device):
    import paper_2506_06988_b200 as hgs
    d = load_golden("stage1")
    gs, cam = _scene(d, tag)
    out = hgs.render_depth(hgs.GaussianSet.from_any(gs), hgs.Camera.from_any(cam))
    assert out.dtype == torch.float64 and tuple(out.shape) == d[f"{tag}_depth"].shape
    assert _same_depth(out.cpu().numpy(), d[f"{tag}_depth"])


@pytest.mark.gpu
def test_render_depth_c2_matches_oracle(cuda_device):
    """Larger case against the oracle restatement (pinned above)."""
    import paper_2506_06988_b200 as hgs
    sc = syn.small_scene(seed=5, n=20000, width=160, height=128)
    cam = sc.cameras[0]
    ref = orc.render_depth(sc.gaussians, cam)
    out = hgs.render_depth(hgs.GaussianSet.from_any(sc.gaussians), hgs.Camera.from_any(cam)).cpu().numpy()
    assert np.isfinite(ref).sum() > 1000
    assert _same_depth(out, ref)


@pytest.mark.gpu
def test_init_texture_matches_reference(cuda_device):
    import paper_2506_06988_b200 as hgs
    from paper_2506_06988_b200.meshraster import init_texture
    d = load_golden("stage1")
    cams, imgs = _it_inputs(d)
    mesh = hgs.TexturedMesh(d["it_vertices"].astype(np.float64), d["it_triangles"], d["it_uvs"].astype(np.float64),
                            d["it_texture_in"].astype(np.float64))
    out = init_texture(mesh, imgs, [hgs.Camera.from_any(c) for c in cams], iters=5, lr=0.05)
    assert np.abs(out.texture.cpu().numpy() - d["it_texture_out"]).max() < 1e-5
    const = init_texture(mesh, imgs, cams, mode="constant")
    assert bool((const.texture == 0.5).all())
    with pytest.raises(ValueError):
        init_texture(mesh, imgs, cams, mode="bogus")
    with pytest.raises(ValueError):
        init_texture(mesh, imgs[:1], cams)
