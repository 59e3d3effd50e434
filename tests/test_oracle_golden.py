"""Pins the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from _util import assert_close, golden_scene, load_golden
from oracle import oracle as orc

CASES = ["small_sh0", "small_sh1", "c1"]


@pytest.fixture(scope="module", params=CASES)
def case(request):
    d = load_golden(request.param)
    gs, cam, mesh = golden_scene(d)
    return request.param, d, gs, cam, mesh


def test_project_matches_reference(case):
    name, d, gs, cam, _ = case
    p = orc.project(gs, cam)
    assert np.array_equal(p.kept, d["p_kept"]), "kept set differs"
    for k in ("mean2d", "depth", "cov2d", "conic", "alpha", "color", "radius", "t_cam", "color_pre"):
        assert_close(getattr(p, k), d["p_" + k], atol=1e-12, rtol=1e-12, what=k)
    if "p_view_dir" in d:
        assert_close(p.view_dir, d["p_view_dir"], atol=1e-13, what="view_dir")


def test_tiles_bit_exact(case):
    name, d, gs, cam, _ = case
    p = orc.project(gs, cam)
    t = orc.build_tiles(p, cam.width, cam.height)
    assert np.array_equal(t.tile_starts, d["t_starts"]), "tile_starts differ"
    assert np.array_equal(t.entries, d["t_entries"]), "entry order differs"


def test_forward_matches_reference(case):
    name, d, gs, cam, mesh = case
    p = orc.project(gs, cam)
    t = orc.build_tiles(p, cam.width, cam.height)
    layer = None
    if mesh is not None:
        fr = orc.rasterize_fragments(mesh.vertices, mesh.triangles, mesh.uvs, cam)
        assert np.array_equal(fr.triangle_id, d["f_tri"]), "triangle ids differ"
        assert_close(fr.depth, d["f_depth"], atol=0, rtol=1e-15, what="frag depth")
        assert_close(fr.uv, d["f_uv"], atol=1e-15, what="uv")
        if "f_bary" in d:
            assert_close(fr.bary, d["f_bary"], atol=1e-15, what="bary")
        mc = orc.sample_texture(mesh.texture, fr.uv, fr.valid)
        if "f_color" in d:
            assert_close(mc, d["f_color"], atol=1e-15, what="mesh colour")
        layer = orc.Mesh(mc, fr.depth, fr.triangle_id)
    color, depth, tt, last = orc.rasterize_forward(p, t, cam.width, cam.height, d["bg"], layer)
    assert np.array_equal(last, d["r_last"]), "last-consumed index differs"
    assert_close(color, d["r_color"], atol=1e-12, what="color")
    assert_close(tt, d["r_t"], atol=1e-12, what="T")
    assert_close(depth, d["r_depth"], atol=1e-10, what="depth")
    if "r0_color" in d:
        color, depth, tt, last = orc.rasterize_forward(p, t, cam.width, cam.height, d["bg"], None)
        assert np.array_equal(last, d["r0_last"])
        assert_close(color, d["r0_color"], atol=1e-12, what="color (no mesh)")
        assert_close(tt, d["r0_t"], atol=1e-12, what="T (no mesh)")


def _ctx(d, gs, cam, mesh, with_mesh=True):
    layer = None
    if with_mesh and mesh is not None:
        fr = orc.rasterize_fragments(mesh.vertices, mesh.triangles, mesh.uvs, cam)
        layer = orc.Mesh(orc.sample_texture(mesh.texture, fr.uv, fr.valid), fr.depth, fr.triangle_id)
    return orc.render(gs, cam, d["bg"], layer)


def test_backward_matches_reference(case):
    name, d, gs, cam, mesh = case
    if "b_centers" not in d:
        pytest.skip("fixture has no backward vectors")
    for with_mesh, pre in ((True, "b_"), (False, "b0_")):
        *_, ctx = _ctx(d, gs, cam, mesh, with_mesh)
        g = orc.backward(ctx, d["b_grad_color"], d["b_grad_t"])
        for k in ("centers", "rotations", "log_scales", "logit_opacities", "colors_dc"):
            ref = d[pre + k]
            assert_close(getattr(g, k), ref, atol=1e-9, rtol=1e-9, what=pre + k)
        if with_mesh:
            assert_close(g.densify_norm, d["b_densify_norm"], atol=1e-9, rtol=1e-9, what="densify_norm")
            assert np.array_equal(g.visible, d["b_visible"])
            if "b_colors_rest" in d:
                assert_close(g.colors_rest, d["b_colors_rest"], atol=1e-9, rtol=1e-9, what="colors_rest")
            if "b_mesh_color" in d:
                assert_close(g.mesh_color, d["b_mesh_color"], atol=1e-15, what="mesh_color")


def test_texture_backward_matches_reference(case):
    name, d, gs, cam, mesh = case
    if "tb_grad" not in d:
        pytest.skip("no texture-backward vectors")
    fr = orc.rasterize_fragments(mesh.vertices, mesh.triangles, mesh.uvs, cam)
    g = orc.texture_backward(fr, d["tb_grad"], mesh.texture.shape[:2])
    assert_close(g, d["tb_out"], atol=1e-12, what="texture grad")


class _Cfg:
    """TrainConfig.desk_scale(texture_weight=0.1) fields used by composite_loss."""
    dssim_weight = 0.2
    zero_dssim_after_densify = False
    densify_until_iter = 1500
    warmup_iters = 300
    texture_weight = 0.1
    mask_sharpness = 20.0
    mask_variant = "sigmoid"
    lr_position, lr_position_final, max_iters = 1.6e-4, 1.6e-6, 3000
    lr_rotation, lr_scale, lr_opacity, lr_color, lr_texture = 1e-3, 5e-3, 0.05, 2.5e-3, 1e-2


def test_loss_and_train_step_match_reference():
    d = load_golden("small_sh0")
    gs, cam, mesh = golden_scene(d)
    color, depth, tt, ctx = _ctx(d, gs, cam, mesh, True)
    layer = ctx["mesh"]
    cfg = _Cfg()
    it = cfg.warmup_iters + 1
    bd, gih, gim, gtt = orc.composite_loss(d["l_target"], color, layer.color, layer.valid, tt, it, cfg)
    ref = d["l_values"]
    got = np.array([bd["l1"], bd["dssim"], bd["l_c"], bd["l_t"], bd["total"], bd["mean_T_on_mesh"]])
    assert_close(got, ref, atol=1e-12, rtol=1e-10, what="loss values")
    assert_close(gih, d["l_grad_ih"], atol=1e-15, rtol=1e-9, what="grad_ih")
    assert_close(gim, d["l_grad_im"], atol=1e-15, rtol=1e-9, what="grad_im")
    assert_close(gtt, d["l_grad_t"], atol=1e-15, rtol=1e-9, what="grad_t")
    g = orc.backward(ctx, gih, gtt)
    lr_pos = float(np.exp(np.log(cfg.lr_position) * (1 - it / cfg.max_iters) + np.log(cfg.lr_position_final) * (it / cfg.max_iters)))
    assert abs(lr_pos - d["a_pos_lr"][0]) < 1e-18
    lrs = {"centers": lr_pos, "rotations": cfg.lr_rotation, "log_scales": cfg.lr_scale,
           "logit_opacities": cfg.lr_opacity, "colors_dc": cfg.lr_color}
    for k, lr in lrs.items():
        p = np.ascontiguousarray(getattr(gs, k), dtype=np.float64).copy()
        m, v = np.zeros_like(p), np.zeros_like(p)
        orc.adam_step(p, m, v, getattr(g, k), lr, 1)
        if k == "rotations":
            p /= np.linalg.norm(p, axis=1, keepdims=True)
        assert_close(p, d["a_" + k], atol=1e-12, what="adam " + k)
    gtex = orc.texture_backward(orc.rasterize_fragments(mesh.vertices, mesh.triangles, mesh.uvs, cam),
                                g.mesh_color + gim, mesh.texture.shape[:2])
    assert_close(gtex, d["a_grad_texture"], atol=1e-15, rtol=1e-9, what="texture grad")
    tex = np.ascontiguousarray(mesh.texture, dtype=np.float64).copy()
    orc.adam_step(tex, np.zeros_like(tex), np.zeros_like(tex), gtex, cfg.lr_texture, 1)
    np.clip(tex, 0.0, 1.0, out=tex)
    assert_close(tex, d["a_texture"], atol=1e-12, what="texture after step")


def test_edge_cases():
    d = load_golden("edge")
    gs = type("G", (), {})()
    gs.centers = np.array([[0.1, 0, 3.0], [-0.1, 0, 3.0], [0, 0.1, 3.0]])
    gs.rotations = np.tile([1.0, 0, 0, 0], (3, 1))
    gs.log_scales = np.full((3, 3), -1.0)
    gs.logit_opacities = np.zeros(3)
    gs.colors_dc = np.zeros((3, 3))
    gs.colors_rest = None
    from paper_2506_06988_b200.synthetic import HostCamera
    cam = HostCamera(60.0, 60.0, 32.0, 32.0, 64, 64, np.eye(4), 0.05, 100.0)
    p = orc.project(gs, cam)
    t = orc.build_tiles(p, 64, 64)
    assert np.array_equal(t.tile_starts, d["eq_starts"]) and np.array_equal(t.entries, d["eq_entries"])
    color, depth, tt, _ = orc.render(gs, cam, (0.2, 0.4, 0.6))
    assert_close(color, d["eq_color"], atol=1e-14, what="eq color")
    verts = np.array([[-1.0, -1.0, 2.0], [1.0, -1.0, 2.0], [1.0, 1.0, 2.0], [-1.0, 1.0, 2.0]])
    tris = np.array([[0, 1, 2], [0, 2, 3]], dtype=np.int32)
    uvs = np.array([[[0, 0], [1, 0], [1, 1]], [[0, 0], [1, 1], [0, 1]]], dtype=np.float64)
    cam32 = HostCamera(32.0, 32.0, 16.0, 16.0, 32, 32, np.eye(4), 0.05, 100.0)
    fr = orc.rasterize_fragments(verts, tris, uvs, cam32)
    assert np.array_equal(fr.triangle_id, d["se_tri"])
    assert_close(fr.bary, d["se_bary"], atol=0, what="shared-edge bary")
    cam_b = HostCamera(30.0, 30.0, 16.0, 12.0, 32, 24, np.eye(4), 0.05, 100.0)
    fr = orc.rasterize_fragments(verts * np.array([3.0, 3.0, 1.0]), tris, uvs, cam_b)
    assert np.array_equal(fr.triangle_id, d["fs_tri"])
    cam48 = HostCamera(43.2, 43.2, 24.0, 24.0, 48, 48, np.eye(4), 0.05, 100.0)
    fr = orc.rasterize_fragments(d["soup_v"].astype(np.float64), d["soup_f"], None, cam48)
    assert np.array_equal(fr.triangle_id, d["soup_tri"])
    assert_close(fr.depth, d["soup_depth"], atol=0, what="soup depth")
    assert_close(fr.bary, d["soup_bary"], atol=0, what="soup bary")


def test_oracle_threads_do_not_change_results():
    d = load_golden("c1")
    gs, cam, mesh = golden_scene(d)
    p = orc.project(gs, cam, nthreads=1)
    t1 = orc.build_tiles(p, cam.width, cam.height, nthreads=1)
    t4 = orc.build_tiles(p, cam.width, cam.height, nthreads=4)
    assert np.array_equal(t1.entries, t4.entries)
    a = orc.rasterize_forward(p, t1, cam.width, cam.height, d["bg"], None, nthreads=1)
    b = orc.rasterize_forward(p, t1, cam.width, cam.height, d["bg"], None, nthreads=4)
    for x, y in zip(a, b):
        assert np.array_equal(x, y, equal_nan=True)


# ---- at scale: reference-written c2 (forward + backward) and c3 (forward)
# fixtures (tests/golden/make_golden_scale.py): integer outputs as SHA-256
# digests (bit-exact), floats at fixed sampled pixels / rows plus sums.

def _digest(a):
    import hashlib
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_oracle_matches_reference_at_scale(cfg):
    import hashlib
    from paper_2506_06988_b200 import synthetic as syn
    d = load_golden(f"scale_{cfg}")
    sc = syn.make_config(cfg, seed=0)
    g, m = sc.gaussians, sc.mesh
    h = hashlib.sha256()
    for p in (g.centers, g.rotations, g.log_scales, g.logit_opacities, g.colors_dc, m.vertices, m.triangles, m.uvs,
              m.texture):
        h.update(np.ascontiguousarray(p, dtype=np.float64 if p.dtype.kind == "f" else np.int64).tobytes())
    assert h.hexdigest() == str(d["input_sha"]), "synthetic generator no longer reproduces the fixture's inputs"
    cam = sc.cameras[0]
    fr = orc.rasterize_fragments(m.vertices, m.triangles, m.uvs, cam)
    assert _digest(fr.triangle_id.astype(np.int32)) == str(d["sha_tri"]), "triangle ids differ"
    mc = orc.sample_texture(m.texture, fr.uv, fr.valid)
    color, depth, tt, octx = orc.render(g, cam, (0.0, 0.0, 0.0), orc.Mesh(mc, fr.depth, fr.triangle_id))
    assert len(octx["tiles"].entries) == int(d["k_entries"])
    assert _digest(octx["tiles"].tile_starts.astype(np.int64)) == str(d["sha_tile_starts"]), "tile_starts differ"
    assert _digest(octx["tiles"].entries.astype(np.int32)) == str(d["sha_entries"]), "entry order differs"
    assert _digest(octx["last"].astype(np.int32)) == str(d["sha_last"]), "last-consumed indices differ"
    pi = d["pix_idx"]
    assert_close(color.reshape(-1, 3)[pi], d["color_s"], atol=1e-12, what="color")
    assert_close(tt.reshape(-1)[pi], d["t_s"], atol=1e-12, what="T")
    assert_close(depth.reshape(-1)[pi], d["depth_s"], atol=1e-10, what="depth")
    assert_close(color.sum(axis=(0, 1)), d["color_sum"], atol=1e-8, rtol=1e-12, what="colour sum")
    assert int(np.isnan(depth).sum()) == int(d["depth_nan"])
    if "row_idx" in d:
        rng = np.random.default_rng(9)
        gc = syn.q32(rng.uniform(-1, 1, (cam.height, cam.width, 3)))
        gt = syn.q32(rng.uniform(-1, 1, (cam.height, cam.width)))
        og = orc.backward(octx, gc, gt)
        ri = d["row_idx"]
        for k in ("centers", "rotations", "log_scales", "logit_opacities", "colors_dc"):
            a = np.asarray(getattr(og, k))
            assert_close(a[ri], d["g_" + k], atol=1e-9, rtol=1e-9, what=k)
            assert abs(np.abs(a).sum() - float(d["gsum_" + k])) <= 1e-9 * float(d["gsum_" + k]), k
