"""Generate golden vectors by running the REFERENCE (gsmesh, /root/reference)
on seeded fp32-quantised inputs.  Run in the build container only:

    PYTHONPATH=/root/reference/pkg/src:/root/repo NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz (inputs stored as float32 -- exact, they are
fp32-quantised -- outputs as produced by the reference, float64/int).
The GPU box never needs /root/reference: tests read these files.
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
from gsmesh.meshraster import (rasterize_fragments, sample_texture, texture_backward)  # noqa: E402
from gsmesh.scene import Camera, GaussianSet, TexturedMesh  # noqa: E402
from gsmesh.splat import MeshLayer, build_tiles, project, rasterize_backward, render  # noqa: E402
from gsmesh.train.adam import Adam, exponential_lr  # noqa: E402
from gsmesh.train.losses import composite_loss  # noqa: E402

from paper_2506_06988_b200 import synthetic as syn  # noqa: E402


def ref_gs(h: syn.HostGaussians) -> GaussianSet:
    return GaussianSet(h.centers, h.rotations, h.log_scales, h.logit_opacities, h.colors_dc, h.colors_rest)


def ref_cam(c: syn.HostCamera) -> Camera:
    return Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.world_to_camera, c.near, c.far)


def pack_inputs(d, gs, cam, mesh):
    d["g_centers"] = gs.centers.astype(np.float32)
    d["g_rotations"] = gs.rotations.astype(np.float32)
    d["g_log_scales"] = gs.log_scales.astype(np.float32)
    d["g_logits"] = gs.logit_opacities.astype(np.float32)
    d["g_dc"] = gs.colors_dc.astype(np.float32)
    if gs.colors_rest is not None:
        d["g_rest"] = gs.colors_rest.astype(np.float32)
    d["cam_intr"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, cam.near, cam.far])
    d["cam_w2c"] = np.asarray(cam.world_to_camera)
    if mesh is not None:
        d["m_vertices"] = mesh.vertices.astype(np.float32)
        d["m_triangles"] = mesh.triangles.astype(np.int32)
        d["m_uvs"] = mesh.uvs.astype(np.float32)
        d["m_texture"] = mesh.texture.astype(np.float32)


def run_case(name, scene: syn.Scene, bg=(0.1, 0.2, 0.3), seed=7, backward=True, train=True, lean=False):
    rng = np.random.default_rng(seed)
    hcam = scene.cameras[0]
    gs, cam = ref_gs(scene.gaussians), ref_cam(hcam)
    d = {}
    pack_inputs(d, scene.gaussians, hcam, scene.mesh)
    W, H = cam.width, cam.height
    proj = project(gs, cam)
    for k in ("kept", "mean2d", "depth", "cov2d", "conic", "alpha", "color", "radius", "t_cam", "color_pre"):
        d["p_" + k] = getattr(proj, k)
    if proj.view_dir is not None:
        d["p_view_dir"], d["p_view_dist"] = proj.view_dir, proj.view_dist
    tiles = build_tiles(proj, W, H)
    d["t_starts"], d["t_entries"] = tiles.tile_starts, tiles.entries
    layer = None
    if scene.mesh is not None:
        m = scene.mesh
        rm = TexturedMesh(m.vertices, m.triangles, m.uvs, m.texture)
        fr = rasterize_fragments(rm, cam)
        d["f_tri"], d["f_bary"], d["f_depth"], d["f_uv"] = fr.triangle_id, fr.bary, fr.depth, fr.uv
        mc = sample_texture(rm.texture, fr.uv, fr.valid)
        d["f_color"] = mc
        layer = MeshLayer(color=mc, depth=fr.depth, triangle_id=fr.triangle_id)
    d["bg"] = np.asarray(bg, dtype=np.float64)
    out, ctx = render(gs, cam, background=bg, mesh=layer)
    d["r_color"], d["r_depth"], d["r_t"], d["r_last"] = out.color, out.depth, out.transmittance, ctx.last_consumed
    out0, ctx0 = render(gs, cam, background=bg, mesh=None)
    d["r0_color"], d["r0_depth"], d["r0_t"], d["r0_last"] = out0.color, out0.depth, out0.transmittance, ctx0.last_consumed
    if backward:
        gc = syn.q32(rng.uniform(-1, 1, (H, W, 3)))
        gt = syn.q32(rng.uniform(-1, 1, (H, W)))
        d["b_grad_color"], d["b_grad_t"] = gc, gt
        gr = rasterize_backward(ctx, gc, grad_transmittance=gt)
        for k in ("centers", "rotations", "log_scales", "logit_opacities", "colors_dc", "densify_norm", "visible"):
            d["b_" + k] = getattr(gr, k)
        if gr.colors_rest is not None:
            d["b_colors_rest"] = gr.colors_rest
        if gr.mesh_color is not None:
            d["b_mesh_color"] = gr.mesh_color
        gr0 = rasterize_backward(ctx0, gc, grad_transmittance=gt)
        for k in ("centers", "rotations", "log_scales", "logit_opacities", "colors_dc"):
            d["b0_" + k] = getattr(gr0, k)
        if scene.mesh is not None:
            gimg = syn.q32(rng.uniform(-1, 1, (H, W, 3)))
            d["tb_grad"] = gimg
            d["tb_out"] = texture_backward(fr, gimg, scene.mesh.texture.shape[:2])
    if train and scene.mesh is not None:
        # one reference training iteration with the texture window active
        cfg = TrainConfig.desk_scale(texture_weight=0.1)
        it = cfg.warmup_iters + 1
        target = syn.q32(rng.uniform(0, 1, (H, W, 3)))
        d["l_target"] = target
        bd, gih, gim, gtt = composite_loss(target, out.color, layer.color, layer.valid, out.transmittance, it, cfg)
        d["l_values"] = np.array([bd.l1, bd.dssim, bd.l_c, bd.l_t, bd.total, bd.mean_t_on_mesh])
        d["l_grad_ih"], d["l_grad_im"], d["l_grad_t"] = gih, gim, gtt
        grads = rasterize_backward(ctx, gih, grad_transmittance=gtt)
        params = {"centers": gs.centers.copy(), "rotations": gs.rotations.copy(), "log_scales": gs.log_scales.copy(),
                  "logit_opacities": gs.logit_opacities.copy(), "colors_dc": gs.colors_dc.copy()}
        lrs = {"centers": cfg.lr_position, "rotations": cfg.lr_rotation, "log_scales": cfg.lr_scale,
               "logit_opacities": cfg.lr_opacity, "colors_dc": cfg.lr_color}
        opt = Adam(params, lrs)
        opt.lrs["centers"] = exponential_lr(cfg.lr_position, cfg.lr_position_final, cfg.max_iters)(it)
        opt.step({k: getattr(grads, k) for k in params})
        q = opt.params["rotations"]
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        for k, v in opt.params.items():
            d["a_" + k] = v
        d["a_pos_lr"] = np.array([opt.lrs["centers"]])
        tex = scene.mesh.texture.copy()
        topt = Adam({"texture": tex}, {"texture": cfg.lr_texture})
        gtex = texture_backward(fr, grads.mesh_color + gim, tex.shape[:2])
        d["a_grad_texture"] = gtex
        topt.step({"texture": gtex})
        np.clip(tex, 0.0, 1.0, out=tex)
        d["a_texture"] = tex
    if lean:  # keep the large-image fixture small: drop what other fixtures already pin
        for k in ("f_bary", "f_color", "r0_color", "r0_depth", "r0_t", "r0_last"):
            d.pop(k, None)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **d)
    print(f"{name}: N={len(scene.gaussians)} M={len(proj)} K={len(tiles.entries)} -> {os.path.getsize(path) / 1e6:.2f} MB")


def edge_cases():
    """Reference pins from test_splat_project/forward and test_meshraster."""
    d = {}
    # equal depths ordered by index (test_splat_project.py:116-128)
    gs = GaussianSet(np.array([[0.1, 0, 3.0], [-0.1, 0, 3.0], [0, 0.1, 3.0]]), np.tile([1.0, 0, 0, 0], (3, 1)),
                     np.full((3, 3), -1.0), np.zeros(3), np.zeros((3, 3)))
    cam = Camera(60.0, 60.0, 32.0, 32.0, 64, 64, np.eye(4), 0.05, 100.0)
    proj = project(gs, cam)
    t = build_tiles(proj, 64, 64)
    d["eq_starts"], d["eq_entries"] = t.tile_starts, t.entries
    out, ctx = render(gs, cam, background=(0.2, 0.4, 0.6))
    d["eq_color"], d["eq_t"] = out.color, out.transmittance
    # shared-edge quad (test_meshraster.py:78-88), full-screen quad, behind-camera quad
    verts = np.array([[-1.0, -1.0, 2.0], [1.0, -1.0, 2.0], [1.0, 1.0, 2.0], [-1.0, 1.0, 2.0]])
    tris = np.array([[0, 1, 2], [0, 2, 3]], dtype=np.int32)
    uvs = np.array([[[0, 0], [1, 0], [1, 1]], [[0, 0], [1, 1], [0, 1]]], dtype=np.float64)
    cam32 = Camera(32.0, 32.0, 16.0, 16.0, 32, 32, np.eye(4), 0.05, 100.0)
    fr = rasterize_fragments(TexturedMesh(verts, tris, uvs, np.full((16, 16, 3), 0.25)), cam32)
    d["se_tri"], d["se_depth"], d["se_bary"], d["se_uv"] = fr.triangle_id, fr.depth, fr.bary, fr.uv
    big = verts * np.array([3.0, 3.0, 1.0])
    cam_b = Camera(30.0, 30.0, 16.0, 12.0, 32, 24, np.eye(4), 0.05, 100.0)
    fr = rasterize_fragments(TexturedMesh(big, tris, uvs, np.full((8, 8, 3), 0.6)), cam_b)
    d["fs_tri"], d["fs_depth"] = fr.triangle_id, fr.depth
    # random triangle soup with overlaps (test_meshraster.py:54-63)
    rng = np.random.default_rng(3)
    n = 60
    v = np.column_stack([rng.uniform(-2, 2, 3 * n), rng.uniform(-2, 2, 3 * n), rng.uniform(1.5, 5.0, 3 * n)])
    v = syn.q32(v)
    f = np.arange(3 * n, dtype=np.int32).reshape(-1, 3)
    cam48 = Camera(43.2, 43.2, 24.0, 24.0, 48, 48, np.eye(4), 0.05, 100.0)
    fr = rasterize_fragments(TexturedMesh(v, f), cam48)
    d["soup_v"], d["soup_f"] = v.astype(np.float32), f
    d["soup_tri"], d["soup_depth"], d["soup_bary"] = fr.triangle_id, fr.depth, fr.bary
    np.savez_compressed(os.path.join(HERE, "edge.npz"), **d)
    print("edge cases written")


if __name__ == "__main__":
    run_case("small_sh0", syn.small_scene(seed=0))
    run_case("small_sh1", syn.small_scene(seed=1, sh_degree=1, with_mesh=True), train=False)
    run_case("c1", syn.make_config("c1", seed=0), backward=False, train=False, lean=True)
    edge_cases()
