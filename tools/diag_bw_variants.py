"""Per-group gradient error vs the oracle at c3 for several library builds
(HGS_LIB variants): which precision change closes the 1e-4 contract.
usage: diag_bw_variants.py lib1.so lib2.so ...  (oracle cached in /tmp)"""
import os, subprocess, sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
CACHE = '/tmp/diag_c3_oracle.npz'
GROUPS = ("centers", "rotations", "log_scales", "logit_opacities", "colors_dc")


def oracle():
    from paper_2506_06988_b200 import synthetic as syn
    from oracle import oracle as orc
    sc = syn.make_config("c3", seed=0); cam = sc.cameras[0]
    fr = orc.rasterize_fragments(sc.mesh.vertices, sc.mesh.triangles, sc.mesh.uvs, cam)
    ml = orc.Mesh(orc.sample_texture(sc.mesh.texture, fr.uv, fr.valid), fr.depth, fr.triangle_id)
    color, depth, tt, octx = orc.render(sc.gaussians, cam, (0, 0, 0), ml)
    rng = np.random.default_rng(9)
    gc = syn.q32(rng.uniform(-1, 1, (cam.height, cam.width, 3))); gt = syn.q32(rng.uniform(-1, 1, (cam.height, cam.width)))
    og = orc.backward(octx, gc, gt)
    np.savez(CACHE, color=color, depth=depth, t=tt, **{k: getattr(og, k) for k in GROUPS})


def device():
    import torch
    import paper_2506_06988_b200 as hgs
    from paper_2506_06988_b200 import meshraster as mr, synthetic as syn
    sc = syn.make_config("c3", seed=0); cam = sc.cameras[0]
    g = hgs.GaussianSet.from_any(sc.gaussians); c = hgs.Camera.from_any(cam); m = hgs.TexturedMesh.from_any(sc.mesh)
    layer = mr.mesh_layer(m, c)
    out, ctx = hgs.render(g, c, background=(0, 0, 0), mesh=layer)
    rng = np.random.default_rng(9)
    gc = syn.q32(rng.uniform(-1, 1, (cam.height, cam.width, 3))); gt = syn.q32(rng.uniform(-1, 1, (cam.height, cam.width)))
    gr = hgs.rasterize_backward(ctx, gc, gt)
    torch.cuda.synchronize()
    o = np.load(CACHE)
    print("lib", os.environ.get("HGS_LIB"))
    for k, a in (("color", out.color), ("depth", out.depth), ("t", out.transmittance)):
        a = a.cpu().numpy().astype(np.float64); b = o[k]; f = np.isfinite(b)
        print(f"  {k:16s} max err {np.abs(a[f] - b[f]).max():.3e}  nan-pattern-equal {np.array_equal(np.isnan(a), np.isnan(b))}")
    for k in GROUPS:
        a = getattr(gr, k).detach().cpu().numpy().astype(np.float64); b = o[k]
        err = np.abs(a - b); i = np.unravel_index(err.argmax(), err.shape)
        print(f"  {k:16s} max|b| {np.abs(b).max():10.4g}  max err {err.max():.3e} at |b|={abs(b[i]):.4g}  "
              f"rel-to-scale {err.max() / np.abs(b).max():.2e}  n(err>1e-4) {(err > 1e-4).sum()}", flush=True)


if __name__ == "__main__":
    if sys.argv[1:2] == ["--device"]:
        device()
    else:
        if not os.path.exists(CACHE):
            oracle()
        for lib in sys.argv[1:]:
            env = dict(os.environ, HGS_LIB=os.path.abspath(lib))
            subprocess.run([sys.executable, __file__, "--device"], env=env, check=False)
