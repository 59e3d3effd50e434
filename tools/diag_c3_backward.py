import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import meshraster as mr, synthetic as syn
from oracle import oracle as orc
sc = syn.make_config("c3", seed=0); cam = sc.cameras[0]
g = hgs.GaussianSet.from_any(sc.gaussians); c = hgs.Camera.from_any(cam); m = hgs.TexturedMesh.from_any(sc.mesh)
fr = orc.rasterize_fragments(sc.mesh.vertices, sc.mesh.triangles, sc.mesh.uvs, cam)
ml = orc.Mesh(orc.sample_texture(sc.mesh.texture, fr.uv, fr.valid), fr.depth, fr.triangle_id)
color, depth, tt, octx = orc.render(sc.gaussians, cam, (0, 0, 0), ml)
layer = mr.mesh_layer(m, c)
out, ctx = hgs.render(g, c, background=(0, 0, 0), mesh=layer)
rng = np.random.default_rng(9)
gc = syn.q32(rng.uniform(-1, 1, (cam.height, cam.width, 3))); gt = syn.q32(rng.uniform(-1, 1, (cam.height, cam.width)))
og = orc.backward(octx, gc, gt); gr = hgs.rasterize_backward(ctx, gc, gt)
for k in ("centers", "rotations", "log_scales", "logit_opacities", "colors_dc"):
    a = getattr(gr, k).detach().cpu().numpy().astype(np.float64); b = getattr(og, k)
    err = np.abs(a - b); i = np.unravel_index(err.argmax(), err.shape)
    norm = err / np.maximum(1.0, np.abs(b))
    print(f"{k:16s} max|b| {np.abs(b).max():10.4g}  max err {err.max():.3e} at |b|={abs(b[i]):.4g}  max rel-to-scale {err.max()/np.abs(b).max():.2e}  max norm {norm.max():.2e}  n(err>1e-4) {(err>1e-4).sum()}")
