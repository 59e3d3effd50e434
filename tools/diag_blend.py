import sys, os
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np, torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import meshraster as mr, splat as sp, synthetic as syn
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
sc = syn.make_config(cfg, seed=0)
cam = sc.cameras[0]
g = hgs.GaussianSet.from_any(sc.gaussians); c = hgs.Camera.from_any(cam); m = hgs.TexturedMesh.from_any(sc.mesh)
layer = mr.mesh_layer(m, c)
cam_dev = sp._upload_camera(c, g.device)
proj = sp._preprocess(g, c, cam_dev, 16, extras=False)
tiles, _ = sp._tiles_core(proj, c.width, c.height, 16, None)
out = sp._blend(proj, tiles, c.width, c.height, layer, np.zeros(3))
torch.cuda.synchronize()
fx = sp.SCRATCH.bufs[("fixup", g.device)].view(torch.int32)
ntiles = tiles.tiles_x * tiles.tiles_y

nflag = int(fx[0])
print("flagged", nflag, "of", c.width * c.height)
if nflag:
    idx = fx[1:1 + min(nflag, 10)].cpu().numpy()
    print("first flagged", idx)
cull = proj.cull.view(-1, 4)[:5].cpu().numpy()
print("cull sample", cull)
rec = proj.rec.view(torch.float64)[:50].view(5, 10).cpu().numpy()
print("rec sample", rec[:, :7])
