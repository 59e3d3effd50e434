import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.engine import HybridRenderer
for cfg in ("c3", "c4", "c5"):
    sc = syn.make_config(cfg, seed=0) if cfg != "c4" else syn.make_config("c4", seed=0, n_views=4)
    g = hgs.GaussianSet.from_any(sc.gaussians); m = hgs.TexturedMesh.from_any(sc.mesh); c = hgs.Camera.from_any(sc.cameras[0])
    r = HybridRenderer(g, m, c.width, c.height)
    r.frame(c, sync_check=True); torch.cuda.synchronize()
    print(cfg, "flagged", int(r.fixup[0]), "of", c.width * c.height, flush=True)
