"""Pixels the fast blend hands to the exact fp64 replay (hgs_blend_out.stats[2],
counted by the STATS variant of the blend) for c3, c4 (first view) and c5."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.engine import HybridRenderer
for cfg in ("c3", "c4", "c5"):
    sc = syn.make_config(cfg, seed=0) if cfg != "c4" else syn.make_config("c4", seed=0, n_views=4)
    g = hgs.GaussianSet.from_any(sc.gaussians); m = hgs.TexturedMesh.from_any(sc.mesh); c = hgs.Camera.from_any(sc.cameras[0])
    r = HybridRenderer(g, m, c.width, c.height, collect_stats=True)
    r.frame(c, sync_check=True); torch.cuda.synchronize()
    r.stats.zero_()
    r.frame(c, sync_check=True); torch.cuda.synchronize()
    print(cfg, "flagged", int(r.stats[2]), "of", c.width * c.height, flush=True)
