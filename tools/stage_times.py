"""Per-stage device timings of one hybrid frame (CUDA events, after warm-up)."""
import argparse
import sys
import os
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
import torch

import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import meshraster as mr
from paper_2506_06988_b200 import splat as sp
from paper_2506_06988_b200 import synthetic as syn

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
t0 = time.time()
sc = syn.make_config(a.config, seed=0)
print(f"scene gen {time.time()-t0:.1f}s")
cam = sc.cameras[0]
g = hgs.GaussianSet.from_any(sc.gaussians)
c = hgs.Camera.from_any(cam)
m = hgs.TexturedMesh.from_any(sc.mesh)
dev = g.device
cam_dev = sp._upload_camera(c, dev)
W, H = c.width, c.height
stats = torch.zeros(3, dtype=torch.int64, device=dev)


def frame(stats_t=None):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record()
    fr = mr.rasterize_fragments(m, c, with_bary=False)
    ev[1].record()
    layer = mr.mesh_layer(m, c, fr)
    ev[2].record()
    proj = sp._preprocess(g, c, cam_dev, 16, extras=False)
    ev[3].record()
    tiles, counters = sp._tiles_core(proj, W, H, 16, cap)
    ev[4].record()
    out = sp._blend(proj, tiles, W, H, layer, np.zeros(3), stats=stats_t)
    ev[5].record()
    torch.cuda.synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) for i in range(5)], counters, out, layer


cap = None
proj = sp._preprocess(g, c, cam_dev, 16, extras=False)
K = int(proj.count.sum().item())
cap = int(K * 1.1) + 1024
print(f"N={len(g)} M={int((proj.count>0).sum())} K={K} F={m.n_faces}")
for _ in range(3):
    frame()
times = []
for _ in range(a.iters):
    t, counters, out, layer = frame()
    times.append(t)
stats.zero_()
frame(stats)
st = stats.cpu().numpy()
med = np.median(np.array(times), axis=0)
names = ["raster", "texture", "preprocess", "tiles", "blend"]
for n_, v in zip(names, med):
    print(f"{n_:12s} {v*1000:9.1f} us")
print(f"total {med.sum()*1000:.1f} us -> {1000/med.sum():.0f} FPS (full hybrid); rasterizer-only {1000/med[2:].sum():.0f} FPS")
print("counters", counters.cpu().numpy(), "walked", st[0], "blended", st[1], "walked/px", st[0] / (W * H))
cov = (layer.triangle_id >= 0).float().mean().item()
tt = out[2]
print(f"coverage {cov:.3f} meanT_on_mesh {tt[layer.triangle_id>=0].mean().item():.4f}")
