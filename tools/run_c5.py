"""Stress config c5 (5M Gaussians, 1M-triangle mesh, 1920x1080): full
hybrid frame through the engine + forward/backward through the API; prints
timings and sizes."""
import os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np, torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import meshraster as mr, synthetic as syn
from paper_2506_06988_b200.engine import HybridRenderer
t0 = time.time()
sc = syn.make_config("c5", seed=0)
print("scene built", round(time.time() - t0, 1), "s", len(sc.gaussians), sc.mesh.n_faces, flush=True)
g = hgs.GaussianSet.from_any(sc.gaussians); m = hgs.TexturedMesh.from_any(sc.mesh); c = hgs.Camera.from_any(sc.cameras[0])
r = HybridRenderer(g, m, c.width, c.height)
r.frame(c, sync_check=True)
mv, k, ovf = r.check()
print("M", mv, "K", k, "overflow", ovf, flush=True)
r.capture()
for _ in range(3): r.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): r.replay()
e1.record(); torch.cuda.synchronize()
print("c5 frame ms", e0.elapsed_time(e1) / 10, flush=True)
layer = mr.mesh_layer(m, c)
out, ctx = hgs.render(g, c, mesh=layer)
rng = np.random.default_rng(0)
gc = torch.as_tensor(rng.uniform(-1, 1, (c.height, c.width, 3)), dtype=torch.float32, device="cuda")
torch.cuda.synchronize(); t1 = time.time()
gr = hgs.rasterize_backward(ctx, gc)
torch.cuda.synchronize()
print("c5 backward s", round(time.time() - t1, 3), "grad finite", bool(torch.isfinite(gr.centers).all()),
      "mem GB", round(torch.cuda.max_memory_allocated() / 1e9, 1), flush=True)
