"""Profile one c4 training step (per-kernel times via ncu launch list)."""
import os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.config import TrainConfig
from paper_2506_06988_b200.train import HybridTrainer
nv = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sc = syn.make_config("c4", seed=0, n_views=nv)
gs = hgs.GaussianSet.from_any(sc.gaussians); mesh = hgs.TexturedMesh.from_any(sc.mesh)
cams = [hgs.Camera.from_any(c) for c in sc.cameras]
dev = gs.device
H, W = cams[0].height, cams[0].width
tr = HybridTrainer(gs, mesh, cams, [torch.zeros(H, W, 3, device=dev) for _ in cams], TrainConfig())
for v in range(nv):
    tr.images[v] = (tr.mesh_layer(v).color + 0.05).clamp_(0, 1)
it = 3001
for _ in range(2):
    tr.step(it, list(range(nv)))
torch.cuda.synchronize()
t0 = time.time()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    tr.step(it, list(range(nv)))
e1.record(); torch.cuda.synchronize()
print(f"{nv} views: {e0.elapsed_time(e1)/steps:.2f} ms/step (gpu), {1000*(time.time()-t0)/steps:.2f} ms wall; per view {e0.elapsed_time(e1)/steps/nv:.2f} ms")
