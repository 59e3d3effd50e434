"""Host-side cost of the training step: wall time of one c4 step vs the host
time spent issuing the per-view work (view_grads), to tell whether the GPU
is kept fed."""
import os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.config import TrainConfig
from paper_2506_06988_b200.train import HybridTrainer
nv = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc = syn.make_config("c4", seed=0, n_views=nv)
gs = hgs.GaussianSet.from_any(sc.gaussians); mesh = hgs.TexturedMesh.from_any(sc.mesh)
cams = [hgs.Camera.from_any(c) for c in sc.cameras]
tr = HybridTrainer(gs, mesh, cams, [torch.zeros(cams[0].height, cams[0].width, 3, device="cuda") for _ in cams], TrainConfig())
for v in range(nv):
    tr.images[v] = (tr.mesh_layer(v).color + 0.05).clamp_(0, 1)
it = 3001
for _ in range(2):
    tr.step(it, list(range(nv)))
torch.cuda.synchronize()
orig = tr.view_grads
acc = [0.0]
def timed(*a, **k):
    t = time.perf_counter()
    r = orig(*a, **k)
    acc[0] += time.perf_counter() - t
    return r
tr.view_grads = timed
t0 = time.perf_counter()
tr.step(it, list(range(nv)))
torch.cuda.synchronize()
t1 = time.perf_counter()
print("step wall %.1f ms; host time inside view_grads %.1f ms (%.3f ms/view)" % ((t1 - t0) * 1e3, acc[0] * 1e3, acc[0] * 1e3 / nv), flush=True)
