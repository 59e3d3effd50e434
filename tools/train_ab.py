"""A/B timing of the c4 training step (64 views) for libhgs variants
(HGS_LIB=...): 3 warm-up steps, K timed (CUDA events); prints ms/step and
the loss so variants can be compared."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.config import TrainConfig
from paper_2506_06988_b200.train import HybridTrainer
if os.environ.get('HGS_LANES'):
    HybridTrainer.N_LANES = int(os.environ['HGS_LANES'])
k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dev = torch.device("cuda:0")
sc = syn.make_config("c4", seed=0, n_views=nv)
gs = hgs.GaussianSet.from_any(sc.gaussians); mesh = hgs.TexturedMesh.from_any(sc.mesh)
cams = [hgs.Camera.from_any(c) for c in sc.cameras]
cfg = TrainConfig(); it = cfg.warmup_iters + 1
H, W = cams[0].height, cams[0].width
tr = HybridTrainer(gs, mesh, cams, [torch.zeros(H, W, 3, device=dev) for _ in cams], cfg)
g = torch.Generator(device=dev).manual_seed(1234)
for v in range(nv):
    tr.images[v] = (tr.mesh_layer(v).color + 0.05 * torch.rand(H, W, 3, device=dev, generator=g)).clamp_(0, 1)
views = list(range(nv))
for _ in range(3):
    tr.step(it, views)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(k):
    loss = tr.step(it, views)
e1.record(); torch.cuda.synchronize()
print(f"{os.path.basename(os.environ.get('HGS_LIB', 'libhgs.so'))} lanes={HybridTrainer.N_LANES} train ms/step {e0.elapsed_time(e1)/k:.2f} loss {float(loss[4]):.9f}", flush=True)
