"""Per-kernel device time of c4 training steps (torch.profiler / CUPTI):
usage: train_kernels.py [views] [steps]  (HGS_LIB selects a build)."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.config import TrainConfig
from paper_2506_06988_b200.train import HybridTrainer

nv = int(sys.argv[1]) if len(sys.argv) > 1 else 16
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda:0")
sc = syn.make_config("c4", seed=0, n_views=nv)
gs = hgs.GaussianSet.from_any(sc.gaussians); mesh = hgs.TexturedMesh.from_any(sc.mesh)
cams = [hgs.Camera.from_any(c) for c in sc.cameras]
cfg = TrainConfig(); it = cfg.warmup_iters + 1
H, W = cams[0].height, cams[0].width
tr = HybridTrainer(gs, mesh, cams, [torch.zeros(H, W, 3, device=dev) for _ in cams], cfg)
for v in range(nv):
    tr.images[v] = (tr.mesh_layer(v).color + 0.05 * torch.rand(H, W, 3, device=dev)).clamp_(0, 1)
views = list(range(nv))
for _ in range(2):
    tr.step(it, views)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        tr.step(it, views)
    torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        t = tot.setdefault(e.name, [0, 0.0])
        t[0] += 1
        t[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
grand = sum(v[1] for v in tot.values())
print(f"{os.path.basename(os.environ.get('HGS_LIB', 'libhgs.so'))}: {nv} views x {steps} steps, "
      f"kernel time per view {grand / (nv * steps) / 1e3:.3f} ms")
for name, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:16]:
    print(f"  {name[:70]:70s} n={n:5d} per-view {us / (nv * steps):8.1f} us  {100 * us / grand:5.1f}%")
