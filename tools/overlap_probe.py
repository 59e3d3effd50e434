"""Upper bound of two-stream view overlap in training: two independent
HybridTrainers (own Gaussians and buffers), their per-view work interleaved
on two streams vs run back to back on one stream."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.config import TrainConfig
from paper_2506_06988_b200.train import HybridTrainer
nv = 16
dev = torch.device("cuda:0")
sc = syn.make_config("c4", seed=0, n_views=nv)
cams = [hgs.Camera.from_any(c) for c in sc.cameras]
cfg = TrainConfig(); it = cfg.warmup_iters + 1
H, W = cams[0].height, cams[0].width
trs = []
for _ in range(2):
    gs = hgs.GaussianSet.from_any(sc.gaussians); mesh = hgs.TexturedMesh.from_any(sc.mesh)
    tr = HybridTrainer(gs, mesh, cams, [torch.zeros(H, W, 3, device=dev) for _ in cams], cfg)
    for v in range(nv):
        tr.images[v] = (tr.mesh_layer(v).color + 0.05).clamp_(0, 1)
    trs.append(tr)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(overlap):
    main = torch.cuda.current_stream()
    s1.wait_stream(main); s2.wait_stream(main)
    for v in range(nv):
        for k, tr in enumerate(trs):
            st = (s1 if k == 0 else s2) if overlap else main
            with torch.cuda.stream(st):
                tr.view_grads(v, it, 1.0 / nv)
    main.wait_stream(s1); main.wait_stream(s2)
for mode in (False, True, False, True):
    run(mode); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        run(mode)
    e1.record(); torch.cuda.synchronize()
    print(f"overlap={mode}: {e0.elapsed_time(e1)/3/(2*nv):.3f} ms per view", flush=True)
