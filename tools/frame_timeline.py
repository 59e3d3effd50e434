"""Kernel timeline of one c3 frame graph replay (torch.profiler / CUPTI):
start / end of every kernel relative to the first, to see the overlap of
the PDL chain, the ready-queue hand-offs and the mesh side stream."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.engine import HybridRenderer
from torch.profiler import profile, ProfilerActivity
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
sc = syn.make_config(cfg, seed=0)
g = hgs.GaussianSet.from_any(sc.gaussians); m = hgs.TexturedMesh.from_any(sc.mesh)
c = hgs.Camera.from_any(sc.cameras[0])
r = HybridRenderer(g, None if os.environ.get("NOMESH") else m, c.width, c.height)
r.frame(c, sync_check=True)
r.capture()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    flush.fill_(1); r.replay()
torch.cuda.synchronize()
flush.fill_(2)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r.replay()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
end = max(e.time_range.end for e in ev)
print(f"frame span {end - t0:.1f} us, {len(ev)} kernels")
for e in ev:
    print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} {e.time_range.end - e.time_range.start:7.1f}  {e.name[:70]}")
