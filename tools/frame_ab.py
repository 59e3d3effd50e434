"""A/B timing of the c3 hybrid frame for libhgs variants (HGS_LIB=...):
CUDA-graph replay, L2 flushed between frames, median of N; prints a
checksum of the frame so variants can be checked bit-identical."""
import os, sys, hashlib
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np, torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.engine import HybridRenderer
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
sc = syn.make_config(cfg, seed=0)
g = hgs.GaussianSet.from_any(sc.gaussians); m = hgs.TexturedMesh.from_any(sc.mesh)
c = hgs.Camera.from_any(sc.cameras[0])
r = HybridRenderer(g, m, c.width, c.height)
r.frame(c, sync_check=True)
r.capture()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(n + 3):
    flush.fill_(i & 255)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r.replay(); e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
h = hashlib.sha1(r.color.cpu().numpy().tobytes() + r.trans.cpu().numpy().tobytes()).hexdigest()[:12]
print(f"{os.path.basename(os.environ.get('HGS_LIB', 'libhgs.so'))} {cfg} median {np.median(ts)*1e3:.1f} us  min {min(ts)*1e3:.1f}  sha {h}", flush=True)
