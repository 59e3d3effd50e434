import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.engine import HybridRenderer
sc = syn.make_config("c3", seed=0)
g = hgs.GaussianSet.from_any(sc.gaussians); m = hgs.TexturedMesh.from_any(sc.mesh)
cam = sc.cameras[0]; c = hgs.Camera.from_any(cam)
r = HybridRenderer(g, m, c.width, c.height)
r.frame(c, sync_check=True); r.capture()
H, W = c.height, c.width
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
host = [(torch.empty(H, W, 3).pin_memory(), torch.empty(H, W).pin_memory(), torch.empty(H, W).pin_memory()) for _ in range(2)]
stream = torch.cuda.current_stream()
def run(n, do_flush=True, do_host=True, do_cam=True):
    pending = [None, None]
    for i in range(2):
        r.render_to_host(cam, *host[i])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(n):
        if do_flush: flush.fill_(i & 255)
        if do_host:
            if pending[i & 1] is not None: pending[i & 1].synchronize()
            pending[i & 1] = r.render_to_host(cam, *host[i & 1])
        else:
            if do_cam: r.set_camera(cam)
            r.replay()
    for ev in pending:
        if ev is not None: stream.wait_event(ev)
    e1.record(stream); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
for name, kw in [("e2e as bench", {}), ("no flush", dict(do_flush=False)), ("replay only + flush", dict(do_host=False)),
                 ("replay only, no cam", dict(do_host=False, do_cam=False)), ("replay only, no flush", dict(do_host=False, do_flush=False))]:
    ts = [run(50, **kw) for _ in range(3)]
    print(f"{name:28s} {min(ts):8.1f} us/frame")
