import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from _util import golden_scene, load_golden
import paper_2506_06988_b200 as hgs
from paper_2506_06988_b200 import meshraster as mr
for name in ["small_sh0", "small_sh1", "c1"]:
    d = load_golden(name); _, gs, cam, mesh = (name,) + golden_scene(d)
    g = hgs.GaussianSet.from_any(gs); c = hgs.Camera.from_any(cam)
    m = hgs.TexturedMesh.from_any(mesh) if mesh is not None else None
    layer = mr.mesh_layer(m, c) if m is not None else None
    for mesh_on in (True, False):
        out, ctx = hgs.render(g, c, background=d["bg"], mesh=layer if mesh_on else None)
        last = ctx.last_consumed.cpu().numpy()
        ref = d["r_last"] if mesh_on else d.get("r0_last")
        if ref is None: continue
        bad = np.argwhere(last != ref)
        print(name, "mesh" if mesh_on else "nomesh", "bad", len(bad), "of", last.size)
        for (y, x) in bad[:8]:
            print("  px", x, y, "dev", last[y, x], "ref", ref[y, x], "T", out.transmittance[y, x].item(), "ref T", d["r_t"][y, x] if mesh_on else None)
