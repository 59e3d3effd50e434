"""The data-parallel branch of HybridTrainer.step through the real
torch.distributed all_reduce (train.py: ``dist.all_reduce(self.bucket)``):
two processes on one GPU with the gloo backend over CUDA tensors (NCCL
refuses two ranks on one device; no kernel of one rank waits on the other
-- the exchange is the host-side collective).  Both replicas must end
bit-identical and equal to the one-process step over the whole batch up to
fp32 summation order (gsmesh/train/loop.py:181-224 per-view semantics, the
shards' gradients summed)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_VIEWS = 6


def _scene():
    import torch
    import paper_2506_06988_b200 as hgs
    from paper_2506_06988_b200 import synthetic as syn
    sc = syn.make_config("c2", seed=0)
    rng = np.random.default_rng(5)
    views = [syn.look_at((0.15 * k, -0.1, -0.2), (0.0, 0.0, 5.0), width=320, height=240) for k in range(N_VIEWS)]
    cams = [hgs.Camera.from_any(v) for v in views]
    images = [torch.as_tensor(rng.uniform(0, 1, (240, 320, 3)), dtype=torch.float32) for _ in cams]
    return sc, cams, images


def _trainer(rank, world):
    import paper_2506_06988_b200 as hgs
    from paper_2506_06988_b200.config import TrainConfig
    from paper_2506_06988_b200.train import HybridTrainer
    sc, cams, images = _scene()
    gs = hgs.GaussianSet.from_any(sc.gaussians)
    mesh = hgs.TexturedMesh.from_any(sc.mesh)
    return HybridTrainer(gs, mesh, cams, images, TrainConfig(), rank=rank, world=world, density_control=True,
                         extent=1.0)


def _rank_main(rank, world, port, out_dir):
    import sys
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    from paper_2506_06988_b200.config import TrainConfig
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        tr = _trainer(rank, world)
        loss = tr.step(TrainConfig().warmup_iters + 1, list(range(N_VIEWS)))
        torch.cuda.synchronize()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), params=tr.gs.params.detach().cpu().numpy(),
                 texture=tr.mesh.texture.detach().cpu().numpy(), loss=loss.cpu().numpy(),
                 accum=tr.dstate.grad_accum.cpu().numpy(), denom=tr.dstate.denom.cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_step_matches_single_process(cuda_device, tmp_path):
    import socket
    import torch
    import torch.multiprocessing as mp
    from paper_2506_06988_b200.config import TrainConfig
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    r0, r1 = (np.load(tmp_path / f"rank{r}.npz") for r in range(2))
    for k in ("params", "texture", "loss", "accum", "denom"):
        assert np.array_equal(r0[k], r1[k]), f"replicas differ in {k}"
    single = _trainer(0, 1)
    loss = single.step(TrainConfig().warmup_iters + 1, list(range(N_VIEWS)))
    torch.cuda.synchronize()
    assert np.abs(r0["params"] - single.gs.params.detach().cpu().numpy()).max() < 1e-6
    assert np.abs(r0["texture"] - single.mesh.texture.detach().cpu().numpy()).max() < 1e-6
    assert np.allclose(r0["loss"], loss.cpu().numpy(), rtol=1e-6, atol=1e-9)
    assert np.array_equal(r0["denom"], single.dstate.denom.cpu().numpy())
    acc1 = single.dstate.grad_accum.cpu().numpy()
    assert np.abs(r0["accum"] - acc1).max() <= 1e-5 * max(1.0, np.abs(acc1).max())
