"""View-sharded data parallelism, host logic, on CPU with the gloo backend
(world_size 2): each rank computes the gradients of its contiguous block of
the view batch (shard_views) scaled by 1/B, ONE all_reduce(SUM) of the flat
bucket gives the batch-mean gradient, and the identical Adam update keeps
replicas bit-identical -- the same protocol HybridTrainer.step runs over
NCCL on GPUs.  The oracle stands in for the device compute here."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_06988_b200 import synthetic as syn
from paper_2506_06988_b200.train import shard_views

GROUPS = ("centers", "rotations", "log_scales", "logit_opacities", "colors_dc")


def _views():
    sc = syn.small_scene(seed=3, n=120, width=48, height=40, with_mesh=False)
    base = sc.cameras[0]
    cams = []
    rng = np.random.default_rng(0)
    for k in range(4):
        eye = np.array([0.3, -0.2, -0.1]) + rng.normal(0, 0.05, 3)
        cams.append(syn.look_at(eye, (0.6, 0.1, 5.0), width=48, height=40))
    grads_in = [(syn.q32(rng.uniform(-1, 1, (40, 48, 3))), syn.q32(rng.uniform(-1, 1, (40, 48)))) for _ in cams]
    return sc.gaussians, cams, grads_in


def _bucket(gs, cams, grads_in, views, scale):
    from oracle import oracle as orc
    tot = None
    for v in views:
        *_, ctx = orc.render(gs, cams[v], (0, 0, 0), None)
        g = orc.backward(ctx, *grads_in[v])
        flat = np.concatenate([np.asarray(getattr(g, k), dtype=np.float64).reshape(-1) for k in GROUPS]) * scale
        tot = flat if tot is None else tot + flat
    if tot is None:
        tot = np.zeros(sum(np.asarray(getattr(gs, k)).size for k in GROUPS))
    return tot


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gs, cams, grads_in = _views()
    b = len(cams)
    mine = shard_views(b, rank, world)
    bucket = torch.from_numpy(_bucket(gs, cams, grads_in, mine, 1.0 / b))
    dist.all_reduce(bucket)
    # identical Adam step on every replica
    from oracle import oracle as orc
    p = np.concatenate([np.asarray(getattr(gs, k), dtype=np.float64).reshape(-1) for k in GROUPS])
    m, v = np.zeros_like(p), np.zeros_like(p)
    orc.adam_step(p, m, v, bucket.numpy(), 1e-3, 1)
    gathered = [torch.zeros_like(bucket) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(p))
    if rank == 0:
        out_q.put((bucket.numpy(), [t.numpy() for t in gathered]))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.timeout(300)
def test_two_rank_allreduce_equals_single_process_mean():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    bucket, replicas = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    gs, cams, grads_in = _views()
    ref = _bucket(gs, cams, grads_in, range(len(cams)), 1.0 / len(cams))
    np.testing.assert_allclose(bucket, ref, rtol=1e-12, atol=1e-12)
    assert np.array_equal(replicas[0], replicas[1]), "replicas diverged after the Adam step"
