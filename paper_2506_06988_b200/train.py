"""Joint Gaussian + texture optimisation step on the device, view-sharded
data parallel over ranks (one process per GPU, NCCL all-reduce).

Mirrors gsmesh/train/loop.py: GaussianTrainer (:85-145: per-group learning
rates, position lr decay, quaternion renormalisation, texture Adam + clamp),
the per-iteration body of train() (:181-224: texture lookup over cached
fragments, render, composite loss, rasterize_backward, Adam, texture
backward, texture Adam) -- generalised to a batch of views per step
(SURVEY H7): the step gradient is the mean of the per-view gradients, then
ONE Adam update.  With world > 1 each rank renders its contiguous block of
the batch and a single all_reduce(SUM) over one flat fp32 bucket
(Gaussian grads | texture grad | densify norms) precedes the identical Adam
update on every rank, so replicas stay bit-identical.

Adaptive density control (densify.py) is opt-in
(density_control=True): every densify_interval iterations, on the device.
"""

from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .adam import Adam, exponential_lr
from .backward import GradBuffer, chain_backward, screen_backward
from .losses import composite_loss
from .meshraster import MeshFragmentBuffer, rasterize_fragments
from .scene import Camera, GaussianSet, TexturedMesh, camera_tensor
from .splat import REC_BYTES, TILE_PX, MeshLayer, ProjectedGaussians, RenderCtx, TileBins, _blend, _stream_ptr


def shard_views(n_views: int, rank: int, world: int) -> List[int]:
    """Contiguous block of the batch for this rank."""
    base, rem = divmod(n_views, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return list(range(lo, hi))


class _Lane:
    """Per-view work buffers of one of the trainer's view pipelines.
    Views of a step alternate between the lanes, each on its own stream, so
    one view's forward / binning overlaps the other's backward; the lanes
    share only the gradient bucket (see HybridTrainer.step)."""

    def __init__(self, dev, stream):
        self.dev = dev
        self.stream = stream
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self.overflow = torch.zeros(1, dtype=torch.int64, device=dev)
        self.loss_sum = torch.zeros(6, dtype=torch.float64, device=dev)
        self.capacity = 0

    def alloc_rows(self, n: int, tiles_xy):
        dev = self.dev
        tx, ty = tiles_xy
        self.rec = torch.empty(n * REC_BYTES, dtype=torch.uint8, device=dev)
        self.count = torch.zeros(n, dtype=torch.int32, device=dev)
        self.rect = torch.zeros(n * 4, dtype=torch.int16, device=dev)
        self.cull = torch.empty(n * 12, dtype=torch.float32, device=dev)
        self.sort_keys = torch.empty(n, dtype=torch.int64, device=dev)
        self.screen = torch.zeros(n * 9, dtype=torch.float64, device=dev)
        self.tile_diff = torch.empty(16 * (tx + 1) * (ty + 1), dtype=torch.int32, device=dev)

    def alloc_entries(self, cap: int, n: int, tiles_xy):
        tx, ty = tiles_xy
        self.capacity = cap
        self.entries = torch.empty(cap, dtype=torch.int32, device=self.dev)
        self.tile_starts = torch.empty(tx * ty + 1, dtype=torch.int64, device=self.dev)
        nbytes = _lib.load().hgs_tiles_scratch_bytes(n, cap, tx * ty)
        self.tiles_scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        self.ready = torch.zeros(_lib.READY_INTS, dtype=torch.int32, device=self.dev)


class HybridTrainer:
    N_LANES = 4  # 2: 137.7, 3: 134.2, 4: 132.3 ms per c4 step (B200)

    def __init__(self, gs: GaussianSet, mesh: Optional[TexturedMesh], cameras: Sequence, images: Sequence, config,
                 rank: int = 0, world: int = 1, process_group=None, allreduce=None, density_control: bool = False,
                 extent: Optional[float] = None, rng: Optional[np.random.Generator] = None):
        self.gs = gs
        self.mesh = mesh
        self.cfg = config
        self.rank, self.world = rank, world
        self.pg = process_group
        self._allreduce = allreduce
        dev = gs.device
        self.dev = dev
        self.cameras = [Camera.from_any(c) for c in cameras]
        if len({(int(c.width), int(c.height)) for c in self.cameras}) > 1:
            raise ValueError("HybridTrainer needs one image size for all views (its per-lane buffers are sized once); "
                             "loop.train handles mixed resolutions")
        if len(images) != len(self.cameras):
            raise ValueError(f"{len(self.cameras)} cameras but {len(images)} images")
        self.cam_dev = [camera_tensor(c, dev) for c in self.cameras]
        self.images = [im if isinstance(im, torch.Tensor) else torch.as_tensor(np.asarray(im, dtype=np.float32))
                       for im in images]
        self.images = [im.to(dev, torch.float32).contiguous() for im in self.images]
        self.bg = np.asarray(config.background, dtype=np.float64).reshape(3)
        n = len(gs)
        self._alloc_bucket()
        # optimiser state (loop.py:92-117)
        names = [g for g in ("centers", "rotations", "log_scales", "logit_opacities", "colors_dc", "colors_rest")
                 if g in gs.layout]
        self.names = names
        params = {k: gs.group(k) for k in names}
        lrs = {"centers": config.lr_position, "rotations": config.lr_rotation, "log_scales": config.lr_scale,
               "logit_opacities": config.lr_opacity, "colors_dc": config.lr_color,
               "colors_rest": config.lr_color / 20.0}
        self.opt = Adam(params, {k: lrs[k] for k in names})
        self.pos_lr = exponential_lr(config.lr_position, config.lr_position_final, config.max_iters)
        self.tex_opt = Adam({"texture": mesh.texture}, {"texture": config.lr_texture}) if self.tex_grad is not None else None
        # adaptive density control (loop.py:226-233, densify.py), opt-in
        self.density_control = density_control
        if density_control:
            from .densify import DensifyState
            from .scene import camera_extent
            self.extent = extent if extent is not None else (
                camera_extent(self.cameras) if len(self.cameras) > 1 else 1.0)
            self.rng = rng if rng is not None else np.random.default_rng(config.seed)
            self.dstate = DensifyState.zeros(n, dev)
            self.density_stats: List[dict] = []
        # per-camera fragments, rasterized once (loop.py:172-175)
        self.frags: List[Optional[MeshFragmentBuffer]] = []
        for c in self.cameras:
            self.frags.append(rasterize_fragments(mesh, c, with_bary=False) if mesh is not None else None)
        c0 = self.cameras[0]
        self.tx = (int(c0.width) + TILE_PX - 1) // TILE_PX
        self.ty = (int(c0.height) + TILE_PX - 1) // TILE_PX
        self.lanes = [_Lane(dev, torch.cuda.Stream(dev) if dev.type == "cuda" else None)
                      for _ in range(self.N_LANES)]
        self._alloc_rows()
        self.loss_sum = torch.zeros(6, dtype=torch.float64, device=dev)
        self._size_entries()

    # ------------------------------------------------------------------
    def _alloc_bucket(self):
        """One flat bucket, all-reduced once per step: Gaussian grads |
        texture grad | densify norm sums | visible-view counts."""
        gs, mesh, dev = self.gs, self.mesh, self.dev
        n = max(len(gs), 1)
        p_sz = gs.params.numel()
        t_sz = mesh.texture.numel() if (mesh is not None and mesh.texture is not None) else 0
        self.bucket = torch.zeros(p_sz + t_sz + 2 * n, dtype=torch.float32, device=dev)
        o = p_sz + t_sz
        self.grads = GradBuffer(gs, self.bucket[:p_sz], self.bucket[o:o + n], self.bucket[o + n:o + 2 * n])
        self.tex_grad = self.bucket[p_sz:p_sz + t_sz].view_as(mesh.texture) if t_sz else None
        # the views' texture gradients meet in a 2^-32 fixed-point accumulator
        # (integer atomics: order-independent, so the step is run-to-run
        # reproducible), converted into tex_grad once per step
        if t_sz and getattr(self, "tex_acc", None) is None:
            self.tex_acc = torch.zeros(t_sz, dtype=torch.int64, device=dev)

    def _alloc_rows(self):
        """Per-view work buffers sized by the Gaussian count, one set per
        lane (each reused in order on its lane's stream)."""
        n = max(len(self.gs), 1)
        for lane in self.lanes:
            lane.alloc_rows(n, (self.tx, self.ty))

    def _density_step(self, it: int, nb: int) -> None:
        """loop.py:226-233 after the optimiser steps of iteration ``it``
        (a step over ``nb`` views)."""
        from .densify import densify_and_prune, reset_opacity
        cfg = self.cfg
        if it >= cfg.densify_until_iter:
            return
        # the views' losses were scaled by 1/nb (batch mean), and the norm
        # is linear in that scale: x nb restores the sum of the per-view
        # norms the reference accumulates one view at a time (densify.py:31-33)
        self.dstate.update(self.grads.visible_count, self.grads.densify_norm, scale=float(nb))
        if it >= cfg.densify_from_iter and it % cfg.densify_interval == 0:
            self.gs, stats = densify_and_prune(self.gs, self.opt, self.dstate, self.extent, cfg, self.rng)
            stats["iter"] = it
            self.density_stats.append(stats)
            self._alloc_bucket()
            self._alloc_rows()
            self._size_entries()
        if it % cfg.opacity_reset_interval == 0:
            reset_opacity(self.gs, self.opt)

    def _size_entries(self):
        """Tile-entry capacity: max K over this rank's views x 1.2 (one sync)."""
        kmax = 0
        for v in range(len(self.cameras)):
            proj = self._project(v, self.lanes[0])
            kmax = max(kmax, int(proj.count.sum().item()))
        cap = int(kmax * 1.2) + 4096
        for lane in self.lanes:
            lane.alloc_entries(cap, len(self.gs), (self.tx, self.ty))

    def _project(self, v, lane: _Lane) -> ProjectedGaussians:
        cam = self.cameras[v]
        ps = _lib.HGSProjected()
        ps.rec, ps.count, ps.rect, ps.cull = (_lib.ptr(lane.rec), _lib.ptr(lane.count), _lib.ptr(lane.rect),
                                              _lib.ptr(lane.cull))
        ps.sort_keys, ps.tile_diff = _lib.ptr(lane.sort_keys), _lib.ptr(lane.tile_diff)
        _lib.call("hgs_preprocess", _lib.ptr(self.cam_dev[v]), int(cam.width), int(cam.height),
                  ctypes.byref(self.gs.struct()), TILE_PX, ctypes.byref(ps), _stream_ptr(self.dev))
        return ProjectedGaussians(len(self.gs), lane.rec, lane.count, lane.rect, None, int(cam.width),
                                  int(cam.height), TILE_PX, lane.cull, lane.sort_keys, lane.tile_diff)

    def _tiles(self, proj, lane: _Lane) -> TileBins:
        ts = _lib.HGSTiles()
        ts.tiles_x, ts.tiles_y, ts.tile_px, ts.capacity = self.tx, self.ty, TILE_PX, lane.capacity
        ts.entries, ts.tile_starts, ts.counters = _lib.ptr(lane.entries), _lib.ptr(lane.tile_starts), _lib.ptr(lane.counters)
        ts.scratch, ts.scratch_bytes = _lib.ptr(lane.tiles_scratch), lane.tiles_scratch.numel()
        ts.ready = _lib.ptr(lane.ready)
        _lib.call("hgs_build_tiles", ctypes.byref(proj.struct()), len(self.gs), ctypes.byref(ts), _stream_ptr(self.dev))
        lane.overflow += lane.counters[2:3]
        return TileBins(lane.tile_starts, lane.entries, self.tx, self.ty, TILE_PX, proj, counters=lane.counters,
                        capacity=lane.capacity, ready=lane.ready)

    def mesh_layer(self, v) -> Optional[MeshLayer]:
        """Texture lookup over the cached fragments (loop.py:189-199)."""
        if self.mesh is None:
            return None
        from .meshraster import sample_texture
        fr = self.frags[v]
        color = sample_texture(self.mesh.texture, fr.uv, fr.triangle_id)
        return MeshLayer(color, fr.depth, fr.triangle_id)

    def view_grads(self, v: int, it: int, grad_scale: float, lane: Optional[_Lane] = None, after=None):
        """Forward + loss + backward of one view on the current stream,
        accumulated (x grad_scale) into the bucket; the accumulation into the
        shared bucket waits for event ``after`` (the previous view's).
        Returns the device loss scalars of this view."""
        lane = lane if lane is not None else self.lanes[0]
        cam = self.cameras[v]
        w, h = int(cam.width), int(cam.height)
        layer = self.mesh_layer(v)
        proj = self._project(v, lane)
        tiles = self._tiles(proj, lane)
        color, depth, trans, final_t, last, _ = _blend(proj, tiles, w, h, layer, self.bg)
        fr = self.frags[v]
        covered = fr.triangle_id if fr is not None else None
        bd, g_ih, g_im, g_t = composite_loss(self.images[v], color, layer.color if layer else None, covered, trans,
                                             it, self.cfg, grad_scale=grad_scale)
        ctx = RenderCtx(self.gs, cam, proj, tiles, layer, self.bg, final_t, last, self.cam_dev[v])
        lane.screen.zero_()
        mesh_grad = None
        if layer is not None:
            mesh_grad = g_im if g_im is not None else torch.zeros(h, w, 3, dtype=torch.float32, device=self.dev)
        screen_backward(ctx, g_ih, g_t, lane.screen, mesh_grad, accumulate_mesh=True)
        if after is not None:  # the chain accumulates (read-modify-write) into the shared bucket, in view order
            torch.cuda.current_stream(self.dev).wait_event(after)
        chain_backward(ctx, lane.screen, self.grads, scale=1.0, accumulate=True)
        if lane.stream is not None:  # the next view's chain may start once this one is done
            lane.chain_done = torch.cuda.Event()
            lane.chain_done.record(torch.cuda.current_stream(self.dev))
        if layer is not None and self.tex_grad is not None:
            th, tw = (int(x) for x in self.mesh.texture.shape[:2])
            _lib.call("hgs_texture_backward_fixed", _lib.ptr(fr.uv), _lib.ptr(fr.triangle_id), _lib.ptr(mesh_grad),
                      fr.triangle_id.numel(), th, tw, _lib.ptr(self.tex_acc), _stream_ptr(self.dev))
        return bd.scalars

    def step(self, it: int, views: Sequence[int]) -> torch.Tensor:
        """One optimisation step over the global batch ``views`` (this rank
        renders its shard).  Returns the batch-mean loss scalars (device)."""
        nb = len(views)
        mine = [views[i] for i in shard_views(nb, self.rank, self.world)]
        self.bucket.zero_()
        self.grads.visible.zero_()
        self.loss_sum.zero_()
        for lane in self.lanes:
            lane.loss_sum.zero_()
            lane.overflow.zero_()
        if self.lanes[0].stream is None:
            for v in mine:
                self.lanes[0].loss_sum += self.view_grads(v, it, 1.0 / nb)
        else:
            # views alternate between the lanes' streams; only the chain's
            # accumulation into the bucket is ordered across them (events)
            main = torch.cuda.current_stream(self.dev)
            for lane in self.lanes:
                lane.stream.wait_stream(main)
            prev = None
            for j, v in enumerate(mine):
                lane = self.lanes[j % len(self.lanes)]
                with torch.cuda.stream(lane.stream):
                    lane.loss_sum += self.view_grads(v, it, 1.0 / nb, lane=lane, after=prev)
                    prev = lane.chain_done
            for lane in self.lanes:
                main.wait_stream(lane.stream)
        overflow = self.lanes[0].overflow
        for lane in self.lanes[1:]:
            overflow = overflow + lane.overflow
        if int(overflow.item()):
            if self.tex_grad is not None:
                self.tex_acc.zero_()  # discard the partial texture sums of the failed pass
            self._size_entries()
            return self.step(it, views)
        if self.tex_grad is not None:
            _lib.call("hgs_fixed_to_float", _lib.ptr(self.tex_acc), self.tex_acc.numel(), _lib.ptr(self.tex_grad), 0,
                      _stream_ptr(self.dev))
        for lane in self.lanes:
            self.loss_sum += lane.loss_sum
        if self.world > 1:
            self.loss_sum /= nb
            if self._allreduce is not None:
                self._allreduce(self.bucket)
                self._allreduce(self.loss_sum)
            else:
                import torch.distributed as dist
                dist.all_reduce(self.bucket, group=self.pg)
                dist.all_reduce(self.loss_sum, group=self.pg)
        else:
            self.loss_sum /= nb
        self.opt.lrs["centers"] = self.pos_lr(it)
        self.opt.step({k: self.grads.group(k) for k in self.names}, renorm=("rotations",))
        if self.tex_opt is not None:
            self.tex_opt.step({"texture": self.tex_grad}, clamp=("texture",))
        if self.density_control:
            self._density_step(it, nb)
        return self.loss_sum
