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

Density control (densify.py) is out of scope for this path.
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
from .splat import (REC_BYTES, TILE_PX, MeshLayer, ProjectedGaussians, RenderCtx, TileBins, _blend, _stream_ptr,
                    SCRATCH)


def shard_views(n_views: int, rank: int, world: int) -> List[int]:
    """Contiguous block of the batch for this rank."""
    base, rem = divmod(n_views, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return list(range(lo, hi))


class HybridTrainer:
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
        self._alloc_rows()
        c0 = self.cameras[0]
        self.tx = (int(c0.width) + TILE_PX - 1) // TILE_PX
        self.ty = (int(c0.height) + TILE_PX - 1) // TILE_PX
        self.tile_diff = torch.empty(16 * (self.tx + 1) * (self.ty + 1), dtype=torch.int32, device=dev)
        self.capacity = 0
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self.overflow = torch.zeros(1, dtype=torch.int64, device=dev)
        self.loss_sum = torch.zeros(6, dtype=torch.float64, device=dev)
        self.scalars = torch.zeros(6, dtype=torch.float64, device=dev)
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

    def _alloc_rows(self):
        """Per-view work buffers sized by the Gaussian count (reused
        sequentially on one stream)."""
        n, dev = max(len(self.gs), 1), self.dev
        self.rec = torch.empty(n * REC_BYTES, dtype=torch.uint8, device=dev)
        self.count = torch.zeros(n, dtype=torch.int32, device=dev)
        self.rect = torch.zeros(n * 4, dtype=torch.int16, device=dev)
        self.cull = torch.empty(n * 12, dtype=torch.float32, device=dev)
        self.sort_keys = torch.empty(n, dtype=torch.int64, device=dev)
        self.screen = torch.zeros(n * 9, dtype=torch.float64, device=dev)

    def _density_step(self, it: int) -> None:
        """loop.py:226-233 after the optimiser steps of iteration ``it``."""
        from .densify import densify_and_prune, reset_opacity
        cfg = self.cfg
        if it >= cfg.densify_until_iter:
            return
        self.dstate.update(self.grads.visible_count, self.grads.densify_norm)
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
        from .splat import _preprocess
        kmax = 0
        for v in range(len(self.cameras)):
            proj = self._project(v)
            kmax = max(kmax, int(proj.count.sum().item()))
        self._alloc_entries(int(kmax * 1.2) + 4096)

    def _alloc_entries(self, cap):
        self.capacity = cap
        self.entries = torch.empty(cap, dtype=torch.int32, device=self.dev)
        cam0 = self.cameras[0]
        tx = (int(cam0.width) + TILE_PX - 1) // TILE_PX
        ty = (int(cam0.height) + TILE_PX - 1) // TILE_PX
        self.tile_starts = torch.empty(tx * ty + 1, dtype=torch.int64, device=self.dev)
        nbytes = _lib.load().hgs_tiles_scratch_bytes(len(self.gs), cap, tx * ty)
        self.tiles_scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        self.tx, self.ty = tx, ty

    def _project(self, v) -> ProjectedGaussians:
        cam = self.cameras[v]
        ps = _lib.HGSProjected()
        ps.rec, ps.count, ps.rect, ps.cull = (_lib.ptr(self.rec), _lib.ptr(self.count), _lib.ptr(self.rect),
                                              _lib.ptr(self.cull))
        ps.sort_keys, ps.tile_diff = _lib.ptr(self.sort_keys), _lib.ptr(self.tile_diff)
        _lib.call("hgs_preprocess", _lib.ptr(self.cam_dev[v]), int(cam.width), int(cam.height),
                  ctypes.byref(self.gs.struct()), TILE_PX, ctypes.byref(ps), _stream_ptr(self.dev))
        return ProjectedGaussians(len(self.gs), self.rec, self.count, self.rect, None, int(cam.width),
                                  int(cam.height), TILE_PX, self.cull, self.sort_keys, self.tile_diff)

    def _tiles(self, proj) -> TileBins:
        ts = _lib.HGSTiles()
        ts.tiles_x, ts.tiles_y, ts.tile_px, ts.capacity = self.tx, self.ty, TILE_PX, self.capacity
        ts.entries, ts.tile_starts, ts.counters = _lib.ptr(self.entries), _lib.ptr(self.tile_starts), _lib.ptr(self.counters)
        ts.scratch, ts.scratch_bytes = _lib.ptr(self.tiles_scratch), self.tiles_scratch.numel()
        _lib.call("hgs_build_tiles", ctypes.byref(proj.struct()), len(self.gs), ctypes.byref(ts), _stream_ptr(self.dev))
        self.overflow += self.counters[2:3]
        return TileBins(self.tile_starts, self.entries, self.tx, self.ty, TILE_PX, proj)

    def mesh_layer(self, v) -> Optional[MeshLayer]:
        """Texture lookup over the cached fragments (loop.py:189-199)."""
        if self.mesh is None:
            return None
        from .meshraster import sample_texture
        fr = self.frags[v]
        color = sample_texture(self.mesh.texture, fr.uv, fr.triangle_id)
        return MeshLayer(color, fr.depth, fr.triangle_id)

    def view_grads(self, v: int, it: int, grad_scale: float):
        """Forward + loss + backward of one view, accumulated (x grad_scale)
        into the bucket.  Returns the device loss scalars of this view."""
        cam = self.cameras[v]
        w, h = int(cam.width), int(cam.height)
        layer = self.mesh_layer(v)
        proj = self._project(v)
        tiles = self._tiles(proj)
        color, depth, trans, final_t, last, _ = _blend(proj, tiles, w, h, layer, self.bg)
        fr = self.frags[v]
        covered = fr.triangle_id if fr is not None else None
        bd, g_ih, g_im, g_t = composite_loss(self.images[v], color, layer.color if layer else None, covered, trans,
                                             it, self.cfg, grad_scale=grad_scale)
        ctx = RenderCtx(self.gs, cam, proj, tiles, layer, self.bg, final_t, last, self.cam_dev[v])
        self.screen.zero_()
        mesh_grad = None
        if layer is not None:
            mesh_grad = g_im if g_im is not None else torch.zeros(h, w, 3, dtype=torch.float32, device=self.dev)
        screen_backward(ctx, g_ih, g_t, self.screen, mesh_grad, accumulate_mesh=True)
        chain_backward(ctx, self.screen, self.grads, scale=1.0, accumulate=True)
        if layer is not None and self.tex_grad is not None:
            from .meshraster import texture_backward
            texture_backward(fr, mesh_grad, tuple(self.mesh.texture.shape[:2]), out=self.tex_grad)
        return bd.scalars

    def step(self, it: int, views: Sequence[int]) -> torch.Tensor:
        """One optimisation step over the global batch ``views`` (this rank
        renders its shard).  Returns the batch-mean loss scalars (device)."""
        nb = len(views)
        mine = [views[i] for i in shard_views(nb, self.rank, self.world)]
        self.bucket.zero_()
        self.grads.visible.zero_()
        self.loss_sum.zero_()
        self.overflow.zero_()
        for v in mine:
            self.loss_sum += self.view_grads(v, it, 1.0 / nb)
        if int(self.overflow.item()):
            self._size_entries()
            return self.step(it, views)
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
            self._density_step(it)
        return self.loss_sum
