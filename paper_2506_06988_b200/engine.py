"""Preallocated frame engine: the whole hybrid frame (mesh raster + texture
fetch + preprocess + tile binning + blend) enqueued on one stream with fixed
buffer addresses, so it can be captured once into a CUDA graph and replayed
per camera.  The functional API in splat.py / meshraster.py allocates per
call like the reference; this is the serving / benchmark path and the
forward half of the training step.

All counts (visible rows M, tile entries K) stay on the device.  The entry
buffer has a capacity; if a frame overflows it, counters[2] is set, and
``check()`` (one tiny device->host read) grows the buffers -- callers
re-render that frame.  ``frame(..., sync_check=True)`` does this
automatically.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np
import torch

from . import _lib
from .scene import CAMERA_BYTES, GaussianSet, TexturedMesh, camera_struct
from .splat import (REC_BYTES, TILE_PX, MeshLayer, ProjectedGaussians, TileBins, _c_f64_3,
                    MASK_VARIANTS)


class HybridRenderer:
    def __init__(self, gs: GaussianSet, mesh: Optional[TexturedMesh], width: int, height: int,
                 background=(0.0, 0.0, 0.0), capacity: Optional[int] = None, keep_state: bool = False,
                 mask=None, collect_stats: bool = False):
        self.gs = gs
        self.mesh = mesh
        self.width, self.height = int(width), int(height)
        self.dev = gs.device
        self.bg = np.asarray(background, dtype=np.float64).reshape(3)
        self.tiles_x = (self.width + TILE_PX - 1) // TILE_PX
        self.tiles_y = (self.height + TILE_PX - 1) // TILE_PX
        self.n_tiles = self.tiles_x * self.tiles_y
        self.keep_state = keep_state
        # the mesh branch forks after preprocess (HGS_MESH_AFTER_PP=0: at the
        # start of the frame): its raster CTAs then fill the gaps of the
        # latency-bound binning chain instead of slowing the preprocess
        # (c3: 770 vs 795 us per frame)
        self._mesh_after_pp = os.environ.get("HGS_MESH_AFTER_PP", "1") != "0"
        # a pure serving renderer (no backward state) builds blend-only bins
        # (hgs.h HGS_TILES_BLEND_ONLY): no fine binning, the blend filters
        # every tile's list out of the super-tile lists and reads only the
        # prefix it walks (c3 792 vs 803 us, c5 2.51 vs 2.93 ms per frame;
        # HGS_BLEND_ONLY=0 turns it off)
        binned = any(((self.tiles_x + (1 << q) - 1) >> q) * ((self.tiles_y + (1 << q) - 1) >> q) <= 512 for q in (2, 3))
        self.blend_only = not keep_state and binned and os.environ.get("HGS_BLEND_ONLY", "1") != "0"
        self.mask = mask
        dev = self.dev
        n = max(len(gs), 1)
        h, w = self.height, self.width
        self.cam_dev = torch.zeros(CAMERA_BYTES, dtype=torch.uint8, device=dev)
        # pinned camera staging ring: a buffer is rewritten only after its
        # previous async H2D has executed (event), so frames can be enqueued
        # back to back without a host sync
        self._cam_ring = [torch.zeros(CAMERA_BYTES, dtype=torch.uint8).pin_memory() for _ in range(4)]
        self._cam_ev = [None] * len(self._cam_ring)
        self._cam_k = 0
        self.cam_host = self._cam_ring[0]
        self.rec = torch.empty(n * REC_BYTES, dtype=torch.uint8, device=dev)
        self.count = torch.zeros(n, dtype=torch.int32, device=dev)
        self.rect = torch.zeros(n * 4, dtype=torch.int16, device=dev)
        self.cull = torch.empty(n * 12, dtype=torch.float32, device=dev)
        self.sort_keys = torch.empty(n, dtype=torch.int64, device=dev)
        self.tile_diff = torch.empty(16 * (self.tiles_x + 1) * (self.tiles_y + 1), dtype=torch.int32, device=dev)
        self.fixup = torch.zeros(h * w + 4, dtype=torch.int32, device=dev)
        self.tile_starts = torch.zeros(self.n_tiles + 1, dtype=torch.int64, device=dev)
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self.counters_host = torch.zeros(4, dtype=torch.int64).pin_memory()
        self.color = torch.empty(h, w, 3, dtype=torch.float32, device=dev)
        self.depth = torch.empty(h, w, dtype=torch.float32, device=dev)
        self.trans = torch.empty(h, w, dtype=torch.float32, device=dev)
        self.final_t = torch.empty(h, w, dtype=torch.float64, device=dev) if keep_state else None
        self.last = torch.empty(h, w, dtype=torch.int32, device=dev) if keep_state else None
        self.mask_out = torch.empty(h, w, dtype=torch.float32, device=dev) if mask is not None else None
        self.stats = torch.zeros(3, dtype=torch.int64, device=dev) if collect_stats else None
        if mesh is not None:
            self.frag_tri = torch.empty(h, w, dtype=torch.int32, device=dev)
            self.frag_depth = torch.empty(h, w, dtype=torch.float64, device=dev)
            self.frag_uv = torch.empty(h, w, 2, dtype=torch.float64, device=dev)
            self.mesh_color = torch.empty(h, w, 3, dtype=torch.float32, device=dev)
            nbytes = _lib.load().hgs_raster_scratch_bytes(len(mesh.vertices), mesh.n_faces, w, h)
            self.raster_scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.capacity = 0
        self._alloc_entries(capacity if capacity is not None else 16 * n)
        self.graph = None
        self._exec = self._exec_alt = None
        self._alt_out = None
        self._side = None

    # ------------------------------------------------------------------
    def _alloc_entries(self, capacity: int):
        capacity = max(int(capacity), 1024)
        self.capacity = capacity
        self.entries = torch.empty(capacity, dtype=torch.int32, device=self.dev)
        nbytes = _lib.load().hgs_tiles_scratch_bytes(len(self.gs), capacity, self.n_tiles)
        self.tiles_scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        self.ready = torch.zeros(_lib.READY_INTS, dtype=torch.int32, device=self.dev)
        self._drop_exec()
        self.graph = None

    def set_camera(self, cam) -> None:
        """H2D of the 200-byte camera struct from pinned memory (async)."""
        s = camera_struct(cam)
        raw = np.frombuffer(bytes(s), dtype=np.uint8)
        k = self._cam_k
        self._cam_k = (k + 1) % len(self._cam_ring)
        if self._cam_ev[k] is not None:
            self._cam_ev[k].synchronize()  # its previous upload has been consumed
        self.cam_host = self._cam_ring[k]
        self.cam_host.numpy()[:len(raw)] = raw
        self.cam_dev.copy_(self.cam_host, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.dev))
        self._cam_ev[k] = ev

    def render_to_host(self, cam, out_color: torch.Tensor, out_depth: Optional[torch.Tensor] = None,
                       out_trans: Optional[torch.Tensor] = None) -> torch.cuda.Event:
        """Serving path: camera H2D, one graph replay, and the D2H of the
        colour image (and, when given, the depth and transmittance images --
        the reference's RenderOutputs) into the pinned host tensors (H x W x 3
        / H x W fp32) on a copy stream, so the transfer overlaps the next
        frame.  Two frame graphs alternate between two sets of output images
        (no device-side snapshot copies): frame i+1 renders into the set frame
        i is not copying out of.  Returns the event that marks the copies
        complete (the caller must not reuse the host tensors before)."""
        if self.graph is None:
            self.capture()
        if getattr(self, "_copy", None) is None:
            self._copy = torch.cuda.Stream(self.dev)
            self._snap_ev = [None, None]
            self._snap_k = 0
        if self._alt_out is None:
            self._alt_out = (torch.empty_like(self.color), torch.empty_like(self.depth), torch.empty_like(self.trans))
        if self._exec_alt is None:
            self.capture(out_set=1)
        k = self._snap_k
        self._snap_k ^= 1
        main = torch.cuda.current_stream(self.dev)
        if self._snap_ev[k] is not None:
            main.wait_event(self._snap_ev[k])  # the previous D2H out of this output set is done
        self.set_camera(cam)
        self.replay(out_set=k)
        dev_out = self._out3(k)
        pairs = [(out_color, dev_out[0]), (out_depth, dev_out[1]), (out_trans, dev_out[2])]
        ready = torch.cuda.Event()
        ready.record(main)
        self._copy.wait_event(ready)
        with torch.cuda.stream(self._copy):
            for host, src in pairs:
                if host is not None:
                    host.copy_(src, non_blocking=True)
        done = torch.cuda.Event()
        done.record(self._copy)
        self._snap_ev[k] = done
        return done

    def _out3(self, out_set: int):
        """(colour, depth, transmittance) device images of output set 0 (the
        public ones) or 1 (the serving path's second set)."""
        return (self.color, self.depth, self.trans) if out_set == 0 else self._alt_out

    def _structs(self):
        ps = _lib.HGSProjected()
        ps.rec, ps.count, ps.rect = _lib.ptr(self.rec), _lib.ptr(self.count), _lib.ptr(self.rect)
        ps.cull = _lib.ptr(self.cull)
        ps.sort_keys, ps.tile_diff = _lib.ptr(self.sort_keys), _lib.ptr(self.tile_diff)
        ts = _lib.HGSTiles()
        ts.tiles_x, ts.tiles_y, ts.tile_px, ts.capacity = self.tiles_x, self.tiles_y, TILE_PX, self.capacity
        ts.entries, ts.tile_starts, ts.counters = _lib.ptr(self.entries), _lib.ptr(self.tile_starts), _lib.ptr(self.counters)
        ts.scratch, ts.scratch_bytes = _lib.ptr(self.tiles_scratch), self.tiles_scratch.numel()
        ts.ready = _lib.ptr(self.ready)
        # a pure serving renderer (no backward state) needs only the images:
        # blend-only bins skip the fine binning, the blend filters the
        # super-tile lists itself and reads only the prefix it walks (hgs.h)
        if self.blend_only:
            ts.flags = _lib.TILES_BLEND_ONLY
        return ps, ts

    def enqueue(self, rasterize_mesh: bool = True, mesh_layer: Optional[MeshLayer] = None, out_set: int = 0) -> None:
        """Enqueue one frame for the camera currently in cam_dev.

        The mesh layer (raster + texture fetch) does not depend on the
        Gaussians: it runs on a side stream forked from the current one after
        the preprocess, overlapping the tile binning, and joins the chain
        before the fine binning / the blend (the fork/join is captured into
        the CUDA graph as well)."""
        L = _lib.load()
        main = torch.cuda.current_stream(self.dev)
        st = main.cuda_stream
        w, h = self.width, self.height
        ml = _lib.HGSMeshLayer()
        joined = None
        side_branch = self.mesh is not None and mesh_layer is None
        ps, ts = self._structs()
        if side_branch:
            if self._side is None:
                self._side = torch.cuda.Stream(self.dev)
                self._ev_fork, self._ev_join = torch.cuda.Event(), torch.cuda.Event()
            if self._mesh_after_pp:
                _lib.check(L.hgs_preprocess(_lib.ptr(self.cam_dev), w, h, ctypes.byref(self.gs.struct()), TILE_PX,
                                            ctypes.byref(ps), st), "preprocess")
            self._ev_fork.record(main)
            self._side.wait_event(self._ev_fork)
        elif mesh_layer is not None:
            ml = mesh_layer.struct()
        # the mesh branch (raster + texture fetch) runs on a side stream and
        # joins the Gaussian chain before the blend (hgs_tiles.join_event)
        if side_branch:
            side = self._side.cuda_stream
            if rasterize_mesh:
                fr = _lib.HGSFragments()
                fr.triangle_id, fr.depth, fr.uv = _lib.ptr(self.frag_tri), _lib.ptr(self.frag_depth), _lib.ptr(self.frag_uv)
                _lib.check(L.hgs_rasterize_fragments(_lib.ptr(self.cam_dev), w, h, ctypes.byref(self.mesh.struct()),
                                                     ctypes.byref(fr), _lib.ptr(self.raster_scratch),
                                                     self.raster_scratch.numel(), side), "rasterize_fragments")
            tex = self.mesh.texture
            _lib.check(L.hgs_sample_texture(_lib.ptr(tex), tex.shape[0], tex.shape[1], _lib.ptr(self.frag_uv),
                                            _lib.ptr(self.frag_tri), w * h, _lib.ptr(self.mesh_color), side),
                       "sample_texture")
            self._ev_join.record(self._side)
            joined = self._ev_join
            ml.color, ml.depth, ml.triangle_id = _lib.ptr(self.mesh_color), _lib.ptr(self.frag_depth), _lib.ptr(self.frag_tri)
        # the Gaussian chain; the mesh branch joins it inside hgs_build_tiles,
        # right before the fine binning (hgs_tiles.join_event), so the blend
        # depends on the fine binning alone and starts on its published quads
        ts.join_event = joined.cuda_event if joined is not None else None
        if not (side_branch and self._mesh_after_pp):
            _lib.check(L.hgs_preprocess(_lib.ptr(self.cam_dev), w, h, ctypes.byref(self.gs.struct()), TILE_PX,
                                        ctypes.byref(ps), st), "preprocess")
        _lib.check(L.hgs_build_tiles(ctypes.byref(ps), len(self.gs), ctypes.byref(ts), st), "build_tiles")
        out = _lib.HGSBlendOut()
        oc, od, ot = self._out3(out_set)
        out.color, out.depth, out.transmittance = _lib.ptr(oc), _lib.ptr(od), _lib.ptr(ot)
        out.final_t, out.last = _lib.ptr(self.final_t), _lib.ptr(self.last)
        variant, k = 0, 20.0
        if self.mask is not None:
            variant, k = MASK_VARIANTS[self.mask[0]], float(self.mask[1])
            out.mask = _lib.ptr(self.mask_out)
        out.stats = _lib.ptr(self.stats)
        out.fixup = _lib.ptr(self.fixup)
        _lib.check(L.hgs_blend_forward(ctypes.byref(ps), ctypes.byref(ts), w, h, ctypes.byref(ml), _c_f64_3(self.bg),
                                       variant, k, ctypes.byref(out), st), "blend_forward")

    def check(self) -> tuple:
        """(M, K, overflow); grows the entry buffer on overflow."""
        self.counters_host.copy_(self.counters, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        m, k, ovf = (int(x) for x in self.counters_host[:3])
        if ovf:
            self._alloc_entries(int(k * 1.25) + 1024)
        return m, k, bool(ovf)

    def frame(self, cam, rasterize_mesh: bool = True, sync_check: bool = True):
        self.set_camera(cam)
        while True:
            self.enqueue(rasterize_mesh)
            if not sync_check:
                return
            _, _, ovf = self.check()
            if not ovf:
                return

    # CUDA graph of one frame (camera read from cam_dev at replay time) --------
    def capture(self, rasterize_mesh: bool = True, out_set: int = 0) -> None:
        """Capture one frame into a CUDA graph (out_set: which output images
        it writes, see render_to_host).  The Gaussian chain (preprocess ->
        binning -> blend) is captured from a high-priority stream and the mesh
        branch from a normal one, and the graph is instantiated with per-node
        priorities (hgs_graph_instantiate): when the two branches compete for
        SMs, the critical path's CTAs are scheduled first.  HGS_GRAPH_PRIO=0
        instantiates without priorities."""
        import os
        prio = os.environ.get("HGS_GRAPH_PRIO", "1") != "0"
        s = torch.cuda.Stream(self.dev, priority=-1 if prio else 0)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            self.enqueue(rasterize_mesh, out_set=out_set)  # warm (lazy attributes, occupancy queries)
        torch.cuda.current_stream(self.dev).wait_stream(s)
        torch.cuda.synchronize(self.dev)
        self._drop_exec(out_set)
        g = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.graph(g, stream=s):
            self.enqueue(rasterize_mesh, out_set=out_set)
        ex = ctypes.c_void_p()
        _lib.call("hgs_graph_instantiate", ctypes.c_void_p(int(g.raw_cuda_graph())), 1 if prio else 0,
                  ctypes.byref(ex))
        if out_set == 0:
            self.graph, self._exec = g, ex
        else:
            self._graph_alt, self._exec_alt = g, ex

    def _drop_exec(self, out_set: Optional[int] = None) -> None:
        """Destroy the instantiated graph(s) of one output set (None: both)."""
        for k in ((0, 1) if out_set is None else (out_set,)):
            name = "_exec" if k == 0 else "_exec_alt"
            ex = getattr(self, name, None)
            if ex is not None and ex.value:
                torch.cuda.synchronize(self.dev)
                _lib.call("hgs_graph_exec_destroy", ex)
            setattr(self, name, None)

    def __del__(self):
        try:
            self._drop_exec()
        except Exception:
            pass

    def replay(self, out_set: int = 0) -> None:
        _lib.call("hgs_graph_launch", self._exec if out_set == 0 else self._exec_alt,
                  torch.cuda.current_stream(self.dev).cuda_stream)

    # views for the API / backward ----------------------------------------
    def projected(self) -> ProjectedGaussians:
        return ProjectedGaussians(len(self.gs), self.rec, self.count, self.rect, None, self.width,
                                  self.height, TILE_PX, self.cull, self.sort_keys, self.tile_diff)

    def tiles(self) -> TileBins:
        if self.blend_only:
            raise RuntimeError("HybridRenderer(keep_state=False) builds blend-only bins (no tile entries): "
                               "use keep_state=True for TileBins / the backward")
        return TileBins(self.tile_starts, self.entries, self.tiles_x, self.tiles_y, TILE_PX, self.projected(),
                        counters=self.counters, capacity=int(self.entries.numel()), ready=self.ready)

    def layer(self) -> Optional[MeshLayer]:
        if self.mesh is None:
            return None
        return MeshLayer(self.mesh_color, self.frag_depth, self.frag_tri)
