"""The split visibility pass on the device and the reference's backend
strategy objects (renderer.py:593-700), plus the per-sample pass and a
progressive render loop (renderer.py:743-861) that drive it.

``VisibilityEngine`` is the hot path: rays already in HBM ->
phase-1 gather (fp64 classify + ordered compaction into outer/inner
queues) -> per-ray OR seeded with the hybrid BVH result -> fused
encode+MLP+threshold per family (tcgen05) -> occlusion bytes per ray.
Every launch is stream-ordered with no host synchronisation, so a fixed
ray count can be captured once in a CUDA graph and replayed.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .scene import QueryRecords, Scene, ShadowRays

GAMMA = 1.0 / 2.2
PSNR_SENTINEL = math.inf


def _torch():
    import torch
    return torch


def rays_to_device(rays: ShadowRays, device):
    torch = _torch()
    o = torch.from_numpy(np.ascontiguousarray(rays.origins, np.float64)).to(device)
    d = torch.from_numpy(np.ascontiguousarray(rays.dirs, np.float64)).to(device)
    t = torch.from_numpy(np.ascontiguousarray(rays.tmaxs, np.float64)).to(device)
    return o, d, t


# record slots per ray the queues start with: a shadow ray meets only a few
# network-routed boxes (C2: 1.16 records per ray, C3: 1.2); the gather bounds
# its writes and reports true totals, so callers grow on overflow
DEFAULT_SLOTS_PER_RAY = 4


class GatherBuffers:
    """Device outputs of nif_gather_dev for up to `n` rays, `slots` record
    slots per ray per queue (default: n_net_obj, the worst case the
    reference allocates, renderer.py:619-624)."""

    def __init__(self, n, n_net_obj, device, interleaved=False, slots=None):
        torch = _torch()
        slots = max(1, n_net_obj) if slots is None else max(1, min(slots, max(1, n_net_obj)))
        cap = max(1, n * slots)
        self.n = n
        self.n_net = max(1, n_net_obj)
        self.slots = slots
        self.cap = cap
        i32 = dict(dtype=torch.int32, device=device)
        f32 = dict(dtype=torch.float32, device=device)
        self.outer_obj = torch.empty(cap, **i32)
        self.outer_ray = torch.empty(cap, **i32)
        self.outer_coord = torch.empty(cap * 4, **f32)
        self.inner_obj = torch.empty(cap, **i32)
        self.inner_ray = torch.empty(cap, **i32)
        self.inner_coord = torch.empty(cap * 4, **f32)
        self.inner_r = torch.empty(cap, **f32)
        self.bvh_occ = torch.empty(max(n, 1), dtype=torch.uint8, device=device)
        self.counts = torch.zeros(4, dtype=torch.int64, device=device)
        self.interleaved = interleaved
        if interleaved:
            self.rec_kind = torch.empty(cap, dtype=torch.uint8, device=device)
            self.rec_obj = torch.empty(cap, **i32)
            self.rec_ray = torch.empty(cap, **i32)
            self.rec_coord = torch.empty(cap * 5, dtype=torch.float64, device=device)
        ws = _lib.lib().nif_gather_workspace_bytes(max(n, 1))
        # zero-filled once: the hot-path gather keeps its counters re-armed
        self.workspace = torch.zeros(ws, dtype=torch.uint8, device=device)
        p = _lib.ptr
        self.out = _lib.GatherOut(
            outer_obj=p(self.outer_obj), outer_ray=p(self.outer_ray),
            outer_coord=p(self.outer_coord), inner_obj=p(self.inner_obj),
            inner_ray=p(self.inner_ray), inner_coord=p(self.inner_coord),
            inner_r=p(self.inner_r), cap_outer=cap, cap_inner=cap,
            rec_kind=p(self.rec_kind) if interleaved else None,
            rec_obj=p(self.rec_obj) if interleaved else None,
            rec_ray=p(self.rec_ray) if interleaved else None,
            rec_coord=p(self.rec_coord) if interleaved else None,
            cap_total=cap if interleaved else 0, bvh_occ=p(self.bvh_occ),
            counts=p(self.counts))


def gather_dev(dscene, route_dev, o, d, t, n, buf: GatherBuffers, stream=None):
    L = _lib.lib()
    L.nif_gather_dev(dscene.view, _lib.ptr(route_dev), _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), n,
                     buf.out, _lib.ptr(buf.workspace), buf.workspace.numel(),
                     _lib.stream_ptr(stream))


def overflowed(buf: GatherBuffers, counts) -> bool:
    """True when the last gather into `buf` emitted more records than its
    queues hold (counts: host copy of buf.counts)."""
    if max(int(counts[0]), int(counts[1])) > buf.cap:
        return True
    return buf.interleaved and int(counts[2]) > buf.cap


def slots_for(counts, n) -> int:
    """Record slots per ray that hold the totals in `counts` (+25 %)."""
    need = max(int(counts[0]), int(counts[1]), int(counts[2]))
    return max(1, -(-(need + need // 4) // max(n, 1)))


def gather_sized(dscene, route_dev, o, d, t, n, n_net, device, interleaved=True):
    """gather_dev into buffers sized from a small per-ray bound, re-run once
    with exact-fit buffers if a queue overflowed; returns (buf, counts)."""
    buf = GatherBuffers(n, n_net, device, interleaved=interleaved, slots=DEFAULT_SLOTS_PER_RAY)
    gather_dev(dscene, route_dev, o, d, t, n, buf)
    counts = buf.counts.cpu().numpy()
    if overflowed(buf, counts):
        buf = GatherBuffers(n, n_net, device, interleaved=interleaved, slots=slots_for(counts, n))
        gather_dev(dscene, route_dev, o, d, t, n, buf)
        counts = buf.counts.cpu().numpy()
    return buf, counts


def gather_queries(scene: Scene, rays: ShadowRays, route: np.ndarray, threads: int = 1):
    """renderer.py:613-644 on the device. Returns (QueryRecords,
    bvh_occluded) with records in the reference's order (ray-major, top-level
    DFS order within a ray). `threads` is accepted for signature parity."""
    torch = _torch()
    ds = scene.device()
    n = len(rays)
    if n == 0:
        return QueryRecords(np.zeros(0, np.uint8), np.zeros(0, np.int32), np.zeros(0, np.int32),
                            np.zeros((0, 5)), 0), np.zeros(0, bool)
    o, d, t = rays_to_device(rays, ds.device)
    n_net = int(np.asarray(route, np.uint8).sum())
    buf, counts = gather_sized(ds, ds.route(route), o, d, t, n, n_net, ds.device)
    m = int(counts[2])
    rec = QueryRecords(kind=buf.rec_kind[:m].cpu().numpy(), obj=buf.rec_obj[:m].cpu().numpy(),
                       ray=buf.rec_ray[:m].cpu().numpy(),
                       coord=buf.rec_coord[:m * 5].view(m, 5).cpu().numpy(),
                       degenerate_count=int(counts[3]))
    return rec, buf.bvh_occ[:n].cpu().numpy().astype(bool)


def label_visible(scene: Scene, records: QueryRecords, rays: ShadowRays) -> np.ndarray:
    """bvh.py:904-916 via nif_label_visible_dev: uint8, 1 = visible."""
    torch = _torch()
    ds = scene.device()
    m = len(records)
    if m == 0:
        return np.zeros(0, np.uint8)
    o, d, t = rays_to_device(rays, ds.device)
    ro = torch.from_numpy(np.ascontiguousarray(records.obj, np.int32)).to(ds.device)
    rr = torch.from_numpy(np.ascontiguousarray(records.ray, np.int32)).to(ds.device)
    vis = torch.empty(m, dtype=torch.uint8, device=ds.device)
    _lib.lib().nif_label_visible_dev(ds.view, _lib.ptr(ro), _lib.ptr(rr), m, _lib.ptr(o),
                                     _lib.ptr(d), _lib.ptr(t), _lib.ptr(vis), _lib.stream_ptr())
    return vis.cpu().numpy()


def oracle_predictor(scene: Scene, records: QueryRecords, rays: ShadowRays,
                     threads: int = 1) -> np.ndarray:
    """renderer.py:647-662: ground-truth answers from per-object trees."""
    return label_visible(scene, records, rays) == 0


class BvhBackend:
    """renderer.py:593-610 on the device (two-level fp64 any-hit)."""

    name = "bvh"

    def occluded(self, scene: Scene, rays: ShadowRays, threads: int = 1) -> np.ndarray:
        torch = _torch()
        ds = scene.device()
        n = len(rays)
        if n == 0:
            return np.zeros(0, bool)
        o, d, t = rays_to_device(rays, ds.device)
        return self.occluded_dev(scene, o, d, t).cpu().numpy().astype(bool)

    def occluded_dev(self, scene: Scene, o, d, t):
        """Device rays in, device uint8 answer out (no host round trip)."""
        torch = _torch()
        ds = scene.device()
        n = int(t.numel())
        out = torch.empty(max(n, 1), dtype=torch.uint8, device=ds.device)
        if n:
            _lib.lib().nif_bvh_occluded_dev(ds.view, _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), n,
                                            _lib.ptr(out), _lib.stream_ptr())
        return out[:n]


class PredictorBackend:
    """renderer.py:665-683: gather, answer records, OR per ray."""

    name = "predictor"

    def __init__(self, predictor, hybrid_threshold: Optional[int] = None):
        self.predictor = predictor
        self.hybrid_threshold = hybrid_threshold
        self.last_records: Optional[QueryRecords] = None

    def occluded(self, scene: Scene, rays: ShadowRays, threads: int = 1) -> np.ndarray:
        route = scene.nif_route_mask(self.hybrid_threshold)
        records, occ = gather_queries(scene, rays, route, threads)
        self.last_records = records
        if len(records):
            rec_occ = self.predictor(scene, records, rays, threads)
            occ = occ.copy()
            occ[records.ray[rec_occ]] = True
        return occ


class OracleBackend(PredictorBackend):
    """renderer.py:686-693: must match BvhBackend pixel for pixel."""

    name = "oracle"

    def __init__(self, hybrid_threshold: Optional[int] = None):
        super().__init__(oracle_predictor, hybrid_threshold)


def _require_occlusion_head(model):
    """nif.py:470-471: visibility needs the occlusion head."""
    if model is not None and model.config.head != "occlusion":
        raise ValueError("model was built with the geometry head")


class VisibilityEngine:
    """Device-resident split visibility pass for one (scene, model, route).

    Buffers are sized for `capacity` rays; `run(n)` enqueues the whole pass
    for the first n rays already in `origins/dirs/tmaxs` and leaves one byte
    per ray in `occ` (1 = shadowed). No host synchronisation inside.

    The record queues hold `slots` records per ray (default
    DEFAULT_SLOTS_PER_RAY, not the n_obj worst case); the gather never
    writes past them and reports the true totals. `checked_run` (and the
    synchronous callers) re-run with grown queues when a batch overflowed;
    `capture` sizes the queues from an eager run of the same rays first.
    """

    def __init__(self, scene: Scene, model, capacity: int, hybrid_threshold=None,
                 impl: int = _lib.IMPL_AUTO, slots: Optional[int] = None):
        torch = _torch()
        _require_occlusion_head(model)
        self.scene = scene
        self.ds = scene.device()
        self.model = model
        self.impl = impl
        self.capacity = capacity
        route = scene.nif_route_mask(hybrid_threshold)
        self.route_np = route
        self.route = self.ds.route(route)
        dev = self.ds.device
        self.origins = torch.empty((capacity, 3), dtype=torch.float64, device=dev)
        self.dirs = torch.empty((capacity, 3), dtype=torch.float64, device=dev)
        self.tmaxs = torch.empty(capacity, dtype=torch.float64, device=dev)
        self.side = torch.cuda.Stream(device=dev)
        self._views = None
        self.graphs = {}
        self._alloc(DEFAULT_SLOTS_PER_RAY if slots is None else slots)

    def _alloc(self, slots):
        torch = _torch()
        dev = self.ds.device
        self.buf = GatherBuffers(self.capacity, int(self.route_np.sum()), dev, slots=slots)
        # the gather writes the hybrid any-hit result straight into the
        # per-ray answer, which the query kernels then OR into
        self.occ = self.buf.bvh_occ
        # per_object sharing: per-family scratch for the bucketed tensor-core query
        self.bucket = None
        if self.model is not None and self.model.outer.n_heads > 1:
            L = _lib.lib()
            nb = int(L.nif_bucket_scratch_bytes(self.buf.cap, self.model.outer.n_obj))
            # zero-filled once: the bucketed query re-zeroes its histogram
            self.bucket = (torch.zeros(nb, dtype=torch.uint8, device=dev),
                           torch.zeros(nb, dtype=torch.uint8, device=dev))
        self.graphs = {}

    def _family_views(self):
        if self._views is None or self.model.outer.dirty or self.model.inner.dirty:
            self._views = (self.model.outer.view(with_fast=True),
                           self.model.inner.view(with_fast=True))
        return self._views

    def load(self, rays: ShadowRays, non_blocking=False):
        torch = _torch()
        n = len(rays)
        if n > self.capacity:
            raise ValueError(f"{n} rays exceed the engine capacity {self.capacity}")
        self.origins[:n].copy_(torch.from_numpy(np.ascontiguousarray(rays.origins, np.float64)),
                               non_blocking=non_blocking)
        self.dirs[:n].copy_(torch.from_numpy(np.ascontiguousarray(rays.dirs, np.float64)),
                            non_blocking=non_blocking)
        self.tmaxs[:n].copy_(torch.from_numpy(np.ascontiguousarray(rays.tmaxs, np.float64)),
                             non_blocking=non_blocking)
        return n

    def run(self, n: int, stream=None):
        self.run_range(0, n, stream)

    def overflowed(self) -> bool:
        """Did the last run emit more records than the queues hold? (syncs)"""
        return overflowed(self.buf, self.counts())

    def checked_run(self, n: int, stream=None):
        """run(n), then (one host read of the record totals) grow the queues
        and re-run if they overflowed; the answer in `occ` is then exact."""
        self.run(n, stream)
        counts = self.counts()
        if overflowed(self.buf, counts):
            self._alloc(slots_for(counts, n))
            self.run(n, stream)

    def _query(self, vo, vi, occ, side_sp, main_sp):
        """Outer family on the side stream, inner on the main one; per_object
        models go through the bucketed tensor-core query."""
        L = _lib.lib()
        b = self.buf
        p = _lib.ptr
        cnt = b.counts.data_ptr()
        if self.bucket is not None and self.impl in (_lib.IMPL_AUTO, _lib.IMPL_TCGEN05):
            L.nif_query_bucketed_dev(vo, p(b.outer_obj), p(b.outer_ray), p(b.outer_coord), None,
                                     cnt, b.cap, occ, None, p(self.bucket[0]), side_sp)
            L.nif_query_bucketed_dev(vi, p(b.inner_obj), p(b.inner_ray), p(b.inner_coord),
                                     p(b.inner_r), cnt + 8, b.cap, occ, None, p(self.bucket[1]),
                                     main_sp)
            return
        L.nif_query_dev(vo, p(b.outer_obj), p(b.outer_ray), p(b.outer_coord), None, cnt, b.cap,
                        occ, None, self.impl, side_sp)
        L.nif_query_dev(vi, p(b.inner_obj), p(b.inner_ray), p(b.inner_coord), p(b.inner_r),
                        cnt + 8, b.cap, occ, None, self.impl, main_sp)

    def run_range(self, s0: int, s1: int, stream=None):
        """The pass over rays [s0, s1) of the resident buffers (ray ids and
        the per-ray answer offset by s0); queues are reused, so ranges on
        one stream run back to back."""
        L = _lib.lib()
        torch = _torch()
        n = s1 - s0
        if n < 0 or (n == 0 and s0 > 0):
            return
        b = self.buf
        sp = _lib.stream_ptr(stream)
        vo = vi = None
        if self.model is not None:
            vo, vi = self._family_views()  # (re)pack before the gather is queued
        out = _lib.GatherOut.from_buffer_copy(b.out)
        out.bvh_occ = b.bvh_occ.data_ptr() + s0
        L.nif_gather_dev(self.ds.view, _lib.ptr(self.route), self.origins.data_ptr() + 24 * s0,
                         self.dirs.data_ptr() + 24 * s0, self.tmaxs.data_ptr() + 8 * s0, n, out,
                         _lib.ptr(b.workspace), b.workspace.numel(), sp)
        if self.model is None:
            return
        occ = self.occ.data_ptr() + s0
        main = stream if stream is not None else torch.cuda.current_stream()
        # the two families are independent: outer on a side stream, inner on
        # the main one, joined before returning (fork/join is graph-capturable)
        self.side.wait_stream(main)
        self._query(vo, vi, occ, self.side.cuda_stream, sp)
        main.wait_stream(self.side)

    def occluded_host(self, ho, hd, ht, hocc, n: int, chunks: int = 4):
        """Host -> visibility -> host with the transfers overlapped: rays in
        pinned host tensors ho/hd (n,3) f64 and ht (n,) f64, answer into the
        pinned uint8 tensor hocc. Chunk k+1 is copied in on a copy stream
        while chunk k is classified and queried; the answer of chunk k is
        copied out as soon as it is final. (The queues must already hold a
        chunk's records: size them with one checked_run first.)"""
        torch = _torch()
        if n > self.capacity:
            raise ValueError(f"{n} rays exceed the engine capacity {self.capacity}")
        self._family_views()
        if not hasattr(self, "_h2d"):
            self._h2d = torch.cuda.Stream(device=self.ds.device)
            self._d2h = torch.cuda.Stream(device=self.ds.device)
        main = torch.cuda.current_stream()
        step = -(-n // max(1, chunks))
        bounds = [(s, min(n, s + step)) for s in range(0, n, step)]
        self._h2d.wait_stream(main)  # previous users of the ray buffers are done
        evs = []
        with torch.cuda.stream(self._h2d):
            for s0, s1 in bounds:
                self.origins[s0:s1].copy_(ho[s0:s1], non_blocking=True)
                self.dirs[s0:s1].copy_(hd[s0:s1], non_blocking=True)
                self.tmaxs[s0:s1].copy_(ht[s0:s1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self._h2d)
                evs.append(ev)
        for (s0, s1), ev in zip(bounds, evs):
            main.wait_event(ev)
            self.run_range(s0, s1, main)
            done = torch.cuda.Event()
            done.record(main)
            self._d2h.wait_event(done)
            with torch.cuda.stream(self._d2h):
                hocc[s0:s1].copy_(self.occ[s0:s1], non_blocking=True)
        main.wait_stream(self._d2h)

    def capture(self, n: int):
        """CUDA-graph the pass for a fixed ray count (replayed by `replay`).
        The rays to replay must already be resident: an eager checked run
        over them sizes the queues before the capture."""
        torch = _torch()
        self._family_views()  # pack outside the capture
        s = torch.cuda.Stream(device=self.ds.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.checked_run(n, s)  # warm (kernel attributes, lazy module load) + sizing
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(n)
        self.graphs[n] = g
        return g

    def counts(self):
        return self.buf.counts.cpu().numpy()


class NativeEngine:
    """The whole pass behind the native engine object (nif_engine_*): host
    rays in, per-ray answer out, one C-ABI call -- what a ctypes stub inside
    the reference binds for PredictorBackend.occluded.
    Pageable numpy rays are staged through the engine's pinned ring (host
    copy threads, upload and device pass of neighbouring chunks overlap)."""

    def __init__(self, scene: Scene, model, capacity: int, hybrid_threshold=None):
        _require_occlusion_head(model)
        self.scene, self.model, self.capacity = scene, model, capacity
        self.ds = scene.device()
        route = scene.nif_route_mask(hybrid_threshold)
        self.route_np = route
        self.route = self.ds.route(route)
        L = _lib.lib()
        # the packs (if the model is dirty) are enqueued on torch's current
        # stream; the engine's streams wait for that stream before reading
        vo = model.outer.view(with_fast=True)
        vi = model.inner.view(with_fast=True)
        h = C.c_void_p()
        L.nif_engine_create(self.ds.view, _lib.ptr(self.route), int(route.sum()), vo, vi,
                            int(capacity), _lib.stream_ptr(), C.byref(h))
        self.handle = h

    def update_model(self):
        """After optimiser steps: repack and point the engine at the blobs
        (the engine waits for the repack's stream)."""
        _lib.lib().nif_engine_update_model(self.handle, self.model.outer.view(with_fast=True),
                                           self.model.inner.view(with_fast=True),
                                           _lib.stream_ptr())

    def info(self) -> dict:
        out = np.zeros(4, np.int64)
        _lib.lib().nif_engine_info(self.handle, out.ctypes.data)
        return {"chunk_rays": int(out[0]), "slots_per_ray": int(out[1]),
                "staging_threads": int(out[2]), "overflow_reruns": int(out[3])}

    def occluded_into(self, origins, dirs, tmaxs, out: np.ndarray, chunks: int = 0):
        """Host arrays in (f64 [n,3], [n,3], [n]), uint8 answer into `out`."""
        n = len(tmaxs)
        if n:
            if self.model.outer.dirty or self.model.inner.dirty:
                self.update_model()
            o = np.ascontiguousarray(origins, np.float64)
            d = np.ascontiguousarray(dirs, np.float64)
            t = np.ascontiguousarray(tmaxs, np.float64)
            _lib.lib().nif_engine_occluded_host(self.handle, o.ctypes.data, d.ctypes.data,
                                                t.ctypes.data, n, out.ctypes.data, int(chunks))
        return out

    def occluded(self, rays: ShadowRays, chunks: int = 0) -> np.ndarray:
        n = len(rays)
        out = np.empty(n, np.uint8)
        self.occluded_into(rays.origins, rays.dirs, rays.tmaxs, out, chunks)
        return out.view(bool)

    def close(self):
        if getattr(self, "handle", None):
            _lib.lib().nif_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


class NifBackend(PredictorBackend):
    """nif.py:486-499: visibility from the learned model, optionally hybrid.
    occluded() (host rays) runs the whole pass behind the native engine
    handle (C-ABI, pinned staging); occluded_dev() (device rays) runs the
    device-resident VisibilityEngine; predict() keeps the record API.
    Engines are cached per (scene, route mask) -- the mask is recomputed on
    every call like the reference's PredictorBackend.occluded, so edits to
    scene.nif_enabled or hybrid_threshold take effect -- keeping the most
    recent few."""

    MAX_ENGINES = 4

    def __init__(self, model, hybrid_threshold: Optional[int] = None,
                 impl: int = _lib.IMPL_AUTO, keep_records: bool = False):
        if model is None:
            raise ValueError("the learned backend needs a model")
        from .nif import infer_records
        self.model = model
        self.impl = impl
        self.keep_records = keep_records

        def predict(scene, records, rays, threads=1):
            return infer_records(model, records, impl)

        super().__init__(predict, hybrid_threshold)
        self.name = "nif" if hybrid_threshold is None else "hybrid"
        from collections import OrderedDict
        self._engines = OrderedDict()

    def _cached(self, kind, scene, n, make):
        route = scene.nif_route_mask(self.hybrid_threshold)
        key = (kind, id(scene), bytes(route))
        eng = self._engines.pop(key, None)
        if eng is not None and (eng.scene is not scene or eng.capacity < n):
            eng = None
        if eng is None:
            eng = make(max(n, 1024))
        self._engines[key] = eng
        while len(self._engines) > self.MAX_ENGINES:
            _, old = self._engines.popitem(last=False)
            if hasattr(old, "close"):
                old.close()
        return eng

    def engine(self, scene: Scene, n: int) -> VisibilityEngine:
        return self._cached("dev", scene, n, lambda cap: VisibilityEngine(
            scene, self.model, cap, self.hybrid_threshold, self.impl))

    def native_engine(self, scene: Scene, n: int) -> NativeEngine:
        return self._cached("host", scene, n, lambda cap: NativeEngine(
            scene, self.model, cap, self.hybrid_threshold))

    def occluded(self, scene: Scene, rays: ShadowRays, threads: int = 1) -> np.ndarray:
        _require_occlusion_head(self.model)
        if self.keep_records:
            return super().occluded(scene, rays, threads)
        n = len(rays)
        if n == 0:
            return np.zeros(0, bool)
        if self.impl not in (_lib.IMPL_AUTO, _lib.IMPL_TCGEN05):
            eng = self.engine(scene, n)
            eng.load(rays)
            eng.checked_run(n)
            return eng.occ[:n].cpu().numpy().astype(bool)
        return self.native_engine(scene, n).occluded(rays)

    def occluded_dev(self, scene: Scene, o, d, t):
        """Device rays in, device uint8 answer out (valid until the next
        call on this scene); the engine's buffers are filled device to
        device. One host read of the record totals guards queue overflow."""
        _require_occlusion_head(self.model)
        n = int(t.numel())
        eng = self.engine(scene, max(n, 1))
        if n:
            eng.origins[:n].copy_(o)
            eng.dirs[:n].copy_(d)
            eng.tmaxs[:n].copy_(t)
            eng.checked_run(n)
        return eng.occ[:n]


def shade_pass_nif(scene: Scene, rays: ShadowRays, predictor, hybrid_threshold=None,
                   threads: int = 1) -> np.ndarray:
    return PredictorBackend(predictor, hybrid_threshold).occluded(scene, rays, threads)


# ---------------------------------------------------------------------------
# per-sample pass and render (renderer.py:743-861)
# ---------------------------------------------------------------------------


def camera_struct(camera) -> _lib.Camera:
    fwd, right, up, tan_half, aspect = camera.basis()
    c = _lib.Camera()
    for k in range(3):
        c.pos[k] = float(camera.position[k])
        c.fwd[k] = float(fwd[k])
        c.right[k] = float(right[k])
        c.up[k] = float(up[k])
    c.tan_half = tan_half
    c.aspect = aspect
    c.width = camera.width
    c.height = camera.height
    return c


class _LightsDev:
    def __init__(self, scene: Scene, device):
        torch = _torch()
        if scene.lights:
            cum, kind, data = scene.light_tables()
        else:
            cum, kind, data = np.ones(1), np.zeros(1, np.uint8), np.zeros((1, 16))
        self.cum = torch.from_numpy(np.ascontiguousarray(cum, np.float64)).to(device)
        self.kind = torch.from_numpy(np.ascontiguousarray(kind, np.uint8)).to(device)
        self.data = torch.from_numpy(np.ascontiguousarray(data, np.float64)).to(device)
        self.view = _lib.LightsView(n_lights=len(scene.lights), pad0=0, kind=_lib.ptr(self.kind),
                                    data=_lib.ptr(self.data), cum=_lib.ptr(self.cum))


def sample_pass_dev(scene: Scene, camera, sample: int, seed: int, sampler="importance",
                    pix0: int = 0, n_pix: Optional[int] = None):
    """renderer.py:743-805 on the device; returns a dict of torch tensors
    for pixels [pix0, pix0 + n_pix) (image-tile sharding)."""
    torch = _torch()
    if sampler not in ("importance", "uniform"):
        raise ValueError(f"unknown sampler {sampler!r}")
    ds = scene.device()
    dev = ds.device
    n = camera.width * camera.height - pix0 if n_pix is None else n_pix
    key = ("lights", str(dev))
    lights = scene._device.get(key)
    if lights is None:
        lights = scene._device[key] = _LightsDev(scene, dev)
    f64 = dict(dtype=torch.float64, device=dev)
    out = {"hit": torch.empty(n, dtype=torch.uint8, device=dev), "t": torch.empty(n, **f64),
           "obj": torch.empty(n, dtype=torch.int32, device=dev),
           "point": torch.empty((n, 3), **f64), "normal": torch.empty((n, 3), **f64),
           "pdir": torch.empty((n, 3), **f64), "ldir": torch.empty((n, 3), **f64),
           "tmax": torch.empty(n, **f64), "pdf": torch.empty(n, **f64),
           "emit": torch.empty((n, 3), **f64)}
    po = _lib.PassOut(**{k: _lib.ptr(v) for k, v in out.items()})
    _lib.lib().nif_sample_pass_dev(ds.view, camera_struct(camera), lights.view, int(seed),
                                   int(sample), 0 if sampler == "importance" else 1, int(pix0),
                                   int(n), po, _lib.stream_ptr())
    return out


def sample_pass(scene: Scene, camera, sample: int, seed: int, threads: int = 1,
                sampler: str = "importance"):
    """renderer.py:743-805 (host arrays, same keys as the reference)."""
    d = sample_pass_dev(scene, camera, sample, seed, sampler)
    out = {k: v.cpu().numpy() for k, v in d.items()}
    out["hit"] = out["hit"].astype(bool)
    return out


def shadow_rays_dev(data, require_emit=True):
    """Cast filter of renderer.py:831-832 (cli.py:170-183 drops the emit
    test): returns (mask, origins, dirs, tmaxs) as device tensors."""
    nl = data["normal"] * data["ldir"]
    cos = (nl[:, 0] + nl[:, 2]) + nl[:, 1]  # np.einsum's pairing (renderer.py:829)
    cast = (data["hit"] != 0) & (cos > 0.0) & (data["pdf"] > 0.0)
    if require_emit:
        cast &= data["emit"].amax(dim=1) > 0.0
    idx = cast.nonzero().squeeze(1)
    return cast, data["point"][idx].contiguous(), data["ldir"][idx].contiguous(), \
        data["tmax"][idx].contiguous()


@dataclass
class RenderConfig:
    spp: int = 16
    sample_offset: int = 0
    seed: Optional[int] = None
    threads: Optional[int] = None


@dataclass
class HdrImage:
    sum: np.ndarray
    count: int
    timings: dict = field(default_factory=dict)

    def mean(self) -> np.ndarray:
        if self.count == 0:
            return np.zeros_like(self.sum)
        return self.sum / self.count

    def merge(self, other: "HdrImage") -> "HdrImage":
        if self.sum.shape != other.sum.shape:
            raise ValueError("image shapes differ")
        return HdrImage(self.sum + other.sum, self.count + other.count)


def render(scene: Scene, camera=None, config: RenderConfig = None, backend=None) -> HdrImage:
    """renderer.py:808-861: progressive direct lighting, one shadow ray
    per pixel sample, visibility from `backend`."""
    torch = _torch()
    config = config or RenderConfig()
    camera = camera or scene.camera
    if camera is None:
        raise ValueError("no camera given and the scene has none")
    backend = backend or BvhBackend()
    seed = scene.seed if config.seed is None else config.seed
    w, h = camera.width, camera.height
    dev = scene.device().device
    buf = torch.zeros((w * h, 3), dtype=torch.float64, device=dev)
    albedo = scene.device().albedo
    on_device = hasattr(backend, "occluded_dev")
    L = _lib.lib()
    t0 = time.perf_counter()
    for s in range(config.sample_offset, config.sample_offset + config.spp):
        data = sample_pass_dev(scene, camera, s, seed)
        cast, o, d, t = shadow_rays_dev(data)
        idx = cast.nonzero().squeeze(1)
        n_cast = int(idx.numel())
        if n_cast == 0:
            continue
        if on_device:  # sample pass -> visibility -> shading, all in HBM
            occ = backend.occluded_dev(scene, o, d, t)
        else:  # generic predictor backends answer on the host
            rays = ShadowRays(o.cpu().numpy(), d.cpu().numpy(), t.cpu().numpy())
            occ = torch.from_numpy(backend.occluded(scene, rays, 1).astype(np.uint8)).to(dev)
        po = _lib.PassOut(**{k: _lib.ptr(v) for k, v in data.items()})
        L.nif_shade_accumulate_dev(po, _lib.ptr(albedo), _lib.ptr(idx), _lib.ptr(occ), n_cast,
                                   _lib.ptr(buf), _lib.stream_ptr())
    img = HdrImage(buf.view(h, w, 3).cpu().numpy(), config.spp)
    img.timings = {"total": time.perf_counter() - t0}
    return img


def render_dev(scene: Scene, backend, spp: int = 1, camera=None, seed=None, sample_offset=0):
    """The renderer's per-sample loop with everything resident: returns the
    fp64 HDR sum buffer as a device tensor (h, w, 3) -- for ms/frame
    measurement and device-side PSNR (psnr_dev)."""
    torch = _torch()
    camera = camera or scene.camera
    seed = scene.seed if seed is None else seed
    dev = scene.device().device
    w, h = camera.width, camera.height
    buf = torch.zeros((w * h, 3), dtype=torch.float64, device=dev)
    albedo = scene.device().albedo
    L = _lib.lib()
    for s in range(sample_offset, sample_offset + spp):
        data = sample_pass_dev(scene, camera, s, seed)
        cast, o, d, t = shadow_rays_dev(data)
        idx = cast.nonzero().squeeze(1)
        n_cast = int(idx.numel())
        if n_cast == 0:
            continue
        occ = backend.occluded_dev(scene, o, d, t)
        po = _lib.PassOut(**{k: _lib.ptr(v) for k, v in data.items()})
        L.nif_shade_accumulate_dev(po, _lib.ptr(albedo), _lib.ptr(idx), _lib.ptr(occ), n_cast,
                                   _lib.ptr(buf), _lib.stream_ptr())
    return buf.view(h, w, 3)


def psnr_dev(a_sum, b_sum, count_a: int, count_b: int) -> float:
    """renderer.py:881-891 on device HDR sums: tonemap to 8 bits, MSE, dB."""
    torch = _torch()

    def tm(x):
        return torch.round(torch.clamp(x, 0.0, 1.0).pow(GAMMA) * 255.0)
    ta, tb = tm(a_sum / max(count_a, 1)), tm(b_sum / max(count_b, 1))
    mse = float(((ta - tb) ** 2).mean())
    if mse == 0.0:
        return PSNR_SENTINEL
    return 10.0 * math.log10(255.0 ** 2 / mse)


def tonemap_srgb8(linear) -> np.ndarray:
    x = np.clip(np.asarray(linear, np.float64), 0.0, 1.0)
    return np.rint(np.power(x, GAMMA) * 255.0).astype(np.uint8)


def psnr(a, b) -> float:
    """renderer.py:881-891 on tonemapped 8-bit images."""
    la = a.mean() if isinstance(a, HdrImage) else np.asarray(a, np.float64)
    lb = b.mean() if isinstance(b, HdrImage) else np.asarray(b, np.float64)
    ta = tonemap_srgb8(la).astype(np.float64)
    tb = tonemap_srgb8(lb).astype(np.float64)
    if ta.shape != tb.shape:
        raise ValueError("image shapes differ")
    mse = float(np.mean((ta - tb) ** 2))
    if mse == 0.0:
        return PSNR_SENTINEL
    return 10.0 * math.log10(255.0 ** 2 / mse)
