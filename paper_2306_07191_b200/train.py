"""Online training on the device: sample collection (BVH labels), the
per-batch optimiser step and the epoch loop (nif.py:507-795).

Samples stay in HBM. The epoch loop reproduces the reference's schedule
exactly -- per-epoch RNG `default_rng(SeedSequence([seed, 0x7472])
.spawn(epochs)[e])`, outer family permuted first then inner with the same
generator, batches `perm[k:k+bs]` -- and on one GPU every full batch is a
replay of a captured three-launch step (batch counts + Adam step counters,
fused forward/backward + grid scatter, dense Adam over touched grids + MLP)
with no host synchronisation until the losses are read back after the last
epoch; the host draws the next permutation while the GPU replays.

Data parallel (torch.distributed over NCCL): samples are collected per
rank on its own band of pixel rows and all-gathered into the reference's
global order, so every rank holds the same sample set and draws the same
global permutation; rank r processes rows r, r+W, r+2W, ... of each global
batch (per-object normalisation uses the global batch counts), one
all-reduce per step sums the exchange buffer [input gradients of the batch
rows | MLP gradients] (see _Sink), every rank scatters the whole batch
into its grids and applies the identical Adam update, so replicas stay
identical without a broadcast.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .nif import NifModel
from .scene import Scene


def _torch():
    import torch
    return torch


@dataclass
class SampleSet:
    """nif.py:507-529, arrays as device tensors (host copies on demand)."""

    head: str
    outer_obj: object
    outer_coord: object   # (n, 4) f64
    outer_label: object   # (n,) f32
    outer_ray: object
    inner_obj: object
    inner_coord: object   # (m, 5) f64
    inner_label: object
    inner_ray: object
    n_rays: int = 0
    stats: dict = field(default_factory=dict)

    @property
    def n_outer(self) -> int:
        return int(self.outer_obj.shape[0])

    @property
    def n_inner(self) -> int:
        return int(self.inner_obj.shape[0])

    def host(self):
        return {k: getattr(self, k).cpu().numpy() for k in (
            "outer_obj", "outer_coord", "outer_label", "outer_ray", "inner_obj", "inner_coord",
            "inner_label", "inner_ray")}

    @staticmethod
    def from_host(d: dict, head="occlusion", device=None) -> "SampleSet":
        torch = _torch()
        dev = device or torch.device("cuda", torch.cuda.current_device())
        dt = {"outer_obj": np.int64, "inner_obj": np.int64, "outer_ray": np.int64,
              "inner_ray": np.int64, "outer_coord": np.float64, "inner_coord": np.float64,
              "outer_label": np.float32, "inner_label": np.float32}
        t = {k: torch.from_numpy(np.ascontiguousarray(d[k], dt[k])).to(dev) for k in dt}
        return SampleSet(head, **t)


def collect_samples(scene: Scene, camera=None, spp: int = 4, sampler: str = "importance",
                    labeler=None, seed: Optional[int] = None,
                    threads: Optional[int] = None, group=None,
                    sample_offset: int = 0) -> SampleSet:
    """nif.py:569-674 on the device: per sample index, the primary pass,
    every hit pixel's shadow ray (no cosine filter), the gather in the
    reference's record order and per-object BVH labels (1 = visible).
    labeler="geometry" follows the primary rays instead (uniform sampler,
    camera origin, infinite t_max) and labels each record with the closest
    hit in its own object (unit normal, t / diagonal), keeping hit rows.

    Under torch.distributed (or with `group`), rank r traces only its own
    band of pixel rows (parallel.tile_pixels) and one ordered all-gather
    per array rebuilds the reference's global order -- sample-major, then
    ray-major across the bands in rank order (nif.py:606-647) -- so every
    rank ends with the single-process SampleSet. sample_offset shifts the
    sample indices (and the ray ids) -- one pass of an online schedule."""
    torch = _torch()
    from .parallel import allgather_ordered, tile_pixels, world_rank
    from .pipeline import gather_sized, sample_pass_dev
    camera = camera or scene.camera
    if camera is None:
        raise ValueError("no camera given and the scene has none")
    if sampler not in ("importance", "uniform"):
        raise ValueError(f"unknown sampler {sampler!r}")
    if labeler not in (None, "geometry"):
        raise NotImplementedError("custom labeler callables are not on the device path")
    head = "geometry" if labeler == "geometry" else "occlusion"
    if head == "occlusion" and not scene.lights:
        raise ValueError("sample collection needs at least one light")
    seed = scene.seed if seed is None else seed
    ds = scene.device()
    dev = ds.device
    route = scene.nif_enabled.copy()
    n_pix_all = camera.width * camera.height
    world, rank = world_rank(group)
    pix0, n_pix = tile_pixels(camera.width, camera.height, rank, world)
    keys = ("oo", "oc", "ol", "or_", "io", "ic", "il", "ir")
    lt = () if head == "occlusion" else (4,)
    tails = {"oo": ((), torch.int64), "oc": ((4,), torch.float64), "ol": (lt, torch.float32),
             "or_": ((), torch.int64), "io": ((), torch.int64), "ic": ((5,), torch.float64),
             "il": (lt, torch.float32), "ir": ((), torch.int64)}
    # one (possibly empty) tensor per sample index and array: the segments of
    # the ordered all-gather
    acc = {k: [] for k in keys}
    stat = torch.zeros(3, dtype=torch.int64)  # rays, shadow rays, degenerate queries
    L = _lib.lib()
    cam_pos = torch.from_numpy(np.ascontiguousarray(
        np.broadcast_to(np.asarray(camera.position, np.float64), (n_pix, 3)))).to(dev)
    inf_tmax = torch.full((n_pix,), math.inf, dtype=torch.float64, device=dev)

    def empty(k):
        tail, dt = tails[k]
        return torch.zeros((0,) + tail, dtype=dt, device=dev)

    for s in range(sample_offset, sample_offset + spp):
        got = {}
        data = sample_pass_dev(scene, camera, s, seed,
                               "uniform" if head == "geometry" else sampler, pix0, n_pix)
        if head == "geometry":
            idx = torch.arange(n_pix, device=dev)
            n = n_pix
            o, d, t = cam_pos, data["pdir"].contiguous(), inf_tmax
        else:
            mask = data["hit"] != 0
            idx = mask.nonzero().squeeze(1)
            n = int(idx.numel())
            o = data["point"][idx].contiguous()
            d = data["ldir"][idx].contiguous()
            t = data["tmax"][idx].contiguous()
        m = 0
        if n:
            buf, counts = gather_sized(ds, ds.route(route), o, d, t, n, int(route.sum()), dev)
            m = int(counts[2])
            stat[1] += n
            stat[2] += int(counts[3])
        if m:
            stat[0] += n
            rec_obj = buf.rec_obj[:m]
            rec_ray = buf.rec_ray[:m]
            if head == "geometry":
                lab = torch.empty((m, 4), dtype=torch.float32, device=dev)
                keep = torch.empty(m, dtype=torch.uint8, device=dev)
                L.nif_label_geometry_dev(ds.view, _lib.ptr(rec_obj), _lib.ptr(rec_ray), m,
                                         _lib.ptr(o), _lib.ptr(d), float(scene.diagonal),
                                         _lib.ptr(lab), _lib.ptr(keep), _lib.stream_ptr())
                keep = keep != 0
            else:
                vis = torch.empty(m, dtype=torch.uint8, device=dev)
                L.nif_label_visible_dev(ds.view, _lib.ptr(rec_obj), _lib.ptr(rec_ray), m,
                                        _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), _lib.ptr(vis),
                                        _lib.stream_ptr())
                lab, keep = vis.float(), None
            kind = buf.rec_kind[:m]
            coord = buf.rec_coord[:m * 5].view(m, 5)
            # global ray id: sample-major over the whole image (nif.py:640)
            ray_ids = s * n_pix_all + pix0 + idx
            for k, (ko, kc, kl, kr), width in ((0, ("oo", "oc", "ol", "or_"), 4),
                                               (1, ("io", "ic", "il", "ir"), 5)):
                selm = kind == k
                if keep is not None:
                    selm &= keep
                sel = selm.nonzero().squeeze(1)
                got[ko] = rec_obj[sel].long()
                got[kc] = coord[sel, :width].contiguous()
                got[kl] = lab[sel]
                got[kr] = ray_ids[rec_ray[sel].long()]
        for k in keys:
            acc[k].append(got.get(k, empty(k)))

    if world > 1:
        import torch.distributed as dist
        st = stat.to(dev)
        dist.all_reduce(st, group=group)
        stat = st.cpu()
        for k in keys:
            acc[k] = allgather_ordered(acc[k], group)

    def cat(k):
        parts = [a for a in acc[k] if a.shape[0]]
        return torch.cat(parts).contiguous() if parts else empty(k)

    out = SampleSet(head, *(cat(k) for k in keys), n_rays=int(stat[0]))
    out.stats = {"pixel_samples": spp * n_pix_all, "shadow_rays": int(stat[1]),
                 "degenerate_queries": int(stat[2]),
                 "outer_per_object": np.bincount(out.outer_obj.cpu().numpy(),
                                                 minlength=scene.n_objects),
                 "inner_per_object": np.bincount(out.inner_obj.cpu().numpy(),
                                                 minlength=scene.n_objects)}
    return out


collect_samples_dev = collect_samples


class _Step:
    """Launch helper for one family's optimiser step."""

    def __init__(self, model: NifModel, which: str):
        torch = _torch()
        self.model = model
        self.fam = model.family(which)
        self.sq = torch.zeros(1, dtype=torch.float64, device=model.device)
        # the flat parameter buffers never move: build the C views once
        self.fv = self.fam.view()
        self.tv = self.fam.train_view()

    def run(self, obj, coord, label, idx, n_rows, stream=None, idx_ptr=None):
        """One optimiser step over rows idx[0:n_rows] (device tensors; or a raw
        device pointer idx_ptr into an int64 row list); leaves this batch's
        squared-error sum added into self.sq. (Data-parallel steps go
        through _Sink.)"""
        L = _lib.lib()
        fam, model = self.fam, self.model
        sp = _lib.stream_ptr(stream)
        fv, tv = self.fv, self.tv
        p = _lib.ptr
        ip = idx_ptr if idx_ptr is not None else p(idx)
        L.nif_batch_counts_dev(p(obj), ip, n_rows, fam.n_obj, p(fam.counts), sp)
        L.nif_train_fwdbwd_dev(fv, tv, p(obj), p(coord), p(label), ip, n_rows, 0, 1,
                               p(self.sq), sp)
        a = model.config.adam
        L.nif_adam_dev(fv, tv, model.learning_rate, a.beta1, a.beta2, a.epsilon, sp)
        fam.dirty = True


class _Sink:
    """Gradient routing of one family's step when the grid scatter is not
    fused into the forward/backward kernel: data parallel and / or
    deterministic.

    One flat fp32 exchange buffer per family, ``comm = [dx | mlp]``:
    ``dx[g, k]`` is the input gradient of global batch row g (written only by
    the rank that owns row g, zero elsewhere) and ``mlp`` the MLP gradients
    in the family's [w | pad | b] layout. Per optimiser step: zero comm,
    fused forward/backward of this rank's rows into it, ONE all-reduce
    (sum) of comm, then on every rank the grid scatter of *all* batch rows
    from dx (grids.py:171-202; identical on every rank, deterministic mode
    sums each cell in np.add.at's order) and the MLP gradients copied into
    the family buffer, then the same dense Adam everywhere -- replicas stay
    identical without a broadcast. Exchanged per step: bs x IN + n_mlp
    floats (outer 2^11 x 6 + 4,673; inner 2^12 x 13 + 5,425), independent
    of how many objects the batch touches, against 1.6 MB / 0.7 MB per
    touched object for a dense grid-gradient all-reduce."""

    def __init__(self, step: "_Step", bs: int, world: int, rank: int, group, deterministic: bool,
                 scatter_mode: Optional[int] = None):
        torch = _torch()
        L = _lib.lib()
        fam = step.fam
        dev = step.model.device
        self.step, self.bs, self.world, self.rank, self.group = step, bs, world, rank, group
        self.det = bool(deterministic)
        # Every rank scatters the whole batch into its own replica, so the
        # scatter must not depend on the atomics' order or the replicas would
        # drift apart in the last bits: deterministic=True uses the sorted
        # scatter (np.add.at's order), data parallel otherwise the
        # order-independent fixed-point one (about the atomic scatter's cost)
        self.scatter_mode = 1 if self.det else (2 if group is not None else 0)
        if scatter_mode is not None:
            self.scatter_mode = scatter_mode
        self.IN = int(fam.dims[0])
        self.dx_len = (bs * self.IN + 63) // 64 * 64
        off_w = fam.offsets["w"][0]
        off_b, size_b = fam.offsets["b"]
        self.n_mlp = off_b - off_w + size_b
        self.comm = torch.zeros(self.dx_len + self.n_mlp, dtype=torch.float32, device=dev)
        self.dx = self.comm[:self.dx_len]
        self.mlp = self.comm[self.dx_len:]
        self.grad_mlp = fam.grad[off_w:off_w + self.n_mlp]
        self.part = self.ws = None
        self.part_n = 0
        if self.scatter_mode:
            nb = int(L.nif_grid_scatter_ws_bytes(step.fv, step.tv, bs, self.scatter_mode))
            self.ws = torch.zeros(max(nb, 1), dtype=torch.uint8, device=dev)
        if self.det:
            self.part_n = int(L.nif_train_part_floats(step.fv, step.tv, bs))
            self.part = torch.empty(max(self.part_n, 1), dtype=torch.float32, device=dev)

    def enqueue(self, obj, coord, label, idx_ptr, cursor_ptr, n_rows, sq_ptr, sp):
        """Everything from the batch counts to the gradients, stream-ordered
        on the current stream (capturable: no host synchronisation)."""
        L = _lib.lib()
        st = self.step
        p = _lib.ptr
        self.comm.zero_()
        L.nif_train_prologue_cur_dev(st.fv, st.tv, p(obj), idx_ptr, cursor_ptr, n_rows, sp)
        L.nif_train_fwdbwd_ex_dev(st.fv, st.tv, p(obj), p(coord), p(label), idx_ptr, cursor_ptr,
                                  n_rows, self.rank, self.world, sq_ptr, p(self.dx),
                                  p(self.mlp), p(self.part), self.part_n, sp)
        if self.group is not None:  # one collective per step
            import torch.distributed as dist
            dist.all_reduce(self.comm, group=self.group)
        L.nif_grid_scatter_dev(st.fv, st.tv, p(obj), p(coord), idx_ptr, cursor_ptr, n_rows,
                               p(self.dx), self.scatter_mode, p(self.ws),
                               0 if self.ws is None else int(self.ws.numel()), sp)
        self.grad_mlp.copy_(self.mlp)


class _GraphStep:
    """One family's optimiser step captured as a CUDA graph and replayed
    for every full batch of an epoch: the batch start lives on the device
    (a cursor into a persistent permutation buffer, advanced by the graph
    itself), so an epoch is one async H2D copy of the permutation (from a
    pinned staging buffer) plus one graph launch per batch -- no per-step
    host work and no host synchronisation: the host is free to draw the
    next permutation while the GPU replays this one.

    With a _Sink (data parallel / deterministic) the captured step also
    holds the exchange buffer's all-reduce (NCCL collectives are capturable;
    each family has its own communicator so the two families' graphs can
    replay concurrently). capture=False runs the same launches eagerly per
    batch (gloo, which cannot be captured)."""

    def __init__(self, step: "_Step", obj, coord, label, n: int, bs: int, sink=None,
                 capture: bool = True):
        torch = _torch()
        self.step, self.bs = step, bs
        self.sink, self.capture = sink, capture
        dev = step.model.device
        self.perm = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        self.cursor = torch.zeros(1, dtype=torch.int64, device=dev)
        # two pinned staging buffers: epoch e+1's permutation is written
        # while epoch e's copy may still be queued
        self.host = [torch.empty(max(n, 1), dtype=torch.int64, pin_memory=True) for _ in range(2)]
        self.copied = [None, None]
        self.turn = 0
        self.obj, self.coord, self.label = obj, coord, label
        self.graph = None

    def _enqueue(self, n_rows: int, advance: bool):
        L = _lib.lib()
        st, fam, model = self.step, self.step.fam, self.step.model
        p = _lib.ptr
        sp = _lib.stream_ptr()
        a = model.config.adam
        if self.sink is not None:
            self.sink.enqueue(self.obj, self.coord, self.label, p(self.perm), p(self.cursor),
                              n_rows, p(st.sq), sp)
        else:
            # three launches: counts + step counters, fused fwd/bwd, dense Adam
            # (which also moves the cursor on)
            L.nif_train_prologue_cur_dev(st.fv, st.tv, p(self.obj), p(self.perm),
                                         p(self.cursor), n_rows, sp)
            L.nif_train_fwdbwd_cur_dev(st.fv, st.tv, p(self.obj), p(self.coord), p(self.label),
                                       p(self.perm), p(self.cursor), n_rows, 0, 1, p(st.sq), sp)
        L.nif_adam_units_dev(st.fv, st.tv, model.learning_rate, a.beta1, a.beta2, a.epsilon,
                             p(self.cursor) if advance else None, n_rows, sp)

    def epoch(self, perm_host: np.ndarray):
        """Queue one epoch of this family (returns without synchronising)."""
        torch = _torch()
        n = len(perm_host)
        k = self.turn
        self.turn ^= 1
        if self.copied[k] is not None:
            self.copied[k].synchronize()  # that buffer's previous copy is done
        # torch's copy runs on the intra-op thread pool (C3: 0.7 GB per epoch)
        self.host[k][:n].copy_(torch.from_numpy(perm_host))
        self.perm[:n].copy_(self.host[k][:n], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.copied[k] = ev
        self.cursor.zero_()
        n_full = n // self.bs
        if n_full and self.capture and self.graph is None:
            s = torch.cuda.Stream(device=self.perm.device)
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            # capture_begin/end directly: the torch.cuda.graph context manager
            # runs gc.collect() + empty_cache() first (~100 ms per capture)
            with torch.cuda.stream(s):
                g.capture_begin()
                self._enqueue(self.bs, True)
                g.capture_end()
            torch.cuda.current_stream().wait_stream(s)
            self.graph = g
        for _ in range(n_full):
            if self.capture:
                self.graph.replay()
            else:
                self._enqueue(self.bs, True)
        if n - n_full * self.bs:
            self._enqueue(n - n_full * self.bs, False)
        # the prologue overwrites counts; leave them zero for the
        # accumulate-style step (_Step.run) as nif_adam_dev does
        self.step.fam.counts.zero_()
        self.step.fam.dirty = True


def train_batch(model: NifModel, which: str, obj, coord, label) -> float:
    """nif.py:682-749 _train_batch with host arrays; returns the batch mean
    loss (sum of squared errors / rows)."""
    torch = _torch()
    dev = model.device
    obj = np.asarray(obj, np.int64)
    n = len(obj)
    if n == 0:
        raise ValueError("empty batch")
    for o in np.unique(obj):
        model._check_object(int(o))
    width = 4 if which == "outer" else 5
    t_obj = torch.from_numpy(obj).to(dev)
    t_coord = torch.from_numpy(np.ascontiguousarray(np.asarray(coord, np.float64)[:, :width])).to(dev)
    lab = np.asarray(label, np.float32).reshape(n, -1)
    t_lab = torch.from_numpy(np.ascontiguousarray(lab)).to(dev)
    step = _Step(model, which)
    step.run(t_obj, t_coord, t_lab, None, n)
    return float(step.sq.item()) / (n * lab.shape[1])


_train_batch = train_batch


_FAMILY_GROUPS = {}  # (ranks, backend) -> {family: process group}
_GRAPH_CACHE_MAX_SAMPLES = 1 << 24  # train(): captured step graphs kept up to this family size


def train(model: NifModel, samples, epochs: Optional[int] = None, seed: Optional[int] = None,
          group=None, deterministic: bool = False, dp_mode: str = "parity") -> np.ndarray:
    """nif.py:752-795: shuffled mini-batch epochs over both families; loss
    curve (epochs, 3) = outer, inner, combined (NaN for an empty family).

    With torch.distributed initialised (or `group` given) every rank holds
    the same samples and draws the same global permutation; rank r takes
    rows r, r+W, ... of each global batch (per-object loss scale from the
    global batch counts) and the step exchanges one buffer [batch input
    gradients | MLP gradients] with a single all-reduce (_Sink), captured
    in the step's CUDA graph under NCCL. deterministic=True makes the
    gradients bit-reproducible run to run: grid cells summed in np.add.at's
    order after a sort, MLP gradients reduced over CTAs in order.

    dp_mode="parity" (default) keeps the reference's global batch sizes, so
    W ranks split each batch (the same schedule as one process);
    dp_mode="throughput" gives every rank a full reference
    batch -- the global batch is W times the configured size, W times fewer
    optimiser steps per epoch -- so an epoch's work per GPU shrinks W-fold."""
    torch = _torch()
    if isinstance(samples, dict):
        samples = SampleSet.from_host(samples, device=model.device)
    if samples.head != model.config.head:
        raise ValueError(f"sample head {samples.head!r} does not match the "
                         f"model head {model.config.head!r}")
    if samples.n_outer == 0 and samples.n_inner == 0:
        raise ValueError("no training samples")
    epochs = model.config.epochs if epochs is None else epochs
    seed = model.config.seed if seed is None else seed
    curve = np.zeros((epochs, 3))
    if epochs == 0:
        return curve
    from .parallel import world_rank
    world, rank = world_rank(group)
    import torch.distributed as dist
    epoch_ss = np.random.SeedSequence([seed, 0x7472]).spawn(epochs)
    if dp_mode not in ("parity", "throughput"):
        raise ValueError(f"unknown dp_mode {dp_mode!r}")
    scale = world if dp_mode == "throughput" else 1
    bo = model.config.outer.batch_size * scale
    bi = model.config.inner.batch_size * scale
    steps = {"outer": _Step(model, "outer"), "inner": _Step(model, "inner")}
    cache = model.__dict__.setdefault("_train_graphs", {})  # family -> (key, step, graph step)
    on_gpu = model.device.type == "cuda"
    # every full batch is a replay of one captured step: always on one GPU,
    # under NCCL with the all-reduce inside the graph; gloo runs eagerly
    capture = on_gpu and (world == 1 or (dist.get_backend(group) == "nccl"
                                         and os.environ.get("NIF_DP_GRAPH", "1") != "0"))
    use_sink = world > 1 or deterministic
    fam_groups = {}
    if world > 1:
        # one communicator per family: the two families' steps (and their
        # collectives) run on separate streams, concurrently; created once
        # per (ranks, backend) and reused by later train() calls
        ranks = list(range(world)) if group is None else dist.get_process_group_ranks(group)
        key = (tuple(ranks), dist.get_backend(group))
        if key not in _FAMILY_GROUPS:
            _FAMILY_GROUPS[key] = {which: dist.new_group(ranks, backend=key[1])
                                   for which in ("outer", "inner")}
        fam_groups = _FAMILY_GROUPS[key]
    gsteps = {}
    fams = ((0, bo, "outer", samples.outer_obj, samples.outer_coord, samples.outer_label),
            (1, bi, "inner", samples.inner_obj, samples.inner_coord, samples.inner_label))
    # per (epoch, family) squared-error sums, read back once at the end (the
    # graph path never synchronises inside the loop)
    sq = torch.zeros((epochs, 2), dtype=torch.float64, device=model.device)
    counts = np.zeros(2, np.int64)
    sizes = [int(f[3].shape[0]) for f in fams]

    def epoch_perms(e):
        # outer first, then inner, from the epoch's generator (nif.py:769-788)
        rng = np.random.default_rng(epoch_ss[e])
        return [rng.permutation(n) if n else None for n in sizes]

    # Later epochs' permutations are drawn on host threads while this epoch is
    # queued and replayed: each epoch has its own generator, so epochs are
    # independent, and numpy's shuffle releases the GIL. One 2.7M-sample
    # permutation takes ~47 ms on one core -- more than the GPU's epoch at
    # C2 -- so several epochs are drawn at once (at C3, 107M samples, one
    # epoch's permutations are 0.86 GB and take ~1.9 s on one core: up to
    # 4 GB, and a quarter of the free host memory, are kept in flight).
    from collections import deque
    from concurrent.futures import ThreadPoolExecutor
    per_epoch_bytes = 8 * max(1, sum(sizes))
    budget = 4e9
    try:
        import psutil
        budget = min(budget, 0.25 * psutil.virtual_memory().available)
    except Exception:  # noqa: BLE001 -- psutil is optional
        pass
    depth = max(1, min(4, epochs, (os.cpu_count() or 2) // 2, int(budget // per_epoch_bytes)))
    pool = ThreadPoolExecutor(max_workers=depth)
    ahead = deque(pool.submit(epoch_perms, k) for k in range(min(depth, epochs)))
    # The two families are independent optimisers (disjoint parameters,
    # counts and step counters), so each runs its own sequence of steps --
    # in the reference's order within the family -- on its own stream, and
    # the latency-bound steps of one overlap the other's.
    fam_streams = {}
    if on_gpu:
        cur = torch.cuda.current_stream(model.device)
        for which in ("outer", "inner"):
            fam_streams[which] = torch.cuda.Stream(device=model.device)
            fam_streams[which].wait_stream(cur)
    for e in range(epochs):
        perms = ahead.popleft().result()
        if e + depth < epochs:
            ahead.append(pool.submit(epoch_perms, e + depth))
        for fam, bs, which, obj, coord, label in fams:
            n = int(obj.shape[0])
            if n == 0:
                continue
            with torch.cuda.stream(fam_streams[which]):
                if which not in gsteps:
                    # a later train() call on the same samples and settings
                    # replays the graphs captured by the previous one (one
                    # entry per family is kept: buffers are sample-sized)
                    a = model.config.adam  # (baked into the captured Adam launch)
                    key = (bs, world, rank, bool(deterministic), capture,
                           id(fam_groups.get(which)), n, obj.data_ptr(), coord.data_ptr(),
                           label.data_ptr(), model.learning_rate, a.beta1, a.beta2, a.epsilon)
                    hit = cache.get(which)
                    if hit is not None and hit[0] == key:
                        steps[which], gsteps[which] = hit[1], hit[2]
                    else:
                        st = steps[which]
                        sink = None
                        if use_sink:
                            sink = _Sink(st, bs, world, rank, fam_groups.get(which), deterministic)
                            if world > 1:  # communicator set up outside any capture
                                dist.all_reduce(sink.comm, group=fam_groups[which])
                        gsteps[which] = _GraphStep(st, obj, coord, label, n, bs, sink, capture)
                        # small sample sets only: a cached entry keeps its
                        # sample-sized permutation buffers (8 B/sample on the
                        # device + 16 B pinned) alive with the model; for
                        # large sets the one-off capture is negligible anyway
                        if n <= _GRAPH_CACHE_MAX_SAMPLES:
                            cache[which] = (key, st, gsteps[which])
                        else:
                            cache.pop(which, None)
                st = steps[which]
                st.sq.zero_()
                gsteps[which].epoch(perms[fam])
                if world > 1:  # each rank summed the squared errors of its own rows
                    dist.all_reduce(st.sq, group=fam_groups[which])
                # the reference's per-batch loss is the mean over rows x outputs
                width = int(label.shape[1]) if label.dim() > 1 else 1
                sq[e, fam].copy_(st.sq[0] / width)
            counts[fam] = n
    for s_ in fam_streams.values():
        torch.cuda.current_stream(model.device).wait_stream(s_)
    pool.shutdown()
    sums_all = sq.cpu().numpy()
    for e in range(epochs):
        sums = sums_all[e]
        om = sums[0] / counts[0] if counts[0] else math.nan
        im = sums[1] / counts[1] if counts[1] else math.nan
        curve[e] = (om, im, sums.sum() / counts.sum())
    return curve


def train_online(model: NifModel, scene: Scene, spp: int, epochs_per_pass: int = 1,
                 camera=None, seed: Optional[int] = None, group=None,
                 deterministic: bool = False, dp_mode: str = "parity"):
    """Online schedule (north_star "online train step"): for
    each progressive sample index s, collect that pass's samples on the
    device (collect_samples(spp=1, sample_offset=s)) and train
    `epochs_per_pass` epochs on them before the next pass, so the model
    improves while the frame accumulates. The reference trains after
    collecting all passes (collect_samples + train, nif.py:569-795); this
    composes the same two steps per pass. The epochs of pass s draw their
    permutations from SeedSequence([seed, s]). Returns the per-pass loss
    curves (spp, epochs_per_pass, 3)."""
    seed = model.config.seed if seed is None else seed
    curves = []
    for s in range(spp):
        smp = collect_samples(scene, camera, spp=1, seed=scene.seed, group=group,
                              sample_offset=s)
        if smp.n_outer == 0 and smp.n_inner == 0:
            curves.append(np.full((epochs_per_pass, 3), math.nan))
            continue
        pass_seed = int(np.random.SeedSequence([seed, s]).generate_state(1)[0])
        curves.append(train(model, smp, epochs=epochs_per_pass, seed=pass_seed, group=group,
                            deterministic=deterministic, dp_mode=dp_mode))
    return np.stack(curves) if curves else np.zeros((0, epochs_per_pass, 3))
