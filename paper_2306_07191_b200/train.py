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

Data parallel (torch.distributed over NCCL): every rank holds the same
sample set and the same global permutation; rank r processes rows
r, r+W, r+2W, ... of each global batch (per-object normalisation uses the
global batch counts), the flat fp32 gradient buffer of the family plus the
squared-error accumulator are summed with one all-reduce, and every rank
applies the identical Adam update, so replicas stay identical without a
broadcast.
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
                    threads: Optional[int] = None) -> SampleSet:
    """nif.py:569-674 on the device: per sample index, the primary pass,
    every hit pixel's shadow ray (no cosine filter), the gather in the
    reference's record order and per-object BVH labels (1 = visible).
    labeler="geometry" follows the primary rays instead (uniform sampler,
    camera origin, infinite t_max) and labels each record with the closest
    hit in its own object (unit normal, t / diagonal), keeping hit rows."""
    torch = _torch()
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
    n_pix = camera.width * camera.height
    acc = {k: [] for k in ("oo", "oc", "ol", "or_", "io", "ic", "il", "ir")}
    n_rays = shadow_rays = degenerate = 0
    L = _lib.lib()
    cam_pos = torch.from_numpy(np.ascontiguousarray(
        np.broadcast_to(np.asarray(camera.position, np.float64), (n_pix, 3)))).to(dev)
    inf_tmax = torch.full((n_pix,), math.inf, dtype=torch.float64, device=dev)
    for s in range(spp):
        data = sample_pass_dev(scene, camera, s, seed,
                               "uniform" if head == "geometry" else sampler)
        if head == "geometry":
            idx = torch.arange(n_pix, device=dev)
            n = n_pix
            o, d, t = cam_pos, data["pdir"].contiguous(), inf_tmax
        else:
            mask = data["hit"] != 0
            idx = mask.nonzero().squeeze(1)
            n = int(idx.numel())
            if n == 0:
                continue
            o = data["point"][idx].contiguous()
            d = data["ldir"][idx].contiguous()
            t = data["tmax"][idx].contiguous()
        buf, counts = gather_sized(ds, ds.route(route), o, d, t, n, int(route.sum()), dev)
        m = int(counts[2])
        shadow_rays += n
        degenerate += int(counts[3])
        if m == 0:
            continue
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
        ray_ids = s * n_pix + idx
        for k, (ko, kc, kl, kr), width in ((0, ("oo", "oc", "ol", "or_"), 4),
                                           (1, ("io", "ic", "il", "ir"), 5)):
            selm = kind == k
            if keep is not None:
                selm &= keep
            sel = selm.nonzero().squeeze(1)
            if sel.numel() == 0:
                continue
            acc[ko].append(rec_obj[sel].long())
            acc[kc].append(coord[sel, :width].contiguous())
            acc[kl].append(lab[sel])
            acc[kr].append(ray_ids[rec_ray[sel].long()])
        n_rays += n

    def cat(key, tail, dt):
        if acc[key]:
            return torch.cat(acc[key]).contiguous()
        return torch.zeros((0,) + tail, dtype=dt, device=dev)

    lt = () if head == "occlusion" else (4,)
    out = SampleSet(head, cat("oo", (), torch.int64), cat("oc", (4,), torch.float64),
                    cat("ol", lt, torch.float32), cat("or_", (), torch.int64),
                    cat("io", (), torch.int64), cat("ic", (5,), torch.float64),
                    cat("il", lt, torch.float32), cat("ir", (), torch.int64), n_rays=n_rays)
    out.stats = {"pixel_samples": spp * n_pix, "shadow_rays": shadow_rays,
                 "degenerate_queries": degenerate,
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

    def run(self, obj, coord, label, idx, n_rows, rank=0, world=1, group=None, stream=None,
            idx_ptr=None):
        """One optimiser step over rows idx[0:n_rows] (device tensors; or a raw
        device pointer idx_ptr into an int64 row list); leaves this batch's
        squared-error sum added into self.sq."""
        torch = _torch()
        L = _lib.lib()
        fam, model = self.fam, self.model
        sp = _lib.stream_ptr(stream)
        fv, tv = self.fv, self.tv
        p = _lib.ptr
        if idx_ptr is not None:
            idx = None
        ip = idx_ptr if idx_ptr is not None else p(idx)
        L.nif_batch_counts_dev(p(obj), ip, n_rows, fam.n_obj, p(fam.counts), sp)
        if world > 1:
            sq_local = torch.zeros(1, dtype=torch.float64, device=model.device)
            L.nif_train_fwdbwd_dev(fv, tv, p(obj), p(coord), p(label), ip, n_rows, rank,
                                   world, p(sq_local), sp)
            import torch.distributed as dist
            dist.all_reduce(fam.grad, group=group)
            dist.all_reduce(sq_local, group=group)
            self.sq += sq_local
        else:
            L.nif_train_fwdbwd_dev(fv, tv, p(obj), p(coord), p(label), ip, n_rows, 0, 1,
                                   p(self.sq), sp)
        a = model.config.adam
        L.nif_adam_dev(fv, tv, model.learning_rate, a.beta1, a.beta2, a.epsilon, sp)
        fam.dirty = True


class _GraphStep:
    """One family's optimiser step captured as a CUDA graph and replayed
    for every full batch of an epoch: the batch start lives on the device
    (a cursor into a persistent permutation buffer, advanced by the graph
    itself), so an epoch is one async H2D copy of the permutation (from a
    pinned staging buffer) plus one graph launch per batch -- no per-step
    host work and no host synchronisation: the host is free to draw the
    next permutation while the GPU replays this one."""

    def __init__(self, step: "_Step", obj, coord, label, n: int, bs: int):
        torch = _torch()
        self.step, self.bs = step, bs
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
        # three launches: counts + step counters, fused fwd/bwd, dense Adam
        # (which also moves the cursor on)
        L.nif_train_prologue_cur_dev(st.fv, st.tv, p(self.obj), p(self.perm), p(self.cursor),
                                     n_rows, sp)
        L.nif_train_fwdbwd_cur_dev(st.fv, st.tv, p(self.obj), p(self.coord), p(self.label),
                                   p(self.perm), p(self.cursor), n_rows, 0, 1, p(st.sq), sp)
        a = model.config.adam
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
        if n_full and self.graph is None:
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
            self.graph.replay()
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


def train(model: NifModel, samples, epochs: Optional[int] = None, seed: Optional[int] = None,
          group=None) -> np.ndarray:
    """nif.py:752-795: shuffled mini-batch epochs over both families; loss
    curve (epochs, 3) = outer, inner, combined (NaN for an empty family).
    With torch.distributed initialised (or `group` given) the batches are
    split across ranks and gradients all-reduced once per step."""
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
    world, rank = 1, 0
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    epoch_ss = np.random.SeedSequence([seed, 0x7472]).spawn(epochs)
    bo = model.config.outer.batch_size
    bi = model.config.inner.batch_size
    steps = {"outer": _Step(model, "outer"), "inner": _Step(model, "inner")}
    # single GPU: every full batch is a replay of one captured step
    use_graph = world == 1 and model.device.type == "cuda"
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
    # counts and step counters), so on one GPU each runs its own sequence of
    # steps -- in the reference's order within the family -- on its own
    # stream, and the latency-bound steps of one overlap the other's.
    import contextlib
    fam_streams = {}
    if use_graph:
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
            perm_np = perms[fam]
            st = steps[which]
            ctx = torch.cuda.stream(fam_streams[which]) if use_graph else contextlib.nullcontext()
            with ctx:
                st.sq.zero_()
                if use_graph:
                    if which not in gsteps:
                        gsteps[which] = _GraphStep(st, obj, coord, label, n, bs)
                    gsteps[which].epoch(perm_np)
                else:
                    perm = torch.from_numpy(perm_np).to(model.device)
                    base = perm.data_ptr()
                    for k in range(0, n, bs):
                        m = min(bs, n - k)
                        st.run(obj, coord, label, None, m, rank, world, group,
                               idx_ptr=base + 8 * k)
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
