"""Multi-GPU layout: one process per GPU (torchrun), NCCL over NVLink.

Inference shards by image tile with no data-path collective: rank r owns
a contiguous band of pixel rows, generates its own primary/shadow rays
(the sample pass takes a pixel offset, the RNG is keyed by the global
pixel index, so the union of the bands is exactly the single-GPU frame)
and resolves their visibility on its own device (sample pass ->
visibility -> shading stay in HBM). The only exchange is the final gather
of the tile images to rank 0.

Training is data parallel (reference nif.py:606-647 and
752-795): each rank collects the samples of its own band, one ordered
all-gather rebuilds the reference's global sample order (spp-major, then
ray-major across the bands), every rank draws the same global permutation,
and each optimiser step exchanges one buffer [input gradients of the batch
rows | MLP gradients] with a single all-reduce (see train.py).
"""

from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np


def band(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, stop) share of n items for `rank` (sizes differ
    by at most one; lower ranks take the remainder)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    q, r = divmod(n, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


def tile_pixels(width: int, height: int, rank: int, world: int) -> Tuple[int, int]:
    """Pixel range (pix0, n_pix) of the row band owned by `rank`."""
    y0, y1 = band(height, rank, world)
    return y0 * width, (y1 - y0) * width


def rank_strips(width: int, height: int, rank: int, world: int,
                strips_per_rank: int = 1) -> List[Tuple[int, int]]:
    """Pixel ranges [(pix0, n_pix), ...] owned by `rank` when the frame is
    cut into world * strips_per_rank row strips dealt round-robin (strip s
    to rank s mod world). strips_per_rank=1 is `tile_pixels`' contiguous
    band; more strips spread every rank over the whole image height, so
    the ranks' shares of costly regions (and of ray-less sky) even out.
    Ranges are in increasing pixel order; touching strips are merged."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if strips_per_rank < 1:
        raise ValueError("strips_per_rank must be >= 1")
    ns = world * strips_per_rank
    out: List[Tuple[int, int]] = []
    for s in range(rank, ns, world):
        y0, y1 = band(height, s, ns)
        if y1 == y0:
            continue
        if out and out[-1][0] + out[-1][1] == y0 * width:
            out[-1] = (out[-1][0], out[-1][1] + (y1 - y0) * width)
        else:
            out.append((y0 * width, (y1 - y0) * width))
    return out


def world_rank(group=None) -> Tuple[int, int]:
    """(world, rank) of `group` (1, 0 without torch.distributed)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def allgather_ordered(parts: Sequence, group=None) -> List:
    """Ordered concatenation across ranks of per-segment local tensors.

    ``parts[s]`` is this rank's tensor for segment s (all ranks pass the same
    number of segments and the same trailing shape / dtype). Returns, on every
    rank, ``[cat over ranks r of parts_r[s] for s]`` -- segment-major, rank
    order inside a segment: the reference's spp-major, band-ordered sample
    order when the segments are sample indices and the ranks own pixel bands
    in order. Two collectives: the per-segment row counts, then the rows
    (padded to the largest rank). Device-agnostic (NCCL or gloo).
    """
    import torch
    import torch.distributed as dist
    world, rank = world_rank(group)
    if world == 1:
        return list(parts)
    ref = parts[0]
    dev = ref.device
    if dist.get_backend(group) == "gloo" and dev.type != "cpu":
        # gloo gathers host tensors: stage through the host and come back
        return [t.to(dev) for t in allgather_ordered([p.cpu() for p in parts], group)]
    n_seg = len(parts)
    counts = torch.tensor([int(p.shape[0]) for p in parts], dtype=torch.int64, device=dev)
    all_counts = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts, group=group)
    cnt = torch.stack(all_counts).cpu().numpy()  # [world, n_seg]
    tail = tuple(ref.shape[1:])
    local = torch.cat(list(parts)) if n_seg else ref.new_zeros((0,) + tail)
    mx = int(cnt.sum(axis=1).max())
    pad = local.new_zeros((mx,) + tail)
    pad[:local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    offs = np.concatenate([np.zeros((world, 1), np.int64), np.cumsum(cnt, axis=1)], axis=1)
    out = []
    for s in range(n_seg):
        out.append(torch.cat([bufs[r][offs[r, s]:offs[r, s + 1]] for r in range(world)]))
    return out


def render_band(scene, backend, spp: int, pix0: int, n_pix: int, seed=None, camera=None,
                sample_offset: int = 0):
    """renderer.py:808-861 for pixels [pix0, pix0 + n_pix): the fp64 HDR sum
    of `spp` progressive samples as a device tensor (n_pix, 3). Sample pass,
    cast filter, visibility (``backend.occluded_dev`` when the backend has
    it) and shading all stay on the device."""
    import torch

    from . import _lib
    from .pipeline import ShadowRays, sample_pass_dev, shadow_rays_dev
    camera = camera or scene.camera
    seed = scene.seed if seed is None else seed
    ds = scene.device()
    dev = ds.device
    buf = torch.zeros((n_pix, 3), dtype=torch.float64, device=dev)
    L = _lib.lib()
    on_device = hasattr(backend, "occluded_dev")
    for s in range(sample_offset, sample_offset + spp):
        data = sample_pass_dev(scene, camera, s, seed, "importance", pix0, n_pix)
        cast, o, d, t = shadow_rays_dev(data)
        idx = cast.nonzero().squeeze(1)
        n_cast = int(idx.numel())
        if n_cast == 0:
            continue
        if on_device:
            occ = backend.occluded_dev(scene, o, d, t)
        else:
            rays = ShadowRays(o.cpu().numpy(), d.cpu().numpy(), t.cpu().numpy())
            occ = torch.from_numpy(backend.occluded(scene, rays, 1).astype(np.uint8)).to(dev)
        po = _lib.PassOut(**{k: _lib.ptr(v) for k, v in data.items()})
        L.nif_shade_accumulate_dev(po, _lib.ptr(ds.albedo), _lib.ptr(idx), _lib.ptr(occ),
                                   n_cast, _lib.ptr(buf), _lib.stream_ptr())
    return buf


def render_sharded(scene, backend, spp: int, seed=None, group=None, camera=None,
                   sample_offset: int = 0) -> Optional[np.ndarray]:
    """Progressive direct-lighting render, image split in row bands across
    ranks; returns the full linear image (mean of the samples) on rank 0
    and None elsewhere."""
    camera = camera or scene.camera
    world, rank = world_rank(group)
    pix0, n_pix = tile_pixels(camera.width, camera.height, rank, world)
    buf = render_band(scene, backend, spp, pix0, n_pix, seed, camera, sample_offset)
    if world == 1:
        return (buf / spp).view(camera.height, camera.width, 3).cpu().numpy()
    full = allgather_ordered([buf], group)[0]
    if rank != 0:
        return None
    return (full / spp).view(camera.height, camera.width, 3).cpu().numpy()


def split_rows(n_rows: int, rank: int, world: int) -> Tuple[int, int]:
    """(row0, row_step) of `rank` inside one global batch: interleaved rows
    r, r + W, r + 2W, ... (every rank gets a share of every object group)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return rank, world


def rows_of(n_rows: int, rank: int, world: int) -> np.ndarray:
    """Batch positions a rank processes (host-side mirror of split_rows)."""
    r0, st = split_rows(n_rows, rank, world)
    return np.arange(r0, n_rows, st, dtype=np.int64)

