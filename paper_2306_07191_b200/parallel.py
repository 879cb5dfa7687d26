"""Multi-GPU layout: one process per GPU (torchrun), NCCL over NVLink.

Inference shards by image tile with no data-path collective: rank r owns
a contiguous band of pixel rows, generates its own primary/shadow rays
(the sample pass takes a pixel offset, the RNG is keyed by the global
pixel index, so the union of the bands is exactly the single-GPU frame)
and resolves their visibility locally. The only exchange is the final
gather of the tile images to rank 0.

Training is data parallel: see train.train (global permutation, rows
interleaved across ranks, one all-reduce of the flat gradient buffer per
optimiser step, identical Adam on every replica).
"""

from __future__ import annotations

import math
from typing import Tuple

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


def render_sharded(scene, backend, spp: int, seed=None, group=None):
    """Progressive direct-lighting render, image split in row bands across
    ranks; returns the full linear image on rank 0 (None elsewhere)."""
    import torch
    import torch.distributed as dist

    from .pipeline import ShadowRays, sample_pass_dev, shadow_rays_dev

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    cam = scene.camera
    pix0, n_pix = tile_pixels(cam.width, cam.height, rank, world)
    seed = scene.seed if seed is None else seed
    ds = scene.device()
    dev = ds.device
    buf = torch.zeros((n_pix, 3), dtype=torch.float64, device=dev)
    inv_pi = 1.0 / math.pi
    for s in range(spp):
        data = sample_pass_dev(scene, cam, s, seed, "importance", pix0, n_pix)
        cos = (data["normal"] * data["ldir"]).sum(dim=1)
        cast, o, d, t = shadow_rays_dev(data)
        if int(cast.sum()) == 0:
            continue
        occ = backend.occluded(scene, ShadowRays(o.cpu().numpy(), d.cpu().numpy(),
                                                 t.cpu().numpy()))
        vis = torch.zeros(n_pix, dtype=torch.float64, device=dev)
        vis[cast] = torch.from_numpy(~occ).to(dev).double()
        obj = data["obj"].long().clamp(min=0)
        scale = torch.where(cast, vis * cos / torch.where(cast, data["pdf"], 1.0), 0.0)
        contrib = ds.albedo[obj] * inv_pi * data["emit"] * scale[:, None]
        buf += torch.where(cast[:, None], contrib, 0.0)
    if world == 1:
        return (buf / spp).view(cam.height, cam.width, 3).cpu().numpy()
    sizes = [tile_pixels(cam.width, cam.height, r, world)[1] for r in range(world)]
    mx = max(sizes)
    pad = torch.zeros((mx, 3), dtype=torch.float64, device=dev)
    pad[:n_pix] = buf
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    if rank != 0:
        return None
    full = torch.cat([p[:sz] for p, sz in zip(parts, sizes)])
    return (full / spp).view(cam.height, cam.width, 3).cpu().numpy()
