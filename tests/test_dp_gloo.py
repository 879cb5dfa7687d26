"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 host logic:

* image-tile sharding covers every pixel exactly once and the per-rank
  RNG keys equal the single-process keys;
* the data-parallel gradient decomposition used by train.train -- rows of
  a global batch interleaved across ranks, per-object normalisation by the
  GLOBAL batch counts, one all-reduce(sum) -- reproduces the single-process
  gradient of the reference step (nif.py:682-749), computed here with the
  oracle's numpy restatement.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_07191_b200.parallel import band, rank_strips, tile_pixels


def test_band_partition_exact():
    for n in (0, 1, 7, 1080, 2161):
        for w in (1, 2, 3, 8):
            seen = []
            for r in range(w):
                a, b = band(n, r, w)
                seen.extend(range(a, b))
            assert seen == list(range(n))
    total = sum(tile_pixels(1920, 1080, r, 8)[1] for r in range(8))
    assert total == 1920 * 1080


def test_rank_strips_partition_exact():
    for wd, ht in ((7, 5), (64, 33), (3840, 2160)):
        for w in (1, 2, 3, 8):
            for k in (1, 2, 8):
                seen = np.zeros(wd * ht, np.int32)
                for r in range(w):
                    strips = rank_strips(wd, ht, r, w, k)
                    if k == 1:
                        assert strips == [tile_pixels(wd, ht, r, w)] or strips == []
                    for (a, m), nxt in zip(strips, strips[1:] + [None]):
                        assert m > 0 and a % wd == 0 and m % wd == 0
                        if nxt is not None:
                            assert a + m < nxt[0]  # increasing, touching strips merged
                        seen[a:a + m] += 1
                assert (seen == 1).all(), (wd, ht, w, k)
    # every rank reaches into every part of the frame's height
    for r in range(8):
        ys = [a // 3840 for a, _ in rank_strips(3840, 2160, r, 8, 8)]
        assert min(ys) < 2160 // 8 and max(ys) >= 2160 * 7 // 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partitioned_grads(rank, world, obj, coord, label, om_factory, which):
    """Gradient of rows rank::world of the batch with global counts."""
    from oracle import oracle as O
    om = om_factory()
    mlp = om.outer if which == "outer" else om.inner
    n_obj = len(om.grids)
    counts = np.bincount(obj, minlength=n_obj)
    rows = np.arange(rank, len(obj), world)
    for o in np.unique(obj[rows]):
        sel = rows[obj[rows] == o]
        g = om.grids[o]
        uv_p, uv_d = coord[sel, 0:2], coord[sel, 2:4]
        if which == "outer":
            n_lat = g["outer_pos"].latents.shape[2]
            x = np.concatenate([O.lookup_2d(g["outer_pos"], uv_p),
                                O.lookup_2d(g["outer_dir"], uv_d)], axis=1)
        else:
            n_lat = g["inner_pos"].latents.shape[2]
            x = np.concatenate([O.lookup_2d(g["inner_pos"], uv_p),
                                O.lookup_2d(g["inner_dir"], uv_d),
                                O.lookup_1d(g["inner_dist"], coord[sel, 4])], axis=1)
        pred = mlp.forward(x.astype(np.float32))
        diff = pred - label[sel][:, None].astype(np.float32)
        gout = diff * np.float32(2.0 / counts[o])   # global group size
        gx = mlp.backward(gout)
        if which == "outer":
            O.grad_2d(g["outer_pos"], uv_p, gx[:, :n_lat])
            O.grad_2d(g["outer_dir"], uv_d, gx[:, n_lat:])
        else:
            O.grad_2d(g["inner_pos"], uv_p, gx[:, :n_lat])
            O.grad_2d(g["inner_dir"], uv_d, gx[:, n_lat:2 * n_lat])
            O.grad_1d(g["inner_dist"], coord[sel, 4], gx[:, 2 * n_lat:])
    flat = [l.gw.reshape(-1) for l in mlp.layers] + [l.gb for l in mlp.layers]
    for g in om.grids:
        for k in g:
            flat.append(g[k].grad.reshape(-1))
    return np.concatenate(flat).astype(np.float64)


def _worker(rank, world, port, payload, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    obj, coord, label, which, init = payload

    def factory():
        from oracle.oracle import OModel
        return OModel(*init)

    g = torch.from_numpy(_partitioned_grads(rank, world, obj, coord, label, factory, which))
    dist.all_reduce(g)
    if rank == 0:
        q.put(g.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("which", ["outer", "inner"])
def test_dp_gradient_allreduce_equals_full_batch(which, golden, scenes):
    from golden_cfg import small_config
    from oracle.oracle import OModel
    from paper_2306_07191_b200.nif import init_arrays
    g = golden("overlap")
    n = 256 if which == "outer" else 512
    obj = g[f"samples_{which}_obj"][:n]
    coord = g[f"samples_{which}_coord"][:n]
    label = g[f"samples_{which}_label"][:n]
    outer, inner, grids, _, _ = init_arrays(small_config(), scenes("overlap").n_objects)
    init = (outer[0], inner[0], grids)
    ref = _partitioned_grads(0, 1, obj, coord, label, lambda: OModel(*init), which)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, (obj, coord, label, which, init), q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    scale = np.abs(ref).max()
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-6 * scale)


def _gather_worker(rank, world, port, q):
    from paper_2306_07191_b200.parallel import allgather_ordered
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # segment s of rank r: (s, r, j) rows; rank 1 has an empty segment 1,
    # segment lengths differ per rank
    parts = []
    for s in range(3):
        n = 0 if (rank == 1 and s == 1) else 2 + s + 3 * rank
        parts.append(torch.tensor([[s, rank, j] for j in range(n)], dtype=torch.int64)
                     .reshape(n, 3))
    out = allgather_ordered(parts)
    q.put((rank, [o.numpy() for o in out]))
    dist.destroy_process_group()


def test_allgather_ordered_is_segment_major_rank_ordered():
    """parallel.allgather_ordered (the package's sample-merging collective):
    every rank receives segment-major, rank-ordered rows -- the reference's
    spp-major, band-ordered sample order (nif.py:606-647)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = []
    for s in range(3):
        rows = []
        for r in range(world):
            n = 0 if (r == 1 and s == 1) else 2 + s + 3 * r
            rows += [[s, r, j] for j in range(n)]
        expect.append(np.array(rows, np.int64).reshape(-1, 3))
    for _, out in got:
        assert len(out) == 3
        for a, b in zip(out, expect):
            np.testing.assert_array_equal(a, b)
