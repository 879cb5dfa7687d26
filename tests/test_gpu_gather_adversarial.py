"""Gather parity on adversarial rays, for the exact API gather (bit-exact
records vs the CPU oracle, which walks the reference's top-level DFS
literally) and the hot-path unordered gather (same record multiset, same
bvh_occ, same degenerate count): axis-aligned directions with exact and
signed zeros, origins exactly on box faces / edges / corners, origins at
box centres (the degenerate inner record), t_max of 0, tiny and inf, and
direction components below the fp32 prefilter's 1e-20 cut-off."""

import numpy as np
import pytest

from test_gpu_gather import _check, _spheres_scene

pytestmark = pytest.mark.gpu


def _adversarial_rays(scene, seed=0):
    from paper_2306_07191_b200 import ShadowRays
    rng = np.random.default_rng(seed)
    pk = scene.pack
    lo, hi = pk.obox_lo, pk.obox_hi
    ctr = 0.5 * (lo + hi)
    o, d, t = [], [], []
    axes = [np.array(v, float) for v in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0),
                                         (0, 0, 1), (0, 0, -1))]
    for k in range(len(lo)):
        # face / edge / corner origins and the centre
        pts = [lo[k], hi[k], ctr[k],
               np.array([lo[k][0], ctr[k][1], ctr[k][2]]),
               np.array([hi[k][0], hi[k][1], ctr[k][2]]),
               np.array([ctr[k][0], lo[k][1], hi[k][2]])]
        for p in pts:
            for a in axes:
                o.append(p)
                d.append(a)
                t.append(rng.choice([0.0, 1e-12, 0.3, 5.0, np.inf]))
            # signed zeros in the direction
            o.append(p)
            d.append(np.array([-0.0, 0.6, -0.8]))
            t.append(np.inf)
            o.append(p)
            d.append(np.array([0.0, -0.0, 1.0]))
            t.append(2.0)
        # from outside straight through the centre, and grazing a face
        for a in axes:
            o.append(ctr[k] - 3.0 * a)
            d.append(a)
            t.append(np.inf)
            off = np.where(a != 0, 0.0, hi[k] - ctr[k])
            o.append(ctr[k] - 3.0 * a + off)
            d.append(a)
            t.append(6.0)
    # tiny components: below the fp32 prefilter cut-off (exact path only)
    for s_ in (1e-25, 1e-300, 5e-324):
        v = np.array([s_, 0.7, -0.7])
        o.append(ctr[0] - 2.0 * v)
        d.append(v / np.linalg.norm(v))
        t.append(np.inf)
    o, d, t = np.array(o), np.array(d), np.array(t)
    return ShadowRays(o, d, t)


def _fast_check(scene, rays, route):
    """Hot-path unordered gather vs the oracle: same (kind, ray, obj)
    multiset, same per-ray hybrid answer, same degenerate count."""
    from oracle import oracle
    from paper_2306_07191_b200.pipeline import GatherBuffers, gather_dev, rays_to_device
    osc = oracle.OracleScene(scene.pack, scene.epsilon_t)
    kind, obj, ray, _, bvh_occ, n_deg = oracle.gather(osc, rays.origins, rays.dirs, rays.tmaxs,
                                                      route)
    ds = scene.device()
    o, d, t = rays_to_device(rays, ds.device)
    buf = GatherBuffers(len(rays), int(route.sum()), ds.device)
    gather_dev(ds, ds.route(route), o, d, t, len(rays), buf)
    c = buf.counts.cpu().numpy()
    no, ni = int(c[0]), int(c[1])
    got = sorted(zip([0] * no, buf.outer_ray[:no].cpu().tolist(), buf.outer_obj[:no].cpu().tolist()))
    got += sorted(zip([1] * ni, buf.inner_ray[:ni].cpu().tolist(), buf.inner_obj[:ni].cpu().tolist()))
    want = sorted(zip((kind == 1).astype(int).tolist(), ray.tolist(), obj.tolist()))
    assert sorted(got) == want
    np.testing.assert_array_equal(buf.bvh_occ[:len(rays)].cpu().numpy().astype(bool), bvh_occ)
    assert int(c[3]) == n_deg


@pytest.mark.parametrize("n_obj,route_every", [(1, 0), (3, 0), (7, 3), (40, 4)])
def test_gather_adversarial_exact(n_obj, route_every, cuda):
    s = _spheres_scene(n_obj, seed=17 + n_obj, route_every=route_every)
    rays = _adversarial_rays(s, seed=n_obj)
    _check(s, rays, s.nif_route_mask(None))


@pytest.mark.parametrize("n_obj,route_every", [(1, 0), (3, 0), (7, 3), (20, 4)])
def test_gather_adversarial_hot_path(n_obj, route_every, cuda):
    s = _spheres_scene(n_obj, seed=17 + n_obj, route_every=route_every)
    rays = _adversarial_rays(s, seed=n_obj)
    _fast_check(s, rays, s.nif_route_mask(None))
