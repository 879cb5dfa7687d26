"""Gather edge cases against the CPU oracle (which walks the reference's
top-level DFS literally): many objects (fused single-pass kernel up to 32
objects, two-pass kernel beyond), empty batches, rays missing everything,
overlapping boxes, hybrid routing."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _spheres_scene(n_obj, seed=0, route_every=0):
    from paper_2306_07191_b200 import meshgen
    from paper_2306_07191_b200.scene import (Camera, PointLight, Scene, SceneObject,
                                             build_bottom)
    rng = np.random.default_rng(seed)
    base = meshgen.mesh_arrays(*meshgen.icosphere(1, 1.0))
    objs = []
    for k in range(n_obj):
        c = rng.uniform(-2, 2, 3)
        c[2] = abs(c[2])
        r = rng.uniform(0.1, 0.5)
        arrays = meshgen.transformed(base, r, c)
        nif = not (route_every and k % route_every == 0)
        objs.append(SceneObject(f"s{k}", build_bottom(arrays), np.ones(3) * 0.5, nif))
    cam = Camera(np.array([0.0, -6.0, 3.0]), np.zeros(3), np.array([0.0, 0.0, 1.0]), 50.0,
                 64, 48)
    return Scene(objs, [PointLight(np.array([1.0, -1.0, 6.0]), np.ones(3) * 30)], cam, 7)


def _random_rays(scene, n, seed=1):
    from paper_2306_07191_b200 import ShadowRays
    rng = np.random.default_rng(seed)
    o = rng.uniform(-3, 3, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t = rng.uniform(0.5, 8.0, n)
    t[::7] = np.inf
    return ShadowRays(o, d, t)


def _check(scene, rays, route):
    from oracle import oracle
    from paper_2306_07191_b200 import gather_queries
    osc = oracle.OracleScene(scene.pack, scene.epsilon_t)
    kind, obj, ray, coord, bvh_occ, n_deg = oracle.gather(osc, rays.origins, rays.dirs,
                                                          rays.tmaxs, route)
    rec, occ = gather_queries(scene, rays, route)
    np.testing.assert_array_equal(rec.kind, kind)
    np.testing.assert_array_equal(rec.obj, obj)
    np.testing.assert_array_equal(rec.ray, ray)
    np.testing.assert_allclose(rec.coord, coord, rtol=0, atol=1e-14)
    np.testing.assert_array_equal(occ, bvh_occ)
    assert rec.degenerate_count == n_deg
    return len(rec)


@pytest.mark.parametrize("n_obj", [2, 31, 32, 33, 48])
def test_gather_many_objects(n_obj, cuda):
    s = _spheres_scene(n_obj, seed=n_obj, route_every=5)
    rays = _random_rays(s, 5000, seed=n_obj)
    m = _check(s, rays, s.nif_route_mask(None))
    assert m > 0


def test_gather_empty_and_miss_all(cuda):
    from paper_2306_07191_b200 import ShadowRays, gather_queries
    s = _spheres_scene(3)
    rec, occ = gather_queries(s, ShadowRays(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0)),
                              s.nif_route_mask(None))
    assert len(rec) == 0 and len(occ) == 0
    # rays far away pointing up: no box touched -> visible, no records
    o = np.tile([50.0, 50.0, 50.0], (100, 1))
    d = np.tile([0.0, 0.0, 1.0], (100, 1))
    rec, occ = gather_queries(s, ShadowRays(o, d, np.full(100, 10.0)), s.nif_route_mask(None))
    assert len(rec) == 0 and not occ.any()


def test_gather_hybrid_threshold_routes_everything_to_bvh(cuda):
    s = _spheres_scene(10, seed=3)
    rays = _random_rays(s, 3000, seed=4)
    route = s.nif_route_mask(10 ** 9)  # every object below the threshold
    assert route.sum() == 0
    assert _check(s, rays, route) == 0


def test_fast_queue_coords_close_to_exact(cuda):
    """Hot-path fp32 queue coordinates vs the exact fp64 records."""
    import torch
    from paper_2306_07191_b200 import gather_queries
    from paper_2306_07191_b200.pipeline import GatherBuffers, gather_dev, rays_to_device
    s = _spheres_scene(20, seed=9)
    rays = _random_rays(s, 4000, seed=9)
    route = s.nif_route_mask(None)
    rec, _ = gather_queries(s, rays, route)
    ds = s.device()
    o, d, t = rays_to_device(rays, ds.device)
    buf = GatherBuffers(len(rays), int(route.sum()), ds.device)
    gather_dev(ds, ds.route(route), o, d, t, len(rays), buf)
    c = buf.counts.cpu().numpy()
    no, ni = int(c[0]), int(c[1])
    oc = buf.outer_coord[:no * 4].view(no, 4).cpu().numpy()
    ic = buf.inner_coord[:ni * 4].view(ni, 4).cpu().numpy()
    ir = buf.inner_r[:ni].cpu().numpy()
    # the hot-path queues are unordered: bring both sides to (ray, object)
    # order first
    ko, ki = rec.kind == 0, rec.kind == 1
    qo = np.lexsort((rec.obj[ko], rec.ray[ko]))
    qi = np.lexsort((rec.obj[ki], rec.ray[ki]))
    ex_o, ex_i = rec.coord[ko][qo], rec.coord[ki][qi]
    oray, oobj = buf.outer_ray[:no].cpu().numpy(), buf.outer_obj[:no].cpu().numpy()
    iray, iobj = buf.inner_ray[:ni].cpu().numpy(), buf.inner_obj[:ni].cpu().numpy()
    po, pi = np.lexsort((oobj, oray)), np.lexsort((iobj, iray))
    oc, ic, ir = oc[po], ic[pi], ir[pi]
    np.testing.assert_array_equal(oray[po], rec.ray[ko][qo])
    np.testing.assert_array_equal(oobj[po], rec.obj[ko][qo])
    np.testing.assert_array_equal(iobj[pi], rec.obj[ki][qi])
    np.testing.assert_array_equal(iray[pi], rec.ray[ki][qi])
    # u wraps at 1 -> compare on the circle
    def cdist(a, b):
        dd = np.abs(a - b)
        return np.minimum(dd, 1 - dd)
    assert cdist(oc[:, 0], ex_o[:, 0]).max() < 2e-6
    assert np.abs(oc[:, 1:4] - ex_o[:, 1:4]).max() < 2e-6 or cdist(oc[:, 2], ex_o[:, 2]).max() < 2e-6
    assert np.abs(ic[:, 1] - ex_i[:, 1]).max() < 2e-6
    assert np.abs(ir - ex_i[:, 4]).max() < 1e-6
