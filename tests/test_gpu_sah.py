"""The GPU SAH builder (nif_build_sah_dev) reproduces the host build --
itself node-for-node the reference's _build_sah (bvh.py:34-303), pinned by
the golden scene hashes -- byte for byte: node bounds (incl. the sign of
zero bounds), child ids in the reference's depth-first numbering, leaf
ranges and the primitive order. Cases cover meshes, uniform random
triangles, both leaf sizes (4 bottom, 1 top), collapsed centroids (the
halving path), single / two primitives and signed-zero ties."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mesh_bounds(sub):
    from paper_2306_07191_b200.meshgen import icosphere
    v, f, _ = icosphere(sub)
    t = v[f]
    return _bounds(t[:, 0], t[:, 1], t[:, 2])


def _bounds(v0, v1, v2):
    lo = np.minimum(np.minimum(v0, v1), v2)
    hi = np.maximum(np.maximum(v0, v1), v2)
    return lo, hi, (lo + hi) * 0.5


def _random(n, seed, scale=1.0):
    g = np.random.default_rng(seed)
    base = g.uniform(-10, 10, (n, 3))
    return _bounds(base, base + g.normal(0, scale, (n, 3)), base + g.normal(0, scale, (n, 3)))


def _compare(lo, hi, ce, max_leaf, dev):
    import torch
    from paper_2306_07191_b200.scene import _build_sah, build_sah_dev
    want = _build_sah(lo, hi, ce, max_leaf)
    t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (lo, hi, ce)]
    got = [x.cpu().numpy() for x in build_sah_dev(*t, max_leaf=max_leaf)]
    names = ("node_lo", "node_hi", "node_a", "node_b", "node_leaf", "order")
    for nm, w, g in zip(names, want, got):
        assert w.shape == g.shape, (nm, w.shape, g.shape)
        assert w.tobytes() == g.tobytes(), nm


@pytest.mark.parametrize("sub", [0, 2, 4, 6])
@pytest.mark.parametrize("max_leaf", [4, 1])
def test_sah_dev_icosphere(sub, max_leaf, cuda):
    _compare(*_mesh_bounds(sub), max_leaf, cuda)


@pytest.mark.parametrize("n,seed", [(3, 1), (37, 2), (1000, 3), (65537, 4), (300000, 5)])
def test_sah_dev_random(n, seed, cuda):
    _compare(*_random(n, seed), 4, cuda)


def test_sah_dev_top_level_boxes(cuda):
    # build_top's case: object boxes, one per leaf
    lo, hi, ce = _random(5000, 9, scale=0.3)
    _compare(lo, hi, ce, 1, cuda)


def test_sah_dev_degenerate(cuda):
    one = np.zeros((1, 3)), np.ones((1, 3)), np.full((1, 3), 0.5)
    _compare(*one, 4, cuda)
    _compare(*one, 1, cuda)
    two = _random(2, 3)
    _compare(*two, 1, cuda)
    # all centroids identical: no axis has extent -> halving by order
    lo = np.zeros((1000, 3))
    hi = np.ones((1000, 3))
    _compare(lo, hi, (lo + hi) * 0.5, 4, cuda)
    # centroids collapsed on two axes, boxes tied
    g = np.random.default_rng(7)
    lo = np.zeros((4096, 3))
    lo[:, 0] = g.integers(0, 8, 4096)
    hi = lo + 1.0
    _compare(lo, hi, (lo + hi) * 0.5, 4, cuda)


def test_sah_dev_signed_zero_ties(cuda):
    # -0.0 / +0.0 bounds compare equal; the first occurrence in segment order
    # sets the node's stored bound, as in the reference's sequential scan
    g = np.random.default_rng(11)
    n = 20000
    lo = g.integers(-2, 3, (n, 3)).astype(np.float64)
    lo[g.random((n, 3)) < 0.3] = -0.0
    hi = lo + g.integers(0, 3, (n, 3))
    hi[(hi == 0) & (g.random((n, 3)) < 0.5)] = -0.0
    _compare(lo, hi, (lo + hi) * 0.5, 4, cuda)


def test_build_bottoms_on_device(cuda):
    """Scene-level use: per-object trees built on the GPU equal host builds."""
    from paper_2306_07191_b200 import meshgen
    from paper_2306_07191_b200.scene import build_bottoms
    base = meshgen.mesh_arrays(*meshgen.icosphere(5, 0.35))
    arrays = [meshgen.transformed(base, 1.0, (0.3 * k, -0.2 * k, 0.35)) for k in range(3)]
    arrays.append(meshgen.mesh_arrays(*meshgen.torus()))
    host = build_bottoms(arrays, workers=1)
    dev = build_bottoms(arrays, device=cuda)
    for h, d in zip(host, dev):
        for nm in ("node_lo", "node_hi", "node_a", "node_b", "node_leaf", "order", "v0", "n2"):
            assert getattr(h, nm).tobytes() == getattr(d, nm).tobytes(), nm


@pytest.mark.parametrize("seed", [21, 22, 23])
def test_sah_dev_clustered_and_skewed(seed, cuda):
    """Quantised coordinates (many equal centroids, bin-boundary ties) and
    heavy-tailed sizes, so segments cross the warp / CTA / chunked classes
    at many depths."""
    g = np.random.default_rng(seed)
    n = int(g.integers(9000, 60000))
    base = np.round(g.exponential(2.0, (n, 3)) * 4) / 4 * g.choice([-1, 1], (n, 3))
    ext = g.exponential(0.05, (n, 3)) * (g.random((n, 1)) < 0.9)
    lo, hi = base, base + ext
    _compare(lo, hi, (lo + hi) * 0.5, 4 if seed != 23 else 1, cuda)
