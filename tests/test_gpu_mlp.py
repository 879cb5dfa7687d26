"""Numerics of the fused query kernels on models whose logits are O(1):
latents drawn U(-1, 1) (the C5 microbench distribution) and non-zero
biases, so both the encode and every layer (bias folding included) are
exercised. Reference: the oracle's fp64 encode + row-sequential forward
(nif.py:286-359 restated)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LOGIT_TOL_TC = 2e-2
LOGIT_TOL_SIMT = 1e-4


def _randomize(model, seed=1):
    import torch
    g = torch.Generator(device=model.device)
    g.manual_seed(seed)
    for fam in (model.outer, model.inner):
        for key in ("pos", "dir", "dist"):
            if key == "dist" and fam.family == 0:
                continue
            p = fam.part(key)
            p.copy_(torch.rand(p.shape, generator=g, device=model.device) * 2 - 1)
        b = fam.part("b")
        b.copy_((torch.rand(b.shape, generator=g, device=model.device) * 2 - 1) * 0.5)
        fam.dirty = True


def _oracle_logits(model, fam, obj, coord):
    from oracle import oracle
    hl = model.host_layers(fam)[0]
    w = np.concatenate([a.reshape(-1) for a, _ in hl])
    b = np.concatenate([bb for _, bb in hl])
    dims = [hl[0][0].shape[1]] + [a.shape[0] for a, _ in hl]
    grids = model.host_grids()
    pos = np.stack([gg[f"{fam}_pos"] for gg in grids])
    dr = np.stack([gg[f"{fam}_dir"] for gg in grids])
    dist = np.stack([gg["inner_dist"] for gg in grids]) if fam == "inner" else None
    x = oracle.encode(pos, dr, dist, obj, coord)
    return oracle.dense_forward(w, b, dims, x, sigmoid_head=0)[:, 0]


def _records(n, n_obj, seed=0):
    rng = np.random.default_rng(seed)
    obj = rng.integers(0, n_obj, n)
    coord = rng.random((n, 5))
    return obj, coord


@pytest.mark.parametrize("cfgname", ["default", "wide", "deep"])
def test_tc_logits_random_latents(cfgname, cuda):
    from paper_2306_07191_b200.nif import NifConfig, NifModel, query_family
    cfg = NifConfig(seed=3)
    if cfgname == "wide":
        cfg.outer.hidden_width = 128
        cfg.inner.hidden_width = 128
    elif cfgname == "deep":
        cfg.outer.hidden_layers = 4
        cfg.inner.hidden_layers = 4
    cfg.outer.grid_resolution = 64
    cfg.inner.grid_resolution = 64
    m = NifModel(cfg, 3)
    _randomize(m)
    obj, coord = _records(20000, 3)
    for fam, width in (("outer", 4), ("inner", 5)):
        ref = _oracle_logits(m, fam, obj, coord[:, :width])
        assert np.abs(ref).mean() > 0.05, "logits too small to test anything"
        simt = query_family(m, fam, obj, coord[:, :width], impl=1).astype(np.float64)
        tc = query_family(m, fam, obj, coord[:, :width], impl=2).astype(np.float64)
        e_simt = np.abs(simt - ref).max()
        e_tc = np.abs(tc - ref).max()
        assert e_simt <= LOGIT_TOL_SIMT, (fam, e_simt)
        assert e_tc <= LOGIT_TOL_TC, (fam, e_tc, np.abs(tc - ref).mean())
        decided = np.abs(ref) > LOGIT_TOL_TC
        agree = np.mean((tc[decided] < 0) == (ref[decided] < 0))
        assert agree == 1.0


def test_tc_partial_tiles_and_empty(cuda):
    """Record counts that are not multiples of the 128-row tile, and zero."""
    from paper_2306_07191_b200.nif import NifConfig, NifModel, query_family
    m = NifModel(NifConfig(seed=5), 2)
    _randomize(m, 7)
    for n in (1, 127, 129, 1000):
        obj, coord = _records(n, 2, seed=n)
        ref = _oracle_logits(m, "inner", obj, coord)
        tc = query_family(m, "inner", obj, coord, impl=2)
        assert np.abs(tc - ref).max() <= LOGIT_TOL_TC
    assert query_family(m, "outer", np.zeros(0, np.int64), np.zeros((0, 4)), impl=2).size == 0


def test_unknown_object_raises(cuda):
    from paper_2306_07191_b200.nif import NifConfig, NifModel, encode_outer_arrays
    m = NifModel(NifConfig(seed=0), 2)
    with pytest.raises(ValueError, match="has no grids"):
        encode_outer_arrays(m, np.array([5]), np.zeros((1, 4)))
