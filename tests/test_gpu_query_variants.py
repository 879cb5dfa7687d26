"""Every tensor-core query kernel agrees with the oracle (fp64 encode +
row-sequential forward, nif.py:286-359 restated) within the north-star
logit tolerance, and they agree with each other: the production fused
kernel with A in TMEM (in its CTA configurations), the runtime-shape
generic kernel and the split (standalone encoding + MLP)
path. Records cover full 128-row tiles, a partial last tile and tiny
batches; latents are U(-1, 1) with non-zero biases so logits are O(1)."""

import numpy as np
import pytest

from test_gpu_mlp import LOGIT_TOL_TC, _oracle_logits, _randomize, _records

pytestmark = pytest.mark.gpu

# nif_debug_set_query_variant: 0 production (TMEM A operand, CUDA-core head),
# 2 generic runtime-shape kernel, 11 TMEM A operand with one tile per CTA
# (6 per SM), 12 the round-1 inner configuration (2 CTAs x 3 warpgroups per SM)
VARIANTS = [0, 2, 11, 12]


@pytest.mark.parametrize("n", [1, 127, 128, 129, 3000, 40000])
def test_query_variants_agree(n, cuda):
    from paper_2306_07191_b200 import _lib
    from paper_2306_07191_b200.nif import NifConfig, NifModel, query_family
    m = NifModel(NifConfig(seed=11), 3)
    _randomize(m, 5)
    obj, coord = _records(n, 3, seed=n)
    L = _lib.lib()
    for fam, width in (("outer", 4), ("inner", 5)):
        ref = _oracle_logits(m, fam, obj, coord[:, :width])
        got = {}
        try:
            for v in VARIANTS:
                L.nif_debug_set_query_variant(v)
                got[v] = query_family(m, fam, obj, coord[:, :width], impl=2).astype(np.float64)
        finally:
            L.nif_debug_set_query_variant(0)
        got["split"] = query_family(m, fam, obj, coord[:, :width], split=True).astype(np.float64)
        for k, v in got.items():
            err = np.abs(v - ref).max()
            assert err <= LOGIT_TOL_TC, (fam, k, err)
            assert np.abs(v - got[2]).max() <= 5e-3, (fam, k)
        # same fp16 operands and fp32 head in both TMEM-operand paths
        np.testing.assert_allclose(got["split"], got[0], atol=1e-5)


def test_split_path_shapes(cuda):
    """The split path covers the C5 sweep widths / depths."""
    from paper_2306_07191_b200.nif import NifConfig, NifModel, query_family
    for width, layers in ((64, 3), (128, 2), (48, 4)):
        cfg = NifConfig(seed=2)
        cfg.outer.hidden_width = width
        cfg.inner.hidden_width = width
        cfg.outer.hidden_layers = layers
        cfg.inner.hidden_layers = layers
        cfg.outer.grid_resolution = 64
        cfg.inner.grid_resolution = 64
        m = NifModel(cfg, 2)
        _randomize(m, 3)
        obj, coord = _records(5000, 2, seed=width)
        for fam, w in (("outer", 4), ("inner", 5)):
            ref = _oracle_logits(m, fam, obj, coord[:, :w])
            got = query_family(m, fam, obj, coord[:, :w], split=True).astype(np.float64)
            assert np.abs(got - ref).max() <= LOGIT_TOL_TC, (width, layers, fam)
