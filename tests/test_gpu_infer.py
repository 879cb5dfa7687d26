"""Query-object API against the reference (golden tests/golden/infer.npz,
made by tests/golden/make_infer.py from the reference itself):
infer_occlusion (nif.py:428-442) and infer_geometry (nif.py:445-464) at the
default resolutions (R 256/128) with O(1) latents and biases, plus the
SPEC.md:412-426 known answers -- zero MLP gives p = 0.5 -> visible, empty
batch -> empty output, batch / permutation invariance, unit normals."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_OBJ = 3
DIAGONAL = 7.25


@pytest.fixture(scope="module")
def gold(golden):
    return golden("infer")


def _model(head, sharing, seed, pseed):
    from golden_cfg import perturb_arrays
    from paper_2306_07191_b200.nif import NifConfig, NifModel, init_arrays
    cfg = NifConfig(seed=seed, head=head, sharing=sharing)
    m = NifModel(cfg, N_OBJ, DIAGONAL)
    outer, inner, grids, _, _ = init_arrays(cfg, N_OBJ)
    perturb_arrays(outer, inner, grids, seed=pseed)
    m.load_arrays(outer, inner, grids)
    return m


def _queries(g):
    from paper_2306_07191_b200.scene import InnerQuery, OuterQuery, SphericalCoord
    out = []
    for k, o, c in zip(g["kind"], g["obj"], g["coord"]):
        p, d = SphericalCoord(c[0], c[1]), SphericalCoord(c[2], c[3])
        out.append(OuterQuery(int(o), p, d) if k == 0 else InnerQuery(int(o), p, d, float(c[4])))
    return out


@pytest.mark.parametrize("sharing", ["shared", "per_object"])
def test_infer_occlusion_matches_reference(sharing, gold, cuda):
    from paper_2306_07191_b200.nif import (encode_inner_arrays, encode_outer_arrays,
                                           forward_inner_arrays, forward_outer_arrays,
                                           infer_occlusion)
    m = _model("occlusion", sharing, 0, int(gold[f"pseed_{sharing}"]))
    qs = _queries(gold)
    ref = gold[f"occ_{sharing}"]
    assert 0.2 < ref.mean() < 0.8
    # exact path: bit-identical bits and probabilities
    got = infer_occlusion(m, qs)
    assert np.array_equal(got, ref)
    kind, obj, coord = gold["kind"], gold["obj"], gold["coord"]
    prob = np.zeros(len(kind))
    for k, enc, fwd, w in ((0, encode_outer_arrays, forward_outer_arrays, 4),
                           (1, encode_inner_arrays, forward_inner_arrays, 5)):
        sel = kind == k
        prob[sel] = fwd(m, obj[sel], enc(m, obj[sel], coord[sel, :w]))[:, 0]
    # logits are bit-exact (test_gpu_parity); the sigmoid's exp is CUDA's
    # (<= 1 ulp from numba's libm), so probabilities agree to a few ulps
    np.testing.assert_allclose(prob, gold[f"prob_{sharing}"], rtol=4e-16, atol=0)
    # tensor-core path: identical wherever the reference's probability is
    # decided beyond the logit tolerance (|logit| > 2e-2)
    fast = infer_occlusion(m, qs, exact=False)
    p = gold[f"prob_{sharing}"]
    logit = np.log(p) - np.log1p(-p)
    decided = np.abs(logit) > 2e-2
    assert np.array_equal(fast[decided], ref[decided])
    assert np.mean(fast == ref) >= 0.999


def test_infer_occlusion_known_answers(gold, cuda):
    """zero MLP -> p = 0.5 -> visible; empty batch ->
    empty; batching / permutation equivalence bit for bit."""
    from paper_2306_07191_b200.nif import NifConfig, NifModel, infer_occlusion
    qs = _queries(gold)
    z = NifModel(NifConfig(seed=0), N_OBJ, DIAGONAL)
    for fam in (z.outer, z.inner):
        fam.part("w").zero_()
        fam.part("b").zero_()
        fam.dirty = True
    assert np.array_equal(infer_occlusion(z, qs), gold["occ_zero"])
    assert not infer_occlusion(z, qs).any()
    assert not infer_occlusion(z, qs, exact=False).any()  # logit exactly 0 -> visible
    assert infer_occlusion(z, []).shape == (0,)
    m = _model("occlusion", "shared", 0, int(gold["pseed_shared"]))
    full = infer_occlusion(m, qs)
    perm = np.random.default_rng(0).permutation(len(qs))
    assert np.array_equal(infer_occlusion(m, [qs[i] for i in perm]), full[perm])
    one = np.array([infer_occlusion(m, [qs[i]])[0] for i in range(0, len(qs), 97)])
    assert np.array_equal(one, full[::97])
    with pytest.raises(TypeError, match="not a ray query"):
        infer_occlusion(m, [object()])


def test_infer_geometry_matches_reference(gold, cuda):
    """4-wide identity head: exact path equals the reference; the fused
    tensor-core path (fp16 operands, 4-wide CUDA-core head from the fp32
    accumulator) is within the logit tolerance on the raw outputs."""
    from paper_2306_07191_b200.nif import infer_geometry, infer_occlusion, query_family
    m = _model("geometry", "shared", 1, 101)
    qs = _queries(gold)
    n_ref, d_ref = gold["geo_normal"], gold["geo_depth"]
    n_ex, d_ex = infer_geometry(m, qs, exact=True)
    assert np.array_equal(n_ex, n_ref) and np.array_equal(d_ex, d_ref)
    n_tc, d_tc = infer_geometry(m, qs)
    assert np.allclose(np.linalg.norm(n_tc, axis=1), 1.0, atol=1e-12)
    assert np.abs(d_tc - d_ref).max() <= 2e-2 * DIAGONAL
    # raw head outputs of the tensor-core kernel vs the exact ones
    kind, obj, coord = gold["kind"], gold["obj"], gold["coord"]
    from paper_2306_07191_b200.nif import _encode, _forward
    for k, fam, w in ((0, "outer", 4), (1, "inner", 5)):
        sel = kind == k
        raw_tc = query_family(m, fam, obj[sel], coord[sel, :w]).reshape(-1, 4)
        raw_ex = _forward(m, fam, obj[sel], _encode(m, fam, obj[sel], coord[sel, :w]))
        assert np.abs(raw_tc - raw_ex).max() <= 2e-2, fam
        assert np.abs(raw_ex).mean() > 0.05
    # angular error of the renormalised normals where the raw normal is not tiny
    raw_norm = np.linalg.norm(np.concatenate([
        _forward(m, "outer", obj[kind == 0], _encode(m, "outer", obj[kind == 0],
                                                     coord[kind == 0, :4]))[:, :3],
        _forward(m, "inner", obj[kind == 1], _encode(m, "inner", obj[kind == 1],
                                                     coord[kind == 1, :5]))[:, :3]]), axis=1)
    assert raw_norm.min() > 0.1
    cosang = np.clip(np.sum(n_tc * n_ref, axis=1), -1, 1)
    assert np.degrees(np.arccos(cosang)).max() < 5.0
    assert infer_geometry(m, [])[0].shape == (0, 3)
    with pytest.raises(ValueError, match="occlusion head"):
        infer_geometry(_model("occlusion", "shared", 0, 100), qs[:3])
    with pytest.raises(ValueError, match="geometry head"):
        infer_occlusion(m, qs[:3])


def test_backends_reject_geometry_head(cuda):
    """a geometry-head model behind the visibility backends
    raises the reference's ValueError instead of answering from the hybrid
    bits alone."""
    from paper_2306_07191_b200 import NativeEngine, NifBackend, build_model, synthetic
    from paper_2306_07191_b200.nif import NifConfig
    from paper_2306_07191_b200.pipeline import ShadowRays, VisibilityEngine
    scene = synthetic.c1(32, 32, subdiv=2)
    m = build_model(NifConfig(seed=0, head="geometry"), scene)
    rays = ShadowRays(np.zeros((4, 3)), np.tile([0.0, 0.0, 1.0], (4, 1)), np.ones(4))
    with pytest.raises(ValueError, match="geometry head"):
        NifBackend(m).occluded(scene, rays)
    with pytest.raises(ValueError, match="geometry head"):
        VisibilityEngine(scene, m, 16)
    with pytest.raises(ValueError, match="geometry head"):
        NativeEngine(scene, m, 16)
