"""sharing="per_object" (one MLP per object; nif.py:91-92, 230-234,
380-397, 731-749) against the reference (tests/golden/make_per_object.py):
seeded init (CPU), per-object logits / bits through the exact API and the
SIMT query kernel, one optimiser step and a 2-epoch loss curve (GPU)."""

import hashlib

import numpy as np
import pytest


def _cfg():
    from golden_cfg import small_config
    cfg = small_config(seed=6)
    cfg.sharing = "per_object"
    return cfg


def _hash(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_per_object_init_matches_reference(golden, scenes):
    from paper_2306_07191_b200.nif import NifModel
    s = scenes("overlap")
    m = NifModel(_cfg(), s.n_objects, s.diagonal, device="cpu")
    assert m.outer.n_heads == s.n_objects and m.inner.n_heads == s.n_objects
    assert _hash(m.model_arrays()) == bytes(golden("per_object")["model_hash"]).decode()


@pytest.mark.gpu
def test_per_object_logits_and_bits(cuda, golden, scenes):
    from paper_2306_07191_b200 import build_model, infer_records
    from paper_2306_07191_b200.nif import (encode_inner_arrays, encode_outer_arrays,
                                           logits_arrays, query_family)
    from paper_2306_07191_b200.scene import QueryRecords
    g, gp = golden("overlap"), golden("per_object")
    m = build_model(_cfg(), scenes("overlap"))
    kind, obj, coord = g["rec_kind"], g["rec_obj"].astype(np.int64), g["rec_coord"]
    for fam, k, width, enc in (("outer", 0, 4, encode_outer_arrays),
                               ("inner", 1, 5, encode_inner_arrays)):
        sel = kind == k
        x = enc(m, obj[sel], coord[sel, :width])
        ref = gp[f"logit_{fam}"]
        np.testing.assert_array_equal(logits_arrays(m, fam, obj[sel], x), ref)
        simt = query_family(m, fam, obj[sel], coord[sel, :width], impl=1)
        assert np.abs(simt - ref[:, 0]).max() <= 1e-4
    rec = QueryRecords(kind, g["rec_obj"], g["rec_ray"], coord, int(g["rec_degenerate"]))
    # fp32 SIMT: the reference's bits exactly; fp16 tensor cores (bucketed):
    # the north-star thresholded agreement
    np.testing.assert_array_equal(infer_records(m, rec, impl=1), gp["infer_bits"])
    assert np.mean(infer_records(m, rec) == gp["infer_bits"]) >= 0.999


@pytest.mark.gpu
def test_per_object_training_matches_reference(cuda, golden, scenes):
    from paper_2306_07191_b200 import build_model
    from paper_2306_07191_b200.train import SampleSet, train, train_batch
    g, gp = golden("overlap"), golden("per_object")
    m = build_model(_cfg(), scenes("overlap"))
    loss = train_batch(m, "outer", g["samples_outer_obj"][:256], g["samples_outer_coord"][:256],
                       g["samples_outer_label"][:256])
    assert loss == pytest.approx(float(gp["step_loss_outer"]), rel=1e-5)
    loss = train_batch(m, "inner", g["samples_inner_obj"][:512], g["samples_inner_coord"][:512],
                       g["samples_inner_label"][:512])
    assert loss == pytest.approx(float(gp["step_loss_inner"]), rel=1e-5)
    close = total = 0
    for i, arr in enumerate(m.model_arrays()):
        ref = gp[f"step_param_{i:03d}"]
        close += int(np.sum(np.abs(arr - ref) <= 1e-6))
        total += arr.size
    assert close / total >= 0.995, close / total
    m2 = build_model(_cfg(), scenes("overlap"))
    smp = SampleSet.from_host({k: g["samples_" + k] for k in (
        "outer_obj", "outer_coord", "outer_label", "outer_ray", "inner_obj", "inner_coord",
        "inner_label", "inner_ray")})
    curve = train(m2, smp, epochs=2)
    np.testing.assert_allclose(curve, gp["curve"], rtol=0.05)


@pytest.mark.gpu
def test_per_object_tensor_core_bucketed(cuda, golden, scenes):
    """nif_query_bucketed_dev: records counting-sorted by object into
    128-row tiles, each tile on its object's MLP with A in TMEM; logits
    within the tensor-core tolerance of the reference, and the device pass
    (VisibilityEngine) answers like the fp32 SIMT path."""
    import torch
    from test_gpu_mlp import LOGIT_TOL_TC, _randomize
    from paper_2306_07191_b200 import build_model
    from paper_2306_07191_b200.nif import NifConfig, NifModel, query_family
    from paper_2306_07191_b200.pipeline import VisibilityEngine, sample_pass_dev, shadow_rays_dev
    from paper_2306_07191_b200.synthetic import c2
    g, gp = golden("overlap"), golden("per_object")
    m = build_model(_cfg(), scenes("overlap"))
    kind, obj, coord = g["rec_kind"], g["rec_obj"].astype(np.int64), g["rec_coord"]
    for fam, k, width in (("outer", 0, 4), ("inner", 1, 5)):
        sel = kind == k
        tc = query_family(m, fam, obj[sel], coord[sel, :width], impl=2).astype(np.float64)
        assert np.abs(tc - gp[f"logit_{fam}"][:, 0]).max() <= LOGIT_TOL_TC
    # O(1) logits, many objects, partial tiles per object
    cfg = NifConfig(seed=9, sharing="per_object")
    mm = NifModel(cfg, 7)
    _randomize(mm, 2)
    rng = np.random.default_rng(3)
    for n in (1, 130, 5000):
        o = rng.integers(0, 7, n)
        c = rng.random((n, 5))
        for fam, width in (("outer", 4), ("inner", 5)):
            simt = query_family(mm, fam, o, c[:, :width], impl=1).astype(np.float64)
            tc = query_family(mm, fam, o, c[:, :width], impl=2).astype(np.float64)
            assert np.abs(tc - simt).max() <= LOGIT_TOL_TC, (fam, n)
    # whole pass on a 13-object scene
    scene = c2(320, 180)
    model = build_model(NifConfig(seed=0, sharing="per_object"), scene)
    data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
    _, oo, dd, tt = shadow_rays_dev(data, require_emit=False)
    n = int(tt.numel())
    occ = {}
    for impl in (0, 1):
        eng = VisibilityEngine(scene, model, n, impl=impl)
        assert eng.bucket is not None
        eng.origins[:n].copy_(oo)
        eng.dirs[:n].copy_(dd)
        eng.tmaxs[:n].copy_(tt)
        eng.run(n)
        torch.cuda.synchronize()
        occ[impl] = eng.occ[:n].cpu().numpy().copy()
    assert np.mean(occ[0] == occ[1]) >= 0.999
