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
    np.testing.assert_array_equal(infer_records(m, rec), gp["infer_bits"])


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
