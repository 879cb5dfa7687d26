"""Pin the oracle's numpy restatement of the training step against the
reference's own _train_batch / train outputs (golden). CPU only."""

import numpy as np
import pytest

from scenes import RECIPES


def _golden_model(name, golden, scenes):
    from golden_cfg import small_config
    from oracle.oracle import OModel
    from paper_2306_07191_b200.nif import init_arrays
    s = scenes(name)
    outer, inner, grids, _, _ = init_arrays(small_config(), s.n_objects)
    return OModel(outer[0], inner[0], grids)


def _model_arrays(m):
    out = []
    for mlp in (m.outer, m.inner):
        for l in mlp.layers:
            out += [l.w, l.b]
    for g in m.grids:
        out += [g[k].latents for k in ("outer_pos", "outer_dir", "inner_pos", "inner_dir",
                                       "inner_dist")]
    return out


@pytest.mark.parametrize("name", ["c1s", "overlap", "area"])
def test_oracle_train_batch_matches_reference(name, golden, scenes):
    g = golden(name)
    m = _golden_model(name, golden, scenes)
    if "step_loss_outer" in g:
        n = min(256, len(g["samples_outer_obj"]))
        loss = m.train_batch("outer", g["samples_outer_obj"][:n], g["samples_outer_coord"][:n],
                             g["samples_outer_label"][:n])
        assert loss == pytest.approx(float(g["step_loss_outer"]), rel=1e-12)
    if "step_loss_inner" in g:
        n = min(512, len(g["samples_inner_obj"]))
        loss = m.train_batch("inner", g["samples_inner_obj"][:n], g["samples_inner_coord"][:n],
                             g["samples_inner_label"][:n])
        assert loss == pytest.approx(float(g["step_loss_inner"]), rel=1e-12)
    got = _model_arrays(m)
    for i, arr in enumerate(got):
        ref = g[f"step_param_{i:03d}"]
        np.testing.assert_array_equal(arr, ref, err_msg=f"param {i}")


@pytest.mark.parametrize("name", ["c1s", "overlap"])
def test_oracle_train_curve_matches_reference(name, golden, scenes):
    g = golden(name)
    m = _golden_model(name, golden, scenes)
    samples = {k: g["samples_" + k] for k in ("outer_obj", "outer_coord", "outer_label",
                                             "inner_obj", "inner_coord", "inner_label")}
    curve = m.train(samples, epochs=2, seed=0, bo=256, bi=512)
    np.testing.assert_allclose(curve, g["curve"], rtol=1e-10)
