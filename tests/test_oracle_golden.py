"""Pin the scene build and the CPU oracle against the reference's golden
vectors (tests/golden/*.npz, produced by make_golden.py from the reference
itself). CPU only."""

import hashlib

import numpy as np
import pytest

from scenes import RECIPES

SCENES = list(RECIPES)


def _pack_hash(pack):
    h = hashlib.sha256()
    for k in ("t_lo", "t_hi", "t_a", "t_b", "t_leaf", "t_order", "roots", "b_lo", "b_hi",
              "b_a", "b_b", "b_leaf", "v0", "v1", "v2", "n0", "n1", "n2", "src", "obox_lo",
              "obox_hi"):
        h.update(np.ascontiguousarray(getattr(pack, k)).tobytes())
    return h.hexdigest()


def _hash(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", SCENES)
def test_scene_pack_matches_reference(name, golden, scenes):
    """meshgen + native SAH builder + pack reproduce the reference trees
    byte for byte (bvh.py:34-303, 1000-1045)."""
    g = golden(name)
    s = scenes(name)
    assert _pack_hash(s.pack) == bytes(g["pack_hash"]).decode()
    assert s.diagonal == float(g["diagonal"])
    assert s.epsilon_t == float(g["epsilon_t"])


@pytest.mark.parametrize("name", SCENES)
def test_oracle_gather_bit_exact(name, golden, scenes):
    from oracle import oracle
    g = golden(name)
    s = scenes(name)
    osc = oracle.OracleScene(s.pack, s.epsilon_t)
    kind, obj, ray, coord, bvh_occ, n_deg = oracle.gather(
        osc, g["origins"], g["dirs"], g["tmaxs"], g["route"])
    np.testing.assert_array_equal(kind, g["rec_kind"])
    np.testing.assert_array_equal(obj, g["rec_obj"])
    np.testing.assert_array_equal(ray, g["rec_ray"])
    np.testing.assert_array_equal(coord, g["rec_coord"])
    np.testing.assert_array_equal(bvh_occ, g["bvh_occ"])
    assert n_deg == int(g["rec_degenerate"])


@pytest.mark.parametrize("name", SCENES)
def test_oracle_labels_and_bvh_bit_exact(name, golden, scenes):
    from oracle import oracle
    g = golden(name)
    s = scenes(name)
    osc = oracle.OracleScene(s.pack, s.epsilon_t)
    vis = oracle.label_visible(osc, g["rec_obj"], g["rec_ray"], g["origins"], g["dirs"],
                               g["tmaxs"])
    np.testing.assert_array_equal(vis.astype(np.float32), g["labels"])
    occ = oracle.bvh_occluded(osc, g["origins"], g["dirs"], g["tmaxs"])
    np.testing.assert_array_equal(occ, g["bvh_backend"])


@pytest.mark.parametrize("name", SCENES)
def test_oracle_sample_pass_bit_exact(name, golden, scenes):
    from oracle import oracle
    g = golden(name)
    s = scenes(name)
    osc = oracle.OracleScene(s.pack, s.epsilon_t)
    cum, kind, data = s.light_tables()
    out = oracle.sample_pass(osc, s.camera, cum, kind, data, s.seed, 0)
    got = _hash([out[k] for k in ("hit", "t", "obj", "point", "normal", "pdir", "ldir", "tmax",
                                  "pdf", "emit")])
    assert got == bytes(g["pass0_hash"]).decode()
    u = oracle.sample_pass(osc, s.camera, cum, kind, data, s.seed, 1, sampler="uniform")
    np.testing.assert_array_equal(u["hit"], g["pass1u_hit"])
    np.testing.assert_array_equal(u["point"], g["pass1u_point"])
    np.testing.assert_allclose(u["ldir"], g["pass1u_ldir"], rtol=0, atol=1e-15)
