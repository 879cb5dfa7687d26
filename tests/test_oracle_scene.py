"""The oracle's own restatement of the reference's scene build and model
init (oracle/refscene.py: meshgen, _build_sah in C, pack_scene, seeded
init) -- what the reference arm of bench.py runs without the package --
pinned to the reference's golden pack hashes and model hashes, and to the
package's C2 bench scene. CPU only."""

import hashlib

import numpy as np
import pytest

from scenes import RECIPES

KEYS = ("t_lo", "t_hi", "t_a", "t_b", "t_leaf", "t_order", "roots", "b_lo", "b_hi", "b_a",
        "b_b", "b_leaf", "v0", "v1", "v2", "n0", "n1", "n2", "src", "obox_lo", "obox_hi")


def _pack_hash(pack):
    h = hashlib.sha256()
    for k in KEYS:
        h.update(np.ascontiguousarray(getattr(pack, k)).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", list(RECIPES))
def test_oracle_scene_matches_reference(name, golden):
    from oracle import refscene
    g = golden(name)
    s = refscene.from_recipe(RECIPES[name])
    assert _pack_hash(s.pack) == bytes(g["pack_hash"]).decode()
    assert s.diagonal == float(g["diagonal"])
    assert s.epsilon_t == float(g["epsilon_t"])


def test_oracle_shadow_rays_match_reference(golden):
    """cli.py:170-183 rays from the oracle's own scene equal the golden rays."""
    from oracle import refscene
    g = golden("c1s")
    o, d, t = refscene.from_recipe(RECIPES["c1s"]).shadow_rays(0)
    assert np.array_equal(o, g["origins"]) and np.array_equal(d, g["dirs"])
    assert np.array_equal(t, g["tmaxs"])


def test_oracle_init_matches_reference(golden):
    """nif.py:181-223 seeded init restated: the reference's model hash."""
    from oracle import refscene
    from golden_cfg import small_config  # noqa: F401  (documents the config)
    g = golden("c1s")
    o_heads, i_heads, grids = refscene.init_model(
        2, seed=0, outer=(6, 64, 2, 32, 3), inner=(13, 48, 3, 16, 5, 16, 3))
    h = hashlib.sha256()
    for heads in (o_heads, i_heads):
        for layers in heads:
            for w, b in layers:
                h.update(np.ascontiguousarray(w).tobytes())
                h.update(np.ascontiguousarray(b).tobytes())
    for gr in grids:
        for k in ("outer_pos", "outer_dir", "inner_pos", "inner_dir", "inner_dist"):
            h.update(np.ascontiguousarray(gr[k]).tobytes())
    assert h.hexdigest() == bytes(g["model_hash"]).decode()


def test_oracle_c2_scene_matches_package():
    """The bench's C2 scene built by the oracle alone equals the package's
    build (pack, diagonal, route mask, light tables, camera basis)."""
    from oracle import refscene
    from paper_2306_07191_b200 import synthetic
    ref = refscene.c2(192, 108)
    pkg = synthetic.c2(192, 108)
    assert _pack_hash(ref.pack) == _pack_hash(pkg.pack)
    assert ref.diagonal == pkg.diagonal and ref.epsilon_t == pkg.epsilon_t
    assert np.array_equal(ref.nif_route_mask(None), pkg.nif_route_mask(None))
    for a, b in zip(ref.light_tables(), pkg.light_tables()):
        assert np.array_equal(a, b)
    for a, b in zip(ref.camera.basis(), pkg.camera.basis()):
        assert np.array_equal(np.asarray(a), np.asarray(b))
