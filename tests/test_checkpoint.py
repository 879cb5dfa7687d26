"""NIF1 checkpoints (scene_io.py:308-387): the package reads files written
by the reference (golden, tests/golden/make_checkpoint.py) array for
array, writes them back byte for byte, and raises the reference's
SceneFormatError on malformed input. CPU only (the model lives on the
CPU device here)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).parent / "golden"
INFO = json.loads((GOLD / "ckpt.json").read_text())


@pytest.mark.parametrize("sharing", ["shared", "per_object"])
def test_reads_reference_checkpoint(sharing, tmp_path):
    from paper_2306_07191_b200.checkpoint import load_checkpoint, save_checkpoint
    info = INFO[sharing]
    src = GOLD / f"ckpt_{sharing}.nif1"
    m = load_checkpoint(src, device="cpu")
    assert m.n_objects == info["n_objects"]
    assert m.scene_diagonal == info["scene_diagonal"]
    assert m.config.to_dict() == info["config"]
    got = [hashlib.sha256(np.ascontiguousarray(a, "<f4").tobytes()).hexdigest()
           for a in m.model_arrays()]
    assert got == info["arrays_sha256"]
    # round trip: the package writes the identical file
    out = tmp_path / "rt.nif1"
    save_checkpoint(m, out)
    assert out.read_bytes() == src.read_bytes()


def test_load_into_and_mismatch(tmp_path):
    from paper_2306_07191_b200.checkpoint import SceneFormatError, load_checkpoint
    from paper_2306_07191_b200.nif import NifConfig, NifModel
    src = GOLD / "ckpt_shared.nif1"
    m = load_checkpoint(src, device="cpu")
    into = NifModel(NifConfig.from_dict(INFO["shared"]["config"]), 2, 1.0, device="cpu")
    load_checkpoint(src, into=into)
    for a, b in zip(m.model_arrays(), into.model_arrays()):
        np.testing.assert_array_equal(a, b)
    other = NifModel(NifConfig(seed=0), 2, 1.0, device="cpu")
    with pytest.raises(SceneFormatError, match="does not match the model"):
        load_checkpoint(src, into=other)


def test_malformed_files(tmp_path):
    from paper_2306_07191_b200.checkpoint import SceneFormatError, load_checkpoint
    data = (GOLD / "ckpt_shared.nif1").read_bytes()
    cases = {"magic": (b"XXXX" + data[4:], "not a model checkpoint"),
             "version": (data[:4] + (2).to_bytes(4, "little") + data[8:], "unsupported"),
             "truncated": (data[:-5], "truncated"),
             "trailing": (data + b"\0", "trailing bytes")}
    for name, (blob, msg) in cases.items():
        p = tmp_path / f"{name}.nif1"
        p.write_bytes(blob)
        with pytest.raises(SceneFormatError, match=msg):
            load_checkpoint(p, device="cpu")


def test_adam_sidecar_round_trip(tmp_path):
    import torch
    from paper_2306_07191_b200.checkpoint import load_checkpoint, save_checkpoint
    m = load_checkpoint(GOLD / "ckpt_shared.nif1", device="cpu")
    g = torch.Generator().manual_seed(0)
    for fam in (m.outer, m.inner):
        fam.m.copy_(torch.rand(fam.m.shape, generator=g))
        fam.v.copy_(torch.rand(fam.v.shape, generator=g))
        fam.grid_steps.fill_(7)
        fam.mlp_steps.fill_(9)
    p = tmp_path / "m.nif1"
    save_checkpoint(m, p, adam=True)
    # the NIF1 part is unchanged (the reference can still read it)
    assert p.read_bytes() == (GOLD / "ckpt_shared.nif1").read_bytes()
    m2 = load_checkpoint(p, device="cpu")
    for fam, fam2 in ((m.outer, m2.outer), (m.inner, m2.inner)):
        assert torch.equal(fam.m, fam2.m) and torch.equal(fam.v, fam2.v)
        assert int(fam2.grid_steps[0]) == 7 and int(fam2.mlp_steps[0]) == 9


def test_adam_sidecar_stale(tmp_path):
    """A re-save without optimiser state removes the old sidecar; a sidecar
    belonging to different weights is rejected."""
    import shutil
    from paper_2306_07191_b200.checkpoint import (SceneFormatError, load_checkpoint,
                                                  save_checkpoint)
    m = load_checkpoint(GOLD / "ckpt_shared.nif1", device="cpu")
    m.outer.grid_steps.fill_(5)
    p = tmp_path / "m.nif1"
    save_checkpoint(m, p, adam=True)
    side = tmp_path / "m.nif1.adam"
    assert side.exists()
    keep = tmp_path / "old.adam"
    shutil.copy(side, keep)
    save_checkpoint(m, p)  # weights only
    assert not side.exists()
    m2 = load_checkpoint(p, device="cpu")
    assert int(m2.outer.grid_steps[0]) == 0
    # a sidecar written for other weights
    m.outer.part("w").add_(1.0)
    save_checkpoint(m, p)
    shutil.copy(keep, side)
    with pytest.raises(SceneFormatError, match="different checkpoint"):
        load_checkpoint(p, device="cpu")
