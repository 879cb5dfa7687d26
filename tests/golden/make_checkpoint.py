"""Golden NIF1 checkpoints written by the REFERENCE (scene_io.py:325-341).

Run in the development container only (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_checkpoint.py

Writes tests/golden/ckpt_shared.nif1 and ckpt_per_object.nif1 (small
configs: R = 8/4, so the files are a few tens of KB) plus a JSON with the
sha256 of every array, so the package's reader/writer are pinned byte for
byte against the reference's.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from niftrace.nif import NifConfig, NifModel  # noqa: E402
from niftrace.scene_io import _model_arrays, save_checkpoint  # noqa: E402

OUT = Path(__file__).resolve().parent


def small_config(sharing, seed):
    cfg = NifConfig(seed=seed, sharing=sharing)
    cfg.outer.grid_resolution = 8
    cfg.inner.grid_resolution = 4
    cfg.inner.dist_resolution = 6
    cfg.outer.hidden_width = 16
    cfg.inner.hidden_width = 16
    return cfg


def main():
    info = {}
    for sharing, seed, n_obj in (("shared", 3, 2), ("per_object", 5, 3)):
        cfg = small_config(sharing, seed)
        model = NifModel(cfg, n_obj, 2.5, dtype=np.float32)
        # perturb so a loader that silently keeps init values is caught
        rng = np.random.default_rng(seed)
        for a in _model_arrays(model):
            a += rng.standard_normal(a.shape).astype(a.dtype) * 0.01
        path = OUT / f"ckpt_{sharing}.nif1"
        save_checkpoint(model, path)
        info[sharing] = {
            "n_objects": n_obj, "scene_diagonal": 2.5, "config": cfg.to_dict(),
            "file_sha256": hashlib.sha256(path.read_bytes()).hexdigest(),
            "arrays_sha256": [hashlib.sha256(np.ascontiguousarray(a, "<f4").tobytes()).hexdigest()
                              for a in _model_arrays(model)],
        }
    (OUT / "ckpt.json").write_text(json.dumps(info, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
