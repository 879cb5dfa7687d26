"""Golden fixtures for sharing="per_object" (one MLP per object,
nif.py:91-92, 230-234, 380-397 and the per-object Adam of nif.py:731-749),
written by running the REFERENCE.

Run in the development container only (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_per_object.py

Writes tests/golden/per_object.npz on the "overlap" recipe (3 objects):
model-init hash, per-object logits of every gathered record, inference
bits, one outer + one inner _train_batch step (losses + all parameters)
and a 2-epoch loss curve on the occlusion samples in overlap.npz.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import niftrace as nt  # noqa: E402
from niftrace.nif import SampleSet  # noqa: E402
from niftrace.renderer import QueryRecords  # noqa: E402
from niftrace.nif import (  # noqa: E402
    _flat_mlp, _k_dense_forward, _train_batch, encode_inner_arrays, encode_outer_arrays,
    infer_records,
)
from niftrace.scene_io import _model_arrays  # noqa: E402

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT))
sys.path.insert(0, str(OUT.parent))
from make_golden import arrays_hash, build_ref_scene, small_config  # noqa: E402
from scenes import RECIPES  # noqa: E402


def main():
    scene = build_ref_scene(RECIPES["overlap"])
    g = np.load(OUT / "overlap.npz")
    cfg = small_config(seed=6)
    cfg.sharing = "per_object"
    model = nt.build_model(cfg, scene)
    d = {"model_hash": np.frombuffer(arrays_hash(list(_model_arrays(model))).encode(), np.uint8)}
    kind, obj, coord = g["rec_kind"], g["rec_obj"].astype(np.int64), g["rec_coord"]
    for fam, k, width, enc, mlps in (("outer", 0, 4, encode_outer_arrays, model.outer_mlps),
                                     ("inner", 1, 5, encode_inner_arrays, model.inner_mlps)):
        m = kind == k
        x = enc(model, obj[m], coord[m, :width])
        out = np.empty((int(m.sum()), 1), np.float64)
        for o in np.unique(obj[m]):
            sel = obj[m] == o
            w, b, dims = _flat_mlp(mlps[int(o)])
            part = np.empty((int(sel.sum()), 1), np.float64)
            _k_dense_forward(w, b, dims, 0, np.ascontiguousarray(x[sel]), part, 0, len(part))
            out[sel] = part
        d[f"logit_{fam}"] = out
    rec = QueryRecords(kind, g["rec_obj"], g["rec_ray"], coord, int(g["rec_degenerate"]))
    d["infer_bits"] = infer_records(model, rec)
    step_model = nt.build_model(cfg, scene)
    so, sc, sl = g["samples_outer_obj"], g["samples_outer_coord"], g["samples_outer_label"]
    io_, ic, il = g["samples_inner_obj"], g["samples_inner_coord"], g["samples_inner_label"]
    d["step_loss_outer"] = np.float64(_train_batch(step_model, "outer", so[:256], sc[:256],
                                                   sl[:256]))
    d["step_loss_inner"] = np.float64(_train_batch(step_model, "inner", io_[:512], ic[:512],
                                                   il[:512]))
    for i, arr in enumerate(_model_arrays(step_model)):
        d[f"step_param_{i:03d}"] = np.array(arr)
    samples = SampleSet(head="occlusion", outer_obj=so, outer_coord=sc, outer_label=sl,
                           outer_ray=g["samples_outer_ray"], inner_obj=io_, inner_coord=ic,
                           inner_label=il, inner_ray=g["samples_inner_ray"])
    curve_model = nt.build_model(cfg, scene)
    d["curve"] = nt.train(curve_model, samples, epochs=2)
    np.savez_compressed(OUT / "per_object.npz", **d)
    print("per_object:", {k: np.shape(v) for k, v in d.items() if not k.startswith("step_param")})


if __name__ == "__main__":
    main()
