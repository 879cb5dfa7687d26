"""Golden fixtures for the query-object API (nif.py:428-464
infer_occlusion / infer_geometry), written by running the
REFERENCE.

Run in the development container only (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_infer.py

Writes tests/golden/infer.npz: for 3 objects at the default resolutions
(R 256/128), models with O(1) latents and biases (golden_cfg.perturb_arrays,
the same draws the tests apply to the package model), a mixed batch of
outer/inner queries (golden_cfg.random_queries), the reference's
infer_occlusion bits and forward probabilities (occlusion head, shared and
per_object), infer_geometry normals and depth (geometry head), and the
zero-MLP known answer of SPEC.md:415.
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
from niftrace.nif import (  # noqa: E402
    encode_inner_arrays, encode_outer_arrays, forward_inner_arrays, forward_outer_arrays,
    infer_geometry, infer_occlusion,
)

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parent))
from golden_cfg import perturb_arrays, random_queries  # noqa: E402

N_OBJ = 3
N_Q = 6000
DIAGONAL = 7.25


def ref_model(head, sharing, seed, pseed):
    cfg = nt.NifConfig(seed=seed)
    cfg.head = head
    cfg.sharing = sharing
    m = nt.NifModel(cfg, N_OBJ, DIAGONAL)
    grids = [{"outer_pos": g.outer_pos.latents, "outer_dir": g.outer_dir.latents,
              "inner_pos": g.inner_pos.latents, "inner_dir": g.inner_dir.latents,
              "inner_dist": g.inner_dist.latents} for g in m.grids]
    outer = [[(l.w, l.b) for l in mlp.layers] for mlp in m.outer_mlps]
    inner = [[(l.w, l.b) for l in mlp.layers] for mlp in m.inner_mlps]
    perturb_arrays(outer, inner, grids, seed=pseed)
    return m


def queries(kind, obj, coord):
    out = []
    for k, o, c in zip(kind, obj, coord):
        p = nt.SphericalCoord(float(c[0]), float(c[1]))
        d = nt.SphericalCoord(float(c[2]), float(c[3]))
        if k == 0:
            out.append(nt.OuterQuery(int(o), p, d))
        else:
            out.append(nt.InnerQuery(int(o), p, d, float(c[4])))
    return out


def main():
    kind, obj, coord = random_queries(N_Q, N_OBJ, seed=7)
    qs = queries(kind, obj, coord)
    d = {"kind": kind, "obj": obj, "coord": coord}
    for sharing in ("shared", "per_object"):
        # the first perturbation seed whose answers are mixed (not all one bit)
        for pseed in range(100, 300):
            m = ref_model("occlusion", sharing, 0, pseed)
            occ = infer_occlusion(m, qs)
            if 0.25 < occ.mean() < 0.75:
                break
        d[f"pseed_{sharing}"] = np.int64(pseed)
        d[f"occ_{sharing}"] = occ
        prob = np.zeros(N_Q)
        for k, enc, fwd, w in ((0, encode_outer_arrays, forward_outer_arrays, 4),
                               (1, encode_inner_arrays, forward_inner_arrays, 5)):
            sel = kind == k
            prob[sel] = fwd(m, obj[sel], enc(m, obj[sel], coord[sel, :w]))[:, 0]
        d[f"prob_{sharing}"] = prob
    g = ref_model("geometry", "shared", 1, 101)
    normals, depth = infer_geometry(g, qs)
    d["geo_normal"], d["geo_depth"] = normals, depth
    # an untrained model with a zero MLP gives p = 0.5 -> visible
    z = nt.NifModel(nt.NifConfig(seed=0), N_OBJ, DIAGONAL)
    for mlp in z.outer_mlps + z.inner_mlps:
        for layer in mlp.layers:
            layer.w[...] = 0.0
            layer.b[...] = 0.0
    d["occ_zero"] = infer_occlusion(z, qs)
    assert not d["occ_zero"].any()
    assert len(infer_occlusion(z, [])) == 0
    np.savez_compressed(OUT / "infer.npz", **d)
    print({k: v.shape for k, v in d.items()}, "occluded:", d["occ_shared"].mean(),
          d["occ_per_object"].mean(), d["pseed_shared"], d["pseed_per_object"])


if __name__ == "__main__":
    main()
