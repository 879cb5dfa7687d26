"""Golden geometry-head samples + training written by the REFERENCE
(nif.py:547-566 _label_geometry, 569-674 collect_samples(labeler="geometry"),
682-795 training with head="geometry").

Run in the development container only (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_geometry.py

Note: the shipped reference cannot run this path (bvh.py uses math without
importing it); see the in-memory binding below.

Writes tests/golden/geometry.npz: the SampleSet of 2 spp on the "overlap"
recipe scene at 48x40 and the 2-epoch loss curve of a geometry-head model
(small grids) trained on it.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import math  # noqa: E402

import numpy as np  # noqa: E402

import niftrace.bvh as _ref_bvh  # noqa: E402
from niftrace.nif import NifConfig, NifModel, collect_samples, train  # noqa: E402

# The reference's _k_label_geometry (bvh.py:920-950) calls math.sqrt but
# bvh.py never imports math, so the geometry labeler raises NameError as
# shipped. Bind the module attribute in memory (no file is modified) so the
# reference's own kernel compiles and runs with its evident semantics.
if not hasattr(_ref_bvh, "math"):
    _ref_bvh.math = math

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT))
sys.path.insert(0, str(OUT.parent))
from make_golden import build_ref_scene  # noqa: E402
from scenes import RECIPES  # noqa: E402


RECIPE = "overlap"


def geometry_config():
    cfg = NifConfig(seed=4, head="geometry")
    cfg.outer.grid_resolution = 32
    cfg.inner.grid_resolution = 16
    return cfg


def main():
    recipe = dict(RECIPES[RECIPE])
    recipe["camera"] = {**recipe["camera"], "width": 48, "height": 40}
    scene = build_ref_scene(recipe)
    s = collect_samples(scene, spp=2, labeler="geometry", seed=scene.seed, threads=1)
    model = NifModel(geometry_config(), scene.n_objects, scene.diagonal, dtype=np.float32)
    curve = train(model, s, epochs=2)
    np.savez_compressed(
        OUT / "geometry.npz", outer_obj=s.outer_obj, outer_coord=s.outer_coord,
        outer_label=s.outer_label, outer_ray=s.outer_ray, inner_obj=s.inner_obj,
        inner_coord=s.inner_coord, inner_label=s.inner_label, inner_ray=s.inner_ray,
        curve=curve)


if __name__ == "__main__":
    main()
