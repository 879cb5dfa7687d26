"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the development container only (the reference lives at
/root/reference and is not available on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes tests/golden/<scene>.npz. Every array is produced by the
reference's own public functions on scenes built from the reference's
meshgen; the package and the oracle are pinned against these files.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import niftrace as nt  # noqa: E402
from niftrace import meshgen  # noqa: E402
from niftrace.bvh import build_bottom  # noqa: E402
from niftrace.cli import _bench_shadow_rays  # noqa: E402
from niftrace.nif import (  # noqa: E402
    _flat_mlp, _k_dense_forward, _label_occlusion, _train_batch, collect_samples,
    encode_inner_arrays, encode_outer_arrays, forward_inner_arrays, forward_outer_arrays,
    infer_records,
)
from niftrace.renderer import gather_queries, sample_pass  # noqa: E402

OUT = Path(__file__).resolve().parent

# Scene recipes shared with tests/scenes.py (same parameters on both sides).
sys.path.insert(0, str(OUT.parent))
from scenes import RECIPES  # noqa: E402


def build_ref_scene(recipe):
    objs = []
    for od in recipe["objects"]:
        kind, args = od["mesh"]
        v, f, n = getattr(meshgen, kind)(*args)
        v0, v1, v2, n0, n1, n2 = meshgen.mesh_arrays(v, f, n)
        s = od.get("scale", 1.0)
        t = np.asarray(od.get("translate", (0.0, 0.0, 0.0)), np.float64)
        v0, v1, v2 = v0 * s + t, v1 * s + t, v2 * s + t
        objs.append(nt.SceneObject(od["name"], build_bottom((v0, v1, v2, n0, n1, n2)),
                                   np.asarray(od["albedo"], np.float64),
                                   od.get("nif_enabled", True)))
    lights = []
    for ld in recipe["lights"]:
        if ld["kind"] == "point":
            lights.append(nt.PointLight(np.asarray(ld["position"], np.float64),
                                        np.asarray(ld["intensity"], np.float64)))
        else:
            lights.append(nt.AreaLight.from_corners(ld["corners"], ld["radiance"]))
    c = recipe["camera"]
    cam = nt.Camera(np.asarray(c["position"], np.float64), np.asarray(c["look_at"], np.float64),
                    np.asarray(c.get("up", (0, 0, 1)), np.float64), c["fov"], c["width"],
                    c["height"])
    return nt.Scene(objs, lights, cam, recipe["seed"])


def pack_hash(pack) -> str:
    h = hashlib.sha256()
    for k in ("t_lo", "t_hi", "t_a", "t_b", "t_leaf", "t_order", "roots", "b_lo", "b_hi",
              "b_a", "b_b", "b_leaf", "v0", "v1", "v2", "n0", "n1", "n2", "src", "obox_lo",
              "obox_hi"):
        h.update(np.ascontiguousarray(getattr(pack, k)).tobytes())
    return h.hexdigest()


def arrays_hash(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def model_arrays(model):
    for mlp in model.outer_mlps + model.inner_mlps:
        for layer in mlp.layers:
            yield layer.w
            yield layer.b
    for g in model.grids:
        yield g.outer_pos.latents
        yield g.outer_dir.latents
        yield g.inner_pos.latents
        yield g.inner_dir.latents
        yield g.inner_dist.latents


def small_config(seed=0):
    cfg = nt.NifConfig(seed=seed)
    cfg.outer.grid_resolution = 32
    cfg.inner.grid_resolution = 16
    cfg.inner.dist_resolution = 16
    cfg.outer.batch_size = 256
    cfg.inner.batch_size = 512
    return cfg


def main():
    for name, recipe in RECIPES.items():
        scene = build_ref_scene(recipe)
        d = {}
        d["pack_hash"] = np.frombuffer(pack_hash(scene.pack).encode(), np.uint8)
        d["diagonal"] = np.float64(scene.diagonal)
        d["epsilon_t"] = np.float64(scene.epsilon_t)
        # sample pass (s = 0), pinned by hash; shadow rays kept verbatim
        data = sample_pass(scene, scene.camera, 0, scene.seed, 1)
        d["pass0_hash"] = np.frombuffer(arrays_hash(
            [data[k] for k in ("hit", "t", "obj", "point", "normal", "pdir", "ldir", "tmax",
                               "pdf", "emit")]).encode(), np.uint8)
        data_u = sample_pass(scene, scene.camera, 1, scene.seed, 1, sampler="uniform")
        d["pass1u_hit"] = data_u["hit"]
        d["pass1u_obj"] = data_u["obj"]
        d["pass1u_point"] = data_u["point"]
        d["pass1u_ldir"] = data_u["ldir"]
        rays = _bench_shadow_rays(scene, 1, 1)
        d["origins"], d["dirs"], d["tmaxs"] = rays.origins, rays.dirs, rays.tmaxs
        route = scene.nif_route_mask(None)
        d["route"] = route
        rec, bvh_occ = gather_queries(scene, rays, route, 1)
        d["rec_kind"], d["rec_obj"], d["rec_ray"], d["rec_coord"] = (
            rec.kind, rec.obj, rec.ray, rec.coord)
        d["rec_degenerate"] = np.int64(rec.degenerate_count)
        d["bvh_occ"] = bvh_occ
        d["labels"] = _label_occlusion(scene, rec, rays, 1)
        d["bvh_backend"] = nt.BvhBackend().occluded(scene, rays, 1)
        # model (small grids), features, logits, bits
        cfg = small_config()
        model = nt.build_model(cfg, scene)
        d["model_hash"] = np.frombuffer(arrays_hash(list(model_arrays(model))).encode(), np.uint8)
        om = rec.kind == 0
        im = rec.kind == 1
        o_obj = rec.obj[om].astype(np.int64)
        i_obj = rec.obj[im].astype(np.int64)
        xo = encode_outer_arrays(model, o_obj, rec.coord[om, 0:4])
        xi = encode_inner_arrays(model, i_obj, rec.coord[im, 0:5])
        d["feat_outer"], d["feat_inner"] = xo, xi
        d["prob_outer"] = forward_outer_arrays(model, o_obj, xo)
        d["prob_inner"] = forward_inner_arrays(model, i_obj, xi)
        for fam, x, mlp in (("outer", xo, model.outer_mlps[0]), ("inner", xi, model.inner_mlps[0])):
            w, b, dims = _flat_mlp(mlp)
            out = np.empty((len(x), 1), np.float64)
            if len(x):
                _k_dense_forward(w, b, dims, 0, np.ascontiguousarray(x), out, 0, len(x))
            d[f"logit_{fam}"] = out
        d["infer_bits"] = infer_records(model, rec)
        # training: samples (2 spp), one outer + one inner step, 2-epoch curve
        samples = collect_samples(scene, spp=2, seed=scene.seed, threads=1)
        for k in ("outer_obj", "outer_coord", "outer_label", "outer_ray", "inner_obj",
                  "inner_coord", "inner_label", "inner_ray"):
            d["samples_" + k] = getattr(samples, k)
        step_model = nt.build_model(cfg, scene)
        n_o = min(256, samples.n_outer)
        n_i = min(512, samples.n_inner)
        if n_o:
            d["step_loss_outer"] = np.float64(_train_batch(
                step_model, "outer", samples.outer_obj[:n_o], samples.outer_coord[:n_o],
                samples.outer_label[:n_o]))
        if n_i:
            d["step_loss_inner"] = np.float64(_train_batch(
                step_model, "inner", samples.inner_obj[:n_i], samples.inner_coord[:n_i],
                samples.inner_label[:n_i]))
        for i, arr in enumerate(model_arrays(step_model)):
            d[f"step_param_{i:03d}"] = np.array(arr)
        curve_model = nt.build_model(cfg, scene)
        d["curve"] = nt.train(curve_model, samples, epochs=2)
        d["curve_model_hash"] = np.frombuffer(
            arrays_hash(list(model_arrays(curve_model))).encode(), np.uint8)
        np.savez_compressed(OUT / f"{name}.npz", **d)
        print(f"{name}: rays {len(rays)} records {len(rec)} outer {om.sum()} inner {im.sum()} "
              f"samples {samples.n_outer}/{samples.n_inner}")

    # default-size model init (seed 0, 2 objects) pinned by hash
    cfg = nt.NifConfig(seed=0)
    m = nt.NifModel(cfg, 2, 1.0)
    np.savez_compressed(OUT / "model_default.npz",
                        hash=np.frombuffer(arrays_hash(list(model_arrays(m))).encode(), np.uint8))


if __name__ == "__main__":
    main()
