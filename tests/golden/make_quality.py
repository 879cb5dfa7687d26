"""Reference quality numbers at the C1 configuration (run here, where the
reference is importable; writes tests/golden/quality_c1.json):

scene   icosphere(5, r=0.9) at z = 0.9 + BVH-routed ground plane, 256x256,
        point light (2.2, -1.6, 2.8) I = 28, seed 11
train   collect_samples(spp=8) + train(epochs=10), NifConfig(seed=0)
eval    render 4 spp with NifBackend vs BvhBackend -> PSNR; thresholded
        agreement with the BVH labels on the spp-0 shadow-ray records.
"""

import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import niftrace as nt  # noqa: E402
from niftrace import meshgen  # noqa: E402
from niftrace.bvh import build_bottom  # noqa: E402
from niftrace.cli import _bench_shadow_rays  # noqa: E402
from niftrace.nif import _label_occlusion, infer_records  # noqa: E402
from niftrace.renderer import gather_queries  # noqa: E402


def c1_scene(w=256, h=256):
    v0, v1, v2, n0, n1, n2 = meshgen.mesh_arrays(*meshgen.icosphere(5, 0.9))
    t = np.array([0.0, 0.0, 0.9])
    sphere = build_bottom((v0 * 1.0 + t, v1 * 1.0 + t, v2 * 1.0 + t, n0, n1, n2))
    plane = build_bottom(meshgen.mesh_arrays(*meshgen.ground_plane(4.0)))
    cam = nt.Camera(np.array([0.0, -3.4, 1.7]), np.array([0.0, 0.0, 0.45]),
                    np.array([0.0, 0.0, 1.0]), 38.0, w, h)
    return nt.Scene([nt.SceneObject("sphere", sphere, np.array([0.75, 0.33, 0.27])),
                     nt.SceneObject("plane", plane, np.array([0.62, 0.62, 0.6]), False)],
                    [nt.PointLight(np.array([2.2, -1.6, 2.8]), np.array([28.0, 28.0, 28.0]))],
                    cam, 11)


def main():
    scene = c1_scene()
    cfg = nt.NifConfig(seed=0)
    model = nt.build_model(cfg, scene)
    t0 = time.perf_counter()
    samples = nt.collect_samples(scene, spp=8, seed=scene.seed)
    curve = nt.train(model, samples, epochs=10)
    t_train = time.perf_counter() - t0
    ref = nt.render(scene, config=nt.RenderConfig(spp=4), backend=nt.BvhBackend())
    img = nt.render(scene, config=nt.RenderConfig(spp=4), backend=nt.NifBackend(model))
    p = nt.psnr(img, ref)
    rays = _bench_shadow_rays(scene, 1, 8)
    rec, _ = gather_queries(scene, rays, scene.nif_route_mask(None), 8)
    labels = _label_occlusion(scene, rec, rays, 8)
    bits = infer_records(model, rec)
    agree = float(np.mean(bits == (labels == 0)))
    out = {"psnr_nif_vs_bvh_db": p, "agreement": agree, "records": int(len(rec)),
           "n_outer_samples": samples.n_outer, "n_inner_samples": samples.n_inner,
           "curve": curve.tolist(), "train_seconds_cpu": t_train}
    (Path(__file__).resolve().parent / "quality_c1.json").write_text(json.dumps(out, indent=1))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
