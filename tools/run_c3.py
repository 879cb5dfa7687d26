"""BASELINE.json configs[2]: synthetic 31.46M-triangle
scene (24 x icosphere(8) + plane) at 1920x1080, online training from
`--spp` samples per pixel on the device, then NIF vs CUDA-BVH any-hit
ms/frame and quality against the BVH ground truth.

    python tools/run_c3.py [--spp 64] [--epochs 30] [--render-spp 4] [--out f.json]

Everything runs on cuda:0: the sample pass, the ordered gather, the
bit-exact BVH labels, the reference's epoch schedule (train.train), the
graph-captured visibility pass and the BVH comparator on the same rays.
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2306_07191_b200 import BvhBackend, NifBackend, RenderConfig, _lib, build_model, psnr, render  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.pipeline import VisibilityEngine, sample_pass_dev, shadow_rays_dev  # noqa: E402
from paper_2306_07191_b200.synthetic import c3  # noqa: E402
from paper_2306_07191_b200.train import collect_samples, train  # noqa: E402


def ev_time(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spp", type=int, default=64)
    ap.add_argument("--epochs", type=int, default=30)
    ap.add_argument("--render-spp", type=int, default=4)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    res = {"config": "C3: 24 x icosphere(8) + NIF plane, 1920x1080, point light",
           "spp_train": a.spp, "epochs": a.epochs}
    t0 = time.perf_counter()
    scene = c3(a.width, a.height, build_device=torch.device("cuda", 0))
    ds = scene.device()
    res["triangles"] = int(sum(o.n_triangles for o in scene.objects))
    res["build_s"] = time.perf_counter() - t0

    model = build_model(NifConfig(seed=0), scene)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    samples = collect_samples(scene, spp=a.spp, seed=scene.seed)
    torch.cuda.synchronize()
    res["collect_s"] = time.perf_counter() - t0
    res["samples_outer"], res["samples_inner"] = samples.n_outer, samples.n_inner
    steps_per_epoch = (-(-samples.n_outer // model.config.outer.batch_size)
                       - (-samples.n_inner // model.config.inner.batch_size))
    t0 = time.perf_counter()
    curve = train(model, samples, epochs=a.epochs)
    torch.cuda.synchronize()
    res["train_s"] = time.perf_counter() - t0
    res["optimizer_steps"] = steps_per_epoch * a.epochs
    res["optimizer_steps_per_s"] = res["optimizer_steps"] / res["train_s"]
    res["train_samples_per_s"] = (samples.n_outer + samples.n_inner) * a.epochs / res["train_s"]
    res["loss_curve"] = curve.tolist()
    del samples
    torch.cuda.empty_cache()

    # visibility pass vs BVH any-hit on one 1-spp frame of shadow rays
    data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
    _, o, d, t = shadow_rays_dev(data, require_emit=False)
    n = int(t.numel())
    eng = VisibilityEngine(scene, model, n)
    eng.origins[:n].copy_(o)
    eng.dirs[:n].copy_(d)
    eng.tmaxs[:n].copy_(t)
    g = eng.capture(n)
    res["rays_per_frame"] = n
    res["nif_ms_per_frame"] = ev_time(g.replay)
    bvh = torch.empty(n, dtype=torch.uint8, device=o.device)
    L = _lib.lib()
    res["bvh_ms_per_frame"] = ev_time(lambda: L.nif_bvh_occluded_dev(
        ds.view, o.data_ptr(), d.data_ptr(), t.data_ptr(), n, bvh.data_ptr(), _lib.stream_ptr()))
    g.replay()
    torch.cuda.synchronize()
    nif = eng.occ[:n].clone()
    res["ray_agreement_vs_bvh"] = float((nif == bvh).float().mean())
    res["counts"] = [int(x) for x in eng.counts()[:3]]

    # rendered image quality (shading from the same sample pass) vs BVH
    cfg = RenderConfig(spp=a.render_spp)
    ref = render(scene, config=cfg, backend=BvhBackend())
    img = render(scene, config=cfg, backend=NifBackend(model))
    res["psnr_nif_vs_bvh_db"] = float(psnr(img, ref))
    print(json.dumps(res))
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
