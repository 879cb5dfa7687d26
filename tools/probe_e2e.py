"""e2e through the drop-in plugin (NifBackend.occluded -> native engine,
pinned staging ring) on the C2 frame, one configuration per process
(staging knobs are read from NIF_STAGING_THREADS / _NT / _CHUNK at engine
creation). Prints one JSON line: ms per call (median of 20) and rays/s."""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2306_07191_b200 import NifBackend, build_model, synthetic
    from paper_2306_07191_b200.nif import NifConfig
    from paper_2306_07191_b200.pipeline import ShadowRays, sample_pass_dev, shadow_rays_dev
    torch.cuda.set_device(0)
    scene = synthetic.c2(build_device=torch.device("cuda", 0))
    data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
    _, o, d, t = shadow_rays_dev(data, require_emit=False)
    rays = ShadowRays(o.cpu().numpy(), d.cpu().numpy(), t.cpu().numpy())
    model = build_model(NifConfig(seed=0), scene)
    be = NifBackend(model)
    for _ in range(5):
        be.occluded(scene, rays)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        be.occluded(scene, rays)
        ts.append(time.perf_counter() - t0)
    # pure host staging copy bandwidth (numpy, one thread) for reference
    buf = np.empty_like(rays.origins)
    t0 = time.perf_counter()
    for _ in range(5):
        np.copyto(buf, rays.origins)
    np_gbs = 5 * buf.nbytes / (time.perf_counter() - t0) / 1e9
    ms = float(np.median(ts)) * 1e3
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("NIF_STAGING")},
                      "ms": ms, "min_ms": float(np.min(ts)) * 1e3, "rays_per_s": len(rays) / ms * 1e3,
                      "info": be.native_engine(scene, len(rays)).info(),
                      "numpy_copy_1t_gbs": np_gbs, "cpus": os.cpu_count()}))


if __name__ == "__main__":
    main()
