"""Small end-to-end exercise of every device path for compute-sanitizer
(tools/gpu_sanitize.sh): ordered + unordered gather, labels, sample
collection, one training epoch (tiled fwd/bwd, per-head per-row kernel,
unit-major Adam), the split data-parallel / deterministic training steps
(exchange buffer, all three grid-scatter modes, ordered MLP reduction),
fused / split / bucketed (per_object) queries, the native engine, device
shading and the GPU SAH build (all three segment classes)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2306_07191_b200 import (BvhBackend, NativeEngine, NifBackend, RenderConfig,  # noqa: E402
                                   build_model, render)
from paper_2306_07191_b200.nif import NifConfig, query_family  # noqa: E402
from paper_2306_07191_b200.pipeline import sample_pass  # noqa: E402
from paper_2306_07191_b200.scene import ShadowRays  # noqa: E402
from paper_2306_07191_b200.synthetic import c1, lattice  # noqa: E402
from paper_2306_07191_b200.train import collect_samples, train  # noqa: E402

torch.cuda.set_device(0)
scene = lattice(3, 2, 0.35, 48, 32)
for sharing in ("shared", "per_object"):
    cfg = NifConfig(seed=0, sharing=sharing)
    cfg.outer.grid_resolution = 32
    cfg.inner.grid_resolution = 16
    model = build_model(cfg, scene)
    smp = collect_samples(scene, spp=1, seed=scene.seed)
    train(model, smp, epochs=1)
    data = sample_pass(scene, scene.camera, 0, scene.seed)
    rays = ShadowRays(data["point"][data["hit"]], data["ldir"][data["hit"]],
                      data["tmax"][data["hit"]])
    occ = NifBackend(model).occluded(scene, rays)
    eng = NativeEngine(scene, model, len(rays))
    assert np.array_equal(eng.occluded(rays, chunks=2), occ)
    eng.close()
    rng = np.random.default_rng(0)
    o = rng.integers(0, scene.n_objects, 300)
    c = rng.random((300, 5))
    for fam, w in (("outer", 4), ("inner", 5)):
        query_family(model, fam, o, c[:, :w])
        if sharing == "shared":
            query_family(model, fam, o, c[:, :w], split=True)
# split steps: the sink with the warp-aggregated, fixed-point and sorted
# scatters (+ ordered MLP partials), eager and graph-replayed
from paper_2306_07191_b200.train import _GraphStep, _Sink, _Step  # noqa: E402
cfg = NifConfig(seed=0)
cfg.outer.grid_resolution = 32
cfg.inner.grid_resolution = 16
cfg.outer.batch_size = 256
cfg.inner.batch_size = 512
model = build_model(cfg, scene)
smp = collect_samples(scene, spp=1, seed=scene.seed)
for which, bs in (("outer", 256), ("inner", 512)):
    n = getattr(smp, f"n_{which}")
    for mode, det in ((0, False), (2, False), (1, True)):
        st = _Step(model, which)
        sink = _Sink(st, bs, 1, 0, None, deterministic=det, scatter_mode=mode)
        for cap in (False, True):
            gs = _GraphStep(st, getattr(smp, f"{which}_obj"), getattr(smp, f"{which}_coord"),
                            getattr(smp, f"{which}_label"), n, bs, sink, capture=cap)
            gs.epoch(np.random.default_rng(mode).permutation(n))
render(c1(32, 24, subdiv=2), config=RenderConfig(spp=1), backend=BvhBackend())
from paper_2306_07191_b200 import meshgen  # noqa: E402
from paper_2306_07191_b200.scene import build_bottoms  # noqa: E402
meshes = [meshgen.mesh_arrays(*meshgen.icosphere(5)), meshgen.mesh_arrays(*meshgen.torus())]
for h, d in zip(build_bottoms(meshes, workers=1), build_bottoms(meshes, device="cuda")):
    assert h.order.tobytes() == d.order.tobytes() and h.node_a.tobytes() == d.node_a.tobytes()
torch.cuda.synchronize()
print("sanitize paths ok")
