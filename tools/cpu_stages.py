"""Per-stage timing of the reference CPU path (oracle port) beside the GPU
path, at C2 (SURVEY.md 8(d) "Timing the reference CPU path beside it"):
BVH any-hit, gather, encode/forward per family, labels and one training
step per family. CPU: the oracle C port (OpenMP; run once with
OMP_NUM_THREADS=1 and once with all host threads) on a bounded sample,
1 warm-up + median of 3; the training step is the numpy restatement
(single-threaded numpy + BLAS). GPU: the same stages on the full frame,
CUDA events, median of 5. Prints one JSON object.

    OMP_NUM_THREADS=1 python tools/cpu_stages.py > gpurun_out/cpu_stages_t1.json
    python tools/cpu_stages.py > gpurun_out/cpu_stages_all.json
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle  # noqa: E402  (CPU baseline only)
from paper_2306_07191_b200 import _lib, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig, init_arrays  # noqa: E402
from paper_2306_07191_b200.pipeline import VisibilityEngine, gather_dev, sample_pass_dev, shadow_rays_dev  # noqa: E402,E501
from paper_2306_07191_b200.synthetic import c2  # noqa: E402
from paper_2306_07191_b200.train import train_batch  # noqa: E402

N_CPU = int(os.environ.get("CPU_STAGE_RAYS", "20000"))


def med(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def gpu_med(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return float(np.median(ts))


torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
scene = c2(build_device=dev)
model = build_model(NifConfig(seed=0), scene)
data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
_, o, d, t = shadow_rays_dev(data, require_emit=False)
n = int(t.shape[0])
rays_np = [x.cpu().numpy() for x in (o, d, t)]
L = _lib.lib()
res = {"omp_threads": oracle.max_threads(), "cpu_sample_rays": N_CPU, "gpu_rays": n,
       "host_cpus": os.cpu_count(), "stages": {}}

# ---- CPU (oracle port) ------------------------------------------------------
osc = oracle.OracleScene(scene.pack, scene.epsilon_t)
route = scene.nif_route_mask(None)
stride = max(1, n // N_CPU)  # a strided sample: every image region, both families
co, cd, ct = (np.ascontiguousarray(x[::stride][:N_CPU]) for x in rays_np)
cpu = {}
cpu["bvh_anyhit"] = (med(lambda: oracle.bvh_occluded(osc, co, cd, ct)), N_CPU, "rays")
cpu["gather"] = (med(lambda: oracle.gather(osc, co, cd, ct, route)), N_CPU, "rays")
kind, obj, ray, coord, _, _ = oracle.gather(osc, co, cd, ct, route)
grids = model.host_grids()
for fam, k, width in (("outer", 0, 4), ("inner", 1, 5)):
    hl = model.host_layers(fam)[0]
    w = np.concatenate([a.reshape(-1) for a, _ in hl])
    b = np.concatenate([bb for _, bb in hl])
    dims = [hl[0][0].shape[1]] + [a.shape[0] for a, _ in hl]
    pos = np.stack([g[f"{fam}_pos"] for g in grids])
    dirg = np.stack([g[f"{fam}_dir"] for g in grids])
    dist = np.stack([g["inner_dist"] for g in grids]) if fam == "inner" else None
    sel = kind == k
    ob, cc = obj[sel], coord[sel, :width]
    cpu[f"encode_{fam}"] = (med(lambda: oracle.encode(pos, dirg, dist, ob, cc)), int(sel.sum()),
                            "records")
    x = oracle.encode(pos, dirg, dist, ob, cc)
    cpu[f"forward_{fam}"] = (med(lambda: oracle.dense_forward(w, b, dims, x)), int(sel.sum()),
                             "records")
cpu["label"] = (med(lambda: oracle.label_visible(osc, obj, ray, co, cd, ct)), len(obj), "records")
outer_i, inner_i, grids_i, _, _ = init_arrays(NifConfig(seed=0), scene.n_objects)
rng = np.random.default_rng(0)
for fam, bs, width in (("outer", 2 ** 11, 4), ("inner", 2 ** 12, 5)):
    ob = rng.integers(0, scene.n_objects, bs)
    cc = rng.random((bs, width))
    lab = (rng.random(bs) < 0.5).astype(np.float32)
    om = oracle.OModel(outer_i[0], inner_i[0], grids_i)
    cpu[f"train_step_{fam}"] = (med(lambda: om.train_batch(fam, ob, cc, lab), reps=3), 1,
                                "optimiser steps")

# ---- GPU (this package) -----------------------------------------------------
eng = VisibilityEngine(scene, model, n)
eng.origins[:n].copy_(o)
eng.dirs[:n].copy_(d)
eng.tmaxs[:n].copy_(t)
eng.run_range(0, n)
torch.cuda.synchronize()
b = eng.buf
counts = eng.counts()
vo, vi = eng._family_views()
sp = _lib.stream_ptr()
gpu = {}
gpu["gather"] = (gpu_med(lambda: gather_dev(eng.ds, eng.route, eng.origins, eng.dirs, eng.tmaxs,
                                            n, b)), n, "rays")
gpu["query_outer"] = (gpu_med(lambda: L.nif_query_dev(
    vo, b.outer_obj.data_ptr(), b.outer_ray.data_ptr(), b.outer_coord.data_ptr(), None,
    b.counts.data_ptr(), b.cap, eng.occ.data_ptr(), None, 0, sp)), int(counts[0]), "records")
gpu["query_inner"] = (gpu_med(lambda: L.nif_query_dev(
    vi, b.inner_obj.data_ptr(), b.inner_ray.data_ptr(), b.inner_coord.data_ptr(),
    b.inner_r.data_ptr(), b.counts.data_ptr() + 8, b.cap, eng.occ.data_ptr(), None, 0, sp)),
    int(counts[1]), "records")
bvh_out = torch.empty(n, dtype=torch.uint8, device=dev)
gpu["bvh_anyhit"] = (gpu_med(lambda: L.nif_bvh_occluded_dev(
    eng.ds.view, o.data_ptr(), d.data_ptr(), t.data_ptr(), n, bvh_out.data_ptr(), sp)), n, "rays")
for fam, bs, width in (("outer", 2 ** 11, 4), ("inner", 2 ** 12, 5)):
    ob = rng.integers(0, scene.n_objects, bs)
    cc = rng.random((bs, width))
    lab = (rng.random(bs) < 0.5).astype(np.float32)
    # eager host-array step (uploads + one sync included: a conservative GPU figure)
    t_step = med(lambda: train_batch(model, fam, ob, cc, lab), reps=5)
    gpu[f"train_step_{fam}"] = (t_step, 1, "optimiser steps (eager, host arrays)")

for k, (sec, units, unit) in cpu.items():
    res["stages"].setdefault(k, {})["cpu"] = {"s": sec, "units": units, "unit": unit,
                                              "per_s": units / sec}
for k, (sec, units, unit) in gpu.items():
    res["stages"].setdefault(k, {})["gpu"] = {"s": sec, "units": units, "unit": unit,
                                              "per_s": units / sec}
print(json.dumps(res))
