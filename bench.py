"""NIF shadow-ray visibility benchmark (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--config c1|c2|c3|c4]

Workload (BASELINE.json configs[1], the default at N=1):
synthetic multi-object scene, 12 x icosphere(6) + NIF-enabled ground plane
= 983,042 triangles in 13 objects, 1920x1080, 1 spp direct-illumination
shadow rays, inference only. One step = one NIF visibility pass over the
frame's shadow rays: phase-1 gather (top-level culling + fp64 T_outer /
T_inner) -> fused grid encoding + visibility MLP (tcgen05) -> p < 0.5 ->
per-ray OR. Rays are generated on the GPU by the sample pass (not timed).

Multi-GPU (torchrun, one process per GPU): ONE frame
cut into 32N row strips dealt round-robin to the ranks
(parallel.rank_strips; contiguous bands left the top ranks with the ray-less
sky: tools/band_balance.py); rank r generates its strips' shadow rays and
resolves them in one pass -- no collective on the data path (strong
scaling, total work = one frame). Default config under torchrun:
C4 = the C2 scene at 3840x2160 (5.2M shadow rays), so per-GPU shares stay
large at 8 GPUs; --config c2 splits the 1080p frame instead.

value : shadow rays of the frame resolved per second (all ranks), rays
        resident in HBM, L2 flushed (256 MiB write) between steps, CUDA
        events on the launching stream, max over ranks.
e2e   : the same metric through the drop-in plugin NifBackend.occluded
        (renderer.py:675-683) on pageable numpy rays -> bool[n]: the native
        engine's C-ABI, staging through its pinned ring, H2D of the rays and
        D2H of the answer every step; host clock around each synchronous
        call, max over ranks.
--impl reference: the reference CPU path restated in oracle/ (scene build,
        seeded init, gather + encode + row-sequential MLP + OR) on the same
        frame, host cores only; the B200 package is never imported.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "NIF shadow-ray queries/s per GPU; secondary-ray cast ms/frame vs BVH"
UNIT = "shadow rays/s"
WORKLOAD = ("C2: 12x icosphere(6) + NIF plane, 983,042 tris, 13 objects, 1920x1080, "
            "1 spp point-light shadow rays, inference only")
WORKLOADS = {
    "c1": "C1: icosphere(5) + BVH-routed plane, 20,480 NIF tris, 256x256, 1 spp shadow rays",
    "c2": WORKLOAD,
    "c3": ("C3: 24x icosphere(8) + NIF plane, 31,457,282 tris, 25 objects, 1920x1080, "
           "1 spp point-light shadow rays, inference"),
    "c4": ("C4: C2 scene (12x icosphere(6) + NIF plane, 983,042 tris) at 3840x2160, "
           "1 spp point-light shadow rays, inference, frame split in row strips across GPUs"),
}
RESOLUTION = {"c1": (256, 256), "c2": (1920, 1080), "c3": (1920, 1080), "c4": (3840, 2160)}
# kernels of one visibility pass (names as ncu reports them) and their
# algorithmic work: see DESIGN.md section 4
STRIPS_PER_RANK = 32  # row strips per rank when a frame is split across GPUs
K_GATHER = "gather_warp_kernel"
K_OUTER = "query_ts_kernel<3, 0, 64, 2, 2, 4, 0, 1, 0>"
K_INNER = "query_ts_kernel<5, 3, 48, 3, 1, 4, 0, 1, 1>"


def workload_label(args):
    """The workload string of the configuration actually run (resolution
    overrides included)."""
    base = WORKLOADS[args.config]
    w0, h0 = RESOLUTION[args.config]
    if (args.width, args.height) != (w0, h0):
        base = base.replace(f"{w0}x{h0}", f"{args.width}x{args.height}")
    return base


def config_of(args, ws, n_frame, counts):
    """The `config` object: identical on both arms for the same run."""
    return {"workload": workload_label(args), "rays_per_frame": int(n_frame),
            "outer_records": int(counts[0]), "inner_records": int(counts[1]),
            "model": f"NifConfig() defaults (R 256/128, seed 0, random init), "
                     f"sharing={args.sharing}",
            "trained_epochs": args.train_epochs,
            "parallelism": (f"one frame cut in {ws * STRIPS_PER_RANK} row strips dealt "
                            f"round-robin to {ws} GPUs" if ws > 1 else "one frame, one GPU")}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default=None, choices=["c1", "c2", "c3", "c4"],
                   help="default: c2 on one GPU, c4 (4K frame in row strips) under torchrun")
    p.add_argument("--width", type=int, default=None)
    p.add_argument("--height", type=int, default=None)
    p.add_argument("--train-epochs", type=int, default=0,
                   help="epochs of GPU training on 1 spp before timing (0 = random init)")
    p.add_argument("--sharing", default="shared", choices=["shared", "per_object"],
                   help="NifConfig.sharing (per_object: one MLP per object, bucketed query)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-train-leg", action="store_true",
                   help="skip the online-training epoch measured after the visibility pass")
    p.add_argument("--e2e-chunks", type=int, default=4,
                   help="chunks of the e2e host path (H2D of chunk k+1 overlaps chunk k)")
    p.add_argument("--profile", action="store_true", help="few steps, no clocks / cpu leg")
    args = p.parse_args()
    if args.config is None:
        args.config = "c2" if int(os.environ.get("WORLD_SIZE", "1")) == 1 else "c4"
    w0, h0 = RESOLUTION[args.config]
    args.width = w0 if args.width is None else args.width
    args.height = h0 if args.height is None else args.height
    return args


def dist_setup(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" else "gloo"
        # NIF_BENCH_BACKEND=gloo + NIF_BENCH_ONE_GPU=1: every rank on cuda:0 (a
        # smoke test of the N>1 code path on a one-GPU box; not a measurement)
        backend = os.environ.get("NIF_BENCH_BACKEND", backend)
        if args.impl == "ours":
            torch.cuda.set_device(0 if os.environ.get("NIF_BENCH_ONE_GPU") else local)
        dist.init_process_group(backend)
    elif args.impl == "ours":
        torch.cuda.set_device(0)
    return rank, ws, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def build_workload(args, rank, build_device=None):
    from paper_2306_07191_b200 import synthetic
    if args.config == "c1":
        return synthetic.c1(min(args.width, 256), min(args.height, 256))
    # scene setup (untimed); build_device: per-object SAH builds on the GPU
    # (identical trees) -- the reference arm keeps the host builder
    if args.config == "c3":
        return synthetic.c3(args.width, args.height, build_device=build_device)
    return synthetic.c2(args.width, args.height, build_device=build_device)  # c2, c4


def cpu_path_step(scene, model, rays_np, n):
    """One step of the reference CPU path (oracle port) over the first n
    rays: gather + encode + row-sequential forward + per-ray OR."""
    from oracle import oracle
    o, d, t = (np.ascontiguousarray(a[:n]) for a in rays_np)
    osc = oracle.OracleScene(scene.pack, scene.epsilon_t)
    route = scene.nif_route_mask(None)
    grids = model.host_grids()
    fams = {}
    for fam in ("outer", "inner"):
        hl = model.host_layers(fam)[0]
        fams[fam] = dict(
            w=np.concatenate([a.reshape(-1) for a, _ in hl]),
            b=np.concatenate([bb for _, bb in hl]),
            dims=[hl[0][0].shape[1]] + [a.shape[0] for a, _ in hl],
            pos=np.stack([g[f"{fam}_pos"] for g in grids]),
            dir=np.stack([g[f"{fam}_dir"] for g in grids]),
            dist=np.stack([g["inner_dist"] for g in grids]) if fam == "inner" else None)

    def one():
        kind, obj, ray, coord, bvh_occ, _ = oracle.gather(osc, o, d, t, route)
        occ = bvh_occ.copy()
        for fam, k, width in (("outer", 0, 4), ("inner", 1, 5)):
            sel = kind == k
            if sel.any():
                f = fams[fam]
                x = oracle.encode(f["pos"], f["dir"], f["dist"], obj[sel], coord[sel, :width])
                p = oracle.dense_forward(f["w"], f["b"], f["dims"], x)
                occ[ray[sel][p[:, 0] < 0.5]] = True
        return occ

    return one


def cpu_baseline_leg(scene, model, rays_np, config, budget_s=20.0):
    """Oracle port of the reference CPU path on the whole frame, all host
    threads (cmd_bench method: 1 warm-up + median of up to 5 within the
    budget)."""
    from oracle import oracle
    n = len(rays_np[0])
    one = cpu_path_step(scene, model, rays_np, n)
    one()
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < 5 and (time.perf_counter() < t_end or len(times) < 1):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    med = float(np.median(times))
    return {"value": n / med, "unit": UNIT, "cores": oracle.max_threads(), "kind": "port",
            "sample": f"the whole {config.upper()} frame ({n} shadow rays): gather + encode + "
                      f"row-sequential MLP + per-ray OR, median of {len(times)}"}


def run_reference(args, rank, ws):
    """--impl reference: the reference's CPU path on the host cores, built
    and run from oracle/ alone (oracle.refscene restates the scene build --
    meshgen, _build_sah, pack -- and the seeded init; nif_oracle.c the
    gather / encode / dense forward), on this run's whole frame. The Python
    reference itself cannot travel to the GPU box. Under torchrun rank 0
    alone runs and prints; the other ranks exit without work."""
    if rank != 0:
        return
    # every host thread: torchrun starts its workers with OMP_NUM_THREADS=1,
    # which the OpenMP runtime has already read
    from oracle import oracle, refscene
    oracle.set_threads(len(os.sched_getaffinity(0)))
    if args.config == "c1":
        scene = refscene.c1(args.width, args.height)
    elif args.config == "c3":
        scene = refscene.lattice(24, 8, 0.3, args.width, args.height, cols=6)
    else:
        scene = refscene.lattice(12, 6, 0.35, args.width, args.height)
    if args.sharing != "shared" or args.train_epochs:
        print(json.dumps({"impl": "reference", "unavailable":
                          "reference arm restates the shared, untrained default model only"}))
        return
    rays = scene.shadow_rays(0)
    n = len(rays[2])
    o_heads, i_heads, grids = refscene.init_model(scene.n_objects, seed=0)
    fams = {"outer": refscene.family_arrays(o_heads, grids, "outer"),
            "inner": refscene.family_arrays(i_heads, grids, "inner")}
    osc = oracle.OracleScene(scene.pack, scene.epsilon_t)
    kind = oracle.gather(osc, *rays, scene.nif_route_mask(None))[0]
    counts = (int((kind == 0).sum()), int((kind == 1).sum()))
    for _ in range(args.warmup):
        refscene.visibility_pass(scene, fams, rays)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        refscene.visibility_pass(scene, fams, rays)
        times.append(time.perf_counter() - t0)
    per = float(np.sum(times)) / args.steps
    value = n / per
    base = {"value": value, "unit": UNIT, "cores": oracle.max_threads(), "kind": "port",
            "sample": f"the whole frame per step ({n} shadow rays): gather + encode + "
                      "row-sequential MLP + per-ray OR, all host threads (OpenMP)"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": config_of(args, ws, n, counts),
            "cpu_baseline": base,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    args = parse()
    rank, ws, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, rank, ws)
        return
    import torch
    from paper_2306_07191_b200 import NifBackend, _lib, build_model
    from paper_2306_07191_b200.nif import NifConfig
    from paper_2306_07191_b200.pipeline import (VisibilityEngine, sample_pass_dev,
                                                shadow_rays_dev)
    dev = torch.device("cuda", torch.cuda.current_device())
    scene = build_workload(args, rank, build_device=dev)
    # this rank's row strips of the frame (the whole frame at N=1); the sample
    # pass keys its RNG by the global pixel index, so the strips' rays are
    # exactly the single-GPU frame's
    from paper_2306_07191_b200.parallel import rank_strips
    parts = []
    for pix0, n_pix in rank_strips(scene.camera.width, scene.camera.height, rank, ws,
                                   STRIPS_PER_RANK if ws > 1 else 1):
        data = sample_pass_dev(scene, scene.camera, 0, scene.seed, "importance", pix0, n_pix)
        parts.append(shadow_rays_dev(data, require_emit=False)[1:])
        del data
    o, d, t = (torch.cat([p_[k] for p_ in parts]) for k in range(3))
    del parts
    n = int(t.numel())
    model = build_model(NifConfig(seed=0, sharing=args.sharing), scene)
    if args.train_epochs > 0:
        import importlib
        tr = importlib.import_module("paper_2306_07191_b200.train")
        samples = tr.collect_samples_dev(scene, spp=1, seed=scene.seed)
        tr.train(model, samples, epochs=args.train_epochs)
    eng = VisibilityEngine(scene, model, n)
    eng.origins[:n].copy_(o)
    eng.dirs[:n].copy_(d)
    eng.tmaxs[:n].copy_(t)
    graph = eng.capture(n)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # --- device-resident timed loop -----------------------------------------
    for _ in range(args.warmup):
        graph.replay()
    barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    clocks = ClockSampler(local)
    with clocks:
        # the timed region of one frame is a few ms, shorter than nvidia-smi's
        # sampling period: keep the same work running for ~1 s first (untimed)
        # so the clock samples see the GPU under this load
        t_soak = time.perf_counter() + (0.0 if args.profile else 1.0)
        while time.perf_counter() < t_soak:
            for _ in range(20):
                flush.fill_(1.0)
                graph.replay()
            torch.cuda.synchronize()
        barrier()
        # gate the stream behind a sleep on a side stream while all K steps
        # are queued, so host jitter (the clock sampler, the OS) can never
        # leave the GPU idle inside a timed step
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            torch.cuda._sleep(int(50e6))  # ~25 ms at 1.9 GHz
        gate = torch.cuda.Event()
        gate.record(side)
        stream.wait_event(gate)
        for e0, e1 in evs:
            flush.fill_(1.0)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
        barrier()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    ms_local = float(np.sum(step_ms))
    counts = eng.counts()

    # --- per-kernel breakdown (eager, events on the launching stream) -------
    L = _lib.lib()
    b = eng.buf
    vo, vi = eng._family_views()
    kt = {}
    reps = max(3, min(args.steps, 10))

    def timed(name, fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        acc = 0.0
        for _ in range(reps):
            flush.fill_(1.0)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            acc += e0.elapsed_time(e1)
        kt[name] = acc / reps

    from paper_2306_07191_b200.pipeline import gather_dev
    sp = _lib.stream_ptr()
    timed("gather", lambda: gather_dev(eng.ds, eng.route, eng.origins, eng.dirs, eng.tmaxs, n, b))
    if eng.bucket is not None:  # per_object: the bucketed tensor-core query, as in the frame
        timed("query_outer", lambda: L.nif_query_bucketed_dev(
            vo, b.outer_obj.data_ptr(), b.outer_ray.data_ptr(), b.outer_coord.data_ptr(), None,
            b.counts.data_ptr(), b.cap, eng.occ.data_ptr(), None, eng.bucket[0].data_ptr(), sp))
        timed("query_inner", lambda: L.nif_query_bucketed_dev(
            vi, b.inner_obj.data_ptr(), b.inner_ray.data_ptr(), b.inner_coord.data_ptr(),
            b.inner_r.data_ptr(), b.counts.data_ptr() + 8, b.cap, eng.occ.data_ptr(), None,
            eng.bucket[1].data_ptr(), sp))
    else:
        timed("query_outer", lambda: L.nif_query_dev(
            vo, b.outer_obj.data_ptr(), b.outer_ray.data_ptr(), b.outer_coord.data_ptr(), None,
            b.counts.data_ptr(), b.cap, eng.occ.data_ptr(), None, 0, sp))
        timed("query_inner", lambda: L.nif_query_dev(
            vi, b.inner_obj.data_ptr(), b.inner_ray.data_ptr(), b.inner_coord.data_ptr(),
            b.inner_r.data_ptr(), b.counts.data_ptr() + 8, b.cap, eng.occ.data_ptr(), None, 0, sp))
    bvh_out = torch.empty(n, dtype=torch.uint8, device=dev)
    timed("bvh_anyhit", lambda: L.nif_bvh_occluded_dev(
        eng.ds.view, o.data_ptr(), d.data_ptr(), t.data_ptr(), n, bvh_out.data_ptr(), sp))

    # --- full frame of the renderer (sample pass -> cast -> visibility ->
    # shading), everything resident, NIF vs BVH visibility (informational)
    from paper_2306_07191_b200 import BvhBackend
    from paper_2306_07191_b200.pipeline import render_dev
    nif_be = NifBackend(model)
    render_ms = {}
    for name, be in ((("nif", nif_be), ("bvh", BvhBackend())) if ws == 1 else ()):
        for _ in range(2):
            render_dev(scene, be, spp=1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            render_dev(scene, be, spp=1)
        e1.record(stream)
        e1.synchronize()
        render_ms[name] = e0.elapsed_time(e1) / 5
    del nif_be

    # the e2e roofline: pinned host -> device copy bandwidth of this box,
    # measured before the plugin's staging threads exist (they are
    # spinning copy workers; measured after them the copy reads ~half),
    # measured on the same stream with one copy of a step's input bytes
    h2d_src = torch.empty(n * 56, dtype=torch.uint8).pin_memory()
    h2d_dst = torch.empty(n * 56, dtype=torch.uint8, device=dev)
    for _ in range(2):
        h2d_dst.copy_(h2d_src, non_blocking=True)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h2d_gbs = 0.0
    for _ in range(8):  # best of eight trials of five copies (the link is noisy)
        c0.record(stream)
        for _ in range(5):
            h2d_dst.copy_(h2d_src, non_blocking=True)
        c1.record(stream)
        c1.synchronize()
        h2d_gbs = max(h2d_gbs, n * 56 * 5 / (c0.elapsed_time(c1) / 1e3) / 1e9)
    del h2d_src, h2d_dst

    # --- e2e through the drop-in plugin: NifBackend.occluded (the reference's
    # PredictorBackend.occluded, renderer.py:675-683) on pageable numpy rays,
    # answered through the native engine's C-ABI (pinned staging ring,
    # upload / staging copy / device pass of neighbouring chunks overlapped);
    # synchronous host call, timed on the host clock around each call
    from paper_2306_07191_b200.pipeline import ShadowRays
    rays_host = ShadowRays(o.cpu().numpy(), d.cpu().numpy(), t.cpu().numpy())
    plugin = NifBackend(model)
    want = eng.occ[:n].cpu().numpy().astype(bool)
    got = plugin.occluded(scene, rays_host)
    e2e_parity = bool(np.array_equal(got, want))
    for _ in range(args.warmup):
        plugin.occluded(scene, rays_host)
    barrier()
    e2e_s = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plugin.occluded(scene, rays_host)
        e2e_s.append(time.perf_counter() - t0)
    barrier()
    e2e_ms_local = float(np.sum(e2e_s)) * 1e3
    staging = plugin.native_engine(scene, n).info()

    # the same on pinned torch tensors through VisibilityEngine.occluded_host
    # (the bound the staging ring is measured against)
    ho = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    hd = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    ht = torch.empty(n, dtype=torch.float64).pin_memory()
    ho.copy_(o)
    hd.copy_(d)
    ht.copy_(t)
    hocc = torch.empty(n, dtype=torch.uint8).pin_memory()
    for _ in range(args.warmup):
        eng.occluded_host(ho, hd, ht, hocc, n, chunks=args.e2e_chunks)
    torch.cuda.synchronize()
    p_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)]
    for e0, e1 in p_evs:
        flush.fill_(1.0)
        e0.record(stream)
        eng.occluded_host(ho, hd, ht, hocc, n, chunks=args.e2e_chunks)
        e1.record(stream)
    torch.cuda.synchronize()
    pinned_ms = float(np.sum([e0.elapsed_time(e1) for e0, e1 in p_evs]))

    # --- the C4 frame (3840x2160, the same scene) on this one GPU: the N=1
    # point of the multi-GPU curve, whose N>1 runs split this frame in row strips
    c4_single = None
    if ws == 1 and args.config == "c2" and not args.profile:
        import dataclasses
        cam4 = dataclasses.replace(scene.camera, width=3840, height=2160)
        d4 = sample_pass_dev(scene, cam4, 0, scene.seed)
        _, o4, dd4, t4 = shadow_rays_dev(d4, require_emit=False)
        n4 = int(t4.numel())
        del d4
        eng4 = VisibilityEngine(scene, model, n4)
        eng4.origins[:n4].copy_(o4)
        eng4.dirs[:n4].copy_(dd4)
        eng4.tmaxs[:n4].copy_(t4)
        g4 = eng4.capture(n4)
        for _ in range(args.warmup):
            g4.replay()
        torch.cuda.synchronize()
        ev4 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for e0, e1 in ev4:
            flush.fill_(1.0)
            e0.record(stream)
            g4.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        ms4 = float(np.mean([e0.elapsed_time(e1) for e0, e1 in ev4]))
        c4_single = {"workload": WORKLOADS["c4"].replace(", frame split in row strips across GPUs",
                                                         ", one GPU"),
                     "rays_per_frame": n4, "frame_ms": ms4, "value": n4 / (ms4 / 1e3),
                     "unit": UNIT, "note": "N=1 point of the C4 curve (bench.py under torchrun "
                                           "splits this frame in 32N row strips)"}
        del eng4, g4, o4, dd4, t4

    # --- online training: one spp of samples collected
    # band-sharded across the ranks (ordered all-gather into the reference's
    # global order), then one epoch of the reference schedule; under torchrun
    # every optimiser step is the data-parallel step -- one all-reduce of
    # [batch input gradients | MLP gradients], captured in the step's CUDA
    # graph. Host clock around the synchronous train() call, max over ranks.
    train_leg = None
    if not args.no_train_leg and not args.profile:
        import importlib
        tr = importlib.import_module("paper_2306_07191_b200.train")
        smp = tr.collect_samples(scene, spp=1, seed=scene.seed)
        tm = build_model(NifConfig(seed=0, sharing=args.sharing), scene)
        tr.train(tm, smp, epochs=1)  # warm: graph capture, communicators
        barrier()
        t0 = time.perf_counter()
        curve = tr.train(tm, smp, epochs=1)
        barrier()
        ep_s = time.perf_counter() - t0
        if ws > 1:
            te = torch.tensor([ep_s], device=dev)
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
            ep_s = float(te[0])
        cfgt = tm.config
        n_steps = -(-smp.n_outer // cfgt.outer.batch_size) - (-smp.n_inner // cfgt.inner.batch_size)
        train_leg = {"epoch_ms": ep_s * 1e3, "optimizer_steps": int(n_steps),
                     "steps_per_s": n_steps / ep_s, "samples": smp.n_outer + smp.n_inner,
                     "spp": 1, "loss": float(curve[-1, 2]),
                     "mode": (f"data parallel over {ws} GPUs: one "
                              f"{torch.distributed.get_backend()} all-reduce per step "
                              + ("inside the step graph" if torch.distributed.get_backend() == "nccl"
                                 else "(eager)") + ", fixed-point grid scatter")
                     if ws > 1 else "single GPU: captured 3-launch step per batch"}
        del tm, smp

    # --- reduce over ranks (max time) ---------------------------------------
    ms, e2e_ms = ms_local, e2e_ms_local
    n_total = n
    frame_counts = [int(counts[0]), int(counts[1])]
    band_ms = [ms_local / args.steps]
    if ws > 1:
        tt = torch.tensor([ms_local, e2e_ms_local], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms, e2e_ms = float(tt[0]), float(tt[1])
        nn = torch.tensor([n, int(counts[0]), int(counts[1])], device=dev, dtype=torch.int64)
        torch.distributed.all_reduce(nn)
        n_total = int(nn[0])
        frame_counts = [int(nn[1]), int(nn[2])]
        per = torch.zeros(ws, device=dev, dtype=torch.float64)
        per[rank] = ms_local / args.steps
        torch.distributed.all_reduce(per)
        band_ms = per.cpu().tolist()
    if rank != 0:
        return
    value = n_total * args.steps / (ms / 1e3)
    e2e_value = n_total * args.steps / (e2e_ms / 1e3)

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
    n_outer, n_inner = int(counts[0]), int(counts[1])
    cfgm = model.config
    fl_o = 2 * (cfgm.outer.input_dim * cfgm.outer.hidden_width
                + (cfgm.outer.hidden_layers - 1) * cfgm.outer.hidden_width ** 2
                + cfgm.outer.hidden_width)
    fl_i = 2 * (cfgm.inner.input_dim * cfgm.inner.hidden_width
                + (cfgm.inner.hidden_layers - 1) * cfgm.inner.hidden_width ** 2
                + cfgm.inner.hidden_width)
    # algorithmic bytes of one gather launch: rays in (origins, dirs, tmaxs
    # f64 = 56 B), bvh_occ out (1 B), records out (outer obj+ray+coord4 = 24 B,
    # inner + r = 28 B); algorithmic FLOPs of the MLPs (useful MACs only)
    gather_bytes = 56 * n + 1 * n + 24 * n_outer + 28 * n_inner
    tr = {}
    tj = ROOT / "profiles" / "traffic.json"
    if tj.exists():
        tr = json.loads(tj.read_text())

    def roof_of(k):
        if k == "gather":
            r = {"bound": "hbm", "kernel": f"{K_GATHER} (classify + unordered compaction)",
                 "achieved": gather_bytes / (kt["gather"] / 1e3) / 1e9,
                 "peak": peaks["hbm_gbs"], "unit": "GB/s", "work_per_launch_bytes": gather_bytes}
            key = K_GATHER
        else:
            nrec = n_outer if k == "query_outer" else n_inner
            fl = fl_o if k == "query_outer" else fl_i
            key = K_OUTER if k == "query_outer" else K_INNER
            r = {"bound": "tensor", "kernel": f"{key} (fused encode + MLP, {k})",
                 "achieved": nrec * fl / (kt[k] / 1e3) / 1e12,
                 "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                 "work_per_launch_flop": nrec * fl}
        r["frac"] = r["achieved"] / r["peak"]
        r["traffic"] = None
        if key in tr:
            r["traffic"] = tr[key]["dram_bytes_read"] + tr[key]["dram_bytes_write"]
            r["traffic_source"] = tr["_source"]
        r["peak_source"] = "MEASURED_PEAKS.json (burst)"
        return r

    dominant = max(("gather", "query_outer", "query_inner"), key=lambda k: kt[k])
    roof = roof_of(dominant)
    rooflines = {k: roof_of(k) for k in ("gather", "query_outer", "query_inner")}

    cpu = None
    if not args.no_cpu_baseline and not args.profile and ws == 1:
        try:
            rays_np = (rays_host.origins, rays_host.dirs, rays_host.tmaxs)
            cpu = cpu_baseline_leg(scene, model, rays_np, args.config)
        except Exception as e:  # the checker must never hide the main number
            cpu = {"value": None, "error": str(e)[:200]}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp16-mma/fp32-acc (fp64 gather)",
        "data": "synthetic",
        "config": config_of(args, ws, n_total, frame_counts),
        "l2": "flushed (256 MiB write) between steps",
        "frame_ms": ms / args.steps,
        "band_ms_per_rank": band_ms,
        # SURVEY 8(d) metric (i) also asks for (ray, object) records per second
        "records_per_s": sum(frame_counts) * args.steps / (ms / 1e3),
        "bvh_ms_per_frame": kt["bvh_anyhit"],
        "render_ms_per_frame_1spp": render_ms,
        "kernel_ms": kt,
        "roofline": roof,
        "rooflines": rooflines,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": int(n_total * 56), "d2h_bytes_per_step": int(n_total),
                "api": "NifBackend.occluded(scene, ShadowRays of numpy f64 arrays) -> bool[n] "
                       "(native engine, C-ABI nif_engine_occluded_host)",
                "parity_with_device_path": e2e_parity,
                "staging": staging,
                # bound: the host -> device link (the pass itself is ~10x faster)
                "h2d_achieved_gbs": n * 56 * args.steps / (e2e_ms / 1e3) / 1e9,
                "h2d_peak_gbs": h2d_gbs,
                "h2d_frac": (n * 56 * args.steps / (e2e_ms / 1e3) / 1e9) / h2d_gbs,
                "pinned_torch_value": n_total * args.steps / (pinned_ms / 1e3)},
        # per step: gather_warp_kernel, query_ts_kernel outer (side stream) and
        # inner (no memset nodes: the gather re-arms its own counters); the
        # per_object mode adds the bucketing kernels (histogram, scan, scatter)
        # of both families
        "gpu_launches": args.steps * (3 + (6 if args.sharing == "per_object" else 0)),
        "train": train_leg,
        "c4_single_gpu": c4_single,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
