"""Chunk-pipelined visibility pass at C2: the frame's rays split in K chunks;
chunk k+1's gather runs on its own stream while chunk k's two queries run
(double-buffered record queues), with the gather / query grids capped per
SM so both can be resident. Captured as one CUDA graph; GPU time per frame
(CUDA events around graph replays, L2 flushed) against the serial pass.

    python tools/probe_pipeline.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import _lib, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.pipeline import (GatherBuffers, VisibilityEngine,  # noqa: E402
                                            sample_pass_dev, shadow_rays_dev)
from paper_2306_07191_b200.synthetic import c2  # noqa: E402

torch.cuda.set_device(0)
L = _lib.lib()
scene = c2()
ds = scene.device()
data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
_, o, d, t = shadow_rays_dev(data)
n = int(t.numel())
model = build_model(NifConfig(seed=0), scene)
eng = VisibilityEngine(scene, model, n)
eng.origins[:n].copy_(o)
eng.dirs[:n].copy_(d)
eng.tmaxs[:n].copy_(t)
eng.checked_run(n)
ref = eng.occ[:n].clone()
vo, vi = eng._family_views()
route = eng.route
n_net = int(eng.route_np.sum())
flush = torch.empty(64 * 1024 * 1024, device="cuda")
p = _lib.ptr


def timeit(fn, reps=30):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        flush.fill_(1)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def build(K, gcpsm, qcpsm):
    step = -(-n // K)
    bounds = [(s, min(n, s + step)) for s in range(0, n, step)]
    bufs = [GatherBuffers(step, n_net, ds.device, slots=4) for _ in range(2)]
    occ = torch.zeros(n, dtype=torch.uint8, device="cuda")
    sg, so, si = (torch.cuda.Stream() for _ in range(3))
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    L.nif_debug_set_gather_grid(gcpsm)
    L.nif_debug_set_query_grid(qcpsm)
    with torch.cuda.stream(cap):
        g.capture_begin()
        for s_ in (sg, so, si):
            s_.wait_stream(cap)
        released = [None, None]
        for k, (s0, s1) in enumerate(bounds):
            b = bufs[k % 2]
            if released[k % 2] is not None:
                for ev in released[k % 2]:
                    sg.wait_event(ev)
            out = _lib.GatherOut.from_buffer_copy(b.out)
            out.bvh_occ = occ.data_ptr() + s0
            L.nif_gather_dev(ds.view, p(route), eng.origins.data_ptr() + 24 * s0,
                             eng.dirs.data_ptr() + 24 * s0, eng.tmaxs.data_ptr() + 8 * s0,
                             s1 - s0, out, p(b.workspace), b.workspace.numel(), sg.cuda_stream)
            ge = torch.cuda.Event()
            ge.record(sg)
            so.wait_event(ge)
            si.wait_event(ge)
            cnt = b.counts.data_ptr()
            L.nif_query_dev(vo, p(b.outer_obj), p(b.outer_ray), p(b.outer_coord), None, cnt,
                            b.cap, occ.data_ptr() + s0, None, _lib.IMPL_AUTO, so.cuda_stream)
            L.nif_query_dev(vi, p(b.inner_obj), p(b.inner_ray), p(b.inner_coord), p(b.inner_r),
                            cnt + 8, b.cap, occ.data_ptr() + s0, None, _lib.IMPL_AUTO,
                            si.cuda_stream)
            eo, ei = torch.cuda.Event(), torch.cuda.Event()
            eo.record(so)
            ei.record(si)
            released[k % 2] = (eo, ei)
        for s_ in (sg, so, si):
            cap.wait_stream(s_)
        g.capture_end()
    torch.cuda.current_stream().wait_stream(cap)
    L.nif_debug_set_gather_grid(0)
    L.nif_debug_set_query_grid(0)
    return g, occ


g_serial = eng.capture(n)
base = timeit(lambda: g_serial.replay())
print(f"serial pass: {base:.1f} us", flush=True)
for K in (2, 3, 4, 6):
    for gc, qc in ((0, 0), (1, 1), (2, 1), (1, 2)):
        try:
            g, occ = build(K, gc, qc)
            g.replay()
            torch.cuda.synchronize()
            ok = torch.equal(occ, ref)
            tt = timeit(lambda: g.replay())
            print(f"K={K} gather cpsm {gc} query cpsm {qc}: {tt:.1f} us  same bits {ok}",
                  flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"K={K} {gc},{qc}: {e}", flush=True)
