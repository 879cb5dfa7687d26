"""Where the fixed cost of a visibility pass goes: %globaltimer timelines of
the hot-path gather (per warp) and of the fused inner query launched behind
it with programmatic dependent launch (per warpgroup), as in the frame.
Rays: the C2 frame, and a 650k-ray block (one rank's share of the 4K frame
on 8 GPUs). L2 flushed before each pass.

    python tools/probe_timeline.py -> JSON lines (us relative to the first
    gather warp's entry)
"""
import dataclasses
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import _lib, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.pipeline import (VisibilityEngine, gather_dev,  # noqa: E402
                                            sample_pass_dev, shadow_rays_dev)
from paper_2306_07191_b200.synthetic import c2  # noqa: E402

torch.cuda.set_device(0)
L = _lib.lib()
scene = c2()
model = build_model(NifConfig(seed=0), scene)
flush = torch.empty(64 * 1024 * 1024, device="cuda")


def rays(w, h):
    cam = dataclasses.replace(scene.camera, width=w, height=h)
    data = sample_pass_dev(scene, cam, 0, scene.seed)
    _, o, d, t = shadow_rays_dev(data, require_emit=False)
    return o, d, t


def q(v, ps=(0, 50, 90, 99, 100)):
    v = np.asarray(v, np.float64)
    return {f"p{p}": round(float(np.percentile(v, p)), 2) for p in ps}


def probe(name, o, d, t, reps=5):
    n = int(t.numel())
    eng = VisibilityEngine(scene, model, n)
    eng.origins[:n].copy_(o)
    eng.dirs[:n].copy_(d)
    eng.tmaxs[:n].copy_(t)
    eng.checked_run(n)
    b = eng.buf
    vo, vi = eng._family_views()
    sp = _lib.stream_ptr()
    gtl = torch.zeros(148 * 8 * 8 * 4, dtype=torch.int64, device="cuda")
    qtl = torch.zeros(148 * 8 * 5, dtype=torch.int64, device="cuda")
    out = []
    for fam in ("inner", "outer"):
        for rep in range(reps):
            gtl.zero_()
            qtl.zero_()
            flush.fill_(1.0)
            torch.cuda.synchronize()
            L.nif_debug_set_timeline_gather(gtl.data_ptr())
            L.nif_debug_set_timeline_query(qtl.data_ptr())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gather_dev(eng.ds, eng.route, eng.origins, eng.dirs, eng.tmaxs, n, b)
            if fam == "inner":
                L.nif_query_dev(vi, b.inner_obj.data_ptr(), b.inner_ray.data_ptr(),
                                b.inner_coord.data_ptr(), b.inner_r.data_ptr(),
                                b.counts.data_ptr() + 8, b.cap, eng.occ.data_ptr(), None, 0, sp)
            else:
                L.nif_query_dev(vo, b.outer_obj.data_ptr(), b.outer_ray.data_ptr(),
                                b.outer_coord.data_ptr(), None, b.counts.data_ptr(), b.cap,
                                eng.occ.data_ptr(), None, 0, sp)
            e1.record()
            torch.cuda.synchronize()
            L.nif_debug_set_timeline_gather(None)
            L.nif_debug_set_timeline_query(None)
            g = gtl.view(-1, 4).cpu().numpy().astype(np.float64)
            g = g[g[:, 0] > 0]
            qq = qtl.view(-1, 5).cpu().numpy().astype(np.float64)
            qq = qq[qq[:, 0] > 0]
            t0 = g[:, 0].min()
            rec = {"case": name, "rays": n, "family": fam, "rep": rep,
                   "events_us": round(e0.elapsed_time(e1) * 1e3, 2),
                   "gather_warps": len(g),
                   "gather_entry": q((g[:, 0] - t0) / 1e3),
                   "gather_ready": q((g[:, 1] - t0) / 1e3),
                   "gather_exit": q((g[:, 2] - t0) / 1e3),
                   "gather_chunks": {"min": int(g[:, 3].min()), "mean": float(g[:, 3].mean()),
                                     "max": int(g[:, 3].max())},
                   "query_wgs": len(qq),
                   "query_entry": q((qq[:, 0] - t0) / 1e3),
                   "query_wait_done": q((qq[:, 1] - t0) / 1e3),
                   "query_first_tile": q((qq[qq[:, 4] > 0, 2] - t0) / 1e3) if (qq[:, 4] > 0).any()
                   else None,
                   "query_exit": q((qq[:, 3] - t0) / 1e3),
                   "query_tiles": {"min": int(qq[:, 4].min()), "mean": float(qq[:, 4].mean()),
                                   "max": int(qq[:, 4].max())}}
            if rep == reps - 1:
                print(json.dumps(rec), flush=True)
            out.append(rec)
    del eng
    return out


o, d, t = rays(1920, 1080)
probe("C2 frame", o, d, t)
o, d, t = rays(3840, 2160)
N = int(t.numel())
a = (N - 650000) // 2
probe("650k block of the 4K frame", o[a:a + 650000], d[a:a + 650000], t[a:a + 650000])
