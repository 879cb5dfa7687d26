"""Visibility-pass time against ray count (the fixed cost that bounds the
strong scaling of a band-split frame): contiguous blocks of n rays from
the middle of the C4 (3840x2160) frame, captured pass, L2 flushed, CUDA
events; gather alone and the two queries alone beside it.

    python tools/pass_vs_n.py -> JSON lines
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
scene = c2()
cam = dataclasses.replace(scene.camera, width=3840, height=2160)
model = build_model(NifConfig(seed=0), scene)
data = sample_pass_dev(scene, cam, 0, scene.seed)
_, O, D, T = shadow_rays_dev(data, require_emit=False)
del data
N = int(T.numel())
flush = torch.empty(64 * 1024 * 1024, device="cuda")
stream = torch.cuda.current_stream()
L = _lib.lib()


def med(fn, reps=20):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for _ in range(3):
        fn()
    for e0, e1 in evs:
        flush.fill_(1.0)
        e0.record(stream)
        fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return float(np.median([e0.elapsed_time(e1) for e0, e1 in evs])) * 1e3


sizes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else
                          "0,1000,10000,50000,100000,200000,400000,650000,1000000,1300000,"
                          "2600000,5234811".split(","))]
for n in sizes:
    n = min(n, N)
    a = (N - n) // 2
    eng = VisibilityEngine(scene, model, max(n, 1))
    eng.origins[:n].copy_(O[a:a + n])
    eng.dirs[:n].copy_(D[a:a + n])
    eng.tmaxs[:n].copy_(T[a:a + n])
    g = eng.capture(n)
    t_pass = med(g.replay)
    b = eng.buf
    t_gather = med(lambda: gather_dev(eng.ds, eng.route, eng.origins, eng.dirs, eng.tmaxs, n, b))
    vo, vi = eng._family_views()
    sp = _lib.stream_ptr()
    t_outer = med(lambda: L.nif_query_dev(vo, b.outer_obj.data_ptr(), b.outer_ray.data_ptr(),
                                          b.outer_coord.data_ptr(), None, b.counts.data_ptr(),
                                          b.cap, eng.occ.data_ptr(), None, 0, sp))
    t_inner = med(lambda: L.nif_query_dev(vi, b.inner_obj.data_ptr(), b.inner_ray.data_ptr(),
                                          b.inner_coord.data_ptr(), b.inner_r.data_ptr(),
                                          b.counts.data_ptr() + 8, b.cap, eng.occ.data_ptr(),
                                          None, 0, sp))
    c = eng.counts()
    print(json.dumps({"rays": n, "outer": int(c[0]), "inner": int(c[1]),
                      "pass_us": round(t_pass, 2), "gather_us": round(t_gather, 2),
                      "outer_us": round(t_outer, 2), "inner_us": round(t_inner, 2)}), flush=True)
    del eng, g
