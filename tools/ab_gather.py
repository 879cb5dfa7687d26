"""A/B of the hot-path gather variants at C2 (nif_debug_set_gather_variant):
gather alone and the whole visibility pass, CUDA events, L2 flushed.

    python tools/ab_gather.py [variants, default 3,0]
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import _lib, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.pipeline import (GatherBuffers, VisibilityEngine, gather_dev,  # noqa: E402
                                            sample_pass_dev, shadow_rays_dev)
from paper_2306_07191_b200.synthetic import c2  # noqa: E402

torch.cuda.set_device(0)
variants = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "3,0").split(",")]
scene = c2()
ds = scene.device()
data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
_, o, d, t = shadow_rays_dev(data)
n = int(t.numel())
route = scene.nif_route_mask(None)
buf = GatherBuffers(n, int(route.sum()), ds.device)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
model = build_model(NifConfig(seed=0), scene)
eng = VisibilityEngine(scene, model, n)
eng.origins[:n].copy_(o)
eng.dirs[:n].copy_(d)
eng.tmaxs[:n].copy_(t)


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


for rep in range(2):
    for v in variants:
        _lib.lib().nif_debug_set_gather_variant(v)
        g = timeit(lambda: gather_dev(ds, ds.route(route), o, d, t, n, buf))
        if os.environ.get("GATHER_ONLY"):  # queue formats under test the queries cannot read
            print(f"variant {v}: gather {g:.1f} us", flush=True)
            continue
        f = timeit(lambda: eng.run(n))
        occ = eng.occ[:n].clone()
        print(f"variant {v}: gather {g:.1f} us  pass {f:.1f} us  occluded {int(occ.sum())}",
              flush=True)
_lib.lib().nif_debug_set_gather_variant(0)
