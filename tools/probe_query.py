"""Phase timing of the tcgen05 query kernel (clock64 stamps per CTA).

    python tools/probe_query.py   (on the GPU box)
"""

import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2306_07191_b200 import _lib, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.pipeline import (VisibilityEngine, sample_pass_dev,  # noqa: E402
                                            shadow_rays_dev)
from paper_2306_07191_b200.synthetic import c2  # noqa: E402

torch.cuda.set_device(0)
scene = c2()
data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
_, o, d, t = shadow_rays_dev(data, require_emit=False)
n = int(t.numel())
model = build_model(NifConfig(seed=0), scene)
eng = VisibilityEngine(scene, model, n)
eng.origins[:n].copy_(o)
eng.dirs[:n].copy_(d)
eng.tmaxs[:n].copy_(t)
eng.run(n)
torch.cuda.synchronize()
L = _lib.lib()
L.nif_debug_set_prof.argtypes = [C.c_void_p]
prof = torch.zeros(148 * 8 * 4 * 16, dtype=torch.int64, device="cuda")
b = eng.buf
vo, vi = eng._family_views()
for name, v, obj, ray, c4, r, cnt in (
        ("outer", vo, b.outer_obj, b.outer_ray, b.outer_coord, None, b.counts.data_ptr()),
        ("inner", vi, b.inner_obj, b.inner_ray, b.inner_coord, b.inner_r, b.counts.data_ptr() + 8)):
    prof.zero_()
    L.nif_debug_set_prof(prof.data_ptr())
    L.nif_query_dev(v, obj.data_ptr(), ray.data_ptr(), c4.data_ptr(),
                    r.data_ptr() if r is not None else None, cnt, b.cap, eng.occ.data_ptr(), None,
                    0, _lib.stream_ptr())
    torch.cuda.synchronize()
    L.nif_debug_set_prof(None)
    p = prof.view(-1, 4, 16).cpu().numpy()
    ok = p[:, :, 0] != 0
    rows = p[ok]
    last = 14 if name == "inner" else 11
    print(f"== {name}: {len(rows)} tiles sampled")
    names = {1: "encode", 2: "sync", 3: "issue+prefetch", 4: "wait L1"}
    for l in range(1, 5):
        names[3 + 3 * l] = f"epilogue {l}"
        names[4 + 3 * l] = f"sync {l}"
        names[5 + 3 * l] = f"wait MMA {l + 1}"
    prev = 0
    for k in range(1, 16):
        if k not in names or not np.any(rows[:, k]):
            continue
        dt = rows[:, k] - rows[:, prev]
        print(f"  {names[k]:16s} median {np.median(dt):8.0f}  p90 {np.percentile(dt, 90):8.0f} cycles")
        prev = k
    tot = rows[:, :16].max(axis=1) - rows[:, 0]
    print(f"  tile total median {np.median(tot):.0f} cycles")
