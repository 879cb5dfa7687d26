"""Per-phase cycles (clock64 stamps, nif_debug_set_prof) of the production
fused query kernel at C2, tiles 2..7 of every warpgroup (steady state):
encode, barrier, MMA round trips, epilogues, head, and the tile period.

    tools/build_variant.sh prof query.cu -DNIF_TS_PROF=1
    NIF_B200_LIB=variants/libnif_prof.so python tools/probe_phases.py

(the stamps cost ~8 % of the kernel, so they are compiled in only on demand)
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import _lib, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.pipeline import VisibilityEngine, sample_pass_dev, shadow_rays_dev  # noqa: E402
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
b = eng.buf
vo, vi = eng._family_views()
slots = 148 * 8 * 8 * 16
prof = torch.zeros(slots, dtype=torch.int64, device="cuda")
out = {}
for name, v, obj, ray, c4, r, cnt, nl in (
        ("outer", vo, b.outer_obj, b.outer_ray, b.outer_coord, None, b.counts.data_ptr(), 2),
        ("inner", vi, b.inner_obj, b.inner_ray, b.inner_coord, b.inner_r, b.counts.data_ptr() + 8, 3)):
    for rep in range(2):
        prof.zero_()
        L.nif_debug_set_prof(prof.data_ptr())
        L.nif_query_dev(v, obj.data_ptr(), ray.data_ptr(), c4.data_ptr(),
                        r.data_ptr() if r is not None else None, cnt, b.cap, eng.occ.data_ptr(),
                        None, _lib.IMPL_TCGEN05, torch.cuda.current_stream().cuda_stream)
        L.nif_debug_set_prof(None)
        torch.cuda.synchronize()
    p = prof.view(-1, 8, 16).cpu().numpy().astype(np.float64)
    used = p[:, :, 0] > 0
    names = ["encode", "sync0", "mma1"]
    for layer in range(1, nl):
        names += [f"epi{layer}", f"sync{layer}", f"mma{layer + 1}"]
    names += ["head"]
    stamps = [0, 1, 2, 3] + [x for layer in range(1, nl) for x in (1 + 3 * layer, 2 + 3 * layer,
                                                                  3 + 3 * layer)] + [15]
    res = {}
    sel = used[:, 2:8]
    for nm, a, bb in zip(names, stamps[:-1], stamps[1:]):
        dur = (p[:, 2:8, bb] - p[:, 2:8, a])[sel]
        res[nm] = round(float(np.mean(dur)), 1)
    per = (p[:, 3:8, 0] - p[:, 2:7, 0])[used[:, 3:8] & used[:, 2:7]]
    res["tile_period"] = round(float(np.mean(per)), 1)
    res["sum_phases"] = round(sum(v for k, v in res.items() if k != "tile_period"), 1)
    out[name] = res
    print(name, json.dumps(res), flush=True)
if "--json" in sys.argv:
    Path(sys.argv[sys.argv.index("--json") + 1]).write_text(json.dumps(out, indent=1) + "\n")
