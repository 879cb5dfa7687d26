"""Phase timing (clock64 stamps) of the split-path tcgen05 MLP kernel at C2.

    python tools/probe_mlp.py [flags]   (on the GPU box)
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2306_07191_b200 import _lib, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.pipeline import VisibilityEngine, sample_pass_dev, shadow_rays_dev  # noqa: E402
from paper_2306_07191_b200.synthetic import c2  # noqa: E402

flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
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
feat = torch.empty(int(L.nif_feat_scratch_bytes(b.cap)), dtype=torch.uint8, device="cuda")
prof = torch.zeros(148 * 8 * 4 * 16, dtype=torch.int64, device="cuda")
for name, v, obj, ray, c4, r, cnt in (
        ("outer", vo, b.outer_obj, b.outer_ray, b.outer_coord, None, b.counts.data_ptr()),
        ("inner", vi, b.inner_obj, b.inner_ray, b.inner_coord, b.inner_r, b.counts.data_ptr() + 8)):
    for rep in range(3):
        prof.zero_()
        L.nif_debug_set_prof(prof.data_ptr())
        L.nif_query_split_dev(v, obj.data_ptr(), ray.data_ptr(), c4.data_ptr(),
                              r.data_ptr() if r is not None else None, cnt, b.cap,
                              eng.occ.data_ptr(), None, feat.data_ptr(), flags, _lib.stream_ptr())
        torch.cuda.synchronize()
        L.nif_debug_set_prof(None)
    p = prof.view(-1, 4, 16).cpu().numpy()
    rows = p[p[:, :, 0] != 0].copy()
    rows[:, 11:14] = 0
    print(f"== {name}: {len(rows)} tiles sampled")
    names = {1: "feat st + sync", 2: "MMA1 round trip"}
    for l in range(1, 5):
        names[3 * l] = f"epilogue {l}"
        names[3 * l + 1] = f"named sync {l}"
        names[3 * l + 2] = f"MMA {l + 1} round trip"
    names[15] = "head (CUDA cores)"
    prev = 0
    for k in range(1, 16):
        if k not in names or not np.any(rows[:, k]):
            continue
        dt = rows[:, k] - rows[:, prev]
        print(f"  {names[k]:16s} median {np.median(dt):8.0f}  p90 {np.percentile(dt, 90):8.0f} cycles")
        prev = k
    tot = rows[:, 15] - rows[:, 0]
    rows[:, 14] = 0
    print(f"  tile total median {np.median(tot):.0f} cycles")
    first = p[:, 0, :]
    okw = first[:, 0] != 0
    span = (first[okw, 14] - first[okw, 0])
    cnt = first[okw, 13]
    print(f"  warpgroups {okw.sum()}  tiles/wg median {np.median(cnt):.0f} max {cnt.max()}  "
          f"loop span median {np.median(span):.0f} max {span.max()} cycles  "
          f"per tile {np.median(span / np.maximum(cnt, 1)):.0f}")
    ns = first[okw, 12] - first[okw, 11]
    print(f"  loop wall median {np.median(ns)/1e3:.1f} us max {ns.max()/1e3:.1f} us -> "
          f"clock {np.median(span / np.maximum(ns, 1)):.3f} GHz; first start to last end "
          f"{(first[okw, 12].max() - first[okw, 11].min())/1e3:.1f} us")
    # time between consecutive tiles of one warpgroup
    st = p[:, :, 0]
    ok = (st[:, 1:] != 0) & (st[:, :-1] != 0)
    print(f"  tile-to-tile median {np.median((st[:, 1:] - st[:, :-1])[ok]):.0f} cycles")
