"""Time the GPU SAH build (nif_build_sah_dev) against the host build on
icosphere meshes; checks the two trees are byte-identical."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200.meshgen import icosphere  # noqa: E402
from paper_2306_07191_b200.scene import MAX_LEAF, _build_sah, build_sah_dev  # noqa: E402

out = []
for sub in [int(s) for s in (sys.argv[1:] or ["5", "6", "7", "8"])]:
    v, f, _ = icosphere(sub)
    t = v[f]
    lo = np.minimum(np.minimum(t[:, 0], t[:, 1]), t[:, 2])
    hi = np.maximum(np.maximum(t[:, 0], t[:, 1]), t[:, 2])
    ce = (lo + hi) * 0.5
    t0 = time.perf_counter()
    want = _build_sah(lo, hi, ce, MAX_LEAF)
    host_ms = (time.perf_counter() - t0) * 1e3
    d = [torch.from_numpy(x).cuda() for x in (lo, hi, ce)]
    build_sah_dev(*d)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        got = build_sah_dev(*d)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
    same = all(w.tobytes() == g.cpu().numpy().tobytes() for w, g in zip(want, got))
    rec = {"tris": len(f), "nodes": len(want[2]), "host_ms": round(host_ms, 2),
           "gpu_ms": round(min(times), 2), "identical": same}
    print(json.dumps(rec), flush=True)
    out.append(rec)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/probe_sah.json").write_text(json.dumps(out, indent=1))
