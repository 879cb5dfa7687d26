"""Phase timing of the fused gather kernel (clock64 stamps of warp 0 per tile)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import _lib  # noqa: E402
from paper_2306_07191_b200.pipeline import GatherBuffers, gather_dev, sample_pass_dev, shadow_rays_dev  # noqa: E402
from paper_2306_07191_b200.synthetic import c2  # noqa: E402

torch.cuda.set_device(0)
scene = c2()
ds = scene.device()
data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
_, o, d, t = shadow_rays_dev(data, require_emit=False)
n = int(t.numel())
route = scene.nif_route_mask(None)
buf = GatherBuffers(n, int(route.sum()), ds.device)
gather_dev(ds, ds.route(route), o, d, t, n, buf)
torch.cuda.synchronize()
L = _lib.lib()
fn = L.nif_debug_set_prof_gather
fn.argtypes = [C.c_void_p]
prof = torch.zeros(8192 * 8, dtype=torch.int64, device="cuda")
fn(prof.data_ptr())
gather_dev(ds, ds.route(route), o, d, t, n, buf)
torch.cuda.synchronize()
fn(None)
p = prof.view(-1, 8).cpu().numpy()
p = p[p[:, 0] != 0]
names = ["", "classify", "block scan+sync", "publish+anyhit", "look-back", "sync", "write"]
print(f"{len(p)} tiles")
for k in range(1, 7):
    dt = p[:, k] - p[:, k - 1]
    print(f"  {names[k]:16s} median {np.median(dt):8.0f}  p90 {np.percentile(dt, 90):8.0f}")
print(f"  total median {np.median(p[:, 6] - p[:, 0]):.0f}")
