"""Time the gather (and the full pass) for the library named by NIF_B200_LIB."""
import os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import build_model
from paper_2306_07191_b200.nif import NifConfig
from paper_2306_07191_b200.pipeline import GatherBuffers, gather_dev, sample_pass_dev, shadow_rays_dev, VisibilityEngine
from paper_2306_07191_b200.synthetic import c2
torch.cuda.set_device(0)
scene = c2(); ds = scene.device()
data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
_, o, d, t = shadow_rays_dev(data, require_emit=False)
n = int(t.numel()); route = scene.nif_route_mask(None)
buf = GatherBuffers(n, int(route.sum()), ds.device)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
def timeit(fn, reps=20):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); tot = 0.0
    for _ in range(3): fn()
    for _ in range(reps):
        flush.fill_(1); e0.record(); fn(); e1.record(); e1.synchronize(); tot += e0.elapsed_time(e1)
    return tot / reps * 1e3
g = timeit(lambda: gather_dev(ds, ds.route(route), o, d, t, n, buf))
model = build_model(NifConfig(seed=0), scene)
eng = VisibilityEngine(scene, model, n)
eng.origins[:n].copy_(o); eng.dirs[:n].copy_(d); eng.tmaxs[:n].copy_(t)
f = timeit(lambda: eng.run(n))
print(f"{os.environ.get('NIF_B200_LIB','default')}: gather {g:.1f} us  pass {f:.1f} us")
