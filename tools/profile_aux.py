"""One launch each of the non-query kernels at C2 for an ncu capture:
label_kernel (collect_samples), bvh_occluded_kernel (BvhBackend), and the
training step kernels (fused step and the data-parallel split step).

    ncu --set full -k regex:"label_kernel|bvh_occluded|train_|adam_units|scatter_" \
        -o gpurun_out/aux python tools/profile_aux.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import BvhBackend, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.pipeline import sample_pass_dev, shadow_rays_dev  # noqa: E402
from paper_2306_07191_b200.synthetic import c2  # noqa: E402
from paper_2306_07191_b200.train import _GraphStep, _Sink, _Step, collect_samples  # noqa: E402

torch.cuda.set_device(0)
scene = c2(build_device=torch.device("cuda", 0))
smp = collect_samples(scene, spp=1, seed=scene.seed)  # label_kernel on the C2 records
print("records", smp.n_outer + smp.n_inner, flush=True)
data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
_, o, d, t = shadow_rays_dev(data)
BvhBackend().occluded_dev(scene, o, d, t)  # bvh_occluded_kernel on the C2 shadow rays
print("rays", int(t.numel()), flush=True)
for which, bs in (("outer", 2048), ("inner", 4096)):
    obj = getattr(smp, f"{which}_obj")
    n = int(obj.shape[0])
    for det in (None, True):
        model = build_model(NifConfig(seed=0), scene)
        st = _Step(model, which)
        sink = None if det is None else _Sink(st, bs, 1, 0, None, deterministic=True)
        g = _GraphStep(st, obj, getattr(smp, f"{which}_coord"), getattr(smp, f"{which}_label"),
                       min(n, 3 * bs), bs, sink, capture=False)
        g.epoch(np.random.default_rng(0).permutation(min(n, 3 * bs)))
torch.cuda.synchronize()
print("done")
