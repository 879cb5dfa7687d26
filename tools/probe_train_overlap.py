"""Per-family epoch time at C2 (2 spp): outer alone, inner alone, both
(the two families run on their own streams): do they overlap?"""
import dataclasses
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.synthetic import c2  # noqa: E402
from paper_2306_07191_b200.train import collect_samples, train  # noqa: E402

torch.cuda.set_device(0)
scene = c2(build_device=torch.device("cuda", 0))
smp = collect_samples(scene, spp=2, seed=scene.seed)
empty = {k: getattr(smp, k)[:0] for k in ("outer_obj", "outer_coord", "outer_label", "outer_ray",
                                           "inner_obj", "inner_coord", "inner_label", "inner_ray")}
only_outer = dataclasses.replace(smp, **{k: v for k, v in empty.items() if k.startswith("inner")})
only_inner = dataclasses.replace(smp, **{k: v for k, v in empty.items() if k.startswith("outer")})
for name, s in (("outer", only_outer), ("inner", only_inner), ("both", smp)):
    model = build_model(NifConfig(seed=0), scene)
    train(model, s, epochs=1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    train(model, s, epochs=5)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"{name}: {dt * 1e3:.1f} ms/epoch ({s.n_outer} outer + {s.n_inner} inner samples)")
