"""Training-step timing at C2 (GPU box): wall time per optimiser step vs
the kernels' own time (run under ncu for the per-kernel split).

    python tools/probe_train.py [spp] [epochs] [train_variant]
"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2306_07191_b200 import build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.synthetic import c2  # noqa: E402
from paper_2306_07191_b200.train import collect_samples, train  # noqa: E402

spp = int(sys.argv[1]) if len(sys.argv) > 1 else 2
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
variant = int(sys.argv[3]) if len(sys.argv) > 3 else 0
torch.cuda.set_device(0)
from paper_2306_07191_b200 import _lib  # noqa: E402
_lib.lib().nif_debug_set_train_variant(variant)
scene = c2()
model = build_model(NifConfig(seed=0), scene)
samples = collect_samples(scene, spp=spp, seed=scene.seed)
train(model, samples, epochs=1)  # warm
torch.cuda.synchronize()
steps = (-(-samples.n_outer // 2048) - (-samples.n_inner // 4096)) * epochs
t0 = time.perf_counter()
curve = train(model, samples, epochs=epochs)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"variant {variant}  samples {samples.n_outer}+{samples.n_inner}  steps {steps}  {dt:.3f} s  "
      f"{steps / dt:.0f} steps/s  {dt / steps * 1e6:.1f} us/step  loss {curve[-1]}")
t0 = time.perf_counter()
curve = train(model, samples, epochs=5)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"5 epochs: {5 * steps / dt:.0f} steps/s  {dt / (5 * steps) * 1e6:.1f} us/step")
