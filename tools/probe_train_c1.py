"""C1 training throughput (the reference's 8 spp x 10 epochs schedule)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2306_07191_b200 import build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.synthetic import c1  # noqa: E402
from paper_2306_07191_b200.train import collect_samples, train  # noqa: E402

torch.cuda.set_device(0)
scene = c1(256, 256)
model = build_model(NifConfig(seed=0), scene)
t0 = time.perf_counter()
s = collect_samples(scene, spp=8, seed=scene.seed)
torch.cuda.synchronize()
t1 = time.perf_counter()
train(model, s, epochs=1)
torch.cuda.synchronize()
t2 = time.perf_counter()
curve = train(model, s, epochs=10)
torch.cuda.synchronize()
t3 = time.perf_counter()
steps = (-(-s.n_outer // 2048) - (-s.n_inner // 4096)) * 10
print(f"collect {t1 - t0:.3f} s; 10 epochs {t3 - t2:.3f} s = {steps} steps, "
      f"{(t3 - t2) / steps * 1e6:.1f} us/step; loss {curve[-1]}")
