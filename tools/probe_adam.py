"""Dense Adam kernel timing at C2 with trained (sparse) moments: every
object touched, CUDA events around 50 launches, per family, per variant
(0 production select form, 4 plain expression)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import _lib, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.synthetic import c2  # noqa: E402
from paper_2306_07191_b200.train import collect_samples, train  # noqa: E402

torch.cuda.set_device(0)
L = _lib.lib()
scene = c2(build_device=torch.device("cuda", 0))
model = build_model(NifConfig(seed=0), scene)
samples = collect_samples(scene, spp=2, seed=scene.seed)
train(model, samples, epochs=int(sys.argv[1]) if len(sys.argv) > 1 else 1)
torch.cuda.synchronize()
a = model.config.adam
for which in ("outer", "inner"):
    fam = model.family(which)
    fv, tv = fam.view(), fam.train_view()
    elems = sum(t.numel() for t in (fam.params,)) if hasattr(fam, "params") else 0
    for variant in (4, 0, 4, 0):
        L.nif_debug_set_train_variant(variant)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for it in range(60):
            if it == 10:
                e0.record()
            fam.counts.fill_(1)
            L.nif_adam_dev(fv, tv, model.learning_rate, a.beta1, a.beta2, a.epsilon,
                           _lib.stream_ptr(None))
        e1.record()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for it in range(50):
            fam.counts.fill_(1)
        f1.record()
        torch.cuda.synchronize()
        us = (e0.elapsed_time(e1) - f0.elapsed_time(f1)) / 50 * 1e3
        print(f"{which} variant {variant}: {us:.1f} us per Adam step ({fam.n_obj} objects)")
L.nif_debug_set_train_variant(0)
