"""GPU time of one captured training step (steady state, CUDA events
around 200 back-to-back replays) per family at C2, and of each of its
three kernels launched eagerly in the same loop shape."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import _lib, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.synthetic import c2  # noqa: E402
from paper_2306_07191_b200.train import _GraphStep, _Step, collect_samples, train  # noqa: E402

torch.cuda.set_device(0)
VARIANT = int(sys.argv[1]) if len(sys.argv) > 1 else 0
scene = c2(build_device=torch.device("cuda", 0))
smp = collect_samples(scene, spp=2, seed=scene.seed)
model = build_model(NifConfig(seed=0), scene)
train(model, smp, epochs=1)
torch.cuda.synchronize()
L = _lib.lib()
for which, bs in (("outer", 2048), ("inner", 4096)):
    obj = getattr(smp, f"{which}_obj")
    coord = getattr(smp, f"{which}_coord")
    label = getattr(smp, f"{which}_label")
    n = int(obj.shape[0])
    st = _Step(model, which)
    _lib.lib().nif_debug_set_train_variant(VARIANT)
    g = _GraphStep(st, obj, coord, label, n, bs)
    g.epoch(np.random.default_rng(0).permutation(n))  # captures the graph
    torch.cuda.synchronize()
    reps = min(200, n // bs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.cursor.zero_()
    e0.record()
    for _ in range(reps):
        g.graph.replay()
    e1.record()
    torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) / reps * 1e3
    # the three kernels eagerly, each timed over the same number of steps
    p = _lib.ptr
    sp = _lib.stream_ptr()
    a = model.config.adam
    parts = {}
    for name, fn in (
        ("prologue", lambda: L.nif_train_prologue_cur_dev(st.fv, st.tv, p(obj), p(g.perm),
                                                          p(g.cursor), bs, sp)),
        ("fwdbwd", lambda: L.nif_train_fwdbwd_cur_dev(st.fv, st.tv, p(obj), p(coord), p(label),
                                                      p(g.perm), p(g.cursor), bs, 0, 1,
                                                      p(st.sq), sp)),
        ("adam", lambda: L.nif_adam_units_dev(st.fv, st.tv, model.learning_rate, a.beta1,
                                              a.beta2, a.epsilon, None, bs, sp))):
        g.cursor.zero_()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        parts[name] = e0.elapsed_time(e1) / reps * 1e3
    print(f"{which}: graph step {t_graph:.1f} us; eager kernels " +
          ", ".join(f"{k} {v:.1f} us" for k, v in parts.items()))
