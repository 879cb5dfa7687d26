"""GPU time per optimiser step (steady state: CUDA events around back-to-back
graph replays) at C2 for the step variants of train.py, per family:

  fused      -- single GPU: prologue, fwd/bwd with the grid scatter fused, Adam
  split      -- _Sink world 1: exchange buffer, batch-wide warp-aggregated
                atomic scatter, MLP copy, Adam
  split-fx   -- _Sink with the order-independent fixed-point scatter
  split-det  -- _Sink deterministic: sorted scatter + ordered MLP reduction
  dp-nccl    -- _Sink with a (world-size 1) NCCL group: the all-reduce of the
                exchange buffer captured in the graph, sorted scatter

    python tools/probe_dp_step.py [--json out.json]
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.synthetic import c2  # noqa: E402
from paper_2306_07191_b200.train import _GraphStep, _Sink, _Step, collect_samples  # noqa: E402

torch.cuda.set_device(0)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import torch.distributed as dist  # noqa: E402
dist.init_process_group("nccl", rank=0, world_size=1)
scene = c2(build_device=torch.device("cuda", 0))
smp = collect_samples(scene, spp=2, seed=scene.seed)
out = {"workload": "C2 samples (2 spp), NifConfig defaults, batch 2^11 outer / 2^12 inner",
       "unit": "us per optimiser step (GPU, graph replay)"}
for which, bs in (("outer", 2048), ("inner", 4096)):
    obj = getattr(smp, f"{which}_obj")
    coord = getattr(smp, f"{which}_coord")
    label = getattr(smp, f"{which}_label")
    n = int(obj.shape[0])
    res = {}
    modes = ("fused", "split", "split-fx", "split-det", "dp-nccl")
    if "--mode" in sys.argv:
        modes = sys.argv[sys.argv.index("--mode") + 1].split(",")
    for mode in modes:
        model = build_model(NifConfig(seed=0), scene)
        st = _Step(model, which)
        sink = None
        if mode != "fused":
            grp = dist.new_group([0]) if mode == "dp-nccl" else None
            sink = _Sink(st, bs, 1, 0, grp, deterministic=mode == "split-det",
                         scatter_mode=2 if mode == "split-fx" else None)
            if grp is not None:
                dist.all_reduce(sink.comm, group=grp)
        g = _GraphStep(st, obj, coord, label, n, bs, sink, capture=True)
        g.epoch(np.random.default_rng(0).permutation(n))  # captures + one epoch
        torch.cuda.synchronize()
        reps = min(int(os.environ.get("NIF_REPS", 200)), n // bs)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.cursor.zero_()
        e0.record()
        for _ in range(reps):
            g.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        res[mode] = round(e0.elapsed_time(e1) / reps * 1e3, 2)
    out[which] = res
    print(which, res, flush=True)
if "--json" in sys.argv:
    Path(sys.argv[sys.argv.index("--json") + 1]).write_text(json.dumps(out, indent=1) + "\n")
dist.destroy_process_group()
