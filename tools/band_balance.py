"""Projected strong scaling of the band-split frame (bench.py under torchrun)
on ONE GPU: each rank's share of the frame is resolved here in turn and
timed exactly like bench.py's step (captured visibility pass, L2 flushed,
CUDA events); the N-GPU frame time is the slowest share (the ranks run
independently, no collective on the data path). Two assignments of pixel
rows to ranks:

  contiguous   rank r owns rows band(H, r, N)                (round-2 bench)
  interleaved  the frame cut in N*K row strips, rank r owns strips r, r+N, ...

    python tools/band_balance.py [width height] [K] [scene c2|c3] -> JSON lines
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_07191_b200 import build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.parallel import band, rank_strips  # noqa: E402
from paper_2306_07191_b200.pipeline import (VisibilityEngine, sample_pass_dev,  # noqa: E402
                                            shadow_rays_dev)
from paper_2306_07191_b200 import synthetic  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 2 else 3840
H = int(sys.argv[2]) if len(sys.argv) > 2 else 2160
K = int(sys.argv[3]) if len(sys.argv) > 3 else 8
SCENE = sys.argv[4] if len(sys.argv) > 4 else "c2"
torch.cuda.set_device(0)
import dataclasses  # noqa: E402

scene = getattr(synthetic, SCENE)(build_device=torch.device("cuda", 0))
cam = dataclasses.replace(scene.camera, width=W, height=H)
model = build_model(NifConfig(seed=0), scene)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
stream = torch.cuda.current_stream()


def rays_of(strips):
    parts = []
    for pix0, n_pix in strips:
        data = sample_pass_dev(scene, cam, 0, scene.seed, "importance", pix0, n_pix)
        _, o, d, t = shadow_rays_dev(data, require_emit=False)
        parts.append((o, d, t))
    return (torch.cat([p[0] for p in parts]), torch.cat([p[1] for p in parts]),
            torch.cat([p[2] for p in parts]))


def frame_ms(strips, steps=20):
    o, d, t = rays_of(strips)
    n = int(t.numel())
    eng = VisibilityEngine(scene, model, max(n, 1))
    eng.origins[:n].copy_(o)
    eng.dirs[:n].copy_(d)
    eng.tmaxs[:n].copy_(t)
    g = eng.capture(n)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for e0, e1 in evs:
        flush.fill_(1.0)
        e0.record(stream)
        g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    ms = float(np.median([e0.elapsed_time(e1) for e0, e1 in evs]))
    occ = int(eng.occ[:n].sum())
    del eng, g
    return ms, n, occ


t1, n1, occ1 = frame_ms([(0, W * H)])
print(json.dumps({"scene": SCENE, "frame": f"{W}x{H}", "n_gpus": 1, "frame_ms": t1, "rays": n1}),
      flush=True)
for N in (2, 4, 8):
    for mode in ("contiguous", "interleaved"):
        per = []
        for r in range(N):
            if mode == "contiguous":
                y0, y1 = band(H, r, N)
                strips = [(y0 * W, (y1 - y0) * W)]
            else:
                strips = rank_strips(W, H, r, N, K)
            per.append(frame_ms(strips))
        ms = [p[0] for p in per]
        rays = [p[1] for p in per]
        assert sum(rays) == n1 and sum(p[2] for p in per) == occ1
        print(json.dumps({"scene": SCENE, "frame": f"{W}x{H}", "n_gpus": N, "mode": mode,
                          "strips_per_rank": 1 if mode == "contiguous" else K,
                          "band_ms": [round(x, 4) for x in ms], "rays": rays,
                          "max_ms": max(ms), "mean_ms": float(np.mean(ms)),
                          "projected_speedup": t1 / max(ms),
                          "projected_efficiency": t1 / max(ms) / N}), flush=True)
