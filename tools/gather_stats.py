"""Culling statistics of the hot-path gather at C2 (GPU box):

    tools/build_variant.sh stats gather.cu -DNIF_GATHER_STATS
    NIF_B200_LIB=build/libnif_stats.so python tools/gather_stats.py

Measured (round 1): 1.52 objects/ray survive the warp-bundle cull, 1.21
the per-ray fp32 prefilter, 1.16 are hits -- the fp64 classification runs
on near-minimal candidates.
"""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, "/root/repo")
import torch
from paper_2306_07191_b200 import _lib
from paper_2306_07191_b200.pipeline import GatherBuffers, gather_dev, sample_pass_dev, shadow_rays_dev
from paper_2306_07191_b200.synthetic import c2
torch.cuda.set_device(0)
scene = c2(); ds = scene.device()
data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
_, o, d, t = shadow_rays_dev(data, require_emit=False)
n = int(t.numel()); route = scene.nif_route_mask(None)
buf = GatherBuffers(n, int(route.sum()), ds.device)
L = _lib.lib()
out = (C.c_ulonglong * 4)()
L.nif_debug_gather_stats.argtypes = [C.c_void_p]
L.nif_debug_gather_stats(C.addressof(out))
gather_dev(ds, ds.route(route), o, d, t, n, buf); torch.cuda.synchronize()
L.nif_debug_gather_stats(C.addressof(out))
rays, wm, pm, hits = list(out)
print(f"rays {rays} bundle survivors/ray {wm/rays:.2f} prefilter survivors/ray {pm/rays:.2f} classified hits/ray {hits/rays:.2f}; records {buf.counts.cpu().numpy()}")
