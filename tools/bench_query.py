"""Time the fused query kernels per variant at C2 (GPU box).

    python tools/bench_query.py [--train-epochs 0]

Variants (nif_debug_set_query_variant): 0 production (A operand in TMEM);
2 runtime-shape generic kernel; 11 TMEM operand, one tile per CTA (6 per
SM); 12 the round-1 inner configuration (2 CTAs x 3 warpgroups per SM); "S0" the
split path (encoding kernel + MLP kernel); "P" the fp32 SIMT kernel. Logits of every variant are
compared with the generic kernel on the same records.
"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2306_07191_b200 import _lib, build_model  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.pipeline import VisibilityEngine, sample_pass_dev, shadow_rays_dev  # noqa: E402
from paper_2306_07191_b200.synthetic import c2  # noqa: E402

torch.cuda.set_device(0)
scene = c2()
data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
_, o, d, t = shadow_rays_dev(data, require_emit=False)
n = int(t.numel())
model = build_model(NifConfig(seed=0), scene)
eng = VisibilityEngine(scene, model, n)
eng.origins[:n].copy_(o)
eng.dirs[:n].copy_(d)
eng.tmaxs[:n].copy_(t)
eng.run(n)
torch.cuda.synchronize()
L = _lib.lib()
L.nif_debug_set_query_variant.argtypes = [C.c_int]
b = eng.buf
vo, vi = eng._family_views()
counts = b.counts.cpu().numpy()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
st = torch.cuda.current_stream()
fams = (("outer", vo, b.outer_obj, b.outer_ray, b.outer_coord, None, b.counts.data_ptr(), counts[0]),
        ("inner", vi, b.inner_obj, b.inner_ray, b.inner_coord, b.inner_r, b.counts.data_ptr() + 8,
         counts[1]))
ref = {}
VARIANTS = [(v if v[0] in "SP" else int(v)) for v in sys.argv[1].split(',')] if len(sys.argv) > 1 else [2, 0, 12]
if 2 not in VARIANTS:
    VARIANTS = [2] + VARIANTS
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 30
feat = torch.empty(int(L.nif_feat_scratch_bytes(b.cap)), dtype=torch.uint8, device="cuda")
for variant in VARIANTS:
    if not isinstance(variant, str):
        L.nif_debug_set_query_variant(variant)
    for name, v, obj, ray, c4, r, cnt, m in fams:
        logits = torch.zeros(b.cap, dtype=torch.float32, device="cuda")

        def run(lg=None):
            if variant == "P":  # the fp32 SIMT kernel (per_object / geometry path)
                rc = L.nif_query_dev(v, obj.data_ptr(), ray.data_ptr(), c4.data_ptr(),
                                     r.data_ptr() if r is not None else None, cnt, b.cap,
                                     eng.occ.data_ptr(), lg, _lib.IMPL_SIMT, st.cuda_stream)
            elif isinstance(variant, str):
                rc = L.nif_query_split_dev(v, obj.data_ptr(), ray.data_ptr(), c4.data_ptr(),
                                           r.data_ptr() if r is not None else None, cnt, b.cap,
                                           eng.occ.data_ptr(), lg, feat.data_ptr(),
                                           int(variant[1:]), st.cuda_stream)
            else:
                rc = L.nif_query_dev(v, obj.data_ptr(), ray.data_ptr(), c4.data_ptr(),
                                     r.data_ptr() if r is not None else None, cnt, b.cap,
                                     eng.occ.data_ptr(), lg, _lib.IMPL_TCGEN05, st.cuda_stream)
            if rc != 0:
                raise RuntimeError(L.nif_last_error().decode())
        run(logits.data_ptr())
        torch.cuda.synchronize()
        lg = logits[:m].clone()
        if variant == 2:
            ref[name] = lg
            err = 0.0
        else:
            err = float((lg - ref[name]).abs().max())
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        tot = 0.0
        reps = REPS
        for _ in range(3):
            run()
        for _ in range(reps):
            flush.fill_(1)
            e0.record()
            run()
            e1.record()
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        us = tot / reps * 1e3
        flop = (9088 if name == "outer" else 10560) * m
        print(f"variant {variant} {name}: {us:7.1f} us  {flop / us / 1e6:7.1f} TFLOP/s  "
              f"records {m}  max|dlogit| vs generic {err:.2e}")
L.nif_debug_set_query_variant(0)
