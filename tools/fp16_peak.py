"""the fused MLP runs fp16 operands and is measured against
the measured bf16 dense peak (MEASURED_PEAKS.json); fp16 and bf16 share the
kind::f16 tensor rate -- confirm with one fp16 and one bf16 GEMM on this box
(torch.matmul 8192^3, best of 10, CUDA events).

    python tools/fp16_peak.py -> JSON line
"""
import json

import torch

torch.cuda.set_device(0)
N = 8192
out = {"gemm": f"torch.matmul {N}^3, 2*N^3 flop, best of 10"}
for name, dt in (("fp16", torch.float16), ("bf16", torch.bfloat16)):
    a = torch.randn(N, N, device="cuda", dtype=dt)
    b = torch.randn(N, N, device="cuda", dtype=dt)
    for _ in range(3):
        a @ b
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[f"{name}_tflops"] = round(2 * N ** 3 / (best / 1e3) / 1e12, 1)
out["fp16_over_bf16"] = round(out["fp16_tflops"] / out["bf16_tflops"], 3)
print(json.dumps(out))
