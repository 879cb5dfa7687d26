"""Host cost of torch.cuda.CUDAGraph.replay() vs the raw cudaGraphLaunch of
the same (tiny) graph: is the training epoch loop host-bound?"""
import ctypes
import time

import torch

torch.cuda.set_device(0)
x = torch.zeros(1, device="cuda")
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    g.capture_begin()
    x.add_(1)
    g.capture_end()
torch.cuda.current_stream().wait_stream(s)
for _ in range(10):
    g.replay()
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    g.replay()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"torch replay: host {1e6 * (t1 - t0) / n:.1f} us/launch, total {1e6 * (t2 - t0) / n:.1f} us/launch")
rt = ctypes.CDLL("libcudart.so.12") if False else None
try:
    exec_ = g.raw_cuda_graph_exec() if hasattr(g, "raw_cuda_graph_exec") else None
except Exception as e:  # noqa: BLE001
    exec_ = None
print("raw exec handle:", exec_)
