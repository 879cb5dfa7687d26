"""C5 microbenchmark (BASELINE.json configs[4]): grid
resolution x MLP width/depth sweep reporting the grid-encoding kernel's
achieved HBM GB/s and the MLP kernel's tensor-pipe utilisation.

    python tools/sweep_c5.py [--records 4194304] [--out profiles/r1_c5_sweep.json]

Records: 2^22 per launch, obj uniform over {1, 16} objects, coordinates
U[0,1)^4 (+ r ~ U[0,1]) from PCG64(seed 0) -- the incoherent worst case --
either in that order ("random") or sorted by object ("sorted"); latents
U(-1, 1), Xavier MLP. Stages are timed separately through the split path
(nif_query_split_dev flags: 2 = encoding kernel only, 4 = MLP kernel only)
and the production fused kernel (nif_query_dev) end to end.

Algorithmic work:
  encoding bytes / record = record in (obj i32 + 4 x f32 coords [+ f32 r])
                            + features out (outer 6 fp16, inner 13 fp16)
                            -> outer 20 + 12 = 32 B, inner 24 + 26 = 50 B
                            ("frac_hbm"); the kernel writes the MMA-ready
                            row (outer 16 B: 6 features + bias + pad; inner
                            32 B), so it moves outer 36 B, inner 56 B
                            ("frac_hbm_written"); table bytes are gathered
                            from L2 (reported separately as the
                            distinct-table footprint)
  MLP useful FLOP / record = 2 (in W + (L-1) W^2 + W)
  MLP executed MMA FLOP / record = 2 (16 W + (L-1) Kp W), Kp = ceil((W+1)/16)*16
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2306_07191_b200 import _lib  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig, NifModel  # noqa: E402


def timeit(fn, reps=20, flush=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1.0)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps * 1e-3  # seconds


def randomize(model, seed=1):
    g = torch.Generator(device=model.device)
    g.manual_seed(seed)
    for fam in (model.outer, model.inner):
        for key in ("pos", "dir", "dist"):
            if key == "dist" and fam.family == 0:
                continue
            p = fam.part(key)
            p.copy_(torch.rand(p.shape, generator=g, device=model.device) * 2 - 1)
        fam.dirty = True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", type=int, default=1 << 22)
    ap.add_argument("--out", default="")
    ap.add_argument("--enc-only", action="store_true", help="skip the MLP / fused sweeps")
    ap.add_argument("--fam", default="outer,inner")
    ap.add_argument("--R", default="", help="comma list overriding the resolutions")
    ap.add_argument("--objs", default="1,16")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
        if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else \
        {"hbm_gbs": 6553.0, "bf16_tflops": 1645.7}
    m = a.records
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    rng = np.random.Generator(np.random.PCG64(0))
    coords = rng.random((m, 5))
    results = {"records": m, "peaks": peaks, "encode": [], "mlp": [], "fused": []}
    cnt = torch.tensor([m], dtype=torch.int64, device=dev)
    ray = torch.arange(m, dtype=torch.int32, device=dev) % (1 << 20)
    occ = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)
    feat = torch.empty(int(L.nif_feat_scratch_bytes(m)), dtype=torch.uint8, device=dev)
    c4 = torch.from_numpy(coords[:, :4].astype(np.float32)).to(dev)
    rr = torch.from_numpy(coords[:, 4].astype(np.float32)).to(dev)
    sp = _lib.stream_ptr()

    def run_split(v, obj, which, flags):
        rc = L.nif_query_split_dev(v, obj.data_ptr(), ray.data_ptr(), c4.data_ptr(),
                                   rr.data_ptr() if which == "inner" else None, cnt.data_ptr(), m,
                                   occ.data_ptr(), None, feat.data_ptr(), flags, sp)
        if rc != 0:
            raise RuntimeError(L.nif_last_error().decode())

    def run_fused(v, obj, which):
        rc = L.nif_query_dev(v, obj.data_ptr(), ray.data_ptr(), c4.data_ptr(),
                             rr.data_ptr() if which == "inner" else None, cnt.data_ptr(), m,
                             occ.data_ptr(), None, _lib.IMPL_TCGEN05, sp)
        if rc != 0:
            raise RuntimeError(L.nif_last_error().decode())

    # ---- encoding kernel: resolution x objects x order ----------------------
    fams = a.fam.split(",")
    r_over = [int(x) for x in a.R.split(",")] if a.R else None
    for which, Rs in (("outer", (64, 128, 256, 512, 1024)), ("inner", (64, 128, 256))):
        if which not in fams:
            continue
        for R in (r_over or Rs):
            for n_obj in [int(x) for x in a.objs.split(",")]:
                cfg = NifConfig(seed=0)
                cfg.outer.grid_resolution = R
                cfg.inner.grid_resolution = R
                model = NifModel(cfg, n_obj)
                randomize(model)
                fam = model.family(which)
                v = fam.view(with_fast=True)
                obj_np = rng.integers(0, n_obj, m)
                for order in ("random", "sorted"):
                    o_np = np.sort(obj_np) if order == "sorted" else obj_np
                    obj = torch.from_numpy(o_np.astype(np.int32)).to(dev)
                    t = timeit(lambda: run_split(v, obj, which, 2), flush=flush)
                    rec_b = 20 if which == "outer" else 24
                    b = m * (rec_b + (12 if which == "outer" else 26))
                    bw = m * (rec_b + (16 if which == "outer" else 32))
                    N = fam.N
                    npad = 4 if N <= 4 else 8
                    table = n_obj * 2 * R * R * npad * 2
                    results["encode"].append({
                        "family": which, "R": R, "objects": n_obj, "order": order,
                        "us": t * 1e6, "records_per_s": m / t,
                        "achieved_GBps": b / t / 1e9, "frac_hbm": b / t / 1e9 / peaks["hbm_gbs"],
                        "written_GBps": bw / t / 1e9,
                        "frac_hbm_written": bw / t / 1e9 / peaks["hbm_gbs"],
                        "algorithmic_bytes": b, "table_bytes_fp16": table})
                    print(json.dumps(results["encode"][-1]), flush=True)
                del model
                torch.cuda.empty_cache()

    # ---- MLP kernel: width x depth (features from the encoding kernel) -------
    for which in (() if a.enc_only else ("outer", "inner")):
        for W in (64, 128):
            for Lh in (2, 3, 4):
                cfg = NifConfig(seed=0)
                cfg.outer.grid_resolution = 128
                cfg.inner.grid_resolution = 128
                for c in (cfg.outer, cfg.inner):
                    c.hidden_width = W
                    c.hidden_layers = Lh
                model = NifModel(cfg, 16)
                randomize(model)
                fam = model.family(which)
                v = fam.view(with_fast=True)
                obj = torch.from_numpy(rng.integers(0, 16, m).astype(np.int32)).to(dev)
                run_split(v, obj, which, 2)  # features
                t = timeit(lambda: run_split(v, obj, which, 4), flush=flush)
                IN = fam.dims[0]
                useful = 2 * (IN * W + (Lh - 1) * W * W + W)
                kp = ((W + 1) + 15) // 16 * 16
                executed = 2 * (16 * W + (Lh - 1) * kp * W)
                tf = m * useful / t / 1e12
                results["mlp"].append({
                    "family": which, "width": W, "hidden_layers": Lh, "us": t * 1e6,
                    "records_per_s": m / t, "useful_TFLOPs": tf,
                    "frac_tensor_peak": tf / peaks["bf16_tflops"],
                    "executed_mma_TFLOPs": m * executed / t / 1e12,
                    "executed_frac": m * executed / t / 1e12 / peaks["bf16_tflops"]})
                print(json.dumps(results["mlp"][-1]), flush=True)
                tfz = timeit(lambda: run_fused(v, obj, which), flush=flush)
                results["fused"].append({
                    "family": which, "width": W, "hidden_layers": Lh, "R": 128, "objects": 16,
                    "us": tfz * 1e6, "records_per_s": m / tfz,
                    "useful_TFLOPs": m * useful / tfz / 1e12,
                    "frac_tensor_peak": m * useful / tfz / 1e12 / peaks["bf16_tflops"]})
                print(json.dumps(results["fused"][-1]), flush=True)
                del model
                torch.cuda.empty_cache()
    if a.out:
        Path(a.out).write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
