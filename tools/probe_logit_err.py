"""Max |logit - oracle| of the fused query variants on the bench's C2 frame
with O(1) logits (latents U(-1,1), biases U(-0.5,0.5)) and with a model
trained one epoch -- the bars of tests/test_gpu_bench_parity.py, per
nif_debug_set_query_variant.

    python tools/probe_logit_err.py [variants, default 0] [--long]
"""
import importlib
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2306_07191_b200 import _lib, build_model, synthetic  # noqa: E402
from paper_2306_07191_b200.nif import NifConfig  # noqa: E402
from paper_2306_07191_b200.pipeline import (VisibilityEngine, sample_pass_dev,  # noqa: E402
                                            shadow_rays_dev)
from test_gpu_bench_parity import _compare, _hot_path  # noqa: E402
from test_gpu_mlp import _randomize  # noqa: E402

def _binned(scene, model, rays, hot):
    """max |dlogit| per |logit_ref| bin, per family (records matched by (ray, obj))."""
    from oracle import oracle
    from test_gpu_bench_parity import _oracle_family
    o, d, t = rays
    osc = oracle.OracleScene(scene.pack, scene.epsilon_t)
    kind, obj, ray, coord, _, _ = oracle.gather(osc, o, d, t, scene.nif_route_mask(None))
    out = {}
    for fam, k, width in (("outer", 0, 4), ("inner", 1, 5)):
        sel = kind == k
        r_obj, r_ray = obj[sel].astype(np.int64), ray[sel].astype(np.int64)
        f = _oracle_family(model, fam)
        x = oracle.encode(f["pos"], f["dir"], f["dist"], r_obj, coord[sel, :width])
        ref = oracle.dense_forward(f["w"], f["b"], f["dims"], x, sigmoid_head=0)[:, 0]
        h = hot[fam]
        nob = scene.n_objects
        kr, kh = r_ray * nob + r_obj, h["ray"] * nob + h["obj"]
        orr, oh = np.argsort(kr, kind="stable"), np.argsort(kh, kind="stable")
        refs, got = ref[orr], h["logit"][oh].astype(np.float64)
        err = np.abs(got - refs)
        a = np.abs(refs)
        bins = [0, 0.1, 1, 3, 10, 1e9]
        out[fam] = {f"<{hi:g}": [float(err[(a >= lo) & (a < hi)].max(initial=0)),
                                int(((a >= lo) & (a < hi)).sum())]
                    for lo, hi in zip(bins[:-1], bins[1:])}
        out[fam]["max_abs_logit"] = float(a.max(initial=0))
    return out


torch.cuda.set_device(0)
args = [a for a in sys.argv[1:] if not a.startswith("--")]
variants = [int(v) for v in (args[0] if args else "0").split(",")]
scene = synthetic.c2(build_device=torch.device("cuda", 0))
data = sample_pass_dev(scene, scene.camera, 0, scene.seed)
_, o, d, t = shadow_rays_dev(data, require_emit=False)
n = int(t.numel())
rays = (o.cpu().numpy(), d.cpu().numpy(), t.cpu().numpy())
models = {}
m = build_model(NifConfig(seed=0), scene)
_randomize(m, seed=11)
models["random O(1)"] = m
tr = importlib.import_module("paper_2306_07191_b200.train")
m2 = build_model(NifConfig(seed=0), scene)
tr.train(m2, tr.collect_samples(scene, spp=1, seed=scene.seed), epochs=1)
models["trained 1 epoch"] = m2
if "--long" in sys.argv:
    m3 = build_model(NifConfig(seed=0), scene)
    tr.train(m3, tr.collect_samples(scene, spp=4, seed=scene.seed), epochs=10)
    models["trained 10 epochs on 4 spp"] = m3
    g = [np.abs(a).max() for a in m3.model_arrays()]
    print(json.dumps({"max_abs_param_10ep": float(max(g))}), flush=True)
for name, model in models.items():
    eng = VisibilityEngine(scene, model, n)
    eng.origins[:n].copy_(o)
    eng.dirs[:n].copy_(d)
    eng.tmaxs[:n].copy_(t)
    for v in variants:
        _lib.lib().nif_debug_set_query_variant(v)
        hot = _hot_path(eng, n)
        binned = _binned(scene, model, rays, hot)
        print(json.dumps({"model": name, "variant": v, "error_by_abs_logit": binned}), flush=True)
        try:
            s = _compare(scene, model, rays, hot)
        except AssertionError as e:
            print(json.dumps({"model": name, "variant": v, "fails_2e-2": str(e)[:200]}), flush=True)
            continue
        print(json.dumps({"model": name, "variant": v, "outer_max_err": s["outer"]["max_logit_err"],
                          "inner_max_err": s["inner"]["max_logit_err"],
                          "agreement": s["agreement"], "undecided": s["undecided_rays"]}),
              flush=True)
    _lib.lib().nif_debug_set_query_variant(0)
