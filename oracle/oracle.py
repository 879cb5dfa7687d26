"""TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.

CPU oracle for the NIF path: ctypes binding of nif_oracle.c (the fp64
kernels: gather, labels, BVH any-hit, sample pass, encode, dense forward)
plus a numpy restatement of the training step (mlp.py:82-167,
grids.py:31-56 / 153-202, nif.py:682-795). Only tests/, smoke() and the
cpu_baseline leg of bench.py may import this module; the product never
does. Pinned against golden vectors produced by the reference
(tests/golden/make_golden.py, test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None


def _build():
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
                    "-fopenmp", "-o", str(LIB), str(HERE / "nif_oracle.c"), "-lm"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists() or LIB.stat().st_mtime < (HERE / "nif_oracle.c").stat().st_mtime:
            _build()
        _lib = C.CDLL(str(LIB))
    return _lib


class OScene(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in (
        "t_lo", "t_hi", "t_a", "t_b", "t_leaf", "t_order", "roots", "b_lo", "b_hi", "b_a",
        "b_b", "b_leaf", "v0", "v1", "v2", "n0", "n1", "n2", "obox_lo", "obox_hi")] + [
        ("n_obj", C.c_int64), ("eps", C.c_double)]


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


class OracleScene:
    """Keeps contiguous copies of a ScenePack (reference layout) alive."""

    def __init__(self, pack, epsilon_t: float):
        keys = ("t_lo", "t_hi", "t_a", "t_b", "t_leaf", "t_order", "roots", "b_lo", "b_hi",
                "b_a", "b_b", "b_leaf", "v0", "v1", "v2", "n0", "n1", "n2", "obox_lo",
                "obox_hi")
        dt = {"t_a": np.int64, "t_b": np.int64, "t_order": np.int64, "roots": np.int64,
              "b_a": np.int64, "b_b": np.int64, "t_leaf": np.uint8, "b_leaf": np.uint8}
        self.arrays = {k: np.ascontiguousarray(getattr(pack, k), dt.get(k, np.float64))
                       for k in keys}
        self.s = OScene(**{k: _p(v).value for k, v in self.arrays.items()},
                        n_obj=len(self.arrays["roots"]), eps=float(epsilon_t))


def _c64(a):
    return np.ascontiguousarray(a, np.float64)


def gather(osc: OracleScene, origins, dirs, tmaxs, route, tol=1e-6):
    """renderer.py:613-644 gather_queries -> (kind, obj, ray, coord, bvh_occ, n_deg)."""
    o, d, t = _c64(origins), _c64(dirs), _c64(tmaxs)
    n = len(t)
    n_obj = int(osc.s.n_obj)
    kind = np.full(n * n_obj, 255, np.uint8)
    obj = np.zeros(n * n_obj, np.int32)
    ray = np.zeros(n * n_obj, np.int32)
    coord = np.zeros((n * n_obj, 5), np.float64)
    bvh_occ = np.zeros(n, np.uint8)
    n_deg = C.c_int64(0)
    route = np.ascontiguousarray(route, np.uint8)
    L = lib()
    L.oracle_gather(C.byref(osc.s), _p(route), _p(o), _p(d), _p(t), C.c_int64(n),
                    C.c_double(tol), _p(kind), _p(obj), _p(ray), _p(coord), _p(bvh_occ),
                    C.byref(n_deg))
    keep = kind != 255
    return kind[keep], obj[keep], ray[keep], coord[keep], bvh_occ.astype(bool), n_deg.value


def label_visible(osc: OracleScene, rec_obj, rec_ray, origins, dirs, tmaxs):
    """bvh.py:904-916: 1 = visible."""
    ro = np.ascontiguousarray(rec_obj, np.int32)
    rr = np.ascontiguousarray(rec_ray, np.int32)
    o, d, t = _c64(origins), _c64(dirs), _c64(tmaxs)
    vis = np.zeros(len(ro), np.uint8)
    lib().oracle_label_visible(C.byref(osc.s), _p(ro), _p(rr), C.c_int64(len(ro)), _p(o), _p(d),
                               _p(t), _p(vis))
    return vis


def bvh_occluded(osc: OracleScene, origins, dirs, tmaxs):
    o, d, t = _c64(origins), _c64(dirs), _c64(tmaxs)
    out = np.zeros(len(t), np.uint8)
    lib().oracle_occluded(C.byref(osc.s), _p(o), _p(d), _p(t), C.c_int64(len(t)), _p(out))
    return out.astype(bool)


def sample_pass(osc: OracleScene, camera, lights_cum, l_kind, l_data, seed, sample,
                sampler="importance"):
    fwd, right, up, tan_half, aspect = camera.basis()
    cam = np.ascontiguousarray(np.concatenate([camera.position, fwd, right, up,
                                               [tan_half, aspect]]), np.float64)
    n = camera.width * camera.height
    out = dict(hit=np.zeros(n, np.uint8), t=np.zeros(n), obj=np.zeros(n, np.int32),
               point=np.zeros((n, 3)), normal=np.zeros((n, 3)), pdir=np.zeros((n, 3)),
               ldir=np.zeros((n, 3)), tmax=np.zeros(n), pdf=np.zeros(n), emit=np.zeros((n, 3)))
    k = np.ascontiguousarray(l_kind, np.uint8)
    dd = np.ascontiguousarray(l_data, np.float64)
    cum = np.ascontiguousarray(lights_cum, np.float64)
    lib().oracle_sample_pass(
        C.byref(osc.s), _p(cam), C.c_int64(camera.width), C.c_int64(camera.height), _p(k),
        _p(dd), _p(cum), C.c_int64(len(cum)), C.c_uint64(seed), C.c_uint64(sample),
        C.c_int(0 if sampler == "importance" else 1), *[_p(out[q]) for q in (
            "hit", "t", "obj", "point", "normal", "pdir", "ldir", "tmax", "pdf", "emit")])
    out["hit"] = out["hit"].astype(bool)
    return out


def encode(pos, dirg, dist, obj, coord):
    """nif.py:286-311; pos/dir [n_obj,R,R,N] f32, dist [n_obj,Rd,Nd] or None."""
    pos = np.ascontiguousarray(pos, np.float32)
    dirg = np.ascontiguousarray(dirg, np.float32)
    R, N = pos.shape[1], pos.shape[3]
    Rd = Nd = 0
    if dist is not None:
        dist = np.ascontiguousarray(dist, np.float32)
        Rd, Nd = dist.shape[1], dist.shape[2]
    obj = np.ascontiguousarray(obj, np.int64)
    coord = _c64(coord)
    cw = coord.shape[1] if coord.ndim == 2 else 4
    out = np.zeros((len(obj), 2 * N + Nd), np.float64)
    lib().oracle_encode(_p(pos), _p(dirg), _p(dist), C.c_int64(R), C.c_int64(N), C.c_int64(Rd),
                        C.c_int64(Nd), _p(obj), _p(coord), C.c_int64(len(obj)), C.c_int64(cw),
                        _p(out))
    return out


def dense_forward(w_flat, b_flat, dims, x, sigmoid_head=1):
    """nif.py:321-359; returns f64[m, dims[-1]] (logits when sigmoid_head=0)."""
    w = np.ascontiguousarray(w_flat, np.float32)
    b = np.ascontiguousarray(b_flat, np.float32)
    dm = np.ascontiguousarray(dims, np.int64)
    x = _c64(x)
    out = np.zeros((len(x), int(dm[-1])), np.float64)
    if len(x):
        lib().oracle_dense_forward(_p(w), _p(b), _p(dm), C.c_int64(len(dm)), C.c_int(sigmoid_head),
                                   _p(x), C.c_int64(len(x)), _p(out))
    return out


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def set_threads(n: int) -> None:
    """OpenMP threads of the following oracle calls."""
    lib().oracle_set_threads(int(n))


# ---------------------------------------------------------------------------
# numpy restatement of the training step
# ---------------------------------------------------------------------------

SLOPE = 0.01  # mlp.py:17


@dataclass
class Adam:
    """grids.py:19-28 AdamParams."""
    learning_rate: float = 0.005
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-15
    step_count: int = 0


def int_power(a: float, e: int) -> float:
    """numba's float ** int (numba/cpython/numbers.py int_power_impl):
    binary exponentiation up to 0x10000, libm pow beyond."""
    if e > 0x10000:
        return math.pow(a, float(e))
    r = 1.0
    while e:
        if e & 1:
            r *= a
        e >>= 1
        a *= a
    return r


def adam_update(param, grad, m, v, p: Adam):
    """grids.py:31-56: fp64 moments over fp32 storage, bias corrected,
    gradient cleared. `b1 ** t` is numba's integer power."""
    p.step_count += 1
    t = p.step_count
    b1, b2, lr, eps = p.beta1, p.beta2, p.learning_rate, p.epsilon
    c1 = 1.0 - int_power(b1, t)
    c2 = 1.0 - int_power(b2, t)
    g = grad.astype(np.float64)
    mi = b1 * m.astype(np.float64) + (1.0 - b1) * g
    vi = b2 * v.astype(np.float64) + (1.0 - b2) * g * g
    m[...] = mi
    v[...] = vi
    mh = mi / c1
    vh = vi / c2
    param[...] = param.astype(np.float64) - lr * mh / (np.sqrt(vh) + eps)
    grad[...] = 0.0


class OLayer:
    def __init__(self, w, b):
        self.w = np.array(w, np.float32)
        self.b = np.array(b, np.float32)
        self.gw = np.zeros_like(self.w)
        self.gb = np.zeros_like(self.b)
        self.mw = np.zeros_like(self.w)
        self.vw = np.zeros_like(self.w)
        self.mb = np.zeros_like(self.b)
        self.vb = np.zeros_like(self.b)
        self.adam_w = Adam()
        self.adam_b = Adam()


def _leaky(z):
    return np.where(z > 0, z, z * np.float32(SLOPE))


def _sigmoid(x):
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


class OMlp:
    """mlp.py:50-129 restated."""

    def __init__(self, layers: List[OLayer], sigmoid_head=True):
        self.layers = layers
        self.sigmoid_head = sigmoid_head
        self._cache = None

    def forward(self, x):
        x = np.ascontiguousarray(x, np.float32)
        inputs, pres = [x], []
        a = x
        last = len(self.layers) - 1
        for i, l in enumerate(self.layers):
            z = a @ l.w.T + l.b
            pres.append(z)
            if i < last:
                a = _leaky(z)
                inputs.append(a)
            elif self.sigmoid_head:
                a = _sigmoid(z)
            else:
                a = z
        self._cache = (inputs, pres, a)
        return a

    def backward(self, up):
        inputs, pres, out = self._cache
        up = np.asarray(up, np.float32)
        dz = up * out * (1.0 - out) if self.sigmoid_head else up
        slope = np.float32(SLOPE)
        for i in range(len(self.layers) - 1, -1, -1):
            l = self.layers[i]
            l.gw += dz.T @ inputs[i]
            l.gb += dz.sum(axis=0)
            dx = dz @ l.w
            if i > 0:
                dz = np.where(pres[i - 1] > 0, dx, dx * slope)
        return dx

    def adam_step(self):
        for l in self.layers:
            adam_update(l.w, l.gw, l.mw, l.vw, l.adam_w)
            adam_update(l.b, l.gb, l.mb, l.vb, l.adam_b)


def l2_loss(pred, target):
    """mlp.py:159-167."""
    target = np.asarray(target, pred.dtype)
    diff = pred - target
    loss = float(np.mean(np.square(diff, dtype=np.float64)))
    return loss, diff * pred.dtype.type(2.0 / diff.size)


class OGrid:
    def __init__(self, latents, wrap_u=True):
        self.latents = np.array(latents, np.float32)
        self.grad = np.zeros_like(self.latents)
        self.m = np.zeros_like(self.latents)
        self.v = np.zeros_like(self.latents)
        self.adam = Adam()
        self.wrap_u = wrap_u
        self.R = self.latents.shape[0]


def _axis(x, R, wrap):
    xc = x * R - 0.5
    x0 = np.floor(xc)
    w = xc - x0
    i0 = x0.astype(np.int64)
    i1 = i0 + 1
    if wrap:
        i0, i1 = i0 % R, i1 % R
    else:
        i0, i1 = np.clip(i0, 0, R - 1), np.clip(i1, 0, R - 1)
    return i0, i1, w


def _bil(g: OGrid, uv):
    u = np.asarray(uv[:, 0], np.float64)
    v = np.asarray(uv[:, 1], np.float64)
    iu0, iu1, wu = _axis(u, g.R, True)
    iv0, iv1, wv = _axis(v, g.R, False)
    return (iu0, iu1, iv0, iv1), ((1.0 - wu) * (1.0 - wv), (1.0 - wu) * wv, wu * (1.0 - wv), wu * wv)


def lookup_2d(g: OGrid, uv):
    (iu0, iu1, iv0, iv1), (w00, w01, w10, w11) = _bil(g, uv)
    L = g.latents
    out = (w00[:, None] * L[iu0, iv0] + w01[:, None] * L[iu0, iv1]
           + w10[:, None] * L[iu1, iv0] + w11[:, None] * L[iu1, iv1])
    return out.astype(np.float32)


def grad_2d(g: OGrid, uv, up):
    (iu0, iu1, iv0, iv1), (w00, w01, w10, w11) = _bil(g, uv)
    up = np.asarray(up, np.float64)
    np.add.at(g.grad, (iu0, iv0), (w00[:, None] * up).astype(np.float32))
    np.add.at(g.grad, (iu0, iv1), (w01[:, None] * up).astype(np.float32))
    np.add.at(g.grad, (iu1, iv0), (w10[:, None] * up).astype(np.float32))
    np.add.at(g.grad, (iu1, iv1), (w11[:, None] * up).astype(np.float32))


def lookup_1d(g: OGrid, x):
    i0, i1, w = _axis(np.asarray(x, np.float64), g.R, False)
    L = g.latents
    return ((1.0 - w)[:, None] * L[i0] + w[:, None] * L[i1]).astype(np.float32)


def grad_1d(g: OGrid, x, up):
    i0, i1, w = _axis(np.asarray(x, np.float64), g.R, False)
    up = np.asarray(up, np.float64)
    np.add.at(g.grad, i0, ((1.0 - w)[:, None] * up).astype(np.float32))
    np.add.at(g.grad, i1, (w[:, None] * up).astype(np.float32))


class OModel:
    """The trainable state of a NifModel (shared MLPs), restated."""

    def __init__(self, outer_layers, inner_layers, grids, lr=0.005, beta1=0.9, beta2=0.999,
                 eps=1e-15):
        self.outer = OMlp([OLayer(w, b) for w, b in outer_layers])
        self.inner = OMlp([OLayer(w, b) for w, b in inner_layers])
        self.grids = [{k: OGrid(v, wrap_u=(k != "inner_dist")) for k, v in g.items()}
                      for g in grids]
        for mlp in (self.outer, self.inner):
            for l in mlp.layers:
                for p in (l.adam_w, l.adam_b):
                    p.learning_rate, p.beta1, p.beta2, p.epsilon = lr, beta1, beta2, eps
        for g in self.grids:
            for gr in g.values():
                gr.adam = Adam(lr, beta1, beta2, eps)

    def train_batch(self, which, obj, coord, label, apply=True) -> float:
        """nif.py:682-749 _train_batch (shared sharing mode). apply=False
        stops before the Adam updates (gradients left in the .grad arrays)."""
        order = np.argsort(obj, kind="stable")
        obj, coord, label = obj[order], coord[order], label[order]
        bounds = np.flatnonzero(np.diff(obj)) + 1
        starts = np.concatenate([[0], bounds])
        stops = np.concatenate([bounds, [len(obj)]])
        total = 0.0
        touched = []
        mlp = self.outer if which == "outer" else self.inner
        for a, b in zip(starts, stops):
            o = int(obj[a])
            g = self.grids[o]
            touched.append(o)
            uv_p, uv_d = coord[a:b, 0:2], coord[a:b, 2:4]
            if which == "outer":
                n_lat = g["outer_pos"].latents.shape[2]
                x = np.concatenate([lookup_2d(g["outer_pos"], uv_p),
                                    lookup_2d(g["outer_dir"], uv_d)], axis=1)
            else:
                n_lat = g["inner_pos"].latents.shape[2]
                r = coord[a:b, 4]
                x = np.concatenate([lookup_2d(g["inner_pos"], uv_p),
                                    lookup_2d(g["inner_dir"], uv_d),
                                    lookup_1d(g["inner_dist"], r)], axis=1)
            tgt = label[a:b]
            if tgt.ndim == 1:
                tgt = tgt[:, None]
            pred = mlp.forward(x.astype(np.float32))
            loss, gout = l2_loss(pred, tgt.astype(pred.dtype))
            gx = mlp.backward(gout)
            if which == "outer":
                grad_2d(g["outer_pos"], uv_p, gx[:, :n_lat])
                grad_2d(g["outer_dir"], uv_d, gx[:, n_lat:2 * n_lat])
            else:
                grad_2d(g["inner_pos"], uv_p, gx[:, :n_lat])
                grad_2d(g["inner_dir"], uv_d, gx[:, n_lat:2 * n_lat])
                grad_1d(g["inner_dist"], r, gx[:, 2 * n_lat:])
            total += loss * (b - a)
        if not apply:
            return total / len(obj)
        for o in touched:
            g = self.grids[o]
            names = ("outer_pos", "outer_dir") if which == "outer" else (
                "inner_pos", "inner_dir", "inner_dist")
            for nm in names:
                gr = g[nm]
                adam_update(gr.latents, gr.grad, gr.m, gr.v, gr.adam)
        mlp.adam_step()
        return total / len(obj)

    def train(self, samples, epochs, seed, bo=2 ** 11, bi=2 ** 12):
        """nif.py:752-795 train (epoch RNG and family order restated)."""
        curve = np.zeros((epochs, 3))
        if epochs == 0:
            return curve
        epoch_ss = np.random.SeedSequence([seed, 0x7472]).spawn(epochs)
        for e in range(epochs):
            rng = np.random.default_rng(epoch_ss[e])
            sums = np.zeros(2)
            counts = np.zeros(2, np.int64)
            for fam, bs, (obj, coord, label) in (
                    (0, bo, (samples["outer_obj"], samples["outer_coord"], samples["outer_label"])),
                    (1, bi, (samples["inner_obj"], samples["inner_coord"], samples["inner_label"]))):
                n = len(obj)
                if n == 0:
                    continue
                perm = rng.permutation(n)
                which = "outer" if fam == 0 else "inner"
                for k in range(0, n, bs):
                    idx = perm[k:k + bs]
                    loss = self.train_batch(which, obj[idx], coord[idx], label[idx])
                    sums[fam] += loss * len(idx)
                    counts[fam] += len(idx)
            om = sums[0] / counts[0] if counts[0] else math.nan
            im = sums[1] / counts[1] if counts[1] else math.nan
            curve[e] = (om, im, sums.sum() / counts.sum())
        return curve
