"""Learned secondary-ray visibility on the B200: configuration, the
HBM-resident model, and the reference's array/record inference API.

Drop-in for pkg/src/niftrace/nif.py (names, argument meaning, error
types and messages follow the reference): NifConfig / OuterConfig /
InnerConfig (nif.py:59-156), NifModel (nif.py:173-255, identical seeded
initialisation), encode_*_arrays (286-311), forward_*_arrays (380-397),
infer_records (467-483), infer_occlusion (428-442), NifBackend (486-499).

All parameters live in HBM as fp32 masters (torch tensors, one flat
allocation per family) beside their Adam state; the fused query kernel
reads an fp16 "fast blob" (canonical UMMA weight tiles + fp16 latent
tables) re-packed on demand after every optimizer step.
"""

from __future__ import annotations

import math
from dataclasses import asdict, dataclass, field
from typing import List, Optional, Sequence, Union

import numpy as np

from . import _lib

# ---------------------------------------------------------------------------
# configuration (nif.py:59-156, grids.py:19-28)
# ---------------------------------------------------------------------------


@dataclass
class AdamParams:
    learning_rate: float = 0.005
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-15
    step_count: int = 0


@dataclass
class OuterConfig:
    hidden_layers: int = 2
    hidden_width: int = 64
    grid_resolution: int = 256
    grid_latents: int = 3
    batch_size: int = 2 ** 11

    @property
    def input_dim(self) -> int:
        return 2 * self.grid_latents


@dataclass
class InnerConfig:
    hidden_layers: int = 3
    hidden_width: int = 48
    grid_resolution: int = 128
    grid_latents: int = 5
    dist_resolution: int = 128
    dist_latents: int = 3
    batch_size: int = 2 ** 12

    @property
    def input_dim(self) -> int:
        return 2 * self.grid_latents + self.dist_latents


SHARING_MODES = ("shared", "per_object")
HEAD_MODES = ("occlusion", "geometry")


@dataclass
class NifConfig:
    outer: OuterConfig = field(default_factory=OuterConfig)
    inner: InnerConfig = field(default_factory=InnerConfig)
    learning_rate: float = 0.005
    adam: AdamParams = field(default_factory=AdamParams)
    epochs: int = 30
    sharing: str = "shared"
    head: str = "occlusion"
    seed: int = 0

    def __post_init__(self):
        for blk in (self.outer, self.inner):
            if blk.hidden_layers < 1 or blk.hidden_width < 1:
                raise ValueError("network depth and width must be at least 1")
            if blk.grid_resolution < 1 or blk.grid_latents < 1:
                raise ValueError("grid resolution and latent count must be at least 1")
            if blk.batch_size < 1:
                raise ValueError("batch size must be at least 1")
        if self.inner.dist_resolution < 1 or self.inner.dist_latents < 1:
            raise ValueError("distance grid sizes must be at least 1")
        if self.sharing not in SHARING_MODES:
            raise ValueError(f"sharing must be one of {SHARING_MODES}")
        if self.head not in HEAD_MODES:
            raise ValueError(f"head must be one of {HEAD_MODES}")
        if not (self.learning_rate > 0):
            raise ValueError("learning rate must be positive")
        if self.epochs < 0:
            raise ValueError("epoch count cannot be negative")

    @property
    def head_dim(self) -> int:
        return 1 if self.head == "occlusion" else 4

    @property
    def head_activation(self) -> str:
        return "sigmoid" if self.head == "occlusion" else "identity"

    def to_dict(self) -> dict:
        d = asdict(self)
        d["adam"] = {"learning_rate": self.adam.learning_rate, "beta1": self.adam.beta1,
                     "beta2": self.adam.beta2, "epsilon": self.adam.epsilon}
        return d

    @staticmethod
    def from_dict(d: dict) -> "NifConfig":
        adam = dict(d.get("adam", {}))
        adam.pop("step_count", None)
        return NifConfig(outer=OuterConfig(**d["outer"]), inner=InnerConfig(**d["inner"]),
                         learning_rate=d["learning_rate"], adam=AdamParams(**adam),
                         epochs=d["epochs"], sharing=d["sharing"], head=d["head"],
                         seed=d["seed"])


# ---------------------------------------------------------------------------
# seeded initialisation, restating nif.py:181-223 / mlp.py:142-156 /
# grids.py:99-117 with the same SeedSequence tree and PCG64 draws
# ---------------------------------------------------------------------------

INIT_SCALE = 1e-4  # grids.py:99


def _xavier(dims, seed) -> List[tuple]:
    rng = np.random.Generator(np.random.PCG64(seed))
    layers = []
    for i in range(len(dims) - 1):
        n_in, n_out = dims[i], dims[i + 1]
        limit = np.sqrt(6.0 / (n_in + n_out))
        w = rng.uniform(-limit, limit, (n_out, n_in)).astype(np.float32)
        layers.append((w, np.zeros(n_out, np.float32)))
    return layers


def _grid_init(shape, seed) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-INIT_SCALE, INIT_SCALE, shape).astype(np.float32)


def init_arrays(config: NifConfig, n_objects: int):
    """Host arrays of a freshly built reference NifModel:
    (outer_layers[heads], inner_layers[heads], grids[objects])."""
    root = np.random.SeedSequence(config.seed)
    mlp_ss, grid_ss = root.spawn(2)
    n_heads = 1 if config.sharing == "shared" else n_objects
    children = mlp_ss.spawn(2 * n_heads)
    o, i = config.outer, config.inner
    odims = [o.input_dim] + [o.hidden_width] * o.hidden_layers + [config.head_dim]
    idims = [i.input_dim] + [i.hidden_width] * i.hidden_layers + [config.head_dim]
    outer = [_xavier(odims, children[2 * h]) for h in range(n_heads)]
    inner = [_xavier(idims, children[2 * h + 1]) for h in range(n_heads)]
    grids = []
    for obj_ss in grid_ss.spawn(n_objects):
        s = obj_ss.spawn(5)
        grids.append({
            "outer_pos": _grid_init((o.grid_resolution, o.grid_resolution, o.grid_latents), s[0]),
            "outer_dir": _grid_init((o.grid_resolution, o.grid_resolution, o.grid_latents), s[1]),
            "inner_pos": _grid_init((i.grid_resolution, i.grid_resolution, i.grid_latents), s[2]),
            "inner_dir": _grid_init((i.grid_resolution, i.grid_resolution, i.grid_latents), s[3]),
            "inner_dist": _grid_init((i.dist_resolution, i.dist_latents), s[4]),
        })
    return outer, inner, grids, odims, idims


# ---------------------------------------------------------------------------
# device model
# ---------------------------------------------------------------------------

FAMILIES = ("outer", "inner")


class FamilyParams:
    """One network family in HBM.

    ``params`` is a single flat fp32 tensor [pos | dir | dist | w | b] so the
    optimizer, the gradient all-reduce and checkpointing see one buffer;
    ``grad``, ``m`` and ``v`` mirror it element for element.
    """

    def __init__(self, which, dims, R, N, Rd, Nd, n_obj, n_heads, sigmoid_head, device):
        import torch
        self.which = which
        self.family = 0 if which == "outer" else 1
        self.dims = list(dims)
        self.R, self.N, self.Rd, self.Nd = R, N, Rd, Nd
        self.n_obj, self.n_heads = n_obj, n_heads
        self.sigmoid_head = sigmoid_head
        self.w_stride = sum(dims[k] * dims[k + 1] for k in range(len(dims) - 1))
        self.b_stride = sum(dims[k + 1] for k in range(len(dims) - 1))
        g2 = n_obj * R * R * N
        g1 = n_obj * Rd * Nd
        sizes = {"pos": g2, "dir": g2, "dist": g1, "w": n_heads * self.w_stride,
                 "b": n_heads * self.b_stride}
        self.offsets = {}
        off = 0
        for k in ("pos", "dir", "dist", "w", "b"):
            self.offsets[k] = (off, sizes[k])
            off += (sizes[k] + 63) // 64 * 64
        self.numel = off
        self.device = device
        self.params = torch.zeros(off, dtype=torch.float32, device=device)
        self.grad = torch.zeros_like(self.params)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        # per-tensor Adam step counters (device): one per object grid set,
        # one per head MLP; batch row counts per object
        self.grid_steps = torch.zeros(n_obj, dtype=torch.int64, device=device)
        self.mlp_steps = torch.zeros(n_heads, dtype=torch.int64, device=device)
        self.counts = torch.zeros(n_obj, dtype=torch.int32, device=device)
        self._fast = None
        self.dirty = True

    def train_view(self):
        t = _lib.TrainView()
        t.params = _lib.ptr(self.params)
        t.grad = _lib.ptr(self.grad)
        t.m = _lib.ptr(self.m)
        t.v = _lib.ptr(self.v)
        t.numel = self.numel
        t.off_pos = self.offsets["pos"][0]
        t.off_dir = self.offsets["dir"][0]
        t.off_dist = self.offsets["dist"][0]
        t.off_w = self.offsets["w"][0]
        t.off_b = self.offsets["b"][0]
        t.grid_steps = _lib.ptr(self.grid_steps)
        t.mlp_steps = _lib.ptr(self.mlp_steps)
        t.counts = _lib.ptr(self.counts)
        return t

    def part(self, key, t=None):
        off, size = self.offsets[key]
        return (self.params if t is None else t)[off:off + size]

    @property
    def pos(self):
        return self.part("pos").view(self.n_obj, self.R, self.R, self.N)

    @property
    def dir(self):
        return self.part("dir").view(self.n_obj, self.R, self.R, self.N)

    @property
    def dist(self):
        if self.family == 0:
            return None
        return self.part("dist").view(self.n_obj, self.Rd, self.Nd)

    def view(self, with_fast=False):
        v = _lib.FamilyView()
        v.family = self.family
        v.n_obj = self.n_obj
        v.R, v.N = self.R, self.N
        v.Rd, v.Nd = (self.Rd, self.Nd) if self.family == 1 else (0, 0)
        v.n_layers = len(self.dims) - 1
        for k, d in enumerate(self.dims):
            v.dims[k] = d
        v.n_heads = self.n_heads
        v.sigmoid_head = self.sigmoid_head
        v.w_stride, v.b_stride = self.w_stride, self.b_stride
        v.pos = _lib.ptr(self.part("pos"))
        v.dir = _lib.ptr(self.part("dir"))
        v.dist = _lib.ptr(self.part("dist")) if self.family == 1 else None
        v.w = _lib.ptr(self.part("w"))
        v.b = _lib.ptr(self.part("b"))
        v.fast = _lib.ptr(self.fast_blob()) if with_fast else None
        return v

    def fast_blob(self):
        """fp16 tables + canonical weight tiles, rebuilt after updates."""
        import torch
        if self._fast is None or self.dirty:
            L = _lib.lib()
            v = self.view(with_fast=False)
            nbytes = L.nif_fast_pack_bytes(v)
            if self._fast is None or self._fast.numel() != nbytes:
                self._fast = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            L.nif_fast_pack_dev(v, _lib.ptr(self._fast), _lib.stream_ptr())
            self.dirty = False
        return self._fast


class NifModel:
    """Per-object grids plus the outer/inner networks, resident in HBM
    (nif.py:173-255). Initialisation is bit-identical to the reference for
    the same config/seed."""

    def __init__(self, config: NifConfig, n_objects: int, scene_diagonal: float = 1.0,
                 dtype=np.float32, device=None):
        import torch
        if n_objects < 1:
            raise ValueError("a model needs at least one object")
        if np.dtype(dtype) != np.float32:
            raise ValueError("the B200 engine stores fp32 master parameters")
        self.config = config
        self.n_objects = n_objects
        self.scene_diagonal = float(scene_diagonal)
        self.dtype = np.dtype(np.float32)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        outer, inner, grids, odims, idims = init_arrays(config, n_objects)
        n_heads = 1 if config.sharing == "shared" else n_objects
        sig = 1 if config.head == "occlusion" else 0
        o, i = config.outer, config.inner
        self.outer = FamilyParams("outer", odims, o.grid_resolution, o.grid_latents, 0, 0,
                                  n_objects, n_heads, sig, self.device)
        self.inner = FamilyParams("inner", idims, i.grid_resolution, i.grid_latents,
                                  i.dist_resolution, i.dist_latents, n_objects, n_heads, sig,
                                  self.device)
        self.load_arrays(outer, inner, grids)
        self.set_learning_rate(config.learning_rate)

    # -- host <-> device -------------------------------------------------------
    def family(self, which: str) -> FamilyParams:
        return self.outer if which == "outer" else self.inner

    def load_arrays(self, outer_layers, inner_layers, grids):
        import torch
        for fam, heads, keys in ((self.outer, outer_layers, ("outer_pos", "outer_dir", None)),
                                 (self.inner, inner_layers,
                                  ("inner_pos", "inner_dir", "inner_dist"))):
            host = np.zeros(fam.numel, np.float32)

            def put(key, arr):
                off, size = fam.offsets[key]
                host[off:off + size] = np.asarray(arr, np.float32).reshape(-1)

            put("pos", np.stack([g[keys[0]] for g in grids]))
            put("dir", np.stack([g[keys[1]] for g in grids]))
            if keys[2]:
                put("dist", np.stack([g[keys[2]] for g in grids]))
            put("w", np.stack([np.concatenate([w.reshape(-1) for w, _ in h]) for h in heads]))
            put("b", np.stack([np.concatenate([b for _, b in h]) for h in heads]))
            fam.params.copy_(torch.from_numpy(host).to(fam.device))
            fam.dirty = True

    def host_layers(self, which: str):
        """[(w, b) per layer] per head, as numpy (reference Mlp layout)."""
        fam = self.family(which)
        w = fam.part("w").detach().cpu().numpy().reshape(fam.n_heads, fam.w_stride)
        b = fam.part("b").detach().cpu().numpy().reshape(fam.n_heads, fam.b_stride)
        heads = []
        for h in range(fam.n_heads):
            layers, wo, bo = [], 0, 0
            for k in range(len(fam.dims) - 1):
                nin, nout = fam.dims[k], fam.dims[k + 1]
                layers.append((w[h, wo:wo + nin * nout].reshape(nout, nin).copy(),
                               b[h, bo:bo + nout].copy()))
                wo += nin * nout
                bo += nout
            heads.append(layers)
        return heads

    def host_grids(self):
        o, i = self.outer, self.inner
        op, od = o.pos.cpu().numpy(), o.dir.cpu().numpy()
        ip, idr, idi = i.pos.cpu().numpy(), i.dir.cpu().numpy(), i.dist.cpu().numpy()
        return [{"outer_pos": op[k], "outer_dir": od[k], "inner_pos": ip[k], "inner_dir": idr[k],
                 "inner_dist": idi[k]} for k in range(self.n_objects)]

    def model_arrays(self):
        """Arrays in the NIF1 checkpoint order (scene_io.py:312-323)."""
        out = []
        for h in range(self.outer.n_heads):
            for w, b in self.host_layers("outer")[h]:
                out += [w, b]
        for h in range(self.inner.n_heads):
            for w, b in self.host_layers("inner")[h]:
                out += [w, b]
        for g in self.host_grids():
            out += [g["outer_pos"], g["outer_dir"], g["inner_pos"], g["inner_dir"],
                    g["inner_dist"]]
        return out

    def _check_object(self, object_id: int):
        if not (0 <= object_id < self.n_objects):
            raise ValueError(f"object {object_id} has no grids "
                             f"(model covers {self.n_objects})")

    def set_learning_rate(self, lr: float):
        self.learning_rate = float(lr)

    def n_parameters(self) -> int:
        total = 0
        for fam in (self.outer, self.inner):
            total += fam.n_heads * (fam.w_stride + fam.b_stride)
            total += 2 * fam.n_obj * fam.R * fam.R * fam.N
            if fam.family == 1:
                total += fam.n_obj * fam.Rd * fam.Nd
        return total

    def mark_dirty(self):
        self.outer.dirty = True
        self.inner.dirty = True


def build_model(config: NifConfig, scene, dtype=np.float32, device=None) -> NifModel:
    return NifModel(config, scene.n_objects, scene.diagonal, dtype, device)


# ---------------------------------------------------------------------------
# array API (exact: fp64 interpolation weights / fp64 accumulation)
# ---------------------------------------------------------------------------


def _to_dev(a, dtype, device):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype)).to(device)


def _encode(model: NifModel, which: str, obj, coord) -> np.ndarray:
    import torch
    fam = model.family(which)
    obj = np.asarray(obj, np.int64)
    width = 4 if which == "outer" else 5
    coord = np.asarray(coord, np.float64).reshape(-1, width) if len(obj) else np.zeros((0, width))
    out = np.empty((len(obj), fam.dims[0]), np.float64)
    if len(obj) == 0:
        return out
    for o in np.unique(obj):
        model._check_object(int(o))
    d_obj = _to_dev(obj, np.int64, model.device)
    d_coord = _to_dev(coord, np.float64, model.device)
    d_out = torch.empty((len(obj), fam.dims[0]), dtype=torch.float64, device=model.device)
    _lib.lib().nif_encode_dev(fam.view(), _lib.ptr(d_obj), _lib.ptr(d_coord), len(obj),
                              _lib.ptr(d_out), _lib.stream_ptr())
    return d_out.cpu().numpy()


def encode_outer_arrays(model: NifModel, obj, coord) -> np.ndarray:
    """nif.py:286-296; coord columns (p_u, p_v, d_u, d_v)."""
    return _encode(model, "outer", obj, coord)


def encode_inner_arrays(model: NifModel, obj, coord) -> np.ndarray:
    """nif.py:299-311; coord columns (p_u, p_v, d_u, d_v, r)."""
    return _encode(model, "inner", obj, coord)


def _forward(model: NifModel, which: str, obj, x, sigmoid_head=None) -> np.ndarray:
    import torch
    fam = model.family(which)
    x = np.asarray(x, np.float64)
    m = len(x)
    od = fam.dims[-1]
    if m == 0:
        return np.empty((0, od), np.float64)
    obj = np.zeros(m, np.int64) if obj is None else np.asarray(obj, np.int64)
    head = fam.sigmoid_head if sigmoid_head is None else int(sigmoid_head)
    d_x = _to_dev(x.reshape(m, fam.dims[0]), np.float64, model.device)
    d_obj = _to_dev(obj, np.int64, model.device)
    d_out = torch.empty((m, od), dtype=torch.float64, device=model.device)
    _lib.lib().nif_forward_dev(fam.view(), _lib.ptr(d_obj), _lib.ptr(d_x), m, head,
                               _lib.ptr(d_out), _lib.stream_ptr())
    return d_out.cpu().numpy()


def forward_outer_arrays(model: NifModel, obj, x) -> np.ndarray:
    """nif.py:380-387: probabilities (sigmoid head) per row."""
    return _forward(model, "outer", obj, x)


def forward_inner_arrays(model: NifModel, obj, x) -> np.ndarray:
    """nif.py:390-397."""
    return _forward(model, "inner", obj, x)


def logits_arrays(model: NifModel, which: str, obj, x) -> np.ndarray:
    """The reference's _k_dense_forward with sigmoid_head=0 (pre-sigmoid)."""
    return _forward(model, which, obj, x, sigmoid_head=0)


# ---------------------------------------------------------------------------
# record / query inference through the fused query kernels
# ---------------------------------------------------------------------------


def query_family(model: NifModel, which: str, obj, coord, impl: int = _lib.IMPL_AUTO,
                 want_logits: bool = True, split: bool = False):
    """Run the fused encode+MLP kernel over host records; returns fp32
    logits (pre-sigmoid). impl selects tcgen05 / SIMT (AUTO = tcgen05 when
    the configuration is covered). split=True runs the two-kernel variant
    (standalone grid encoding, then the tcgen05 MLP over its features)."""
    import torch
    fam = model.family(which)
    obj = np.asarray(obj, np.int64)
    m = len(obj)
    if m == 0:
        return np.zeros(0, np.float32)
    for o in np.unique(obj):
        model._check_object(int(o))
    coord = np.asarray(coord, np.float64)
    dev = model.device
    d_obj = _to_dev(obj, np.int32, dev)
    d_ray = torch.zeros(m, dtype=torch.int32, device=dev)
    d_c4 = _to_dev(coord[:, 0:4], np.float32, dev)
    d_r = _to_dev(coord[:, 4], np.float32, dev) if which == "inner" else None
    d_cnt = torch.tensor([m], dtype=torch.int64, device=dev)
    d_log = torch.empty(m * fam.dims[-1], dtype=torch.float32, device=dev)
    if fam.n_heads > 1 and fam.dims[-1] != 1 and impl == _lib.IMPL_AUTO:
        impl = _lib.IMPL_SIMT  # per-object geometry heads: no bucketed 4-wide kernel
    if fam.n_heads > 1 and impl in (_lib.IMPL_AUTO, _lib.IMPL_TCGEN05) and not split:
        # per_object sharing: bucket by object, then the tensor-core kernel
        L = _lib.lib()
        scratch = torch.zeros(int(L.nif_bucket_scratch_bytes(m, fam.n_obj)), dtype=torch.uint8,
                              device=dev)
        L.nif_query_bucketed_dev(fam.view(with_fast=True), _lib.ptr(d_obj), _lib.ptr(d_ray),
                                 _lib.ptr(d_c4), _lib.ptr(d_r), _lib.ptr(d_cnt), m, None,
                                 _lib.ptr(d_log), _lib.ptr(scratch), _lib.stream_ptr())
    elif split:
        L = _lib.lib()
        feat = torch.empty(int(L.nif_feat_scratch_bytes(m)), dtype=torch.uint8, device=dev)
        L.nif_query_split_dev(fam.view(with_fast=True), _lib.ptr(d_obj), _lib.ptr(d_ray),
                              _lib.ptr(d_c4), _lib.ptr(d_r), _lib.ptr(d_cnt), m, None,
                              _lib.ptr(d_log), _lib.ptr(feat), 0, _lib.stream_ptr())
    else:
        _lib.lib().nif_query_dev(fam.view(with_fast=True), _lib.ptr(d_obj), _lib.ptr(d_ray),
                                 _lib.ptr(d_c4), _lib.ptr(d_r), _lib.ptr(d_cnt), m, None,
                                 _lib.ptr(d_log), impl, _lib.stream_ptr())
    return d_log.cpu().numpy()


def infer_records(model: NifModel, records, impl: int = _lib.IMPL_AUTO) -> np.ndarray:
    """nif.py:467-483: True = occluded (p < 0.5, i.e. logit < 0)."""
    if model.config.head != "occlusion":
        raise ValueError("model was built with the geometry head")
    occ = np.zeros(len(records), bool)
    om = records.kind == 0
    if om.any():
        occ[om] = query_family(model, "outer", records.obj[om], records.coord[om, 0:4],
                               impl) < 0.0
    im = records.kind == 1
    if im.any():
        occ[im] = query_family(model, "inner", records.obj[im], records.coord[im, 0:5],
                               impl) < 0.0
    return occ


def _split_queries(queries):
    from .scene import InnerQuery, OuterQuery
    o_idx, o_obj, o_coord, i_idx, i_obj, i_coord = [], [], [], [], [], []
    for j, q in enumerate(queries):
        if isinstance(q, InnerQuery):
            i_idx.append(j)
            i_obj.append(q.object_id)
            i_coord.append((q.p_prime.u, q.p_prime.v, q.d_prime.u, q.d_prime.v, q.r_prime))
        elif isinstance(q, OuterQuery):
            o_idx.append(j)
            o_obj.append(q.object_id)
            o_coord.append((q.p_prime.u, q.p_prime.v, q.d_prime.u, q.d_prime.v))
        else:
            raise TypeError(f"not a ray query: {type(q).__name__}")
    return (np.asarray(o_idx, np.int64), np.asarray(o_obj, np.int64),
            np.asarray(o_coord, np.float64).reshape(-1, 4), np.asarray(i_idx, np.int64),
            np.asarray(i_obj, np.int64), np.asarray(i_coord, np.float64).reshape(-1, 5))


def infer_occlusion(model: NifModel, queries, exact: bool = True) -> np.ndarray:
    """nif.py:428-442: True = occluded (p < 0.5; exactly 0.5 is visible).
    Outer batch first, then inner, results in query order. exact=True runs
    the reference's arithmetic (fp64 weights / accumulation, stable
    sigmoid: bit-identical to the reference, so SPEC.md's batching
    invariant holds bit for bit); exact=False runs the fused tensor-core
    query (fp16 operands, logit < 0)."""
    if model.config.head != "occlusion":
        raise ValueError("model was built with the geometry head")
    o_idx, o_obj, o_coord, i_idx, i_obj, i_coord = _split_queries(queries)
    out = np.zeros(len(queries), bool)
    for idx, obj, coord, which in ((o_idx, o_obj, o_coord, "outer"),
                                   (i_idx, i_obj, i_coord, "inner")):
        if not len(idx):
            continue
        if exact:
            p = _forward(model, which, obj, _encode(model, which, obj, coord))
            out[idx] = p[:, 0] < 0.5
        else:
            out[idx] = query_family(model, which, obj, coord) < 0.0
    return out


def infer_geometry(model: NifModel, queries, exact: bool = False):
    """nif.py:445-464: (unit normal [q,3], depth [q]) per query from the
    4-wide identity head; normals renormalised (a zero vector maps to +z),
    depth rescaled by the scene diagonal. exact=False runs the fused
    tensor-core query with the 4-wide head (fp16 operands, fp32 head);
    exact=True the reference's fp64-accumulation arithmetic."""
    if model.config.head != "geometry":
        raise ValueError("model was built with the occlusion head")
    o_idx, o_obj, o_coord, i_idx, i_obj, i_coord = _split_queries(queries)
    raw = np.zeros((len(queries), 4), np.float64)
    for idx, obj, coord, which in ((o_idx, o_obj, o_coord, "outer"),
                                   (i_idx, i_obj, i_coord, "inner")):
        if not len(idx):
            continue
        if exact:
            raw[idx] = _forward(model, which, obj, _encode(model, which, obj, coord))
        else:
            raw[idx] = query_family(model, which, obj, coord).reshape(-1, 4)
    normals = raw[:, 0:3]
    norms = np.linalg.norm(normals, axis=1)
    ok = norms > 1e-20
    normals = np.where(ok[:, None], normals / np.maximum(norms, 1e-300)[:, None],
                       np.array([0.0, 0.0, 1.0]))
    depth = raw[:, 3] * model.scene_diagonal
    return normals, depth
