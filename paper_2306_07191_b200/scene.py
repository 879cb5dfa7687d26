"""Scene description, host-side BVH build and the device-resident scene.

Mirrors the reference's scene surface (renderer.py:113-445, bvh.py:306-1045)
for what the NIF hot path consumes: per-object bottom-level trees, the
top-level tree, the packed arrays and the derived constants
(scene diagonal, epsilon_t, route mask). The SAH build runs in native code
(csrc/sah_builder.cpp) and reproduces the reference trees node for node;
the packed arrays are uploaded once to HBM as ``DeviceScene``.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _lib

MAX_LEAF = 4          # bvh.py:21
N_BINS = 16           # bvh.py:22
COST_TRAVERSAL = 1.0  # bvh.py:23
COST_INTERSECT = 1.5  # bvh.py:24
MAX_DEPTH = 120       # bvh.py:26 (reference stack budget)
DEVICE_STACK = 120    # traversal stack of the CUDA kernels (bvh.py:26 MAX_DEPTH)
EPSILON_SCALE = 1e-4  # renderer.py:43
CONTAINMENT_TOL = 1e-6  # geometry.py:20

NODE_DTYPE = np.dtype([("lo", "<f8", 3), ("hi", "<f8", 3), ("a", "<i4"), ("b", "<i4"),
                       ("leaf", "<i4"), ("pad", "<i4")])
assert NODE_DTYPE.itemsize == 64


def vec3(x, y, z) -> np.ndarray:
    return np.array([x, y, z], dtype=np.float64)


def _length(v) -> float:
    # geometry.py:29-30, same Python float arithmetic
    return math.sqrt(float(v[0]) ** 2 + float(v[1]) ** 2 + float(v[2]) ** 2)


def normalize(v) -> np.ndarray:
    n = _length(v)
    if n == 0.0:
        raise ValueError("cannot normalize a zero vector")
    return np.asarray(v, dtype=np.float64) / n


@dataclass(frozen=True)
class Aabb:
    min: np.ndarray
    max: np.ndarray

    @property
    def center(self):
        return 0.5 * (self.min + self.max)

    @property
    def half_diagonal(self):
        return 0.5 * (self.max - self.min)

    @property
    def diagonal(self) -> float:
        return _length(self.max - self.min)


# ---------------------------------------------------------------------------
# BVH build (native)
# ---------------------------------------------------------------------------


def _build_sah(lo, hi, ce, max_leaf):
    n = lo.shape[0]
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    ce = np.ascontiguousarray(ce, np.float64)
    cap = max(2 * n, 1)
    node_lo = np.empty((cap, 3))
    node_hi = np.empty((cap, 3))
    node_a = np.zeros(cap, np.int64)
    node_b = np.zeros(cap, np.int64)
    node_leaf = np.zeros(cap, np.uint8)
    order = np.empty(n, np.int64)
    n_nodes = C.c_int64(0)
    _lib.lib().nif_build_sah(
        _lib.ptr(lo), _lib.ptr(hi), _lib.ptr(ce), n, max_leaf, N_BINS,
        COST_TRAVERSAL, COST_INTERSECT, _lib.ptr(node_lo), _lib.ptr(node_hi),
        _lib.ptr(node_a), _lib.ptr(node_b), _lib.ptr(node_leaf), _lib.ptr(order),
        C.byref(n_nodes))
    k = n_nodes.value
    return (node_lo[:k].copy(), node_hi[:k].copy(), node_a[:k].copy(),
            node_b[:k].copy(), node_leaf[:k].copy(), order)


def build_sah_dev(lo, hi, ce, max_leaf=MAX_LEAF, stream=None):
    """_build_sah on the GPU (nif_build_sah_dev): lo/hi/ce are [n, 3] float64
    CUDA tensors; returns (node_lo, node_hi, node_a, node_b, node_leaf, order)
    as CUDA tensors, identical to the host build."""
    import torch
    n = lo.shape[0]
    if n == 0:
        raise ValueError("cannot build a tree over zero primitives")
    dev = lo.device
    lo, hi, ce = (t.to(torch.float64).contiguous() for t in (lo, hi, ce))
    cap = 2 * n
    node_lo = torch.empty((cap, 3), dtype=torch.float64, device=dev)
    node_hi = torch.empty((cap, 3), dtype=torch.float64, device=dev)
    node_a = torch.zeros(cap, dtype=torch.int64, device=dev)
    node_b = torch.zeros(cap, dtype=torch.int64, device=dev)
    node_leaf = torch.zeros(cap, dtype=torch.uint8, device=dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    n_nodes = C.c_int64(0)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    ws_bytes = _lib.lib().nif_build_sah_workspace_bytes(n)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    _lib.lib().nif_build_sah_dev(
        lo.data_ptr(), hi.data_ptr(), ce.data_ptr(), n, max_leaf, N_BINS,
        COST_TRAVERSAL, COST_INTERSECT, node_lo.data_ptr(), node_hi.data_ptr(),
        node_a.data_ptr(), node_b.data_ptr(), node_leaf.data_ptr(), order.data_ptr(),
        C.byref(n_nodes), ws.data_ptr(), ws_bytes, C.c_void_p(st.cuda_stream))
    k = n_nodes.value
    return node_lo[:k], node_hi[:k], node_a[:k], node_b[:k], node_leaf[:k], order


class _FlatBvh:
    def __init__(self, node_lo, node_hi, node_a, node_b, node_leaf, order):
        self.node_lo = node_lo
        self.node_hi = node_hi
        self.node_a = node_a
        self.node_b = node_b
        self.node_leaf = node_leaf
        self.order = order

    @property
    def n_nodes(self) -> int:
        return len(self.node_a)

    def depth(self) -> int:
        """bvh.py:337-346 depth, computed one frontier per level."""
        frontier = np.zeros(1, np.int64)
        d = 0
        while frontier.size:
            d += 1
            inner = frontier[self.node_leaf[frontier] == 0]
            frontier = np.concatenate((self.node_a[inner], self.node_b[inner]))
        return d


class BottomLevelBvh(_FlatBvh):
    """Per-object tree; triangle arrays stored in leaf order (bvh.py:361-377)."""

    def __init__(self, nodes, order, v0, v1, v2, n0, n1, n2, src):
        super().__init__(*nodes, order)
        self.v0, self.v1, self.v2 = v0, v1, v2
        self.n0, self.n1, self.n2 = n0, n1, n2
        self.src = src
        self.bounds = Aabb(self.node_lo[0].copy(), self.node_hi[0].copy())

    @property
    def n_triangles(self) -> int:
        return len(self.v0)


class TopLevelBvh(_FlatBvh):
    pass


def build_bottom(arrays, device=None) -> BottomLevelBvh:
    """bvh.py:402-428: tree over one object's triangles from
    (v0, v1, v2, n0, n1, n2) arrays. With a CUDA ``device`` the SAH build
    runs there (nif_build_sah_dev, the identical tree)."""
    v0, v1, v2, n0, n1, n2 = (np.ascontiguousarray(a, np.float64) for a in arrays)
    if len(v0) == 0:
        raise ValueError("cannot build a tree over zero triangles")
    lo = np.minimum(np.minimum(v0, v1), v2)
    hi = np.maximum(np.maximum(v0, v1), v2)
    ce = (lo + hi) * 0.5
    if device is None:
        *nodes, order = _build_sah(lo, hi, ce, MAX_LEAF)
    else:
        import torch
        t = [torch.from_numpy(x).to(device) for x in (lo, hi, ce)]
        *nodes, order = (x.cpu().numpy() for x in build_sah_dev(*t, max_leaf=MAX_LEAF))
    bvh = BottomLevelBvh(tuple(nodes), order, v0[order].copy(), v1[order].copy(),
                         v2[order].copy(), n0[order].copy(), n1[order].copy(),
                         n2[order].copy(), order.copy())
    if bvh.depth() > MAX_DEPTH - 8:
        raise ValueError("tree depth exceeds the traversal stack budget")
    return bvh


def build_bottoms(arrays_list, workers: Optional[int] = None, device=None):
    """build_bottom over many objects: on host threads (the native builder
    and numpy release the GIL), or one after another on a CUDA ``device``;
    trees are identical to sequential host builds."""
    from concurrent.futures import ThreadPoolExecutor
    arrays_list = list(arrays_list)
    if device is not None:
        return [build_bottom(a, device) for a in arrays_list]
    if workers is None:
        workers = min(len(arrays_list), os.cpu_count() or 1)
    if workers <= 1 or len(arrays_list) <= 1:
        return [build_bottom(a) for a in arrays_list]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(build_bottom, arrays_list))


def build_top(boxes: Sequence[Aabb]) -> TopLevelBvh:
    if len(boxes) == 0:
        raise ValueError("cannot build a tree over zero boxes")
    lo = np.stack([b.min for b in boxes]).astype(np.float64)
    hi = np.stack([b.max for b in boxes]).astype(np.float64)
    ce = (lo + hi) * 0.5
    *nodes, order = _build_sah(lo, hi, ce, 1)
    return TopLevelBvh(*nodes, order)


@dataclass
class ScenePack:
    """Flat arrays concatenated over objects (bvh.py:958-1045)."""

    t_lo: np.ndarray
    t_hi: np.ndarray
    t_a: np.ndarray
    t_b: np.ndarray
    t_leaf: np.ndarray
    t_order: np.ndarray
    roots: np.ndarray
    b_lo: np.ndarray
    b_hi: np.ndarray
    b_a: np.ndarray
    b_b: np.ndarray
    b_leaf: np.ndarray
    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray
    n0: np.ndarray
    n1: np.ndarray
    n2: np.ndarray
    src: np.ndarray
    prim_off: np.ndarray
    obox_lo: np.ndarray
    obox_hi: np.ndarray
    tri_counts: np.ndarray

    @property
    def n_objects(self) -> int:
        return len(self.roots)


def pack_scene(bvhs: List[BottomLevelBvh], top: TopLevelBvh) -> ScenePack:
    node_off = np.zeros(len(bvhs) + 1, np.int64)
    prim_off = np.zeros(len(bvhs) + 1, np.int64)
    for i, b in enumerate(bvhs):
        node_off[i + 1] = node_off[i] + b.n_nodes
        prim_off[i + 1] = prim_off[i] + b.n_triangles
    a_parts, b_parts = [], []
    for i, b in enumerate(bvhs):
        a = b.node_a.copy()
        bb = b.node_b.copy()
        leaf = b.node_leaf == 1
        a[leaf] += prim_off[i]
        a[~leaf] += node_off[i]
        bb[~leaf] += node_off[i]
        a_parts.append(a)
        b_parts.append(bb)
    cat = np.concatenate
    return ScenePack(
        t_lo=top.node_lo, t_hi=top.node_hi, t_a=top.node_a, t_b=top.node_b,
        t_leaf=top.node_leaf, t_order=top.order, roots=node_off[:-1].copy(),
        b_lo=cat([b.node_lo for b in bvhs]), b_hi=cat([b.node_hi for b in bvhs]),
        b_a=cat(a_parts), b_b=cat(b_parts), b_leaf=cat([b.node_leaf for b in bvhs]),
        v0=cat([b.v0 for b in bvhs]), v1=cat([b.v1 for b in bvhs]),
        v2=cat([b.v2 for b in bvhs]), n0=cat([b.n0 for b in bvhs]),
        n1=cat([b.n1 for b in bvhs]), n2=cat([b.n2 for b in bvhs]),
        src=cat([b.src for b in bvhs]), prim_off=prim_off,
        obox_lo=np.stack([b.bounds.min for b in bvhs]),
        obox_hi=np.stack([b.bounds.max for b in bvhs]),
        tri_counts=np.array([b.n_triangles for b in bvhs], np.int64),
    )


def top_dfs_order(top: TopLevelBvh) -> np.ndarray:
    """Objects in the order the reference's left-first top-level DFS meets
    their leaves (bvh.py:801-841). Leaves hold one object each and a
    left-first DFS visits leaves by increasing first slot, so this is the
    leaf-order array itself; verified here rather than assumed."""
    leaves = [(int(top.node_a[i]), int(top.node_b[i])) for i in range(top.n_nodes)
              if top.node_leaf[i]]
    seq = []
    stack = [0]
    while stack:
        i = stack.pop()
        if top.node_leaf[i]:
            seq.extend(int(top.order[k]) for k in range(top.node_a[i],
                                                         top.node_a[i] + top.node_b[i]))
        else:
            stack.append(int(top.node_b[i]))
            stack.append(int(top.node_a[i]))
    assert all(c == 1 for _, c in leaves)
    return np.asarray(seq, np.int32)


# ---------------------------------------------------------------------------
# camera, lights, scene
# ---------------------------------------------------------------------------


@dataclass
class Camera:
    position: np.ndarray
    look_at: np.ndarray
    up: np.ndarray
    vertical_fov: float
    width: int
    height: int

    def basis(self):
        # renderer.py:122-128
        fwd = normalize(self.look_at - self.position)
        right = normalize(np.cross(fwd, self.up))
        true_up = np.cross(right, fwd)
        tan_half = math.tan(math.radians(self.vertical_fov) * 0.5)
        aspect = self.width / self.height
        return fwd, right, true_up, tan_half, aspect


@dataclass
class PointLight:
    position: np.ndarray
    intensity: np.ndarray


@dataclass
class AreaLight:
    corner: np.ndarray
    edge_u: np.ndarray
    edge_v: np.ndarray
    radiance: np.ndarray

    @staticmethod
    def from_corners(corners, radiance) -> "AreaLight":
        c = [vec3(*p) for p in corners]
        return AreaLight(c[0], c[1] - c[0], c[3] - c[0], vec3(*radiance))

    @property
    def normal(self):
        return normalize(np.cross(self.edge_u, self.edge_v))

    @property
    def area(self) -> float:
        return float(np.linalg.norm(np.cross(self.edge_u, self.edge_v)))


def _light_flux(light) -> float:
    if isinstance(light, PointLight):
        return float(np.mean(light.intensity)) * 4.0 * math.pi
    if isinstance(light, AreaLight):
        return float(np.mean(light.radiance)) * math.pi * light.area
    raise TypeError(f"unknown light type {type(light).__name__}")


def build_light_cdf(lights) -> np.ndarray:
    """Flux CDF (renderer.py:198-214); environment lights are out of scope."""
    w = np.asarray([_light_flux(l) for l in lights], np.float64)
    if len(w) == 0:
        raise ValueError("no lights to sample")
    total = w.sum()
    if not (total > 0.0):
        raise ValueError("lights have zero total flux")
    cum = np.cumsum(w) / total
    cum[-1] = 1.0
    return cum


def pack_lights(lights):
    """renderer.py:223-259 _pack_lights for point/area lights."""
    kind = np.zeros(len(lights), np.uint8)
    data = np.zeros((len(lights), 16), np.float64)
    for i, l in enumerate(lights):
        if isinstance(l, PointLight):
            kind[i] = 0
            data[i, 0:3] = l.position
            data[i, 3:6] = l.intensity
        elif isinstance(l, AreaLight):
            kind[i] = 1
            data[i, 0:3] = l.corner
            data[i, 3:6] = l.edge_u
            data[i, 6:9] = l.edge_v
            data[i, 9:12] = l.radiance
            data[i, 12:15] = l.normal
            data[i, 15] = l.area
        else:
            raise TypeError(f"unknown light type {type(l).__name__}")
    return kind, data


@dataclass
class SceneObject:
    name: str
    bvh: BottomLevelBvh
    albedo: np.ndarray
    nif_enabled: bool = True

    @property
    def n_triangles(self) -> int:
        return self.bvh.n_triangles

    @property
    def bounds(self) -> Aabb:
        return self.bvh.bounds


class SphericalCoord(tuple):
    """(u, v): azimuth in [0,1) wraps, polar in [0,1] clamps (geometry.py:55-57)."""

    def __new__(cls, u, v):
        return super().__new__(cls, (float(u), float(v)))

    @property
    def u(self):
        return self[0]

    @property
    def v(self):
        return self[1]


@dataclass(frozen=True)
class OuterQuery:
    """geometry.py:128-134."""
    object_id: int
    p_prime: SphericalCoord
    d_prime: SphericalCoord


@dataclass(frozen=True)
class InnerQuery:
    """geometry.py:137-144."""
    object_id: int
    p_prime: SphericalCoord
    d_prime: SphericalCoord
    r_prime: float


@dataclass
class ShadowRays:
    """renderer.py:569-576: origins/dirs f64[n,3], tmaxs f64[n]."""

    origins: np.ndarray
    dirs: np.ndarray
    tmaxs: np.ndarray

    def __len__(self):
        return len(self.origins)


@dataclass
class QueryRecords:
    """renderer.py:579-590: kind 0 outer / 1 inner, obj, ray, coord[n,5]."""

    kind: np.ndarray
    obj: np.ndarray
    ray: np.ndarray
    coord: np.ndarray
    degenerate_count: int = 0

    def __len__(self):
        return len(self.kind)


class Scene:
    """Runtime scene (renderer.py:401-445) plus its HBM-resident copy."""

    def __init__(self, objects: Sequence[SceneObject], lights: Sequence = (),
                 camera: Optional[Camera] = None, seed: int = 0):
        self.objects = list(objects)
        if not self.objects:
            raise ValueError("the B200 engine needs at least one object")
        self.lights = list(lights)
        self.camera = camera
        self.seed = seed
        self.environment = None
        self.top = build_top([o.bounds for o in self.objects])
        self.pack = pack_scene([o.bvh for o in self.objects], self.top)
        self.bounds = Aabb(self.pack.t_lo[0].copy(), self.pack.t_hi[0].copy())
        self.diagonal = self.bounds.diagonal
        self.albedo = np.stack([o.albedo for o in self.objects]).astype(np.float64)
        self.epsilon_t = EPSILON_SCALE * self.diagonal
        self.nif_enabled = np.array([o.nif_enabled for o in self.objects], np.uint8)
        self.dfs_order = top_dfs_order(self.top)
        self._device = {}

    @property
    def n_objects(self) -> int:
        return len(self.objects)

    def nif_route_mask(self, hybrid_threshold: Optional[int] = None) -> np.ndarray:
        route = self.nif_enabled.copy()
        if hybrid_threshold is not None:
            route &= (self.pack.tri_counts >= hybrid_threshold).astype(np.uint8)
        return route

    def light_tables(self):
        cum = build_light_cdf(self.lights)
        kind, data = pack_lights(self.lights)
        return cum, kind, data

    def device(self, device=None) -> "DeviceScene":
        import torch
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        key = str(dev)
        if key not in self._device:
            self._device[key] = DeviceScene(self, dev)
        return self._device[key]


def max_depth(pack: ScenePack) -> int:
    best = 0
    for r in pack.roots:
        stack = [(int(r), 1)]
        while stack:
            i, d = stack.pop()
            best = max(best, d)
            if not pack.b_leaf[i]:
                stack.append((int(pack.b_a[i]), d + 1))
                stack.append((int(pack.b_b[i]), d + 1))
    return best


class DeviceScene:
    """HBM copy of the packed scene and the view struct the kernels take.

    Layout: 64-byte nodes (both child words in the same line as the box),
    triangles as 72-byte v0|v1|v2 records in leaf order, object boxes as
    48-byte lo|hi records, all fp64 (the classification and labels must be
    bit-exact against the reference's fp64 arithmetic).
    """

    def __init__(self, scene: Scene, device):
        import torch
        pk = scene.pack
        if pk.b_a.max(initial=0) >= 2 ** 31 or len(pk.v0) >= 2 ** 31:
            raise NotImplementedError("scene exceeds 32-bit node/triangle indices")
        depth = max_depth(pk)
        if depth > DEVICE_STACK - 2:
            raise NotImplementedError(f"tree depth {depth} exceeds the device stack")
        nodes = np.zeros(len(pk.b_a), NODE_DTYPE)
        nodes["lo"] = pk.b_lo
        nodes["hi"] = pk.b_hi
        nodes["a"] = pk.b_a.astype(np.int32)
        nodes["b"] = pk.b_b.astype(np.int32)
        nodes["leaf"] = pk.b_leaf.astype(np.int32)
        tris = np.ascontiguousarray(np.concatenate([pk.v0, pk.v1, pk.v2], axis=1))
        norms = np.ascontiguousarray(np.concatenate([pk.n0, pk.n1, pk.n2], axis=1))
        obox = np.ascontiguousarray(np.concatenate([pk.obox_lo, pk.obox_hi], axis=1))

        def up(a, dt=None):
            t = torch.from_numpy(np.ascontiguousarray(a))
            return t.to(device)

        self.device = device
        self.nodes = up(nodes.view(np.uint8).reshape(-1))
        self.tris = up(tris)
        self.normals = up(norms)
        self.obox = up(obox)
        dfs = getattr(scene, "dfs_order", None)
        if dfs is None:  # a reference niftrace.Scene
            dfs = top_dfs_order(scene.top)
        self.t_order = up(np.asarray(dfs, np.int32))
        self.roots = up(pk.roots.astype(np.int32))
        self.albedo = up(scene.albedo)
        top = scene.top
        tnodes = np.zeros(top.n_nodes, NODE_DTYPE)
        tnodes["lo"] = top.node_lo
        tnodes["hi"] = top.node_hi
        tnodes["a"] = top.node_a.astype(np.int32)
        tnodes["b"] = top.node_b.astype(np.int32)
        tnodes["leaf"] = top.node_leaf.astype(np.int32)
        self.top_nodes = up(tnodes.view(np.uint8).reshape(-1))
        self.top_order = up(top.order.astype(np.int32))
        self.n_obj = scene.n_objects
        self.view = _lib.SceneView(
            n_obj=scene.n_objects, pad0=0, n_nodes=len(nodes), n_tris=len(pk.v0),
            eps=scene.epsilon_t, tol=CONTAINMENT_TOL, obox=_lib.ptr(self.obox),
            t_order=_lib.ptr(self.t_order), roots=_lib.ptr(self.roots),
            nodes=_lib.ptr(self.nodes), tris=_lib.ptr(self.tris),
            normals=_lib.ptr(self.normals), obj_albedo=_lib.ptr(self.albedo),
            top_nodes=_lib.ptr(self.top_nodes), top_order=_lib.ptr(self.top_order),
            n_top=top.n_nodes)
        self.scene_bytes = (self.nodes.numel() + self.tris.numel() * 8
                            + self.normals.numel() * 8 + self.obox.numel() * 8)
        self._route = {}

    def route(self, mask: np.ndarray):
        import torch
        key = bytes(np.asarray(mask, np.uint8))
        if key not in self._route:
            self._route[key] = torch.from_numpy(
                np.ascontiguousarray(mask, np.uint8)).to(self.device)
        return self._route[key]
