"""TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.

Scene construction and model initialisation of the reference, restated on
the oracle side so the reference arm of bench.py (`--impl reference`) and
the CPU tests build their workloads without importing the B200 package:

  meshgen.py:16-102   icosphere / torus / ground_plane / mesh_arrays
  bvh.py:34-303       _build_sah        (nif_oracle.c oracle_build_sah)
  bvh.py:400-437      build_bottom / build_top
  bvh.py:1000-1045    pack_scene
  renderer.py:113-128 Camera.basis;  renderer.py:198-259 light CDF / pack
  renderer.py:401-424 Scene (diagonal, epsilon_t), 439-445 nif_route_mask
  nif.py:181-223, mlp.py:142-156, grids.py:99-117  seeded NifModel init

Pinned: tests/test_oracle_scene.py checks the packs of every golden scene
against the reference's own pack hashes and the C2 bench scene against the
package's build; the init against the reference's model hashes.
"""

from __future__ import annotations

import ctypes as C
import math
from types import SimpleNamespace
from typing import Dict, List, Tuple

import numpy as np

from . import oracle

MAX_LEAF = 4            # bvh.py:21
N_BINS = 16             # bvh.py:22
COST_TRAVERSAL = 1.0    # bvh.py:23
COST_INTERSECT = 1.5    # bvh.py:24
EPSILON_SCALE = 1e-4    # renderer.py:43
INIT_SCALE = 1e-4       # grids.py:99

# ---------------------------------------------------------------------------
# meshgen.py
# ---------------------------------------------------------------------------


def icosphere(subdivisions: int = 3, radius: float = 1.0):
    """meshgen.py:16-54, the same midpoint recursion and vertex order."""
    phi = (1.0 + math.sqrt(5.0)) / 2.0
    raw = np.array([
        (-1, phi, 0), (1, phi, 0), (-1, -phi, 0), (1, -phi, 0),
        (0, -1, phi), (0, 1, phi), (0, -1, -phi), (0, 1, -phi),
        (phi, 0, -1), (phi, 0, 1), (-phi, 0, -1), (-phi, 0, 1),
    ], np.float64)
    verts = [v / np.linalg.norm(v) for v in raw]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
             (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
             (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
             (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdivisions):
        cache: Dict[Tuple[int, int], int] = {}

        def mid(a, b):
            key = (a, b) if a < b else (b, a)
            k = cache.get(key)
            if k is None:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                k = cache[key] = len(verts) - 1
            return k

        nxt = []
        for a, b, c in faces:
            ab = mid(a, b)  # creation order of the reference's comprehension
            ca = mid(c, a)
            bc = mid(b, c)
            nxt += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nxt
    unit = np.asarray(verts)
    return unit * radius, np.asarray(faces, np.int64), unit


def torus(nu: int = 32, nv: int = 16, major: float = 1.0, minor: float = 0.35):
    """meshgen.py:57-84."""
    us = 2.0 * math.pi * np.arange(nu) / nu
    vs = 2.0 * math.pi * np.arange(nv) / nv
    uu, vv = np.meshgrid(us, vs, indexing="ij")
    cu, su, cv, sv = np.cos(uu), np.sin(uu), np.cos(vv), np.sin(vv)
    ring = major + minor * cv
    verts = np.stack([ring * cu, ring * su, minor * sv], axis=2).reshape(-1, 3)
    normals = np.stack([cv * cu, cv * su, sv], axis=2).reshape(-1, 3)
    faces = []
    for i in range(nu):
        for j in range(nv):
            a, b = (i % nu) * nv + j % nv, ((i + 1) % nu) * nv + j % nv
            c, d = ((i + 1) % nu) * nv + (j + 1) % nv, (i % nu) * nv + (j + 1) % nv
            faces += [(a, b, c), (a, c, d)]
    return verts, np.asarray(faces, np.int64), normals


def ground_plane(half_extent: float = 4.0, z: float = 0.0):
    """meshgen.py:87-93."""
    h = float(half_extent)
    verts = np.array([(-h, -h, z), (h, -h, z), (h, h, z), (-h, h, z)], np.float64)
    return verts, np.array([(0, 1, 2), (0, 2, 3)], np.int64), np.tile((0.0, 0.0, 1.0), (4, 1))


def mesh_arrays(verts, faces, normals):
    """meshgen.py:96-102."""
    v, n, f = np.asarray(verts, np.float64), np.asarray(normals, np.float64), np.asarray(faces)
    return v[f[:, 0]], v[f[:, 1]], v[f[:, 2]], n[f[:, 0]], n[f[:, 1]], n[f[:, 2]]


def transformed(arrays, scale=1.0, translate=(0.0, 0.0, 0.0)):
    """The scene builders' per-object transform: v * scale + t."""
    t = np.asarray(translate, np.float64)
    v0, v1, v2, n0, n1, n2 = arrays
    return v0 * scale + t, v1 * scale + t, v2 * scale + t, n0, n1, n2


# ---------------------------------------------------------------------------
# bvh.py
# ---------------------------------------------------------------------------


def build_sah(lo, hi, ce, max_leaf):
    """bvh.py:34-303 through nif_oracle.c."""
    lo, hi, ce = (np.ascontiguousarray(a, np.float64) for a in (lo, hi, ce))
    n = len(lo)
    node_lo, node_hi = np.empty((2 * n, 3)), np.empty((2 * n, 3))
    node_a, node_b = np.zeros(2 * n, np.int64), np.zeros(2 * n, np.int64)
    node_leaf, order = np.zeros(2 * n, np.uint8), np.empty(n, np.int64)
    L = oracle.lib()
    L.oracle_build_sah.restype = C.c_int64
    p = oracle._p
    k = L.oracle_build_sah(p(lo), p(hi), p(ce), C.c_int64(n), C.c_int64(max_leaf),
                           C.c_int64(N_BINS), C.c_double(COST_TRAVERSAL),
                           C.c_double(COST_INTERSECT), p(node_lo), p(node_hi), p(node_a),
                           p(node_b), p(node_leaf), p(order))
    return (node_lo[:k].copy(), node_hi[:k].copy(), node_a[:k].copy(), node_b[:k].copy(),
            node_leaf[:k].copy(), order)


def build_bottom(arrays):
    """bvh.py:402-428: one object's tree, triangles stored in leaf order."""
    v0, v1, v2, n0, n1, n2 = (np.ascontiguousarray(a, np.float64) for a in arrays)
    lo = np.minimum(np.minimum(v0, v1), v2)
    hi = np.maximum(np.maximum(v0, v1), v2)
    node_lo, node_hi, node_a, node_b, node_leaf, order = build_sah(lo, hi, (lo + hi) * 0.5,
                                                                   MAX_LEAF)
    return SimpleNamespace(node_lo=node_lo, node_hi=node_hi, node_a=node_a, node_b=node_b,
                           node_leaf=node_leaf, order=order, v0=v0[order].copy(),
                           v1=v1[order].copy(), v2=v2[order].copy(), n0=n0[order].copy(),
                           n1=n1[order].copy(), n2=n2[order].copy(), src=order.copy(),
                           lo=node_lo[0].copy(), hi=node_hi[0].copy())


def build_top(bottoms):
    """bvh.py:431-437: tree over object boxes, one object per leaf."""
    lo = np.stack([b.lo for b in bottoms]).astype(np.float64)
    hi = np.stack([b.hi for b in bottoms]).astype(np.float64)
    node_lo, node_hi, node_a, node_b, node_leaf, order = build_sah(lo, hi, (lo + hi) * 0.5, 1)
    return SimpleNamespace(node_lo=node_lo, node_hi=node_hi, node_a=node_a, node_b=node_b,
                           node_leaf=node_leaf, order=order)


def pack_scene(bottoms, top):
    """bvh.py:1000-1045."""
    n_nodes = [len(b.node_a) for b in bottoms]
    n_tris = [len(b.v0) for b in bottoms]
    node_off = np.concatenate([[0], np.cumsum(n_nodes)]).astype(np.int64)
    prim_off = np.concatenate([[0], np.cumsum(n_tris)]).astype(np.int64)
    a_parts, b_parts = [], []
    for i, b in enumerate(bottoms):
        a, bb = b.node_a.copy(), b.node_b.copy()
        leaf = b.node_leaf == 1
        a[leaf] += prim_off[i]
        a[~leaf] += node_off[i]
        bb[~leaf] += node_off[i]
        a_parts.append(a)
        b_parts.append(bb)
    cat = np.concatenate
    return SimpleNamespace(
        t_lo=top.node_lo, t_hi=top.node_hi, t_a=top.node_a, t_b=top.node_b,
        t_leaf=top.node_leaf, t_order=top.order, roots=node_off[:-1].copy(),
        b_lo=cat([b.node_lo for b in bottoms]), b_hi=cat([b.node_hi for b in bottoms]),
        b_a=cat(a_parts), b_b=cat(b_parts), b_leaf=cat([b.node_leaf for b in bottoms]),
        v0=cat([b.v0 for b in bottoms]), v1=cat([b.v1 for b in bottoms]),
        v2=cat([b.v2 for b in bottoms]), n0=cat([b.n0 for b in bottoms]),
        n1=cat([b.n1 for b in bottoms]), n2=cat([b.n2 for b in bottoms]),
        src=cat([b.src for b in bottoms]), prim_off=prim_off,
        obox_lo=np.stack([b.lo for b in bottoms]), obox_hi=np.stack([b.hi for b in bottoms]),
        tri_counts=np.array(n_tris, np.int64))


# ---------------------------------------------------------------------------
# renderer.py: camera, lights, scene
# ---------------------------------------------------------------------------


def _length(v) -> float:
    """geometry.py:29-30 (Python float arithmetic)."""
    return math.sqrt(float(v[0]) ** 2 + float(v[1]) ** 2 + float(v[2]) ** 2)


def _normalize(v):
    return np.asarray(v, np.float64) / _length(v)


class RefCamera:
    """renderer.py:113-128."""

    def __init__(self, position, look_at, up, fov, width, height):
        self.position = np.asarray(position, np.float64)
        self.look_at = np.asarray(look_at, np.float64)
        self.up = np.asarray(up, np.float64)
        self.vertical_fov, self.width, self.height = fov, width, height

    def basis(self):
        fwd = _normalize(self.look_at - self.position)
        right = _normalize(np.cross(fwd, self.up))
        true_up = np.cross(right, fwd)
        return (fwd, right, true_up, math.tan(math.radians(self.vertical_fov) * 0.5),
                self.width / self.height)


class RefScene:
    """renderer.py:401-445 for the oracle: objects = [(arrays, albedo,
    nif_enabled)], lights = recipe-style dicts (point / area)."""

    def __init__(self, objects, lights, camera: RefCamera, seed: int):
        self.bottoms = [build_bottom(a) for a, _, _ in objects]
        self.albedo = np.stack([np.asarray(al, np.float64) for _, al, _ in objects])
        self.nif_enabled = np.array([bool(e) for _, _, e in objects], np.uint8)
        self.top = build_top(self.bottoms)
        self.pack = pack_scene(self.bottoms, self.top)
        self.diagonal = _length(self.pack.t_hi[0] - self.pack.t_lo[0])
        self.epsilon_t = EPSILON_SCALE * self.diagonal
        self.lights, self.camera, self.seed = list(lights), camera, seed

    @property
    def n_objects(self) -> int:
        return len(self.bottoms)

    def nif_route_mask(self, hybrid_threshold=None):
        route = self.nif_enabled.copy()
        if hybrid_threshold is not None:
            route &= (self.pack.tri_counts >= hybrid_threshold).astype(np.uint8)
        return route

    def light_tables(self):
        """renderer.py:198-259 for point / area lights: (cum, kind, data)."""
        w, kind, data = [], np.zeros(len(self.lights), np.uint8), np.zeros((len(self.lights), 16))
        for i, l in enumerate(self.lights):
            if l["kind"] == "point":
                w.append(float(np.mean(np.asarray(l["intensity"], np.float64))) * 4.0 * math.pi)
                data[i, 0:3] = l["position"]
                data[i, 3:6] = l["intensity"]
            else:
                c = [np.asarray(p, np.float64) for p in l["corners"]]
                eu, ev = c[1] - c[0], c[3] - c[0]
                cr = np.cross(eu, ev)
                area = float(np.linalg.norm(cr))
                rad = np.asarray(l["radiance"], np.float64)
                w.append(float(np.mean(rad)) * math.pi * area)
                kind[i] = 1
                data[i, 0:3], data[i, 3:6], data[i, 6:9] = c[0], eu, ev
                data[i, 9:12], data[i, 12:15], data[i, 15] = rad, _normalize(cr), area
        w = np.asarray(w, np.float64)
        cum = np.cumsum(w) / w.sum()
        cum[-1] = 1.0
        return cum, kind, data

    def shadow_rays(self, sample: int = 0):
        """cli.py:170-183 (_bench_shadow_rays): the sample pass, then every
        hit pixel with a positive cosine and pdf casts its light ray."""
        osc = oracle.OracleScene(self.pack, self.epsilon_t)
        cum, kind, data = self.light_tables()
        sp = oracle.sample_pass(osc, self.camera, cum, kind, data, self.seed, sample)
        cos = np.einsum("ij,ij->i", sp["normal"], sp["ldir"])
        cast = sp["hit"] & (cos > 0) & (sp["pdf"] > 0)
        return sp["point"][cast].copy(), sp["ldir"][cast].copy(), sp["tmax"][cast].copy()


def from_recipe(recipe) -> RefScene:
    """tests/scenes.py recipe dict -> RefScene."""
    objs = []
    for od in recipe["objects"]:
        kind, args = od["mesh"]
        arrays = mesh_arrays(*globals()[kind](*args))
        arrays = transformed(arrays, od.get("scale", 1.0), od.get("translate", (0.0, 0.0, 0.0)))
        objs.append((arrays, od["albedo"], od.get("nif_enabled", True)))
    c = recipe["camera"]
    cam = RefCamera(c["position"], c["look_at"], c.get("up", (0.0, 0.0, 1.0)), c["fov"],
                    c["width"], c["height"])
    return RefScene(objs, recipe["lights"], cam, recipe["seed"])


LIGHT = {"kind": "point", "position": (2.2, -1.6, 2.8), "intensity": (28.0, 28.0, 28.0)}


def lattice(n_spheres, subdiv, radius, width=1920, height=1080, cols=4) -> RefScene:
    """spheres on a lattice + NIF-enabled plane,
    camera (0,-4.4,2.2) -> (0,0,0.3), fov 45, point light, seed 11."""
    base = mesh_arrays(*icosphere(subdiv, radius))
    rows = (n_spheres + cols - 1) // cols
    pitch = 1.2 if n_spheres <= 12 else 3.6 / max(cols - 1, 1)
    objs = []
    for k in range(n_spheres):
        x = -1.8 + pitch * (k % cols)
        y = -0.6 + 1.2 * (k // cols) - (0.6 * (rows - 3) if rows > 3 else 0.0)
        objs.append((transformed(base, 1.0, (x, y, radius)), (0.75, 0.33, 0.27), True))
    objs.append((mesh_arrays(*ground_plane(4.0)), (0.62, 0.62, 0.6), True))
    cam = RefCamera((0.0, -4.4, 2.2), (0.0, 0.0, 0.3), (0.0, 0.0, 1.0), 45.0, width, height)
    return RefScene(objs, [LIGHT], cam, 11)


def c1(width=256, height=256, subdiv=5) -> RefScene:
    """C1: icosphere(5, r=0.9) at z=0.9 + BVH-routed plane."""
    sphere = transformed(mesh_arrays(*icosphere(subdiv, 0.9)), 1.0, (0.0, 0.0, 0.9))
    cam = RefCamera((0.0, -3.4, 1.7), (0.0, 0.0, 0.45), (0.0, 0.0, 1.0), 38.0, width, height)
    return RefScene([(sphere, (0.75, 0.33, 0.27), True),
                     (mesh_arrays(*ground_plane(4.0)), (0.62, 0.62, 0.6), False)],
                    [LIGHT], cam, 11)


def c2(width=1920, height=1080) -> RefScene:
    return lattice(12, 6, 0.35, width, height)


# ---------------------------------------------------------------------------
# nif.py:181-223 seeded initialisation (default NifConfig shapes)
# ---------------------------------------------------------------------------


def init_model(n_objects, seed=0, sharing="shared", outer=(6, 64, 2, 256, 3),
               inner=(13, 48, 3, 128, 5, 128, 3), head_dim=1):
    """Host arrays of a fresh reference NifModel: (outer_heads, inner_heads,
    grids) with heads = [[(w f32[out,in], b f32[out]) per layer]] and
    grids = [{outer_pos, outer_dir, inner_pos, inner_dir, inner_dist}].
    outer = (in, width, hidden layers, R, N); inner = (in, width, hidden
    layers, R, N, Rd, Nd)."""
    def xavier(dims, ss):
        rng = np.random.Generator(np.random.PCG64(ss))
        out = []
        for i in range(len(dims) - 1):
            lim = np.sqrt(6.0 / (dims[i] + dims[i + 1]))
            out.append((rng.uniform(-lim, lim, (dims[i + 1], dims[i])).astype(np.float32),
                        np.zeros(dims[i + 1], np.float32)))
        return out

    def grid(shape, ss):
        return np.random.Generator(np.random.PCG64(ss)).uniform(
            -INIT_SCALE, INIT_SCALE, shape).astype(np.float32)

    mlp_ss, grid_ss = np.random.SeedSequence(seed).spawn(2)
    heads = 1 if sharing == "shared" else n_objects
    ch = mlp_ss.spawn(2 * heads)
    odims = [outer[0]] + [outer[1]] * outer[2] + [head_dim]
    idims = [inner[0]] + [inner[1]] * inner[2] + [head_dim]
    o_heads = [xavier(odims, ch[2 * h]) for h in range(heads)]
    i_heads = [xavier(idims, ch[2 * h + 1]) for h in range(heads)]
    grids = []
    for oss in grid_ss.spawn(n_objects):
        s = oss.spawn(5)
        grids.append({"outer_pos": grid((outer[3], outer[3], outer[4]), s[0]),
                      "outer_dir": grid((outer[3], outer[3], outer[4]), s[1]),
                      "inner_pos": grid((inner[3], inner[3], inner[4]), s[2]),
                      "inner_dir": grid((inner[3], inner[3], inner[4]), s[3]),
                      "inner_dist": grid((inner[5], inner[6]), s[4])})
    return o_heads, i_heads, grids


def family_arrays(heads, grids, fam):
    """The flat arrays oracle.encode / oracle.dense_forward take for one
    family (shared MLP: head 0)."""
    hl = heads[0]
    return dict(w=np.concatenate([w.reshape(-1) for w, _ in hl]),
                b=np.concatenate([b for _, b in hl]),
                dims=[hl[0][0].shape[1]] + [w.shape[0] for w, _ in hl],
                pos=np.stack([g[f"{fam}_pos"] for g in grids]),
                dir=np.stack([g[f"{fam}_dir"] for g in grids]),
                dist=np.stack([g["inner_dist"] for g in grids]) if fam == "inner" else None)


def visibility_pass(scene: RefScene, fams, rays):
    """The reference CPU path of one shadow-ray batch: gather_queries
    (renderer.py:613-644) -> encode_*_arrays + _k_dense_forward
    (nif.py:286-397) -> p < 0.5 -> per-ray OR seeded with the hybrid bits
    (renderer.py:675-683). Returns bool[n]."""
    o, d, t = rays
    osc = oracle.OracleScene(scene.pack, scene.epsilon_t)
    kind, obj, ray, coord, bvh_occ, _ = oracle.gather(osc, o, d, t, scene.nif_route_mask(None))
    occ = bvh_occ.copy()
    for fam, k, width in (("outer", 0, 4), ("inner", 1, 5)):
        sel = kind == k
        if sel.any():
            f = fams[fam]
            x = oracle.encode(f["pos"], f["dir"], f["dist"], obj[sel], coord[sel, :width])
            p = oracle.dense_forward(f["w"], f["b"], f["dims"], x)
            occ[ray[sel][p[:, 0] < 0.5]] = True
    return occ
