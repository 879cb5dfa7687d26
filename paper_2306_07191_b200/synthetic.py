"""Synthetic scenes of the benchmark configurations.

C1: icosphere(5, r=0.9) at z=0.9 + BVH-routed ground plane, 256x256.
C2: 12 x icosphere(6, r=0.35) on a 4x3 lattice + NIF-enabled plane
    (983,042 triangles, 13 objects), 1920x1080.
C3: 24 x icosphere(8) (31.46M triangles) + plane, 1920x1080.
All use the point light (2.2, -1.6, 2.8), I = 28 and scene seed 11.
Geometry is generated with the reference's meshgen constructions, so the
same parameters give the same scene on both sides.
"""

from __future__ import annotations

import numpy as np

from . import meshgen
from .scene import Camera, PointLight, Scene, SceneObject, build_bottom, build_bottoms

LIGHT = PointLight(np.array([2.2, -1.6, 2.8]), np.array([28.0, 28.0, 28.0]))


def _obj(name, arrays, albedo, nif=True):
    return SceneObject(name, build_bottom(arrays), np.asarray(albedo, np.float64), nif)


def c1(width=256, height=256, subdiv=5, plane_nif=False) -> Scene:
    sphere = meshgen.transformed(meshgen.mesh_arrays(*meshgen.icosphere(subdiv, 0.9)), 1.0,
                                 (0.0, 0.0, 0.9))
    plane = meshgen.mesh_arrays(*meshgen.ground_plane(4.0))
    cam = Camera(np.array([0.0, -3.4, 1.7]), np.array([0.0, 0.0, 0.45]),
                 np.array([0.0, 0.0, 1.0]), 38.0, width, height)
    return Scene([_obj("sphere", sphere, (0.75, 0.33, 0.27)),
                  _obj("plane", plane, (0.62, 0.62, 0.6), plane_nif)], [LIGHT], cam, 11)


def lattice(n_spheres: int, subdiv: int, radius: float, width=1920, height=1080,
            cols: int = 4, build_device=None) -> Scene:
    base = meshgen.mesh_arrays(*meshgen.icosphere(subdiv, radius))
    rows = (n_spheres + cols - 1) // cols
    pitch = 1.2 if n_spheres <= 12 else 3.6 / max(cols - 1, 1)
    arrays = []
    for k in range(n_spheres):
        x = -1.8 + pitch * (k % cols)
        y = -0.6 + 1.2 * (k // cols) - (0.6 * (rows - 3) if rows > 3 else 0.0)
        arrays.append(meshgen.transformed(base, 1.0, (x, y, radius)))
    arrays.append(meshgen.mesh_arrays(*meshgen.ground_plane(4.0)))
    # the per-object trees are independent: build them on all host cores, or
    # on the GPU (identical trees)
    trees = build_bottoms(arrays, device=build_device)
    objs = [SceneObject(f"sphere{k}", trees[k], np.asarray((0.75, 0.33, 0.27), np.float64), True)
            for k in range(n_spheres)]
    objs.append(SceneObject("plane", trees[-1], np.asarray((0.62, 0.62, 0.6), np.float64), True))
    cam = Camera(np.array([0.0, -4.4, 2.2]), np.array([0.0, 0.0, 0.3]),
                 np.array([0.0, 0.0, 1.0]), 45.0, width, height)
    return Scene(objs, [LIGHT], cam, 11)


def c2(width=1920, height=1080, build_device=None) -> Scene:
    return lattice(12, 6, 0.35, width, height, build_device=build_device)


def c3(width=1920, height=1080, subdiv=8, build_device=None) -> Scene:
    return lattice(24, subdiv, 0.3, width, height, cols=6, build_device=build_device)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3}
