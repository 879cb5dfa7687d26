"""Scene recipes shared by the golden generator (reference side) and the
tests / bench (package side): identical parameters on both sides."""

from __future__ import annotations

import numpy as np

_CAM = {"position": (0.0, -3.4, 1.7), "look_at": (0.0, 0.0, 0.45), "up": (0.0, 0.0, 1.0),
        "fov": 38.0}

RECIPES = {
    # C1 analogue at small size: sphere + BVH-routed ground plane
    "c1s": {
        "objects": [
            {"name": "sphere", "mesh": ("icosphere", (3, 0.9)), "translate": (0.0, 0.0, 0.9),
             "albedo": (0.75, 0.33, 0.27)},
            {"name": "plane", "mesh": ("ground_plane", (4.0,)), "albedo": (0.62, 0.62, 0.6),
             "nif_enabled": False},
        ],
        "lights": [{"kind": "point", "position": (2.2, -1.6, 2.8), "intensity": (28.0, 28.0, 28.0)}],
        "camera": {**_CAM, "width": 64, "height": 64},
        "seed": 11,
    },
    # NIF-enabled plane: exercises the flat-box top-level culling quirk
    "c1s_flat": {
        "objects": [
            {"name": "sphere", "mesh": ("icosphere", (3, 0.9)), "translate": (0.0, 0.0, 0.9),
             "albedo": (0.75, 0.33, 0.27)},
            {"name": "plane", "mesh": ("ground_plane", (4.0,)), "albedo": (0.62, 0.62, 0.6),
             "nif_enabled": True},
        ],
        "lights": [{"kind": "point", "position": (2.2, -1.6, 2.8), "intensity": (28.0, 28.0, 28.0)}],
        "camera": {**_CAM, "width": 64, "height": 64},
        "seed": 11,
    },
    # overlapping boxes: rays whose origin lies in two boxes
    "overlap": {
        "objects": [
            {"name": "torus", "mesh": ("torus", (32, 18, 1.0, 0.38)), "scale": 0.85,
             "translate": (0.0, 0.0, 0.3), "albedo": (0.3, 0.52, 0.75)},
            {"name": "ball", "mesh": ("icosphere", (2, 1.0)), "scale": 0.5,
             "translate": (0.35, 0.0, 0.3), "albedo": (0.78, 0.35, 0.25)},
            {"name": "plane", "mesh": ("ground_plane", (4.0,)), "translate": (0.0, 0.0, -0.65),
             "albedo": (0.6, 0.6, 0.58), "nif_enabled": False},
        ],
        "lights": [{"kind": "point", "position": (1.8, -2.2, 3.0), "intensity": (30.0, 30.0, 30.0)}],
        "camera": {**_CAM, "look_at": (0.0, 0.0, 0.25), "width": 64, "height": 48},
        "seed": 23,
    },
    # area light + three objects (sphere_torus_plane bundled scene analogue)
    "area": {
        "objects": [
            {"name": "sphere", "mesh": ("icosphere", (3, 1.0)), "scale": 0.72,
             "translate": (-0.85, 0.05, 0.72), "albedo": (0.74, 0.31, 0.25)},
            {"name": "torus", "mesh": ("torus", (32, 18, 1.0, 0.38)), "scale": 0.62,
             "translate": (0.9, 0.15, 0.26), "albedo": (0.26, 0.45, 0.78)},
            {"name": "plane", "mesh": ("ground_plane", (4.0,)), "albedo": (0.62, 0.62, 0.6),
             "nif_enabled": False},
        ],
        "lights": [{"kind": "area",
                    "corners": [[-0.7, -0.45, 2.6], [0.7, -0.45, 2.6], [0.7, 0.95, 2.6],
                                [-0.7, 0.95, 2.6]],
                    "radiance": (11.0, 11.0, 10.5)}],
        "camera": {**_CAM, "width": 48, "height": 48},
        "seed": 5,
    },
    # one object: the top-level root is a leaf (never box-tested)
    "single": {
        "objects": [
            {"name": "ball", "mesh": ("icosphere", (2, 1.0)), "albedo": (0.7, 0.7, 0.7)},
        ],
        "lights": [{"kind": "point", "position": (2.0, -2.0, 3.0), "intensity": (20.0, 20.0, 20.0)}],
        "camera": {**_CAM, "look_at": (0.0, 0.0, 0.0), "width": 40, "height": 40},
        "seed": 3,
    },
}


def build_scene(recipe):
    """The same scene through the B200 package (no reference import)."""
    from paper_2306_07191_b200 import meshgen
    from paper_2306_07191_b200.scene import (AreaLight, Camera, PointLight, Scene, SceneObject,
                                             build_bottom)

    objs = []
    for od in recipe["objects"]:
        kind, args = od["mesh"]
        arrays = meshgen.mesh_arrays(*getattr(meshgen, kind)(*args))
        arrays = meshgen.transformed(arrays, od.get("scale", 1.0), od.get("translate", (0, 0, 0)))
        objs.append(SceneObject(od["name"], build_bottom(arrays),
                                np.asarray(od["albedo"], np.float64), od.get("nif_enabled", True)))
    lights = []
    for ld in recipe["lights"]:
        if ld["kind"] == "point":
            lights.append(PointLight(np.asarray(ld["position"], np.float64),
                                     np.asarray(ld["intensity"], np.float64)))
        else:
            lights.append(AreaLight.from_corners(ld["corners"], ld["radiance"]))
    c = recipe["camera"]
    cam = Camera(np.asarray(c["position"], np.float64), np.asarray(c["look_at"], np.float64),
                 np.asarray(c.get("up", (0, 0, 1)), np.float64), c["fov"], c["width"], c["height"])
    return Scene(objs, lights, cam, recipe["seed"])
