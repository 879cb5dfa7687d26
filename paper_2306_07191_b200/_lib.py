"""ctypes binding of libnif_b200.so (include/nif_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2306_07191_b200.build``). There is no fallback: if the
shared object is missing every entry point raises, so a GPU run can never
silently answer from a CPU path.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("NIF_B200_LIB", _HERE / "libnif_b200.so"))

NIF_OK = 0
NIF_ERR_VALUE = 1
NIF_ERR_TYPE = 2
NIF_ERR_CUDA = 3
NIF_ERR_UNSUPPORTED = 4
NIF_MAX_LAYERS = 8

IMPL_AUTO = 0
IMPL_SIMT = 1
IMPL_TCGEN05 = 2
IMPL_TCGEN05_GENERIC = 3


class NifNode(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3), ("a", C.c_int32),
                ("b", C.c_int32), ("leaf", C.c_int32), ("pad", C.c_int32)]


class SceneView(C.Structure):
    _fields_ = [
        ("n_obj", C.c_int32), ("pad0", C.c_int32), ("n_nodes", C.c_int64),
        ("n_tris", C.c_int64), ("eps", C.c_double), ("tol", C.c_double),
        ("obox", C.c_void_p), ("t_order", C.c_void_p), ("roots", C.c_void_p),
        ("nodes", C.c_void_p), ("tris", C.c_void_p), ("normals", C.c_void_p),
        ("obj_albedo", C.c_void_p), ("top_nodes", C.c_void_p), ("top_order", C.c_void_p),
        ("n_top", C.c_int64),
    ]


class GatherOut(C.Structure):
    _fields_ = [
        ("outer_obj", C.c_void_p), ("outer_ray", C.c_void_p), ("outer_coord", C.c_void_p),
        ("inner_obj", C.c_void_p), ("inner_ray", C.c_void_p), ("inner_coord", C.c_void_p),
        ("inner_r", C.c_void_p), ("cap_outer", C.c_int64), ("cap_inner", C.c_int64),
        ("rec_kind", C.c_void_p), ("rec_obj", C.c_void_p), ("rec_ray", C.c_void_p),
        ("rec_coord", C.c_void_p), ("cap_total", C.c_int64), ("bvh_occ", C.c_void_p),
        ("counts", C.c_void_p),
    ]


class FamilyView(C.Structure):
    _fields_ = [
        ("family", C.c_int32), ("n_obj", C.c_int32), ("R", C.c_int32), ("N", C.c_int32),
        ("Rd", C.c_int32), ("Nd", C.c_int32), ("n_layers", C.c_int32),
        ("dims", C.c_int32 * (NIF_MAX_LAYERS + 1)), ("n_heads", C.c_int32),
        ("sigmoid_head", C.c_int32), ("w_stride", C.c_int32), ("b_stride", C.c_int32),
        ("pos", C.c_void_p), ("dir", C.c_void_p), ("dist", C.c_void_p),
        ("w", C.c_void_p), ("b", C.c_void_p), ("fast", C.c_void_p),
    ]


class Camera(C.Structure):
    _fields_ = [("pos", C.c_double * 3), ("fwd", C.c_double * 3), ("right", C.c_double * 3),
                ("up", C.c_double * 3), ("tan_half", C.c_double), ("aspect", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class LightsView(C.Structure):
    _fields_ = [("n_lights", C.c_int32), ("pad0", C.c_int32), ("kind", C.c_void_p),
                ("data", C.c_void_p), ("cum", C.c_void_p)]


class PassOut(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in
                ("hit", "t", "obj", "point", "normal", "pdir", "ldir", "tmax", "pdf", "emit")]


class TrainView(C.Structure):
    _fields_ = [
        ("params", C.c_void_p), ("grad", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p),
        ("numel", C.c_int64), ("off_pos", C.c_int64), ("off_dir", C.c_int64),
        ("off_dist", C.c_int64), ("off_w", C.c_int64), ("off_b", C.c_int64),
        ("grid_steps", C.c_void_p), ("mlp_steps", C.c_void_p), ("counts", C.c_void_p),
    ]


_lib = None


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    """Load the extension, failing loudly when it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(the engine has no CPU fallback)")
        _lib = C.CDLL(str(LIB_PATH))
        _declare(_lib)
    return _lib


def _check(status, func, args):
    if status == NIF_OK:
        return status
    msg = _lib.nif_last_error().decode()
    if status == NIF_ERR_VALUE:
        raise ValueError(msg)
    if status == NIF_ERR_TYPE:
        raise TypeError(msg)
    if status == NIF_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"{func.__name__}: {msg}")


P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
D = C.c_double

_SIGS = {
    "nif_abi_version": (C.c_int, []),
    "nif_device_check": (C.c_int, [C.c_int]),
    "nif_build_sah": (C.c_int, [P, P, P, I64, I64, I64, D, D, P, P, P, P, P, P, P]),
    "nif_build_sah_workspace_bytes": (C.c_size_t, [I64]),
    "nif_build_sah_dev": (C.c_int, [P, P, P, I64, I64, I64, D, D, P, P, P, P, P, P, P, P,
                                    C.c_size_t, P]),
    "nif_gather_workspace_bytes": (C.c_size_t, [I64]),
    "nif_gather_dev": (C.c_int, [C.POINTER(SceneView), P, P, P, P, I64,
                                 C.POINTER(GatherOut), P, C.c_size_t, P]),
    "nif_label_visible_dev": (C.c_int, [C.POINTER(SceneView), P, P, I64, P, P, P, P, P]),
    "nif_bvh_occluded_dev": (C.c_int, [C.POINTER(SceneView), P, P, P, I64, P, P]),
    "nif_encode_dev": (C.c_int, [C.POINTER(FamilyView), P, P, I64, P, P]),
    "nif_forward_dev": (C.c_int, [C.POINTER(FamilyView), P, P, I64, I32, P, P]),
    "nif_fast_pack_bytes": (C.c_size_t, [C.POINTER(FamilyView)]),
    "nif_fast_pack_dev": (C.c_int, [C.POINTER(FamilyView), P, P]),
    "nif_query_dev": (C.c_int, [C.POINTER(FamilyView), P, P, P, P, P, I64, P, P, I32, P]),
    "nif_occ_init_dev": (C.c_int, [P, I64, P, P]),
    "nif_feat_scratch_bytes": (C.c_size_t, [I64]),
    "nif_bucket_scratch_bytes": (C.c_size_t, [I64, I32]),
    "nif_engine_create": (C.c_int, [C.POINTER(SceneView), P, I32, C.POINTER(FamilyView),
                                    C.POINTER(FamilyView), I64, P, C.POINTER(C.c_void_p)]),
    "nif_engine_update_model": (C.c_int, [P, C.POINTER(FamilyView), C.POINTER(FamilyView), P]),
    "nif_engine_info": (C.c_int, [P, P]),
    "nif_engine_occluded_host": (C.c_int, [P, P, P, P, I64, P, I32]),
    "nif_engine_destroy": (C.c_int, [P]),
    "nif_query_bucketed_dev": (C.c_int, [C.POINTER(FamilyView), P, P, P, P, P, I64, P, P, P, P]),
    "nif_query_split_dev": (C.c_int, [C.POINTER(FamilyView), P, P, P, P, P, I64, P, P, P, I32, P]),
    "nif_debug_set_prof": (C.c_int, [P]),
    "nif_debug_set_prof_gather": (C.c_int, [P]),
    "nif_debug_set_gather_variant": (C.c_int, [C.c_int]),
    "nif_debug_set_gather_grid": (C.c_int, [C.c_int]),
    "nif_debug_set_gather_dynamic": (C.c_int, [C.c_int]),
    "nif_debug_set_timeline_gather": (C.c_int, [C.c_void_p]),
    "nif_debug_set_timeline_query": (C.c_int, [C.c_void_p]),
    "nif_debug_set_query_grid": (C.c_int, [C.c_int]),
    "nif_debug_set_query_variant": (C.c_int, [C.c_int]),
    "nif_debug_set_train_variant": (C.c_int, [C.c_int]),
    "nif_batch_counts_dev": (C.c_int, [P, P, I64, I32, P, P]),
    "nif_batch_counts_cur_dev": (C.c_int, [P, P, P, I64, I32, P, P]),
    "nif_train_fwdbwd_cur_dev": (C.c_int, [C.POINTER(FamilyView), C.POINTER(TrainView), P, P, P,
                                           P, P, I64, I64, I64, P, P]),
    "nif_cursor_advance_dev": (C.c_int, [P, I64, P]),
    "nif_train_prologue_cur_dev": (C.c_int, [C.POINTER(FamilyView), C.POINTER(TrainView), P, P,
                                             P, I64, P]),
    "nif_adam_units_dev": (C.c_int, [C.POINTER(FamilyView), C.POINTER(TrainView), D, D, D, D,
                                     P, I64, P]),
    "nif_train_fwdbwd_dev": (C.c_int, [C.POINTER(FamilyView), C.POINTER(TrainView), P, P, P, P,
                                       I64, I64, I64, P, P]),
    "nif_adam_dev": (C.c_int, [C.POINTER(FamilyView), C.POINTER(TrainView), D, D, D, D, P]),
    "nif_train_fwdbwd_ex_dev": (C.c_int, [C.POINTER(FamilyView), C.POINTER(TrainView), P, P, P,
                                          P, P, I64, I64, I64, P, P, P, P, I64, P]),
    "nif_train_part_floats": (C.c_int64, [C.POINTER(FamilyView), C.POINTER(TrainView), I64]),
    "nif_grid_scatter_ws_bytes": (C.c_size_t, [C.POINTER(FamilyView), C.POINTER(TrainView),
                                               I64, C.c_int]),
    "nif_grid_scatter_dev": (C.c_int, [C.POINTER(FamilyView), C.POINTER(TrainView), P, P, P, P,
                                       I64, P, C.c_int, P, C.c_size_t, P]),
    "nif_sample_pass_dev": (C.c_int, [C.POINTER(SceneView), C.POINTER(Camera),
                                      C.POINTER(LightsView), I64, I64, I32, I64, I64,
                                      C.POINTER(PassOut), P]),
    "nif_shade_accumulate_dev": (C.c_int, [C.POINTER(PassOut), P, P, P, I64, P, P]),
    "nif_label_geometry_dev": (C.c_int, [C.POINTER(SceneView), P, P, I64, P, P, D, P, P, P]),
}


def _declare(L):
    L.nif_last_error.restype = C.c_char_p
    L.nif_last_error.argtypes = []
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
        if res is C.c_int and name not in ("nif_abi_version", "nif_device_check"):
            fn.errcheck = _check


def declared_symbols():
    """Every function the public header declares (for the export test)."""
    import re
    hdr = (_HERE.parent / "include" / "nif_b200.h").read_text()
    hdr += (_HERE.parent / "include" / "nif_b200_debug.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(nif_\w+)\s*\(",
                                 hdr, re.M)))


def ptr(t) -> int:
    """Raw device/host address of a torch tensor or numpy array (or None)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
