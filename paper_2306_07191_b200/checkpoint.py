"""NIF1 model checkpoints, byte-compatible with the reference
(scene_io.py:308-387 save_checkpoint / load_checkpoint).

Layout (little endian): b"NIF1", u32 version (1), u64 length + JSON
metadata {"config", "n_objects", "scene_diagonal"} (sorted keys), then
every array in the NIF1 order (NifModel.model_arrays: per head the outer
then inner MLP layers' w, b; per object outer_pos, outer_dir, inner_pos,
inner_dir, inner_dist) as u32 ndim, u64 shape[ndim], f32 data. A file
written here loads in the reference and vice versa; malformed files raise
SceneFormatError with the reference's messages.

Optimiser state (not part of NIF1, whose reader rejects trailing bytes) is
written to an optional sidecar `<path>.adam` (b"NIFA", the sha256 of the
NIF1 file it belongs to, then per family the flat m / v buffers and the
per-tensor step counters) so training can resume on the device. Saving
without `adam` removes a stale sidecar; a sidecar whose digest does not
match the checkpoint beside it is rejected.
"""

from __future__ import annotations

import json
import struct
from pathlib import Path
from typing import Optional

import numpy as np

from .nif import NifConfig, NifModel

CHECKPOINT_MAGIC = b"NIF1"
CHECKPOINT_VERSION = 1
ADAM_MAGIC = b"NIFA"


class SceneFormatError(ValueError):
    """scene_io.py SceneFormatError: malformed scene / checkpoint input."""


def save_checkpoint(model: NifModel, path, adam: bool = False) -> None:
    meta = {"config": model.config.to_dict(), "n_objects": model.n_objects,
            "scene_diagonal": model.scene_diagonal}
    blob = json.dumps(meta, sort_keys=True).encode()
    with open(path, "wb") as fh:
        fh.write(CHECKPOINT_MAGIC)
        fh.write(struct.pack("<I", CHECKPOINT_VERSION))
        fh.write(struct.pack("<Q", len(blob)))
        fh.write(blob)
        for arr in model.model_arrays():
            a = np.ascontiguousarray(arr, "<f4")
            fh.write(struct.pack("<I", a.ndim))
            fh.write(struct.pack(f"<{a.ndim}Q", *a.shape))
            fh.write(a.tobytes())
    side = Path(str(path) + ".adam")
    if adam:
        _save_adam(model, side, _digest(path))
    elif side.exists():
        # a sidecar from an earlier save would otherwise be restored with
        # these weights on the next load
        side.unlink()


def _digest(path) -> bytes:
    """sha256 of a NIF1 file: binds an Adam sidecar to the exact weights."""
    import hashlib
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for block in iter(lambda: fh.read(1 << 20), b""):
            h.update(block)
    return h.digest()


def _read_exact(fh, n: int, path) -> bytes:
    data = fh.read(n)
    if len(data) != n:
        raise SceneFormatError(f"{path}: truncated checkpoint")
    return data


def load_checkpoint(path, into: Optional[NifModel] = None, device=None) -> NifModel:
    """Rebuild a model from disk (scene_io.py:355-386). With `into`, the file
    must echo that model's configuration exactly; weights load in place."""
    path = Path(path)
    with open(path, "rb") as fh:
        if _read_exact(fh, 4, path) != CHECKPOINT_MAGIC:
            raise SceneFormatError(f"{path}: not a model checkpoint")
        (version,) = struct.unpack("<I", _read_exact(fh, 4, path))
        if version != CHECKPOINT_VERSION:
            raise SceneFormatError(f"{path}: unsupported checkpoint version {version}")
        (blob_len,) = struct.unpack("<Q", _read_exact(fh, 8, path))
        meta = json.loads(_read_exact(fh, blob_len, path))
        config = NifConfig.from_dict(meta["config"])
        if into is not None:
            if into.config.to_dict() != config.to_dict() or into.n_objects != meta["n_objects"]:
                raise SceneFormatError(
                    f"{path}: checkpoint configuration does not match the model")
            model = into
            model.scene_diagonal = float(meta["scene_diagonal"])
        else:
            model = NifModel(config, meta["n_objects"], meta["scene_diagonal"],
                             dtype=np.float32, device=device)
        arrays = [np.array(a) for a in model.model_arrays()]
        for arr in arrays:
            (ndim,) = struct.unpack("<I", _read_exact(fh, 4, path))
            shape = struct.unpack(f"<{ndim}Q", _read_exact(fh, 8 * ndim, path))
            if shape != arr.shape:
                raise SceneFormatError(
                    f"{path}: stored array shape {shape} does not match {arr.shape}")
            count = int(np.prod(shape))
            data = np.frombuffer(_read_exact(fh, 4 * count, path), "<f4")
            arr[...] = data.reshape(shape)
        if fh.read(1):
            raise SceneFormatError(f"{path}: trailing bytes after checkpoint payload")
    _install(model, arrays)
    side = Path(str(path) + ".adam")
    if side.exists():
        _load_adam(model, side, _digest(path))
    return model


def _install(model: NifModel, arrays) -> None:
    """Arrays in NIF1 order -> the device-resident flat parameter buffers."""
    it = iter(arrays)
    heads = {}
    for which in ("outer", "inner"):
        fam = model.family(which)
        heads[which] = [[(next(it), next(it)) for _ in range(len(fam.dims) - 1)]
                        for _ in range(fam.n_heads)]
    grids = []
    for _ in range(model.n_objects):
        grids.append({k: next(it) for k in ("outer_pos", "outer_dir", "inner_pos", "inner_dir",
                                            "inner_dist")})
    model.load_arrays(heads["outer"], heads["inner"], grids)


def _save_adam(model: NifModel, path: Path, digest: bytes) -> None:
    with open(path, "wb") as fh:
        fh.write(ADAM_MAGIC)
        fh.write(digest)
        for fam in (model.outer, model.inner):
            for t in (fam.m, fam.v):
                a = t.detach().cpu().numpy().astype("<f4")
                fh.write(struct.pack("<Q", a.size))
                fh.write(a.tobytes())
            for t in (fam.grid_steps, fam.mlp_steps):
                a = t.detach().cpu().numpy().astype("<i8")
                fh.write(struct.pack("<Q", a.size))
                fh.write(a.tobytes())


def _load_adam(model: NifModel, path: Path, digest: bytes) -> None:
    import torch
    with open(path, "rb") as fh:
        if _read_exact(fh, 4, path) != ADAM_MAGIC:
            raise SceneFormatError(f"{path}: not an optimiser-state sidecar")
        if _read_exact(fh, 32, path) != digest:
            raise SceneFormatError(
                f"{path}: optimiser state belongs to a different checkpoint")
        for fam in (model.outer, model.inner):
            for t, dt, w in ((fam.m, "<f4", 4), (fam.v, "<f4", 4), (fam.grid_steps, "<i8", 8),
                             (fam.mlp_steps, "<i8", 8)):
                (n,) = struct.unpack("<Q", _read_exact(fh, 8, path))
                if n != t.numel():
                    raise SceneFormatError(f"{path}: optimiser state does not match the model")
                a = np.frombuffer(_read_exact(fh, w * n, path), dt)
                t.copy_(torch.from_numpy(a.astype(t.cpu().numpy().dtype)).to(t.device))
        if fh.read(1):
            raise SceneFormatError(f"{path}: trailing bytes after optimiser state")
