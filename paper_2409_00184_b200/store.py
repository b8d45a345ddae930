"""Store reader: manifest.json + level-N/i_j_k.mfa (FORMAT.md:89-155).

load_model_bytes / load_model mirror the reference's read side
(store.py:33-47).  device_loader returns a loader for runtime.ModelCache
that reads a block file and uploads it straight into a DeviceStore slot
(raw bytes H2D, realigned on device), so the cache holds HBM handles.
The encoder-side write_store is provided for tests and synthetic stores.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from . import model
from .errors import FormatError

__all__ = ["write_store", "load_model_bytes", "load_model", "store_size_bytes", "device_loader"]


def write_store(store_root, manifest, models: dict) -> Path:
    root = Path(store_root)
    for addr in sorted(models):
        blob = models[addr] if isinstance(models[addr], (bytes, bytearray)) else model.serialize(models[addr])
        target = root / addr.file_name
        target.parent.mkdir(parents=True, exist_ok=True)
        target.write_bytes(blob)
        ent = manifest.entries[addr]
        ent.path, ent.nbytes = addr.file_name, len(blob)
    manifest.save(root)
    return root


def load_model_bytes(store_root, manifest, addr) -> bytes:
    ent = manifest.entries.get(addr)
    if ent is None or not ent.path:
        raise FormatError(f"manifest has no model file for block {addr.key}")
    path = Path(store_root) / ent.path
    if not path.exists():
        raise FormatError(f"missing model file {path}")
    return path.read_bytes()


def load_model(store_root, manifest, addr) -> model.MicroModel:
    ent = manifest.entries[addr]
    return model.deserialize(load_model_bytes(store_root, manifest, addr), ncp=ent.ncp, extent=ent.extent,
                             lod=addr.lod)


def store_size_bytes(store_root, manifest) -> int:
    root = Path(store_root)
    return sum((root / e.path).stat().st_size for e in manifest.entries.values() if e.path)


def device_loader(store_root, manifest, dstore, stream=None, source=None):
    """addr -> DeviceBlock.  Block files are read natively into pinned
    staging and uploaded asynchronously (afam_store_put_file);
    `source(addr) -> bytes` overrides the file read (e.g. an in-memory /
    pinned host store)."""

    def load(addr):
        ent = manifest.entries.get(addr)
        if source is None:
            if ent is None or not ent.path:
                raise FormatError(f"manifest has no model file for block {addr.key}")
            return dstore.load_file(Path(store_root) / ent.path, ent.ncp, ent.extent, addr.lod, stream)
        data = source(addr)
        if ent is None:
            raise FormatError(f"manifest has no model file for block {addr.key}")
        # afam_store_put_mfa validates like model.deserialize (FormatError on
        # length / degree byte, ValueError on non-finite control points)
        buf = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        return dstore.load_mfa(buf, ent.ncp, ent.extent, addr.lod, stream)

    return load
