"""Test helpers: golden fixture loading with minimal, product-independent
stand-ins for the reference's data types (so the oracle can be pinned to the
golden vectors without importing the product package)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path
from types import SimpleNamespace
from typing import NamedTuple

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


class Addr(NamedTuple):
    lod: int
    ijk: tuple


def addr_from_key(key: str) -> Addr:
    lod, ijk = key.split("/")
    return Addr(int(lod), tuple(int(v) for v in ijk.split("_")))


@lru_cache(maxsize=None)
def npz(name: str):
    return dict(np.load(GOLDEN / name, allow_pickle=False))


def parse_mfa(data: bytes, ncp: int, extent, lod: int = 1):
    """FORMAT.md:16-70 restated: [u8 d][3*(ncp+d) f32 knots t1..][ncp^3 f32, x fastest]."""
    d = data[0]
    stored = ncp + d
    assert len(data) == 1 + (stored * 3 + ncp ** 3) * 4
    knots = np.zeros((3, stored + 1), dtype=np.float32)
    off = 1
    for a in range(3):
        knots[a, 1:] = np.frombuffer(data, dtype="<f4", count=stored, offset=off)
        off += stored * 4
    ctrl = np.frombuffer(data, dtype="<f4", count=ncp ** 3, offset=off).reshape((ncp,) * 3, order="F").copy()
    return SimpleNamespace(degree=int(d), knots=knots, control=ctrl,
                           extent=np.asarray(extent, dtype=np.float64).reshape(3, 2), lod=lod)


def manifest_ns(obj: dict):
    entries = {}
    for key, e in obj["entries"].items():
        entries[addr_from_key(key)] = SimpleNamespace(extent=np.asarray(e["extent"], dtype=np.float64),
                                                      ncp=e.get("ncp"), path=e.get("path", ""),
                                                      nbytes=e.get("nbytes"))
    return SimpleNamespace(levels=int(obj["levels"]), finest_blocks_per_axis=int(obj["finest_blocks_per_axis"]),
                           micro_dims=tuple(obj["micro_dims"]), entries=entries, raw=obj)


@lru_cache(maxsize=None)
def golden_store(name: str):
    """(manifest namespace, {Addr: model namespace}, {Addr: raw bytes})."""
    z = npz(f"store_{name}.npz")
    man = manifest_ns(json.loads(bytes(z["manifest"]).decode()))
    blob = bytes(z["blob"])
    offs = z["offsets"]
    models, raw = {}, {}
    for i, key in enumerate(z["keys"]):
        a = addr_from_key(str(key))
        data = blob[offs[i]:offs[i + 1]]
        e = man.entries[a]
        raw[a] = data
        models[a] = parse_mfa(data, e.ncp, e.extent, a.lod)
    return man, models, raw


def pov_ns(row):
    row = np.asarray(row, dtype=np.float64)
    return SimpleNamespace(position=row[0:3], direction=row[3:6], up=row[6:9], fov_y=float(row[9]))


def params_ns(row):
    w, h, sd, omax, ref, near, amb, dif, spe, shi = [float(v) for v in row]
    return SimpleNamespace(width=int(w), height=int(h), sample_distance=sd, o_max=omax,
                           reference_step=None if np.isnan(ref) else ref, near=near, ambient=amb,
                           diffuse=dif, specular=spe, shininess=shi)


def tf_ns(raw):
    obj = json.loads(bytes(raw).decode())
    return SimpleNamespace(color_points=np.asarray(obj["color"], dtype=np.float64),
                           opacity_points=np.asarray(obj["opacity"], dtype=np.float64),
                           domain=tuple(obj["domain"]))


def vis_for(table: np.ndarray, pov_index: int, col1: int):
    rows = table[(table[:, 0] == pov_index) & (table[:, 1] == col1)]
    return [tuple(int(v) for v in r[2:]) for r in rows]
