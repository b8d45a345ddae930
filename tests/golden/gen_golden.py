"""Generate golden vectors from the UNMODIFIED reference (splinecast).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

Every fixture is produced by calling the reference's own public functions on
seeded inputs; nothing here re-implements reference arithmetic.  The
fixtures pin oracle/ (tests/test_oracle_golden.py) and the product path
(tests/test_*_gpu.py) to the reference.

Outputs (tests/golden/):
  bspline.npz        evaluate_points[_with_gradient], find_spans, basis,
                     decode_tensor_product / MicroModel.decode_grid cases
  store_<name>.npz   packed stores (manifest JSON + .mfa bytes) encoded by
                     the reference encoder
  visible.npz        select_visible outputs over many POVs and manifests
  frames.npz         render() frames, sample counts and error messages
"""

from __future__ import annotations

import io
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from splinecast import bspline, model, render, runtime  # noqa: E402
from splinecast.encoder import encode_volume  # noqa: E402
from splinecast.errors import MissingBlockError  # noqa: E402
from splinecast.partition import BlockAddress, LODManifest, ManifestEntry, _extent  # noqa: E402
from splinecast.volume import AnalyticField, marschner_lobb, sample_grid  # noqa: E402

OUT = Path(__file__).resolve().parent


def smooth_field():
    """The reference test suite's smooth field (tests/test_render.py:26-37)."""

    def val(x, y, z):
        return 0.5 + 0.3 * np.sin(2 * x) * np.cos(1.5 * y) + 0.1 * z

    def grad(x, y, z):
        return (
            0.6 * np.cos(2 * x) * np.cos(1.5 * y),
            -0.45 * np.sin(2 * x) * np.sin(1.5 * y),
            0.1 * np.ones_like(np.asarray(z, dtype=float)),
        )

    return AnalyticField(val, grad, np.array([[0.0, 1.0]] * 3))


# ------------------------------------------------------------------ stores
def pack_store(manifest: LODManifest, models: dict) -> dict:
    keys, blobs, offs = [], [], [0]
    for addr in sorted(models):
        blob = model.serialize(models[addr])
        entry = manifest.entries[addr]
        entry.path = addr.file_name
        entry.nbytes = len(blob)
        keys.append(addr.key)
        blobs.append(blob)
        offs.append(offs[-1] + len(blob))
    return {
        "manifest": np.frombuffer(json.dumps(manifest.to_json()).encode(), dtype=np.uint8),
        "keys": np.array(keys),
        "blob": np.frombuffer(b"".join(blobs), dtype=np.uint8),
        "offsets": np.array(offs, dtype=np.int64),
    }


def build_stores():
    stores = {}
    t = time.time()
    vol = sample_grid(smooth_field(), (33, 33, 33))
    m, models, _ = encode_volume(vol, levels=3, micro_dims=5, degree=2, error_bound=1e-4)
    stores["smooth33"] = (m, models)
    print(f"smooth33: {len(models)} blocks {time.time() - t:.1f}s", flush=True)

    t = time.time()
    vol = sample_grid(marschner_lobb(), (65, 65, 65))
    m, models, _ = encode_volume(vol, levels=2, micro_dims=17, degree=3, error_bound=1e-3, coarsest=2)
    stores["ml65_p3"] = (m, models)
    print(f"ml65_p3: {len(models)} blocks {time.time() - t:.1f}s", flush=True)

    # BASELINE config 1: 64^3 ML, degree 2, 8^3 micro-blocks, single LOD.
    t = time.time()
    vol = sample_grid(marschner_lobb(), (64, 64, 64))
    m, models, _ = encode_volume(vol, levels=1, micro_dims=8, coarsest=9, degree=2, error_bound=1e-3)
    stores["config1"] = (m, models)
    print(f"config1: {len(models)} blocks {time.time() - t:.1f}s", flush=True)

    # Constant volume, multi-block vs single-block (tests/test_cli.py:236-261).
    from splinecast.volume import ScalarVolume

    cvol = ScalarVolume(np.full((9, 9, 9), 0.5, dtype=np.float32), np.array([[0.0, 1.0]] * 3))
    m, models, _ = encode_volume(cvol, levels=2, micro_dims=5, coarsest=1)
    stores["const_multi"] = (m, models)
    m, models, _ = encode_volume(cvol, levels=1, micro_dims=9, coarsest=1)
    stores["const_single"] = (m, models)
    for name, (m, models) in stores.items():
        np.savez_compressed(OUT / f"store_{name}.npz", **pack_store(m, models))
    return stores


def skeleton_manifest(levels: int, coarsest: int, micro: int) -> LODManifest:
    """Address/extent-only manifest (partition.py:198-305 without volume data)."""
    finest = coarsest * 2 ** (levels - 1)
    man = LODManifest(levels=levels, micro_dims=(micro,) * 3, finest_blocks_per_axis=finest,
                      volume_dims=(finest * (micro - 1) + 1,) * 3, bounds=np.array([[0.0, 1.0]] * 3))
    for lod in range(1, levels + 1):
        bpa = coarsest * 2 ** (levels - lod)
        for i in range(bpa):
            for j in range(bpa):
                for k in range(bpa):
                    man.entries[BlockAddress(lod, (i, j, k))] = ManifestEntry(extent=_extent((i, j, k), bpa))
    return man


# ------------------------------------------------------------------ bspline
def gen_bspline():
    rng = np.random.default_rng(20261017)
    out = {}
    cases = []
    ci = 0
    for degree in (1, 2, 3):
        for ncp in sorted({degree + 1, 7, 12}):
            coeff = rng.normal(size=(ncp, ncp, ncp))
            n = 300
            u = rng.uniform(0, 1, size=(n, 3))
            kv = bspline.clamped_knots(ncp, degree)
            edge = [0.0, 1.0, -0.3, 1.25] + [float(x) for x in kv[degree:ncp + 1]]
            e = np.array([[a, edge[(i + 1) % len(edge)], edge[(i + 2) % len(edge)]] for i, a in enumerate(edge)])
            u = np.vstack([u, e])
            # default knots (float64 uniform) and stored float32 knots
            v0 = bspline.evaluate_points(coeff, degree, u)
            v1, g1 = bspline.evaluate_points_with_gradient(coeff, degree, u)
            k32 = np.repeat(kv.astype(np.float32)[None, :], 3, axis=0)
            v2, g2 = bspline.evaluate_points_with_gradient(coeff.astype(np.float32), degree, u,
                                                           knots=tuple(k32.astype(np.float64)))
            out[f"c{ci}_coeff"] = coeff.astype(np.float32)
            out[f"c{ci}_coeff64"] = coeff
            out[f"c{ci}_u"] = u
            out[f"c{ci}_v_default"] = v0
            out[f"c{ci}_v"] = v1
            out[f"c{ci}_g"] = g1
            out[f"c{ci}_knots32"] = k32
            out[f"c{ci}_v32"] = v2
            out[f"c{ci}_g32"] = g2
            spans = bspline.find_spans(kv, ncp, degree, np.clip(u[:, 0], 0, 1))
            bv, bd = bspline.basis_values_and_derivatives(kv, degree, spans, np.clip(u[:, 0], 0, 1))
            out[f"c{ci}_spans"] = spans
            out[f"c{ci}_bv"] = bv
            out[f"c{ci}_bd"] = bd
            cases.append((degree, ncp))
            ci += 1
    # non-uniform stored knots (FORMAT.md:53-55: general interiors round-trip)
    degree, ncp = 3, 9
    interior = np.sort(rng.uniform(0.05, 0.95, size=ncp - degree - 1))
    kv = np.concatenate([np.zeros(degree + 1), interior, np.ones(degree + 1)]).astype(np.float32)
    knots = np.stack([kv, np.roll(kv, 0), kv])
    knots[1, degree + 1:ncp] = np.sort(rng.uniform(0.05, 0.95, size=ncp - degree - 1)).astype(np.float32)
    coeff = rng.normal(size=(ncp, ncp, ncp)).astype(np.float32)
    u = rng.uniform(-0.1, 1.1, size=(400, 3))
    v, g = bspline.evaluate_points_with_gradient(coeff, degree, u, knots=tuple(knots.astype(np.float64)))
    out["nu_coeff"], out["nu_knots"], out["nu_u"], out["nu_v"], out["nu_g"] = coeff, knots, u, v, g
    out["nu_degree"] = np.array(degree)
    out["cases"] = np.array(cases)

    # decode_grid (model.py:89-93) on MicroModels built by the reference fit
    dec = []
    for j, (ncp, degree, m) in enumerate([(3, 2, 5), (6, 2, 8), (8, 2, 8), (12, 3, 17), (17, 3, 17), (9, 1, 9), (10, 3, 33)]):
        samples = sample_grid(marschner_lobb(), (m, m, m)).samples
        mm = model.fit(samples, ncp=ncp, degree=degree, extent=[[-1, 1]] * 3, lod=1)
        out[f"d{j}_control"] = mm.control
        out[f"d{j}_grid"] = mm.decode_grid((m, m, m))
        # MicroModel world-space hooks with a non-unit extent (model.py:64-87)
        ext = np.array([[-0.5, 0.25], [0.0, 0.5], [-1.0, -0.25]])
        mw = model.MicroModel(degree=degree, knots=mm.knots, control=mm.control, extent=ext, lod=2)
        pts = rng.uniform(-1.1, 1.1, size=(200, 3))
        out[f"d{j}_pts"] = pts
        out[f"d{j}_values_at"] = mw.values_at(pts)
        out[f"d{j}_gradients_at"] = mw.gradients_at(pts)
        out[f"d{j}_knots"] = mm.knots
        dec.append((ncp, degree, m))
    out["dcases"] = np.array(dec)
    np.savez_compressed(OUT / "bspline.npz", **out)
    print("bspline.npz written", flush=True)


# ------------------------------------------------------------------ visibility
def gen_visible(stores):
    out = {}
    mans = {
        "smooth33": stores["smooth33"][0],
        "ml65_p3": stores["ml65_p3"][0],
        "config3": skeleton_manifest(4, 2, 65),
        "config2": skeleton_manifest(2, 2, 65),
    }
    rng = np.random.default_rng(7)
    povs = []
    for radius in (2.0, 1.3, 3.0):
        povs += runtime.orbit_trajectory(100, radius=radius)
    for _ in range(150):
        pos = rng.uniform(-4, 4, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        fov = float(rng.uniform(20, 100))
        try:
            povs.append(render.PointOfView(pos, d, [0, 1, 0], fov))
        except ValueError:
            pass
    povs.append(render.PointOfView([0.6, 0.5, 1.2], [-0.6, -0.5, -1.2], [0, 1, 0]))
    povs.append(render.PointOfView([2.0, 1.6, 2.6], [-0.55, -0.44, -0.71], [0, 1, 0]))
    out["povs"] = np.array([[*p.position, *p.direction, *p.up, p.fov_y] for p in povs])
    for name, man in mans.items():
        out[f"{name}_manifest"] = np.frombuffer(json.dumps(man.to_json()).encode(), dtype=np.uint8)
        rows = []
        for pi, pov in enumerate(povs):
            for aspect in (1.0, 1.5):
                vis = render.select_visible(pov, man, aspect)
                for a in vis:
                    rows.append((pi, int(aspect * 2), a.lod, *a.ijk))
        out[f"{name}_vis"] = np.array(rows, dtype=np.int32).reshape(-1, 6)
        # custom ranges (render.py:256-261)
        rows = []
        for pi, pov in enumerate(povs[:40]):
            for ri, ranges in enumerate([(1e-9, 2e-9, 3e-9), (1e9, 2e9, 3e9), (0.5, 1.0, 1.7)]):
                rr = ranges[: man.levels - 1]
                vis = render.select_visible(pov, man, 1.0, ranges=rr)
                for a in vis:
                    rows.append((pi, ri, a.lod, *a.ijk))
        out[f"{name}_vis_ranges"] = np.array(rows, dtype=np.int32).reshape(-1, 6)
        print(f"visible {name}: {len(out[f'{name}_vis'])} rows", flush=True)
    # lod_for_distance frozen values (render.py:256-261)
    ds = np.concatenate([np.linspace(0, 4, 401), [0.8, 1.6, 2.4, 3.2, np.nextafter(0.8, 0), np.nextafter(1.6, 0)]])
    out["lod_d"] = ds
    out["lod_l4"] = np.array([render.lod_for_distance(float(d), 4) for d in ds])
    out["lod_l2"] = np.array([render.lod_for_distance(float(d), 2) for d in ds])
    np.savez_compressed(OUT / "visible.npz", **out)


# ------------------------------------------------------------------ frames
class Counting:
    """Wraps a MicroModel to count the samples render() decodes (values_at)."""

    def __init__(self, m, counter):
        self.m, self.c = m, counter
        self.extent = m.extent

    def values_at(self, pts):
        self.c[0] += len(pts)
        return self.m.values_at(pts)

    def gradients_at(self, pts):
        return self.m.gradients_at(pts)


def gen_frames(stores):
    out = {}
    jobs = []
    tf_ml = render.TransferFunction.ml_preset()
    tf_alt = render.TransferFunction(
        color_points=[[0.0, 0.9, 0.1, 0.1], [0.45, 0.2, 0.8, 0.3], [0.7, 0.1, 0.3, 0.9], [1.0, 1.0, 1.0, 1.0]],
        opacity_points=[[0.0, 0.0], [0.3, 0.05], [0.55, 0.6], [0.8, 0.1], [1.0, 0.3]],
        domain=(0.1, 0.9),
    )
    P = render.PointOfView
    jobs.append(("smooth_a", "smooth33", P([0.4, 0.3, 2.0], [-0.1, -0.1, -1.0], [0, 1, 0]), tf_ml,
                 render.RenderParams(width=32, height=32, sample_distance=0.01)))
    jobs.append(("smooth_b", "smooth33", P([2.5, 0.1, 2.5], [-0.7, 0, -0.7], [0, 1, 0], 50.0), tf_alt,
                 render.RenderParams(width=40, height=24, sample_distance=0.008, o_max=1.0)))
    jobs.append(("smooth_c", "smooth33", P([0.5, 0.5, 1.1], [0, 0, -1], [0, 1, 0], 60.0), tf_ml,
                 render.RenderParams(width=24, height=24, sample_distance=0.005, reference_step=0.01,
                                     ambient=0.2, diffuse=0.6, specular=0.3, shininess=16.0)))
    jobs.append(("ml_a", "ml65_p3", P([0.6, 0.5, 1.2], [-0.6, -0.5, -1.2], [0, 1, 0]), tf_ml,
                 render.RenderParams(width=32, height=32, sample_distance=0.01)))
    jobs.append(("ml_b", "ml65_p3", P([2.0, 1.6, 2.6], [-0.55, -0.44, -0.71], [0, 1, 0]), tf_ml,
                 render.RenderParams(width=32, height=24, sample_distance=0.004)))
    jobs.append(("ml_c", "ml65_p3", P([0.1, -0.2, 1.6], [0.05, 0.1, -1.0], [0, 1, 0], 70.0), tf_alt,
                 render.RenderParams(width=28, height=28, sample_distance=0.006, o_max=1.0)))
    jobs.append(("c1_a", "config1", P([0.0, 0.0, 3.0], [0, 0, -1], [0, 1, 0]), tf_ml,
                 render.RenderParams(width=32, height=32, sample_distance=0.01)))
    jobs.append(("const_multi", "const_multi", P([0, 0, 4.0], [0, 0, -1], [0, 1, 0]), tf_ml,
                 render.RenderParams(width=24, height=24, sample_distance=0.02)))
    jobs.append(("const_single", "const_single", P([0, 0, 4.0], [0, 0, -1], [0, 1, 0]), tf_ml,
                 render.RenderParams(width=24, height=24, sample_distance=0.02)))
    names = []
    for name, store, pov, tf, params in jobs:
        man, models = stores[store]
        vis = render.select_visible(pov, man, params.aspect)
        counter = [0]
        resident = {a: Counting(models[a], counter) for a in vis}
        t = time.time()
        fr = render.render(pov, resident, tf, params)
        print(f"frame {name}: {params.width}x{params.height} {counter[0]} samples {time.time() - t:.1f}s", flush=True)
        out[f"{name}_rgba"] = fr.rgba
        out[f"{name}_samples"] = np.array(counter[0])
        out[f"{name}_pov"] = np.array([*pov.position, *pov.direction, *pov.up, pov.fov_y])
        out[f"{name}_params"] = np.array([params.width, params.height, params.sample_distance, params.o_max,
                                          params.reference_step if params.reference_step is not None else np.nan,
                                          params.near, params.ambient, params.diffuse, params.specular,
                                          params.shininess])
        out[f"{name}_tf"] = np.frombuffer(json.dumps(tf.to_json()).encode(), dtype=np.uint8)
        out[f"{name}_store"] = np.array(store)
        out[f"{name}_vis"] = np.array([(a.lod, *a.ijk) for a in vis], dtype=np.int32)
        names.append(name)
    # MissingBlockError (render.py:430-436, tests/test_render.py:354-362)
    man, models = stores["smooth33"]
    pov = P([0, 0, 5.0], [0, 0, -1], [0, 1, 0])
    vis = render.select_visible(pov, man)
    resident = {a: models[a] for a in vis}
    resident.pop(vis[0])
    try:
        render.render(pov, resident, tf_ml, render.RenderParams(width=8, height=8, sample_distance=0.05))
        msg = ""
    except MissingBlockError as exc:
        msg = str(exc)
    out["missing_msg"] = np.array(msg)
    out["missing_dropped"] = np.array([vis[0].lod, *vis[0].ijk])
    out["names"] = np.array(names)
    np.savez_compressed(OUT / "frames.npz", **out)


def main():
    t0 = time.time()
    gen_bspline()
    stores = build_stores()
    gen_visible(stores)
    gen_frames(stores)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
