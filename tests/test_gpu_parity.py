"""GPU parity of the B200 path against the reference's golden vectors and the
float64 oracle.  Gates (BASELINE.json north_star): decoded values within
1e-5 x data range, frames PSNR >= 60 dB, block/LOD selection bit-exact."""

import json

import numpy as np
import pytest

from helpers import Addr, golden_store, npz, params_ns, pov_ns, tf_ns

pytestmark = pytest.mark.gpu

VALUE_TOL = 1e-5  # x data range; all stores here have values in ~[0, 1]


def _torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def cuda():
    return _torch_cuda()


def _to_product(models):
    from paper_2409_00184_b200 import model
    from paper_2409_00184_b200.partition import BlockAddress

    return {BlockAddress(a.lod, a.ijk): model.MicroModel(m.degree, m.knots, m.control, m.extent, a.lod)
            for a, m in models.items()}


# ----------------------------------------------------------------- store (K4)
def test_store_round_trip_and_flags(cuda):
    from paper_2409_00184_b200.device import DeviceStore

    man, models, raw = golden_store("ml65_p3")
    ds = DeviceStore(len(raw), 17)
    for a, data in raw.items():
        blk = ds.load_mfa(data, man.entries[a].ncp, man.entries[a].extent, a.lod)
        ctrl, knots = ds.read(blk.slot)
        np.testing.assert_array_equal(ctrl, models[a].control)
        np.testing.assert_array_equal(knots, models[a].knots)
        info = ds.info(blk.slot)
        assert info["max_abs_ctrl"] == pytest.approx(float(np.abs(models[a].control).max()))
        assert info["fp64"] == (info["max_abs_ctrl"] > 4.0)


def test_store_rejects_bad_images(cuda):
    from paper_2409_00184_b200.device import DeviceStore
    from paper_2409_00184_b200.errors import CapacityError, FormatError

    man, models, raw = golden_store("smooth33")
    a, data = next(iter(raw.items()))
    ds = DeviceStore(2, 9)
    with pytest.raises(FormatError, match="length mismatch"):
        ds.put_mfa(0, data[:-4], man.entries[a].ncp, man.entries[a].extent)
    with pytest.raises(FormatError, match="degree byte"):
        ds.put_mfa(0, bytes([40]) + data[1:], man.entries[a].ncp, man.entries[a].extent)
    ds.alloc(), ds.alloc()
    with pytest.raises(CapacityError):
        ds.alloc()


# ----------------------------------------------------------------- K1 points
def test_eval_points_vs_reference_golden(cuda):
    from paper_2409_00184_b200 import bspline

    z = npz("bspline.npz")
    for ci, (degree, ncp) in enumerate(z["cases"]):
        c = z[f"c{ci}_coeff"]
        u = z[f"c{ci}_u"]
        rng_ = max(1.0, float(np.abs(c).max()))
        v, g = bspline.evaluate_points_with_gradient(c, int(degree), u, knots=tuple(z[f"c{ci}_knots32"]))
        assert np.abs(v - z[f"c{ci}_v32"]).max() <= VALUE_TOL * rng_
        # gradients to the value gate relative to the gradient range (measured worst 9e-7,
        # tools/diag_gradtol.py)
        gr = z[f"c{ci}_g32"]
        np.testing.assert_allclose(g, gr, rtol=0, atol=VALUE_TOL * max(1.0, float(np.abs(gr).max())))
        v0 = bspline.evaluate_points(c, int(degree), u)
        assert np.abs(v0 - z[f"c{ci}_v_default"]).max() <= VALUE_TOL * rng_
    v, g = bspline.evaluate_points_with_gradient(z["nu_coeff"], int(z["nu_degree"]), z["nu_u"],
                                                 knots=tuple(z["nu_knots"]))
    assert np.abs(v - z["nu_v"]).max() <= VALUE_TOL * float(np.abs(z["nu_coeff"]).max())


def test_world_space_hooks_vs_reference_golden(cuda):
    from paper_2409_00184_b200 import model

    z = npz("bspline.npz")
    ext = np.array([[-0.5, 0.25], [0.0, 0.5], [-1.0, -0.25]])
    for j, (ncp, degree, m) in enumerate(z["dcases"]):
        mw = model.MicroModel(int(degree), z[f"d{j}_knots"], z[f"d{j}_control"], ext, 2)
        scale = float(np.abs(z[f"d{j}_control"]).max())
        tol = VALUE_TOL * max(1.0, scale / 4.0)
        assert np.abs(mw.values_at(z[f"d{j}_pts"]) - z[f"d{j}_values_at"]).max() <= tol
        g = mw.gradients_at(z[f"d{j}_pts"])
        gr = z[f"d{j}_gradients_at"]
        assert np.abs(g - gr).max() <= VALUE_TOL * max(1.0, np.abs(gr).max())  # measured worst 1e-6


def test_eval_points_ill_conditioned_fp64_path(cuda, oracle):
    """ncp = m = 65, degree 3: max|c| ~ 1e4..1e7; the fp64 path must hold 1e-5."""
    from paper_2409_00184_b200 import bspline, synth
    from paper_2409_00184_b200.device import DeviceStore

    man, blobs = synth.field_store(levels=1, coarsest=1, micro=65, degree=3, ncp_of=lambda a: 65)
    a = next(iter(blobs))
    ds = DeviceStore(1, 65)
    blk = ds.load_mfa(blobs[a], 65, man.entries[a].extent, 1)
    info = ds.info(blk.slot)
    assert info["fp64"] and info["max_abs_ctrl"] > 100
    ctrl, knots = ds.read(blk.slot)
    u = np.random.default_rng(1).uniform(0, 1, size=(20000, 3))
    v, g = bspline.eval_device(ds, blk.slot, u, gradient=True, param=True)
    vr, gr = oracle.eval_points(ctrl, 3, u, knots=knots)
    assert np.abs(v - vr).max() <= VALUE_TOL


# ----------------------------------------------------------------- K3 decode
def test_decode_grid_vs_reference_golden(cuda):
    from paper_2409_00184_b200 import model

    z = npz("bspline.npz")
    for j, (ncp, degree, m) in enumerate(z["dcases"]):
        mm = model.MicroModel(int(degree), z[f"d{j}_knots"], z[f"d{j}_control"], [[-1, 1]] * 3, 1)
        got = mm.decode_grid((int(m),) * 3)
        want = z[f"d{j}_grid"]
        assert got.shape == want.shape
        assert np.abs(got - want).max() <= VALUE_TOL * max(1.0, float(np.abs(want).max()))


def test_decode_non_cubic_dims_vs_oracle(cuda, oracle):
    """decode_grid / decode_tensor_product on non-cubic dims (the reference
    accepts any dims triple, bspline.py:162-172): linspace(0, 1, 9) and
    linspace(0, 1, 5) are exact sub-lattices of linspace(0, 1, 17), so the
    (9, 17, 5) decode is the oracle's 17^3 decode strided."""
    from paper_2409_00184_b200 import bspline, model

    rng = np.random.default_rng(11)
    for degree, ncp in ((2, 7), (3, 12), (1, 5)):
        ctrl = rng.random((ncp, ncp, ncp)).astype(np.float32)
        want = oracle.decode_grid(ctrl, degree, 17)[::2, :, ::4]
        got = bspline.decode_tensor_product(ctrl, degree, (9, 17, 5))
        assert got.shape == (9, 17, 5)
        assert np.abs(got - want).max() <= VALUE_TOL
        knots = np.repeat(bspline.clamped_knots(ncp, degree)[None, :], 3, axis=0).astype(np.float32)
        mm = model.MicroModel(degree, knots, ctrl, [[-1, 1]] * 3, 1)
        assert np.abs(mm.decode_grid((9, 17, 5)) - want).max() <= VALUE_TOL
        one = mm.decode_grid((1, 17, 17))  # a single u = 0 plane
        assert np.abs(one - oracle.decode_grid(ctrl, degree, 17)[:1]).max() <= VALUE_TOL


def test_decode_config1_all_blocks_vs_oracle(cuda, oracle):
    """BASELINE config 1: all 729 blocks of the 64^3 ML store, 8^3 lattice."""
    from paper_2409_00184_b200.bspline import decode_slots
    from paper_2409_00184_b200.device import DeviceStore

    man, models, raw = golden_store("config1")
    ds = DeviceStore(len(raw), 8)
    addrs = sorted(raw)
    slots = [ds.load_mfa(raw[a], man.entries[a].ncp, man.entries[a].extent, a.lod).slot for a in addrs]
    got = decode_slots(ds, slots, 8)
    for b, a in enumerate(addrs):
        want = oracle.decode_grid(models[a].control, models[a].degree, 8)
        assert np.abs(got[b] - want).max() <= VALUE_TOL


def test_decode_ill_conditioned_vs_oracle(cuda, oracle):
    from paper_2409_00184_b200 import synth
    from paper_2409_00184_b200.bspline import decode_slots
    from paper_2409_00184_b200.device import DeviceStore

    man, blobs = synth.field_store(levels=2, coarsest=1, micro=65, degree=3,
                                   ncp_of=lambda a: 64 if a.lod == 1 else 65)
    ds = DeviceStore(len(blobs), 65)
    addrs = sorted(blobs)[:3]
    slots = [ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod).slot for a in addrs]
    got = decode_slots(ds, slots, 65)
    for b, s in enumerate(slots):
        ctrl, _ = ds.read(s)
        want = oracle.decode_grid(ctrl, 3, 65)
        assert np.abs(got[b] - want).max() <= VALUE_TOL


@pytest.mark.parametrize("degree", [1, 2, 3])
def test_decode_tensor_cores_vs_oracle(cuda, oracle, degree):
    """K3 tcgen05 path (3xTF32 x stage) on the 65^3 lattice: every block given
    to the tensor cores, values within 1e-5 of the float64 oracle and of the
    CUDA-core kernel."""
    from paper_2409_00184_b200 import synth
    from paper_2409_00184_b200.bspline import decode_slots
    from paper_2409_00184_b200.device import DeviceStore

    sizes = [degree + 2, 17, 33, 40, 48, 57, 60, 64 if degree < 3 else 52]
    man, blobs = synth.field_store(levels=1, coarsest=2, micro=65, degree=degree,
                                   ncp_of=lambda a: sizes[(a.ijk[0] * 2 + a.ijk[1]) * 2 + a.ijk[2]])
    ds = DeviceStore(len(blobs), 65)
    addrs = sorted(blobs)
    slots = [ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod).slot for a in addrs]
    info = {}
    got = decode_slots(ds, slots, 65, path="tensor_cores", info=info)
    assert info["tensor_core_blocks"] == len(slots)
    ref = decode_slots(ds, slots, 65, path="cuda_cores")
    for b, s in enumerate(slots):
        ctrl, _ = ds.read(s)
        want = oracle.decode_grid(ctrl, degree, 65)
        assert np.abs(got[b] - want).max() <= VALUE_TOL, (b, ctrl.shape[0])
        assert np.abs(got[b] - ref[b]).max() <= VALUE_TOL


def test_decode_tensor_cores_other_lattice_falls_back(cuda, oracle):
    """m != 65: the tensor-core request falls back to the CUDA-core kernel."""
    from paper_2409_00184_b200 import synth
    from paper_2409_00184_b200.bspline import decode_slots
    from paper_2409_00184_b200.device import DeviceStore

    man, blobs = synth.field_store(levels=1, coarsest=1, micro=9, degree=3, ncp_of=lambda a: 7)
    ds = DeviceStore(len(blobs), 9)
    a = sorted(blobs)[0]
    slot = ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod).slot
    info = {}
    got = decode_slots(ds, [slot], 33, path="tensor_cores", info=info)
    assert info["tensor_core_blocks"] == 0
    ctrl, _ = ds.read(slot)
    assert np.abs(got[0] - oracle.decode_grid(ctrl, 3, 33)).max() <= VALUE_TOL


# ----------------------------------------------------------------- K2 render
FRAME_NAMES = list(npz("frames.npz")["names"])


@pytest.mark.parametrize("name", FRAME_NAMES)
def test_render_vs_reference_frames(cuda, oracle, name):
    from paper_2409_00184_b200 import render

    z = npz("frames.npz")
    man, models, _ = golden_store(str(z[f"{name}_store"]))
    pm = _to_product(models)
    vis = [tuple(int(v) for v in r) for r in z[f"{name}_vis"]]
    from paper_2409_00184_b200.partition import BlockAddress

    resident = {BlockAddress(v[0], v[1:]): pm[BlockAddress(v[0], v[1:])] for v in vis}
    p = params_ns(z[f"{name}_params"])
    params = render.RenderParams(width=p.width, height=p.height, sample_distance=p.sample_distance, o_max=p.o_max,
                                 reference_step=p.reference_step, near=p.near, ambient=p.ambient,
                                 diffuse=p.diffuse, specular=p.specular, shininess=p.shininess)
    t = tf_ns(z[f"{name}_tf"])
    tf = render.TransferFunction(t.color_points, t.opacity_points, t.domain)
    frame = render.render(pov_ns(z[f"{name}_pov"]), resident, tf, params)
    want = z[f"{name}_rgba"]
    assert oracle.psnr(frame.rgba, want) >= 60.0
    assert np.abs(frame.rgba[..., 3].astype(int) - want[..., 3].astype(int)).max() <= 2
    if p.o_max == 1.0:  # no early termination: the sample set is pure float64 geometry
        assert render.render.last_stats["samples"] == int(z[f"{name}_samples"])


def test_constant_volume_multi_vs_single_identical(cuda):
    from paper_2409_00184_b200 import render

    z = npz("frames.npz")
    frames = []
    for name in ("const_multi", "const_single"):
        man, models, _ = golden_store(name)
        pm = _to_product(models)
        pov = pov_ns(z[f"{name}_pov"])
        vis = render.select_visible(pov, man)
        frames.append(render.render(pov, {a: pm[a] for a in vis}, render.TransferFunction.ml_preset(),
                                    render.RenderParams(width=24, height=24, sample_distance=0.02)).rgba)
        np.testing.assert_array_equal(frames[-1], z[f"{name}_rgba"])
    np.testing.assert_array_equal(frames[0], frames[1])


def test_missing_block_message_matches_reference(cuda):
    from paper_2409_00184_b200 import render
    from paper_2409_00184_b200.errors import MissingBlockError
    from paper_2409_00184_b200.partition import BlockAddress

    z = npz("frames.npz")
    man, models, _ = golden_store("smooth33")
    pm = _to_product(models)
    pov = render.PointOfView([0, 0, 5.0], [0, 0, -1], [0, 1, 0])
    vis = render.select_visible(pov, man)
    resident = {a: pm[a] for a in vis}
    d = [int(v) for v in z["missing_dropped"]]
    resident.pop(BlockAddress(d[0], d[1:]))
    with pytest.raises(MissingBlockError, match="finest cell") as exc:
        render.render(pov, resident, render.TransferFunction.ml_preset(),
                      render.RenderParams(width=8, height=8, sample_distance=0.05))
    assert str(exc.value) == str(z["missing_msg"])


def _owner_check(oracle, pov, resident, tf, params, rows=None):
    from paper_2409_00184_b200 import render

    out, info, dbg = render.render_part(pov, resident, tf, params, debug=True)
    want, oinfo = oracle.render(pov, resident, tf, params, debug=True)
    ns = dbg["nsamp"].cpu().numpy().ravel()
    oh = dbg["ohash"].cpu().numpy().view(np.uint64).ravel()
    return out.cpu().numpy(), want, info, oinfo, ns, oh


def test_owner_selection_bit_exact_golden_store(cuda, oracle):
    from paper_2409_00184_b200 import render

    man, models, _ = golden_store("smooth33")
    pm = _to_product(models)
    rng = np.random.default_rng(5)
    for _ in range(4):
        pos = rng.uniform(-2.5, 2.5, 3)
        pos[2] = abs(pos[2]) + 1.2
        pov = render.PointOfView(pos, -pos + rng.normal(scale=0.2, size=3), [0, 1, 0], float(rng.uniform(30, 70)))
        vis = render.select_visible(pov, man)
        resident = {a: pm[a] for a in vis}
        params = render.RenderParams(width=40, height=32, sample_distance=0.007, o_max=1.0)
        got, want, info, oinfo, ns, oh = _owner_check(oracle, pov, resident, render.TransferFunction.ml_preset(),
                                                      params)
        np.testing.assert_array_equal(ns, oinfo["nsamp"])
        np.testing.assert_array_equal(oh, oinfo["ohash"])
        assert info["samples"] == oinfo["samples"]
        assert oracle.psnr(got, want) >= 60.0


def test_ill_conditioned_render_config2_geometry(cuda, oracle):
    """Config-2 geometry (2 LODs, micro 65, degree 3) with ncp 64/65 blocks."""
    from paper_2409_00184_b200 import model, render, synth

    man, blobs = synth.field_store(levels=2, coarsest=2, micro=65, degree=3,
                                   ncp_of=lambda a: 65 if a.lod == 2 else 44 + (sum(a.ijk) % 20))
    pov = render.PointOfView([0.6, 0.5, 1.2], [-0.6, -0.5, -1.2], [0, 1, 0])
    vis = render.select_visible(pov, man)
    resident = {a: model.deserialize(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in vis}
    assert {a.lod for a in vis} == {1, 2}
    params = render.RenderParams(width=48, height=48, sample_distance=0.004, o_max=1.0)
    got, want, info, oinfo, ns, oh = _owner_check(oracle, pov, resident, render.TransferFunction.ml_preset(),
                                                  params)
    assert info["fp64_samples"] > 0
    np.testing.assert_array_equal(ns, oinfo["nsamp"])
    np.testing.assert_array_equal(oh, oinfo["ohash"])
    assert oracle.psnr(got, want) >= 60.0


def test_config3_band_vs_oracle(cuda, oracle):
    """A row band of a config-3 (4,680-block turbulence) 1024^2 frame vs the oracle."""
    from paper_2409_00184_b200 import render, runtime, synth
    from paper_2409_00184_b200.device import DeviceStore

    man, blobs = synth.turbulence_store()
    pov = runtime.orbit_trajectory(100, radius=2.0)[7]
    vis = render.select_visible(pov, man)
    ds = DeviceStore(len(vis), 65)
    resident = {a: ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in vis}
    params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3, o_max=1.0)
    tf = render.TransferFunction.ml_preset()
    out, info, dbg = render.render_part(pov, resident, tf, params, band_rows=8, nparts=64, part=37, debug=True)
    # rows of part 37: bands 37, 101, ... -> compare the first band (rows 296..303)
    from paper_2409_00184_b200.model import deserialize

    host = {a: deserialize(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in vis}
    want, oinfo = oracle.render(pov, host, tf, params, rows=(296, 304), debug=True)
    got = out.cpu().numpy()[:8]
    assert oracle.psnr(got, want) >= 60.0
    np.testing.assert_array_equal(dbg["nsamp"].cpu().numpy()[:8].ravel(), oinfo["nsamp"])
    np.testing.assert_array_equal(dbg["ohash"].cpu().numpy()[:8].view(np.uint64).ravel(), oinfo["ohash"])


def test_parts_stitch_to_full_frame(cuda):
    from paper_2409_00184_b200 import render

    man, models, _ = golden_store("ml65_p3")
    pm = _to_product(models)
    pov = render.PointOfView([0.6, 0.5, 1.2], [-0.6, -0.5, -1.2], [0, 1, 0])
    vis = render.select_visible(pov, man)
    resident = {a: pm[a] for a in vis}
    params = render.RenderParams(width=64, height=50, sample_distance=0.01)
    tf = render.TransferFunction.ml_preset()
    full = render.render(pov, resident, tf, params).rgba
    for nparts, br in ((2, 8), (3, 4), (8, 1)):
        stitched = np.zeros_like(full)
        for part in range(nparts):
            out, _, _ = render.render_part(pov, resident, tf, params, band_rows=br, nparts=nparts, part=part)
            rows = [r for b in range(part, (50 + br - 1) // br, nparts) for r in range(b * br, min(50, (b + 1) * br))]
            stitched[rows] = out.cpu().numpy()
        np.testing.assert_array_equal(stitched, full)


def test_constant_volume_closed_form(cuda):
    """20 equal samples of a constant field: A = 1-(1-a)^20, C = ambient*c*A
    (reference tests/test_render.py:239-254) with a spline constant block."""
    from paper_2409_00184_b200 import model, render
    from paper_2409_00184_b200.bspline import clamped_knots
    from paper_2409_00184_b200.partition import BlockAddress

    kv = np.repeat(clamped_knots(4, 2)[None].astype(np.float32), 3, axis=0)
    blk = model.MicroModel(2, kv, np.full((4, 4, 4), 0.5, np.float32), [[-1, 1]] * 3, 1)
    a_tf = 0.3
    tf = render.TransferFunction([[0.0, 0.8, 0.4, 0.2], [1.0, 0.8, 0.4, 0.2]], [[0.0, a_tf], [1.0, a_tf]])
    params = render.RenderParams(width=2, height=2, sample_distance=0.1, o_max=1.0)
    fr = render.render(render.PointOfView([0, 0, 4.0], [0, 0, -1], [0, 1, 0]), {BlockAddress(1, (0, 0, 0)): blk}, tf,
                       params)
    A = 1.0 - (1.0 - a_tf) ** 20
    want = np.rint(255.0 * np.r_[np.array([0.8, 0.4, 0.2]) * 0.1 * A, A])
    np.testing.assert_allclose(fr.rgba[1, 1].astype(float), want, atol=1.0)
