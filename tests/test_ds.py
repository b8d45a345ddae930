"""Down-sampled (DS) baseline (reference downsample.py): store format and
build on the CPU; GPU render of DS blocks (AFAM_SLOT_DS, trilinear values
and central-difference gradients) against the reference's own frames
(tests/golden/gen_ds_golden.py)."""

import json

import numpy as np
import pytest

from helpers import npz

Z = npz("ds.npz")
NAMES = [str(n) for n in Z["names"]]


def _store(g):
    from paper_2409_00184_b200 import downsample, partition

    man = partition.LODManifest.from_json(json.loads(bytes(Z[f"store_g{g}_manifest"]).decode()))
    blob = bytes(Z[f"store_g{g}_blob"])
    offs = Z[f"store_g{g}_offsets"]
    raw, blocks = {}, {}
    for i, key in enumerate(Z[f"store_g{g}_keys"]):
        a = partition.BlockAddress.from_key(str(key))
        raw[a] = blob[offs[i]:offs[i + 1]]
        blocks[a] = downsample.deserialize_ds(raw[a], man.entries[a].extent, a.lod)
    return man, raw, blocks


def test_ds_store_round_trip_and_errors():
    from paper_2409_00184_b200 import downsample
    from paper_2409_00184_b200.errors import FormatError

    man, raw, blocks = _store(1)
    assert man.kind == "ds" and man.ghost == 1
    for a, data in raw.items():
        assert downsample.serialize_ds(blocks[a]) == data
        assert blocks[a].nbytes == len(data) == man.entries[a].nbytes
    data = next(iter(raw.values()))
    with pytest.raises(FormatError, match="header missing"):
        downsample.deserialize_ds(data[:8], [[-1, 1]] * 3, 1)
    with pytest.raises(FormatError, match="length mismatch"):
        downsample.deserialize_ds(data[:-4], [[-1, 1]] * 3, 1)
    bad = bytearray(data)
    bad[12:16] = (2).to_bytes(4, "little")
    with pytest.raises(ValueError, match="ghost width"):
        downsample.deserialize_ds(bytes(bad), [[-1, 1]] * 3, 1)


def test_build_ds_store_matches_reference_bytes():
    """build_ds_store on the golden 33^3 volume reproduces the reference's
    block files byte for byte (ghosted, edge-clamped strided samples)."""
    from types import SimpleNamespace

    from paper_2409_00184_b200 import downsample

    ez = npz("encoder.npz")
    vol = SimpleNamespace(samples=ez["vol_samples"], bounds=ez["vol_bounds"])
    for g in (0, 1):
        man_ref, raw, _ = _store(g)
        man, blocks = downsample.build_ds_store(vol, levels=2, micro_dims=9, coarsest=2, ghost=g)
        assert sorted(blocks) == sorted(raw)
        for a in raw:
            assert downsample.serialize_ds(blocks[a]) == raw[a], (g, a)
            np.testing.assert_array_equal(man.entries[a].extent, man_ref.entries[a].extent)


def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_render_ds_vs_reference_frames(name, oracle):
    _cuda()
    from paper_2409_00184_b200 import render

    g = int(Z[f"{name}_ghost"])
    man, _, blocks = _store(g)
    pv = Z[f"{name}_pov"]
    pov = render.PointOfView(pv[0:3], pv[3:6], pv[6:9], float(pv[9]))
    w, h, sd, omax, ref, near, amb, dif, spe, shi = [float(v) for v in Z[f"{name}_params"]]
    params = render.RenderParams(width=int(w), height=int(h), sample_distance=sd, o_max=omax,
                                 reference_step=None if np.isnan(ref) else ref, near=near, ambient=amb,
                                 diffuse=dif, specular=spe, shininess=shi)
    vis = render.select_visible(pov, man, params.aspect)
    assert [(a.lod, *a.ijk) for a in vis] == [tuple(r) for r in Z[f"{name}_vis"]]
    frame = render.render(pov, {a: blocks[a] for a in vis}, render.TransferFunction.ml_preset(), params)
    assert render.render.last_stats["samples"] == int(Z[f"{name}_samples"])
    assert oracle.psnr(frame.rgba, Z[f"{name}_rgba"]) >= 60.0


@pytest.mark.gpu
def test_ds_device_loader_replay(tmp_path):
    """make_loader on a DS store with a DeviceStore: HBM-resident DS slots,
    replay frames equal a direct render of host DS blocks."""
    _cuda()
    from paper_2409_00184_b200 import downsample, render, runtime
    from paper_2409_00184_b200.device import DeviceStore

    man, raw, blocks = _store(1)
    downsample.write_ds_store(tmp_path, man, raw)
    ds = DeviceStore(20, 11)
    cache = runtime.ModelCache(16, runtime.make_loader(tmp_path, man, ds))
    povs = runtime.orbit_trajectory(3, radius=2.5)
    params = render.RenderParams(width=24, height=24, sample_distance=0.02)
    tf = render.TransferFunction.ml_preset()
    _, frames, agg = runtime.replay(povs, man, cache, tf, params, prefetch="off")
    assert agg["frames"] == 3
    for pov, fr in zip(povs, frames):
        vis = render.select_visible(pov, man, params.aspect)
        want = render.render(pov, {a: blocks[a] for a in vis}, tf, params)
        np.testing.assert_array_equal(fr.rgba, want.rgba)


@pytest.mark.gpu
def test_ds_point_queries_vs_reference():
    """DsBlock.values_at / gradients_at on the GPU (K1's DS branch) against
    the reference's trilinear queries (tests/golden/gen_ds_points_golden.py),
    ghost 0 and 1, points inside and around each block (clipped)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from helpers import npz

    from paper_2409_00184_b200 import downsample

    z = npz("ds_points.npz")
    for k in range(int(z["nblocks"])):
        b = downsample.DsBlock(z[f"b{k}_samples"], int(z[f"b{k}_ghost"]), z[f"b{k}_extent"], int(z[f"b{k}_lod"]))
        pts = z[f"b{k}_points"]
        v = b.values_at(pts)
        g = b.gradients_at(pts)
        want_v, want_g = z[f"b{k}_values"], z[f"b{k}_grads"]
        rng = max(1.0, float(np.abs(want_v).max()))
        assert np.abs(v - want_v).max() <= 1e-12 * rng, k
        # the central-difference grids are built once at upload and held in
        # float32 (as the DS render reads them): ~1e-8 relative vs float64
        assert np.abs(g - want_g).max() <= 1e-6 * max(1.0, float(np.abs(want_g).max())), k


@pytest.mark.gpu
def test_ds_scratch_store_keeps_the_calls_blocks():
    """Host DS blocks resolved in one call are pinned in the scratch store: a
    full store evicts only blocks of earlier calls and raises CapacityError
    when the call alone overflows it (never a slot reused within the call)."""
    _cuda()
    from paper_2409_00184_b200 import device, downsample
    from paper_2409_00184_b200.errors import CapacityError

    man, raw, blocks = _store(1)
    addrs = sorted(blocks)[:5]
    edge = max(max(blocks[a].samples.shape) for a in addrs)
    sc = device._ScratchStore(edge, 0)
    sc.store = device.DeviceStore(3, edge)
    first = {id(blocks[a]) for a in addrs[:3]}
    slots = [sc.get_ds(blocks[a], downsample.serialize_ds, first).slot for a in addrs[:3]]
    assert len(set(slots)) == 3
    # a new call with two other blocks evicts two of the earlier call's slots
    second = {id(blocks[a]) for a in addrs[3:5]}
    s2 = [sc.get_ds(blocks[a], downsample.serialize_ds, second).slot for a in addrs[3:5]]
    assert len(set(s2)) == 2
    # one call needing four slots of a three-slot store: CapacityError, no silent reuse
    allp = {id(blocks[a]) for a in addrs[:4]}
    with pytest.raises(CapacityError):
        for a in addrs[:4]:
            sc.get_ds(blocks[a], downsample.serialize_ds, allp)
    # DS scratch stores are sized by the sample edge, not a spline NCP bucket
    assert device.scratch_store(edge, 0, exact=True).store.max_ncp == edge


@pytest.mark.gpu
def test_ds_slots_reject_parameter_space_points():
    """Parameter-space evaluation needs a spline (a DS block has no
    parameter space): the per-point slots path raises like the single-slot
    one when a batch names a DS slot, and still evaluates spline-only
    batches of a store that also holds DS blocks."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from helpers import npz

    from paper_2409_00184_b200 import bspline, downsample, model
    from paper_2409_00184_b200.device import DeviceStore

    z = npz("ds_points.npz")
    b = downsample.DsBlock(z["b0_samples"], int(z["b0_ghost"]), z["b0_extent"], int(z["b0_lod"]))
    ds = DeviceStore(2, 65)
    ds.put_ds(0, downsample.serialize_ds(b), b.extent)
    c = np.random.default_rng(0).normal(size=(7, 7, 7)).astype(np.float32)
    m = model.MicroModel(3, np.stack([bspline.clamped_knots(7, 3)] * 3).astype(np.float32), c,
                         np.array([[0, 1.0]] * 3), 1)
    ds.put_model(1, m)
    u = np.random.default_rng(1).uniform(0, 1, size=(64, 3))
    with pytest.raises(ValueError, match="DS block"):
        bspline.eval_device(ds, 0, u, gradient=False, param=True)
    with pytest.raises(ValueError, match="DS block"):
        bspline.eval_device(ds, np.array([1, 0] * 32, dtype=np.int32), u, gradient=False, param=True)
    v = bspline.eval_device(ds, np.ones(64, dtype=np.int32), u, gradient=False, param=True)
    np.testing.assert_allclose(v, bspline.eval_device(ds, 1, u, gradient=False, param=True), rtol=0, atol=0)
