"""GPU tests of the out-of-core path: DeviceStore-backed ModelCache + replay
(reference runtime.py:228-293 semantics) on a store written to disk."""

import numpy as np
import pytest

from helpers import golden_store

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def disk_store(tmp_path_factory):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json

    from helpers import npz
    from paper_2409_00184_b200 import partition, store

    root = tmp_path_factory.mktemp("store")
    man, _, raw = golden_store("smooth33")
    pman = partition.LODManifest.from_json(json.loads(bytes(npz("store_smooth33.npz")["manifest"]).decode()))
    blobs = {partition.BlockAddress(a.lod, a.ijk): data for a, data in raw.items()}
    store.write_store(root, pman, blobs)
    return root, partition.LODManifest.load(root)


def _cache(root, manifest, cap):
    from paper_2409_00184_b200 import runtime
    from paper_2409_00184_b200.device import DeviceStore

    ds = DeviceStore(cap + 1, 9)
    return runtime.ModelCache(cap, runtime.make_loader(root, manifest, ds)), ds


def test_device_cache_replay_matches_direct_render(disk_store):
    from paper_2409_00184_b200 import render, runtime, store

    root, man = disk_store
    tf = render.TransferFunction.ml_preset()
    params = render.RenderParams(width=24, height=24, sample_distance=0.02)
    povs = runtime.orbit_trajectory(6, radius=3.0)
    cache, ds = _cache(root, man, 120)
    timings, frames, agg = runtime.replay(povs, man, cache, tf, params, prefetch="linear")
    assert agg["frames"] == 6 and timings[0].miss_rate == 1.0
    for t in timings:
        assert t.input_latency_ms == pytest.approx(t.caching_ms + t.rendering_ms, abs=1e-6)
    for pov, fr in zip(povs, frames):
        vis = render.select_visible(pov, man)
        host = {a: store.load_model(root, man, a) for a in vis}
        np.testing.assert_array_equal(fr.rgba, render.render(pov, host, tf, params).rgba)


def test_stationary_steady_state_and_slot_reuse(disk_store):
    from paper_2409_00184_b200 import render, runtime

    root, man = disk_store
    tf = render.TransferFunction.ml_preset()
    params = render.RenderParams(width=8, height=8, sample_distance=0.05)
    pov = render.PointOfView([0, 0, 4.0], [0, 0, -1], [0, 1, 0])
    cache, ds = _cache(root, man, 100)
    timings, _, _ = runtime.replay([pov] * 3, man, cache, tf, params, prefetch="static")
    assert [t.miss_rate for t in timings] == [1.0, 0.0, 0.0]
    # a small cache over an orbit evicts, and every eviction returns its slot
    cache, ds = _cache(root, man, 40)
    runtime.replay(runtime.orbit_trajectory(8, radius=1.5), man, cache, tf, params, keep_frames=False)
    assert cache.evictions > 0
    assert ds.free_slots() == ds.slots - len(cache)


def test_linear_prefetch_reduces_misses_on_dolly(disk_store):
    from paper_2409_00184_b200 import render, runtime

    root, man = disk_store
    tf = render.TransferFunction.ml_preset()
    # the prefetch loads only while the frame is on the GPU (the reference's
    # rendering_done check, runtime.py:186): frames big enough that a few
    # 9^3 block uploads fit in one
    params = render.RenderParams(width=256, height=256, sample_distance=0.002)
    povs = [render.PointOfView([0.3, 0.2, 3.2 - 0.05 * i], [0, 0, -1], [0, 1, 0]) for i in range(40)]
    off, _ = _cache(root, man, 500)
    runtime.replay(povs, man, off, tf, params, prefetch="off", keep_frames=False)
    on, _ = _cache(root, man, 500)
    _, frames_on, _ = runtime.replay(povs, man, on, tf, params, prefetch="linear")
    assert off.misses > 0 and on.misses < off.misses


def test_file_loader_round_trip_and_errors(disk_store, tmp_path):
    """afam_store_put_file (native pinned-staging reader) uploads exactly the
    file's model and keeps store.load_model's error semantics (store.py:33-47,
    model.py:121-148): missing / truncated file or bad degree byte ->
    FormatError, non-finite control points -> ValueError."""
    import shutil

    from paper_2409_00184_b200 import model, store
    from paper_2409_00184_b200.device import DeviceStore
    from paper_2409_00184_b200.errors import FormatError

    root, man = disk_store
    ds = DeviceStore(4, 9)
    load = store.device_loader(root, man, ds)
    for a in man.addresses()[:3]:
        blk = load(a)
        want = store.load_model(root, man, a)
        ctrl, knots = ds.read(blk.slot)
        np.testing.assert_array_equal(ctrl, want.control)
        np.testing.assert_array_equal(knots, want.knots)
        assert blk.degree == want.degree and blk.ncp == want.ncp
        ds.release(blk.slot)
    # corrupt copies of one block file
    a = man.addresses()[0]
    work = tmp_path / "s"
    shutil.copytree(root, work)
    path = work / man.entries[a].path
    data = bytearray(path.read_bytes())
    bad = store.device_loader(work, man, ds)
    path.write_bytes(bytes(data[:-4]))
    with pytest.raises(FormatError, match="length mismatch"):
        bad(a)
    path.write_bytes(bytes([man.entries[a].ncp]) + bytes(data[1:]))
    with pytest.raises(FormatError, match="degree byte"):
        bad(a)
    nan = bytearray(data)
    off = 1 + 12 * (man.entries[a].ncp + data[0])
    nan[off:off + 4] = np.array([np.nan], dtype="<f4").tobytes()
    path.write_bytes(bytes(nan))
    with pytest.raises(ValueError, match="non-finite"):
        bad(a)
    path.unlink()
    with pytest.raises(FormatError, match="missing model file"):
        bad(a)
    assert ds.free_slots() == 4
    assert model is not None
