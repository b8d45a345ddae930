"""Host-side semantics of the out-of-core runtime (reference runtime.py:57-225),
checked on CPU with stand-in loaders: LRU order and counters against a
textbook LRU, pinning, the load hook, capacity errors, prefetch preemption
and fault tolerance, and the camera predictors."""

import json
import threading
from collections import OrderedDict

import numpy as np
import pytest

from helpers import npz


class Blob:
    def __init__(self, key, nbytes=100):
        self.key, self.nbytes = key, nbytes


def load_blob(key):
    return Blob(key)


class TextbookLRU:
    def __init__(self, cap):
        self.cap, self.d, self.hits, self.misses, self.evictions = cap, OrderedDict(), 0, 0, 0

    def touch(self, k):
        if k in self.d:
            self.d.move_to_end(k)
            self.hits += 1
            return
        self.misses += 1
        if len(self.d) >= self.cap:
            self.d.popitem(last=False)
            self.evictions += 1
        self.d[k] = 1


@pytest.fixture(scope="module")
def manifest():
    from paper_2409_00184_b200 import partition

    z = npz("store_smooth33.npz")
    return partition.LODManifest.from_json(json.loads(bytes(z["manifest"]).decode()))


def test_lru_matches_textbook_over_random_stream():
    from paper_2409_00184_b200.runtime import ModelCache

    rng = np.random.default_rng(3)
    cache, ref = ModelCache(12, load_blob), TextbookLRU(12)
    for _ in range(20000):
        k = int(rng.integers(0, 40))
        cache.fetch(k)
        ref.touch(k)
    assert cache.resident_addresses() == list(ref.d)
    assert (cache.hits, cache.misses, cache.evictions) == (ref.hits, ref.misses, ref.evictions)


def test_capacity_and_pinning():
    from paper_2409_00184_b200.errors import CapacityError
    from paper_2409_00184_b200.runtime import ModelCache

    with pytest.raises(ValueError):
        ModelCache(0, load_blob)
    c = ModelCache(2, load_blob)
    c.fetch("a"), c.fetch("b")
    c.begin_frame({"a"})
    c.fetch("c")  # the pinned "a" survives although it is the LRU entry
    assert "a" in c and "b" not in c and "c" in c
    c.begin_frame({"a", "c"})
    with pytest.raises(CapacityError):
        c.fetch("d")


def test_evictions_release_device_slots():
    from paper_2409_00184_b200.runtime import ModelCache

    released = []
    c = ModelCache(2, load_blob, on_evict=lambda b: released.append(b.key))
    for k in "abcd":
        c.fetch(k)
    assert released == ["a", "b"]


def test_capacity_error_releases_the_loaded_block():
    """A block loaded for a fetch that then cannot be cached (every entry
    pinned) is handed back to the loader's release hook: with a DeviceStore
    loader its slot would otherwise leak."""
    from paper_2409_00184_b200.errors import CapacityError
    from paper_2409_00184_b200.runtime import ModelCache

    released = []
    c = ModelCache(2, load_blob, on_evict=lambda b: released.append(b.key))
    c.fetch("a"), c.fetch("b")
    c.begin_frame({"a", "b"})
    with pytest.raises(CapacityError):
        c.fetch("c")
    assert released == ["c"] and "c" not in c and len(c) == 2


def test_counters_and_hook():
    from paper_2409_00184_b200.runtime import ModelCache

    ev = []
    c = ModelCache(4, lambda k: Blob(k, 7), on_load=lambda a, s: ev.append((a, s)))
    c.fetch("a"), c.fetch("b"), c.fetch("a"), c.fetch("x", record=False)
    assert c.bytes_loaded == 21
    assert (c.hits, c.misses) == (1, 2)  # the unrecorded prefetch fetch is not counted
    assert ev == [("a", "frame"), ("b", "frame"), ("x", "prefetch")]


def test_failed_load_leaves_cache_untouched():
    from paper_2409_00184_b200.runtime import ModelCache

    def bad(k):
        raise OSError("io")

    c = ModelCache(1, load_blob)
    c.fetch("a")
    c._loader = bad
    with pytest.raises(OSError):
        c.fetch("b")
    assert c.resident_addresses() == ["a"] and c.evictions == 0


def test_cache_frame_and_capacity_error(manifest):
    from paper_2409_00184_b200.errors import CapacityError
    from paper_2409_00184_b200.render import PointOfView, select_visible
    from paper_2409_00184_b200.runtime import ModelCache, cache_frame

    pov = PointOfView([0, 0, 5.0], [0, 0, -1], [0, 1, 0])
    vis = select_visible(pov, manifest)
    c = ModelCache(100, load_blob)
    res = cache_frame(pov, manifest, c)
    assert list(res) == vis and c.misses == len(vis) and c.hits == 0
    cache_frame(pov, manifest, c)
    assert c.hits == len(vis)
    with pytest.raises(CapacityError, match="exceeds cache capacity"):
        cache_frame(pov, manifest, ModelCache(len(vis) - 1, load_blob))


def test_prefetch_preemption_and_faults(manifest):
    from paper_2409_00184_b200.render import PointOfView, select_visible
    from paper_2409_00184_b200.runtime import ModelCache, predict_static, prefetch_loop

    pov = PointOfView([0, 0, 5.0], [0, 0, -1], [0, 1, 0])
    vis = select_visible(pov, manifest)
    done = threading.Event()
    done.set()
    assert prefetch_loop([pov], manifest, ModelCache(100, load_blob), done, predict_static) == 0
    done = threading.Event()
    c = ModelCache(100, load_blob, on_load=lambda a, s: done.set())  # render finishes mid-prefetch
    assert prefetch_loop([pov], manifest, c, done, predict_static) == 1
    calls = []

    def flaky(k):
        calls.append(k)
        if len(calls) == 1:
            raise OSError("transient")
        return Blob(k)

    c = ModelCache(100, flaky)
    assert prefetch_loop([pov], manifest, c, threading.Event(), predict_static) == len(vis) - 1


def test_prefetch_keeps_pinned_set(manifest):
    from paper_2409_00184_b200.render import PointOfView, select_visible
    from paper_2409_00184_b200.runtime import ModelCache, cache_frame, predict_static, prefetch_loop

    pov = PointOfView([0, 0, 5.0], [0, 0, -1], [0, 1, 0])
    c = ModelCache(len(select_visible(pov, manifest)), load_blob)
    res = cache_frame(pov, manifest, c)
    other = PointOfView([0.2, 0.2, 1.2], [0, 0, -1], [0, 1, 0], fov_y=70)
    prefetch_loop([other], manifest, c, threading.Event(), predict_static)
    assert set(res) <= set(c.resident_addresses())


def test_predictors():
    from paper_2409_00184_b200.render import PointOfView
    from paper_2409_00184_b200.runtime import predict_next_linear, predict_static

    a = PointOfView([0, 0, 3.0], [0, 0, -1], [0, 1, 0])
    b = PointOfView([0, 0.1, 2.8], [0, 0, -1], [0, 1, 0])
    assert predict_static([a, b]) is b and predict_static([]) is None
    assert predict_next_linear([a]) is a
    p = predict_next_linear([a, b])
    np.testing.assert_allclose(p.position, [0, 0.2, 2.6], atol=1e-12)
    c = PointOfView([0, 0, 3.0], [0, 0.8, 0.6], [0, 1, 0])
    d = PointOfView([0, 0, 2.9], [0, np.sqrt(0.91), 0.3], [0, 1, 0])
    np.testing.assert_allclose(predict_next_linear([c, d]).direction, d.direction, atol=1e-12)


def test_trajectory_io(tmp_path):
    from paper_2409_00184_b200.errors import FormatError
    from paper_2409_00184_b200.runtime import load_trajectory, orbit_trajectory, save_trajectory

    povs = orbit_trajectory(7, radius=2.0)
    save_trajectory(tmp_path / "t.jsonl", povs)
    back = load_trajectory(tmp_path / "t.jsonl")
    for p, q in zip(povs, back):
        np.testing.assert_allclose(p.position, q.position)
        np.testing.assert_allclose(p.direction, q.direction)
    (tmp_path / "bad.jsonl").write_text('{"pos": [0, 0, 1]}\n')
    with pytest.raises(FormatError):
        load_trajectory(tmp_path / "bad.jsonl")


def test_replay_with_submit_prefetches_while_frame_in_flight(manifest):
    """replay with a render function that splits at its GPU wait
    (`render_fn.submit` -> handle with done()/result()): the prefetch runs on
    the frame thread and loads only while done() is False (the reference's
    rendering_done check, runtime.py:186); frames, timings and the hit/miss
    accounting are the thread path's."""
    from paper_2409_00184_b200.render import PointOfView
    from paper_2409_00184_b200.runtime import ModelCache, replay

    povs = [PointOfView([0.3, 0.2, 3.2 - 0.15 * i], [0, 0, -1], [0, 1, 0]) for i in range(20)]

    class Pending:
        def __init__(self, budget):
            self.polls, self.budget = 0, budget

        def done(self):  # "the GPU" finishes after `budget` polls
            self.polls += 1
            return self.polls > self.budget

        def result(self):
            return ("frame", self.polls)

    def draw(pov, resident, tf, params):
        raise AssertionError("replay must use submit")

    for budget, expect_loads in ((0, False), (10 ** 6, True)):
        draw.submit = lambda pov, resident, tf, params, b=budget: Pending(b)
        cache = ModelCache(500, load_blob)
        params = type("P", (), {"aspect": 1.0})()
        timings, frames, agg = replay(povs, manifest, cache, None, params, prefetch="linear", render_fn=draw)
        assert len(frames) == len(povs) and all(f[0] == "frame" for f in frames)
        assert agg["frames"] == len(povs)
        loaded = sum(t.prefetch_models_loaded for t in timings)
        assert (loaded > 0) == expect_loads
        for t in timings:
            assert t.input_latency_ms == pytest.approx(t.caching_ms + t.rendering_ms, abs=1e-6)


@pytest.mark.parametrize("depth", [1, 2])
def test_replay_pipeline_keeps_the_reference_operation_order(manifest, depth):
    """replay's submit schedule (the next frame's caching, and at depth 2 its
    launch, overlapped with the current frame): the cache sees the
    reference's operation sequence -- caching i, prefetch i, caching i+1 --
    exactly as the strict order does (same loads, same hit/miss counters,
    same residency), at most `depth` frames are launched and uncollected,
    and frames come back in trajectory order."""
    from paper_2409_00184_b200.render import PointOfView
    from paper_2409_00184_b200.runtime import ModelCache, replay

    povs = [PointOfView([0.3 + 0.02 * i, 0.2, 3.2 - 0.15 * i], [0, 0, -1], [0, 1, 0]) for i in range(16)]
    params = type("P", (), {"aspect": 1.0})()

    def run(overlap, d):
        log, inflight, peak = [], [], [0]

        class Pending:
            def __init__(self, i):
                self.i, self.polls = i, 0

            def done(self):  # each frame "finishes" after 3 polls
                self.polls += 1
                return self.polls > 3

            def result(self):
                inflight.remove(self.i)
                return ("frame", self.i)

        def draw(pov, resident, tf, params_):
            raise AssertionError("replay must use submit")

        def submit(pov, resident, tf, params_):
            i = povs.index(pov)
            inflight.append(i)
            peak[0] = max(peak[0], len(inflight))
            log.append(("submit", i, tuple(sorted(resident))))
            return Pending(i)

        draw.submit = submit
        draw.frames_in_flight = d

        def loader(key):
            log.append(("load", key))
            return Blob(key)

        cache = ModelCache(40, loader)
        import os

        os.environ["AFAM_REPLAY_OVERLAP"] = "1" if overlap else "0"
        try:
            timings, frames, _ = replay(povs, manifest, cache, None, params, prefetch="linear", render_fn=draw)
        finally:
            os.environ.pop("AFAM_REPLAY_OVERLAP", None)
        return log, frames, cache, peak[0]

    ref_log, ref_frames, ref_cache, _ = run(False, 1)
    log, frames, cache, peak = run(True, depth)
    assert frames == ref_frames == [("frame", i) for i in range(len(povs))]
    assert [e for e in log if e[0] == "load"] == [e for e in ref_log if e[0] == "load"]
    assert [e for e in log if e[0] == "submit"] == [e for e in ref_log if e[0] == "submit"]
    assert (cache.hits, cache.misses, cache.evictions) == (ref_cache.hits, ref_cache.misses, ref_cache.evictions)
    assert cache.resident_addresses() == ref_cache.resident_addresses()
    assert peak == depth
