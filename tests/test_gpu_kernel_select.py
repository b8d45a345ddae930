"""K2's per-frame instantiation choice (afam_render.cu launch_render): the
all-fast kernel when every block is a clamped-uniform float32 slot of the
frame's degree, the general kernel (exact path for the rest) when a block
has non-uniform knots or another degree, the float64 kernels when a slot is
ill-conditioned -- every choice against the float64 oracle on the same
models (PSNR >= 60 dB, identical sample counts at o_max = 1)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_00184_b200 import model, render, synth

    man, blobs = synth.field_store(levels=2, coarsest=1, micro=9, degree=3, ncp_of=lambda a: 7)
    models = {a: model.deserialize(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
    pov = render.PointOfView([0.2, 0.3, 0.65], [-0.1, -0.2, -1.0], [0, 1, 0], 70.0)  # the finest LOD: 8 blocks
    params = render.RenderParams(width=40, height=40, sample_distance=0.008, o_max=1.0)
    vis = render.select_visible(pov, man, params.aspect)
    assert len(vis) >= 4
    return man, models, pov, params, vis


def _check(oracle, pov, resident, params):
    from paper_2409_00184_b200 import render

    tf = render.TransferFunction.ml_preset()
    frame = render.render(pov, resident, tf, params)
    want, info = oracle.render(pov, resident, tf, params)
    assert oracle.psnr(frame.rgba, want) >= 60.0
    st = render.render.last_stats
    assert st["samples"] == info["samples"]
    return st


def test_all_uniform_frame_takes_no_exact_samples(scene, oracle):
    man, models, pov, params, vis = scene
    st = _check(oracle, pov, {a: models[a] for a in vis}, params)
    assert st["exact_samples"] == 0 and st["fp64_samples"] == 0


def test_non_uniform_knots_take_the_exact_path(scene, oracle):
    from paper_2409_00184_b200 import model

    man, models, pov, params, vis = scene
    resident = {a: models[a] for a in vis}
    a0 = max(vis, key=lambda a: a.lod)  # a coarse block most rays cross
    m = resident[a0]
    kv = np.array(m.knots, dtype=np.float32)
    kv[:, 4] += np.float32(0.03)  # an interior knot moved: still increasing, no longer uniform
    resident[a0] = model.MicroModel(m.degree, kv, m.control, m.extent, m.lod)
    st = _check(oracle, pov, resident, params)
    assert st["exact_samples"] > 0


def test_mixed_degrees_in_one_frame(scene, oracle):
    from paper_2409_00184_b200 import model, synth

    man, models, pov, params, vis = scene
    man2, blobs2 = synth.field_store(levels=2, coarsest=1, micro=9, degree=2, ncp_of=lambda a: 6)
    models2 = {a: model.deserialize(b, man2.entries[a].ncp, man2.entries[a].extent, a.lod) for a, b in blobs2.items()}
    resident = {a: (models2[a] if i % 3 == 0 else models[a]) for i, a in enumerate(vis)}
    assert {m.degree for m in resident.values()} == {2, 3}
    st = _check(oracle, pov, resident, params)
    assert st["exact_samples"] > 0  # the minority degree takes the exact path


def test_ill_conditioned_slot_with_non_uniform_neighbour(scene, oracle):
    from paper_2409_00184_b200 import model

    man, models, pov, params, vis = scene
    resident = {a: models[a] for a in vis}
    big = vis[len(vis) // 2]
    m = resident[big]
    resident[big] = model.MicroModel(m.degree, m.knots, m.control * 40.0 - 20.0, m.extent, m.lod)  # max|c| > 4
    st = _check(oracle, pov, resident, params)
    assert st["fp64_samples"] > 0 and st["exact_samples"] == 0  # the float64 fast path (all-fast F64)
    other = vis[0] if vis[0] != big else vis[1]
    m = resident[other]
    kv = np.array(m.knots, dtype=np.float32)
    kv[:, 4] += np.float32(0.02)
    resident[other] = model.MicroModel(m.degree, kv, m.control, m.extent, m.lod)
    st = _check(oracle, pov, resident, params)
    assert st["fp64_samples"] > 0
