"""Degrees above 3 on the device (the reference takes any degree,
bspline.py:29-38): K1 point queries, K3 grid decode (cubic and non-cubic
lattices, mixed with degree-3 blocks in one call) and K2 frames, against
the reference's own outputs (tests/golden/degree.npz, store_ml33_p5.npz)
and the float64 oracle.  Such blocks take the float64 Cox-de Boor path
(afam_eval.cuh eval_any); the tolerances are the float64 ones."""

import numpy as np
import pytest

from helpers import Addr, golden_store, npz, params_ns, pov_ns, tf_ns

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("ci", range(5))
def test_points_vs_reference(cuda, ci):
    from paper_2409_00184_b200 import bspline

    z = npz("degree.npz")
    deg = int(z[f"p{ci}_degree"])
    k = tuple(z[f"p{ci}_knots32"].astype(np.float64))
    v, g = bspline.evaluate_points_with_gradient(z[f"p{ci}_coeff"], deg, z[f"p{ci}_u"], knots=k)
    v0 = bspline.evaluate_points(z[f"p{ci}_coeff"], deg, z[f"p{ci}_u"], knots=k)
    scale = max(1.0, float(np.abs(z[f"p{ci}_v"]).max()))
    np.testing.assert_allclose(v, z[f"p{ci}_v"], rtol=0, atol=1e-10 * scale)
    np.testing.assert_allclose(v0, z[f"p{ci}_v"], rtol=0, atol=1e-10 * scale)
    np.testing.assert_allclose(g, z[f"p{ci}_g"], rtol=0, atol=1e-9 * max(1.0, float(np.abs(z[f"p{ci}_g"]).max())))


@pytest.mark.parametrize("ci", range(3))
def test_decode_vs_reference(cuda, ci):
    from paper_2409_00184_b200 import bspline

    z = npz("degree.npz")
    want = z[f"d{ci}_grid"]
    m = int(z[f"d{ci}_m"])
    got = bspline.decode_tensor_product(z[f"d{ci}_coeff"], int(z[f"d{ci}_degree"]), (m, m, m))
    rng = float(want.max() - want.min())
    assert np.abs(got - want).max() <= 1e-5 * rng  # float32 output


def test_decode_mixed_degrees_and_noncubic(cuda, oracle):
    """One K3 call over degree-3 and degree-5 slots (the fast kernels and the
    high-degree kernel side by side), and a non-cubic lattice (K1 in
    parameter mode)."""
    from paper_2409_00184_b200 import bspline, model
    from paper_2409_00184_b200.device import DeviceStore

    rng = np.random.default_rng(5)
    blocks = []
    for deg, ncp in ((3, 9), (5, 9), (3, 12), (7, 11), (4, 6)):
        c = rng.normal(size=(ncp, ncp, ncp)).astype(np.float32)
        kv = np.repeat(bspline.clamped_knots(ncp, deg).astype(np.float32)[None, :], 3, axis=0)
        blocks.append(model.MicroModel(deg, kv, c, np.array([[0, 1.0]] * 3), 1))
    store = DeviceStore(slots=len(blocks), max_ncp=12)
    for i, b in enumerate(blocks):
        store.put_model(i, b)
    slots = list(range(len(blocks)))
    for m in (9, 33):
        got = bspline.decode_slots(store, slots, m)
        for i, b in enumerate(blocks):
            want = oracle.decode_grid(b.control, b.degree, m)
            assert np.abs(got[i] - want).max() <= 1e-5 * float(want.max() - want.min()), (b.degree, m)
    b = blocks[1]
    got = b.decode_grid((5, 7, 9))
    u = np.stack(np.meshgrid(*[np.linspace(0, 1, n) for n in (5, 7, 9)], indexing="ij"), -1).reshape(-1, 3)
    want = oracle.eval_points(b.control, b.degree, u, knots=b.knots, gradient=False).reshape(5, 7, 9)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-10 * max(1.0, float(np.abs(want).max())))


@pytest.mark.parametrize("name", ["a", "b"])
def test_degree5_frames_vs_reference(cuda, oracle, name):
    from paper_2409_00184_b200 import model, render
    from paper_2409_00184_b200.partition import BlockAddress

    z = npz("degree.npz")
    man, models, _ = golden_store("ml33_p5")
    vis = [tuple(int(v) for v in r) for r in z[f"f{name}_vis"]]
    resident = {}
    for v in vis:
        m = models[Addr(v[0], v[1:])]
        resident[BlockAddress(v[0], v[1:])] = model.MicroModel(m.degree, m.knots, m.control, m.extent, v[0])
    p = params_ns(z[f"f{name}_params"])
    params = render.RenderParams(width=p.width, height=p.height, sample_distance=p.sample_distance, o_max=p.o_max)
    t = tf_ns(z[f"f{name}_tf"])
    tf = render.TransferFunction(t.color_points, t.opacity_points, t.domain)
    frame = render.render(pov_ns(z[f"f{name}_pov"]), resident, tf, params)
    want = z[f"f{name}_rgba"]
    assert oracle.psnr(frame.rgba, want) >= 60.0
    st = render.render.last_stats
    assert st["fp64_samples"] == st["samples"]  # every degree-5 sample on the float64 path
    if p.o_max == 1.0:
        assert st["samples"] == int(z[f"f{name}_samples"])

