"""Pin the float64 CPU oracle (oracle/) to golden vectors produced by the
unmodified reference (tests/golden/gen_golden.py).  CPU only."""

import json

import numpy as np
import pytest

from helpers import (Addr, golden_store, manifest_ns, npz, params_ns, pov_ns, tf_ns, vis_for)


def test_basis_and_spans_match_reference(oracle):
    z = npz("bspline.npz")
    for ci, (degree, ncp) in enumerate(z["cases"]):
        degree, ncp = int(degree), int(ncp)
        kv = np.concatenate([np.zeros(degree + 1), np.arange(1, ncp - degree) / (ncp - degree), np.ones(degree + 1)])
        u = np.clip(z[f"c{ci}_u"][:, 0], 0, 1)
        for k in range(0, len(u), 7):
            s = oracle.find_span(kv, ncp, degree, u[k])
            assert s == z[f"c{ci}_spans"][k]
            n, d = oracle.basis(kv, degree, s, u[k], derivatives=True)
            np.testing.assert_allclose(n, z[f"c{ci}_bv"][k], rtol=0, atol=1e-14)
            np.testing.assert_allclose(d, z[f"c{ci}_bd"][k], rtol=0, atol=1e-12 * ncp)


def test_eval_points_match_reference(oracle):
    z = npz("bspline.npz")
    for ci, (degree, ncp) in enumerate(z["cases"]):
        degree = int(degree)
        c64 = z[f"c{ci}_coeff64"]
        u = z[f"c{ci}_u"]
        # The oracle stores float32 control points (the .mfa payload type);
        # compare against the reference evaluated on the same float32 grid.
        v, g = oracle.eval_points(z[f"c{ci}_coeff"], degree, u, knots=z[f"c{ci}_knots32"])
        np.testing.assert_allclose(v, z[f"c{ci}_v32"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(g, z[f"c{ci}_g32"], rtol=0, atol=1e-10)
        # default knots path (bspline.py:188-190) on a float32-representable grid
        v0 = oracle.eval_points(c64.astype(np.float32), degree, u, gradient=False)
        ref0 = z[f"c{ci}_v_default"]
        scale = np.abs(c64).max()
        np.testing.assert_allclose(v0, ref0, rtol=0, atol=scale * 2e-7)


def test_eval_points_nonuniform_knots(oracle):
    z = npz("bspline.npz")
    v, g = oracle.eval_points(z["nu_coeff"], int(z["nu_degree"]), z["nu_u"], knots=z["nu_knots"])
    np.testing.assert_allclose(v, z["nu_v"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(g, z["nu_g"], rtol=0, atol=1e-10)


def test_decode_grid_matches_reference(oracle):
    z = npz("bspline.npz")
    for j, (ncp, degree, m) in enumerate(z["dcases"]):
        got = oracle.decode_grid(z[f"d{j}_control"], int(degree), int(m))
        want = z[f"d{j}_grid"]
        scale = max(1.0, np.abs(z[f"d{j}_control"]).max())
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12 * scale)


def test_world_space_hooks(oracle):
    """MicroModel.values_at / gradients_at (model.py:64-87) via the oracle."""
    z = npz("bspline.npz")
    for j, (ncp, degree, m) in enumerate(z["dcases"]):
        ext = np.array([[-0.5, 0.25], [0.0, 0.5], [-1.0, -0.25]])
        pts = z[f"d{j}_pts"]
        u = np.clip((pts - ext[:, 0]) / (ext[:, 1] - ext[:, 0]), 0, 1)
        v, g = oracle.eval_points(z[f"d{j}_control"], int(degree), u, knots=z[f"d{j}_knots"])
        g = g / (ext[:, 1] - ext[:, 0])
        np.testing.assert_allclose(v, z[f"d{j}_values_at"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(g, z[f"d{j}_gradients_at"], rtol=1e-12, atol=1e-10)


def test_lod_for_distance_frozen(oracle):
    z = npz("visible.npz")
    for d, l4, l2 in zip(z["lod_d"], z["lod_l4"], z["lod_l2"]):
        assert oracle.lod_for_distance(float(d), 4) == l4
        assert oracle.lod_for_distance(float(d), 2) == l2


@pytest.mark.parametrize("name", ["smooth33", "ml65_p3", "config3", "config2"])
def test_select_visible_bit_exact(oracle, name):
    z = npz("visible.npz")
    man = manifest_ns(json.loads(bytes(z[f"{name}_manifest"]).decode()))
    table = z[f"{name}_vis"]
    rtable = z[f"{name}_vis_ranges"]
    bad = 0
    for pi, row in enumerate(z["povs"]):
        pov = pov_ns(row)
        for col in (2, 3):
            got = oracle.select_visible(pov, man, aspect=col / 2.0)
            want = vis_for(table, pi, col)
            bad += got != want
        if pi < 40:
            for ri, ranges in enumerate([(1e-9, 2e-9, 3e-9), (1e9, 2e9, 3e9), (0.5, 1.0, 1.7)]):
                got = oracle.select_visible(pov, man, 1.0, ranges=ranges[: man.levels - 1])
                bad += got != vis_for(rtable, pi, ri)
    assert bad == 0


@pytest.mark.parametrize("name", list(npz("frames.npz")["names"]))
def test_render_matches_reference_frames(oracle, name):
    z = npz("frames.npz")
    man, models, _ = golden_store(str(z[f"{name}_store"]))
    vis = [Addr(int(r[0]), tuple(int(v) for v in r[1:])) for r in z[f"{name}_vis"]]
    resident = {a: models[a] for a in vis}
    rgba, info = oracle.render(pov_ns(z[f"{name}_pov"]), resident, tf_ns(z[f"{name}_tf"]),
                               params_ns(z[f"{name}_params"]))
    want = z[f"{name}_rgba"]
    assert info["samples"] == int(z[f"{name}_samples"])
    diff = np.abs(rgba.astype(int) - want.astype(int))
    assert diff.max() <= 1
    assert (diff > 0).mean() < 1e-3
    assert oracle.psnr(rgba, want) >= 80.0


def test_constant_multi_vs_single_identical(oracle):
    z = npz("frames.npz")
    np.testing.assert_array_equal(z["const_multi_rgba"], z["const_single_rgba"])


def test_missing_block_detected(oracle):
    z = npz("frames.npz")
    man, models, _ = golden_store("smooth33")
    from types import SimpleNamespace

    pov = SimpleNamespace(position=np.array([0, 0, 5.0]), direction=np.array([0, 0, -1.0]),
                          up=np.array([0, 1.0, 0]), fov_y=45.0)
    vis = oracle.select_visible(pov, man)
    resident = {Addr(v[0], tuple(v[1:])): models[Addr(v[0], tuple(v[1:]))] for v in vis}
    drop = tuple(int(v) for v in z["missing_dropped"])
    resident.pop(Addr(drop[0], drop[1:]))
    params = SimpleNamespace(width=8, height=8, sample_distance=0.05, o_max=0.99, reference_step=None,
                             near=1e-3, ambient=0.1, diffuse=0.7, specular=0.2, shininess=32.0)
    from helpers import tf_ns as _t  # noqa: F401
    tf = SimpleNamespace(color_points=np.array([[0, 0.1, 0.15, 0.6], [1, 0.8, 0.2, 0.1]]),
                         opacity_points=np.array([[0, 0.0], [1, 0.0]]), domain=(0.0, 1.0))
    _, info = oracle.render(pov, resident, tf, params)
    assert info["missing"] is not None
    assert "finest cell" in str(z["missing_msg"])
