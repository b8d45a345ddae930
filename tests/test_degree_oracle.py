"""Degrees above 3 (the reference takes any degree, bspline.py:29-38): the
oracle pinned to the reference's own outputs (tests/golden/degree.npz,
store_ml33_p5.npz, made by tests/golden/gen_degree_golden.py), and the host
fit operator libafam builds for the encoder at those degrees (no GPU)."""

import ctypes as C

import numpy as np
import pytest

from helpers import Addr, golden_store, npz, params_ns, pov_ns, tf_ns


@pytest.mark.parametrize("ci", range(5))
def test_oracle_points_match_reference(oracle, ci):
    z = npz("degree.npz")
    deg = int(z[f"p{ci}_degree"])
    v, g = oracle.eval_points(z[f"p{ci}_coeff"], deg, z[f"p{ci}_u"], knots=z[f"p{ci}_knots32"])
    np.testing.assert_allclose(v, z[f"p{ci}_v"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(g, z[f"p{ci}_g"], rtol=0, atol=1e-9)


@pytest.mark.parametrize("ci", range(3))
def test_oracle_decode_matches_reference(oracle, ci):
    z = npz("degree.npz")
    got = oracle.decode_grid(z[f"d{ci}_coeff"], int(z[f"d{ci}_degree"]), int(z[f"d{ci}_m"]))
    np.testing.assert_allclose(got, z[f"d{ci}_grid"], rtol=0, atol=1e-11)


@pytest.mark.parametrize("name", ["a", "b"])
def test_oracle_degree5_frames_match_reference(oracle, name):
    z = npz("degree.npz")
    man, models, _ = golden_store("ml33_p5")
    assert {m.degree for m in models.values()} == {5}
    vis = [Addr(int(r[0]), tuple(int(v) for v in r[1:])) for r in z[f"f{name}_vis"]]
    rgba, info = oracle.render(pov_ns(z[f"f{name}_pov"]), {a: models[a] for a in vis}, tf_ns(z[f"f{name}_tf"]),
                               params_ns(z[f"f{name}_params"]))
    assert info["samples"] == int(z[f"f{name}_samples"])
    assert np.abs(rgba.astype(int) - z[f"f{name}_rgba"].astype(int)).max() <= 1


@pytest.mark.parametrize("deg,ncp,m", [(4, 9, 17), (5, 12, 17), (7, 10, 13)])
def test_fit_operator_high_degree(deg, ncp, m):
    """afam_fit_operator (the encoder's host operator, bspline.py:109-159) at
    degrees above 3 against a numpy restatement of the pinned fit."""
    from paper_2409_00184_b200 import _lib, synth

    fit = np.zeros((ncp, m))
    dec = np.zeros((m, ncp))
    _lib.check(_lib.lib().afam_fit_operator(ncp, deg, m, fit.ctypes.data_as(C.c_void_p),
                                            dec.ctypes.data_as(C.c_void_p)))
    np.testing.assert_allclose(fit, synth.fit_operator(m, ncp, deg), rtol=0, atol=1e-9)
