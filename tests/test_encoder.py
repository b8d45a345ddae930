"""Encoder inner loop: endpoint-pinned least-squares
fit + float32 rounding + decode + RMSE, pinned to the reference's own
encoder on golden blocks (tests/golden/gen_encoder_golden.py).

CPU tests check the host fit operator (afam_fit_operator, no device work)
against the reference's fitted coefficients; GPU tests run the batched
float64 kernels (afam_fit_rmse) and the search / cross-level encode."""

import ctypes as C
import warnings

import numpy as np
import pytest

from helpers import npz

Z = npz("encoder.npz")
FIT_CASES = [tuple(int(v) for v in r) for r in Z["fit_cases"]]


def _operator(ncp, deg, m):
    from paper_2409_00184_b200 import _lib

    F = np.zeros((ncp, m))
    B = np.zeros((m, ncp))
    _lib.check(_lib.lib().afam_fit_operator(ncp, deg, m, F.ctypes.data_as(C.c_void_p), B.ctypes.data_as(C.c_void_p)))
    return F, B


def _ulps32(a, b):
    ia = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    ib = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    return np.abs(ia - ib)


@pytest.mark.parametrize("case", range(len(FIT_CASES)))
def test_fit_operator_matches_reference_fit(case):
    """F (x) F (x) F . samples (float64) rounded to float32 reproduces model.fit's
    coefficients (bspline.py:128-159) to within 1 ulp, and B-decode + RMSE
    reproduces encoder.error_rmse (encoder.py:74-78)."""
    m, deg, _ = FIT_CASES[case]
    s = Z[f"fit_{case}_samples"].astype(np.float64)
    rm = Z[f"fit_{case}_rmse"]
    for ncp in range(deg + 1, m + 1):
        F, B = _operator(ncp, deg, m)
        c = np.einsum("ai,ijk->ajk", F, s)
        c = np.einsum("bj,ajk->abk", F, c)
        c = np.einsum("ck,abk->abc", F, c).astype(np.float32)
        want = Z[f"fit_{case}_ctrl_{ncp}"]
        assert _ulps32(c, want).max() <= 1, (ncp, _ulps32(c, want).max())
        d = np.einsum("ia,abc->ibc", B, c.astype(np.float64))
        d = np.einsum("jb,ibc->ijc", B, d)
        d = np.einsum("kc,ijc->ijk", B, d)
        r = float(np.sqrt(np.mean((d - s) ** 2)))
        assert r == pytest.approx(rm[ncp - deg - 1], rel=1e-7)


def test_fit_operator_rejects_bad_arguments():
    from paper_2409_00184_b200 import _lib
    from paper_2409_00184_b200.errors import FormatError  # noqa: F401

    with pytest.raises(ValueError):
        _lib.check(_lib.lib().afam_fit_operator(2, 2, 9, None, None))  # ncp < degree + 1
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().afam_fit_operator(10, 2, 9, None, None))  # ncp > m


# ------------------------------------------------------------------ GPU
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(FIT_CASES)))
def test_fit_rmse_batch_vs_reference(case):
    _cuda()
    from paper_2409_00184_b200 import encoder

    m, deg, _ = FIT_CASES[case]
    s = Z[f"fit_{case}_samples"]
    ncps = list(range(deg + 1, m + 1))
    rmse, ctrls = encoder.fit_rmse_batch([s], deg, [(0, n) for n in ncps], want_ctrl=True)
    np.testing.assert_allclose(rmse, Z[f"fit_{case}_rmse"], rtol=1e-9, atol=1e-14)
    for n, c in zip(ncps, ctrls):
        assert _ulps32(c, Z[f"fit_{case}_ctrl_{n}"]).max() <= 1, n


@pytest.mark.gpu
def test_fit_rmse_batch_many_blocks_and_shuffled_jobs():
    """Jobs over several blocks in arbitrary order give the per-block results."""
    _cuda()
    from paper_2409_00184_b200 import encoder

    cases = [c for c, (m, _, _) in enumerate(FIT_CASES) if m == 17 and FIT_CASES[c][1] == 2]
    cases += [c for c, (m, d, _) in enumerate(FIT_CASES) if m == 17 and d == 3]
    blocks = [Z[f"fit_{c}_samples"] for c in cases]
    deg = 2
    c0 = cases[0]
    jobs = [(0, n) for n in range(3, 18)]
    rng = np.random.default_rng(0)
    order = rng.permutation(len(jobs))
    r, _ = encoder.fit_rmse_batch(blocks, deg, [jobs[i] for i in order])
    want = Z[f"fit_{c0}_rmse"]
    np.testing.assert_allclose(r, want[[jobs[i][1] - 3 for i in order]], rtol=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(Z["search_cases"])))
def test_in_level_search_vs_reference(k):
    _cuda()
    from paper_2409_00184_b200 import encoder

    c, bound, mono = Z["search_cases"][k]
    m, deg, _ = FIT_CASES[int(c)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        r = encoder.in_level_search(Z[f"fit_{int(c)}_samples"], float(bound), deg, assume_monotone=bool(mono))
    star, met, cplx = (int(v) for v in Z[f"search_{k}_star"])
    assert (r.ncp_star, int(r.met_bound), int(r.is_complex)) == (star, met, cplx)
    prof = Z[f"search_{k}_profile"]
    assert sorted(r.profile.rmse_by_ncp) == [int(v) for v in prof[:, 0]]
    np.testing.assert_allclose([r.profile.rmse_by_ncp[int(n)] for n in prof[:, 0]], prof[:, 1], rtol=1e-9)
    assert _ulps32(r.model.control, Z[f"search_{k}_ctrl"]).max() <= 1


@pytest.mark.gpu
def test_in_level_search_warns_when_unmeetable():
    _cuda()
    from paper_2409_00184_b200 import encoder

    with pytest.warns(RuntimeWarning, match="unmeetable"):
        r = encoder.in_level_search(Z["fit_3_samples"], 1e-9, 3)
    assert not r.met_bound and r.ncp_star == 17


@pytest.mark.gpu
@pytest.mark.parametrize("deg", [2, 3])
def test_encode_volume_vs_reference(deg):
    """encode_volume (adaptive) on the 33^3 Marschner-Lobb volume: the same
    NCP and complexity for every block, the same stats, coefficients within
    1 float32 ulp."""
    _cuda()
    from types import SimpleNamespace

    from paper_2409_00184_b200 import encoder

    bound, mono = Z[f"vol_{deg}_case"]
    vol = SimpleNamespace(samples=Z["vol_samples"], bounds=Z["vol_bounds"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        man, models, stats = encoder.encode_volume(vol, levels=2, micro_dims=9, degree=deg, error_bound=float(bound),
                                                   coarsest=2, mode="adaptive", assume_monotone=bool(mono))
    addrs = sorted(man.entries)
    assert [(a.lod, *a.ijk) for a in addrs] == [tuple(r) for r in Z[f"vol_{deg}_addr"]]
    assert [man.entries[a].ncp for a in addrs] == list(Z[f"vol_{deg}_ncp"])
    assert [int(man.entries[a].is_complex) for a in addrs] == list(Z[f"vol_{deg}_complex"])
    assert [stats.total_blocks, stats.searched_blocks, len(stats.unmet_blocks)] == list(Z[f"vol_{deg}_stats"])
    for i, a in enumerate(addrs):
        assert _ulps32(models[a].control, Z[f"vol_{deg}_ctrl_{i}"]).max() <= 1, a
