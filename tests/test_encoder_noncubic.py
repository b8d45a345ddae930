"""Encoder on non-cubic micro-blocks (afam_fit_rmse3), pinned to the
reference's own encoder (tests/golden/gen_encoder_noncubic_golden.py):
_fit_and_measure, in_level_search (sweep and bisection), the reference's
ValueError when the NCP range exceeds a shorter axis, and encode_volume with
micro_dims (5, 9, 9)."""

import warnings

import numpy as np
import pytest

from helpers import npz

Z = npz("encoder_noncubic.npz")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ulps32(a, b):
    ia = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    ib = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    return np.abs(ia - ib)


def test_fit_rmse_noncubic_vs_reference():
    from paper_2409_00184_b200 import encoder

    s = Z["fit_samples"]
    assert s.shape == (5, 9, 7)
    ncps = [3, 4, 5]
    rmse, ctrls = encoder.fit_rmse_batch([s], 2, [(0, n) for n in ncps], want_ctrl=True)
    np.testing.assert_allclose(rmse, Z["fit_rmse"], rtol=1e-9, atol=1e-14)
    for n, c in zip(ncps, ctrls):
        assert c.shape == (n, n, n)
        assert _ulps32(c, Z[f"fit_ctrl_{n}"]).max() <= 1, n


@pytest.mark.parametrize("k", [0, 1])
def test_in_level_search_noncubic_vs_reference(k):
    from paper_2409_00184_b200 import encoder

    bound, mono = Z[f"search_{k}_case"]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        r = encoder.in_level_search(Z["fit_samples"], float(bound), 2, assume_monotone=bool(mono))
    assert (r.ncp_star, int(r.met_bound), int(r.is_complex)) == tuple(int(v) for v in Z[f"search_{k}_star"])
    prof = Z[f"search_{k}_profile"]
    assert sorted(r.profile.rmse_by_ncp) == [int(v) for v in prof[:, 0]]
    np.testing.assert_allclose([r.profile.rmse_by_ncp[int(n)] for n in prof[:, 0]], prof[:, 1], rtol=1e-9)
    assert _ulps32(r.model.control, Z[f"search_{k}_ctrl"]).max() <= 1


def test_ncp_above_a_shorter_axis_raises_like_reference():
    from paper_2409_00184_b200 import encoder

    block = np.full((9, 9, 5), 0.5, np.float32)
    with pytest.raises(ValueError) as exc:
        encoder.in_level_search(block, 1e-2, 2)
    assert str(exc.value) == str(Z["bad_msg"])


def test_encode_volume_noncubic_micro_dims_vs_reference():
    from types import SimpleNamespace

    from paper_2409_00184_b200 import encoder

    vol = SimpleNamespace(samples=Z["vol_samples"], bounds=np.array([[-1.0, 1.0]] * 3))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        man, models, stats = encoder.encode_volume(vol, levels=2, micro_dims=(5, 9, 9), degree=2, error_bound=3e-2,
                                                   coarsest=1, mode="adaptive")
    addrs = sorted(man.entries)
    assert [(a.lod, *a.ijk) for a in addrs] == [tuple(r) for r in Z["vol_addr"]]
    assert [man.entries[a].ncp for a in addrs] == list(Z["vol_ncp"])
    assert [int(man.entries[a].is_complex) for a in addrs] == list(Z["vol_complex"])
    assert [stats.total_blocks, stats.searched_blocks, len(stats.unmet_blocks)] == list(Z["vol_stats"])
    for i, a in enumerate(addrs):
        assert _ulps32(models[a].control, Z[f"vol_ctrl_{i}"]).max() <= 1, a
