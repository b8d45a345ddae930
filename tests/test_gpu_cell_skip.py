"""K2's transparent-cell skip (BlockDesc::crange, afam_store.cu
cell_range_kernel / cell_range4_kernel; afam_render.cu fast_cell_update_k)
against the float64 oracle: transfer functions whose opacity support covers
part, all or none of the data range, domains narrower than the data (values
clamped into the support), degrees 1-3.  Frames within 60 dB PSNR, per-ray
sample counts and owner hashes identical (reference render.py:398-466)."""

import numpy as np
import pytest

from helpers import golden_store

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _check(oracle, pov, resident, tf, params):
    from paper_2409_00184_b200 import render

    out, info, dbg = render.render_part(pov, resident, tf, params, debug=True)
    want, oinfo = oracle.render(pov, resident, tf, params, debug=True)
    np.testing.assert_array_equal(dbg["nsamp"].cpu().numpy().ravel(), oinfo["nsamp"])
    np.testing.assert_array_equal(dbg["ohash"].cpu().numpy().view(np.uint64).ravel(), oinfo["ohash"])
    assert info["samples"] == oinfo["samples"]
    assert oracle.psnr(out.cpu().numpy(), want) >= 60.0
    return out.cpu().numpy(), info


def _tfs(lo, hi):
    from paper_2409_00184_b200 import render

    w = hi - lo
    col = [[0.0, 0.2, 0.4, 0.9], [0.5, 0.9, 0.9, 0.3], [1.0, 0.9, 0.2, 0.1]]
    return {
        # support in the middle of the data range (most cells transparent)
        "narrow": render.TransferFunction(col, [[0.0, 0.0], [0.45, 0.0], [0.5, 0.6], [0.55, 0.0], [1.0, 0.0]],
                                          (lo, hi)),
        # support at the low end of a domain narrower than the data: every
        # value below the domain clamps into the support
        "clamped_low": render.TransferFunction(col, [[0.0, 0.4], [0.2, 0.4], [0.3, 0.0], [1.0, 0.0]],
                                               (lo + 0.45 * w, lo + 0.55 * w)),
        "clamped_high": render.TransferFunction(col, [[0.0, 0.0], [0.7, 0.0], [0.8, 0.4], [1.0, 0.4]],
                                                (lo + 0.45 * w, lo + 0.55 * w)),
        # opacity everywhere: nothing to skip
        "full": render.TransferFunction(col, [[0.0, 0.05], [1.0, 0.2]], (lo, hi)),
        # no opacity anywhere: every sample skipped, transparent frame
        "none": render.TransferFunction(col, [[0.0, 0.0], [1.0, 0.0]], (lo, hi)),
    }


@pytest.mark.parametrize("tfname", ["narrow", "clamped_low", "clamped_high", "full", "none"])
def test_cell_skip_golden_store(cuda, oracle, tfname):
    from paper_2409_00184_b200 import render

    from paper_2409_00184_b200 import model
    from paper_2409_00184_b200.partition import BlockAddress

    man, models, _ = golden_store("smooth33")
    pm = {BlockAddress(a.lod, a.ijk): model.MicroModel(m.degree, m.knots, m.control, m.extent, a.lod)
          for a, m in models.items()}
    ctrl = np.concatenate([np.asarray(m.control).ravel() for m in models.values()])
    tf = _tfs(float(ctrl.min()), float(ctrl.max()))[tfname]
    pov = render.PointOfView([1.3, 0.9, 2.2], [-1.3, -0.9, -2.2], [0, 1, 0], 50.0)
    vis = render.select_visible(pov, man)
    params = render.RenderParams(width=48, height=40, sample_distance=0.005, o_max=0.99)
    got, info = _check(oracle, pov, {a: pm[a] for a in vis}, tf, params)
    if tfname == "none":
        assert not got.any() and info["shaded_samples"] == 0
        assert info["clear_samples"] == info["samples"]  # every cell transparent
    elif tfname == "full":
        assert info["clear_samples"] == 0  # no cell transparent
    elif tfname == "narrow":
        assert 0 < info["clear_samples"] < info["samples"]
    else:  # the clamped supports: whether any cell is opaque depends on the view
        assert info["clear_samples"] <= info["samples"]


@pytest.mark.parametrize("degree", [1, 2, 3])
def test_cell_skip_degrees(cuda, oracle, degree):
    from paper_2409_00184_b200 import model, render, synth

    man, blobs = synth.field_store(levels=2, coarsest=1, micro=17, degree=degree, ncp_of=lambda a: 9 + a.lod * 3)
    models = {a: model.deserialize(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
    ctrl = np.concatenate([np.asarray(m.control).ravel() for m in models.values()])
    pov = render.PointOfView([0.5, 0.5, 1.4], [-0.5, -0.5, -1.4], [0, 1, 0])
    vis = render.select_visible(pov, man)
    params = render.RenderParams(width=40, height=40, sample_distance=0.004, o_max=0.99)
    for name in ("narrow", "clamped_low"):
        _check(oracle, pov, {a: models[a] for a in vis}, _tfs(float(ctrl.min()), float(ctrl.max()))[name], params)
