"""Edge cases of the GPU path against the float64 oracle and the reference's
semantics (render.py:355-466): an empty resident set (MissingBlockError at
the first sample that enters the domain, transparent frame when no ray
enters it), odd and degenerate frame shapes, empty point batches and
zero-block decodes."""

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


def _product(models):
    from paper_2409_00184_b200 import model
    from paper_2409_00184_b200.partition import BlockAddress

    return {BlockAddress(a.lod, a.ijk): model.MicroModel(m.degree, m.knots, m.control, m.extent, a.lod)
            for a, m in models.items()}


def test_empty_resident_set_raises_at_first_domain_sample(cuda, oracle):
    """_BlockIndex over no blocks is one cell of -1 (render.py:363-366): the
    first alive sample raises, with the reference's message."""
    from paper_2409_00184_b200 import render
    from paper_2409_00184_b200.errors import MissingBlockError

    pov = render.PointOfView([0, 0, 3.0], [0, 0, -1], [0, 1, 0])
    params = render.RenderParams(width=6, height=4, sample_distance=0.05)
    tf = render.TransferFunction.ml_preset()
    _, info = oracle.render(pov, {}, tf, params)
    assert info["missing"] is not None
    with pytest.raises(MissingBlockError, match=r"finest cell \(0, 0, 0\)") as exc:
        render.render(pov, {}, tf, params)
    step, ray = info["missing"]
    _, ginfo, _ = render.render_part(pov, {}, tf, params, raise_missing=False)
    assert ginfo["missing_key"] == (step << 32) | ray
    assert "no resident block covers sample" in str(exc.value)


def test_empty_resident_set_looking_away_is_transparent(cuda):
    from paper_2409_00184_b200 import render

    pov = render.PointOfView([0, 0, 3.0], [0, 0, 1], [0, 1, 0])
    fr = render.render(pov, {}, render.TransferFunction.ml_preset(),
                       render.RenderParams(width=5, height=3, sample_distance=0.05))
    assert fr.rgba.shape == (3, 5, 4) and not fr.rgba.any()
    assert render.render.last_stats["samples"] == 0


@pytest.mark.parametrize("wh", [(1, 1), (3, 5), (17, 2), (33, 31)])
def test_odd_frame_shapes_vs_oracle(cuda, oracle, wh):
    """Frames whose sizes are not multiples of the 16x8 CTA tile: every
    pixel (incl. the partial tiles) against the float64 oracle, same sample
    counts per ray."""
    from paper_2409_00184_b200 import render

    man, models, _ = golden_store("smooth33")
    pm = _product(models)
    W, H = wh
    params = render.RenderParams(width=W, height=H, sample_distance=0.01)
    pov = render.PointOfView([0.3, 0.2, 2.2], [-0.1, -0.1, -1.0], [0, 1, 0])
    vis = render.select_visible(pov, man, params.aspect)
    res = {a: pm[a] for a in vis}
    tf = render.TransferFunction.ml_preset()
    out, info, dbg = render.render_part(pov, res, tf, params, debug=True)
    want, oinfo = oracle.render(pov, res, tf, params, debug=True)
    got = out.cpu().numpy()
    assert got.shape == want.shape == (H, W, 4)
    np.testing.assert_array_equal(dbg["nsamp"].cpu().numpy().ravel(), oinfo["nsamp"])
    assert np.abs(got.astype(int) - want.astype(int)).max() <= 2
    assert info["samples"] == oinfo["samples"]


def test_empty_point_batch_and_zero_block_decode(cuda):
    from paper_2409_00184_b200 import bspline, model
    from paper_2409_00184_b200.device import DeviceStore

    kv = np.repeat(bspline.clamped_knots(5, 2)[None, :], 3, axis=0).astype(np.float32)
    mm = model.MicroModel(2, kv, np.zeros((5, 5, 5), np.float32), [[-1, 1]] * 3, 1)
    assert mm.values_at(np.zeros((0, 3))).shape == (0,)
    assert mm.gradients_at(np.zeros((0, 3))).shape == (0, 3)
    ds = DeviceStore(2, 8)
    assert bspline.decode_slots(ds, [], 8).shape == (0, 8, 8, 8)
