"""GPU frame egress: Frame.to_png_bytes with the
deflate payload made on the GPU (afam_png_deflate) decodes -- with PIL and
with zlib -- to exactly the frame's pixels."""

import io
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _decode(png):
    from PIL import Image

    return np.asarray(Image.open(io.BytesIO(png)).convert("RGBA"))


@pytest.mark.parametrize("shape", [(1, 1), (7, 5), (64, 48), (256, 256)])
def test_png_round_trip_random_and_structured(gpu, shape):
    from paper_2409_00184_b200.render import Frame

    H, W = shape
    rng = np.random.default_rng(H * 131 + W)
    frames = [rng.integers(0, 256, size=(H, W, 4), dtype=np.uint8),
              np.zeros((H, W, 4), dtype=np.uint8)]
    g = np.zeros((H, W, 4), dtype=np.uint8)  # gradients + flat runs: exercises Sub/Up filters and long matches
    g[..., 0] = (np.arange(W)[None, :] * 3) % 256
    g[..., 1] = (np.arange(H)[:, None] * 5) % 256
    g[H // 2:, :, 3] = 255
    frames.append(g)
    for rgba in frames:
        png = Frame(W, H, rgba).to_png_bytes()
        np.testing.assert_array_equal(_decode(png), rgba)


def test_png_of_a_rendered_frame(gpu):
    """A real 256^2 render: PIL decodes it identically, zlib accepts the
    stream (adler32 checked), and it is smaller than the raw pixels."""
    from paper_2409_00184_b200 import model, render, synth

    man, blobs = synth.field_store(levels=2, coarsest=1, micro=9, degree=3, ncp_of=lambda a: 7)
    models = {a: model.deserialize(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
    pov = render.PointOfView([0.3, 0.2, 2.2], [-0.1, -0.1, -1.0], [0, 1, 0], 50.0)
    params = render.RenderParams(width=256, height=256, sample_distance=0.01)
    vis = render.select_visible(pov, man)
    fr = render.render(pov, {a: models[a] for a in vis}, render.TransferFunction.ml_preset(), params)
    png = fr.to_png_bytes()
    np.testing.assert_array_equal(_decode(png), fr.rgba)
    # IDAT payload: zlib stream with a valid adler32 trailer
    i = png.index(b"IDAT")
    n = int.from_bytes(png[i - 4:i], "big")
    raw = zlib.decompress(png[i + 4:i + 4 + n])
    assert len(raw) == 256 * (256 * 4 + 1)
    assert len(png) < fr.rgba.nbytes
