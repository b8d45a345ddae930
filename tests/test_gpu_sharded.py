"""Grid decode sharded over ranks (BASELINE config 5):
tiles.decode_grid_sharded against the single-GPU K3 decode."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_decode_grid_sharded_matches_single(cuda):
    """tiles.decode_grid_sharded (config 5 over N ranks): the
    shares of ranks 0..2 of a 3-way split, decoded each in one launch, are
    the single-GPU decode of those blocks, and together cover every block."""
    from paper_2409_00184_b200 import bspline, model, synth, tiles
    from paper_2409_00184_b200.device import DeviceStore

    man, blobs = synth.field_store(levels=2, coarsest=1, micro=9, degree=3, ncp_of=lambda a: 5 + sum(a.ijk) % 3)
    ds = DeviceStore(len(blobs), 9)
    blocks = {a: ds.load_mfa(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
    seen = []
    for r in range(3):
        mine, grids = tiles.decode_grid_sharded(blocks, 17, rank=r, world=3)
        seen += mine
        want = bspline.decode_slots(ds, [blocks[a].slot for a in mine], 17)  # [b, i, j, k]
        got = grids.permute(0, 3, 2, 1).cpu().numpy()
        np.testing.assert_array_equal(got, want)
    assert sorted(seen) == sorted(blocks)
