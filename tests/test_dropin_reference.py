"""The drop-in boundary, proven with the reference's own tests.

INTEGRATION.md's three-line shim is appended to ``splinecast/render.py`` of
an unmodified reference install (``baseline/_ref``: ``pip install --target``
of /root/reference/pkg plus a copy of its ``tests/``, made by
``tools/install_reference.sh``; git-ignored, shipped to the GPU box with the
built libraries), and the reference's own test files run against it in a
subprocess:

* CPU (``-m "not gpu"``): the shim installs, ``paper_2409_00184_b200.errors``
  re-exports the reference's classes, and the reference's visibility tests
  (``TestSelectVisible``, ``TestLodForDistance``) pass through the native
  ``select_visible``;
* GPU: ``tests/test_render.py`` whole (incl. the ``MissingBlockError``
  check at :354-362), ``tests/test_runtime.py`` whole and
  ``tests/test_cli.py::TestEndToEnd`` (:236-261) with every spline frame
  ray-cast by K2 -- the shim's log must show GPU frames.
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

SHIM = """
# --- B200 drop-in (INTEGRATION.md) ---
try:
    from paper_2409_00184_b200.integration import patch_render as _afam_patch
except ImportError:
    pass
else:
    _afam_patch(globals())
"""

IDENTITY_TEST = """
import splinecast.errors as ref_errors
import splinecast.render as ref_render
import splinecast.runtime as ref_runtime
from paper_2409_00184_b200 import errors, integration


def test_errors_are_the_reference_classes():
    assert errors.REFERENCE_CLASSES
    for name in ("FormatError", "PartitionError", "CapacityError", "MissingBlockError"):
        assert getattr(errors, name) is getattr(ref_errors, name)


def test_render_and_select_visible_are_rebound():
    assert ref_render.render.__wrapped_cpu__ is not None
    assert ref_runtime.render is ref_render.render
    assert ref_runtime.select_visible is ref_render.select_visible
    assert ref_render.select_visible.__module__ == integration.__name__
"""


def _shimmed_copy(tmp: Path) -> Path:
    if not (REF / "splinecast").is_dir() or not (REF / "ref_tests").is_dir():
        pytest.skip("baseline/_ref (the reference install + its tests) is missing: run tools/install_reference.sh")
    dst = tmp / "ref"
    shutil.copytree(REF / "splinecast", dst / "splinecast")
    with open(dst / "splinecast" / "render.py", "a") as fh:
        fh.write(SHIM)
    shutil.copytree(REF / "ref_tests", dst / "tests")
    (dst / "tests" / "test_shim_identity.py").write_text(IDENTITY_TEST)
    return dst


def _run(dst: Path, targets, log: Path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(dst), str(ROOT)])
    env["AFAM_SHIM_LOG"] = str(log)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x", *targets]
    return subprocess.run(cmd, cwd=dst, env=env, capture_output=True, text=True, timeout=1800)


def test_shim_cpu_side_reference_tests(tmp_path):
    """Shim install, error identity, and the reference's visibility tests
    through the native select_visible (host code, no device needed)."""
    dst = _shimmed_copy(tmp_path)
    log = tmp_path / "shim.log"
    r = _run(dst, ["tests/test_shim_identity.py", "tests/test_render.py::TestSelectVisible",
                   "tests/test_render.py::TestLodForDistance"], log)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0
    assert "passed" in r.stdout


@pytest.mark.gpu
def test_shim_reference_render_runtime_cli_on_gpu(tmp_path):
    """The reference's render, runtime and CLI end-to-end tests pass with
    every spline frame ray-cast on the B200."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dst = _shimmed_copy(tmp_path)
    log = tmp_path / "shim.log"
    r = _run(dst, ["tests/test_shim_identity.py", "tests/test_render.py", "tests/test_runtime.py",
                   "tests/test_cli.py::TestEndToEnd"], log)
    print(r.stdout[-5000:], r.stderr[-3000:])
    assert r.returncode == 0
    lines = log.read_text().splitlines() if log.exists() else []
    print(f"{len(lines)} frames ray-cast on the GPU through the shim")
    assert len(lines) >= 5
