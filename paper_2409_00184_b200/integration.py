"""Drop-in wiring of the B200 path into an unmodified reference install.

A maintainer adds three lines at the end of the reference's
``splinecast/render.py``:

    try:
        from paper_2409_00184_b200.integration import patch_render as _afam_patch
    except ImportError:
        pass
    else:
        _afam_patch(globals())

``patch_render`` rebinds the module's ``render`` and ``select_visible``
(reference render.py:398-466 and :281-320) before any other reference
module imports them (runtime.py:26, cli.py and service.py bind them at
import or call time), so ``runtime.replay``, ``cli render/replay/compare``
and the service's ``serve_frame`` reach the GPU unchanged:

* ``render(pov, blocks, tf, params)``: when every block is a spline model
  (the reference's ``MicroModel``, duck-typed on ``.control/.knots/.degree``,
  or a resident ``DeviceBlock``) the frame is ray-cast by K2 and returned as
  the reference's own ``Frame``; analytic ``FieldBlock``s
  (``render_ground_truth``) and DS blocks stay on the reference's CPU loop
  (the B200 path has no CPU fallback of its own).
* ``select_visible``: the native, bit-exact traversal, returning the
  reference's ``BlockAddress`` objects.

Errors are the reference's classes: ``paper_2409_00184_b200.errors``
re-exports ``splinecast.errors`` whenever the reference is importable, so a
``MissingBlockError`` from the GPU path is the one ``cli.py:345-351``,
``service.py:255`` and ``tests/test_render.py:360`` catch.

With ``AFAM_SHIM_LOG=<path>`` every frame routed to the GPU appends one line
(``gpu <width>x<height> <blocks>``) to that file, so a test can prove the
B200 path ran.
"""

from __future__ import annotations

import os

__all__ = ["patch_render", "is_spline_block"]


def is_spline_block(block) -> bool:
    """A block the B200 renderer takes: a resident DeviceBlock of a spline
    model, or any object shaped like the reference's MicroModel."""
    from .device import DeviceBlock

    if isinstance(block, DeviceBlock):
        return block.kind == "mfa"
    return all(hasattr(block, k) for k in ("control", "knots", "degree", "extent"))


def _log(line: str) -> None:
    path = os.environ.get("AFAM_SHIM_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(line + "\n")


def patch_render(ns: dict) -> None:
    """Rebind ``render`` and ``select_visible`` in the reference render module's
    namespace ``ns`` (its ``globals()``)."""
    from . import render as b200

    cpu_render = ns["render"]
    frame_cls = ns["Frame"]
    addr_cls = ns["BlockAddress"]

    def render(pov, blocks, tf, params):
        if blocks and all(is_spline_block(b) for b in blocks.values()):
            fr = b200.render(pov, blocks, tf, params)
            _log(f"gpu {fr.width}x{fr.height} {len(blocks)}")
            return frame_cls(width=fr.width, height=fr.height, rgba=fr.rgba)
        return cpu_render(pov, blocks, tf, params)

    def select_visible(pov, manifest, aspect: float = 1.0, near: float = 1e-3, ranges=None):
        return [addr_cls(a.lod, a.ijk) for a in b200.select_visible(pov, manifest, aspect, near, ranges)]

    render.__doc__ = cpu_render.__doc__
    render.__wrapped_cpu__ = cpu_render
    select_visible.__doc__ = ns["select_visible"].__doc__
    ns["render"] = render
    ns["select_visible"] = select_visible
