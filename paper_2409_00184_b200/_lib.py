"""ctypes binding of libafam.so (the sm_100a library behind include/afam.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every device entry point raises.  Build it with
``python __graft_entry__.py`` (or ``make -C paper_2409_00184_b200/csrc``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

from .errors import CapacityError, FormatError, MissingBlockError

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("AFAM_LIB", str(PKG / "libafam.so")))  # override: A/B kernel builds
CSRC = PKG / "csrc"

AFAM_OK = 0
_ERRORS = {1: MissingBlockError, 2: FormatError, 3: CapacityError, 4: ValueError, 5: RuntimeError}

AFAM_MAX_DEGREE = 15
AFAM_FAST_DEGREE = 3
AFAM_MAX_TF_POINTS = 32
AFAM_SLOT_VALID = 1
AFAM_SLOT_FP64 = 2
AFAM_EVAL_PARAM = 1
AFAM_EVAL_OUT_F64 = 2
AFAM_RENDER_DEBUG = 1
AFAM_RENDER_FULL_FRAME = 2

_lib = None


class AfamFrame(C.Structure):
    _fields_ = [
        ("origin", C.c_double * 3),
        ("f", C.c_double * 3),
        ("r", C.c_double * 3),
        ("u", C.c_double * 3),
        ("tan_x", C.c_double),
        ("tan_y", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("band_rows", C.c_int32),
        ("nparts", C.c_int32),
        ("part", C.c_int32),
        ("sample_distance", C.c_double),
        ("power", C.c_double),
        ("o_max", C.c_double),
        ("near_", C.c_double),
        ("ambient", C.c_double),
        ("diffuse", C.c_double),
        ("specular", C.c_double),
        ("shininess", C.c_double),
        ("ncolor", C.c_int32),
        ("nopacity", C.c_int32),
        ("domain_lo", C.c_double),
        ("domain_hi", C.c_double),
        ("color", (C.c_double * 4) * AFAM_MAX_TF_POINTS),
        ("opacity", (C.c_double * 2) * AFAM_MAX_TF_POINTS),
        ("flags", C.c_uint32),
        ("color_pts", C.c_void_p),
        ("opacity_pts", C.c_void_p),
    ]


class AfamRenderStats(C.Structure):
    _fields_ = [("samples", C.c_uint64), ("missing_key", C.c_int64), ("fp64_samples", C.c_uint64),
                ("shaded_samples", C.c_uint64), ("exact_samples", C.c_uint64),
                ("exact_cells", C.c_uint64), ("clear_samples", C.c_uint64)]


# (name, restype, argtypes) for every symbol declared in include/afam.h
SIGNATURES = [
    ("afam_last_error", C.c_char_p, []),
    ("afam_version", C.c_int, []),
    ("afam_device_count", C.c_int, []),
    ("afam_store_create", C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int32, C.c_int32, C.c_double]),
    ("afam_store_destroy", C.c_int, [C.c_void_p]),
    ("afam_store_slots", C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("afam_store_put_ds", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    ("afam_store_put_file", C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    ("afam_store_put_mfa", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p,
                                     C.c_void_p]),
    ("afam_mfa_check", C.c_int, [C.c_void_p, C.c_uint64, C.c_int32, C.POINTER(C.c_int32)]),
    ("afam_store_put_mfa_device", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_uint64, C.c_int32, C.c_int32,
                                            C.c_void_p, C.c_void_p]),
    ("afam_store_put", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p]),
    ("afam_store_evict", C.c_int, [C.c_void_p, C.c_int32]),
    ("afam_store_info", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_uint32), C.POINTER(C.c_float)]),
    ("afam_store_read", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    ("afam_eval_points", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                                   C.c_void_p, C.c_uint32, C.c_void_p]),
    ("afam_decode_grid", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    ("afam_decode_grid_ex", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                      C.c_void_p, C.c_void_p]),
    ("afam_fit_rmse", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("afam_fit_rmse3", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                 C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("afam_fit_operator", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    ("afam_png_deflate", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_uint64,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.c_void_p]),
    ("afam_manifest_create", C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_void_p, C.c_void_p]),
    ("afam_manifest_destroy", C.c_int, [C.c_void_p]),
    ("afam_select_visible", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                      C.c_double, C.c_double, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                      C.POINTER(C.c_int32)]),
    ("afam_render", C.c_int, [C.c_void_p, C.POINTER(AfamFrame), C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p]),
    ("afam_ipc_get_handle", C.c_int, [C.c_void_p, C.c_void_p]),
    ("afam_ipc_open", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    ("afam_ipc_close", C.c_int, [C.c_void_p]),
    ("afam_device_alloc", C.c_int, [C.c_int32, C.c_uint64, C.POINTER(C.c_void_p)]),
    ("afam_device_free", C.c_int, [C.c_void_p]),
    ("afam_copy_to_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    ("afam_render_elapsed", C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    ("afam_render_seq", C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    ("afam_render_elapsed_seq", C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_float)]),
    ("afam_frame_rows", C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    ("afam_owner_grid", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_void_p,
                                  C.c_int32]),
    ("afam_bench_fma", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_float), C.POINTER(C.c_double), C.c_void_p]),
    ("afam_bench_dfma", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_float), C.POINTER(C.c_double), C.c_void_p]),
]


def build(force: bool = False) -> Path:
    """Compile libafam.so for sm_100a with nvcc (cross-compiles without a GPU)."""
    cmd = ["make", "-s", "-C", str(CSRC)]
    if force:
        subprocess.run(["make", "-s", "-C", str(CSRC), "clean"], check=True)
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib():
    """The loaded library; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py` "
                               "(the B200 path has no CPU fallback)")
        handle = C.CDLL(str(LIB_PATH))
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    """Map an afam status code to the reference's exception types (errors.py)."""
    if rc == AFAM_OK:
        return
    msg = lib().afam_last_error().decode(errors="replace")
    raise _ERRORS.get(rc, RuntimeError)(msg)


def require_device() -> None:
    n = lib().afam_device_count()
    if n < 1:
        raise RuntimeError("no CUDA device visible: the B200 path has no CPU fallback")


def device_available() -> bool:
    """True when libafam sees a CUDA device."""
    try:
        return lib().afam_device_count() > 0
    except Exception:  # noqa: BLE001
        return False
