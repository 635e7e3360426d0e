"""ctypes binding of libspst.so (the C ABI declared in include/spst.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``) and loaded from this
package directory.  There is no fallback: if the library or a CUDA device is missing, every
entry point raises.  Status codes map 1:1 onto the reference's exception taxonomy
(reference errors.py:4-33).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_longlong, c_void_p

from . import errors

LIB_PATH = os.environ.get("SPST_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspst.so")

OK, E_SHAPE, E_GEOMETRY, E_CONFIG, E_NONFINITE, E_CUDA, E_OOM, E_UNSUPPORTED, E_EMPTY = range(9)

_EXC = {
    E_SHAPE: errors.ShapeError,
    E_GEOMETRY: errors.GeometryError,
    E_CONFIG: errors.ConfigError,
    E_NONFINITE: errors.NonFiniteError,
    E_CUDA: RuntimeError,
    E_OOM: MemoryError,
    E_UNSUPPORTED: NotImplementedError,
    E_EMPTY: errors.EmptyError,
}

# symbol -> (restype, argtypes); mirrors include/spst.h
SIGNATURES = {
    "spst_abi_version": (c_int, []),
    "spst_status_string": (ctypes.c_char_p, [c_int]),
    "spst_create": (c_int, [c_int, c_int, POINTER(c_int), POINTER(c_int), POINTER(c_int),
                            POINTER(POINTER(c_double)), POINTER(POINTER(c_double)), c_int, POINTER(c_int),
                            c_int, c_int, POINTER(c_double), POINTER(c_double), POINTER(c_void_p)]),
    "spst_destroy": (None, [c_void_p]),
    "spst_last_error": (ctypes.c_char_p, [c_void_p]),
    "spst_set_stream": (c_int, [c_void_p, c_void_p]),
    "spst_set_precision": (c_int, [c_void_p, c_int]),
    "spst_bind": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int]),
    "spst_unbind": (c_int, [c_void_p]),
    "spst_bind_window": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int]),
    "spst_window_dims": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int)]),
    "spst_forward_pitched": (c_int, [c_void_p, c_void_p, c_longlong, c_int]),
    "spst_backward_pitched": (c_int, [c_void_p, c_double, c_void_p, c_longlong]),
    "spst_padded_dims": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int)]),
    "spst_tap_info": (c_int, [c_void_p, c_int, POINTER(c_int), POINTER(c_int), POINTER(c_longlong)]),
    "spst_workspace_bytes": (c_longlong, [c_void_p]),
    "spst_forward": (c_int, [c_void_p, c_void_p, c_int]),
    "spst_stats_ptrs": (c_int, [c_void_p, c_int, POINTER(c_void_p), POINTER(c_void_p)]),
    "spst_capture_content": (c_int, [c_void_p]),
    "spst_content_sqdiff": (c_int, [c_void_p, c_void_p]),
    "spst_content_target": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_longlong), POINTER(c_float)]),
    "spst_set_content_target": (c_int, [c_void_p, c_void_p, c_float]),
    "spst_set_style_ref": (c_int, [c_void_p, c_int, POINTER(c_double), POINTER(c_double), POINTER(c_double),
                                   c_double, c_double, c_double]),
    "spst_finalize": (c_int, [c_void_p, POINTER(c_longlong), POINTER(c_double), POINTER(c_int)]),
    "spst_backward": (c_int, [c_void_p, c_double, c_void_p]),
    "spst_forward_redone": (c_int, [c_void_p]),
    "spst_backward_async": (c_int, [c_void_p, c_double, c_void_p, c_longlong]),
    "spst_backward_resolve": (c_int, [c_void_p, POINTER(c_int)]),
    "spst_vec_partials": (c_int, []),
    "spst_vec_dots": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_longlong,
                              c_void_p, c_void_p, c_void_p]),
    "spst_vec_absmax": (c_int, [c_int, c_void_p, c_longlong, c_void_p, c_void_p, c_void_p]),
    "spst_vec_axpy_dot": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_void_p,
                                  c_longlong, c_void_p, c_void_p]),
    "spst_vec_twoloop_scalar": (c_int, [c_void_p, c_double, c_int, c_void_p, c_void_p, c_void_p]),
    "spst_vec_sum_partials": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "spst_vec_two_loop": (c_int, [c_int, c_void_p, c_void_p, POINTER(c_void_p), POINTER(c_void_p), POINTER(c_double),
                                  c_double, c_int, c_longlong, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "spst_vec_axpy": (c_int, [c_int, c_void_p, c_void_p, c_double, c_longlong, c_void_p, c_void_p]),
    "spst_vec_sy": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_longlong, c_void_p, c_void_p,
                            c_void_p, c_void_p, c_void_p]),
    "spst_timing_enable": (c_int, [c_void_p, c_int]),
    "spst_launch_count": (c_longlong, []),
    "spst_timing_read": (c_int, [c_void_p, POINTER(c_double), POINTER(c_double), POINTER(c_longlong)]),
    "spst_metric_sqdiff": (c_int, [c_int, c_void_p, c_void_p, c_longlong, c_void_p, c_void_p, c_void_p]),
    "spst_metric_ssim": (c_int, [c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "spst_resize_down": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
    "spst_resize_bilinear": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
    "spst_resize_down_typed": (c_int, [c_int, c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
    "spst_resize_bilinear_typed": (c_int, [c_int, c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
    "spst_debug_conv": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                c_void_p]),
    "spst_debug_gram": (c_int, [c_int, c_int, c_longlong, c_void_p, c_void_p]),
    "spst_debug_mask": (c_int, [c_void_p, c_int, c_void_p]),
    "spst_debug_stage_out": (c_int, [c_void_p, c_int, c_void_p]),
    "spst_stage_features": (c_int, [c_void_p, c_int, c_void_p]),
    "spst_feature_affine": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_int, c_longlong, c_void_p, c_void_p,
                                    c_void_p]),
    "spst_vec_scaled_diff": (c_int, [c_int, c_void_p, c_void_p, c_double, c_longlong, c_void_p, c_void_p]),
}

_lib = None


def lib():
    """Load libspst.so once; raise (never fall back) when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int, ctx=None, what: str = "") -> None:
    if status == OK:
        return
    msg = ""
    if ctx is not None:
        raw = lib().spst_last_error(ctx)
        msg = raw.decode() if raw else ""
    if not msg:
        msg = lib().spst_status_string(status).decode()
    exc = _EXC.get(status, RuntimeError)
    raise exc(f"{what}: {msg}" if what else msg)


def ptr(t) -> int:
    """Device pointer of a torch tensor (or 0 for None)."""
    return 0 if t is None else int(t.data_ptr())
