"""ctypes binding of libsegb200.so (include/segb200.h).

There is no fallback: if the library is missing or does not load, every
operator raises. Host-only entry points (shape algebra, counts) work without a
GPU; compute entry points need a CUDA device.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SEGB200_LIB", os.path.join(_HERE, "lib", "libsegb200.so"))

SEGB_OK, SEGB_ERR_SPEC, SEGB_ERR_SHAPE, SEGB_ERR_VALUE, SEGB_ERR_CUDA, SEGB_ERR_UNSUPPORTED = range(6)
F32, F64, BF16 = 0, 1, 2
ENGINE_IDS = {"reference": 0, "segregated": 1}
PATH_IDS = {"auto": 0, "direct": 1, "igemm": 2}

# the exported symbols, with ctypes signatures (also checked by tests/test_host.py)
_i, _i64, _u64, _p = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
_pi = ctypes.POINTER(ctypes.c_int)
SIGNATURES = {
    "segb_abi_version": (_i, []),
    "segb_last_error": (ctypes.c_char_p, []),
    "segb_launch_count": (_i64, []),
    "segb_output_dims": (_i, [_i, _i, _i, _i, _pi, _pi]),
    "segb_effective_padding": (_i, [_i, _pi, _pi]),
    "segb_subkernel_dims": (_i, [_i, _i, _i, _pi, _pi]),
    "segb_mult_count_segregated": (_i64, [_i, _i, _i, _i, _i, _i]),
    "segb_segregate": (_i, [_p, _i, _i64, _i, _p, _p]),
    "segb_merge": (_i, [_p, _i, _i64, _i, _p, _p]),
    "segb_prepare": (_i, [_p, _i, _i, _i, _i, _i, _i, _i, _p, ctypes.POINTER(_p)]),
    "segb_layer_info": (_i, [_p, _pi, _pi, _pi, _pi, _pi, _pi]),
    "segb_forward": (_i, [_p, _p, _i, _i64, _i, _i, _p, _i, _i, _i, _p]),
    "segb_select_path": (_i, [_p, _i, _i64, _i, _i, _i]),
    "segb_release": (_i, [_p]),
    "segb_unit_floats": (_i, [_p, _i, _i64, _u64, _p]),
    "segb_forward_workspace_bytes": (_i, [_p, _i, _i64, _i, _i, _i, _i, _i, ctypes.POINTER(_i64)]),
    "segb_forward_ws": (_i, [_p, _p, _i, _i64, _i, _i, _p, _i, _i, _i, _p, _i64, _p]),
    "segb_layer_reserve_workspace": (_i, [_p, _i64]),
    "segb_describe_path": (_i, [_p, _i, _i64, _i, _i, _i, _i, _i, ctypes.c_char_p, _i]),
    "segb_stack_workspace_bytes": (_i, [ctypes.POINTER(_p), _i, _i64, _i, _i, _i, ctypes.POINTER(_i64)]),
    "segb_stack_workspace_bytes2": (_i, [ctypes.POINTER(_p), _i, _i64, _i, _i, _i, _i, _i,
                                         ctypes.POINTER(_i64)]),
    "segb_stack_forward": (_i, [ctypes.POINTER(_p), _i, _p, _i, _i64, _i, _i, _p, _i, _i, _p, _i64, _p]),
    "segb_u8_hwc_to_chw": (_i, [_p, _i64, _i, _i, _i, _p, _i, _p]),
    "segb_counted_forward": (_i, [_p, _i, _i, _i, _p, _i, _i, _i, _i, _p, _p, _p]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load libsegb200.so once; raise (no fallback) if it is absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"segb200 CUDA library not found at {LIB_PATH}; build it with "
                        "`python -m paper_2502_20493_b200.build` (there is no CPU fallback)")
                handle = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def last_error() -> str:
    return lib().segb_last_error().decode(errors="replace")


def check(rc: int) -> None:
    """Map a segb status code to the reference's exception taxonomy."""
    if rc == SEGB_OK:
        return
    from .errors import ShapeError, SpecError
    msg = last_error()
    if rc == SEGB_ERR_SPEC:
        raise SpecError(msg)
    if rc == SEGB_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == SEGB_ERR_VALUE:
        raise ValueError(msg)
    if rc == SEGB_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"segb200 CUDA error: {msg}")


def launch_count() -> int:
    return int(lib().segb_launch_count())
