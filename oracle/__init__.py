"""CPU oracle for parity checks (TEST INFRASTRUCTURE ONLY -- see segconv_oracle.py).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
leg. The product package never imports it.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build_c_oracle() -> str:
    """Compile oracle/direct_oracle.c into oracle/build/liboracle.so (gcc, OpenMP)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "build", "liboracle.so")


def c_oracle():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "build", "liboracle.so")
        if not os.path.exists(path):
            build_c_oracle()
        lib = ctypes.CDLL(path)
        lib.oracle_forward_f64.restype = ctypes.c_int
        lib.oracle_forward_f64.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] + [ctypes.c_int] * 6
        lib.oracle_mult_count.restype = ctypes.c_int64
        lib.oracle_mult_count.argtypes = [ctypes.c_int] * 6
        _LIB = lib
    return _LIB


def c_forward_f64(x: np.ndarray, bank: np.ndarray, pad: int) -> np.ndarray:
    """Batched (B, c_in, H, W) forward through the C restatement, in fp64."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    bank = np.ascontiguousarray(bank, dtype=np.float64)
    b, c_in, h, w = x.shape
    _, c_out, n, _ = bank.shape
    oh, ow = 2 * h + 2 * pad - n, 2 * w + 2 * pad - n
    out = np.empty((b, c_out, oh, ow), dtype=np.float64)
    rc = c_oracle().oracle_forward_f64(x.ctypes.data, bank.ctypes.data, out.ctypes.data, b, c_in,
                                       c_out, h, w, n, pad)
    if rc != 0:
        raise ValueError("invalid spec for C oracle")
    return out
