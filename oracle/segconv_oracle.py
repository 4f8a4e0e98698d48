"""CPU oracle for the unified kernel-segregated stride-2 transpose convolution.

TEST INFRASTRUCTURE ONLY. This module is a numpy restatement of the reference
algorithm (arxiv 2502.20493, package `segconv`). It exists to *check* the CUDA
path; it is never the thing measured or shipped. Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
leg may import it. The product package `paper_2502_20493_b200` never imports
anything from `oracle/`.

Parity pinning: every function here is checked against golden vectors produced
by the reference itself (`tests/golden/make_golden.py` imports
`/root/reference/pkg/src/segconv` in the build container and freezes its
outputs into `tests/golden/*.npz`; see `tests/test_oracle.py`).

Citations are `path:line` relative to `/root/reference/pkg/src/segconv/`.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

# --------------------------------------------------------------------------
# synth.py:20-56 -- splitmix64 stream, double-rounded to float32

_MASK = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB


def splitmix64(value: int) -> int:
    """synth.py:20-25: stateless splitmix64 output function."""
    z = (value + _GAMMA) & _MASK
    z = ((z ^ (z >> 30)) * _MIX1) & _MASK
    z = ((z ^ (z >> 27)) * _MIX2) & _MASK
    return z ^ (z >> 31)


def unit_floats(count: int, seed: int) -> np.ndarray:
    """synth.py:28-39: element i = float32(float64(splitmix64(seed + i)) * 2**-64)."""
    idx = np.arange(count, dtype=np.uint64) + np.uint64(seed & _MASK)
    z = idx + np.uint64(_GAMMA)
    z ^= z >> np.uint64(30)
    z *= np.uint64(_MIX1)
    z ^= z >> np.uint64(27)
    z *= np.uint64(_MIX2)
    z ^= z >> np.uint64(31)
    return (z.astype(np.float64) * 2.0 ** -64).astype(np.float32)


def gen_synthetic(c: int, h: int, w: int, seed: int) -> np.ndarray:
    """synth.py:42-46."""
    return unit_floats(c * h * w, seed).reshape(c, h, w)


def gen_kernel_bank(c_in: int, c_out: int, n: int, seed: int) -> np.ndarray:
    """synth.py:49-56."""
    return unit_floats(c_in * c_out * n * n, seed).reshape(c_in, c_out, n, n)


def harness_seeds(seed: int, index: int) -> tuple[int, int]:
    """bench.py:299-300: per-layer input and bank seeds of the reference harness."""
    input_seed = splitmix64((seed & _MASK) + 2 * index)
    return input_seed, splitmix64(input_seed + 1)


# --------------------------------------------------------------------------
# shape algebra: engines.py:70-96, segregation.py:53-58,91-96, engines.py:338-347

def output_dims(in_h: int, in_w: int, n: int, pad: int) -> tuple[int, int]:
    """engines.py:93-96: M = 2N + 2P - n per axis."""
    return 2 * in_h + 2 * pad - n, 2 * in_w + 2 * pad - n


def spec_valid(in_h: int, in_w: int, n: int, pad: int, c_in: int = 1, c_out: int = 1,
               stride: int = 2) -> bool:
    """engines.py:70-86: the TransposeConvSpec validity predicate."""
    if stride != 2 or in_h < 1 or in_w < 1 or n < 2 or pad < 0 or c_in < 1 or c_out < 1:
        return False
    oh, ow = output_dims(in_h, in_w, n, pad)
    return oh >= 1 and ow >= 1


def effective_padding(pad: int) -> tuple[int, int]:
    """segregation.py:91-96: P -> (floor(P/2), P odd)."""
    return pad // 2, pad % 2


def subkernel_dims(n: int, r: int, s: int) -> tuple[int, int]:
    """segregation.py:53-58."""
    return ((n + 1) // 2 if r == 0 else n // 2, (n + 1) // 2 if s == 0 else n // 2)


def parity_grid(out_len: int, parity: int, swap: int) -> tuple[int, int, int]:
    """engines.py:338-347: (first output index, count, first window base)."""
    start = (parity + swap) % 2
    count = max(0, (out_len - start + 1) // 2)
    return start, count, (start + parity) // 2


def mult_count_segregated(in_h, in_w, n, pad, c_in=1, c_out=1) -> int:
    """analysis.py:46-57 + 100-103: useful-MAC count (the metric numerator)."""
    oh, ow = output_dims(in_h, in_w, n, pad)
    swap = pad % 2
    total = 0
    for r in (0, 1):
        rows = max(0, (oh - (r + swap) % 2 + 1) // 2)
        for s in (0, 1):
            cols = max(0, (ow - (s + swap) % 2 + 1) // 2)
            sh, sw = subkernel_dims(n, r, s)
            total += rows * cols * sh * sw
    return total * c_in * c_out


def segregate(kernel: np.ndarray) -> list[np.ndarray]:
    """segregation.py:61-70: [k00, k01, k10, k11] with k_rs[u, v] = K[2u+r, 2v+s]."""
    return [kernel[..., r::2, s::2].copy() for r in (0, 1) for s in (0, 1)]


def merge(subs: list[np.ndarray], n: int) -> np.ndarray:
    """segregation.py:73-88: exact inverse of segregate."""
    out = np.empty(subs[0].shape[:-2] + (n, n), dtype=np.result_type(*subs))
    for idx, (r, s) in enumerate(((0, 0), (0, 1), (1, 0), (1, 1))):
        out[..., r::2, s::2] = subs[idx]
    return out


# --------------------------------------------------------------------------
# engines.py:271-291 -- the vectorised segregated forward (one sample)

def prepare_segregated(bank: np.ndarray, dt) -> list[np.ndarray]:
    """engines.py:236-244: per class (r, s) the contiguous (c_out, c_in*R*C) weight matrix
    (PreparedLayer.__init__, once per weight tensor, outside the forward)."""
    c_out = bank.shape[1]
    return [np.ascontiguousarray(bank[:, :, r::2, s::2].transpose(1, 0, 2, 3).reshape(c_out, -1)).astype(dt)
            for r in (0, 1) for s in (0, 1)]


def forward_segregated(x: np.ndarray, bank: np.ndarray, pad: int, prepared=None) -> np.ndarray:
    """engines.py:236-244 (weight layout) + 271-291 (forward) + 309-335 (GEMM units).

    x: (c_in, H, W); bank: (c_in, c_out, n, n). Returns (c_out, M_h, M_w) in
    np.result_type(x, bank). Every output element is written exactly once.
    prepared: prepare_segregated(bank, dt), else built here.
    """
    c_in, h, w = x.shape
    _, c_out, n, _ = bank.shape
    oh, ow = output_dims(h, w, n, pad)
    p, swap = effective_padding(pad)
    dt = np.result_type(x.dtype, bank.dtype)
    flats = prepared if prepared is not None else prepare_segregated(bank, dt)
    padded = np.pad(x.astype(dt, copy=False), ((0, 0), (p, p), (p, p)))
    out = np.empty((c_out, oh, ow), dtype=dt)
    for r in (0, 1):
        for s in (0, 1):
            sh, sw = subkernel_dims(n, r, s)
            flat = flats[2 * r + s]
            r0, rows, rb = parity_grid(oh, r, swap)
            c0, cols, cb = parity_grid(ow, s, swap)
            if rows == 0 or cols == 0:
                continue
            region = padded[:, rb:rb + rows + sh - 1, cb:cb + cols + sw - 1]
            win = sliding_window_view(region, (sh, sw), axis=(1, 2))
            patches = win.transpose(1, 2, 0, 3, 4).reshape(rows * cols, -1)
            out[:, r0::2, c0::2] = (patches @ flat.T).T.reshape(c_out, rows, cols)
    return out


def forward_segregated_batch(x: np.ndarray, bank: np.ndarray, pad: int,
                             workers: int | None = None) -> np.ndarray:
    """Batch = independent map over samples; thread pool over samples."""
    workers = workers or os.cpu_count() or 1
    if workers == 1 or x.shape[0] == 1:
        return np.stack([forward_segregated(xi, bank, pad) for xi in x])
    with ThreadPoolExecutor(max_workers=workers) as pool:
        outs = list(pool.map(lambda xi: forward_segregated(xi, bank, pad), x))
    return np.stack(outs)


# --------------------------------------------------------------------------
# engines.py:134-140, 258-269, tensors.py:76-112 -- Alg. 1 (bed of nails)

def forward_reference(x: np.ndarray, bank: np.ndarray, pad: int, prepared=None) -> np.ndarray:
    """Upsample (zero insertion) -> zero pad P -> valid correlation, unflipped kernel.
    prepared: the (c_out, c_in*n*n) weight matrix (engines.py:232-235), else built here."""
    c_in, h, w = x.shape
    _, c_out, n, _ = bank.shape
    oh, ow = output_dims(h, w, n, pad)
    dt = np.result_type(x.dtype, bank.dtype)
    up = np.zeros((c_in, 2 * h - 1 + 2 * pad, 2 * w - 1 + 2 * pad), dtype=dt)
    up[:, pad:pad + 2 * h - 1:2, pad:pad + 2 * w - 1:2] = x
    win = sliding_window_view(up, (n, n), axis=(1, 2))
    patches = win.transpose(1, 2, 0, 3, 4).reshape(oh * ow, -1)
    flat = prepared if prepared is not None else np.ascontiguousarray(
        bank.transpose(1, 0, 2, 3).reshape(c_out, -1)).astype(dt)
    return (patches @ flat.T).T.reshape(c_out, oh, ow)


# --------------------------------------------------------------------------
# engines.py:379-406 -- literal per-element unified rule (pure Python, small)

def forward_scalar(x: np.ndarray, bank: np.ndarray, pad: int):
    """Per output element: pick sub-kernel by parity (with the odd-P swap), sum
    over ci ascending, then u, v. fp64. Returns (out, mults, writes)."""
    c_in, h, w = x.shape
    _, c_out, n, _ = bank.shape
    oh, ow = output_dims(h, w, n, pad)
    p, swap = effective_padding(pad)
    xs = x.astype(np.float64).tolist()
    ks = bank.astype(np.float64).tolist()
    out = np.zeros((c_out, oh, ow))
    mults = writes = 0
    for co in range(c_out):
        for xx in range(oh):
            r = (xx + swap) % 2
            bx = (xx + r) // 2
            for yy in range(ow):
                s = (yy + swap) % 2
                by = (yy + s) // 2
                sh, sw = subkernel_dims(n, r, s)
                acc = 0.0
                for ci in range(c_in):
                    for u in range(sh):
                        ii = bx + u - p
                        for v in range(sw):
                            jj = by + v - p
                            val = xs[ci][ii][jj] if 0 <= ii < h and 0 <= jj < w else 0.0
                            acc += val * ks[ci][co][2 * u + r][2 * v + s]
                            mults += 1
                out[co, xx, yy] = acc
                writes += 1
    return out, mults, writes


def forward_scalar_reference(m: np.ndarray, k: np.ndarray, pad: int):
    """engines.py:353-376 -- Alg. 1 per element on one map: bed-of-nails upsample
    (tensors.py:85-95), zero pad P, all n x n taps (zeros included). fp64, (u, v) order.
    Returns (out, mults, writes)."""
    h, w = m.shape
    n = k.shape[0]
    oh, ow = output_dims(h, w, n, pad)
    up = np.zeros((2 * h - 1 + 2 * pad, 2 * w - 1 + 2 * pad), dtype=np.float64)
    up[pad:pad + 2 * h - 1:2, pad:pad + 2 * w - 1:2] = m
    ul = up.tolist()
    kl = k.astype(np.float64).tolist()
    out = np.zeros((oh, ow))
    mults = writes = 0
    for xx in range(oh):
        for yy in range(ow):
            acc = 0.0
            for u in range(n):
                for v in range(n):
                    acc += ul[xx + u][yy + v] * kl[u][v]
                    mults += 1
            out[xx, yy] = acc
            writes += 1
    return out, mults, writes


# --------------------------------------------------------------------------
# engines.py:175-198 -- the parity verdict

def compare(a: np.ndarray, b: np.ndarray, rel_tol: float = 1e-5, abs_tol: float = 1e-6) -> dict:
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return {"shapes_match": False, "max_abs_diff": None, "max_rel_diff": None,
                "rel_tol": rel_tol, "abs_tol": abs_tol, "passed": False}
    a64 = a.astype(np.float64)
    b64 = b.astype(np.float64)
    d = np.abs(a64 - b64)
    den = np.maximum(np.abs(a64), np.abs(b64))
    rel = np.divide(d, den, out=np.zeros_like(d), where=den > 0)
    return {"shapes_match": True,
            "max_abs_diff": float(d.max()) if d.size else 0.0,
            "max_rel_diff": float(rel.max()) if rel.size else 0.0,
            "rel_tol": rel_tol, "abs_tol": abs_tol,
            "passed": bool(np.all(d <= abs_tol + rel_tol * np.abs(b64)))}


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 -> float32 (for bf16 parity gates)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32)
