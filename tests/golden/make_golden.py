"""Freeze golden vectors from the reference implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the *unmodified* reference package from /root/reference/pkg/src and
writes tests/golden/reference_golden.npz. The GPU box never has
/root/reference; tests there only read the committed .npz.

Contents (all produced by reference code paths, cited):
  * kat_*       frozen known answers (tests/test_engines.py:65-100)
  * splitmix    splitmix64 / unit_floats samples (synth.py:20-39)
  * counts      mult_count_segregated for many specs (analysis.py:46-57)
  * seg_*       segregate_kernel outputs for n = 2..9 (segregation.py:61-70)
  * case{i}_*   random layer cases: x, bank, pad, the reference's segregated
                engine output in fp32 and fp64, and its reference (Alg. 1)
                engine output in fp64 (engines.py:163-172)
  * gan{i}_*    small GAN-shaped layers driven by the harness seed rule
                (bench.py:299-300) with the reference segregated output
  * cnt{i}_*    the instrumented scalar engines (engines.py:353-406) on small
                maps: output (fp64) and the mults / writes counters of both
                transpose_conv_reference_counted and _segregated_counted
"""

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.dont_write_bytecode = True

import segconv  # noqa: E402  (the reference)
from segconv import analysis, engines, segregation, synth  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")


def main():
    g = {}
    f32 = np.float32
    # --- known answers (test_engines.py:65-100) -------------------------------
    x = np.array([[1, 2], [3, 4]], dtype=f32)
    k = np.array([[1, 2], [3, 4]], dtype=f32)
    g["kat_p0"] = engines.transpose_conv_segregated(x, segregation.segregate_kernel(k), 0)
    g["kat_p1"] = engines.transpose_conv_segregated(x, segregation.segregate_kernel(k), 1)
    g["kat_p1_ref"] = engines.transpose_conv_reference(x, k, 1)
    g["kat_ones"] = engines.transpose_conv_segregated(x, segregation.segregate_kernel(np.ones((2, 2), f32)), 0)
    # --- synth (synth.py) -------------------------------------------------------
    seeds = [0, 1, 42, 2**63, (1 << 64) - 1, -7, 123456789]
    g["splitmix_in"] = np.array([s & ((1 << 64) - 1) for s in seeds], dtype=np.uint64)
    g["splitmix_out"] = np.array([synth.splitmix64(s & ((1 << 64) - 1)) for s in seeds], dtype=np.uint64)
    g["unit_floats_seeds"] = np.array([s & ((1 << 64) - 1) for s in seeds], dtype=np.uint64)
    g["unit_floats"] = np.stack([synth.unit_floats(64, s) for s in seeds])
    g["gen_synthetic_3_5_7_s9"] = synth.gen_synthetic(3, 5, 7, 9)
    g["gen_kernel_bank_2_3_4_s11"] = synth.gen_kernel_bank(2, 3, 4, 11)
    # --- counts (analysis.py) ------------------------------------------------------
    specs = []
    for (h, w, n, p, ci, co) in [(4, 4, 5, 0, 1, 1), (4, 4, 4, 2, 1, 1), (28, 28, 3, 0, 1, 1),
                                 (28, 28, 3, 1, 1, 1), (28, 28, 3, 2, 1, 1), (224, 224, 3, 2, 3, 1),
                                 (224, 224, 4, 2, 3, 1), (224, 224, 5, 2, 3, 1), (512, 512, 5, 2, 3, 1),
                                 (5, 7, 3, 1, 2, 3), (3, 4, 7, 3, 1, 1), (1, 2, 2, 1, 1, 1)]:
        specs.append((h, w, n, p, ci, co))
    for cfg in segconv.GAN_SUITE:
        specs.append((cfg.input_h, cfg.input_w, cfg.kernel_n, cfg.pad, cfg.c_in, cfg.c_out))
    g["count_specs"] = np.array(specs, dtype=np.int64)
    g["count_seg"] = np.array([analysis.mult_count_segregated(engines.TransposeConvSpec(
        in_h=h, in_w=w, kernel_n=n, pad=p, c_in=ci, c_out=co)) for (h, w, n, p, ci, co) in specs],
        dtype=np.int64)
    g["count_ref"] = np.array([analysis.mult_count_reference(engines.TransposeConvSpec(
        in_h=h, in_w=w, kernel_n=n, pad=p, c_in=ci, c_out=co)) for (h, w, n, p, ci, co) in specs],
        dtype=np.int64)
    # --- segregation -----------------------------------------------------------------
    for n in range(2, 10):
        kk = np.arange(n * n, dtype=f32).reshape(n, n)
        subs = segregation.segregate_kernel(kk)
        for name in ("k00", "k01", "k10", "k11"):
            g[f"seg_n{n}_{name}"] = getattr(subs, name)
    # --- random layer cases (test_engines.py:121-143 draw, acceptance ranges) ---------
    rng = np.random.default_rng(20260810)
    cases = 0
    while cases < 160:
        h = int(rng.integers(1, 17))
        w = int(rng.integers(1, 17))
        n = int(rng.integers(2, 10))
        pad = int(rng.integers(0, 5))
        if 2 * h + 2 * pad - n < 1 or 2 * w + 2 * pad - n < 1:
            continue
        ci = int(rng.integers(1, 5))
        co = int(rng.integers(1, 5))
        x64 = rng.random((ci, h, w))
        b64 = rng.random((ci, co, n, n))
        x32, b32 = x64.astype(f32), b64.astype(f32)
        g[f"case{cases}_x"] = x64
        g[f"case{cases}_bank"] = b64
        g[f"case{cases}_pad"] = np.int64(pad)
        g[f"case{cases}_seg32"] = engines.layer_forward(x32, b32, pad, engine=engines.ENGINE_SEGREGATED)
        g[f"case{cases}_seg64"] = engines.layer_forward(x64, b64, pad, engine=engines.ENGINE_SEGREGATED)
        g[f"case{cases}_ref64"] = engines.layer_forward(x64, b64, pad, engine=engines.ENGINE_REFERENCE)
        cases += 1
    g["n_cases"] = np.int64(cases)
    # --- GAN-shaped layers through the harness seed rule -------------------------------
    gan = [("mini_dcgan", 4, 4, 128, 4, 64, 2), ("mini_ebgan7", 16, 16, 64, 4, 64, 2),
           ("mnist_p1", 28, 28, 1, 3, 1, 1), ("ds_k5", 32, 32, 3, 5, 1, 2)]
    for i, (name, h, w, ci, n, co, pad) in enumerate(gan):
        in_seed = synth.splitmix64(7 + 2 * i)
        bank_seed = synth.splitmix64(in_seed + 1)
        xg = synth.gen_synthetic(ci, h, w, in_seed)
        bg = synth.gen_kernel_bank(ci, co, n, bank_seed)
        g[f"gan{i}_meta"] = np.array([h, w, ci, n, co, pad, in_seed, bank_seed], dtype=np.uint64)
        g[f"gan{i}_out"] = engines.layer_forward(xg, bg, pad, engine=engines.ENGINE_SEGREGATED)
    g["n_gan"] = np.int64(len(gan))
    # --- instrumented scalar engines (engines.py:353-406), own RNG stream ---------------
    crng = np.random.default_rng(353)
    cnt = 0
    while cnt < 24:
        h = int(crng.integers(1, 10))
        w = int(crng.integers(1, 10))
        n = int(crng.integers(2, 8))
        pad = int(crng.integers(0, 5))
        if 2 * h + 2 * pad - n < 1 or 2 * w + 2 * pad - n < 1:
            continue
        dt = np.float64 if cnt % 2 else f32
        m = crng.random((h, w)).astype(dt)
        kk = crng.random((n, n)).astype(dt)
        ref_out, cr = engines.transpose_conv_reference_counted(m, kk, pad)
        seg_out, cs = engines.transpose_conv_segregated_counted(m, segregation.segregate_kernel(kk), pad)
        g[f"cnt{cnt}_map"] = m
        g[f"cnt{cnt}_kernel"] = kk
        g[f"cnt{cnt}_pad"] = np.int64(pad)
        g[f"cnt{cnt}_ref"] = ref_out
        g[f"cnt{cnt}_seg"] = seg_out
        g[f"cnt{cnt}_counts"] = np.array([cr.mults, cr.writes, cs.mults, cs.writes], dtype=np.int64)
        cnt += 1
    g["n_cnt"] = np.int64(cnt)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
