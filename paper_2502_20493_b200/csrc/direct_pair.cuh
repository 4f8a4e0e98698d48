// K2p -- the direct kernel for the low-channel layers (dataset images; n = 4, 5, c_out <= 3 and a
// weight tensor of at most kPairWMax floats), fp32 compute with packed FFMA2.
//
// Same per-element rule, summation order and outputs as K2 (direct_impl.cuh; spec
// /root/reference/pkg/src/segconv/engines.py:379-406, ascending ci as engines.py:163-172), so
// the results are bitwise K2's. What differs is the mapping onto the SM:
//   - two samples per thread: every register of the input window and of the accumulators is a
//     float2 (sample b in .x, sample b + 1 in .y), so each multiply-add of the rule is one lane of
//     an FFMA2 (sm_100: two fp32 FMAs per instruction) -- half the FMA instructions of K2, and
//     the pairs come straight from the loads (no register shuffling);
//   - the class-packed weights are a __grid_constant__ kernel parameter: warp-uniform values the
//     FFMA2s read as uniform-register broadcast operands, so they take no vector registers and no
//     shared-memory traffic (K2 stages them through shared memory and holds a tap vector in
//     registers, which spilled for n = 5 under the six-blocks-per-SM register cap).
#pragma once

#include "direct_impl.cuh"
#include "tc_ptx.cuh"

namespace segb {

#ifndef SEGB_DIRECT_PAIR_PIPE  // double-buffered window loads across input channels
#define SEGB_DIRECT_PAIR_PIPE 1
#endif
struct PairWeights {  // kPairWMax (direct_impl.cuh) floats: a 3.5 KB kernel parameter
    float w[kPairWMax];
};

template <typename TX, int N, int COB, int RQ, int CQ, bool PIPE>
// (one channel: 2 x 2 quads, 64 live float registers of window and accumulators -> 5 blocks per
// SM so nothing spills; two: 2 x 1 quads in 80 registers, 6 blocks; three: 4 blocks; PIPE's
// second window: 4 blocks)
__global__ void __launch_bounds__(128, PIPE ? 4 : COB == 1 ? 5 : COB == 2 ? 6 : 4)
    direct_pair_kernel(DirectArgs a, const __grid_constant__ PairWeights W) {
    constexpr int NW = N / 2 + 1;    // input rows/cols under one output quad
    constexpr int WR = RQ + NW - 1;  // window rows for RQ row quads
    constexpr int WC = CQ + NW - 1;  // window cols for CQ column quads
    constexpr int R0 = (N + 1) / 2, R1 = N / 2;
    constexpr int OFF1 = R0 * R0, OFF2 = R0 * R0 + R0 * R1, OFF3 = R0 * R0 + 2 * R0 * R1;
    constexpr int N2P = (N * N + 3) / 4 * 4;
    extern __shared__ __align__(16) unsigned char smem_raw[];

    const int t0 = (blockIdx.x * 32 + threadIdx.x) * CQ;  // first column quad
    const int q0 = (blockIdx.y * kDirectRowsPerBlock + threadIdx.y) * RQ;
    const int64_t b = a.b0 + 2 * (int64_t)blockIdx.z;  // samples b and b + 1 (if it exists)
    const bool two = b + 1 < a.batch;
    const int row0 = q0 - a.swap - a.p, col0 = t0 - a.swap - a.p;
    const int64_t plane = (int64_t)a.h * a.w_in;
    constexpr bool HWC = XLayout<TX>::HWC;
    const int es = HWC ? a.c_in : 1;              // column (element) stride
    const int64_t rs = (int64_t)a.w_in * es;      // row stride
    const int64_t cs = XLayout<TX>::chan(plane);  // channel stride
    const int64_t ss = (int64_t)a.c_in * plane;   // sample stride
    const TX *xb = reinterpret_cast<const TX *>(a.x) + b * ss;

    float2 acc[COB][2 * RQ][2 * CQ];
#pragma unroll
    for (int c = 0; c < COB; ++c)
#pragma unroll
        for (int i = 0; i < 2 * RQ; ++i)
#pragma unroll
            for (int k = 0; k < 2 * CQ; ++k) acc[c][i][k] = make_float2(0.f, 0.f);

    const bool inside = row0 >= 0 && row0 + WR <= a.h && col0 >= 0 && col0 + WC <= a.w_in;
    const bool warp_inside = __all_sync(0xffffffffu, inside) && __all_sync(0xffffffffu, two);
    bool rok[WR], cok[WC];
#pragma unroll
    for (int i = 0; i < WR; ++i) rok[i] = (unsigned)(row0 + i) < (unsigned)a.h;
#pragma unroll
    for (int j = 0; j < WC; ++j) cok[j] = (unsigned)(col0 + j) < (unsigned)a.w_in;
    const TX *xw = xb + (int64_t)row0 * rs + (int64_t)col0 * es;  // window origin (may point outside)

    auto load_win = [&](float2 (&win)[WR][WC], int ci) {
        const TX *xc = xw + (int64_t)ci * cs;
        if (warp_inside) {
#pragma unroll
            for (int i = 0; i < WR; ++i)
#pragma unroll
                for (int j = 0; j < WC; ++j) {
                    const TX *p = xc + i * rs + j * es;
                    win[i][j] = make_float2(load_x<TX, float, false>(p), load_x<TX, float, false>(p + ss));
                }
        } else {
#pragma unroll
            for (int i = 0; i < WR; ++i)
#pragma unroll
                for (int j = 0; j < WC; ++j) {
                    const TX *p = xc + i * rs + j * es;
                    const bool ok = rok[i] && cok[j];
                    win[i][j] = make_float2(ok ? load_x<TX, float, false>(p) : 0.f,
                                            (ok && two) ? load_x<TX, float, false>(p + ss) : 0.f);
                }
        }
    };
    auto compute = [&](const float2 (&win)[WR][WC], int ci) {
#pragma unroll
        for (int c = 0; c < COB; ++c) {
            const float *wv = W.w + (c * a.c_in + ci) * N2P;  // uniform: broadcast operands
            auto fma2 = [&](float2 &d, const float2 &x, float w) { d = __ffma2_rn(x, make_float2(w, w), d); };
#pragma unroll
            for (int qq = 0; qq < RQ; ++qq)
#pragma unroll
                for (int cq = 0; cq < CQ; ++cq) {
#pragma unroll
                    for (int u = 0; u < R0; ++u) {
#pragma unroll
                        for (int v = 0; v < R0; ++v) fma2(acc[c][2 * qq][2 * cq], win[qq + u][cq + v], wv[u * R0 + v]);
#pragma unroll
                        for (int v = 0; v < R1; ++v)
                            fma2(acc[c][2 * qq][2 * cq + 1], win[qq + u][cq + 1 + v], wv[OFF1 + u * R1 + v]);
                    }
#pragma unroll
                    for (int u = 0; u < R1; ++u) {
#pragma unroll
                        for (int v = 0; v < R0; ++v)
                            fma2(acc[c][2 * qq + 1][2 * cq], win[qq + 1 + u][cq + v], wv[OFF2 + u * R0 + v]);
#pragma unroll
                        for (int v = 0; v < R1; ++v)
                            fma2(acc[c][2 * qq + 1][2 * cq + 1], win[qq + 1 + u][cq + 1 + v], wv[OFF3 + u * R1 + v]);
                    }
                }
        }
    };
    float2 wa[WR][WC];
    if constexpr (PIPE) {
        // the next channel's window loads in flight while the current one is multiplied (two
        // window buffers used alternately, no register copies)
        float2 wb[WR][WC];
        load_win(wa, 0);
#pragma unroll 1
        for (int ci = 0; ci < a.c_in; ci += 2) {
            if (ci + 1 < a.c_in) load_win(wb, ci + 1);
            compute(wa, ci);
            if (ci + 1 >= a.c_in) break;
            if (ci + 2 < a.c_in) load_win(wa, ci + 2);
            compute(wb, ci + 1);
        }
    } else {
#pragma unroll 1
        for (int ci = 0; ci < a.c_in; ++ci) {
            load_win(wa, ci);
            compute(wa, ci);
        }
    }

    // stores as K2: staged per warp through shared memory so each store instruction writes 32
    // consecutive outputs of one row; one sample at a time
    constexpr int SC = 64 * CQ;
    float *stg = reinterpret_cast<float *>(smem_raw) + threadIdx.y * (COB * 2 * RQ * SC);
    float *yb = reinterpret_cast<float *>(a.y);
    const int y0 = 2 * (blockIdx.x * 32 * CQ) - a.swap;  // first output column of the warp
#pragma unroll
    for (int sidx = 0; sidx < 2; ++sidx) {
        if (sidx == 1 && !two) break;
#pragma unroll
        for (int c = 0; c < COB; ++c)
#pragma unroll
            for (int i = 0; i < 2 * RQ; ++i)
#pragma unroll
                for (int k = 0; k < 2 * CQ; ++k)
                    stg[(c * 2 * RQ + i) * SC + threadIdx.x * 2 * CQ + k] = sidx ? acc[c][i][k].y : acc[c][i][k].x;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < COB; ++c) {
            float *yc = yb + ((b + sidx) * a.c_out + c) * a.oh * a.ow;
#pragma unroll
            for (int i = 0; i < 2 * RQ; ++i) {
                const int xo = 2 * q0 + i - a.swap;
                if ((unsigned)xo >= (unsigned)a.oh) continue;
                float *row = yc + (int64_t)xo * a.ow;
#pragma unroll
                for (int m = 0; m < 2 * CQ; ++m) {
                    const int col = m * 32 + threadIdx.x;
                    const int yo = y0 + col;
                    if ((unsigned)yo < (unsigned)a.ow) row[yo] = stg[(c * 2 * RQ + i) * SC + col];
                }
            }
        }
        __syncwarp();
    }
}

// K2p with TMA-staged input tiles (fp32 x, W % 4 == 0): per input channel one 4-D TMA box
// (tile columns x tile rows x 1 channel x 2 samples) lands the block's input window in shared
// memory, double-buffered across channels and zero-filled outside the image (no predicated
// loads); threads read their register windows from shared memory. Same rule, order and bits as
// K2p / K2.
// WSM: the weights (too many for the kernel parameter, e.g. dcgan_l5: 128 x 3 x 16) are copied
// from a.w into shared memory at block start and read as broadcast loads
#ifndef SEGB_PAIR_TMA_MINB1  // blocks per SM of the one-channel TMA-staged kernel
#define SEGB_PAIR_TMA_MINB1 6  // measured: ds512_k5 0.117 -> 0.110 ms (8: spills and loses)
#endif
template <int N, int COB, int RQ, int CQ, int TR, int TC, bool WSM = false>
// (three channels: 5 blocks per SM with the weights in the parameter, ds512_k4_c3 0.282 -> 0.256 ms;
// 4 with the weights in shared memory, dcgan_l5 0.120 vs 0.124)
__global__ void __launch_bounds__(128, COB == 1 ? SEGB_PAIR_TMA_MINB1 : COB == 2 ? 6 : (WSM ? 4 : 5))
    direct_pair_tma_kernel(const __grid_constant__ CUtensorMap tmX, DirectArgs a, const __grid_constant__ PairWeights W) {
    constexpr int NW = N / 2 + 1;
    constexpr int WR = RQ + NW - 1, WC = CQ + NW - 1;
    constexpr int R0 = (N + 1) / 2, R1 = N / 2;
    constexpr int OFF1 = R0 * R0, OFF2 = R0 * R0 + R0 * R1, OFF3 = R0 * R0 + 2 * R0 * R1;
    constexpr int N2P = (N * N + 3) / 4 * 4;
    constexpr int TILE = (2 * TR * TC + 31) / 32 * 32;  // floats per buffer ([sample][row][col]), 128-B aligned
    extern __shared__ __align__(128) unsigned char smem_dyn[];
    // TMA destinations: 128-byte aligned (the dynamic shared-memory base is only guaranteed 16)
    unsigned char *smem_raw =
        reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_dyn) + 127) & ~uintptr_t(127));
    float *tiles = reinterpret_cast<float *>(smem_raw);                                   // 2 buffers
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw + 2 * TILE * sizeof(float));   // 2 barriers
    float *stg_base = reinterpret_cast<float *>(smem_raw + 2 * TILE * sizeof(float) + 64);
    const int tid = threadIdx.y * 32 + threadIdx.x;
    // WSM: the weights after the store staging area
    float *sW = stg_base + kDirectRowsPerBlock * COB * 2 * RQ * 64 * CQ;
    if constexpr (WSM) {
        const int nw4 = COB * a.c_in * N2P / 4;  // N2P % 4 == 0
        const float4 *src = reinterpret_cast<const float4 *>(a.w);
        for (int i = tid; i < nw4; i += blockDim.x * blockDim.y) reinterpret_cast<float4 *>(sW)[i] = __ldg(src + i);
    }
    const int qb = blockIdx.y * kDirectRowsPerBlock * RQ, tb = blockIdx.x * 32 * CQ;  // block's first quads
    const int q0 = qb + threadIdx.y * RQ;
    const int64_t b = a.b0 + 2 * (int64_t)blockIdx.z;
    const bool two = b + 1 < a.batch;
    // tile origin in the input; the box's first column is rounded down to a multiple of 4 floats
    // (a TMA box without swizzle must start 16-byte aligned in its inner dimension, negative
    // coordinates included: measured, an unaligned start faults), dc columns before the window
    const int brow = qb - a.swap - a.p, bcol_w = tb - a.swap - a.p;
    const int dc = ((bcol_w % 4) + 4) % 4, bcol = bcol_w - dc;
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    }
    __syncthreads();
    auto issue = [&](int ci) {
        float *dst = tiles + (ci & 1) * TILE;
        mbar_expect_tx(&full[ci & 1], 2 * TR * TC * sizeof(float));
        tma_load_4d(dst, &tmX, &full[ci & 1], bcol, brow, ci, (int)b);
    };
    if (tid == 0) {
        issue(0);
        if (a.c_in > 1) issue(1);
    }
    float2 acc[COB][2 * RQ][2 * CQ];
#pragma unroll
    for (int c = 0; c < COB; ++c)
#pragma unroll
        for (int i = 0; i < 2 * RQ; ++i)
#pragma unroll
            for (int k = 0; k < 2 * CQ; ++k) acc[c][i][k] = make_float2(0.f, 0.f);
    const int wr0 = threadIdx.y * RQ, wc0 = threadIdx.x * CQ + dc;  // this thread's window in the tile
#pragma unroll 1
    for (int ci = 0; ci < a.c_in; ++ci) {
        mbar_wait(&full[ci & 1], (ci >> 1) & 1);
        const float *t0 = tiles + (ci & 1) * TILE;
        float2 win[WR][WC];
#pragma unroll
        for (int i = 0; i < WR; ++i)
#pragma unroll
            for (int j = 0; j < WC; ++j)
                win[i][j] = make_float2(t0[(wr0 + i) * TC + wc0 + j], t0[TR * TC + (wr0 + i) * TC + wc0 + j]);
        __syncthreads();  // every thread has its window: the buffer may be refilled
        if (tid == 0 && ci + 2 < a.c_in) issue(ci + 2);
#pragma unroll
        for (int c = 0; c < COB; ++c) {
            const float *wv = (WSM ? sW : W.w) + (c * a.c_in + ci) * N2P;
            auto fma2 = [&](float2 &d, const float2 &x, float w) { d = __ffma2_rn(x, make_float2(w, w), d); };
#pragma unroll
            for (int qq = 0; qq < RQ; ++qq)
#pragma unroll
                for (int cq = 0; cq < CQ; ++cq) {
#pragma unroll
                    for (int u = 0; u < R0; ++u) {
#pragma unroll
                        for (int v = 0; v < R0; ++v) fma2(acc[c][2 * qq][2 * cq], win[qq + u][cq + v], wv[u * R0 + v]);
#pragma unroll
                        for (int v = 0; v < R1; ++v)
                            fma2(acc[c][2 * qq][2 * cq + 1], win[qq + u][cq + 1 + v], wv[OFF1 + u * R1 + v]);
                    }
#pragma unroll
                    for (int u = 0; u < R1; ++u) {
#pragma unroll
                        for (int v = 0; v < R0; ++v)
                            fma2(acc[c][2 * qq + 1][2 * cq], win[qq + 1 + u][cq + v], wv[OFF2 + u * R0 + v]);
#pragma unroll
                        for (int v = 0; v < R1; ++v)
                            fma2(acc[c][2 * qq + 1][2 * cq + 1], win[qq + 1 + u][cq + 1 + v], wv[OFF3 + u * R1 + v]);
                    }
                }
        }
    }
    // stores as K2p (per-warp shared-memory staging, one sample at a time)
    constexpr int SC = 64 * CQ;
    float *stg = stg_base + threadIdx.y * (COB * 2 * RQ * SC);
    float *yb = reinterpret_cast<float *>(a.y);
    const int y0 = 2 * tb - a.swap;
#pragma unroll
    for (int sidx = 0; sidx < 2; ++sidx) {
        if (sidx == 1 && !two) break;
#pragma unroll
        for (int c = 0; c < COB; ++c)
#pragma unroll
            for (int i = 0; i < 2 * RQ; ++i)
#pragma unroll
                for (int k = 0; k < 2 * CQ; ++k)
                    stg[(c * 2 * RQ + i) * SC + threadIdx.x * 2 * CQ + k] = sidx ? acc[c][i][k].y : acc[c][i][k].x;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < COB; ++c) {
            float *yc = yb + ((b + sidx) * a.c_out + c) * a.oh * a.ow;
#pragma unroll
            for (int i = 0; i < 2 * RQ; ++i) {
                const int xo = 2 * q0 + i - a.swap;
                if ((unsigned)xo >= (unsigned)a.oh) continue;
                float *row = yc + (int64_t)xo * a.ow;
#pragma unroll
                for (int m = 0; m < 2 * CQ; ++m) {
                    const int col = m * 32 + threadIdx.x;
                    const int yo = y0 + col;
                    if ((unsigned)yo < (unsigned)a.ow) row[yo] = stg[(c * 2 * RQ + i) * SC + col];
                }
            }
        }
        __syncwarp();
    }
}

#ifndef SEGB_DIRECT_PAIR_TMA
#define SEGB_DIRECT_PAIR_TMA 1
#endif

template <int N, int COB, bool WSM = false>
int launch_direct_pair_tma_n(const DirectArgs &a, const PairWeights &W, cudaStream_t st) {
    constexpr int RQ = 2, CQ = COB == 1 ? 2 : 1;
    constexpr int NW = N / 2 + 1;
    constexpr int TR = kDirectRowsPerBlock * RQ + NW - 1;
    constexpr int TC = (32 * CQ + NW - 1 + 3 + 3) / 4 * 4;  // 16-byte rows, 3 columns of start alignment
    auto enc = tensor_map_encoder();
    if (!enc) return fail(SEGB_ERR_UNSUPPORTED, "paired direct kernel (TMA): no tensor-map encoder");
    CUtensorMap tm;
    const cuuint64_t dims[4] = {(cuuint64_t)a.w_in, (cuuint64_t)a.h, (cuuint64_t)a.c_in, (cuuint64_t)a.batch};
    const cuuint64_t strides[3] = {(cuuint64_t)a.w_in * 4, (cuuint64_t)a.h * a.w_in * 4,
                                   (cuuint64_t)a.c_in * a.h * a.w_in * 4};
    const cuuint32_t box[4] = {(cuuint32_t)TC, (cuuint32_t)TR, 1, 2};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void *>(a.x), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SEGB_ERR_CUDA, "paired direct kernel: tensor map (%d)", (int)r);
    dim3 block(32, kDirectRowsPerBlock);
    const int64_t nrb = ceil_div(a.nqr, kDirectRowsPerBlock * RQ);
    if (nrb > 65535) return fail(SEGB_ERR_UNSUPPORTED, "output too large for the paired direct kernel grid");
    const size_t smem = 128 + 2 * ((2 * TR * TC + 31) / 32 * 32) * sizeof(float) + 64 +
                        sizeof(float) * kDirectRowsPerBlock * COB * 2 * RQ * 64 * CQ +
                        (WSM ? sizeof(float) * COB * a.c_in * a.n2p : 0);
    auto kern = direct_pair_tma_kernel<N, COB, RQ, CQ, TR, TC, WSM>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t pairs = ceil_div(a.batch, 2);
    for (int64_t p0 = 0; p0 < pairs; p0 += 65535) {
        DirectArgs c = a;
        c.b0 = 2 * p0;
        dim3 grid((unsigned)ceil_div(a.nqc, 32 * CQ), (unsigned)nrb, (unsigned)std::min<int64_t>(65535, pairs - p0));
        kern<<<grid, block, smem, st>>>(tm, c, W);
        note_launch();
        if (int rc = check_launch("direct_pair_tma_kernel")) return rc;
    }
    return SEGB_OK;
}

template <typename TX, int N, int COB>
int launch_direct_pair_n(const DirectArgs &a, const PairWeights &W, cudaStream_t st) {
    // one channel: 2 x 2 quads (window 4 x 4 pairs); two or three channels: 2 x 1
    constexpr int RQ = 2, CQ = COB == 1 ? 2 : 1;
    dim3 block(32, kDirectRowsPerBlock);
    const int64_t nrb = ceil_div(a.nqr, kDirectRowsPerBlock * RQ);
    if (nrb > 65535) return fail(SEGB_ERR_UNSUPPORTED, "output too large for the paired direct kernel grid");
    const size_t smem = sizeof(float) * kDirectRowsPerBlock * COB * 2 * RQ * 64 * CQ;
    const int64_t pairs = ceil_div(a.batch, 2);
    for (int64_t p0 = 0; p0 < pairs; p0 += 65535) {
        DirectArgs c = a;
        c.b0 = 2 * p0;
        dim3 grid((unsigned)ceil_div(a.nqc, 32 * CQ), (unsigned)nrb, (unsigned)std::min<int64_t>(65535, pairs - p0));
        // (measured: three channels ds512_k4_c3 0.302 -> 0.286 ms, n = 5 ds224_k5 0.036 -> 0.034;
        // one channel with n = 4, ds224_k4, 0.032 -> 0.034: the occupancy it costs is not repaid)
        if (SEGB_DIRECT_PAIR_PIPE && a.c_in > 1 && (COB == 3 || N == 5))
            direct_pair_kernel<TX, N, COB, RQ, CQ, true><<<grid, block, smem, st>>>(c, W);
        else
            direct_pair_kernel<TX, N, COB, RQ, CQ, false><<<grid, block, smem, st>>>(c, W);
        note_launch();
        if (int rc = check_launch("direct_pair_kernel")) return rc;
    }
    return SEGB_OK;
}

// fp32 x, W % 4 == 0, n 3..5, c_out <= 3, weights too many for the parameter (direct_pair_wsm_ok):
// the TMA-staged kernel with its weights in shared memory, read from the layer's K2 weights (a.w)
template <int N>
int launch_direct_pair_wsm_n(const DirectArgs &a, cudaStream_t st) {
    static PairWeights unused{};  // (the parameter slot the WSM instance does not read)
    if (a.c_out == 1) return launch_direct_pair_tma_n<N, 1, true>(a, unused, st);
    if (a.c_out == 2) return launch_direct_pair_tma_n<N, 2, true>(a, unused, st);
    return launch_direct_pair_tma_n<N, 3, true>(a, unused, st);
}
inline int launch_direct_pair_wsm_impl(const DirectArgs &a, cudaStream_t st) {
    if (a.n == 3) return launch_direct_pair_wsm_n<3>(a, st);
    if (a.n == 4) return launch_direct_pair_wsm_n<4>(a, st);
    return launch_direct_pair_wsm_n<5>(a, st);
}

inline int launch_direct_pair_tma_n3(const DirectArgs &a, const PairWeights &W, cudaStream_t st) {
    if (a.w_in % 4 != 0) return fail(SEGB_ERR_UNSUPPORTED, "paired direct kernel: n = 3 needs W % 4 == 0");
    if (a.c_out == 1) return launch_direct_pair_tma_n<3, 1>(a, W, st);
    if (a.c_out == 2) return launch_direct_pair_tma_n<3, 2>(a, W, st);
    return launch_direct_pair_tma_n<3, 3>(a, W, st);
}

template <typename TX, int N>
int launch_direct_pair_cob(const DirectArgs &a, const PairWeights &W, cudaStream_t st) {
    if constexpr (sizeof(TX) == 4) {  // fp32 NCHW with 16-byte rows: TMA-staged input tiles
        // (measured, batch 64: ds512_k5 0.130 -> 0.116 ms, ds224_k5 0.035 -> 0.028, ds224_k4
        // 0.032 -> 0.028, ds512_k4_c3 0.286 -> 0.283)
        if (SEGB_DIRECT_PAIR_TMA && direct_pair_tma_enabled() && a.w_in % 4 == 0) {
            if (a.c_out == 1) return launch_direct_pair_tma_n<N, 1>(a, W, st);
            if (a.c_out == 2) return launch_direct_pair_tma_n<N, 2>(a, W, st);
            return launch_direct_pair_tma_n<N, 3>(a, W, st);
        }
    }
    if (a.c_out == 1) return launch_direct_pair_n<TX, N, 1>(a, W, st);
    if (a.c_out == 2) return launch_direct_pair_n<TX, N, 2>(a, W, st);
    return launch_direct_pair_n<TX, N, 3>(a, W, st);
}

// w_host: the K2 class-packed weights [c_out][c_in][n2p] (fp32) on the host
template <typename TX>
int launch_direct_pair(const DirectArgs &a, const float *w_host, cudaStream_t st) {
    PairWeights W;
    const int64_t nw = (int64_t)a.c_in * a.c_out * a.n2p;
    if (!direct_pair_ok(a.c_in, a.c_out, a.n, a.n2p) || !w_host)
        return fail(SEGB_ERR_UNSUPPORTED, "paired direct kernel: unsupported layer");
    for (int64_t i = 0; i < nw; ++i) W.w[i] = w_host[i];
    if constexpr (sizeof(TX) == 4) {
        if (a.n == 3) return launch_direct_pair_tma_n3(a, W, st);
    }
    if (a.n == 4) return launch_direct_pair_cob<TX, 4>(a, W, st);
    return launch_direct_pair_cob<TX, 5>(a, W, st);
}

}  // namespace segb
