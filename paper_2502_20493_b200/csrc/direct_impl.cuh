// K2 -- the direct unified kernel (CUDA cores), templated on element types and
// the kernel side n.
//
// Spec: the per-element unified rule of the reference's instrumented engine,
// /root/reference/pkg/src/segconv/engines.py:379-406, summed over input
// channels as engines.py:163-172 (ascending ci, no bias):
//
//   r = (x + swap) & 1, s = (y + swap) & 1, p = P/2, swap = P & 1
//   out[b,co,x,y] = sum_ci sum_{u<R(r), v<R(s)} X[b,ci,(x+r)/2+u-p,(y+s)/2+v-p] * K[ci,co,2u+r,2v+s]
//
// One launch covers exactly the output elements; the parity is picked per
// output by construction (each thread owns whole parity "quads"), the upsampled
// map is never materialised and the floor(P/2) zero ring is implicit in the
// predicated loads. Odd output dims compute no stored extra elements.
//
// Work decomposition. Let x' = x + swap. A row quad q holds output rows
// x' in {2q, 2q+1} (r = 0 then r = 1); a column quad t holds y' in {2t, 2t+1}.
// For quad q, class r = 0 reads input rows q - swap - p + u (u < R0) and
// class r = 1 reads q + 1 - swap - p + u (u < R1): the union is
// NW = n/2 + 1 consecutive rows. A thread owns RQ row quads x 1 column quad x
// COB output channels (2RQ x 2 x COB outputs, all four parity classes), keeps
// the (RQ + NW - 1) x NW input window of one input channel in registers and
// reuses each loaded value for every tap and channel that needs it. Lanes of a
// warp own consecutive column quads, so loads are coalesced row segments and
// each warp store instruction covers 64 consecutive output columns.
// Weights (class-packed taps, K1 layout [co][ci][n2p]) are staged in shared
// memory per 16-input-channel chunk and read as broadcasts.
#pragma once

#include "common.cuh"

namespace segb {

struct DirectArgs {
    const void *x;
    void *y;
    const void *w;  // [c_out][c_in][n2p] compute type, class-packed taps
    int64_t batch, b0;  // b0: first sample of this launch (grid z chunking)
    int c_in, c_out, h, w_in, oh, ow, n, p, swap, n2p;
    int nqr, nqc;  // row / column quads
};

constexpr int kDirectCiChunk = 16;
constexpr int kDirectRowsPerBlock = 4;  // blockDim.y

template <typename TX, typename TC, bool RBF>
__device__ __forceinline__ TC load_x(const TX *p);
template <> __device__ __forceinline__ float load_x<float, float, false>(const float *p) { return __ldg(p); }
template <> __device__ __forceinline__ float load_x<float, float, true>(const float *p) {
    return round_bf16(__ldg(p));
}
template <> __device__ __forceinline__ float load_x<__nv_bfloat16, float, false>(const __nv_bfloat16 *p) {
    return __bfloat162float(*p);
}
template <> __device__ __forceinline__ double load_x<double, double, false>(const double *p) { return __ldg(p); }
// dataset images: the interleaved u8 PPM payload read in place, decoded on load
// exactly as the reference decodes it, float32(u8) / float32(255) with IEEE division
// (tensor_io.py:52), so the fused path computes on the very values parse_ppm produces
template <> __device__ __forceinline__ float load_x<uint8_t, float, false>(const uint8_t *p) {
    return __fdiv_rn((float)__ldg(p), 255.0f);
}

// Input addressing: NCHW for float inputs; a uint8_t input is the interleaved (B, H, W, C) image
// payload (channel stride 1, column stride C).
template <typename TX> struct XLayout {
    static constexpr bool HWC = sizeof(TX) == 1;
    __device__ __forceinline__ static int64_t chan(int64_t plane) { return HWC ? 1 : plane; }
};

template <typename TY, typename TC> __device__ __forceinline__ void store_y(TY *p, TC v);
template <> __device__ __forceinline__ void store_y<float, float>(float *p, float v) { *p = v; }
template <> __device__ __forceinline__ void store_y<double, double>(double *p, double v) { *p = v; }
template <> __device__ __forceinline__ void store_y<__nv_bfloat16, float>(__nv_bfloat16 *p, float v) {
    *p = __float2bfloat16_rn(v);
}

template <typename TY, typename TC> __device__ __forceinline__ TY cvt_y(TC v);
template <> __device__ __forceinline__ float cvt_y<float, float>(float v) { return v; }
template <> __device__ __forceinline__ double cvt_y<double, double>(double v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt_y<__nv_bfloat16, float>(float v) { return __float2bfloat16_rn(v); }

template <typename TY, typename TC> __device__ __forceinline__ void store_y2(TY *p, TC a, TC b);
template <> __device__ __forceinline__ void store_y2<float, float>(float *p, float a, float b) {
    *reinterpret_cast<float2 *>(p) = make_float2(a, b);
}
template <> __device__ __forceinline__ void store_y2<double, double>(double *p, double a, double b) {
    *reinterpret_cast<double2 *>(p) = make_double2(a, b);
}
template <> __device__ __forceinline__ void store_y2<__nv_bfloat16, float>(__nv_bfloat16 *p, float a, float b) {
    *reinterpret_cast<__nv_bfloat162 *>(p) = __floats2bfloat162_rn(a, b);
}

// vectorised broadcast read of one (co, ci) tap vector from shared memory
template <typename TC, int N2P> __device__ __forceinline__ void load_taps(const TC *wp, TC (&wv)[N2P]);
template <int N2P> __device__ __forceinline__ void load_taps_f(const float *wp, float (&wv)[N2P]) {
#pragma unroll
    for (int k = 0; k < N2P; k += 4) {
        const float4 v = *reinterpret_cast<const float4 *>(wp + k);
        wv[k] = v.x; wv[k + 1] = v.y; wv[k + 2] = v.z; wv[k + 3] = v.w;
    }
}
template <int N2P> __device__ __forceinline__ void load_taps_d(const double *wp, double (&wv)[N2P]) {
#pragma unroll
    for (int k = 0; k < N2P; k += 2) {
        const double2 v = *reinterpret_cast<const double2 *>(wp + k);
        wv[k] = v.x; wv[k + 1] = v.y;
    }
}
template <typename TC, int N2P> __device__ __forceinline__ void load_taps(const TC *wp, TC (&wv)[N2P]) {
    if constexpr (sizeof(TC) == 4) load_taps_f<N2P>(wp, wv);
    else load_taps_d<N2P>(wp, wv);
}

template <typename TX, typename TC, typename TY, bool RBF, int N, int COB, int RQ, int CQ>
// one or two output channels per thread (the dataset layers): at most 80 registers so six
// blocks fit per SM -- more warps to hide the window loads (ds512_k5 0.151 -> 0.141 ms); with
// three channels the register cap spills and loses
__global__ void __launch_bounds__(128, (COB <= 2 && sizeof(TC) == 4) ? 6 : 1) direct_kernel(DirectArgs a) {
    constexpr int NW = N / 2 + 1;          // input rows/cols under one output quad
    constexpr int WR = RQ + NW - 1;        // window rows for RQ row quads
    constexpr int WC = CQ + NW - 1;        // window cols for CQ column quads
    constexpr int R0 = (N + 1) / 2, R1 = N / 2;
    constexpr int OFF1 = R0 * R0, OFF2 = R0 * R0 + R0 * R1, OFF3 = R0 * R0 + 2 * R0 * R1;
    constexpr int N2P = (N * N + 3) / 4 * 4;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TC *ws = reinterpret_cast<TC *>(smem_raw);  // [COB][kDirectCiChunk][N2P]

    const int t0 = (blockIdx.x * 32 + threadIdx.x) * CQ;  // first column quad
    const int nrb = (a.nqr + kDirectRowsPerBlock * RQ - 1) / (kDirectRowsPerBlock * RQ);
    const int q0 = ((blockIdx.y % nrb) * kDirectRowsPerBlock + threadIdx.y) * RQ;
    const int co0 = (blockIdx.y / nrb) * COB;
    const int64_t b = a.b0 + blockIdx.z;
    const int row0 = q0 - a.swap - a.p, col0 = t0 - a.swap - a.p;
    const int64_t plane = (int64_t)a.h * a.w_in;
    const TX *xb = reinterpret_cast<const TX *>(a.x) + b * a.c_in * plane;
    const TC *wsrc = reinterpret_cast<const TC *>(a.w);
    const int tid = threadIdx.y * 32 + threadIdx.x;
    constexpr bool HWC = XLayout<TX>::HWC;
    const int es = HWC ? a.c_in : 1;                  // column (element) stride
    const int64_t rs = (int64_t)a.w_in * es;          // row stride
    const int64_t cs = XLayout<TX>::chan(plane);      // channel stride

    TC acc[COB][2 * RQ][2 * CQ];
#pragma unroll
    for (int c = 0; c < COB; ++c)
#pragma unroll
        for (int i = 0; i < 2 * RQ; ++i)
#pragma unroll
            for (int k = 0; k < 2 * CQ; ++k) acc[c][i][k] = TC(0);

    // interior warps (the whole window of every lane inside the input) load unpredicated
    const bool inside = row0 >= 0 && row0 + WR <= a.h && col0 >= 0 && col0 + WC <= a.w_in;
    const bool warp_inside = __all_sync(0xffffffffu, inside);
    bool rok[WR], cok[WC];
#pragma unroll
    for (int i = 0; i < WR; ++i) rok[i] = (unsigned)(row0 + i) < (unsigned)a.h;
#pragma unroll
    for (int j = 0; j < WC; ++j) cok[j] = (unsigned)(col0 + j) < (unsigned)a.w_in;
    const TX *xw = xb + (int64_t)row0 * rs + (int64_t)col0 * es;  // window origin of channel 0 (may point outside)

    auto load_win = [&](TC (&dst)[WR][WC], int ci_abs) {
        const TX *xc = xw + (int64_t)ci_abs * cs;
        if (warp_inside) {  // one row pointer per window row, immediate column offsets (NCHW)
#pragma unroll
            for (int i = 0; i < WR; ++i) {
                const TX *rp = xc + i * rs;
#pragma unroll
                for (int j = 0; j < WC; ++j) dst[i][j] = load_x<TX, TC, RBF>(rp + j * es);
            }
        } else {
#pragma unroll
            for (int i = 0; i < WR; ++i) {
                const TX *rp = xc + i * rs;
#pragma unroll
                for (int j = 0; j < WC; ++j)
                    dst[i][j] = (rok[i] && cok[j]) ? load_x<TX, TC, RBF>(rp + j * es) : TC(0);
            }
        }
    };
    auto compute = [&](const TC (&win)[WR][WC], int ci) {
#pragma unroll
        for (int c = 0; c < COB; ++c) {
            const TC *wp = ws + (c * kDirectCiChunk + ci) * N2P;
            TC wv[N2P];
            load_taps<TC, N2P>(wp, wv);  // 128-bit shared-memory broadcasts
#pragma unroll
            for (int qq = 0; qq < RQ; ++qq)
#pragma unroll
                for (int cq = 0; cq < CQ; ++cq) {
#pragma unroll
                    for (int u = 0; u < R0; ++u) {
#pragma unroll
                        for (int v = 0; v < R0; ++v)
                            acc[c][2 * qq][2 * cq] += win[qq + u][cq + v] * wv[u * R0 + v];
#pragma unroll
                        for (int v = 0; v < R1; ++v)
                            acc[c][2 * qq][2 * cq + 1] += win[qq + u][cq + 1 + v] * wv[OFF1 + u * R1 + v];
                    }
#pragma unroll
                    for (int u = 0; u < R1; ++u) {
#pragma unroll
                        for (int v = 0; v < R0; ++v)
                            acc[c][2 * qq + 1][2 * cq] += win[qq + 1 + u][cq + v] * wv[OFF2 + u * R0 + v];
#pragma unroll
                        for (int v = 0; v < R1; ++v)
                            acc[c][2 * qq + 1][2 * cq + 1] += win[qq + 1 + u][cq + 1 + v] * wv[OFF3 + u * R1 + v];
                    }
                }
        }
    };

    // Software pipeline over input channels with two window buffers used alternately (no
    // register copies): the next channel's window loads are in flight while the current one
    // is multiplied, and the first window of a weight chunk is loaded before the chunk's
    // weights are staged.
    // Pipelined only with three or more output channels per thread (enough arithmetic per
    // window to cover a load); with fewer the second window's registers cost more occupancy
    // than the overlap gains (measured on the dataset layers).
    constexpr bool PIPE = COB >= 3;
    TC wa[WR][WC], wb[WR][WC];
    for (int ci0 = 0; ci0 < a.c_in; ci0 += kDirectCiChunk) {
        const int nci = min(kDirectCiChunk, a.c_in - ci0);
        if (PIPE) load_win(wa, ci0);
        __syncthreads();
        for (int i = tid; i < COB * nci * N2P; i += 32 * kDirectRowsPerBlock) {
            const int co = i / (nci * N2P);
            const int rem = i - co * nci * N2P;
            const int ci = rem / N2P;
            const int k = rem - ci * N2P;
            ws[(co * kDirectCiChunk + ci) * N2P + k] =
                (co0 + co < a.c_out) ? wsrc[((int64_t)(co0 + co) * a.c_in + ci0 + ci) * N2P + k] : TC(0);
        }
        __syncthreads();
        if constexpr (PIPE) {
            for (int ci = 0; ci < nci; ci += 2) {
                if (ci + 1 < nci) load_win(wb, ci0 + ci + 1);
                compute(wa, ci);
                if (ci + 1 >= nci) break;
                if (ci + 2 < nci) load_win(wa, ci0 + ci + 2);
                compute(wb, ci + 1);
            }
        } else {
#pragma unroll 2
            for (int ci = 0; ci < nci; ++ci) {
                load_win(wa, ci0 + ci);
                compute(wa, ci);
            }
        }
    }

    // Stores, staged per warp through shared memory so each warp store instruction writes 32
    // consecutive outputs of one row (a thread's 2*CQ columns are adjacent, which would
    // otherwise spread one instruction over 16 sectors). Every output element is written
    // exactly once; quad positions outside [0, oh) x [0, ow) (odd dims, the swap shift) are
    // not stored.
    constexpr int SC = 64 * CQ;  // staged columns per warp row
    __syncthreads();             // the weight chunk area is reused for staging
    TY *stg = reinterpret_cast<TY *>(smem_raw) + threadIdx.y * (COB * 2 * RQ * SC);
#pragma unroll
    for (int c = 0; c < COB; ++c)
#pragma unroll
        for (int i = 0; i < 2 * RQ; ++i)
#pragma unroll
            for (int k = 0; k < 2 * CQ; ++k)
                stg[(c * 2 * RQ + i) * SC + threadIdx.x * 2 * CQ + k] = cvt_y<TY, TC>(acc[c][i][k]);
    __syncwarp();
    TY *yb = reinterpret_cast<TY *>(a.y);
    const int y0 = 2 * (blockIdx.x * 32 * CQ) - a.swap;  // first output column of the warp
#pragma unroll
    for (int c = 0; c < COB; ++c) {
        if (co0 + c >= a.c_out) break;
        TY *yc = yb + ((int64_t)b * a.c_out + co0 + c) * a.oh * a.ow;
#pragma unroll
        for (int i = 0; i < 2 * RQ; ++i) {
            const int xo = 2 * q0 + i - a.swap;
            if ((unsigned)xo >= (unsigned)a.oh) continue;
            TY *row = yc + (int64_t)xo * a.ow;
#pragma unroll
            for (int m = 0; m < 2 * CQ; ++m) {
                const int col = m * 32 + threadIdx.x;
                const int yo = y0 + col;
                if ((unsigned)yo < (unsigned)a.ow) row[yo] = stg[(c * 2 * RQ + i) * SC + col];
            }
        }
    }
}

// Generic-n fallback (n > 9): one thread per output element, runtime loops.
template <typename TX, typename TC, typename TY, bool RBF>
__global__ void __launch_bounds__(256) direct_generic_kernel(DirectArgs a) {
    const int64_t total = a.batch * a.c_out * (int64_t)a.oh * a.ow;
    const int64_t plane = (int64_t)a.h * a.w_in;
    const TC *wsrc = reinterpret_cast<const TC *>(a.w);
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int yo = idx % a.ow;
        const int xo = (idx / a.ow) % a.oh;
        const int co = (idx / ((int64_t)a.ow * a.oh)) % a.c_out;
        const int64_t b = idx / ((int64_t)a.ow * a.oh * a.c_out);
        const int r = (xo + a.swap) & 1, s = (yo + a.swap) & 1;
        const int bx = (xo + r) / 2 - a.p, by = (yo + s) / 2 - a.p;
        const int R = sub_len(a.n, r), C = sub_len(a.n, s), off = class_offset(a.n, 2 * r + s);
        TC acc = 0;
        constexpr bool HWC = XLayout<TX>::HWC;
        const int es = HWC ? a.c_in : 1;
        for (int ci = 0; ci < a.c_in; ++ci) {
            const TX *xc = reinterpret_cast<const TX *>(a.x) + b * a.c_in * plane + ci * XLayout<TX>::chan(plane);
            const TC *wp = wsrc + ((int64_t)co * a.c_in + ci) * a.n2p + off;
            for (int u = 0; u < R; ++u) {
                const int ii = bx + u;
                if ((unsigned)ii >= (unsigned)a.h) continue;
                for (int v = 0; v < C; ++v) {
                    const int jj = by + v;
                    if ((unsigned)jj >= (unsigned)a.w_in) continue;
                    acc += load_x<TX, TC, RBF>(xc + ((int64_t)ii * a.w_in + jj) * es) * wp[u * C + v];
                }
            }
        }
        store_y<TY, TC>(reinterpret_cast<TY *>(a.y) + idx, acc);
    }
}

// The reference engine (Alg. 1, engines.py:134-140 / 258-269) on the device:
// correlation of the zero-padded bed-of-nails map with the full n x n kernel,
// evaluated without materialising the map (zero taps are still multiplied, as
// the reference does). Weights: the raw bank in compute type, [co][ci][n*n].
template <typename TX, typename TC, typename TY, bool RBF>
__global__ void __launch_bounds__(256) reference_engine_kernel(DirectArgs a, int pad) {
    const int64_t total = a.batch * a.c_out * (int64_t)a.oh * a.ow;
    const int64_t plane = (int64_t)a.h * a.w_in;
    const TC *wsrc = reinterpret_cast<const TC *>(a.w);
    const int n = a.n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int yo = idx % a.ow;
        const int xo = (idx / a.ow) % a.oh;
        const int co = (idx / ((int64_t)a.ow * a.oh)) % a.c_out;
        const int64_t b = idx / ((int64_t)a.ow * a.oh * a.c_out);
        TC acc = 0;
        constexpr bool HWC = XLayout<TX>::HWC;
        const int es = HWC ? a.c_in : 1;
        for (int ci = 0; ci < a.c_in; ++ci) {
            const TX *xc = reinterpret_cast<const TX *>(a.x) + b * a.c_in * plane + ci * XLayout<TX>::chan(plane);
            const TC *wp = wsrc + ((int64_t)co * a.c_in + ci) * a.n2p;
            for (int u = 0; u < n; ++u) {
                const int uu = xo + u - pad;  // index into the un-padded upsampled map
                const bool rlive = uu >= 0 && (uu & 1) == 0 && (uu >> 1) < a.h;
                for (int v = 0; v < n; ++v) {
                    const int vv = yo + v - pad;
                    const bool live = rlive && vv >= 0 && (vv & 1) == 0 && (vv >> 1) < a.w_in;
                    const TC val =
                        live ? load_x<TX, TC, RBF>(xc + ((int64_t)(uu >> 1) * a.w_in + (vv >> 1)) * es) : TC(0);
                    acc += val * wp[u * n + v];
                }
            }
        }
        store_y<TY, TC>(reinterpret_cast<TY *>(a.y) + idx, acc);
    }
}

template <typename TX, typename TC, typename TY, bool RBF, int N, int COB>
int launch_direct_n(const DirectArgs &a, cudaStream_t st) {
#ifndef SEGB_DIRECT_RQ
#define SEGB_DIRECT_RQ 0
#endif
#ifndef SEGB_DIRECT_CQ
#define SEGB_DIRECT_CQ 0
#endif
    // row / column quads per thread (SEGB_DIRECT_RQ / _CQ override them for A/B builds)
    constexpr int RQ = SEGB_DIRECT_RQ > 0 ? SEGB_DIRECT_RQ : ((N <= 5) ? 4 : 2);
    constexpr int CQ = SEGB_DIRECT_CQ > 0 ? SEGB_DIRECT_CQ : ((N <= 5 && COB <= 2 && sizeof(TC) == 4) ? 2 : 1);
    dim3 block(32, kDirectRowsPerBlock);
    const int64_t nco_blk = ceil_div(a.c_out, COB);
    const int64_t nrb = ceil_div(a.nqr, kDirectRowsPerBlock * RQ);
    if (nco_blk * nrb > 65535 || ceil_div(a.nqc, 32 * CQ) > (1ll << 31) - 1)
        return fail(SEGB_ERR_UNSUPPORTED, "output too large for the direct kernel grid");
    const size_t smem = std::max(sizeof(TC) * COB * kDirectCiChunk * a.n2p,
                                 sizeof(TY) * kDirectRowsPerBlock * COB * 2 * RQ * 64 * CQ);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(direct_kernel<TX, TC, TY, RBF, N, COB, RQ, CQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    for (int64_t b0 = 0; b0 < a.batch; b0 += 65535) {
        DirectArgs c = a;
        c.b0 = b0;
        dim3 grid((unsigned)ceil_div(a.nqc, 32 * CQ), (unsigned)(nco_blk * nrb),
                  (unsigned)std::min<int64_t>(65535, a.batch - b0));
        direct_kernel<TX, TC, TY, RBF, N, COB, RQ, CQ><<<grid, block, smem, st>>>(c);
        note_launch();
        if (int rc = check_launch("direct_kernel")) return rc;
    }
    return SEGB_OK;
}

template <typename TX, typename TC, typename TY, bool RBF, int N>
int launch_direct_cob(const DirectArgs &a, cudaStream_t st) {
    if (a.c_out == 1) return launch_direct_n<TX, TC, TY, RBF, N, 1>(a, st);
    if (a.c_out == 2) return launch_direct_n<TX, TC, TY, RBF, N, 2>(a, st);
    if (a.c_out == 3) return launch_direct_n<TX, TC, TY, RBF, N, 3>(a, st);
    return launch_direct_n<TX, TC, TY, RBF, N, 4>(a, st);
}

template <typename TX, typename TC, typename TY, bool RBF>
int launch_direct_typed(const DirectArgs &a, bool reference_engine, cudaStream_t st) {
    const int64_t total = a.batch * a.c_out * (int64_t)a.oh * a.ow;
    if (reference_engine) {
        const int threads = 256;
        const int64_t blocks = std::min<int64_t>(ceil_div(total, threads), 148 * 64);
        reference_engine_kernel<TX, TC, TY, RBF><<<(unsigned)blocks, threads, 0, st>>>(a, a.p);
        note_launch();
        return check_launch("reference_engine_kernel");
    }
    switch (a.n) {
        case 2: return launch_direct_cob<TX, TC, TY, RBF, 2>(a, st);
        case 3: return launch_direct_cob<TX, TC, TY, RBF, 3>(a, st);
        case 4: return launch_direct_cob<TX, TC, TY, RBF, 4>(a, st);
        case 5: return launch_direct_cob<TX, TC, TY, RBF, 5>(a, st);
        case 6: return launch_direct_cob<TX, TC, TY, RBF, 6>(a, st);
        case 7: return launch_direct_cob<TX, TC, TY, RBF, 7>(a, st);
        case 8: return launch_direct_cob<TX, TC, TY, RBF, 8>(a, st);
        case 9: return launch_direct_cob<TX, TC, TY, RBF, 9>(a, st);
        default: {
            const int threads = 256;
            const int64_t blocks = std::min<int64_t>(ceil_div(total, threads), 148 * 64);
            direct_generic_kernel<TX, TC, TY, RBF><<<(unsigned)blocks, threads, 0, st>>>(a);
            note_launch();
            return check_launch("direct_generic_kernel");
        }
    }
}

// per-dtype-combination entry points (defined in direct_*.cu)
int launch_direct_f32(const DirectArgs &a, bool ref_engine, cudaStream_t st);
int launch_direct_f64(const DirectArgs &a, bool ref_engine, cudaStream_t st);
// bf16 compute: x in {f32 (rounded on load), bf16}, y in {f32, bf16}
int launch_direct_bf16(const DirectArgs &a, int x_dtype, int y_dtype, bool ref_engine, cudaStream_t st);
// fp32 compute on the interleaved u8 image payload (x: (B, H, W, C), decoded on load)
int launch_direct_u8(const DirectArgs &a, bool ref_engine, cudaStream_t st);

// K2p, the paired FFMA2 kernel for low-channel layers (direct_pair.cuh): whether it takes a
// segregated fp32 layer, and its launchers (x f32 / u8 image; w_host = the K2 weights
// [c_out][c_in][n2p] on the host, passed as a kernel parameter)
constexpr int kPairWMax = 896;
inline bool direct_pair_ok(int c_in, int c_out, int n, int n2p) {
    // n <= 3: K2's one-sample 8 x 4 tiles load fewer window values per output and win (ds224_k3
    // 0.025 vs 0.028 ms); n 4, 5: K2p (ds512_k5 0.150 -> 0.129 ms, ds512_k4_c3 0.351 -> 0.298)
    // (n = 3: only its TMA-staged variant, see direct_pair_n_ok)
    return c_out >= 1 && c_out <= 3 && n >= 3 && n <= 5 && (int64_t)c_in * c_out * n2p <= kPairWMax;
}
int launch_direct_pair_f32(const DirectArgs &a, const float *w_host, cudaStream_t st);
// fp32 x with W % 4 == 0 runs K2p with TMA-staged input tiles unless SEGB200_DIRECT_PAIR_TMA=0
inline bool direct_pair_tma_enabled() {
    const char *e = getenv("SEGB200_DIRECT_PAIR_TMA");
    return !(e && !atoi(e));
}
// K2p with the weights in shared memory (TMA-staged input; the layer's K2 weights a.w): fp32 x,
// W % 4 == 0, c_out <= 3, n 3..5, more weights than the kernel parameter holds, <= 12 K floats
inline bool direct_pair_wsm_ok(int c_in, int c_out, int n, int n2p, int in_w) {
    const int64_t nw = (int64_t)c_in * c_out * n2p;
    return c_out >= 1 && c_out <= 3 && n >= 3 && n <= 5 && nw > kPairWMax && nw <= 12288 && in_w % 4 == 0 &&
           direct_pair_tma_enabled();
}
int launch_direct_pair_wsm(const DirectArgs &a, cudaStream_t st);
// per call: n = 3 only on the TMA-staged variant (the register-window K2p loses to K2 there)
inline bool direct_pair_n_ok(int n, bool f32_x, int in_w) {
    return n >= 4 || (f32_x && in_w % 4 == 0 && direct_pair_tma_enabled());
}
int launch_direct_pair_u8(const DirectArgs &a, const float *w_host, cudaStream_t st);

}  // namespace segb
