// K3c -- input-stationary ("scatter") implicit GEMM for narrow outputs, e.g. DCGAN l5
// (32x32x128 -> 64x64x3, n = 4): c_out * n^2 <= 256 and c_out much smaller than c_in.
//
// The output-stationary GEMMs of K3/K3b read every input element once per tap of every
// parity class (n^2 times) to produce c_out columns; with c_out = 3 that is mostly operand
// traffic. Here each input position is read ONCE and multiplied by all n^2 taps at once:
//
//   Z[b, (kx, ky, co), i, j] = sum_ci X[b, ci, i, j] * K[ci, co, kx, ky]
//
// a single dense GEMM (M = positions, K = c_in, N = n^2 c_out) on tcgen05 with the A
// operand TMA-loaded straight from NCHW as an MN-major SWIZZLE_128B tile (no NHWC copy;
// descriptor LBO = 8 KB between the two 64-position atoms, SBO = 1 KB between 8-channel
// atoms, measured by tools/probes/mn_major_probe.cu). A gather kernel then applies the
// unified rule backwards: output (x, y) of parity class (r, s), r = (x + swap) & 1, sums
// Z[(2u + r, 2v + s), (x + r) / 2 + u - p, (y + s) / 2 + v - p] over the class's taps --
// exactly the terms of engines.py:391-404, with out-of-range input rows
// and columns (the floor(P/2) zero ring) contributing nothing. Z is fp32, so the only
// rounding beyond fp32 accumulation is the final cast of the output.
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "igemm.cuh"
#include "tc_ptx.cuh"

namespace segb {

namespace {

constexpr int kScThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kScStages = 6;     // A ring: 64 channels x 128 positions (16 KB) per stage

struct ScatterParams {
    int64_t positions;  // batch * h * w
    int hw, c_in, n_real, n_pad, kb, total_tiles;
    float *z;           // [batch][n_real][hw] fp32
};

__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)(8192 >> 4) << 16;  // LBO: next 64-position atom (second TMA box)
    d |= (uint64_t)(1024 >> 4) << 32;  // SBO: next 8-channel atom
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}

__global__ void __launch_bounds__(kScThreads, 1)
    scatter_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const ScatterParams prm) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int NP = prm.n_pad, KB = prm.kb;
    uint8_t *sB = smem;                                 // [kb][NP rows x 128 B], K-major SW128
    uint8_t *sA = smem + (size_t)KB * NP * 128;         // [stage][2 boxes x 8 KB]
    sA = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sA) + 1023) & ~uintptr_t(1023));
    uint64_t *bars = reinterpret_cast<uint64_t *>(sA + kScStages * 16384);
    uint64_t *b_full = bars, *full = bars + 1, *empty = full + kScStages, *tfull = empty + kScStages,
             *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    if (threadIdx.x == 0) {
        mbar_init(b_full, 1);
        for (int i = 0; i < kScStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    }
    const uint32_t tcols = tmem_pow2(2 * NP);
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            mbar_expect_tx(b_full, KB * NP * 128);
            for (int kb = 0; kb < KB; ++kb) tma_load_3d(sB + (size_t)kb * NP * 128, &tmB, b_full, kb * 64, 0, 0);
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < prm.total_tiles; t += gridDim.x) {
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], 16384);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        // 64 positions of one image (hw % 64 == 0); past the batch the box
                        // lies wholly outside the tensor and is zero-filled
                        const int64_t g = (int64_t)t * 128 + h * 64;
                        const int b = (int)(g / prm.hw), pos = (int)(g % prm.hw);
                        tma_load_3d(sA + stage * 16384 + h * 8192, &tmA, &full[stage], pos, kb * 64, b);
                    }
                    if (++stage == kScStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {  // ---------------- MMA issuer
        mbar_wait(b_full, 0);
        const uint32_t idesc = idesc_bf16_m(128, NP) | (1u << 15);  // A MN-major, B K-major
        const uint32_t leader = elect_one();
        int stage = 0, acc = 0;
        uint32_t phase = 0, acc_phase = 0;
        for (int t = blockIdx.x; t < prm.total_tiles; t += gridDim.x) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d = tmem_base + acc * NP;
            for (int kb = 0; kb < KB; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint32_t a0 = smem_u32(sA + stage * 16384), b0 = smem_u32(sB + (size_t)kb * NP * 128);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)  // 16 channels per MMA: two 8-channel atoms of A, 32 B of B
                    tc_mma_pred(d, desc_mn_sw128(a0 + kk * 2048), desc_k_sw128(b0 + kk * 32), idesc,
                                (kb | kk) != 0, leader);
                if (leader) tc_commit(&empty[stage]);
                __syncwarp();
                if (++stage == kScStages) { stage = 0; phase ^= 1; }
            }
            if (leader) tc_commit(&tfull[acc]);
            __syncwarp();
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    } else {  // ---------------- epilogue: TMEM lane quarter -> Z planes, 128 B per warp store
        const int q = warp & 3;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < prm.total_tiles; t += gridDim.x) {
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int64_t g = (int64_t)t * 128 + q * 32 + lane;
            const bool ok = g < prm.positions;
            const int64_t b = g / prm.hw, pos = g % prm.hw;
            float *zp = prm.z + b * prm.n_real * (int64_t)prm.hw + pos;
            const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16) + acc * NP;
            for (int c0 = 0; c0 < prm.n_real; c0 += 16) {
                uint32_t v[16];
                tmem_ld16(tl + c0, v);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (ok && c0 + j < prm.n_real) zp[(int64_t)(c0 + j) * prm.hw] = __uint_as_float(v[j]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tcols));
    }
}

__device__ __forceinline__ void store_pair(__nv_bfloat16 *p, float a, float b) {
    *reinterpret_cast<__nv_bfloat162 *>(p) = __floats2bfloat162_rn(a, b);
}
__device__ __forceinline__ void store_pair(float *p, float a, float b) {
    *reinterpret_cast<float2 *>(p) = make_float2(a, b);
}

constexpr int kGatherRows = 16;  // output rows per gather block

// Unified rule read backwards over Z. Block (32 x 4 threads) = 16 output rows x 64 columns of
// one (image, output channel) plane, thread = one column pair (2c, 2c + 1), i.e. one column
// of each parity s; no integer division. Classes are picked at run time from the output
// coordinates (r = (x + swap) & 1, s = (y + swap) & 1); the loads of a warp are contiguous
// along j for every (tap, s).
template <typename TY, int NK>
__global__ void __launch_bounds__(128) scatter_gather_kernel(const float *__restrict__ z, TY *__restrict__ y,
                                                             int c_out, int h, int w, int oh, int ow, int n_rt, int p,
                                                             int swap) {
    const int n = NK ? NK : n_rt;  // kernel side, compile-time for the common sizes
    const int plane = blockIdx.x;  // b * c_out + co
    const int co = plane % c_out;
    const int64_t b = plane / c_out;
    const int hw = h * w;
    const float *zb = z + b * ((int64_t)n * n * c_out) * hw + (int64_t)co * hw;  // offsets below fit in int32
    const int tap_stride = c_out * hw;
    const int y0 = (blockIdx.z * 32 + threadIdx.x) * 2;
    // column terms of the two outputs (parities s = (y + swap) & 1), hoisted out of the row loop
    int joff[2][(NK ? NK : 8) / 2 + 1];
    int nv[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int yy = y0 + e;
        const int s = (yy + swap) & 1, j0 = (yy + s) / 2 - p;
        nv[e] = 0;
#pragma unroll
        for (int v = 0; v < (NK ? NK : 8) / 2 + 1; ++v) {
            joff[e][v] = -1;
            const int j = j0 + v;
            if (2 * v + s < n && j >= 0 && j < w && yy < ow) joff[e][v] = (2 * v + s) * tap_stride + j;
        }
    }
    for (int xx = blockIdx.y * kGatherRows + threadIdx.y; xx < min(oh, (int)(blockIdx.y + 1) * kGatherRows); xx += 4) {
        const int r = (xx + swap) & 1, i0 = (xx + r) / 2 - p;
        float out[2] = {0.f, 0.f};
#pragma unroll
        for (int u = 0; u < (NK ? NK : 8) / 2 + 1; ++u) {
            const int i = i0 + u;
            if (2 * u + r >= n || i < 0 || i >= h) continue;
            const float *zr = zb + (2 * u + r) * n * tap_stride + i * w;
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int v = 0; v < (NK ? NK : 8) / 2 + 1; ++v)
                    if (joff[e][v] >= 0) out[e] += __ldg(zr + joff[e][v]);
        }
        TY *row = y + ((int64_t)plane * oh + xx) * ow;
        if (y0 + 1 < ow && (ow & 1) == 0) {  // one 2-element store (row starts stay aligned)
            store_pair(row + y0, out[0], out[1]);
        } else {
            if (y0 < ow) row[y0] = from_float<TY>(out[0]);
            if (y0 + 1 < ow) row[y0 + 1] = from_float<TY>(out[1]);
        }
    }
}

template <typename TY>
static void launch_gather(dim3 grd, cudaStream_t st, const float *z, TY *y, int c_out, int h, int w, int oh, int ow,
                          int n, int p, int swap) {
    dim3 blk(32, 4);
    switch (n) {
        case 2: scatter_gather_kernel<TY, 2><<<grd, blk, 0, st>>>(z, y, c_out, h, w, oh, ow, n, p, swap); break;
        case 3: scatter_gather_kernel<TY, 3><<<grd, blk, 0, st>>>(z, y, c_out, h, w, oh, ow, n, p, swap); break;
        case 4: scatter_gather_kernel<TY, 4><<<grd, blk, 0, st>>>(z, y, c_out, h, w, oh, ow, n, p, swap); break;
        case 5: scatter_gather_kernel<TY, 5><<<grd, blk, 0, st>>>(z, y, c_out, h, w, oh, ow, n, p, swap); break;
        case 6: scatter_gather_kernel<TY, 6><<<grd, blk, 0, st>>>(z, y, c_out, h, w, oh, ow, n, p, swap); break;
        default: scatter_gather_kernel<TY, 0><<<grd, blk, 0, st>>>(z, y, c_out, h, w, oh, ow, n, p, swap); break;
    }
}

// weights for K3c: bf16 [n_pad rows = (kx, ky, co)][c_in_pad (64-multiple)] K-major, zero-padded
template <typename TB>
__global__ void prep_scatter_kernel(const TB *__restrict__ bank, __nv_bfloat16 *__restrict__ dst, int c_in,
                                    int c_in_pad, int c_out, int n, int n_pad) {
    const int64_t total = (int64_t)n_pad * c_in_pad;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int ci = (int)(idx % c_in_pad), row = (int)(idx / c_in_pad);
        float v = 0.f;
        if (ci < c_in && row < n * n * c_out) {
            const int co = row % c_out, tap = row / c_out, kx = tap / n, ky = tap % n;
            v = (float)bank[(((int64_t)ci * c_out + co) * n + kx) * n + ky];
        }
        dst[idx] = __float2bfloat16_rn(v);
    }
}

bool scatter_params(const IgemmShape &s, ScatterParams &prm) {
    if (s.compute != SEGB_BF16 || s.x_dtype != SEGB_BF16) return false;
    if (s.y_dtype != SEGB_BF16 && s.y_dtype != SEGB_F32) return false;
    const int64_t hw = (int64_t)s.h * s.w;
    if (hw % 64 != 0 || hw > INT32_MAX) return false;
    if (s.c_in < 64 || s.c_in > 256) return false;  // whole-tile TMA boxes; B resident for <= 4 blocks
    const int nreal = s.n * s.n * s.c_out;
    if (nreal > 256 || s.n > 8) return false;
    if ((int64_t)nreal * hw > INT32_MAX) return false;  // gather offsets within an image are int32
    // reading the input once instead of n^2 times pays while Z (4 n^2 c_out B per position,
    // written then read back) stays well below the input's n^2 re-reads (2 n^2 c_in B)
    if (4 * s.c_out > s.c_in) return false;
    prm.positions = s.batch * hw;
    const int64_t tiles = ceil_div(prm.positions, 128);
    if (tiles > INT32_MAX) return false;
    // small batches (few 128-position tiles): the output-stationary K3 with split K is faster
    // (dcgan_l5 bf16 at batch 1: 18.4 -> 16.4 us; at batch 16 K3c wins, 18.9 vs 22.5).
    // SEGB200_K3C_MIN_TILES overrides (tests run K3c at small shapes with 0).
    int64_t min_tiles = 64;
    if (const char *mt = getenv("SEGB200_K3C_MIN_TILES")) min_tiles = atoll(mt);
    if (tiles < min_tiles) return false;
    prm.hw = (int)hw;
    prm.c_in = s.c_in;
    prm.n_real = nreal;
    prm.n_pad = (nreal + 15) / 16 * 16;
    prm.kb = (s.c_in + 63) / 64;
    prm.total_tiles = (int)tiles;
    return true;
}

}  // namespace

bool igemm_scatter_supported(const IgemmShape &s) {
    ScatterParams prm;
    const char *e = getenv("SEGB200_IGEMM_NOSCATTER");  // A/B switch: route to K3/K3b instead
    return !(e && atoi(e)) && scatter_params(s, prm) && tensor_map_encoder() != nullptr;
}

int scatter_weight_rows(int c_out, int n) { return (n * n * c_out + 15) / 16 * 16; }

int run_prep_scatter(const void *bank, int bank_dtype, int c_in, int c_in_pad, int c_out, int n, void *dst,
                     cudaStream_t st) {
    const int n_pad = scatter_weight_rows(c_out, n);
    const int64_t total = (int64_t)n_pad * c_in_pad;
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 32);
    __nv_bfloat16 *d = (__nv_bfloat16 *)dst;
    switch (bank_dtype) {
        case SEGB_F32: prep_scatter_kernel<float><<<g, 256, 0, st>>>((const float *)bank, d, c_in, c_in_pad, c_out, n, n_pad); break;
        case SEGB_F64: prep_scatter_kernel<double><<<g, 256, 0, st>>>((const double *)bank, d, c_in, c_in_pad, c_out, n, n_pad); break;
        case SEGB_BF16: prep_scatter_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16 *)bank, d, c_in, c_in_pad, c_out, n, n_pad); break;
        default: return fail(SEGB_ERR_VALUE, "unknown bank dtype %d", bank_dtype);
    }
    note_launch();
    return check_launch("prep_scatter_kernel");
}

int64_t igemm_scatter_workspace_bytes(const IgemmShape &s) {
    ScatterParams prm;
    if (!scatter_params(s, prm)) return 0;
    return (prm.positions * prm.n_real * 4 + 255) / 256 * 256;
}

int run_igemm_scatter(const IgemmShape &s, const void *x, const void *wz, void *y, void *ws, int64_t ws_bytes,
                      cudaStream_t st) {
    ScatterParams prm;
    if (!scatter_params(s, prm)) return fail(SEGB_ERR_UNSUPPORTED, "scatter implicit GEMM: unsupported shape");
    auto encode = tensor_map_encoder();
    if (!encode) return fail(SEGB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int c_in_pad = prm.kb * 64;
    CUtensorMap tmA, tmB;
    cuuint32_t es[3] = {1, 1, 1};
    {
        cuuint64_t dims[3] = {(cuuint64_t)prm.hw, (cuuint64_t)s.c_in, (cuuint64_t)s.batch};
        cuuint64_t strides[2] = {(cuuint64_t)prm.hw * 2, (cuuint64_t)s.c_in * prm.hw * 2};
        cuuint32_t box[3] = {64, 64, 1};
        CUresult r = encode(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(x), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SEGB_ERR_CUDA, "tensor map (scatter A): error %d", (int)r);
    }
    {
        cuuint64_t dims[3] = {(cuuint64_t)c_in_pad, (cuuint64_t)prm.n_pad, 1};
        cuuint64_t strides[2] = {(cuuint64_t)c_in_pad * 2, (cuuint64_t)prm.n_pad * c_in_pad * 2};
        cuuint32_t box[3] = {64, (cuuint32_t)prm.n_pad, 1};
        CUresult r = encode(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(wz), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SEGB_ERR_CUDA, "tensor map (scatter B): error %d", (int)r);
    }
    const int64_t zbytes = prm.positions * prm.n_real * 4;
    if (!ws || ws_bytes < zbytes)
        return fail(SEGB_ERR_VALUE, "scatter implicit GEMM: workspace of %lld bytes needed, got %lld",
                    (long long)zbytes, (long long)ws_bytes);
    prm.z = (float *)ws;  // the tap products Z, in the caller's workspace
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = 1024 + ((size_t)prm.kb * prm.n_pad * 128 + 1023) / 1024 * 1024 + kScStages * 16384 +
                        (1 + 2 * kScStages + 4) * 8 + 16;
    const unsigned grid = (unsigned)std::min<int64_t>(prm.total_tiles, sms);
    cudaFuncSetAttribute(scatter_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    scatter_gemm_kernel<<<grid, kScThreads, smem, st>>>(tmA, tmB, prm);
    note_launch();
    int rc = check_launch("scatter_gemm_kernel");
    if (!rc) {
        const int oh = 2 * s.h + 2 * s.pad - s.n, ow = 2 * s.w + 2 * s.pad - s.n;
        const int64_t planes = s.batch * (int64_t)s.c_out;
        dim3 grd((unsigned)planes, (unsigned)ceil_div(oh, kGatherRows), (unsigned)ceil_div(ow, 64));
        if (s.y_dtype == SEGB_BF16)
            launch_gather(grd, st, prm.z, (__nv_bfloat16 *)y, s.c_out, s.h, s.w, oh, ow, s.n, s.pad / 2, s.pad & 1);
        else
            launch_gather(grd, st, prm.z, (float *)y, s.c_out, s.h, s.w, oh, ow, s.n, s.pad / 2, s.pad & 1);
        note_launch();
        rc = check_launch("scatter_gather_kernel");
    }
    return rc;
}

}  // namespace segb
