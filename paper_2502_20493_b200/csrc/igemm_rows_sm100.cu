// K3b -- row-streaming implicit GEMM for wide class grids (cols % 128 == 0),
// e.g. EB-GAN l7 (128x128x64 -> 256x256x64): all four parity classes of one
// class-grid row (128 positions) per tile, weights resident, input rows loaded
// once.
//
// Same arithmetic as K3 (igemm_sm100.cu, per-class GEMMs of engines.py:271-335)
// but the operand traffic is restructured for layers whose K = taps x c_in is
// small and whose output is large, where K3's per-tap TMA boxes re-read every
// input element n*n times from L2 and the weights once per tile:
//   * weights: every (class, tap, 64-channel block) B tile is TMA-loaded once
//     per CTA and stays resident in shared memory;
//   * activations: NCHW rows are TMA-loaded raw (box {w, 1, 64 ch, 1}; the
//     out-of-range columns/rows -- the floor(P/2) zero ring -- are TMA zero
//     fill), then transposed by four warps into a ring of K-major SWIZZLE_128B
//     "row slots" (slot row = input column, 64 channels = 128 B). No NHWC copy
//     of the input ever touches HBM;
//   * every (class, tap) A operand is a row-shifted view of a slot: the UMMA
//     descriptor start address moves by 128 B per column shift (measured on
//     B200: the SWIZZLE_128B phase follows the absolute smem address, so the
//     descriptor's base-offset field stays 0);
//   * consecutive class-grid rows of a strip share nr - 1 of their nr input rows,
//     so each input row is loaded once per strip;
//   * the epilogue holds all four classes of a position, so it writes the two
//     output columns 2j, 2j+1 of both output rows as packed pairs (fully
//     coalesced 128-B warp stores, every output element written once).
//
// Warps: 0 TMA producer, 1 MMA issuer (+TMEM owner), 2..5 epilogue (TMEM lane
// quarters), 6..9 transposers.
#include <cstdlib>
#include <mutex>

#include "igemm.cuh"
#include "tc_ptx.cuh"

namespace segb {

constexpr int kRowsThreads = 320;
constexpr int kRing = 4;
// raw row buffer: [64 ch][128] main box, then [64][8] left and right halo boxes
constexpr uint32_t kRawMain = 64 * kBlockM * 2, kRawHalo = 64 * 8 * 2;

struct RowsClass {
    int R, C, st_r, st_s, base_r, base_s, tap0;
};

struct RowsParams {
    RowsClass cls[4];
    int c_out, oh, ow, p;
    int rows, msub;          // class-grid rows, 128-position subtiles per row
    int dmin_r, nr;          // first window row offset, input rows per class-grid row
    int dmin_c, slot_rows, raw_w;
    int kbc, ntaps;          // 64-channel blocks, n*n
    int total_tiles, tiles_per_cta;
    uint32_t slot_bytes, raw_bytes, b_tile_bytes;
    void *y;
};

struct RowsSmem {  // byte offsets from the 1024-aligned smem base
    uint32_t b, ring, raw, bars, total;
};

__host__ __device__ inline RowsSmem rows_layout(const RowsParams &p) {
    RowsSmem s;
    s.b = 0;
    s.ring = s.b + p.ntaps * p.kbc * p.b_tile_bytes;
    s.raw = s.ring + kRing * p.kbc * p.slot_bytes;
    s.bars = s.raw + ((p.raw_bytes + 1023) / 1024) * 1024;
    s.total = s.bars + (3 + 2 * kRing * p.kbc + 4) * 8 + 16;
    return s;
}

template <typename TY> __device__ __forceinline__ void store_pair(TY *dst, float lo, float hi);
template <> __device__ __forceinline__ void store_pair<__nv_bfloat16>(__nv_bfloat16 *dst, float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    *reinterpret_cast<__nv_bfloat162 *>(dst) = v;
}
template <> __device__ __forceinline__ void store_pair<float>(float *dst, float lo, float hi) {
    *reinterpret_cast<float2 *>(dst) = make_float2(lo, hi);
}

// number of input-row loads a tile triggers (nr when it starts a strip, else 1)
__device__ __forceinline__ int tile_loads(const RowsParams &p, int t, int t0) {
    return (t == t0 || (t % p.rows) == 0) ? p.nr : 1;
}

template <typename TY>
__global__ void __launch_bounds__(kRowsThreads, 1)
    igemm_rows_kernel(const __grid_constant__ CUtensorMap tmRaw, const __grid_constant__ CUtensorMap tmHalo,
                      const __grid_constant__ CUtensorMap tmB,
                      const RowsParams prm) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const RowsSmem L = rows_layout(prm);
    uint8_t *sB = smem + L.b;
    uint8_t *sRing = smem + L.ring;
    uint8_t *sRaw = smem + L.raw;
    uint64_t *b_full = reinterpret_cast<uint64_t *>(smem + L.bars);
    uint64_t *raw_full = b_full + 1;
    uint64_t *raw_empty = b_full + 2;
    uint64_t *slot_full = b_full + 3;
    uint64_t *slot_empty = slot_full + kRing * prm.kbc;
    uint64_t *tfull = slot_empty + kRing * prm.kbc;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int N = prm.c_out;
    const int nslots = kRing * prm.kbc;

    if (threadIdx.x == 0) {
        mbar_init(b_full, 1);
        mbar_init(raw_full, 1);
        mbar_init(raw_empty, 4);
        for (int i = 0; i < nslots; ++i) {
            mbar_init(&slot_full[i], 4);
            mbar_init(&slot_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmRaw) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmHalo) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    }
    const uint32_t tcols = tmem_pow2(8 * N);  // 2 buffers x 4 classes x N fp32 columns
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int t0 = blockIdx.x * prm.tiles_per_cta;
    const int t1 = min(prm.total_tiles, t0 + prm.tiles_per_cta);

    if (warp == 0) {
        if (lane == 0) {  // ---------------- producer: resident weights, then raw input rows
            mbar_expect_tx(b_full, prm.ntaps * prm.kbc * prm.b_tile_bytes);
            for (int tap = 0; tap < prm.ntaps; ++tap)
                for (int kb = 0; kb < prm.kbc; ++kb)
                    tma_load_3d(sB + (tap * prm.kbc + kb) * prm.b_tile_bytes, &tmB, b_full, kb * 64, 0, tap);
            uint32_t g = 0;
            for (int t = t0; t < t1; ++t) {
                const int i = t % prm.rows, rest = t / prm.rows;
                const int ms = rest % prm.msub, b = rest / prm.msub;
                const int nl = tile_loads(prm, t, t0);
                for (int l = prm.nr - nl; l < prm.nr; ++l) {
                    const int row = i + prm.dmin_r + l;
                    for (int kb = 0; kb < prm.kbc; ++kb, ++g) {
                        mbar_wait(raw_empty, (g & 1) ^ 1);
                        // main 128 columns + 8-column halo boxes left and right (a box
                        // may not be wider than the tensor, so the halo is separate)
                        const int j0 = ms * kBlockM;
                        mbar_expect_tx(raw_full, prm.raw_bytes);
                        tma_load_4d(sRaw, &tmRaw, raw_full, j0, row, kb * 64, b);
                        tma_load_4d(sRaw + kRawMain, &tmHalo, raw_full, j0 - 8, row, kb * 64, b);
                        tma_load_4d(sRaw + kRawMain + kRawHalo, &tmHalo, raw_full, j0 + kBlockM, row, kb * 64, b);
                    }
                }
            }
        }
    } else if (warp >= 6) {  // ---------------- transposers: raw [64 ch][raw_w] -> K-major SW128 slot rows
        const int tw = warp - 6;
        const uint16_t *raw = reinterpret_cast<const uint16_t *>(sRaw);
        const int nblk = (prm.slot_rows + 31) / 32;
        uint32_t g = 0, q = 0;
        for (int t = t0; t < t1; ++t) {
            const int nl = tile_loads(prm, t, t0);
            for (int l = 0; l < nl; ++l, ++q) {
                const int k = q % kRing;
                const uint32_t use = q / kRing;
                for (int kb = 0; kb < prm.kbc; ++kb, ++g) {
                    const int sidx = k * prm.kbc + kb;
                    mbar_wait(&slot_empty[sidx], (use & 1) ^ 1);
                    mbar_wait(raw_full, g & 1);
                    const uint32_t dst = smem_u32(sRing + sidx * prm.slot_bytes);
                    for (int task = tw; task < 8 * nblk; task += 4) {
                        const int k8 = task & 7, rho = (task >> 3) * 32 + lane;
                        if (rho < prm.slot_rows) {
                            uint32_t w[4];
#pragma unroll
                            // slot row rho <-> input column j0 + dmin_c + rho
                            const int o = rho + prm.dmin_c;
                            const uint16_t *src;
                            int pitch;
                            if (o < 0) { src = raw + kRawMain / 2 + 8 + o; pitch = 8; }
                            else if (o >= kBlockM) { src = raw + (kRawMain + kRawHalo) / 2 + (o - kBlockM); pitch = 8; }
                            else { src = raw + o; pitch = kBlockM; }
                            for (int e = 0; e < 4; ++e) {
                                const uint32_t lo = src[(8 * k8 + 2 * e) * pitch];
                                const uint32_t hi = src[(8 * k8 + 2 * e + 1) * pitch];
                                w[e] = lo | (hi << 16);
                            }
                            const uint32_t addr = dst + rho * 128 + ((k8 ^ (rho & 7)) << 4);
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(w[0]),
                                         "r"(w[1]), "r"(w[2]), "r"(w[3])
                                         : "memory");
                        }
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&slot_full[sidx]);
                        mbar_arrive(raw_empty);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            mbar_wait(b_full, 0);
            const uint32_t idesc = idesc_bf16(N);
            const uint32_t ring0 = smem_u32(sRing), b0 = smem_u32(sB);
            int acc = 0;
            uint32_t acc_phase = 0, qe = 0;
            for (int t = t0; t < t1; ++t) {
                qe += tile_loads(prm, t, t0);
                const uint32_t qbase = qe - prm.nr;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                for (int l = 0; l < prm.nr; ++l) {
                    const uint32_t q = qbase + l;
                    for (int kb = 0; kb < prm.kbc; ++kb)
                        mbar_wait(&slot_full[(q % kRing) * prm.kbc + kb], (q / kRing) & 1);
                }
                tc_fence_after();
                for (int c = 0; c < 4; ++c) {
                    const RowsClass &g = prm.cls[c];
                    const uint32_t d = tmem_base + acc * 4 * N + c * N;
                    uint32_t accumulate = 0;
                    for (int u = 0; u < g.R; ++u) {
                        const uint32_t q = qbase + (g.base_r + u - prm.p - prm.dmin_r);
                        for (int v = 0; v < g.C; ++v) {
                            const uint32_t dc = g.base_s + v - prm.p - prm.dmin_c;
                            const int tap = g.tap0 + u * g.C + v;
                            for (int kb = 0; kb < prm.kbc; ++kb) {
                                const uint32_t a_addr = ring0 + ((q % kRing) * prm.kbc + kb) * prm.slot_bytes + dc * 128;
                                const uint32_t b_addr = b0 + (tap * prm.kbc + kb) * prm.b_tile_bytes;
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk) {
                                    // row-shifted start address; the SW128 pattern follows the
                                    // absolute smem address bits, so no base offset is needed
                                    tc_mma(d, desc_k_sw128(a_addr + kk * 32), desc_k_sw128(b_addr + kk * 32),
                                           idesc, accumulate);
                                    accumulate = 1;
                                }
                            }
                        }
                    }
                }
                tc_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                // release input rows no later tile of this strip reads
                const bool cont = (t + 1 < t1) && ((t + 1) % prm.rows != 0);
                const int nrel = cont ? 1 : prm.nr;
                for (int l = 0; l < nrel; ++l) {
                    const uint32_t q = qbase + l;
                    for (int kb = 0; kb < prm.kbc; ++kb) tc_commit(&slot_empty[(q % kRing) * prm.kbc + kb]);
                }
            }
        }
    } else {  // ---------------- epilogue (warps 2..5): TMEM lane quarter = warp % 4
        const int quarter = warp & 3;
        const int m = quarter * 32 + lane;
        const int64_t plane = (int64_t)prm.oh * prm.ow;
        TY *y = reinterpret_cast<TY *>(prm.y);
        // y = 2j + st_s: the class with st_s == 0 fills the even column of the pair
        const int s_even = prm.cls[0].st_s == 0 ? 0 : 1;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = t0; t < t1; ++t) {
            const int i = t % prm.rows, rest = t / prm.rows;
            const int ms = rest % prm.msub, b = rest / prm.msub;
            const int j = ms * kBlockM + m;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            TY *base = y + (int64_t)b * N * plane + 2 * j;
            for (int ch = 0; ch < N; ch += 16) {
                uint32_t v[4][16];
#pragma unroll
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    tmem_ld16(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * 4 * N + c * N + ch, v[c]);
                tmem_wait_ld();
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int x = 2 * i + prm.cls[2 * r].st_r;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float a0 = __uint_as_float(v[2 * r][k]), a1 = __uint_as_float(v[2 * r + 1][k]);
                        store_pair<TY>(base + (int64_t)(ch + k) * plane + (int64_t)x * prm.ow, s_even ? a1 : a0,
                                       s_even ? a0 : a1);
                    }
                }
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

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

static bool rows_params(const IgemmShape &s, RowsParams &prm) {
    if (s.n % 2 != 0 || s.x_dtype != SEGB_BF16) return false;
    if (s.y_dtype != SEGB_BF16 && s.y_dtype != SEGB_F32) return false;
    if (s.c_out < 16 || s.c_out > 64 || s.c_out % 16 != 0) return false;
    if (s.w % 8 != 0) return false;  // TMA: NCHW row pitch must be a multiple of 16 B
    const int oh = 2 * s.h + 2 * s.pad - s.n, ow = 2 * s.w + 2 * s.pad - s.n;
    if (oh < 2 || ow < 2) return false;
    const int p = s.pad / 2, swap = s.pad & 1;
    prm = RowsParams{};
    int dmin_r = 1 << 30, dmax_r = -(1 << 30), dmin_c = 1 << 30, dmax_c = -(1 << 30);
    for (int c = 0; c < 4; ++c) {
        const int r = c >> 1, q = c & 1;
        RowsClass &g = prm.cls[c];
        g.R = sub_len(s.n, r);
        g.C = sub_len(s.n, q);
        g.st_r = (r + swap) % 2;
        g.st_s = (q + swap) % 2;
        g.base_r = (g.st_r + r) / 2;
        g.base_s = (g.st_s + q) / 2;
        g.tap0 = class_offset(s.n, c);
        dmin_r = std::min(dmin_r, g.base_r - p);
        dmax_r = std::max(dmax_r, g.base_r + g.R - 1 - p);
        dmin_c = std::min(dmin_c, g.base_s - p);
        dmax_c = std::max(dmax_c, g.base_s + g.C - 1 - p);
    }
    const int rows = oh / 2, cols = ow / 2;
    if (cols % kBlockM != 0) return false;
    prm.c_out = s.c_out; prm.oh = oh; prm.ow = ow; prm.p = p;
    prm.rows = rows; prm.msub = cols / kBlockM;
    prm.dmin_r = dmin_r; prm.nr = dmax_r - dmin_r + 1;
    prm.dmin_c = dmin_c;
    prm.slot_rows = kBlockM + dmax_c - dmin_c;
    prm.raw_w = kBlockM;
    if (-dmin_c > 8 || dmax_c > 8 || prm.nr > kRing) return false;
    if (s.w < kBlockM) return false;
    prm.kbc = (s.c_in + 63) / 64;
    prm.ntaps = s.n * s.n;
    prm.slot_bytes = (prm.slot_rows * 128 + 1023) / 1024 * 1024;
    prm.raw_bytes = kRawMain + 2 * kRawHalo;
    prm.b_tile_bytes = s.c_out * 128;
    const int64_t total = s.batch * (int64_t)prm.msub * rows;
    if (total > INT32_MAX) return false;
    prm.total_tiles = (int)total;
    return rows_layout(prm).total + 1024 <= 227 * 1024;
}

bool igemm_rows_supported(const IgemmShape &s) {
    RowsParams prm;
    return rows_params(s, prm) && tensor_map_encoder() != nullptr;
}

int run_igemm_rows(const IgemmShape &s, const void *x, const void *wg, void *y, cudaStream_t st) {
    RowsParams prm;
    if (!rows_params(s, prm)) return fail(SEGB_ERR_UNSUPPORTED, "row-streaming implicit GEMM: unsupported shape");
    auto encode = tensor_map_encoder();
    CUtensorMap tmRaw, tmHalo, tmB;
    for (int k = 0; k < 2; ++k) {
        cuuint64_t dims[4] = {(cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)s.c_in, (cuuint64_t)s.batch};
        cuuint64_t strides[3] = {(cuuint64_t)s.w * 2, (cuuint64_t)s.h * s.w * 2, (cuuint64_t)s.c_in * s.h * s.w * 2};
        cuuint32_t box[4] = {k == 0 ? (cuuint32_t)kBlockM : 8u, 1, 64, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = encode(k == 0 ? &tmRaw : &tmHalo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(x), dims,
                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SEGB_ERR_CUDA, "tensor map (raw rows): error %d", (int)r);
    }
    {
        cuuint64_t dims[3] = {(cuuint64_t)s.c_in_pad, (cuuint64_t)s.c_out, (cuuint64_t)s.n * s.n};
        cuuint64_t strides[2] = {(cuuint64_t)s.c_in_pad * 2, (cuuint64_t)s.c_out * s.c_in_pad * 2};
        cuuint32_t box[3] = {64, (cuuint32_t)s.c_out, 1};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = encode(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(wg), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SEGB_ERR_CUDA, "tensor map (weights): error %d", (int)r);
    }
    prm.y = y;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<int64_t>(prm.total_tiles, sms);
    prm.tiles_per_cta = (int)ceil_div(prm.total_tiles, grid);
    const size_t smem = rows_layout(prm).total + 1024;
    if (s.y_dtype == SEGB_BF16) {
        cudaFuncSetAttribute(igemm_rows_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        igemm_rows_kernel<__nv_bfloat16><<<grid, kRowsThreads, smem, st>>>(tmRaw, tmHalo, tmB, prm);
    } else {
        cudaFuncSetAttribute(igemm_rows_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        igemm_rows_kernel<float><<<grid, kRowsThreads, smem, st>>>(tmRaw, tmHalo, tmB, prm);
    }
    note_launch();
    return check_launch("igemm_rows_kernel");
}

}  // namespace segb
