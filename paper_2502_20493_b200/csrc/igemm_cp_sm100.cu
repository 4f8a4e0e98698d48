// K3p -- K3 with column-parity class pairs: one tile computes classes (r, 0) AND (r, 1) of the
// same 128 class-grid positions, as a 2-SM CTA pair (tcgen05.mma.cta_group::2, M = 256).
//
// Why. A per-class K3 tile writes every other output column (stride-2 bf16 stores that only
// half-fill each sector), and the two classes of a row parity read overlapping input windows
// from L2 separately. Class (r, s) tap (u, v) reads input column j + base_s + v - p; the
// windows dc = base_s + v of the two column parities overlap (engines.py:338-347: base_s is
// 0 / 1 for s = 0 / 1 when P is even, 0 / 0 when P is odd). Here one k-step is one window
// (u, dc, channel block): the A operand is loaded once and multiplied by the taps of every
// class that reads it, as ONE MMA whose N spans both classes' accumulators when both do
// (B rows = [class s=0 tap | class s=1 tap]). The accumulator then holds, for each position,
// the output columns 2j and 2j + 1 side by side, so the epilogue writes bf16x2 (fp32x2) pairs:
// full sectors, half the store instructions.
//
// Same arithmetic as K3 (per-class sums over taps and channels, fp32 accumulation of bf16
// products), only the grouping of the MMAs differs. Pairs: CTA r of a 2-CTA cluster holds its
// 128 A rows and half of the step's B rows (the class-s=r tile when both classes are in the
// step, else channel half r of the single class's tile); the leader issues, both CTAs' TMA
// loads complete on the leader's barrier, commits multicast, epilogue completions are
// forwarded by the peer's MMA warp.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "igemm.cuh"
#include "tc_ptx.cuh"

namespace segb {

namespace {

constexpr int kCpThreads = 192;  // warp 0 TMA, warp 1 MMA / forwarder, warps 2-5 epilogue
constexpr int kCpMaxWin = 4;
constexpr int kCpMaxStages = 12;

struct CpWindow {
    int dc;     // window column offset (relative to the class grid position, before - p)
    int mask;   // bit s: class (r, s) reads it
    int v[2];   // tap column of class s in this window
    int fresh;  // first window (in order) touching a class's accumulator: accumulate = 0
};

struct CpParams {
    int R, C;                 // sub-kernel rows / cols (even n: equal for all classes)
    int st_r[2], base_r[2];   // per row parity r
    int st_s[2];              // per column parity s (same for both r)
    int tap0[4];              // class-packed tap index of (u, v) = (0, 0), class c = 2r + s
    int nwin[2];
    CpWindow win[2][kCpMaxWin];
    int rows, cols, batch, c_in, c_out, oh, ow, p;
    int nb_w, n_blocks, k_cblocks, m_tiles, m_pairs, total_tiles, stages;
    int64_t class_positions;
    void *y;
};

template <typename TY> __device__ __forceinline__ void store_pair_out(TY *p, float a, float b);
template <> __device__ __forceinline__ void store_pair_out<__nv_bfloat16>(__nv_bfloat16 *p, float a, float b) {
    *reinterpret_cast<__nv_bfloat162 *>(p) = __floats2bfloat162_rn(a, b);
}
template <> __device__ __forceinline__ void store_pair_out<float>(float *p, float a, float b) {
    *reinterpret_cast<float2 *>(p) = make_float2(a, b);
}

template <typename TY>
__global__ void __launch_bounds__(kCpThreads, 1)
    igemm_cp_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const CpParams prm) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = prm.stages, NB = prm.nb_w;
    constexpr uint32_t a_bytes = kBlockM * 128;          // 128 positions x 64 channels
    const uint32_t b_cta = (uint32_t)NB * 128;            // this CTA's B rows per stage (<= NB)
    uint8_t *sA = smem;
    uint8_t *sB = smem + S * a_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + S * b_cta);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int rank = (int)cluster_ctarank();
    const int t_begin = (int)blockIdx.x / 2, t_step = (int)gridDim.x / 2;
    auto decode = [&](int t, int &r, int &mb, int &nb) {
        r = t & 1;
        const int rest = t >> 1;
        mb = 2 * (rest % prm.m_pairs) + rank;
        nb = rest / prm.m_pairs;
    };

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], rank == 0 ? 5 : 4);  // leader: 4 local epilogue warps + the peer's forward
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    }
    const uint32_t tcols = tmem_pow2(2 * 2 * NB);  // 2 buffers x 2 classes x NB fp32 columns
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            for (int t = t_begin; t < prm.total_tiles; t += t_step) {
                int r, mb, nb;
                decode(t, r, mb, nb);
                const int64_t P0 = (int64_t)mb * kBlockM;  // past the last block: zero-filled boxes
                const int64_t per = (int64_t)prm.rows * prm.cols;
                const int b0 = (int)(P0 / per);
                const int rem = (int)(P0 - b0 * per);
                const int i0 = rem / prm.cols, j0 = rem % prm.cols;
                for (int u = 0; u < prm.R; ++u)
                    for (int wi = 0; wi < prm.nwin[r]; ++wi) {
                        const CpWindow &w = prm.win[r][wi];
                        const bool both = w.mask == 3;
                        const int s1 = w.mask == 2 ? 1 : 0;  // the single class when !both
                        for (int kb = 0; kb < prm.k_cblocks; ++kb) {
                            mbar_wait(&empty[stage], phase ^ 1);
                            const uint32_t fb = mapa_rank(&full[stage], 0);
                            if (rank == 0) mbar_expect_tx(&full[stage], 2 * a_bytes + (both ? 2 : 1) * NB * 128);
                            const int wa = j0 + w.dc - prm.p, ha = i0 + prm.base_r[r] + u - prm.p;
                            tma_load_4d_2sm(sA + stage * a_bytes, &tmA, fb, kb * 64, wa, ha, b0);
                            uint8_t *bdst = sB + stage * b_cta;
                            if (both) {  // CTA r: the whole tile of class (r, s = rank), two half boxes
                                const int tap = prm.tap0[2 * r + rank] + u * prm.C + w.v[rank];
                                tma_load_3d_2sm(bdst, &tmB, fb, kb * 64, nb * NB, tap);
                                tma_load_3d_2sm(bdst + NB / 2 * 128, &tmB, fb, kb * 64, nb * NB + NB / 2, tap);
                            } else {     // CTA r: channel half r of the single class's tile
                                const int tap = prm.tap0[2 * r + s1] + u * prm.C + w.v[s1];
                                tma_load_3d_2sm(bdst, &tmB, fb, kb * 64, nb * NB + rank * (NB / 2), tap);
                            }
                            if (++stage == S) { stage = 0; phase ^= 1; }
                        }
                    }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // ---------------- MMA issuer (leader), branch-free over the warp
            const uint32_t leader = elect_one();
            const uint32_t aLo0 = desc_lo_sw128(smem_u32(sA)), bLo0 = desc_lo_sw128(smem_u32(sB));
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            const uint32_t idesc1 = idesc_bf16_m(2 * kBlockM, NB), idesc2 = idesc_bf16_m(2 * kBlockM, 2 * NB);
            for (int t = t_begin; t < prm.total_tiles; t += t_step) {
                const int r = t & 1;
                mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * 2 * NB;
                for (int u = 0; u < prm.R; ++u)
                    for (int wi = 0; wi < prm.nwin[r]; ++wi) {
                        const CpWindow &w = prm.win[r][wi];
                        const bool both = w.mask == 3;
                        const uint32_t dd = d + (w.mask == 2 ? NB : 0);
                        const uint32_t idesc = both ? idesc2 : idesc1;
                        const bool fresh = u == 0 && w.fresh;
                        for (int kb = 0; kb < prm.k_cblocks; ++kb) {
                            // CTA-scope acquire: the stage is filled by TMA (async proxy) only,
                            // both CTAs' bytes completing on this barrier; a cluster-scope acquire
                            // here invalidated L1 (CCTL.IVALL) once per stage
                            mbar_wait(&full[stage], phase);
                            tc_fence_after();
                            const uint32_t a0 = aLo0 + stage * (a_bytes >> 4), b0 = bLo0 + stage * (b_cta >> 4);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                tc_mma_lo<2>(dd, a0 + kk * 2, b0 + kk * 2, idesc, (fresh && kb == 0 && kk == 0) ? 0u : 1u,
                                             leader);
                            tc_commit_2sm_mc_pred(&empty[stage], 3, leader);
                            __syncwarp();
                            if (++stage == S) { stage = 0; phase ^= 1; }
                        }
                    }
                tc_commit_2sm_mc_pred(&tfull[acc], 3, leader);
                __syncwarp();
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        } else if (lane == 0) {  // ---------------- peer: forward drained TMEM buffers to the leader
            int acc = 0;
            uint32_t acc_phase = 0;
            const uint32_t lt[2] = {mapa_rank(&tempty[0], 0), mapa_rank(&tempty[1], 0)};
            for (int t = t_begin; t < prm.total_tiles; t += t_step) {
                mbar_wait(&tempty[acc], acc_phase);
                mbar_arrive_cluster(lt[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {  // ---------------- epilogue: both column parities of a position -> one paired store
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const int64_t plane = (int64_t)prm.oh * prm.ow;
        TY *y = reinterpret_cast<TY *>(prm.y);
        const int lo = prm.st_s[0] == 0 ? 0 : 1;  // class whose columns are even (2j)
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = t_begin; t < prm.total_tiles; t += t_step) {
            int r, mb, nb;
            decode(t, r, mb, nb);
            const int64_t pos = (int64_t)mb * kBlockM + m;
            const bool valid = pos < prm.class_positions;
            const int64_t per = (int64_t)prm.rows * prm.cols;
            const int64_t b = pos / per;
            const int rem = (int)(pos - b * per);
            const int x = 2 * (rem / prm.cols) + prm.st_r[r], y2 = 2 * (rem % prm.cols);
            TY *dst = y + (b * prm.c_out + (int64_t)nb * NB) * plane + (int64_t)x * prm.ow + y2;
            const int co_left = prm.c_out - nb * NB;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16) + acc * 2 * NB;
            // the next chunk's TMEM loads are in flight while this chunk is stored
            uint32_t v0[8], v1[8];
            tmem_ld8(tl + lo * NB, v0);         // column 2j
            tmem_ld8(tl + (1 - lo) * NB, v1);   // column 2j + 1
            for (int c0 = 0; c0 < NB; c0 += 8) {
                tmem_wait_ld();
                reg_fence8(v0);
                reg_fence8(v1);
                uint32_t w0[8], w1[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) { w0[k] = v0[k]; w1[k] = v1[k]; }
                if (c0 + 8 < NB) {
                    tmem_ld8(tl + lo * NB + c0 + 8, v0);
                    tmem_ld8(tl + (1 - lo) * NB + c0 + 8, v1);
                } else {  // last chunk: the buffer is drained
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                }
                if (valid) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (c0 + k < co_left)
                            store_pair_out<TY>(dst + (int64_t)(c0 + k) * plane, __uint_as_float(w0[k]),
                                               __uint_as_float(w1[k]));
                }
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the leader's MMAs write this CTA's TMEM until both are done
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tcols));
    }
    cluster_sync_all();
}

}  // namespace

// Shapes K3p takes: bf16 compute, even n (all classes share one grid), even output width (the
// two column parities have equal grids and write adjacent columns), two position blocks to
// pair, c_in >= 64. The A operand is K3's NHWC copy; B is K3's weight layout.
bool cp_params(const IgemmShape &s, CpParams &prm) {
    const char *e = getenv("SEGB200_K3_CP");
    if (e && !atoi(e)) return false;
    if (s.compute != SEGB_BF16 || s.n % 2 != 0 || s.c_in < 64 || s.c_in % 8 != 0) return false;
    if (s.x_dtype != SEGB_BF16 && s.x_dtype != SEGB_F32) return false;
    if (s.y_dtype != SEGB_BF16 && s.y_dtype != SEGB_F32) return false;
    if (s.batch > 65535) return false;
    const int oh = 2 * s.h + 2 * s.pad - s.n, ow = 2 * s.w + 2 * s.pad - s.n;
    if (oh < 2 || ow < 2 || ow % 2 != 0 || oh % 2 != 0) return false;
    prm = CpParams{};
    const int p = s.pad / 2, swap = s.pad & 1;
    const int nh = s.n / 2;
    prm.R = prm.C = nh;
    for (int r = 0; r < 2; ++r) {
        prm.st_r[r] = (r + swap) % 2;
        prm.base_r[r] = (prm.st_r[r] + r) / 2;
    }
    int base_s[2];
    for (int q = 0; q < 2; ++q) {
        prm.st_s[q] = (q + swap) % 2;
        base_s[q] = (prm.st_s[q] + q) / 2;
    }
    for (int c = 0; c < 4; ++c) prm.tap0[c] = class_offset(s.n, c);
    // windows: shared ones first so the first k-step of a tile initialises both accumulators
    for (int r = 0; r < 2; ++r) {
        const int lo_dc = std::min(base_s[0], base_s[1]), hi_dc = std::max(base_s[0], base_s[1]) + nh - 1;
        int cnt = 0, covered = 0;
        for (int pass = 0; pass < 2; ++pass)
            for (int dc = lo_dc; dc <= hi_dc; ++dc) {
                int mask = 0;
                CpWindow w{};
                w.dc = dc;
                for (int q = 0; q < 2; ++q)
                    if (dc - base_s[q] >= 0 && dc - base_s[q] < nh) {
                        mask |= 1 << q;
                        w.v[q] = dc - base_s[q];
                    }
                if ((pass == 0) != (mask == 3) || !mask) continue;
                if (cnt >= kCpMaxWin) return false;
                w.mask = mask;
                w.fresh = (mask & ~covered) != 0;
                covered |= mask;
                prm.win[r][cnt++] = w;
            }
        prm.nwin[r] = cnt;
        if (cnt == 0 || covered != 3) return false;
    }
    prm.rows = oh / 2;
    prm.cols = ow / 2;
    // K3's A box (128 positions of the class grid) must tile the grid
    const int cols = prm.cols, rows = prm.rows;
    if (cols >= kBlockM) {
        if (cols % kBlockM) return false;
    } else {
        if (kBlockM % cols) return false;
        const int bh = std::min(rows, kBlockM / cols);
        if (rows % bh) return false;
        if (bh == rows && kBlockM % (cols * rows)) return false;
    }
    // one channel block of <= 128 (the pair of classes fills N <= 256): for wider c_out the
    // per-class K3 with 256-wide tiles measured faster (ebgan l2-l4), so K3p takes c_out <= 128
    const int cop = (int)ceil_div(s.c_out, 32) * 32;
    if (cop > 128) return false;
    int nb_w = cop;
    if (const char *e = getenv("SEGB200_K3P_NB")) {  // A/B experiments: narrower N blocks, more stages
        const int v = atoi(e);
        if (v >= 32 && v % 32 == 0 && cop % v == 0) nb_w = v;
    }
    prm.nb_w = nb_w;
    prm.n_blocks = cop / nb_w;
    prm.batch = (int)s.batch; prm.c_in = s.c_in; prm.c_out = s.c_out; prm.oh = oh; prm.ow = ow; prm.p = p;
    prm.k_cblocks = (s.c_in + 63) / 64;
    prm.class_positions = s.batch * (int64_t)rows * cols;
    prm.m_tiles = (int)ceil_div(prm.class_positions, kBlockM);
    if (prm.m_tiles < 2) return false;
    prm.m_pairs = (prm.m_tiles + 1) / 2;
    const int64_t total = 2ll * prm.m_pairs * prm.n_blocks;
    if (total > INT32_MAX) return false;
    // too few pair tiles to fill half the SM pairs (small batches): K3 with narrow N tiles and
    // split K spreads the layer wider (dcgan_l4 bf16 at batch 1: 24.6 -> 18.4 us; batch 16: 24.6
    // -> 22.5). SEGB200_K3P_MIN_TILES overrides (tests run K3p at small shapes with 0).
    int64_t min_tiles = 37;
    if (const char *mt = getenv("SEGB200_K3P_MIN_TILES")) min_tiles = atoll(mt);
    if (total < min_tiles) return false;
    prm.total_tiles = (int)total;
    const int stage_bytes = kBlockM * 128 + nb_w * 128;
    prm.stages = std::min(kCpMaxStages, (int)((227 * 1024 - 1024 - 256) / stage_bytes));
    return prm.stages >= 2;
}

bool igemm_cp_supported(const IgemmShape &s) {
    CpParams prm;
    return cp_params(s, prm) && tensor_map_encoder() != nullptr;
}

// x_nhwc: K3's channels-last bf16 copy of the input; wg: K3's weights [tap][c_out_pad][c_in_pad]
int run_igemm_cp_core(const IgemmShape &s, const void *x_nhwc, const void *wg, void *y, cudaStream_t st) {
    CpParams prm;
    if (!cp_params(s, prm)) return fail(SEGB_ERR_UNSUPPORTED, "class-pair implicit GEMM: unsupported shape");
    auto encode = tensor_map_encoder();
    // A: NHWC bf16, box {64 ch, box_w, box_h, box_b} = 128 positions (as K3)
    int box_w, box_h, box_b;
    if (prm.cols >= kBlockM) {
        box_w = kBlockM; box_h = 1; box_b = 1;
    } else {
        box_w = prm.cols;
        box_h = std::min(prm.rows, kBlockM / prm.cols);
        box_b = box_h == prm.rows ? kBlockM / (prm.cols * prm.rows) : 1;
    }
    CUtensorMap tmA, tmB;
    cuuint32_t es[4] = {1, 1, 1, 1};
    {
        cuuint64_t dims[4] = {(cuuint64_t)s.c_in, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)s.batch};
        cuuint64_t strides[3] = {(cuuint64_t)s.c_in * 2, (cuuint64_t)s.w * s.c_in * 2,
                                 (cuuint64_t)s.h * s.w * s.c_in * 2};
        cuuint32_t box[4] = {64, (cuuint32_t)box_w, (cuuint32_t)box_h, (cuuint32_t)box_b};
        CUresult r = encode(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(x_nhwc), dims, strides, box,
                            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SEGB_ERR_CUDA, "tensor map (K3p A): error %d", (int)r);
    }
    {
        cuuint64_t dims[3] = {(cuuint64_t)s.c_in_pad, (cuuint64_t)s.c_out_pad, (cuuint64_t)s.n * s.n};
        cuuint64_t strides[2] = {(cuuint64_t)s.c_in_pad * 2, (cuuint64_t)s.c_out_pad * s.c_in_pad * 2};
        cuuint32_t box[3] = {64, (cuuint32_t)(prm.nb_w / 2), 1};
        CUresult r = encode(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(wg), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SEGB_ERR_CUDA, "tensor map (K3p B): error %d", (int)r);
    }
    prm.y = y;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t stage_bytes = (size_t)kBlockM * 128 + (size_t)prm.nb_w * 128;
    const size_t smem = 1024 + prm.stages * stage_bytes + (2 * prm.stages + 4) * 8 + 16;
    const unsigned grid = 2 * (unsigned)std::min<int64_t>(prm.total_tiles, sms / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kCpThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (s.y_dtype == SEGB_BF16) {
        cudaFuncSetAttribute(igemm_cp_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        e = cudaLaunchKernelEx(&cfg, igemm_cp_kernel<__nv_bfloat16>, tmA, tmB, prm);
    } else {
        cudaFuncSetAttribute(igemm_cp_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        e = cudaLaunchKernelEx(&cfg, igemm_cp_kernel<float>, tmA, tmB, prm);
    }
    if (e != cudaSuccess) return fail(SEGB_ERR_CUDA, "igemm_cp_kernel: %s", cudaGetErrorString(e));
    note_launch();
    return check_launch("igemm_cp_kernel");
}

}  // namespace segb
