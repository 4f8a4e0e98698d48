// K3 -- per-parity-class implicit GEMM on the 5th-gen tensor cores (sm_100a).
//
// For parity class (r, s) of the unified rule (engines.py:271-291 computes the
// same per-class product with an explicit im2col + BLAS GEMM, :309-335):
//
//   out[b, co, 2i + st_r, 2j + st_s] = sum_{u<R(r), v<R(s), ci}
//        X[b, ci, i + base_r + u - p, j + base_s + v - p] * K[ci, co, 2u + r, 2v + s]
//
// i.e. a GEMM with M = positions (b, i, j) of the class grid, N = c_out,
// K = (tap (u, v), ci). Nothing is materialised: the A operand of tap (u, v)
// is a TMA box of the channels-last activations at coordinates shifted by the
// tap, and TMA's out-of-bounds zero fill *is* the floor(P/2) zero ring.
//
// Kernel: persistent, warp-specialised, one CTA per SM.
//   warp 0      TMA producer  (A box + B tile per k-step into a 4..8-stage ring)
//   warp 1      MMA issuer    (tcgen05.mma.cta_group::1.kind::f16, M=128, N=n_tile,
//                              fp32 accumulators in TMEM, double-buffered)
//   warps 2..5  epilogue      (tcgen05.ld -> registers -> NCHW stores of the class
//                              positions; each output element written once)
// Operands: A = activations NHWC bf16 (K-major, SWIZZLE_128B, 64 channels =
// 128 B per row), B = K1-prepared weights [tap][c_out][c_in_pad] bf16 (K-major,
// SWIZZLE_128B). Tiles: (class, 128 positions, n_tile output channels); the
// class index varies fastest so the four parity classes of a position block run
// concurrently on neighbouring SMs (shared input windows hit in L2, and their
// interleaved stride-2 output sectors are completed in L2 before write-back).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "f16split.cuh"
#include "igemm.cuh"
#include "tc_ptx.cuh"

namespace segb {

constexpr int kThreads = 192;
// operand modes: bf16 (kind::f16, one MMA per product), fp32 as 3xTF32 (kind::tf32: hi/lo tf32
// planes, three MMAs) or as 3xFP16 (kind::f16 on scaled fp16 hi/lo planes, three MMAs at twice
// the tf32 rate; f16split.cuh)
constexpr int kModeBf16 = 0, kModeTf32x3 = 1, kModeF16x3 = 2;
// A k-step covers one 128-B SWIZZLE_128B row of channels: 64 bf16 / fp16 or 32 fp32 (kind::tf32).
template <int MODE> constexpr int kstep_channels() { return MODE == kModeTf32x3 ? 32 : 64; }
// 3-pass partial-sum depth: the tensor core's fp32 accumulation error grows with the number
// of accumulate steps (measured on B200: ~0.25 ulp per MMA), so every kTf32Chunk k-steps
// (96 MMAs) the partial is moved into fp32 registers.
constexpr int kTf32Chunk = 8;
// 3xFP16 k-steps hold twice the channels (the same 12 MMAs per k-step); its partials are drained
// every 4 k-steps (48 MMAs): measured max rel vs the fp64 oracle 5e-6 with 8 (B=256 EB-GAN)
#ifndef SEGB_F16X3_CHUNK
#define SEGB_F16X3_CHUNK 4
#endif
constexpr int kF16Chunk = SEGB_F16X3_CHUNK;
#ifndef SEGB_K3_NACC3
#define SEGB_K3_NACC3 4
#endif
constexpr int kTf32MaxN = 128;

// instruction descriptor: fp16 x fp16 -> fp32, A and B K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBlockM >> 4) << 24);
}

struct ClassGeom {
    int R, C;             // sub-kernel rows / cols
    int rows, cols;       // class grid
    int st_r, st_s;       // first output row / col of the class
    int base_r, base_s;   // first window base (engines.py:338-347)
    int tap0;             // class-packed tap index of (u, v) = (0, 0)
};

struct IgemmParams {
    ClassGeom cls[4];
    int batch, c_in, c_out, oh, ow, p;
    int n_tile, n_blocks, k_cblocks, m_tiles, total_tiles, stages;
    int m_pairs;              // PAIR: position blocks per CTA pair (m_tiles rounded up / 2)
    int box_w, box_h, box_b;  // A box (positions): cols x rows x samples = 128
    int64_t class_positions;  // batch * rows * cols (identical for all classes here)
    void *y;
    const float *x_partials;  // 3xFP16: the input's partial maxima (its scale 2^k_x)
    float w_unscale;          // 3xFP16: 2^-k_w of the weight planes
    int swap_ab;              // PM 3: weights as the M = 128 side, the few class positions as N
    int ksplit;               // > 1: each tile covers 1/ksplit of K and writes fp32 partial sums
    float *partial;           // ksplit: [ks][class][c_out][class position] fp32 partials
};

template <typename TY> __device__ __forceinline__ TY cvt_out(float v);
template <> __device__ __forceinline__ float cvt_out<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// ---------------------------------------------------------------- the kernel
// MODE kModeTf32x3: fp32 operands as 3xTF32 (A_hi*B_hi + A_hi*B_lo + A_lo*B_hi, ~fp32 accuracy)
// on tcgen05.mma.kind::tf32; each stage then holds hi and lo tiles of both operands.
// PAIR: the grid is made of 2-CTA clusters. The two CTAs of a pair compute adjacent position
// blocks (2 mbp, 2 mbp + 1) of the same class and output-channel block in lockstep, so they
// need the same B tile: each loads one half of it and multicasts it to both, halving the
// weight traffic from L2 per CTA; a stage is refilled only after both CTAs' MMAs released
// it (each commit arrives on the stage's empty barrier in both CTAs).
// PM: 0 = single CTA; 1 = PAIR with the B tile multicast; 2 = PAIR as one 2-SM MMA
// (tcgen05.mma.cta_group::2, M = 256): each CTA holds its 128 A rows and HALF of the B tile
// (N/2 rows) at the same shared-memory offsets, the leader (rank 0) issues the MMAs for both,
// each CTA's TMEM receives its own 128 rows x N columns, the TMA loads of both CTAs signal
// the leader's full barrier, the leader's commits arrive on both CTAs' empty / tfull
// barriers and both CTAs' epilogue warps arrive on the leader's tempty barrier.
// kModeF16x3: the same three products on scaled fp16 planes with kind::f16 MMAs; the epilogue
// multiplies the fp32 sum by 2^-(k_x + k_w).
template <typename TY, int MODE, int PM>
__global__ void __launch_bounds__(kThreads, 1)
    igemm_tconv_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmAlo, const __grid_constant__ CUtensorMap tmBlo,
                       const IgemmParams prm) {
    constexpr bool TF32X3 = MODE != kModeBf16;  // three-pass hi/lo operands (either kind)
    constexpr bool TFK = MODE == kModeTf32x3;   // kind::tf32 MMAs
    constexpr int KCH = kstep_channels<MODE>();
    constexpr int NOP = TF32X3 ? 2 : 1;  // tiles per operand per stage (hi [, lo])
    constexpr int CHUNK = MODE == kModeF16x3 ? kF16Chunk : kTf32Chunk;  // k-steps per TMEM partial
    // TMEM accumulator buffers: the 3-pass modes (N <= 128) keep four, so the MMAs run up to three
    // partials ahead while the epilogue writes a finished tile (with two, a tile's output stores
    // held the next tile's second partial; fp32 ebgan_l5 has only four partials per tile)
    constexpr int NACC = TF32X3 ? SEGB_K3_NACC3 : 2;
    // PM 3 (SWAP): a single CTA with the operands swapped -- A = 128 output channels of weights,
    // B = the tile's class positions (N = 16..128): tiny batches, where a 128-position A box would be
    // mostly zero fill and the weights are the bytes that matter
    constexpr bool PAIR = PM == 1 || PM == 2, TWO = PM == 2, SWAP = PM == 3;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for SWIZZLE_128B atoms
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = prm.stages;
    const uint32_t a_bytes = kBlockM * 128;       // one A tile: 128 rows x 128 B
    const uint32_t b_bytes = prm.n_tile * 128;    // one B tile: n_tile rows x 128 B
    const uint32_t b_cta = TWO ? b_bytes / 2 : b_bytes;  // B bytes held per CTA and stage
    uint8_t *sA = smem;                           // [stage][NOP] A tiles
    uint8_t *sB = smem + S * NOP * a_bytes;       // [stage][NOP] B tiles (TWO: this CTA's half)
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + S * NOP * b_cta);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + NACC;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + NACC);
    float *unscale_slot = reinterpret_cast<float *>(tmem_slot + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int N = prm.n_tile;
    const int rank = PAIR ? (int)cluster_ctarank() : 0;
    // tile iteration: the pair index walks the pair tiles, both CTAs of a pair in lockstep
    const int t_begin = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;
    const int t_step = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;
    // K range of a tile: with split K, tile t covers k-steps [k_lo, k_hi) of its class
    auto krange = [&](int t, int &k_lo, int &k_hi) {
        const ClassGeom &g = prm.cls[t & 3];
        const int nks = g.R * g.C * prm.k_cblocks;
        if (prm.ksplit <= 1) { k_lo = 0; k_hi = nks; return; }
        const int ks = (t >> 2) % prm.ksplit, chunk = (nks + prm.ksplit - 1) / prm.ksplit;
        k_lo = min(nks, ks * chunk);
        k_hi = min(nks, k_lo + chunk);
    };
    auto decode = [&](int t, int &c, int &mb, int &nb) {
        c = t & 3;
        const int rest = (t >> 2) / prm.ksplit;
        if (PAIR) {
            mb = 2 * (rest % prm.m_pairs) + rank;
            nb = rest / prm.m_pairs;
        } else {
            mb = rest % prm.m_tiles;
            nb = rest / prm.m_tiles;
        }
    };

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], PM == 1 ? 2 : 1);
        }
        for (int i = 0; i < NACC; ++i) {
            mbar_init(&tfull[i], 1);
            // TWO: the leader's counts its 4 epilogue warps + 1 forwarded arrival from the peer
            mbar_init(&tempty[i], TWO && rank == 0 ? 5 : 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        if (TF32X3) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmAlo) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmBlo) : "memory");
        }
    }
    if (MODE == kModeF16x3 && warp == 2) {  // the input's scale from the absmax partials
        float m = 0.f;
        for (int i = lane; i < kAbsmaxBlocks; i += 32) m = fmaxf(m, __ldg(prm.x_partials + i));
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if (lane == 0) *unscale_slot = ldexpf(1.f, -f16_scale_exp(m)) * prm.w_unscale;
    }
    if (warp == 1) {  // TMEM: two accumulator buffers of N fp32 columns
        const uint32_t cols = NACC == 2 ? tmem_cols(N) : tmem_pow2(NACC * N);
        if (TWO) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();  // both CTAs' barriers initialised before any multicast lands
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int S_ = S;
    // an epilogue warp hands a TMEM accumulator buffer back on its own CTA's barrier (a
    // cluster-scope release right after the global stores would stall on them); TWO: the peer's
    // idle MMA warp forwards its CTA's completions to the leader
    auto release_acc = [&](int a) { mbar_arrive(&tempty[a]); };

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int t = t_begin; t < prm.total_tiles; t += t_step) {
                int c, mb, nb;
                decode(t, c, mb, nb);
                const ClassGeom &g = prm.cls[c];
                const int64_t P0 = (int64_t)mb * (SWAP ? N : kBlockM);  // past the last block: zero-filled boxes
                const int64_t per = (int64_t)g.rows * g.cols;
                const int b0 = (int)(P0 / per);
                const int rem = (int)(P0 - b0 * per);
                const int i0 = rem / g.cols, j0 = rem % g.cols;
                int k_lo, k_hi;
                krange(t, k_lo, k_hi);
                for (int kf = k_lo; kf < k_hi; ++kf) {
                            const int kb = kf % prm.k_cblocks, uv = kf / prm.k_cblocks;
                            const int u = uv / g.C, v = uv % g.C;
                            mbar_wait(&empty[stage], phase ^ 1);
                            const int wa = j0 + g.base_s + v - prm.p, ha = i0 + g.base_r + u - prm.p;
                            const int tap = g.tap0 + u * g.C + v;
                            if (TWO) {  // own A rows + own half of B, counted on the leader's barrier
                                const uint32_t fb = mapa_rank(&full[stage], 0);
                                if (rank == 0) mbar_expect_tx(&full[stage], NOP * 2 * (a_bytes + b_cta));
                                tma_load_4d_2sm(sA + stage * NOP * a_bytes, &tmA, fb, kb * KCH, wa, ha, b0);
                                tma_load_3d_2sm(sB + stage * NOP * b_cta, &tmB, fb, kb * KCH, nb * N + rank * (N / 2),
                                                tap);
                                if (TF32X3) {
                                    tma_load_4d_2sm(sA + (stage * NOP + 1) * a_bytes, &tmAlo, fb, kb * KCH, wa, ha, b0);
                                    tma_load_3d_2sm(sB + (stage * NOP + 1) * b_cta, &tmBlo, fb, kb * KCH,
                                                    nb * N + rank * (N / 2), tap);
                                }
                                if (++stage == S_) { stage = 0; phase ^= 1; }
                                continue;
                            }
                            mbar_expect_tx(&full[stage], NOP * (a_bytes + b_bytes));
                            if (SWAP) {  // A: 128 channels of the tap's weights; B: the positions
                                tma_load_3d(sA + stage * NOP * a_bytes, &tmB, &full[stage], kb * KCH, nb * kBlockM, tap);
                                tma_load_4d(sB + stage * NOP * b_bytes, &tmA, &full[stage], kb * KCH, wa, ha, b0);
                                if (TF32X3) {
                                    tma_load_3d(sA + (stage * NOP + 1) * a_bytes, &tmBlo, &full[stage], kb * KCH,
                                                nb * kBlockM, tap);
                                    tma_load_4d(sB + (stage * NOP + 1) * b_bytes, &tmAlo, &full[stage], kb * KCH, wa, ha,
                                                b0);
                                }
                                if (++stage == S_) { stage = 0; phase ^= 1; }
                                continue;
                            }
                            tma_load_4d(sA + stage * NOP * a_bytes, &tmA, &full[stage], kb * KCH, wa, ha, b0);
                            if (TF32X3)
                                tma_load_4d(sA + (stage * NOP + 1) * a_bytes, &tmAlo, &full[stage], kb * KCH, wa, ha, b0);
                            if (PAIR) {  // this CTA's half of the B tile, to both CTAs
                                const uint32_t half = b_bytes / 2;
                                tma_load_3d_mc(sB + stage * NOP * b_bytes + rank * half, &tmB, &full[stage], kb * KCH,
                                               nb * N + rank * (N / 2), tap, 3);
                                if (TF32X3)
                                    tma_load_3d_mc(sB + (stage * NOP + 1) * b_bytes + rank * half, &tmBlo, &full[stage],
                                                   kb * KCH, nb * N + rank * (N / 2), tap, 3);
                            } else {
                                tma_load_3d(sB + stage * NOP * b_bytes, &tmB, &full[stage], kb * KCH, nb * N, tap);
                                if (TF32X3)
                                    tma_load_3d(sB + (stage * NOP + 1) * b_bytes, &tmBlo, &full[stage], kb * KCH, nb * N, tap);
                            }
                            if (++stage == S_) { stage = 0; phase ^= 1; }
                        }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (TWO: the leader CTA). The whole warp walks the loop and one
        // elected lane issues (branch-free MMAs keep the descriptor math in uniform registers).
        if (!(TWO && rank != 0)) {
            const uint32_t leader = elect_one();
            const uint32_t aLo0 = desc_lo_sw128(smem_u32(sA)), bLo0 = desc_lo_sw128(smem_u32(sB));
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            const uint32_t idesc0 = MODE == kModeTf32x3 ? idesc_tf32(N) : (MODE == kModeF16x3 ? idesc_f16(N) : idesc_bf16(N));
            const uint32_t idesc = TWO ? idesc0 + ((uint32_t)(256 - kBlockM) >> 4 << 24) : idesc0;
            // commits predicated on the elected lane like the MMAs: no divergent branch in the
            // loop, so ptxas keeps the stage / descriptor arithmetic in uniform registers
            auto commit = [&](uint64_t *bar, bool both) {
                if (TWO) tc_commit_2sm_mc_pred(bar, 3, leader);
                else if (PAIR && both) tc_commit_mc_pred(bar, 3, leader);
                else tc_commit_pred(bar, leader);
                __syncwarp();
            };
            for (int t = t_begin; t < prm.total_tiles; t += t_step) {
                int k_lo, k_hi;
                krange(t, k_lo, k_hi);
                const int ksteps = k_hi - k_lo;
                uint32_t d = 0;
                for (int ks = 0; ks < ksteps; ++ks) {
                    // 3xTF32 accumulates at most kTf32Chunk k-steps per TMEM partial (the
                    // epilogue sums partials in fp32 registers, round-to-nearest)
                    const int kc = TF32X3 ? ks % CHUNK : ks;
                    if (kc == 0) {
                        if (ks > 0) {
                            commit(&tfull[acc], false);
                            if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
                        }
                        mbar_wait(&tempty[acc], acc_phase ^ 1);
                        tc_fence_after();
                        d = tmem_base + acc * N;
                    }
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    // low descriptor words (the start address field moves by 2 per 32 B of K)
                    const uint32_t a0 = aLo0 + stage * (NOP * a_bytes >> 4), b0 = bLo0 + stage * (NOP * b_cta >> 4);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {  // 4 MMAs of 32 B of K (16 bf16 / 8 tf32) per 128-B row
                        if (TF32X3) {
                            const uint32_t ah = a0 + kk * 2, al = a0 + (a_bytes >> 4) + kk * 2;
                            const uint32_t bh = b0 + kk * 2, bl = b0 + (b_cta >> 4) + kk * 2;
                            tc_mma_lo<TWO ? 2 : 1, TFK>(d, ah, bh, idesc, (kc | kk) != 0, leader);
                            tc_mma_lo<TWO ? 2 : 1, TFK>(d, ah, bl, idesc, 1, leader);
                            tc_mma_lo<TWO ? 2 : 1, TFK>(d, al, bh, idesc, 1, leader);
                        } else {
                            tc_mma_lo<TWO ? 2 : 1, false>(d, a0 + kk * 2, b0 + kk * 2, idesc, (ks | kk) != 0, leader);
                        }
                    }
                    commit(&empty[stage], true);
                    if (++stage == S_) { stage = 0; phase ^= 1; }
                }
                commit(&tfull[acc], false);
                if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
            }
        } else if (lane == 0) {  // ---------------- TWO, peer: forward "TMEM buffer drained" to the leader
            int acc = 0;
            uint32_t acc_phase = 0;
            uint32_t lt[NACC];
#pragma unroll
            for (int i = 0; i < NACC; ++i) lt[i] = mapa_rank(&tempty[i], 0);
            for (int t = t_begin; t < prm.total_tiles; t += t_step) {
                int k_lo, k_hi;
                krange(t, k_lo, k_hi);
                const int uses = TF32X3 ? (k_hi - k_lo + CHUNK - 1) / CHUNK : 1;
                for (int k = 0; k < uses; ++k) {
                    mbar_wait(&tempty[acc], acc_phase);
                    mbar_arrive_cluster(lt[acc]);
                    if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
                }
            }
        }
    } else if (SWAP) {  // ---------------- epilogue, swapped: TMEM lane = output channel, column = position
        const int q = warp & 3;
        const float unscale = MODE == kModeF16x3 ? *unscale_slot : 1.f;
        const int64_t plane = (int64_t)prm.oh * prm.ow;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = t_begin; t < prm.total_tiles; t += t_step) {
            int c, mb, nb;
            decode(t, c, mb, nb);
            const ClassGeom &g = prm.cls[c];
            int k_lo, k_hi;
            krange(t, k_lo, k_hi);
            const int nchunks = TF32X3 ? (k_hi - k_lo + CHUNK - 1) / CHUNK : 1;
            const int co = nb * kBlockM + q * 32 + lane;
            float racc[kTf32MaxN];
#pragma unroll
            for (int k = 0; k < kTf32MaxN; ++k) racc[k] = 0.f;
            for (int pc = 0; pc < nchunks; ++pc) {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
#pragma unroll
                for (int ch = 0; ch < kTf32MaxN / 16; ++ch) {
                    if (ch * 16 < N) {
                        uint32_t v[16];
                        tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + acc * N + ch * 16, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int k = 0; k < 16; ++k) racc[ch * 16 + k] += __uint_as_float(v[k]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) release_acc(acc);
                if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
            }
            if (co < prm.c_out) {
                const int64_t per = (int64_t)g.rows * g.cols;
#pragma unroll
                for (int k = 0; k < kTf32MaxN; ++k) {
                    const int64_t pos = (int64_t)mb * N + k;
                    if (k >= N || pos >= prm.class_positions) continue;
                    const float val = MODE == kModeF16x3 ? racc[k] * unscale : racc[k];
                    if (prm.ksplit > 1) {
                        const int ksi = (t >> 2) % prm.ksplit;
                        prm.partial[((int64_t)(ksi * 4 + c) * prm.c_out + co) * prm.class_positions + pos] = val;
                    } else {
                        const int64_t b = pos / per;
                        const int rem = (int)(pos - b * per);
                        const int x = 2 * (rem / g.cols) + g.st_r, yy = 2 * (rem % g.cols) + g.st_s;
                        reinterpret_cast<TY *>(prm.y)[(b * prm.c_out + co) * plane + (int64_t)x * prm.ow + yy] =
                            cvt_out<TY>(val);
                    }
                }
            }
        }
    } else if (TF32X3) {  // ---------------- epilogue, 3-pass: sum the TMEM partials in registers
        const int q = warp & 3;
        const float unscale = MODE == kModeF16x3 ? *unscale_slot : 1.f;
        const int m = q * 32 + lane;
        const int64_t plane = (int64_t)prm.oh * prm.ow;
        float *y = reinterpret_cast<float *>(prm.y);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = t_begin; t < prm.total_tiles; t += t_step) {
            int c, mb, nb;
            decode(t, c, mb, nb);
            const ClassGeom &g = prm.cls[c];
            int k_lo, k_hi;
            krange(t, k_lo, k_hi);
            const int nchunks = (k_hi - k_lo + CHUNK - 1) / CHUNK;
            float racc[kTf32MaxN];
#pragma unroll
            for (int k = 0; k < kTf32MaxN; ++k) racc[k] = 0.f;
            for (int pc = 0; pc < nchunks; ++pc) {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
#pragma unroll
                for (int ch = 0; ch < kTf32MaxN / 32; ++ch) {
                    if (ch * 32 < N) {
                        uint32_t v[32];
                        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * N + ch * 32, v);
#pragma unroll
                        for (int k = 0; k < 32; ++k) racc[ch * 32 + k] += __uint_as_float(v[k]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) release_acc(acc);
                if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
            }
            const int64_t pos = (int64_t)mb * kBlockM + m;
            if (pos < prm.class_positions && prm.ksplit > 1) {  // split K: this range's fp32 partial
                const int ksi = (t >> 2) % prm.ksplit;
                float *pp = prm.partial + ((int64_t)(ksi * 4 + c) * prm.c_out + (int64_t)nb * N) * prm.class_positions + pos;
                const int co_left = prm.c_out - nb * N;
#pragma unroll
                for (int k = 0; k < kTf32MaxN; ++k)
                    if (k < N && k < co_left)
                        pp[(int64_t)k * prm.class_positions] = MODE == kModeF16x3 ? racc[k] * unscale : racc[k];
            } else if (pos < prm.class_positions) {
                const int64_t per = (int64_t)g.rows * g.cols;
                const int64_t b = pos / per;
                const int rem = (int)(pos - b * per);
                const int x = 2 * (rem / g.cols) + g.st_r, yy = 2 * (rem % g.cols) + g.st_s;
                float *dst = y + (b * prm.c_out + (int64_t)nb * N) * plane + (int64_t)x * prm.ow + yy;
                const int co_left = prm.c_out - nb * N;
#pragma unroll
                for (int k = 0; k < kTf32MaxN; ++k)
                    if (k < N && k < co_left) dst[(int64_t)k * plane] = MODE == kModeF16x3 ? racc[k] * unscale : racc[k];
            }
        }
    } else {  // ---------------- epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const int64_t plane = (int64_t)prm.oh * prm.ow;
        TY *y = reinterpret_cast<TY *>(prm.y);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = t_begin; t < prm.total_tiles; t += t_step) {
            int c, mb, nb;
            decode(t, c, mb, nb);
            const ClassGeom &g = prm.cls[c];
            const int64_t pos = (int64_t)mb * kBlockM + m;
            const bool valid = pos < prm.class_positions;
            const int64_t per = (int64_t)g.rows * g.cols;
            const int64_t b = pos / per;
            const int rem = (int)(pos - b * per);
            const int x = 2 * (rem / g.cols) + g.st_r, yy = 2 * (rem % g.cols) + g.st_s;
            TY *dst = y + (b * prm.c_out + (int64_t)nb * N) * plane + (int64_t)x * prm.ow + yy;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            for (int ch = 0; ch < N / 32; ++ch) {
                uint32_t v[32];
                tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * N + ch * 32, v);
                if (valid && prm.ksplit > 1) {  // split K: this range's fp32 partial
                    const int ksi = (t >> 2) % prm.ksplit;
                    float *pp = prm.partial +
                                ((int64_t)(ksi * 4 + c) * prm.c_out + (int64_t)nb * N + ch * 32) * prm.class_positions + pos;
                    const int co_left = prm.c_out - nb * N - ch * 32;
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        if (k < co_left) pp[(int64_t)k * prm.class_positions] = __uint_as_float(v[k]);
                } else if (valid) {
                    const int co_left = prm.c_out - nb * N - ch * 32;  // real channels in this chunk
                    if (co_left >= 32) {
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            dst[(int64_t)(ch * 32 + k) * plane] = cvt_out<TY>(__uint_as_float(v[k]));
                    } else {
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            if (k < co_left) dst[(int64_t)(ch * 32 + k) * plane] = cvt_out<TY>(__uint_as_float(v[k]));
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) release_acc(acc);
            if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (TWO) cluster_sync_all();  // the leader's MMAs write this CTA's TMEM until both are done
    if (warp == 1) {
        tc_fence_after();
        const uint32_t cols = NACC == 2 ? tmem_cols(N) : tmem_pow2(NACC * N);
        if (TWO) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(cols));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(cols));
    }
    if (PAIR) cluster_sync_all();  // the peer may still multicast into / arrive on this CTA
}

// NCHW (bf16 or fp32) -> NHWC bf16 staging: the channels-last A operand.
// Generic fallback (any HW): 32x32 shared-memory tile transpose.
template <typename TX>
__global__ void nchw_to_nhwc_bf16(const TX *__restrict__ x, __nv_bfloat16 *__restrict__ y, int C, int HW) {
    __shared__ float tile[32][33];
    const int64_t b = blockIdx.z;
    const int hw0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    const TX *xb = x + b * C * (int64_t)HW;
    __nv_bfloat16 *yb = y + b * C * (int64_t)HW;
    for (int k = threadIdx.y; k < 32; k += 8) {
        const int c = c0 + k, hw = hw0 + threadIdx.x;
        if (c < C && hw < HW) {
            if constexpr (sizeof(TX) == 2) tile[k][threadIdx.x] = __bfloat162float(xb[(int64_t)c * HW + hw]);
            else tile[k][threadIdx.x] = xb[(int64_t)c * HW + hw];
        }
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += 8) {
        const int hw = hw0 + k, c = c0 + threadIdx.x;
        if (c < C && hw < HW) yb[(int64_t)hw * C + c] = __float2bfloat16_rn(tile[threadIdx.x][k]);
    }
}

// threads per staging block: 256, fewer for small inputs (batch 1: DCGAN l2 stages 256 tiles,
// which as one 256-thread block ran on a single SM)
inline int staging_block(int64_t nthreads) {
    int tpb = 256;
    while (tpb > 32 && ceil_div(nthreads, tpb) < 2 * 148) tpb /= 2;
    return tpb;
}

// The 8-channel x 8-position tile of staging thread i (flat grid of nthreads = B x HW/8 x
// ceil(C/64) x 8): lane bits 0-2 pick the channel group of a 64-channel block (writes: 8 x 16 B
// contiguous), then position chunks, then channel blocks and samples -- every thread has work
// for any HW (a 256-position x 64-channel block per CTA left 15 of 16 threads idle at HW = 16).
__device__ __forceinline__ bool staging_tile(int C, int HW, int64_t nthreads, int64_t &b, int &c0, int &hw0) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nthreads) return false;
    const int nhc = HW / 8, ncb = (C + 63) / 64;
    const int64_t r = i >> 3;
    const int hc = (int)(r % nhc);
    const int64_t r2 = r / nhc;
    c0 = (int)(r2 % ncb) * 64 + (int)(i & 7) * 8;
    b = r2 / ncb;
    hw0 = hc * 8;
    return c0 < C;
}

// Vectorised path (HW % 8 == 0, C % 8 == 0): each thread (staging_tile) loads an 8-channel x
// 8-position tile with 128-bit loads, transposes it in registers with byte permutes and writes
// 8 x 128-bit channels-last rows; no shared memory.
template <typename TX>
__global__ void __launch_bounds__(256) nchw_to_nhwc_bf16_v8(const TX *__restrict__ x, __nv_bfloat16 *__restrict__ y,
                                                             int C, int HW, int64_t nthreads) {
    int64_t b;
    int c0, hw0;
    if (!staging_tile(C, HW, nthreads, b, c0, hw0)) return;
    const TX *src = x + (b * C + c0) * (int64_t)HW + hw0;
    uint32_t r[8][4];  // r[c][k]: channel c, positions 2k, 2k+1 (bf16 pairs)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if constexpr (sizeof(TX) == 2) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(src + (int64_t)c * HW));
            r[c][0] = v.x; r[c][1] = v.y; r[c][2] = v.z; r[c][3] = v.w;
        } else {
            const float4 a = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)c * HW));
            const float4 bb = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)c * HW + 4));
            __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y), p1 = __floats2bfloat162_rn(a.z, a.w);
            __nv_bfloat162 p2 = __floats2bfloat162_rn(bb.x, bb.y), p3 = __floats2bfloat162_rn(bb.z, bb.w);
            r[c][0] = *reinterpret_cast<uint32_t *>(&p0); r[c][1] = *reinterpret_cast<uint32_t *>(&p1);
            r[c][2] = *reinterpret_cast<uint32_t *>(&p2); r[c][3] = *reinterpret_cast<uint32_t *>(&p3);
        }
    }
    __nv_bfloat16 *dst = y + (b * HW + hw0) * (int64_t)C + c0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        uint4 o;
        uint32_t *op = &o.x;
#pragma unroll
        for (int m = 0; m < 4; ++m)
            op[m] = __byte_perm(r[2 * m][w >> 1], r[2 * m + 1][w >> 1], (w & 1) ? 0x7632 : 0x5410);
        *reinterpret_cast<uint4 *>(dst + (int64_t)w * C) = o;
    }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool igemm_available() { return true; }

// NCHW fp32 -> NHWC fp32 hi/lo planes for the 3xTF32 A operand (hi = TF32(x), lo = TF32(x - hi)).
__device__ __forceinline__ float tf32_round(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__global__ void nchw_to_nhwc_tf32x2(const float *__restrict__ x, float *__restrict__ hi, float *__restrict__ lo, int C,
                                    int HW, int64_t total) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {  // e indexes the NHWC output (coalesced stores)
        const int c = (int)(e % C);
        const int64_t bhw = e / C;
        const int64_t b = bhw / HW, hw = bhw % HW;
        const float v = __ldg(x + (b * C + c) * HW + hw);
        const float h = tf32_round(v);
        hi[e] = h;
        lo[e] = tf32_round(v - h);
    }
}

// NCHW fp32 -> NHWC fp16 hi / lo planes of the 3xFP16 A operand, scaled by 2^k_x (k_x from the
// input's absmax partials, f16split.cuh). Each thread (staging_tile) loads an 8-channel x
// 8-position tile with 128-bit loads, splits it and transposes the fp16 pairs
// in registers (byte permutes) into 8 channels-last 16-byte rows per plane. HW % 8 == 0, C % 8 == 0.
#ifndef SEGB_STAGING_MINB  // four 256-thread blocks per SM (<= 64 registers): ebgan_l5 fp32 0.767 -> 0.712 ms,
#define SEGB_STAGING_MINB 4   // l4 0.628 -> 0.601 (six blocks spill and lose)
#endif
__global__ void __launch_bounds__(256, SEGB_STAGING_MINB) nchw_to_nhwc_f16x2_v8(const float *__restrict__ x, __half *__restrict__ hi,
                                                              __half *__restrict__ lo, int C, int HW, int64_t nthreads,
                                                              const float *__restrict__ partials) {
    __shared__ float scale;
    if (threadIdx.x < 32) {
        float m = 0.f;
        for (int i = threadIdx.x; i < kAbsmaxBlocks; i += 32) m = fmaxf(m, __ldg(partials + i));
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if (threadIdx.x == 0) scale = ldexpf(1.f, f16_scale_exp(m));
    }
    __syncthreads();
    const float sc = scale;
    int64_t b;
    int c0, hw0;
    if (!staging_tile(C, HW, nthreads, b, c0, hw0)) return;
    const float *src = x + (b * C + c0) * (int64_t)HW + hw0;
    uint32_t rh[8][4], rl[8][4];  // [channel][k]: positions 2k, 2k+1 as fp16 pairs
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)c * HW));
        const float4 bb = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)c * HW + 4));
        const float v[8] = {a.x, a.y, a.z, a.w, bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            __half h0, l0, h1, l1;
            split_f16(v[2 * k] * sc, h0, l0);
            split_f16(v[2 * k + 1] * sc, h1, l1);
            rh[c][k] = pack_h2(h0, h1);
            rl[c][k] = pack_h2(l0, l1);
        }
    }
    const int64_t off = (b * HW + hw0) * (int64_t)C + c0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        uint4 oh, ol;
        uint32_t *ph = &oh.x, *pl = &ol.x;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const uint32_t sel = (w & 1) ? 0x7632 : 0x5410;
            ph[m] = __byte_perm(rh[2 * m][w >> 1], rh[2 * m + 1][w >> 1], sel);
            pl[m] = __byte_perm(rl[2 * m][w >> 1], rl[2 * m + 1][w >> 1], sel);
        }
        *reinterpret_cast<uint4 *>(hi + off + (int64_t)w * C) = oh;
        *reinterpret_cast<uint4 *>(lo + off + (int64_t)w * C) = ol;
    }
}

// generic-shape 3xFP16 staging: one element per thread, NHWC-indexed (coalesced stores)
__global__ void nchw_to_nhwc_f16x2(const float *__restrict__ x, __half *__restrict__ hi, __half *__restrict__ lo, int C,
                                   int HW, int64_t total, const float *__restrict__ partials) {
    __shared__ float scale;
    if (threadIdx.x < 32) {
        float m = 0.f;
        for (int i = threadIdx.x; i < kAbsmaxBlocks; i += 32) m = fmaxf(m, __ldg(partials + i));
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if (threadIdx.x == 0) scale = ldexpf(1.f, f16_scale_exp(m));
    }
    __syncthreads();
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % C);
        const int64_t bhw = e / C;
        const int64_t b = bhw / HW, hw = bhw % HW;
        __half h, l;
        split_f16(__ldg(x + (b * C + c) * HW + hw) * scale, h, l);
        hi[e] = h;
        lo[e] = l;
    }
}

// Split-K reduction: every output element once, the ksplit partials of its class position summed
// in ascending split order (a fixed order: bitwise reproducible), converted to the output type.
template <typename TY>
__global__ void splitk_reduce_kernel(const float *__restrict__ partial, TY *__restrict__ y, int ksplit, int c_out,
                                     int oh, int ow, int rows, int cols, int swap, int64_t class_positions,
                                     int64_t total) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int yy = (int)(e % ow);
        const int64_t r1 = e / ow;
        const int x = (int)(r1 % oh);
        const int64_t r2 = r1 / oh;
        const int co = (int)(r2 % c_out);
        const int64_t b = r2 / c_out;
        // output (x, y) belongs to class (r, s) = ((x + swap) & 1, (y + swap) & 1) at (x / 2, y / 2)
        const int c = 2 * ((x + swap) & 1) + ((yy + swap) & 1);
        const int64_t pos = (b * rows + (x >> 1)) * cols + (yy >> 1);
        float acc = 0.f;
        for (int ks = 0; ks < ksplit; ++ks)
            acc += __ldcs(partial + ((int64_t)(ks * 4 + c) * c_out + co) * class_positions + pos);
        y[e] = cvt_out<TY>(acc);
    }
}

static int fp32_mode(const IgemmShape &s) {
    if (s.compute != SEGB_F32) return kModeBf16;
    return s.f16x3 ? kModeF16x3 : kModeTf32x3;
}

static bool make_params(const IgemmShape &s, IgemmParams &prm) {
    const int mode = fp32_mode(s);
    const bool tf32 = mode != kModeBf16;  // three-pass operands (hi / lo planes)
    if (s.n % 2 != 0) return false;  // all four classes share one grid
    if (mode == kModeF16x3) {
        // any c_out: a narrow output (dcgan_l5's 3 channels) pads N to 32 on the tensor cores, still
        // faster than the FFMA direct kernel at every batch (small batches: many more CTAs)
        if (s.c_in < 64 || s.c_in % 8 != 0) return false;
        if (s.x_dtype != SEGB_F32 || s.y_dtype != SEGB_F32) return false;
    } else if (tf32) {
        if (s.c_in < 32 || s.c_in % 4 != 0) return false;
        if (s.c_out < 16) return false;  // >2x padded N x 3 passes: the FFMA direct kernel is faster
        if (s.x_dtype != SEGB_F32 || s.y_dtype != SEGB_F32) return false;
    } else {
        if (s.c_in < 64 || s.c_in % 8 != 0) return false;
        if (s.x_dtype != SEGB_BF16 && s.x_dtype != SEGB_F32) return false;
        if (s.y_dtype != SEGB_BF16 && s.y_dtype != SEGB_F32) return false;
    }
    const int cop = s.c_out_pad ? s.c_out_pad : (int)ceil_div(s.c_out, 32) * 32;
    if (s.batch > 65535) return false;
    const int oh = 2 * s.h + 2 * s.pad - s.n, ow = 2 * s.w + 2 * s.pad - s.n;
    if (oh < 2 || ow < 2) return false;
    const int p = s.pad / 2, swap = s.pad & 1;
    prm = IgemmParams{};
    for (int c = 0; c < 4; ++c) {
        const int r = c >> 1, q = c & 1;
        ClassGeom &g = prm.cls[c];
        g.R = sub_len(s.n, r);
        g.C = sub_len(s.n, q);
        g.st_r = (r + swap) % 2;
        g.st_s = (q + swap) % 2;
        g.rows = (oh - g.st_r + 1) / 2;
        g.cols = (ow - g.st_s + 1) / 2;
        g.base_r = (g.st_r + r) / 2;
        g.base_s = (g.st_s + q) / 2;
        g.tap0 = class_offset(s.n, c);
    }
    const int rows = prm.cls[0].rows, cols = prm.cls[0].cols;
    for (int c = 1; c < 4; ++c)
        if (prm.cls[c].rows != rows || prm.cls[c].cols != cols) return false;
    // A box = 128 positions: (cols x rows x samples) rectangle of the class grid
    if (cols >= kBlockM) {
        if (cols % kBlockM) return false;
        prm.box_w = kBlockM; prm.box_h = 1; prm.box_b = 1;
    } else {
        if (kBlockM % cols) return false;
        prm.box_w = cols;
        prm.box_h = std::min(rows, kBlockM / cols);
        if (rows % prm.box_h) return false;
        if (prm.box_h == rows) {
            if (kBlockM % (cols * rows)) return false;
            prm.box_b = kBlockM / (cols * rows);
        } else {
            if (prm.box_w * prm.box_h != kBlockM) return false;
            prm.box_b = 1;
        }
    }
    if (prm.box_b > 256 || prm.box_h > 256 || prm.box_w > 256) return false;
    // N tile over the zero-padded output channels (multiple of 32: the epilogue reads
    // 32-column TMEM chunks); padded channels are computed on zeros and never stored.
    // 3xTF32 stages hold hi and lo tiles of both operands, so its N tile is capped at 128.
    const int nmax = tf32 ? 128 : 256;
    int nt = cop <= nmax ? cop : 0;
    if (!nt)
        for (int cand : {256, 128, 64, 32})
            if (cand <= nmax && cop % cand == 0) { nt = cand; break; }
    // (round 1 used N = 128 for 1024+ output channels; with the current pipeline N = 256 is
    // faster there too: ebgan_l2 bf16 0.222 -> 0.193 ms)
    {  // few position blocks (small batches: DCGAN/EB-GAN l2 at batch 1 has 16 positions per class):
       // narrower N tiles until the four classes' tiles cover the SMs, so the weight stream -- the
       // bytes that bound such a layer -- is read by many SMs at once instead of a handful
        // (2-SM pairs from two position tiles on: count pair tiles against half the 74 pairs -- a
        // wider N tile with most pairs busy beats twice the tiles at half the width: dcgan_l2 at
        // batch 64, N 64 -> 128: 0.040 -> 0.030 ms; dcgan_l3, N 128 -> 256: 0.031 -> 0.028)
        const int64_t mt = ceil_div(s.batch * (int64_t)((oh + 1) / 2) * ((ow + 1) / 2), kBlockM);
        const bool pairs = mt >= 2;
        auto units = [&](int n) { return pairs ? 4 * ((mt + 1) / 2) * (cop / n) : 4 * mt * (cop / n); };
        const int64_t target = pairs ? 37 : 148;
        while (nt > 32 && nt % 64 == 0 && cop % (nt / 2) == 0 && units(nt) < target) nt /= 2;
    }
    if (const char *e = getenv("SEGB200_K3_NTILE")) {  // A/B experiments: force the N tile
        const int v = atoi(e);
        if (v >= 32 && v <= nmax && v % 32 == 0 && cop % v == 0) nt = v;
    }
    // swapped operands (PM 3) for tiny batches: all class positions of the batch (16..128, a
    // multiple of 16) as the N side of one tile, 128-channel weight blocks as the M side
    const int64_t cpos = s.batch * (int64_t)rows * cols;
    // (opt-in, SEGB200_K3_SWAP=1: correct, but measured slower than the narrow-N tiles on DCGAN l2/l3
    // at batch 1 -- 53 vs 21 us for dcgan_l2 bf16 -- so tiny batches keep the output-stationary layout)
    const char *swp = getenv("SEGB200_K3_SWAP");
    if (mode != kModeTf32x3 && cpos <= kTf32MaxN && cpos % 16 == 0 && cop % kBlockM == 0 && rows * cols <= 256 &&
        s.batch <= 256 && swp && atoi(swp)) {
        prm.swap_ab = 1;
        prm.box_w = cols; prm.box_h = rows; prm.box_b = (int)s.batch;
        nt = (int)cpos;
    }
    if (!prm.swap_ab && (nt % 32 || nt > nmax)) return false;
    prm.n_tile = nt;
    prm.n_blocks = prm.swap_ab ? cop / kBlockM : cop / nt;
    prm.batch = (int)s.batch; prm.c_in = s.c_in; prm.c_out = s.c_out; prm.oh = oh; prm.ow = ow; prm.p = p;
    const int kch = mode == kModeTf32x3 ? 32 : 64;
    prm.k_cblocks = (s.c_in + kch - 1) / kch;
    prm.class_positions = s.batch * (int64_t)rows * cols;
    prm.m_tiles = prm.swap_ab ? 1 : (int)ceil_div(prm.class_positions, kBlockM);
    prm.m_pairs = (prm.m_tiles + 1) / 2;
    const int64_t total = 4ll * prm.m_tiles * prm.n_blocks;
    if (total > INT32_MAX) return false;
    prm.total_tiles = (int)total;
    // split K when the tiles cannot cover the SMs (small batches: a weight-streaming layer then runs
    // on a handful of SMs); the partials are summed in a fixed order by splitk_reduce_kernel
    prm.ksplit = 1;
    {
        const int nks = prm.cls[0].R * prm.cls[0].C * prm.k_cblocks;
        // the largest split that still fits one wave (2-SM pairs, the default from two position
        // tiles on: 74 slots of pair tiles; else 148): one more tile per slot would double the
        // critical path (DCGAN l2 at batch 1: split 3 = 192 tiles on 148 SMs 21 us, split 2 ...)
        const bool pairs = prm.m_tiles >= 2 && !prm.swap_ab;
        const int64_t units = pairs ? 4ll * ((prm.m_tiles + 1) / 2) * prm.n_blocks : total;
        const int64_t slots = pairs ? 74 : 148;
        if (2 * units <= slots && nks >= 8)
            prm.ksplit = (int)std::max<int64_t>(1, std::min<int64_t>({8, nks / 4, slots / units}));
        if (const char *e = getenv("SEGB200_K3_KSPLIT")) {  // A/B experiments
            const int v = atoi(e);
            if (v >= 1 && v <= 16 && v <= nks) prm.ksplit = v;
        }
        prm.total_tiles *= prm.ksplit;
    }
    const int stage_bytes = (tf32 ? 2 : 1) * (kBlockM * 128 + nt * 128);
    prm.stages = std::min(8, (int)((227 * 1024 - 1024 - 256) / stage_bytes));
    return prm.stages >= 2;
}

static bool use_rows(const IgemmShape &s) {
    const char *e = getenv("SEGB200_IGEMM_GENERIC");
    return (s.compute == SEGB_BF16 || (s.compute == SEGB_F32 && s.f16x3)) && !(e && atoi(e)) &&
           igemm_rows_supported(s);
}

bool igemm_supported(const IgemmShape &s) {
    IgemmParams prm;
    return igemm_scatter_supported(s) || use_rows(s) || (make_params(s, prm) && tensor_map_encoder() != nullptr);
}

const char *igemm_kernel_name(const IgemmShape &s) {
    // the family, the operand mode and the tile configuration (a different N tile, split or pair
    // layout changes the summation bits, so the name says which one ran)
    static thread_local std::string name;
    char buf[160];
    if (igemm_scatter_supported(s)) return "K3c scatter-GEMM + gather (bf16)";
    if (use_rows(s)) {
        const int ns = igemm_rows_variant(s);
        snprintf(buf, sizeof buf, "K3b row-streaming GEMM (%s%s)%s", s.compute != SEGB_F32 ? "bf16" : "3xFP16",
                 s.compute == SEGB_F32 && s.c_in > 64 ? ", 64-channel passes" : "",
                 ns == 3 || ns == 4 ? " [2-SM pairs]" : ns == 2 ? " [row-parity CTA pairs]" : "");
        name = buf;
        return name.c_str();
    }
    const int mode = fp32_mode(s);
    if (mode == kModeBf16 && igemm_cp_supported(s)) return "K3p class-pair GEMM (bf16)";
    IgemmParams prm;
    if (!make_params(s, prm)) return "K3 implicit GEMM (unsupported shape)";
    const char *pm_env = getenv("SEGB200_K3_PAIR");
    const int pm = prm.swap_ab ? 3 : prm.m_tiles < 2 ? 0 : pm_env ? std::max(0, std::min(2, atoi(pm_env))) : 2;
    snprintf(buf, sizeof buf, "K3 implicit GEMM (%s%s) [N %d%s%s]",
             mode == kModeF16x3 ? "3xFP16" : mode == kModeTf32x3 ? "3xTF32" : "bf16",
             prm.swap_ab ? ", swapped operands" : "", prm.n_tile,
             pm == 2 ? ", 2-SM pairs" : pm == 1 ? ", multicast pairs" : "",
             prm.ksplit > 1 ? (std::string(", split K ") + std::to_string(prm.ksplit)).c_str() : "");
    name = buf;
    return name.c_str();
}

// K3's only workspace: the channels-last A operand (bf16, or fp32 hi followed by fp32 lo for
// 3xTF32), written by the staging launch and read by the GEMM. K3b and K3c's own kernels take
// none from here (K3c's tap products are counted by igemm_scatter_workspace_bytes).
int64_t igemm_workspace_bytes(const IgemmShape &s) {
    if (igemm_scatter_supported(s)) return igemm_scatter_workspace_bytes(s);
    if (use_rows(s)) return igemm_rows_workspace_bytes(s);
    const int mode = fp32_mode(s);
    const int64_t elems = s.batch * (int64_t)s.c_in * s.h * s.w;
    const int64_t bpe = mode == kModeTf32x3 ? 8 : (mode == kModeF16x3 ? 4 : 2);  // bytes per element, all planes
    IgemmParams prm;
    int64_t split = 0;  // split K: fp32 partials of every class position and channel per split
    if (make_params(s, prm) && prm.ksplit > 1)
        split = ((int64_t)prm.ksplit * 4 * s.c_out * prm.class_positions * 4 + 255) / 256 * 256;
    // the A planes, the absmax partials, the split-K partials
    return (elems * bpe + 255) / 256 * 256 + (mode == kModeF16x3 ? kAbsmaxBytes : 0) + split;
}

static int encode_map(CUtensorMap *m, CUtensorMapDataType dt, int rank, const void *ptr, const cuuint64_t *dims,
                      const cuuint64_t *strides, const cuuint32_t *box, const char *what) {
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = tensor_map_encoder()(m, dt, rank, const_cast<void *>(ptr), dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? SEGB_OK : fail(SEGB_ERR_CUDA, "tensor map %s: error %d", what, (int)r);
}

template <typename TY, int MODE, int PM>
static int launch_k3(unsigned grid, size_t smem, cudaStream_t st, const CUtensorMap &tmA, const CUtensorMap &tmB,
                     const CUtensorMap &tmAlo, const CUtensorMap &tmBlo, const IgemmParams &prm) {
    auto kern = igemm_tconv_kernel<TY, MODE, PM>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (PM == 0 || PM == 3) {
        kern<<<grid, kThreads, smem, st>>>(tmA, tmB, tmAlo, tmBlo, prm);
        return SEGB_OK;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmAlo, tmBlo, prm);
    return e == cudaSuccess ? SEGB_OK : fail(SEGB_ERR_CUDA, "igemm_tconv_kernel (pair): %s", cudaGetErrorString(e));
}

int run_igemm(const IgemmShape &s, const void *x, const void *wg, const void *wg_lo, void *y, void *ws,
              int64_t ws_bytes, cudaStream_t st) {
    if (use_rows(s)) return run_igemm_rows(s, x, wg, wg_lo, y, ws, ws_bytes, st);
    IgemmParams prm;
    if (!make_params(s, prm)) return fail(SEGB_ERR_UNSUPPORTED, "implicit GEMM: unsupported shape");
    if (!tensor_map_encoder()) return fail(SEGB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int mode = fp32_mode(s);
    const bool tf32 = mode != kModeBf16;  // hi / lo planes
    const int64_t elems = s.batch * (int64_t)s.c_in * s.h * s.w;
    const int esz = mode == kModeTf32x3 ? 4 : 2;
    void *xs = ws;  // channels-last A operand in the caller's workspace
    if (!xs || ws_bytes < igemm_workspace_bytes(s))
        return fail(SEGB_ERR_VALUE, "implicit GEMM: workspace of %lld bytes needed, got %lld",
                    (long long)igemm_workspace_bytes(s), (long long)ws_bytes);
    void *xs_lo = tf32 ? (void *)((char *)xs + elems * esz) : nullptr;
    float *partials = mode == kModeF16x3 ? (float *)((char *)xs + (2 * elems * esz + 255) / 256 * 256) : nullptr;
    {
        const int hw = s.h * s.w;
        if (mode == kModeF16x3) {
            if (int rc = run_absmax_partials(x, SEGB_F32, elems, partials, st)) return rc;
            if (hw % 8 == 0 && s.c_in % 8 == 0) {
                const int64_t nth = s.batch * (hw / 8) * ceil_div(s.c_in, 64) * 8;
                const int tpb = staging_block(nth);
                nchw_to_nhwc_f16x2_v8<<<(unsigned)ceil_div(nth, tpb), tpb, 0, st>>>(
                    (const float *)x, (__half *)xs, (__half *)xs_lo, s.c_in, hw, nth, partials);
            } else {
                const unsigned g = (unsigned)std::min<int64_t>(ceil_div(elems, 256), 148 * 64);
                nchw_to_nhwc_f16x2<<<g, 256, 0, st>>>((const float *)x, (__half *)xs, (__half *)xs_lo, s.c_in, hw, elems,
                                                      partials);
            }
        } else if (tf32) {
            const unsigned g = (unsigned)std::min<int64_t>(ceil_div(elems, 256), 148 * 64);
            nchw_to_nhwc_tf32x2<<<g, 256, 0, st>>>((const float *)x, (float *)xs, (float *)xs_lo, s.c_in, hw, elems);
        } else if (hw % 8 == 0 && s.c_in % 8 == 0) {
            const int64_t nth = s.batch * (hw / 8) * ceil_div(s.c_in, 64) * 8;
            const int tpb = staging_block(nth);
            const unsigned grd = (unsigned)ceil_div(nth, tpb);
            if (s.x_dtype == SEGB_BF16)
                nchw_to_nhwc_bf16_v8<__nv_bfloat16><<<grd, tpb, 0, st>>>((const __nv_bfloat16 *)x,
                                                                         (__nv_bfloat16 *)xs, s.c_in, hw, nth);
            else
                nchw_to_nhwc_bf16_v8<float><<<grd, tpb, 0, st>>>((const float *)x, (__nv_bfloat16 *)xs, s.c_in, hw,
                                                                 nth);
        } else {
            dim3 blk(32, 8), grd((unsigned)ceil_div(hw, 32), (unsigned)ceil_div(s.c_in, 32), (unsigned)s.batch);
            if (s.x_dtype == SEGB_BF16)
                nchw_to_nhwc_bf16<__nv_bfloat16><<<grd, blk, 0, st>>>((const __nv_bfloat16 *)x, (__nv_bfloat16 *)xs,
                                                                       s.c_in, hw);
            else
                nchw_to_nhwc_bf16<float><<<grd, blk, 0, st>>>((const float *)x, (__nv_bfloat16 *)xs, s.c_in, hw);
        }
        note_launch();
        if (int rc = check_launch("nchw->nhwc staging")) return rc;
    }
    if (!tf32 && igemm_cp_supported(s)) {  // K3p: both column parities per tile
        return run_igemm_cp_core(s, xs, wg, y, st);
    }
    const int kch = mode == kModeTf32x3 ? 32 : 64;
    const CUtensorMapDataType dt = mode == kModeTf32x3 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : mode == kModeF16x3 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                        : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const int cin_pad = mode == kModeTf32x3 ? s.c_in_pad32 : s.c_in_pad;
    CUtensorMap tmA, tmB, tmAlo, tmBlo;
    cuuint64_t adims[4] = {(cuuint64_t)s.c_in, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)s.batch};
    cuuint64_t astr[3] = {(cuuint64_t)s.c_in * esz, (cuuint64_t)s.w * s.c_in * esz, (cuuint64_t)s.h * s.w * s.c_in * esz};
    cuuint32_t abox[4] = {(cuuint32_t)kch, (cuuint32_t)prm.box_w, (cuuint32_t)prm.box_h, (cuuint32_t)prm.box_b};
    cuuint64_t bdims[3] = {(cuuint64_t)cin_pad, (cuuint64_t)s.c_out_pad, (cuuint64_t)s.n * s.n};
    cuuint64_t bstr[2] = {(cuuint64_t)cin_pad * esz, (cuuint64_t)s.c_out_pad * cin_pad * esz};
    // CTA pairs: pm = 2 runs two position blocks as one 2-SM MMA (cta_group::2, M = 256, half
    // of the B tile per CTA: more pipeline stages, half the weight traffic); pm = 1 multicasts B
    // to two single-SM MMAs. Measured with the branch-free MMA warp (profiles/README.md): pm = 2
    // is fastest for every GAN layer in bf16 and 3xTF32, so it is the default.
    // SEGB200_K3_PAIR=0/1/2 overrides (A/B experiments).
    const char *pm_env = getenv("SEGB200_K3_PAIR");
    int pm = pm_env ? std::max(0, std::min(2, atoi(pm_env))) : 2;
    if (prm.m_tiles < 2) pm = 0;
    if (prm.swap_ab) pm = 3;
    const bool pair = pm == 1 || pm == 2;
    if (pair) prm.total_tiles = 4 * prm.m_pairs * prm.n_blocks * prm.ksplit;
    {
        const int64_t bpe = mode == kModeTf32x3 ? 8 : (mode == kModeF16x3 ? 4 : 2);  // all A planes
        prm.partial = prm.ksplit > 1 ? (float *)((char *)ws + (elems * bpe + 255) / 256 * 256 +
                                                (mode == kModeF16x3 ? kAbsmaxBytes : 0))
                                     : nullptr;
    }
    {  // stages: TWO holds only half of the B tile per CTA
        const int b_cta = (pm == 2 ? prm.n_tile / 2 : prm.n_tile) * 128;
        const int stage_bytes = (tf32 ? 2 : 1) * (kBlockM * 128 + b_cta);
        prm.stages = std::min(8, (int)((227 * 1024 - 1024 - 256) / stage_bytes));
    }
    cuuint32_t bbox[3] = {(cuuint32_t)kch,
                          (cuuint32_t)(prm.swap_ab ? kBlockM : (pair ? prm.n_tile / 2 : prm.n_tile)), 1};
    int rc = encode_map(&tmA, dt, 4, xs, adims, astr, abox, "A");
    if (!rc) rc = encode_map(&tmB, dt, 3, wg, bdims, bstr, bbox, "B");
    if (!rc && tf32) rc = encode_map(&tmAlo, dt, 4, xs_lo, adims, astr, abox, "A lo");
    if (!rc && tf32) rc = encode_map(&tmBlo, dt, 3, wg_lo, bdims, bstr, bbox, "B lo");
    if (rc) return rc;
    if (!tf32) { tmAlo = tmA; tmBlo = tmB; }
    prm.y = y;
    prm.x_partials = partials;
    prm.w_unscale = ldexpf(1.f, -s.w_exp);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t b_cta = (size_t)(pm == 2 ? prm.n_tile / 2 : prm.n_tile) * 128;
    const size_t stage_bytes = (size_t)(tf32 ? 2 : 1) * ((size_t)kBlockM * 128 + b_cta);
    const size_t smem = 1024 + prm.stages * stage_bytes + (2 * prm.stages + 8) * 8 + 16;  // up to 4 TMEM buffers
    const unsigned grid = pair ? 2 * (unsigned)std::min<int64_t>(prm.total_tiles, sms / 2)
                               : (unsigned)std::min<int64_t>(prm.total_tiles, sms);
#define SEGB_K3_LAUNCH(TY_, TF_)                                                                       \
    rc = pm == 3   ? launch_k3<TY_, TF_, 3>(grid, smem, st, tmA, tmB, tmAlo, tmBlo, prm)                \
         : pm == 2 ? launch_k3<TY_, TF_, 2>(grid, smem, st, tmA, tmB, tmAlo, tmBlo, prm)                \
         : pm == 1 ? launch_k3<TY_, TF_, 1>(grid, smem, st, tmA, tmB, tmAlo, tmBlo, prm)                \
                   : launch_k3<TY_, TF_, 0>(grid, smem, st, tmA, tmB, tmAlo, tmBlo, prm);
    if (mode == kModeF16x3) {
        SEGB_K3_LAUNCH(float, kModeF16x3)
    } else if (mode == kModeTf32x3) {
        SEGB_K3_LAUNCH(float, kModeTf32x3)
    } else if (s.y_dtype == SEGB_BF16) {
        SEGB_K3_LAUNCH(__nv_bfloat16, kModeBf16)
    } else {
        SEGB_K3_LAUNCH(float, kModeBf16)
    }
#undef SEGB_K3_LAUNCH
    if (rc) return rc;
    note_launch();
    if (int e = check_launch("igemm_tconv_kernel")) return e;
    if (prm.ksplit > 1) {
        const int64_t total = s.batch * (int64_t)s.c_out * prm.oh * prm.ow;
        const unsigned g = (unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
        const ClassGeom &g0 = prm.cls[0];
        if (s.y_dtype == SEGB_BF16)
            splitk_reduce_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(prm.partial, (__nv_bfloat16 *)y, prm.ksplit,
                                                                   s.c_out, prm.oh, prm.ow, g0.rows, g0.cols,
                                                                   s.pad & 1, prm.class_positions, total);
        else
            splitk_reduce_kernel<float><<<g, 256, 0, st>>>(prm.partial, (float *)y, prm.ksplit, s.c_out, prm.oh, prm.ow,
                                                           g0.rows, g0.cols, s.pad & 1, prm.class_positions, total);
        note_launch();
        return check_launch("splitk_reduce_kernel");
    }
    return SEGB_OK;
}

}  // namespace segb
