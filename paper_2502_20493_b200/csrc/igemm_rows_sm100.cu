// K3b -- row-streaming implicit GEMM for wide class grids (cols % 128 == 0),
// e.g. EB-GAN l7 (128x128x64 -> 256x256x64): all four parity classes of one
// class-grid row (128 positions) per tile, weights resident, every input row
// loaded once, output written by TMA.
//
// Same arithmetic as K3 (igemm_sm100.cu, per-class GEMMs of engines.py:271-335)
// with the operand traffic restructured for layers whose K = taps x c_in is
// small and whose output is large (K3's per-tap boxes re-read each input
// element n*n times and the weights once per tile):
//   * weights: every (class, tap, 64-channel block) B tile is TMA-loaded once
//     per CTA and stays resident in shared memory;
//   * activations: four loader warps read NCHW input rows with 128-bit loads
//     (the next row already in flight in registers), transpose 8x8 bf16 tiles
//     with byte permutes and store them into a ring of K-major SWIZZLE_128B
//     "row slots" (slot row = input column, 64 channels = 128 B); columns and
//     rows outside the input -- the floor(P/2) zero ring -- are stored as
//     zeros. No NHWC copy of the input touches HBM;
//   * every A operand is a row-shifted view of a slot: the UMMA descriptor start
//     moves by 128 B per column shift (measured on B200: the SWIZZLE_128B phase
//     follows the absolute smem address, so the base-offset field stays 0);
//   * (class, tap) pairs that read the same shifted window share one MMA: their
//     B tiles are stored contiguously and their TMEM accumulators are adjacent,
//     so e.g. the centre window of a 4x4 / P=2 layer feeds all four classes in a
//     single N = 4*c_out MMA (11 MMAs per k-step instead of 16, 40% less smem
//     operand traffic);
//   * consecutive class-grid rows of a strip share nr - 1 of their nr input rows;
//   * epilogue: four warps (TMEM lane quarters) turn the four class accumulators
//     of a position into bf16 pairs (output columns 2j, 2j+1) and store both
//     output rows with coalesced 4-byte stores (128 B per warp instruction),
//     the next channels' TMEM loads in flight; every output element written once.
//
// Warps: 0 weight TMA, 1 MMA issuer (+TMEM owner), 2..3 idle, 4..7 epilogue (TMEM lane
// quarters), 8..11 row loaders / transposers (registers rebalanced, see kRegsLoad).
#include <cstdlib>
#include <mutex>

#include "f16split.cuh"
#include "igemm.cuh"
#include "tc_ptx.cuh"

namespace segb {

static unsigned long long *g_rows_prof_buf = nullptr;
constexpr int kRowsEpw = 4;  // epilogue warps, one per TMEM lane quarter (8 measured slower: spills)
// Three warpgroups with rebalanced registers (setmaxnreg): warpgroup 0 = weight TMA (warp 0),
// MMA issuer (warp 1), two idle warps, shrunk to kRegsCtl registers; warpgroup 1 = the four
// epilogue warps (TMEM lane quarter warp % 4), kept at the launch budget; warpgroup 2 = the
// four row loaders, grown to kRegsLoad registers so each thread can keep up to 5 input units in
// flight (SEGB_ROWS_LOAD_BUFS; measured: 3 is as fast as 4 or 5 on l6/l7).
constexpr int kEpiWarp0 = 4;
constexpr int kLoaderWarp0 = 8;                               // first of the 4 row-loader warps
constexpr int kRowsThreads = 12 * 32;                         // launch budget: 168 registers
constexpr int kRegsCtl = 96, kRegsLoad = 232;                 // 128 x (96 + 168 + 232) <= 64 K
// 3xFP16: the epilogue holds a whole tile's accumulators (4 classes x 32 columns) at once
#ifndef SEGB_ROWS_BF16_STCS  // the same for the bf16 epilogue
#define SEGB_ROWS_BF16_STCS 1  // measured: ebgan_l7 bf16 0.577 -> 0.567 ms
#endif
#ifndef SEGB_ROWS_F16_RED  // later channel passes add into y with L2 vector atomics (no read-back)
#define SEGB_ROWS_F16_RED 1  // measured: ebgan_l6 fp32 0.969 -> 0.938 ms (the add flushes subnormal sums)
#endif
__device__ __forceinline__ void red_add_f32x2(float *p, float2 v) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
#ifndef SEGB_ROWS_F16_STCS
#define SEGB_ROWS_F16_STCS 1  // measured: ebgan_l7 fp32 1.728 -> 1.681 ms, l6 0.976 -> 0.964
#endif
#ifndef SEGB_ROWS_F16_ST16  // 3xFP16 epilogue stores: 16-byte (lane-pair exchange) or two 8-byte per channel
#define SEGB_ROWS_F16_ST16 0  // measured: 8-byte stores without exchange -3.5% (l7), -8% (l6) vs 16-byte
#endif
// (the 16-byte store variant keeps the read-modify-write accumulation)
static_assert(!(SEGB_ROWS_F16_ST16 && SEGB_ROWS_F16_RED), "SEGB_ROWS_F16_ST16 needs SEGB_ROWS_F16_RED=0");
constexpr int kRegsLoadF16 = 192, kRegsEpiF16 = 216;          // 128 x (96 + 216 + 192) <= 128 x 3 x 168
constexpr int kRingMax = 8;         // input-row slots: as many as shared memory holds, <= 8
// 3xFP16 loaders hand each filled slot to an "arriver" warp (warp 2) through a named barrier;
// the arriver's cluster-scope release arrive then has no outstanding global loads to wait for
// (a release arrive from a loader lane waited for the next units' loads in flight: 1850 cycles
// per unit on ebgan_l7, and the register pipelining of the loads collapsed to one unit)
#ifndef SEGB_ROWS_ARRIVER
#define SEGB_ROWS_ARRIVER 1
#endif
// (loaders and arriver both bar.sync on named barrier 1; measured: loaders that only bar.arrive on
// one barrier per slot, not waiting for the arriver, +1.5% on ebgan_l7)
#ifndef SEGB_ROWS_ARRIVER_BF16  // the same for the bf16 loaders (M = 64 pairs: one barrier per channel-block half)
#define SEGB_ROWS_ARRIVER_BF16 1
#endif
constexpr int kArriverWarp = 2;
constexpr int kSlotBar0 = 1;
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

#ifndef SEGB_ROWS_LOAD_BUFS
#define SEGB_ROWS_LOAD_BUFS 3
#endif
constexpr int kLoadBufs = SEGB_ROWS_LOAD_BUFS;  // input-row units in flight per loader thread

struct RowsClass {
    int st_r, st_s, base_r, base_s, tap0;
};

struct RowsParams {
    RowsClass cls[4];
    int c_in, c_out, h, w, oh, ow, p;
    int rows, msub;  // class-grid rows, 128-position subtiles per row
    int dmin_r, nr;  // first window row offset, input rows per class-grid row (all four classes)
    int dminr_rs[2]; // first window row offset of the classes of row parity r (RS = 2)
    int dmin_c, slot_rows;
    int total_tiles, tiles_per_cta;
    uint32_t slot_bytes, b_tile_bytes;
    int ring;  // input-row slots in the ring (nr <= ring <= kRingMax)
    int half_tiles;  // RS = 3: tiles of one half of the batch (CTA r of a pair takes half r)
    const void *x;
    void *y;
    unsigned long long *prof;  // optional role cycle counters (CTA 0), SEGB200_PROFILE=1
    int ablate;                // SEGB200_ABLATE bits, see ABL()
    // F16 (3xFP16, fp32 in / out): every slot and weight tile holds an fp16 hi plane and a lo
    // plane (f16split.cuh); the input's scale comes from its absmax partials
    uint32_t slot_plane, b_plane;  // byte offset of the lo plane in a slot / in the weight area
    const float *x_partials;
    float w_unscale;               // 2^-k_w of the weight planes
    int ch_base;                   // F16: first input channel of this pass (c_in > 64 runs 64-channel passes)
    int accumulate;                // F16: add this pass's sums to y (passes after the first)
};

// Role ablation for bottleneck experiments, compiled in only with -DSEGB_ROWS_ABLATION
// (SEGB200_ABLATE bit mask: 1 no output stores, 2 no input loads, 4 no MMAs, 8 no TMEM reads,
// 16 no slot stores, 32 no TMEM handshake, 64 no slot handshake). Results are garbage then.
#ifdef SEGB_ROWS_ABLATION
#define ABL(bit) (prm.ablate & (bit))
#else
#define ABL(bit) 0
#endif

// role counters: [0] MMA wait tempty, [1] MMA wait slots, [2] MMA issue, [3] epi wait tfull,
// [4] epi TMEM+convert, [5] epi staging+store, [6] loader wait empty, [7] loader work, [8] tiles
// (compiled in only with -DSEGB_ROWS_PROFILE: its divergent branches cost the MMA warp its
// uniform-register descriptor arithmetic)
#ifdef SEGB_ROWS_PROFILE
#define ROWS_PROF(idx, t0_)                                                                 \
    if (prm.prof && blockIdx.x == 0) {                                                       \
        const long long _n = clock64();                                                      \
        if ((threadIdx.x & 31) == 0) atomicAdd(&prm.prof[idx], (unsigned long long)(_n - t0_)); \
        t0_ = _n;                                                                            \
    }
#else
#define ROWS_PROF(idx, t0_)
#endif

// ---------------------------------------------------------------------------
// Compile-time MMA schedule for even n = 2*NH: A window (du, dc) of the slot
// ring is shared by the classes (r, s) with 0 <= du - base_r < NH and
// 0 <= dc - base_s < NH (base = parity when P is even, 0 when P is odd).
// RSEL < 0: all four classes (du relative to the union row window);
// RSEL = r: only the two classes of row parity r (du = tap row u).
struct MmaGroup {
    int du, dc, c0, nc, b0;  // window, first TMEM class slot, slot count, first B tile
};
template <int NH, int SWAP, int RSEL>
struct Schedule {
    MmaGroup g[(NH + 1) * (NH + 1) * 2];
    int count = 0;
    int ntiles = 0;    // B tiles (one per included (class, tap))
    int btap[16 * 4];  // B tile k -> (class << 8) | (u << 4) | v
    bool fresh[(NH + 1) * (NH + 1) * 2];
};
// TMEM slot of class c = 2r + s when all four classes share a buffer: [0, 1, 3, 2] puts (0, 1)
// next to (1, 1), so the window both row parities read with column parity 1 becomes one N = 2 c_out
// MMA (10 instead of 11 MMAs per k-step for n = 4, P even). The permutation is its own inverse.
#ifndef SEGB_ROWS_CLASS_PERM
#define SEGB_ROWS_CLASS_PERM 1
#endif
__host__ __device__ constexpr int class_slot(int c) { return SEGB_ROWS_CLASS_PERM ? (c < 2 ? c : 5 - c) : c; }

template <int NH, int SWAP, int RSEL>
constexpr Schedule<NH, SWAP, RSEL> make_schedule() {
    Schedule<NH, SWAP, RSEL> s{};
    const int W = SWAP ? NH : NH + 1;  // distinct column windows (and row windows for RSEL < 0)
    const int DU = RSEL < 0 ? W : NH;
    auto slot = [](int c) { return RSEL < 0 ? class_slot(c) : c; };
    int nb = 0;
    // one MMA over TMEM slots p0 .. p0 + nc - 1 (their classes in slot order)
    auto add = [&](int du, int dc, int p0, int nc) {
        s.g[s.count] = MmaGroup{du, dc, p0, nc, nb};
        for (int p = p0; p < p0 + nc; ++p) {
            const int c = slot(p);  // the permutation is an involution
            const int r = c >> 1, q = c & 1;
            const int u = RSEL < 0 ? du - (SWAP ? 0 : r) : du, v = dc - (SWAP ? 0 : q);
            s.btap[nb++] = (c << 8) | (u << 4) | v;
        }
        s.count++;
    };
    // windows feeding every included class first, so one MMA initialises all accumulators
    for (int pass = 0; pass < 2; ++pass)
        for (int du = 0; du < DU; ++du)
            for (int dc = 0; dc < W; ++dc) {
                bool rr[2] = {false, false}, ss[2] = {false, false};
                for (int r = 0; r < 2; ++r) {
                    const int u = du - (SWAP ? 0 : r), v = dc - (SWAP ? 0 : r);
                    rr[r] = RSEL < 0 ? (u >= 0 && u < NH) : (r == RSEL);
                    ss[r] = v >= 0 && v < NH;
                }
                const bool all_r = RSEL < 0 ? (rr[0] && rr[1]) : true;
                const bool full = all_r && ss[0] && ss[1];
                if ((pass == 0) != full) continue;
                if (full) {
                    if (RSEL < 0) add(du, dc, 0, 4);
                    else add(du, dc, 2 * RSEL, 2);
                    continue;
                }
                // both row parities, one column parity q: classes q and 2 + q, one MMA when
                // their slots are adjacent
                if (RSEL < 0 && all_r && ss[0] != ss[1]) {
                    const int q = ss[1] ? 1 : 0;
                    const int a = slot(q), b = slot(2 + q);
                    if (a + 1 == b || b + 1 == a) {
                        add(du, dc, a < b ? a : b, 2);
                        continue;
                    }
                }
                for (int r = 0; r < 2; ++r) {
                    if (!rr[r]) continue;
                    if (ss[0] && ss[1]) {  // both column parities of row r: slots adjacent either way
                        const int a = slot(2 * r), b = slot(2 * r + 1);
                        add(du, dc, a < b ? a : b, 2);
                    } else {
                        for (int q = 0; q < 2; ++q)
                            if (ss[q]) add(du, dc, slot(2 * r + q), 1);
                    }
                }
            }
    s.ntiles = nb;
    bool touched[4] = {false, false, false, false};
    for (int i = 0; i < s.count; ++i) {
        s.fresh[i] = !touched[s.g[i].c0];
        for (int c = s.g[i].c0; c < s.g[i].c0 + s.g[i].nc; ++c) touched[c] = true;
    }
    return s;
}

struct RowsSmem {  // byte offsets from the 1024-aligned smem base
    uint32_t b, ring, bars, total;
};

__host__ __device__ inline RowsSmem rows_layout(const RowsParams &p, int ntaps, int kbc) {
    RowsSmem s;
    s.b = 0;
    s.ring = s.b + ntaps * kbc * p.b_tile_bytes * (p.b_plane ? 2 : 1);  // F16: hi and lo weight planes
    s.bars = s.ring + p.ring * kbc * p.slot_bytes;
    s.total = s.bars + (1 + 2 * p.ring * kbc + 8) * 8 + 16;  // b_full, slots, 4 tfull + 4 tempty, TMEM addr
    return s;
}

// number of input-row loads a tile triggers (nr when it starts a strip, else 1)
__device__ __forceinline__ int tile_loads(const RowsParams &p, int t, int t0) {
    return (t == t0 || (t % p.rows) == 0) ? p.nr : 1;
}


// epilogue TMEM chunk: 8 fp32 columns per class per tcgen05.ld (c_out is a multiple of 16)
#ifndef SEGB_ROWS_EPI_CHUNK
#define SEGB_ROWS_EPI_CHUNK 8
#endif
constexpr int kEpiChunk = SEGB_ROWS_EPI_CHUNK;
__device__ __forceinline__ void tmem_ld_chunk(uint32_t taddr, uint32_t (&v)[kEpiChunk]) {
    if constexpr (kEpiChunk == 16) tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
    else tmem_ld8(taddr, *reinterpret_cast<uint32_t(*)[8]>(&v[0]));
}
__device__ __forceinline__ void reg_fence_chunk(uint32_t (&v)[kEpiChunk]) {
#pragma unroll
    for (int k = 0; k < kEpiChunk; k += 8) reg_fence8(*reinterpret_cast<uint32_t(*)[8]>(&v[k]));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&v);
}

// MMA issue of one tile for schedule (NH, SWAP, RSEL): the whole warp walks the compile-time
// schedule (uniform values), lane `leader` issues each tcgen05.mma (no per-MMA branch). The channel-block loop
// stays rolled so the unrolled schedule's live state stays small.
// CG = 2: one tcgen05.mma.cta_group::2 for a CTA pair (M = 2 MR); each CTA holds the output-
// channel half of every B tile, so a class's accumulator is N/2 TMEM columns (lanes 0-63: first
// channel half, lanes 64-127: second).
// COSPLIT (with CG = 2, M = 128): the pair's B rows are [first channel halves | second halves],
// so class c's accumulator is N/2 columns in both lane halves; otherwise (M = 256) B rows are
// the group's (class, channel) list split in two and every CTA holds all N columns.
// F16: three MMAs per k-chunk on the scaled fp16 planes, hi*hi + hi*lo + lo*hi (the lo planes
// AP16 / BP16 descriptor units after the hi ones), fp16 instruction descriptors.
template <int NH, int KBC, int SWAP, int MR, int RSEL, int CG = 1, bool COSPLIT = true, bool F16 = false>
__device__ __forceinline__ void issue_tile(uint32_t d0, uint32_t aLo0, uint32_t bLo0, uint32_t sq, uint32_t ring,
                                           uint32_t S16, uint32_t B16, int N, uint32_t leader, uint32_t AP16 = 0,
                                           uint32_t BP16 = 0) {
    constexpr Schedule<NH, SWAP, RSEL> SCH = make_schedule<NH, SWAP, RSEL>();
    constexpr int CB = RSEL < 0 ? 0 : 2 * RSEL;  // first class held in this CTA's TMEM
    constexpr int DU = RSEL < 0 ? (SWAP ? NH : NH + 1) : NH;
    // opaque per-tile copies: keeps ptxas from hoisting all 44 loop-invariant B descriptors out
    // of the tile loop (more than the uniform register file holds; they were spilled to vector
    // registers and re-broadcast with R2UR for every MMA)
    asm volatile("mov.b32 %0, %0;" : "+r"(bLo0));
    asm volatile("mov.b32 %0, %0;" : "+r"(B16));
    asm volatile("mov.b32 %0, %0;" : "+r"(d0));
    // low descriptor word of window row du's slot (channel block 0): the only per-tile values
    uint32_t arow[DU];
#pragma unroll
    for (int du = 0; du < DU; ++du) {
        const uint32_t sl = sq + du >= ring ? sq + du - ring : sq + du;
        arow[du] = aLo0 + sl * KBC * S16;
    }
#pragma unroll 1
    for (int kb = 0; kb < KBC; ++kb) {
#pragma unroll
        for (int gi = 0; gi < SCH.count; ++gi) {
            const MmaGroup g = SCH.g[gi];
            const uint32_t a = arow[g.du] + kb * S16 + g.dc * 8;
            const uint32_t b = bLo0 + (kb * SCH.ntiles + g.b0) * B16;
            const uint32_t idesc = F16 ? idesc_bf16_m(MR * CG, g.nc * N) & ~((1u << 7) | (1u << 10))  // fp16 x fp16
                                       : idesc_bf16_m(MR * CG, g.nc * N);
            const uint32_t d = d0 + (g.c0 - CB) * (COSPLIT ? N / CG : N);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                tc_mma_lo<CG>(d, a + kk * 2, b + kk * 2, idesc, (SCH.fresh[gi] && kb == 0 && kk == 0) ? 0u : 1u,
                              leader);
                if constexpr (F16) {
                    tc_mma_lo<CG>(d, a + kk * 2, b + BP16 + kk * 2, idesc, 1u, leader);
                    tc_mma_lo<CG>(d, a + AP16 + kk * 2, b + kk * 2, idesc, 1u, leader);
                }
            }
        }
    }
}

// TMA loads of the resident weights of schedule (NH, SWAP, RSEL), [kb][tile] order
// (RS = 3: this CTA's output-channel half of every tile, b_tile_bytes = half a tile, counted on
// the leader's barrier, which expects both halves)
template <int NH, int KBC, int SWAP, int RSEL>
__device__ __forceinline__ void load_weights(uint8_t *sB, const CUtensorMap *tmB, uint64_t *bar, const RowsParams &prm,
                                             int pair_rank = -1, bool cosplit = true,
                                             const CUtensorMap *tmBlo = nullptr) {
    // tmBlo (F16): the lo plane's tiles go to the same offsets + prm.b_plane
    constexpr Schedule<NH, SWAP, RSEL> SCH = make_schedule<NH, SWAP, RSEL>();
    const int planes = tmBlo ? 2 : 1;
    if (pair_rank >= 0 && !cosplit) {
        // M = 256 pairs: CTA r holds rows [r N/2, (r+1) N/2) of each group's (class, channel)
        // list, as half tiles: whole tiles of classes c0 + r nc/2 .. (nc >= 2) or the channel
        // half r of the single class (nc = 1); a group's halves start at half tile b0
        const uint32_t lb = mapa_rank(bar, 0);
        if (pair_rank == 0) mbar_expect_tx(bar, 2 * planes * SCH.ntiles * KBC * prm.b_tile_bytes);
#pragma unroll
        for (int gi = 0; gi < SCH.count; ++gi) {
            const MmaGroup g = SCH.g[gi];
#pragma unroll
            for (int j = 0; j < g.nc; ++j) {
                const int k = g.b0 + (g.nc >= 2 ? pair_rank * g.nc / 2 + j / 2 : 0);
                const int co_off = g.nc >= 2 ? (j & 1) * (prm.c_out / 2) : pair_rank * (prm.c_out / 2);
                const int c = SCH.btap[k] >> 8, u = (SCH.btap[k] >> 4) & 15, v = SCH.btap[k] & 15;
                const int tap = prm.cls[c].tap0 + u * NH + v;
                for (int kb = 0; kb < KBC; ++kb)
                    for (int pl = 0; pl < planes; ++pl)
                        tma_load_3d_2sm(sB + pl * prm.b_plane + (kb * SCH.ntiles + g.b0 + j) * prm.b_tile_bytes,
                                        pl ? tmBlo : tmB, lb, prm.ch_base + kb * 64, co_off, tap);
            }
        }
        return;
    }
    if (pair_rank >= 0) {
        const uint32_t lb = mapa_rank(bar, 0);
        if (pair_rank == 0) mbar_expect_tx(bar, 2 * planes * SCH.ntiles * KBC * prm.b_tile_bytes);
#pragma unroll
        for (int k = 0; k < SCH.ntiles; ++k) {
            const int c = SCH.btap[k] >> 8, u = (SCH.btap[k] >> 4) & 15, v = SCH.btap[k] & 15;
            const int tap = prm.cls[c].tap0 + u * NH + v;
            for (int kb = 0; kb < KBC; ++kb)
                for (int pl = 0; pl < planes; ++pl)
                    tma_load_3d_2sm(sB + pl * prm.b_plane + (kb * SCH.ntiles + k) * prm.b_tile_bytes, pl ? tmBlo : tmB,
                                    lb, prm.ch_base + kb * 64, pair_rank * (prm.c_out / 2), tap);
        }
        return;
    }
    mbar_expect_tx(bar, planes * SCH.ntiles * KBC * prm.b_tile_bytes);
#pragma unroll
    for (int k = 0; k < SCH.ntiles; ++k) {
        const int c = SCH.btap[k] >> 8, u = (SCH.btap[k] >> 4) & 15, v = SCH.btap[k] & 15;
        const int tap = prm.cls[c].tap0 + u * NH + v;
        for (int kb = 0; kb < KBC; ++kb)
            for (int pl = 0; pl < planes; ++pl)
                tma_load_3d(sB + pl * prm.b_plane + (kb * SCH.ntiles + k) * prm.b_tile_bytes, pl ? tmBlo : tmB, bar,
                            prm.ch_base + kb * 64, 0, tap);
    }
}

// MR: positions per tile (one class-grid row segment) = the MMA M, 128 or 64 (M=64 keeps its
// accumulator in TMEM lanes 32q + [0,16), q = 0..3). RS = 2 splits the four parity classes
// over a CTA pair by row parity (CTA blockIdx % 2 owns classes (r, 0) and (r, 1)): each CTA
// then holds half the weights, writes one of the two output rows of a tile and issues 6
// instead of 11 MMAs per k-step (GAN n = 4, P = 2).
// RS = 3: a CTA pair (2-CTA cluster) runs one tcgen05.mma.cta_group::2 of M = 2 MR per window
// group: CTA r streams the rows of batch half r into its own ring (identical slot sequence in
// both, so one descriptor addresses both) and holds output-channel half r of every weight tile;
// the leader (rank 0) issues the MMAs; each CTA's TMEM gets its own MR positions with the first
// channel half in lanes 0-63 and the second in lanes 64-127 (MR = 64), so all four epilogue
// warps store full 32-lane rows.
// F16 (3xFP16): fp32 input rows are scaled, split into fp16 hi / lo planes by the loaders, the
// MMA warp issues three MMAs per chunk and the epilogue writes fp32 times 2^-(k_x + k_w).
// FM: 0 = bf16, 1 = 3xFP16 (first channel pass: stores y), 2 = 3xFP16 later pass (adds into y);
// the pass kind is a template parameter so the storing instance carries no accumulate code
template <int NH, int KBC, int SWAP, int MR, int RS, int FM = 0>
__global__ void __launch_bounds__(kRowsThreads, 1)
    igemm_rows_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBlo,
                      const RowsParams prm) {
    constexpr bool F16 = FM != 0;
    constexpr bool ACCP = FM == 2;  // this launch adds its channel block's sums into y
    constexpr bool TWO = RS == 3 || RS == 4;  // 2-SM pair: M = 128 (RS 3, MR 64) or 256 (RS 4, MR 128)
    constexpr bool COSPLIT = RS == 3;
    // RS = 5 (HALF): one CTA, every tile issued as two row-parity halves (schedules RSEL 0, 1)
    // into four half-tile TMEM buffers, so the epilogue drains row 2i while the MMAs of row
    // 2i+1 run and the next tile's first half can start as soon as a half buffer is free
    constexpr bool HALF = RS == 5;
    constexpr int NCL = (RS == 2 || HALF) ? 2 : 4;  // parity classes per accumulator buffer
#ifndef SEGB_ROWS_PAIR_NBUF
#define SEGB_ROWS_PAIR_NBUF 2
#endif
    // TMEM accumulator buffers: F16 (64-position tiles) keeps 4; the bf16 pair (RS 3) is an A/B knob
    constexpr int NBUF = (HALF || F16) ? 4 : (RS == 3 ? SEGB_ROWS_PAIR_NBUF : 2);
    // M = 64 rows with two channel blocks: loader warps 0-1 fill block 0, warps 2-3 block 1 of
    // the same input row at once (else each unit is one (row, block) filled by all four)
    constexpr bool PAIRKB = MR == 64 && KBC == 2;
    constexpr int UKB = PAIRKB ? 1 : KBC;  // channel blocks iterated per row by a loader thread
    constexpr bool ARR = F16 ? SEGB_ROWS_ARRIVER : SEGB_ROWS_ARRIVER_BF16;  // slot hand-off via warp 2
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int rsel = RS == 2 ? (int)(blockIdx.x % 2) : -1;
    const int cta = blockIdx.x / ((RS == 1 || HALF) ? 1 : 2);
    const int rank = TWO ? (int)cluster_ctarank() : 0;
    const int toff = TWO ? rank * prm.half_tiles : 0;  // tile index offset of this CTA's batch half
    const int ntiles_b = (RS == 2 ? 2 : 4) * NH * NH;  // resident B tiles
    const RowsSmem L = rows_layout(prm, ntiles_b, KBC);
    uint8_t *sB = smem + L.b;
    uint8_t *sRing = smem + L.ring;
    uint64_t *b_full = reinterpret_cast<uint64_t *>(smem + L.bars);
    uint64_t *slot_full = b_full + 1;
    const int ring = prm.ring;
    uint64_t *slot_empty = slot_full + ring * KBC;
    uint64_t *tfull = slot_empty + ring * KBC;
    uint64_t *tempty = tfull + NBUF;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + NBUF);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int N = prm.c_out;
    constexpr int CG = TWO ? 2 : 1;
    // this CTA's input-row window per class-grid row
    const int dminr = RS == 2 ? prm.dminr_rs[rsel] : prm.dmin_r;
    const int nr = RS == 2 ? NH : prm.nr;

    if (threadIdx.x == 0) {
        mbar_init(b_full, HALF ? 2 : 1);  // HALF: the two schedules' weights, two expect_tx
        for (int i = 0; i < ring * KBC; ++i) {
            // one arrival per loader warp filling the slot (3xFP16 with the arriver: one per CTA)
            mbar_init(&slot_full[i], (ARR ? 1 : PAIRKB ? 2 : 4) * CG);
            mbar_init(&slot_empty[i], 1);
        }
        for (int i = 0; i < NBUF; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kRowsEpw * CG);  // one arrival per epilogue warp (TWO: of both CTAs)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        if (F16) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmBlo) : "memory");
    }
    const CUtensorMap *tmLo = F16 ? &tmBlo : nullptr;
    const uint32_t tcols = tmem_pow2(NBUF * NCL * N / (COSPLIT ? 2 : 1));  // buffers x NCL classes x N (RS 3: N/2)
    if (warp == 1) {
        if (TWO) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(tcols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(tcols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (TWO) cluster_sync_all();  // both CTAs' barriers initialised before remote arrivals
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int t0 = cta * prm.tiles_per_cta;
    const int t1 = min(TWO ? prm.half_tiles : prm.total_tiles, t0 + prm.tiles_per_cta);
    auto loads_of = [&](int t) { return (t == t0 || (t % prm.rows) == 0) ? nr : 1; };

    // setmaxnreg at the top of each warpgroup's branch (all four warps execute it, and it
    // dominates the code it budgets for)
    if (warp < kEpiWarp0) {
#ifndef SEGB_ROWS_NO_SETMAXNREG
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl));
#endif
        if (warp == 0) {
            if (lane == 0) {  // ---------------- the resident weights, in schedule order
                if (TWO) load_weights<NH, KBC, SWAP, -1>(sB, &tmB, b_full, prm, rank, COSPLIT, tmLo);
                else if (RS == 1) load_weights<NH, KBC, SWAP, -1>(sB, &tmB, b_full, prm, -1, true, tmLo);
                else if (HALF) {  // both row parities' schedules, the second after the first's tiles
                    load_weights<NH, KBC, SWAP, 0>(sB, &tmB, b_full, prm);
                    load_weights<NH, KBC, SWAP, 1>(sB + make_schedule<NH, SWAP, 0>().ntiles * KBC * prm.b_tile_bytes,
                                                   &tmB, b_full, prm);
                } else if (rsel == 0) load_weights<NH, KBC, SWAP, 0>(sB, &tmB, b_full, prm);
                else load_weights<NH, KBC, SWAP, 1>(sB, &tmB, b_full, prm);
            }
        } else if (warp == 1) {
            // ---------------- MMA issuer (TWO: the leader CTA issues for the pair)
            if (!(TWO && rank != 0)) {  // (the peer's MMA warp idles)
            if (TWO) mbar_wait_cluster(b_full, 0);
            else mbar_wait(b_full, 0);
            const uint32_t aLo0 = desc_lo_sw128(smem_u32(sRing)), bLo0 = desc_lo_sw128(smem_u32(sB));
            const uint32_t S16 = prm.slot_bytes >> 4, B16 = prm.b_tile_bytes >> 4;
            const uint32_t leader = elect_one();
            int acc = 0;
            uint32_t acc_phase = 0;
            // ring cursor of the first window row of the current tile (slot, phase) and the tile's
            // row in its strip, all advanced incrementally: no runtime division in this loop, so
            // ptxas keeps the slot and descriptor arithmetic in uniform registers (a `% ring` here
            // went through F2I in vector registers and cost an R2UR per MMA operand)
            uint32_t sq = 0, phq = 0;
            int ri = t0 % prm.rows;
            long long pt_ = clock64();
            for (int t = t0; t < t1; ++t) {
                ROWS_PROF(2, pt_)
                if (!HALF && !(ABL(32))) {
                    if (TWO) mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
                    else mbar_wait(&tempty[acc], acc_phase ^ 1);
                }
                ROWS_PROF(0, pt_)
                // only the rows this tile adds: the nr - 1 it shares with the previous tile of the
                // strip were waited for then (fewer cluster-scope acquires per tile)
                const int lw0 = (t == t0 || ri == 0) ? 0 : nr - 1;
                for (int l = lw0; l < nr; ++l) {
                    uint32_t s = sq + l, ph = phq;
                    if (s >= (uint32_t)ring) { s -= ring; ph ^= 1; }
    #pragma unroll
                    for (int kb = 0; kb < KBC; ++kb)
                        if (!(ABL(64))) {
    #ifdef SEGB_ROWS_SLOT_CTA_SCOPE
                            if (TWO) mbar_wait(&slot_full[s * KBC + kb], ph);
    #else
                            if (TWO) mbar_wait_cluster(&slot_full[s * KBC + kb], ph);
    #endif
                            else mbar_wait(&slot_full[s * KBC + kb], ph);
                        }
                }
                tc_fence_after();
                ROWS_PROF(1, pt_)
                const uint32_t d0 = tmem_base + acc * NCL * (COSPLIT ? N / 2 : N);
                if constexpr (HALF) {  // two half tiles: row parity h into its own TMEM buffer
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (!(ABL(32))) mbar_wait(&tempty[acc], acc_phase ^ 1);
                        tc_fence_after();
                        // class row parity h reads the union window from row offset dminr_rs[h] - dmin_r
                        uint32_t sqh = sq + (uint32_t)(prm.dminr_rs[h] - prm.dmin_r);
                        if (sqh >= (uint32_t)ring) sqh -= ring;
                        const uint32_t dh = tmem_base + acc * NCL * N;
                        const uint32_t bh = bLo0 + (uint32_t)(h * make_schedule<NH, SWAP, 0>().ntiles * KBC) * B16;
                        if (ABL(4)) {
                        } else if (h == 0) issue_tile<NH, KBC, SWAP, MR, 0>(dh, aLo0, bh, sqh, ring, S16, B16, N, leader);
                        else issue_tile<NH, KBC, SWAP, MR, 1>(dh, aLo0, bh, sqh, ring, S16, B16, N, leader);
                        if (!(ABL(32))) tc_commit_pred(&tfull[acc], leader);
                        if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
                    }
                } else if (ABL(4)) {
                } else if (TWO) issue_tile<NH, KBC, SWAP, MR, -1, 2, COSPLIT, F16>(d0, aLo0, bLo0, sq, ring, S16, B16, N,
                                                                                    leader, prm.slot_plane >> 4,
                                                                                    prm.b_plane >> 4);
                else if (RS == 1) issue_tile<NH, KBC, SWAP, MR, -1, 1, true, F16>(d0, aLo0, bLo0, sq, ring, S16, B16, N,
                                                                                  leader, prm.slot_plane >> 4,
                                                                                  prm.b_plane >> 4);
                else if (rsel == 0) issue_tile<NH, KBC, SWAP, MR, 0>(d0, aLo0, bLo0, sq, ring, S16, B16, N, leader);
                else issue_tile<NH, KBC, SWAP, MR, 1>(d0, aLo0, bLo0, sq, ring, S16, B16, N, leader);
                // commits, branch-free like the MMAs (lane `leader` issues them)
                if (!HALF && !(ABL(32))) {
                    if (TWO) tc_commit_2sm_mc_pred(&tfull[acc], 3, leader);
                    else tc_commit_pred(&tfull[acc], leader);
                }
                // release input rows no later tile of this strip reads, advance the window
                const int ri_next = ri + 1 == prm.rows ? 0 : ri + 1;
                const bool cont = (t + 1 < t1) && ri_next != 0;
                const int nrel = cont ? 1 : nr;
                for (int l = 0; l < nrel; ++l) {
                    uint32_t s = sq + l;
                    if (s >= (uint32_t)ring) s -= ring;
    #pragma unroll
                    for (int kb = 0; kb < KBC; ++kb)
                        if (!(ABL(64))) {
                            if (TWO) tc_commit_2sm_mc_pred(&slot_empty[s * KBC + kb], 3, leader);
                            else tc_commit_pred(&slot_empty[s * KBC + kb], leader);
                        }
                }
                sq += nrel;
                if (sq >= (uint32_t)ring) { sq -= ring; phq ^= 1; }
                ri = ri_next;
                __syncwarp();
                if (!HALF && ++acc == NBUF) { acc = 0; acc_phase ^= 1; }
            }
            }
        } else if (ARR && warp == kArriverWarp) {
            // ---------------- the arriver: one slot_full arrival per unit the loaders filled, in
            // the loaders' unit order (tile t adds loads_of(t) rows, each of KBC channel blocks;
            // M = 64 pairs: the two blocks of a row are filled at once by loader warps 0-1 / 2-3,
            // each half on its own barrier)
            uint32_t qs = 0;
            for (int t = t0; t < t1; ++t)
                for (int l = loads_of(t); l > 0; --l) {
#pragma unroll
                    for (int kb = 0; kb < KBC; ++kb) {
                        if (PAIRKB) named_bar_sync(kSlotBar0 + kb, 32 * 3);
                        else named_bar_sync(kSlotBar0, 32 * 5);
                        if (lane == 0 && !(ABL(64))) {
                            if (TWO) mbar_arrive_cluster(mapa_rank(&slot_full[qs * KBC + kb], 0));
                            else mbar_arrive(&slot_full[qs * KBC + kb]);
                        }
                        __syncwarp();
                    }
                    if (++qs == (uint32_t)ring) qs = 0;
                }
        }  // warps 2 (unless the arriver), 3: idle (they only take part in warpgroup 0's register release)
    } else if (warp >= kLoaderWarp0) {
#ifndef SEGB_ROWS_NO_SETMAXNREG
        // (3xFP16: the loaders hold 3 x 32 fp32 registers of units; the epilogue gets the rest)
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(F16 ? kRegsLoadF16 : kRegsLoad));
#endif
        // ---------------- row loaders / transposers: NCHW input row (64 channels x MR columns
        // + halo) -> K-major SWIZZLE_128B slot rows. Thread (cg = t & 7, cc = t >> 3) loads 8
        // channels x 8 columns with 128-bit loads (coalesced along the row), transposes the 8x8
        // bf16 tile in registers and stores 8 slot rows x 16 B; the next unit's loads are in
        // flight while the current one is stored.
        const int tt = threadIdx.x - kLoaderWarp0 * 32;
        const int tw = tt >> 5;
        const int cg = tt & 7;
        const int cc = PAIRKB ? (tt >> 3) & 7 : tt >> 3;  // column chunk of 8
        const int kbt = PAIRKB ? tt >> 6 : 0;             // PAIRKB: this thread's channel block
        const int th = PAIRKB ? tt & 63 : tt;             // index among the threads of one slot
        const int HL = -prm.dmin_c, HR = prm.slot_rows - MR - HL;
        const bool col_active = cc < MR / 8;  // MR = 64 (unpaired) uses half the column chunks
        const int64_t plane_in = (int64_t)prm.h * prm.w;
        // unit cursor (tile, row of its window, channel block)
        auto advance = [&](int &ut, int &ul, int &ukb) {
            if (++ukb == UKB) {
                ukb = 0;
                if (++ul == nr && ++ut < t1) ul = nr - loads_of(ut);
            }
        };
        if constexpr (F16) {
            // ---- 3xFP16: fp32 rows (8 channels x 8 columns per thread, 16-byte loads), scaled by
            // 2^k_x, split into fp16 hi / lo, 8x8-transposed in registers into both slot planes
            const float *xf = reinterpret_cast<const float *>(prm.x);
            float mx = 0.f;
            for (int i = lane; i < kAbsmaxBlocks; i += 32) mx = fmaxf(mx, __ldg(prm.x_partials + i));
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
            const float sc = ldexpf(1.f, f16_scale_exp(mx));
            // all 128 loader threads share a unit: thread (cg = t & 7, c4 = t >> 3) owns 8 channels x
            // 4 columns (one 16-byte load per channel), so a unit costs each thread 32 values
            static_assert(MR == 64, "3xFP16 rows: 64-wide tiles (16 column chunks of 4)");
            const int c4 = tt >> 3;
#ifndef SEGB_ROWS_F16_KLB
#define SEGB_ROWS_F16_KLB 3
#endif
            constexpr int KLB = SEGB_ROWS_F16_KLB;  // units in flight per thread (32 fp32 registers each)
            // unit cursor with its tile's (row i, segment ms, sample b) kept incrementally: no
            // runtime divisions per unit
            struct Cur {
                int t, l, i, ms, b;
            };
            auto cur_at = [&](int t) {
                Cur c;
                c.t = t;
                c.l = t < t1 ? nr - loads_of(t) : 0;
                const int ta = t + toff;
                c.i = ta % prm.rows;
                const int rest = ta / prm.rows;
                c.ms = rest % prm.msub;
                c.b = rest / prm.msub;
                return c;
            };
            auto cur_next = [&](Cur &c) {
                if (++c.l < nr) return;
                if (++c.t >= t1) return;
                if (++c.i == prm.rows) {  // a new strip: its first tile loads all nr rows
                    c.i = 0;
                    if (++c.ms == prm.msub) { c.ms = 0; ++c.b; }
                    c.l = 0;
                } else {
                    c.l = nr - 1;  // consecutive tiles of a strip share nr - 1 rows
                }
            };
#ifndef SEGB_ROWS_F16_LOADS_V2
#define SEGB_ROWS_F16_LOADS_V2 1
#endif
            // c_in % 8 == 0 (rows_params): a thread's 8 channels are all valid or all past c_in, so
            // one predicate per unit and a running pointer per channel (the per-channel 64-bit
            // address arithmetic, predicates and zero-fills spilled the base pointer back to the
            // constant bank and stalled on address-register reuse behind queued loads)
            const int64_t plane4 = plane_in / 4;  // plane_in % 4 == 0 (prm.w % 8 == 0)
            auto load_unit = [&](const Cur &u, float4 (&r)[8], float (&hv)[8]) {
                const int row = u.i + dminr + u.l;
                const int j0 = u.ms * MR;
                const bool in_row = row >= 0 && row < prm.h;
                const int ch0 = prm.ch_base + cg * 8;
                const float *src = xf + ((int64_t)u.b * prm.c_in + ch0) * plane_in + (int64_t)row * prm.w + j0;
#if SEGB_ROWS_F16_LOADS_V2
                const bool ok = in_row && ch0 < prm.c_in && !(ABL(2));
                if (ok) {
                    const float4 *q = reinterpret_cast<const float4 *>(src) + c4;
#pragma unroll
                    for (int c = 0; c < 8; ++c) r[c] = __ldg(q + c * plane4);
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) r[c] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int c = 0; c < 8; ++c) hv[c] = 0.f;
                if (th < (HL + HR) * 8) {  // halo column tasks: (halo col, channel group)
                    const int hc = th >> 3;
                    const int col = hc < HL ? j0 - HL + hc : j0 + MR + (hc - HL);
                    if (ok && col >= 0 && col < prm.w) {
                        const float *q = src + (col - j0);
#pragma unroll
                        for (int c = 0; c < 8; ++c) hv[c] = __ldg(q + c * plane_in);
                    }
                }
#else
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    r[c] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (in_row && ch0 + c < prm.c_in && !(ABL(2)))
                        r[c] = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)c * plane_in + c4 * 4));
                }
#pragma unroll
                for (int c = 0; c < 8; ++c) hv[c] = 0.f;
                if (th < (HL + HR) * 8) {  // halo column tasks: (halo col, channel group)
                    const int hc = th >> 3;
                    const int col = hc < HL ? j0 - HL + hc : j0 + MR + (hc - HL);
                    if (in_row && col >= 0 && col < prm.w) {
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            if (ch0 + c < prm.c_in) hv[c] = __ldg(src + (int64_t)c * plane_in + (col - j0));
                    }
                }
#endif
            };
            static_assert(KBC == 1 && !PAIRKB, "3xFP16 rows: one 64-channel block per pass");
            float4 rb[KLB][8];
            float hb[KLB][8];
            bool bv[KLB];
            Cur cu = cur_at(t0);
            // L2 prefetch of the row unit kPrefetch units beyond the register loads: each of the 128
            // threads touches one of the unit's 128-byte lines (64 channels x 2 halves of the row)
#ifndef SEGB_ROWS_F16_PREFETCH
#define SEGB_ROWS_F16_PREFETCH 4
#endif
            constexpr int kPrefetch = SEGB_ROWS_F16_PREFETCH;
            Cur pc = cu;
            auto prefetch_unit = [&](const Cur &u) {
                const int row = u.i + dminr + u.l;
                if (u.t >= t1 || row < 0 || row >= prm.h) return;
                const int ch = prm.ch_base + (tt >> 1);
                if (ch >= prm.c_in) return;
                const float *p = xf + ((int64_t)u.b * prm.c_in + ch) * plane_in + (int64_t)row * prm.w + u.ms * MR +
                                 (tt & 1) * 32;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
            };
            for (int k = 0; k < KLB + kPrefetch && pc.t < t1; ++k) cur_next(pc);
#pragma unroll
            for (int k = 0; k < KLB; ++k) {
                bv[k] = cu.t < t1;
                if (bv[k]) {
                    load_unit(cu, rb[k], hb[k]);
                    cur_next(cu);
                }
            }
            uint32_t qs = 0, qph = 0;
            bool more = bv[0];
            long long pl_ = clock64();
            while (more) {
#pragma unroll
                for (int k = 0; k < KLB; ++k) {
                    if (!bv[k]) {
                        more = false;
                        break;
                    }
                    const int sidx = qs;
                    if (tw == 0) { ROWS_PROF(7, pl_) }
                    if (!(ABL(64))) mbar_wait(&slot_empty[sidx], qph ^ 1);
                    if (tw == 0) { ROWS_PROF(6, pl_) }
                    const uint32_t dst = smem_u32(sRing + sidx * prm.slot_bytes);
                    if (!(ABL(16))) {
                        uint32_t hp[8][2], lp[8][2];  // [channel][q]: columns 2q, 2q+1 as fp16 pairs
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const float v[4] = {rb[k][c].x * sc, rb[k][c].y * sc, rb[k][c].z * sc, rb[k][c].w * sc};
#pragma unroll
                            for (int q = 0; q < 2; ++q)  // packed conversions, bitwise split_f16's
                                split_f16x2(v[2 * q], v[2 * q + 1], hp[c][q], lp[c][q]);
                        }
#pragma unroll
                        for (int w = 0; w < 4; ++w) {  // slot row = column c4*4 + w, 8 channels = 16 B
                            uint32_t oh[4], ol[4];
                            const uint32_t sel = (w & 1) ? 0x7632 : 0x5410;
#pragma unroll
                            for (int m4 = 0; m4 < 4; ++m4) {
                                oh[m4] = __byte_perm(hp[2 * m4][w >> 1], hp[2 * m4 + 1][w >> 1], sel);
                                ol[m4] = __byte_perm(lp[2 * m4][w >> 1], lp[2 * m4 + 1][w >> 1], sel);
                            }
                            const int rho = HL + c4 * 4 + w;
                            const uint32_t addr = dst + rho * 128 + ((cg ^ (rho & 7)) << 4);
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(oh[0]),
                                         "r"(oh[1]), "r"(oh[2]), "r"(oh[3])
                                         : "memory");
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr + prm.slot_plane),
                                         "r"(ol[0]), "r"(ol[1]), "r"(ol[2]), "r"(ol[3])
                                         : "memory");
                        }
                    }
                    if (th < (HL + HR) * 8) {
                        const int hc = th >> 3;
                        const int rho = hc < HL ? hc : HL + MR + (hc - HL);
                        const uint32_t addr = dst + rho * 128 + ((cg ^ (rho & 7)) << 4);
                        uint32_t oh[4], ol[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            __half h0, l0, h1, l1;
                            split_f16(hb[k][2 * q] * sc, h0, l0);
                            split_f16(hb[k][2 * q + 1] * sc, h1, l1);
                            oh[q] = pack_h2(h0, h1);
                            ol[q] = pack_h2(l0, l1);
                        }
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(oh[0]), "r"(oh[1]),
                                     "r"(oh[2]), "r"(oh[3])
                                     : "memory");
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr + prm.slot_plane),
                                     "r"(ol[0]), "r"(ol[1]), "r"(ol[2]), "r"(ol[3])
                                     : "memory");
                    }
                    if (tw == 0) { ROWS_PROF(12, pl_) }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (tw == 0) { ROWS_PROF(14, pl_) }
                    if constexpr (ARR) {
                        named_bar_sync(kSlotBar0, 32 * 5);
                    } else if (lane == 0 && !(ABL(64))) {
                        if (TWO) mbar_arrive_cluster(mapa_rank(&slot_full[sidx], 0));
                        else mbar_arrive(&slot_full[sidx]);
                    }
                    if (tw == 0) { ROWS_PROF(13, pl_) }
                    if (++qs == (uint32_t)ring) { qs = 0; qph ^= 1; }
                    bv[k] = cu.t < t1;
                    if (bv[k]) {
                        load_unit(cu, rb[k], hb[k]);
                        cur_next(cu);
                        if (kPrefetch > 0) {
                            prefetch_unit(pc);
                            cur_next(pc);
                        }
                    }
                }
            }
        } else {
        const __nv_bfloat16 *x = reinterpret_cast<const __nv_bfloat16 *>(prm.x);
        auto load_unit = [&](int t, int l, int kb, uint4 (&r)[8], uint4 &hv) {
            t += toff;
            const int i = t % prm.rows, rest = t / prm.rows;
            const int ms = rest % prm.msub, b = rest / prm.msub;
            const int row = i + dminr + l;
            const int j0 = ms * MR;
            const bool in_row = row >= 0 && row < prm.h;
            const bool rok = in_row && col_active;
            const int ch0 = (PAIRKB ? kbt : kb) * 64 + cg * 8;
            const __nv_bfloat16 *src = x + ((int64_t)b * prm.c_in + ch0) * plane_in + (int64_t)row * prm.w + j0;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                r[c] = make_uint4(0, 0, 0, 0);
                if (rok && ch0 + c < prm.c_in && !(ABL(2)))
                    r[c] = __ldg(reinterpret_cast<const uint4 *>(src + (int64_t)c * plane_in + cc * 8));
            }
            hv = make_uint4(0, 0, 0, 0);
            if (th < (HL + HR) * 8) {  // halo column tasks: (halo col, channel group)
                const int hc = th >> 3;
                const int col = hc < HL ? j0 - HL + hc : j0 + MR + (hc - HL);
                if (in_row && col >= 0 && col < prm.w) {
                    uint32_t h16[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        h16[c] = (ch0 + c < prm.c_in)
                                     ? (uint32_t)__ldg(reinterpret_cast<const unsigned short *>(
                                           src + (int64_t)c * plane_in + (col - j0)))
                                     : 0u;
                    hv = make_uint4(h16[0] | (h16[1] << 16), h16[2] | (h16[3] << 16), h16[4] | (h16[5] << 16),
                                    h16[6] | (h16[7] << 16));
                }
            }
        };
        // kLoadBufs register buffers in rotation, the loop unrolled by as many so that no buffer
        // is ever copied: a unit's loads are issued kLoadBufs units before its slot stores
        // consume them
        // (a `cur = nxt` rotation of register arrays made every iteration wait for the loads it
        // had just issued: one full memory latency per unit)
        uint4 rb[kLoadBufs][8], hb[kLoadBufs];
        int bkb[kLoadBufs];     // channel block of the unit in each buffer
        bool bv[kLoadBufs];     // buffer holds a unit
        int ct = t0, cl = t0 < t1 ? nr - loads_of(t0) : 0, ckb_ = 0;  // next unit to load
        // L2 prefetch of the unit kBfPrefetch units beyond the register loads (one 128-byte line of
        // its row segment per thread: 64 channels x MR columns x 2 B)
        // (measured: 128-wide single-CTA rows, ebgan_l7 0.608 -> 0.575 ms; the 2-SM pair, l6, +2%: off)
#ifndef SEGB_ROWS_BF16_PREFETCH
#define SEGB_ROWS_BF16_PREFETCH ((RS == 1 && MR == 128) ? 4 : 0)
#endif
        constexpr int kBfPrefetch = SEGB_ROWS_BF16_PREFETCH;
        int pt = ct, pl = cl, pkb = ckb_;
        auto prefetch_unit = [&]() {
            if (pt >= t1) return;
            const int ta = pt + toff;
            const int i = ta % prm.rows, rest = ta / prm.rows;
            const int ms = rest % prm.msub, b = rest / prm.msub;
            const int row = i + dminr + pl;
            if (row < 0 || row >= prm.h) return;
            constexpr int LPC = MR * 2 / 128;  // lines per channel row segment
            const int ch = (PAIRKB ? kbt * 64 : pkb * 64) + tt / LPC;
            if (tt >= 64 * LPC || ch >= prm.c_in) return;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(x + ((int64_t)b * prm.c_in + ch) * plane_in +
                                                        (int64_t)row * prm.w + ms * MR + (tt % LPC) * 64));
        };
        if (kBfPrefetch > 0)
            for (int k = 0; k < kLoadBufs + kBfPrefetch && pt < t1; ++k) advance(pt, pl, pkb);
#pragma unroll
        for (int k = 0; k < kLoadBufs; ++k) {
            bv[k] = ct < t1;
            bkb[k] = ckb_;
            if (bv[k]) {
                load_unit(ct, cl, ckb_, rb[k], hb[k]);
                advance(ct, cl, ckb_);
            }
        }
        uint32_t qs = 0, qph = 0;  // ring slot and phase of the current input row
        bool more = bv[0];
        while (more) {
#pragma unroll
            for (int k = 0; k < kLoadBufs; ++k) {
                if (!bv[k]) {
                    more = false;
                    break;
                }
                const int ckb = PAIRKB ? kbt : bkb[k];
                const int sidx = qs * KBC + ckb;
                long long pl_ = clock64();
                if (tw == 0) { ROWS_PROF(7, pl_) }
                if (!(ABL(64))) mbar_wait(&slot_empty[sidx], qph ^ 1);
                if (tw == 0) { ROWS_PROF(6, pl_) }
                const uint32_t dst = smem_u32(sRing + sidx * prm.slot_bytes);
                if (col_active && !(ABL(16))) {
#pragma unroll
                    for (int w = 0; w < 8; ++w) {  // 8x8 transpose: column cc*8 + w, channels cg*8 .. +7
                        uint32_t o[4];
#pragma unroll
                        for (int m = 0; m < 4; ++m) {
                            const uint32_t a = (&rb[k][2 * m].x)[w >> 1], bb = (&rb[k][2 * m + 1].x)[w >> 1];
                            o[m] = __byte_perm(a, bb, (w & 1) ? 0x7632 : 0x5410);
                        }
                        const int rho = HL + cc * 8 + w;
                        const uint32_t addr = dst + rho * 128 + ((cg ^ (rho & 7)) << 4);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(o[0]), "r"(o[1]),
                                     "r"(o[2]), "r"(o[3])
                                     : "memory");
                    }
                }
                if (th < (HL + HR) * 8) {
                    const int hc = th >> 3;
                    const int rho = hc < HL ? hc : HL + MR + (hc - HL);
                    const uint32_t addr = dst + rho * 128 + ((cg ^ (rho & 7)) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(hb[k].x), "r"(hb[k].y),
                                 "r"(hb[k].z), "r"(hb[k].w)
                                 : "memory");
                }
                fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
                __syncwarp();
                if constexpr (ARR) {
                    if (PAIRKB) named_bar_sync(kSlotBar0 + kbt, 32 * 3);
                    else named_bar_sync(kSlotBar0, 32 * 5);
                } else if (lane == 0 && !(ABL(64))) {
                    if (TWO) mbar_arrive_cluster(mapa_rank(&slot_full[sidx], 0));  // the leader's barrier
                    else mbar_arrive(&slot_full[sidx]);
                }
                if (PAIRKB || ckb == KBC - 1) {
                    if (++qs == (uint32_t)ring) { qs = 0; qph ^= 1; }
                }
                // refill this buffer with the unit kLoadBufs ahead
                bv[k] = ct < t1;
                bkb[k] = ckb_;
                if (bv[k]) {
                    load_unit(ct, cl, ckb_, rb[k], hb[k]);
                    advance(ct, cl, ckb_);
                    if (kBfPrefetch > 0) {
                        prefetch_unit();
                        advance(pt, pl, pkb);
                    }
                }
            }
        }
        }
    } else {
#ifndef SEGB_ROWS_NO_SETMAXNREG
        if constexpr (F16) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsEpiF16));
#endif
        // ---------------- epilogue (warps 4..7): warp reads TMEM lane quarter warp % 4. The
        // classes of a position are in registers, so each lane writes the pair of output
        // columns (2j, 2j+1) of each of its output rows as one 4-byte bf16x2 store: a warp
        // store covers 128 (M=64: 64) contiguous bytes of one output row, every output element
        // is written once, and no staging, proxy fence or barrier is needed.
        const int quarter = warp & 3;
        // position of this lane's TMEM row: M=128 -> lane = row; M=64 -> lanes 32q + [0,16)
        // TWO (M = 64 per CTA): lanes 0-63 = positions with the first channel half, 64-127 = the
        // same positions with the second half
        const int m = COSPLIT ? (quarter & 1) * 32 + lane : (MR == 128 ? quarter * 32 + lane : quarter * 16 + (lane & 15));
        const bool lane_active = COSPLIT || MR == 128 || lane < 16;
        const int NE = COSPLIT ? N / 2 : N;              // TMEM columns (= output channels) per class here
        const int chalf = COSPLIT ? (quarter >> 1) : 0;  // this warp's output-channel half
        const int NEW = NE, cw0 = 0;  // channels per class this warp stores, its first one
        auto release_acc = [&](int a) {
#ifdef SEGB_ROWS_RELAXED_ARRIVE  // measured 3% slower on l7 fp32, no change on bf16 l6/l7
            if (TWO) mbar_arrive_relaxed_cluster(mapa_rank(&tempty[a], 0));
            else mbar_arrive_relaxed(&tempty[a]);
#else
            if (TWO) mbar_arrive_cluster(mapa_rank(&tempty[a], 0));
            else mbar_arrive(&tempty[a]);
#endif
        };
        // With even P the classes with row/column parity 0 fill output row 2i and the even
        // columns; with odd P (SWAP) it is the parity-1 classes (engines.py:338-347).
        constexpr int RE = SWAP, SE = SWAP;  // class parities of output row 2i / even columns
        const int64_t plane_b = (int64_t)prm.oh * prm.ow * 2, ow_b = (int64_t)prm.ow * 2;
        // RS = 2: this CTA holds classes (rsel, 0), (rsel, 1) and writes output row 2i + (rsel != RE)
        const int row_off = RS == 2 ? (rsel != RE ? 1 : 0) : 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        constexpr int HT = HALF ? 2 : 1;  // accumulator buffers (half tiles) per tile
        if constexpr (F16) {
            // ---- 3xFP16: fp32 output. A lane holds the four classes of its position, i.e. output
            // columns (2j, 2j+1) of rows 2i and 2i+1: one 8-byte store per row and channel (a warp
            // instruction writes 256 contiguous bytes), times 2^-(k_x + k_w) (exact).
            static_assert(NCL == 4, "3xFP16 rows: all four classes per accumulator buffer");
            float mx = 0.f;
            for (int q = lane; q < kAbsmaxBlocks; q += 32) mx = fmaxf(mx, __ldg(prm.x_partials + q));
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
            const float us = ldexpf(1.f, -f16_scale_exp(mx)) * prm.w_unscale;
            const int64_t plane = (int64_t)prm.oh * prm.ow;
            constexpr int C00 = class_slot(2 * RE + SE), C01 = class_slot(2 * RE + (1 - SE));
            constexpr int C10 = class_slot(2 * (1 - RE) + SE), C11 = class_slot(2 * (1 - RE) + (1 - SE));
            // a later channel pass reads y back: the next tile's lines of this warp (32 channels x 2
            // rows x 256 B) are prefetched into L2 while this tile's accumulators are awaited
            auto prefetch_tile = [&](int tn) {
                const int ta = tn + toff;
                const int i = ta % prm.rows, rest = ta / prm.rows;
                const int ms = rest % prm.msub, b = rest / prm.msub;
                const float *base = reinterpret_cast<const float *>(prm.y) +
                                    ((int64_t)b * prm.c_out + chalf * NE + lane % NE) * plane +
                                    (int64_t)(2 * i + row_off) * prm.ow + (int64_t)ms * 2 * MR + 2 * ((quarter & 1) * 32);
#pragma unroll
                for (int r = 0; r < 2; ++r)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (int64_t)r * prm.ow + h * 32));
            };
            if (!SEGB_ROWS_F16_RED && ACCP && t0 < t1) prefetch_tile(t0);
            // the tile's (row i, segment ms, sample b), advanced incrementally (no per-tile divisions)
            int ei = (t0 + toff) % prm.rows, ems = ((t0 + toff) / prm.rows) % prm.msub,
                eb = ((t0 + toff) / prm.rows) / prm.msub;
            for (int t = t0; t < t1; ++t) {
                const int i = ei, ms = ems, b = eb;
                if (++ei == prm.rows) {
                    ei = 0;
                    if (++ems == prm.msub) { ems = 0; ++eb; }
                }
                if (!SEGB_ROWS_F16_RED && ACCP && t + 1 < t1) prefetch_tile(t + 1);
                long long pe_ = clock64();
                if (warp == kEpiWarp0) { ROWS_PROF(4, pe_) }
                if (!(ABL(32))) mbar_wait(&tfull[acc], acc_phase);
                if (warp == kEpiWarp0) { ROWS_PROF(3, pe_) }
                tc_fence_after();
                const uint32_t tl = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * NCL * NE;
                float *pf = reinterpret_cast<float *>(prm.y) + ((int64_t)b * prm.c_out + chalf * NE) * plane +
                            (int64_t)(2 * i + row_off) * prm.ow + (int64_t)ms * 2 * MR + 2 * m;
                const int odd = lane & 1;
                float *pf4 = pf - 2 * odd + odd * prm.ow;  // even lane: row 2i, col 2m; odd: row 2i+1, col 2m-2
                (void)pf4;
                if (ABL(8)) {  // ablation: no TMEM reads (nor stores)
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0 && !(ABL(32))) release_acc(acc);
                    if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
                    continue;
                }
#ifndef SEGB_ROWS_F16_EPI_WHOLE
#define SEGB_ROWS_F16_EPI_WHOLE 1
#endif
#if SEGB_ROWS_F16_EPI_WHOLE
                {  // (F16: c_out <= 64 split over the pair, so NE <= 32)
                    // the whole tile's accumulators in one go (4 classes x NE columns, one wait), the
                    // TMEM buffer released before any store: the MMAs of the next tiles do not wait
                    // for this tile's output writes
                    uint32_t va[NCL][32];
#pragma unroll
                    for (int c = 0; c < NCL; ++c) {
                        tmem_ld16(tl + c * NE, *reinterpret_cast<uint32_t(*)[16]>(&va[c][0]));
                        if (NE > 16) tmem_ld16(tl + c * NE + 16, *reinterpret_cast<uint32_t(*)[16]>(&va[c][16]));
                    }
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < NCL; ++c)
#pragma unroll
                        for (int k = 0; k < 32; k += 8) reg_fence8(*reinterpret_cast<uint32_t(*)[8]>(&va[c][k]));
                    tc_fence_before();
                    __syncwarp();
                    // relaxed: the accumulators are in registers (waited); a release would first wait
                    // for the previous tile's global stores (ncu: 91% membar stalls on that arrive)
#ifndef SEGB_ROWS_F16_RELEASE_ARRIVE
                    if (lane == 0) {
                        if (TWO) mbar_arrive_relaxed_cluster(mapa_rank(&tempty[acc], 0));
                        else mbar_arrive_relaxed(&tempty[acc]);
                    }
#else
                    if (lane == 0) release_acc(acc);
#endif
#pragma unroll
                    for (int g8 = 0; g8 < 32; g8 += 8) {
                        if (g8 >= NE) break;
                        float4 old[8];
                        if (!SEGB_ROWS_F16_RED && ACCP && lane_active) {
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
#if SEGB_ROWS_F16_ST16
                                old[k] = __ldcs(reinterpret_cast<const float4 *>(pf4 + (int64_t)(g8 + k) * plane));
#else
                                const float2 o0 = __ldcs(reinterpret_cast<const float2 *>(pf + (int64_t)(g8 + k) * plane));
                                const float2 o1 =
                                    __ldcs(reinterpret_cast<const float2 *>(pf + (int64_t)(g8 + k) * plane + prm.ow));
                                old[k] = make_float4(o0.x, o0.y, o1.x, o1.y);
#endif
                            }
                        }
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int co = g8 + k;
                            const float2 r0 = make_float2(__uint_as_float(va[C00][co]) * us, __uint_as_float(va[C01][co]) * us);
                            const float2 r1 = make_float2(__uint_as_float(va[C10][co]) * us, __uint_as_float(va[C11][co]) * us);
#if SEGB_ROWS_F16_ST16
                            const float2 give = odd ? r0 : r1;
                            const float2 got = make_float2(__shfl_xor_sync(0xffffffffu, give.x, 1),
                                                           __shfl_xor_sync(0xffffffffu, give.y, 1));
                            float4 v4 = odd ? make_float4(got.x, got.y, r1.x, r1.y) : make_float4(r0.x, r0.y, got.x, got.y);
                            if (lane_active && !(ABL(1))) {
                                if (ACCP)
                                    v4 = make_float4(old[k].x + v4.x, old[k].y + v4.y, old[k].z + v4.z, old[k].w + v4.w);
                                *reinterpret_cast<float4 *>(pf4 + (int64_t)co * plane) = v4;
                            }
#else  // two 8-byte stores per channel, no lane exchange (old values as two float2 in old[k])
                            if (lane_active && !(ABL(1))) {
                                float2 *d0 = reinterpret_cast<float2 *>(pf + (int64_t)co * plane);
                                float2 a0 = r0, a1 = r1;
                                if (SEGB_ROWS_F16_RED && ACCP) {  // y += this pass (one add per element)
                                    red_add_f32x2(reinterpret_cast<float *>(d0), r0);
                                    red_add_f32x2(pf + (int64_t)co * plane + prm.ow, r1);
                                    continue;
                                }
                                if (ACCP) {
                                    a0 = make_float2(old[k].x + r0.x, old[k].y + r0.y);
                                    a1 = make_float2(old[k].z + r1.x, old[k].w + r1.y);
                                }
#if SEGB_ROWS_F16_STCS  // streaming (evict-first) stores: the output does not push the input rows out of L2
                                __stcs(d0, a0);
                                __stcs(reinterpret_cast<float2 *>(pf + (int64_t)co * plane + prm.ow), a1);
#else
                                d0[0] = a0;
                                *reinterpret_cast<float2 *>(pf + (int64_t)co * plane + prm.ow) = a1;
#endif
                            }
#endif
                        }
                    }
                    if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
                    continue;
                }
#else
                constexpr int CH = kEpiChunk;
                uint32_t v[NCL][CH], v2[NCL][CH];
#pragma unroll
                for (int c = 0; c < NCL; ++c) tmem_ld_chunk(tl + c * NE, v[c]);
                auto chunk = [&](int co0, uint32_t (&cur)[NCL][CH], uint32_t (&nxt)[NCL][CH]) {
                    // a later channel pass adds to y: the chunk's old values are loaded first, all
                    // CH in flight at once (interleaved with the stores they would be serialised:
                    // the compiler cannot prove the plane-strided addresses distinct)
                    float4 old[CH];
                    if (ACCP && lane_active) {
#pragma unroll
                        for (int k = 0; k < CH; ++k)
                            old[k] = __ldcs(reinterpret_cast<const float4 *>(pf4 + (int64_t)(co0 + k) * plane));
                    }
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < NCL; ++c) reg_fence_chunk(cur[c]);
                    if (co0 + CH < NE) {
#pragma unroll
                        for (int c = 0; c < NCL; ++c) tmem_ld_chunk(tl + c * NE + co0 + CH, nxt[c]);
                    } else {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) release_acc(acc);
                    }
#pragma unroll
                    for (int k = 0; k < CH; ++k) {
                        const float2 r0 = make_float2(__uint_as_float(cur[C00][k]) * us, __uint_as_float(cur[C01][k]) * us);
                        const float2 r1 = make_float2(__uint_as_float(cur[C10][k]) * us, __uint_as_float(cur[C11][k]) * us);
                        // 16-byte stores: lanes 2q, 2q+1 (positions j, j+1 = output columns 4q'..4q'+3)
                        // swap one row's pair, so the even lane writes row 2i and the odd lane row 2i+1
                        const float2 give = odd ? r0 : r1;
                        const float2 got = make_float2(__shfl_xor_sync(0xffffffffu, give.x, 1),
                                                       __shfl_xor_sync(0xffffffffu, give.y, 1));
                        const float4 v4 = odd ? make_float4(got.x, got.y, r1.x, r1.y) : make_float4(r0.x, r0.y, got.x, got.y);
                        if (lane_active && !(ABL(1))) {
                            float4 *dst4 = reinterpret_cast<float4 *>(pf4 + (int64_t)(co0 + k) * plane);
                            if (ACCP) {  // a later channel pass: y += this pass's sums
                                const float4 o = old[k];
                                *dst4 = make_float4(o.x + v4.x, o.y + v4.y, o.z + v4.z, o.w + v4.w);
                            } else {
                                *dst4 = v4;
                            }
                        }
                    }
                };
                for (int co0 = 0; co0 < NE; co0 += 2 * CH) {
                    chunk(co0, v, v2);
                    if (co0 + CH < NE) chunk(co0 + CH, v2, v);
                }
                if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
#endif
            }
        } else
        for (int u = t0 * HT; u < t1 * HT; ++u) {
            const int t = u / HT;
            const int ta = t + toff;
            const int i = ta % prm.rows, rest = ta / prm.rows;
            const int ms = rest % prm.msub, b = rest / prm.msub;
            // HALF: buffer u holds the classes of row parity u % 2 -> output row 2i + (h != RE)
            const int row_h = HALF ? ((u & 1) != RE ? 1 : 0) : row_off;
            long long pe_ = clock64();
            if (!(ABL(32))) mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if (warp == kEpiWarp0) { ROWS_PROF(3, pe_) }
            const uint32_t tl = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * NCL * NE;
            char *pc = reinterpret_cast<char *>(prm.y) + ((int64_t)b * prm.c_out + chalf * NE + cw0) * plane_b +
                       (int64_t)(2 * i + row_h) * ow_b + (int64_t)(ms * 2 * MR + 2 * m) * 2;  // (co, row, col 2j)
            // 8-byte store pointer: even position of this lane's pair, channel + (lane & 1)
            const int odd = lane & 1;
            char *pc2 = pc - odd * 4 + odd * plane_b;
            // CH channels per TMEM load per class; the next chunk's loads are in flight while
            // this chunk is converted and stored
            constexpr int CH = kEpiChunk;
            uint32_t v[NCL][CH];
            if (ABL(8)) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0 && !(ABL(32))) release_acc(acc);
                if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
                continue;
            }
#pragma unroll
            for (int c = 0; c < NCL; ++c) tmem_ld_chunk(tl + c * NE + cw0, v[c]);
            // two register buffers used alternately (loop unrolled by two, no copies): after
            // the wait for chunk k's loads, chunk k+1's loads go into the other buffer while
            // chunk k is converted and stored
            uint32_t v2[NCL][CH];
            auto chunk = [&](int co0, uint32_t (&cur)[NCL][CH], uint32_t (&nxt)[NCL][CH]) {
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < NCL; ++c) reg_fence_chunk(cur[c]);
                if (co0 + CH < NEW) {
#pragma unroll
                    for (int c = 0; c < NCL; ++c) tmem_ld_chunk(tl + c * NE + cw0 + co0 + CH, nxt[c]);
                } else {  // last chunk of the tile: release the accumulator buffer
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) release_acc(acc);
                }
                // Stores of 8 B per lane: lanes 2j and 2j+1 (adjacent positions) swap one bf16x2
                // pair per channel pair, so the even lane holds positions 2j, 2j+1 of channel k
                // and the odd lane the same positions of channel k+1 (a warp instruction writes
                // two 128-byte row segments). With 4-byte stores four warps per SM cap HBM
                // writes at ~4.9 TB/s; 8-byte ones reach ~6.2 TB/s (tools/probes/store_width_probe.cu).
#pragma unroll
                for (int k = 0; k < CH; k += 2) {
                    uint32_t mine[2], sent[2];  // [output row]: bf16x2 of channel k + odd (kept), k + !odd (sent)
                    if (RS != 2 && !HALF) {  // class index c = 2r + s; a bf16x2 is the (even, odd) column pair
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk) {
                            constexpr int C00 = class_slot(2 * RE + SE), C01 = class_slot(2 * RE + (1 - SE));
                            constexpr int C10 = class_slot(2 * (1 - RE) + SE), C11 = class_slot(2 * (1 - RE) + (1 - SE));
                            const uint32_t r0 = pack_bf16x2(__uint_as_float(cur[C00][k + kk]),
                                                            __uint_as_float(cur[C01][k + kk]));
                            const uint32_t r1 = pack_bf16x2(__uint_as_float(cur[C10][k + kk]),
                                                            __uint_as_float(cur[C11][k + kk]));
                            if (kk == odd) { mine[0] = r0; mine[1] = r1; } else { sent[0] = r0; sent[1] = r1; }
                        }
                    } else {  // TMEM slot = column parity s
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk) {
                            const uint32_t r0 = pack_bf16x2(__uint_as_float(cur[SE][k + kk]),
                                                            __uint_as_float(cur[1 - SE][k + kk]));
                            if (kk == odd) mine[0] = r0; else sent[0] = r0;
                        }
                    }
#pragma unroll
                    for (int rr = 0; rr < (RS != 2 && !HALF ? 2 : 1); ++rr) {
                        const uint32_t got = __shfl_xor_sync(0xffffffffu, sent[rr], 1);
                        const uint2 v = odd ? make_uint2(got, mine[rr]) : make_uint2(mine[rr], got);
                        if (lane_active && !(ABL(1))) {
                            if (SEGB_ROWS_BF16_STCS) __stcs(reinterpret_cast<uint2 *>(pc2 + rr * ow_b), v);
                            else *reinterpret_cast<uint2 *>(pc2 + rr * ow_b) = v;
                        }
                    }
                    pc2 += 2 * plane_b;
                }
            };
            for (int co0 = 0; co0 < NEW; co0 += 2 * CH) {
                chunk(co0, v, v2);
                if (co0 + CH < NEW) chunk(co0 + CH, v2, v);
            }
            if (warp == kEpiWarp0) { ROWS_PROF(4, pe_) }
            if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
        }
        }
    tc_fence_before();
    __syncthreads();
    if (TWO) cluster_sync_all();  // the leader's MMAs write this CTA's TMEM until both are done
    if (warp == 1) {
        tc_fence_after();
        if (TWO) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tcols));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tcols));
    }
    if (TWO) cluster_sync_all();  // remote arrivals on this CTA's barriers are all done
}

// ---------------------------------------------------------------- host side
static bool rows_f16(const IgemmShape &s) { return s.compute == SEGB_F32 && s.f16x3; }

static bool rows_params(const IgemmShape &s, RowsParams &prm, int &nh, int &kbc, int &swap, int &mr, int &nsplit) {
    const bool f16 = rows_f16(s);
    if (f16) {  // 3xFP16: fp32 in / out, one channel block, the 2-SM pair over batch halves
        if (s.x_dtype != SEGB_F32 || s.y_dtype != SEGB_F32) return false;
        // c_in > 64: 64-channel passes, the later ones accumulating into y (the weights of one
        // channel block, hi and lo, fill half the shared memory of each CTA of the pair)
        if (s.n != 4 || s.c_in > 128 || s.c_in % 8 != 0 || s.batch % 2 != 0 || s.c_out % 32 != 0) return false;
    } else if (s.compute != SEGB_BF16) {
        return false;
    }
    if (s.n % 2 != 0 || s.n > 6 || (!f16 && s.x_dtype != SEGB_BF16)) return false;
    if (!f16 && s.y_dtype != SEGB_BF16) return false;  // fp32 output takes K3
    if (s.c_out < 16 || s.c_out > 64 || s.c_out % 16 != 0) return false;
    if (s.w % 8 != 0 || s.w < 64) return false;
    const int oh = 2 * s.h + 2 * s.pad - s.n, ow = 2 * s.w + 2 * s.pad - s.n;
    if (oh < 2 || ow < 2) return false;
    const int p = s.pad / 2;
    swap = s.pad & 1;
    nh = s.n / 2;
    prm = RowsParams{};
    int dmin_r = 1 << 30, dmax_r = -(1 << 30), dmin_c = 1 << 30, dmax_c = -(1 << 30);
    for (int c = 0; c < 4; ++c) {
        const int r = c >> 1, q = c & 1;
        RowsClass &g = prm.cls[c];
        g.st_r = (r + swap) % 2;
        g.st_s = (q + swap) % 2;
        g.base_r = (g.st_r + r) / 2;
        g.base_s = (g.st_s + q) / 2;
        g.tap0 = class_offset(s.n, c);
        dmin_r = std::min(dmin_r, g.base_r - p);
        dmax_r = std::max(dmax_r, g.base_r + nh - 1 - p);
        dmin_c = std::min(dmin_c, g.base_s - p);
        dmax_c = std::max(dmax_c, g.base_s + nh - 1 - p);
    }
    const int rows = oh / 2, cols = ow / 2;
    if (f16 && cols % 64 != 0) return false;
    if (f16) mr = 64;  // M = 128 pair MMAs over 64-wide tiles: half the weights per CTA
    else if (cols % 128 == 0) mr = 128;
    else if (cols % 64 == 0) mr = 64;  // M=64 MMAs (half rate, but every input row loaded once)
    else return false;
    prm.c_in = s.c_in; prm.h = s.h; prm.w = s.w;
    prm.c_out = s.c_out; prm.oh = oh; prm.ow = ow; prm.p = p;
    prm.rows = rows; prm.msub = cols / mr;
    prm.dmin_r = dmin_r; prm.nr = dmax_r - dmin_r + 1;
    prm.dmin_c = dmin_c;
    prm.slot_rows = mr + dmax_c - dmin_c;
    if (-dmin_c > 8 || dmax_c > 8) return false;
    kbc = f16 ? 1 : (s.c_in + 63) / 64;  // F16: per pass
    if (kbc > 2) return false;
    prm.slot_bytes = (prm.slot_rows * 128 + 1023) / 1024 * 1024;
    prm.slot_plane = prm.b_plane = 0;
    if (f16) {  // hi plane then lo plane per slot (1024-aligned: the same swizzle phase)
        prm.slot_plane = prm.slot_bytes;
        prm.slot_bytes *= 2;
    }
    const int64_t total = s.batch * (int64_t)prm.msub * rows;
    if (total > INT32_MAX) return false;
    prm.total_tiles = (int)total;
    for (int r = 0; r < 2; ++r) prm.dminr_rs[r] = prm.cls[2 * r].base_r - p;
    // 64-wide class grids with an even batch: a 2-SM CTA pair (nsplit = 3, kernel RS = 3) turns
    // the half-rate M=64 MMAs into full-rate M=128 ones; each CTA holds the output-channel half
    // of all weights. SEGB200_ROWS_PAIR=0 disables it (A/B experiments).
    const char *pe = getenv("SEGB200_ROWS_PAIR");
    // 128-wide class grids (nsplit = 4, RS = 4) can likewise pair into M=256 MMAs (half the
    // weights' shared memory, a deeper row ring, half the B operand reads per SM); measured
    // slower on ebgan_l7 (0.70 vs 0.64 ms), so only with SEGB200_ROWS_PAIR=4.
    const bool pair_ok = s.batch % 2 == 0 && s.c_out % 32 == 0 && nh == 2 && (f16 || !(pe && !atoi(pe)));
    const bool pair128 = pe && atoi(pe) == 4;
    if (pair_ok && (mr == 64 || pair128)) {
        prm.b_tile_bytes = s.c_out / 2 * 128;
        if (f16) prm.b_plane = 4 * nh * nh * kbc * prm.b_tile_bytes;
        prm.half_tiles = prm.total_tiles / 2;
        for (prm.ring = kRingMax; prm.ring > std::max(4, prm.nr); --prm.ring)
            if (rows_layout(prm, 4 * nh * nh, kbc).total + 1024 <= 227 * 1024) break;
        if (rows_layout(prm, 4 * nh * nh, kbc).total + 1024 <= 227 * 1024) {
            nsplit = mr == 64 ? 3 : 4;
            return true;
        }
    }
    if (f16) return false;
    prm.b_tile_bytes = s.c_out * 128;
    // all four classes per CTA if their weights fit next to the row ring, else split the
    // classes over a CTA pair by row parity (half the weights each)
    // (the ring gets every slot that fits, up to kRingMax: the slots beyond the nr rows of the
    // current window let the loaders run ahead of the MMAs and hide the handshake latency)
    for (nsplit = 1; nsplit <= 2; nsplit *= 2) {
        const int nr_cta = nsplit == 2 ? nh : prm.nr;
        const int ring_min = std::max(4, nr_cta);
        for (prm.ring = kRingMax; prm.ring > ring_min; --prm.ring)
            if (rows_layout(prm, 4 / nsplit * nh * nh, kbc).total + 1024 <= 227 * 1024) break;
        if (rows_layout(prm, 4 / nsplit * nh * nh, kbc).total + 1024 <= 227 * 1024) {
            // SEGB200_ROWS_HALF=1: one CTA per strip with half-tile TMEM buffers (kernel RS = 5)
            const char *hv = getenv("SEGB200_ROWS_HALF");
            if (nsplit == 1 && nh == 2 && hv && atoi(hv)) nsplit = 5;
            return true;
        }
    }
    return false;
}

// the (NH, KBC, SWAP, MR, NS) variants compiled below
static bool rows_instantiated(int nh, int kbc, int swap, int mr, int nsplit, bool f16 = false) {
    // (odd P with w % 8 == 0 never gives a 64-multiple class grid for n = 4: no SWAP variant)
    if (f16) return nh == 2 && kbc == 1 && mr == 64 && nsplit == 3 && swap == 0;
    if (nsplit == 3) return mr == 64 && nh == 2;
    if (nsplit == 4) return mr == 128 && nh == 2;
    if (mr == 128 && nsplit == 1) return true;
    if (nsplit == 5) return mr == 128 && nh == 2;
    if (mr == 128 && nsplit == 2) return nh == 2 && kbc == 2 && swap == 0;
    if (mr == 64 && nh == 2 && swap == 0) return true;
    return mr == 64 && nh == 2 && kbc == 2 && swap == 1 && nsplit == 2;
}

int igemm_rows_variant(const IgemmShape &s) {
    RowsParams prm;
    int nh, kbc, swap, mr, nsplit;
    return rows_params(s, prm, nh, kbc, swap, mr, nsplit) ? nsplit : 0;
}

bool igemm_rows_supported(const IgemmShape &s) {
    RowsParams prm;
    int nh, kbc, swap, mr, nsplit;
    return rows_params(s, prm, nh, kbc, swap, mr, nsplit) &&
           rows_instantiated(nh, kbc, swap, mr, nsplit, rows_f16(s)) && tensor_map_encoder() != nullptr;
}

template <int NH, int KBC, int SWAP, int MR, int NS, int FM = 0>
static void launch_rows(int grid, size_t smem, cudaStream_t st, const CUtensorMap &tmB, const CUtensorMap &tmBlo,
                        const RowsParams &prm) {
    auto kern = igemm_rows_kernel<NH, KBC, SWAP, MR, NS, FM>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (NS < 3 || NS == 5) {
        kern<<<grid, kRowsThreads, smem, st>>>(tmB, tmBlo, prm);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kRowsThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, tmB, tmBlo, prm);
}

int64_t igemm_rows_workspace_bytes(const IgemmShape &s) { return rows_f16(s) ? kAbsmaxBytes : 0; }

int run_igemm_rows(const IgemmShape &s, const void *x, const void *wg, const void *wg_lo, void *y, void *ws,
                   int64_t ws_bytes, cudaStream_t st) {
    const bool f16 = rows_f16(s);
    RowsParams prm;
    int nh, kbc, swap, mr, nsplit;
    if (!rows_params(s, prm, nh, kbc, swap, mr, nsplit))
        return fail(SEGB_ERR_UNSUPPORTED, "row-streaming implicit GEMM: unsupported shape");
    auto encode = tensor_map_encoder();
    CUtensorMap tmB, tmBlo;
    {
        cuuint64_t dims[3] = {(cuuint64_t)s.c_in_pad, (cuuint64_t)s.c_out_pad, (cuuint64_t)s.n * s.n};
        cuuint64_t strides[2] = {(cuuint64_t)s.c_in_pad * 2, (cuuint64_t)s.c_out_pad * s.c_in_pad * 2};
        cuuint32_t box[3] = {64, (cuuint32_t)((nsplit == 3 || nsplit == 4) ? s.c_out / 2 : s.c_out), 1};
        cuuint32_t es[3] = {1, 1, 1};
        const CUtensorMapDataType dt = f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        CUresult r = encode(&tmB, dt, 3, const_cast<void *>(wg), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SEGB_ERR_CUDA, "tensor map (weights): error %d", (int)r);
        tmBlo = tmB;
        if (f16) {
            r = encode(&tmBlo, dt, 3, const_cast<void *>(wg_lo), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(SEGB_ERR_CUDA, "tensor map (weights lo): error %d", (int)r);
        }
    }
    prm.x_partials = nullptr;
    prm.w_unscale = ldexpf(1.f, -s.w_exp);
    if (f16) {  // the input's scale: absmax partials into the caller's workspace
        if (!ws || ws_bytes < igemm_rows_workspace_bytes(s))
            return fail(SEGB_ERR_VALUE, "row-streaming GEMM: workspace of %lld bytes needed, got %lld",
                        (long long)igemm_rows_workspace_bytes(s), (long long)ws_bytes);
        float *partials = (float *)ws;
        if (int rc = run_absmax_partials(x, SEGB_F32, s.batch * (int64_t)s.c_in * s.h * s.w, partials, st)) return rc;
        prm.x_partials = partials;
    }
    prm.x = x;
    prm.y = y;
    prm.prof = nullptr;
    prm.ablate = 0;
    prm.ch_base = 0;
    prm.accumulate = 0;
    if (const char *ab = getenv("SEGB200_ABLATE")) prm.ablate = atoi(ab);
    if (const char *rg = getenv("SEGB200_ROWS_RING")) {  // debug: cap the ring depth
        const int nr_cta = nsplit == 2 ? nh : prm.nr;
        prm.ring = std::max(std::min(prm.ring, atoi(rg)), std::max(4, nr_cta));
    }
    if (const char *pe = getenv("SEGB200_PROFILE"); pe && atoi(pe)) {
        static unsigned long long *buf = nullptr;
        if (!buf) cudaMalloc(&buf, 64 * sizeof(unsigned long long));
        cudaMemsetAsync(buf, 0, 64 * sizeof(unsigned long long), st);
        prm.prof = buf;
        g_rows_prof_buf = buf;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int grid;
    size_t smem;
    if (nsplit == 3 || nsplit == 4) {  // CTA pairs over the two batch halves
        const int strips = (int)std::min<int64_t>(prm.half_tiles, sms / 2);
        grid = 2 * strips;
        prm.tiles_per_cta = (int)ceil_div(prm.half_tiles, strips);
        smem = rows_layout(prm, 4 * nh * nh, kbc).total + 1024;
    } else {
        const int cps = nsplit == 5 ? 1 : nsplit;  // CTAs per strip
        const int strips = (int)std::min<int64_t>(prm.total_tiles, sms / cps);  // CTAs per channel slice
        grid = strips * cps;
        prm.tiles_per_cta = (int)ceil_div(prm.total_tiles, strips);
        smem = rows_layout(prm, 4 / cps * nh * nh, kbc).total + 1024;
    }
    int rc = SEGB_OK;
#define SEGB_ROWS_CASE(NH_, KBC_, SW_, MR_, NS_)                                                  \
    if (!f16 && nh == NH_ && kbc == KBC_ && swap == SW_ && mr == MR_ && nsplit == NS_)             \
        launch_rows<NH_, KBC_, SW_, MR_, NS_>(grid, smem, st, tmB, tmBlo, prm);                    \
    else
    // 3xFP16 (fp32 in / out): EB-GAN l7's shape family
    if (f16 && nh == 2 && kbc == 1 && swap == 0 && mr == 64 && nsplit == 3) {
        // one launch per 64-channel block of the input, the later ones accumulating into y
        const int passes = (s.c_in + 63) / 64;
        for (int ps = 0; ps < passes; ++ps) {
            prm.ch_base = 64 * ps;
            prm.accumulate = ps > 0;
            if (ps == 0) launch_rows<2, 1, 0, 64, 3, 1>(grid, smem, st, tmB, tmBlo, prm);
            else launch_rows<2, 1, 0, 64, 3, 2>(grid, smem, st, tmB, tmBlo, prm);
            if (ps + 1 < passes) note_launch();
        }
    } else
    // instantiated: n in {2, 4, 6} x channel blocks x P parity for 128-wide rows; the n = 4
    // (GAN) family also for 64-wide rows and with the row-parity split
    SEGB_ROWS_CASE(1, 1, 0, 128, 1) SEGB_ROWS_CASE(1, 1, 1, 128, 1) SEGB_ROWS_CASE(1, 2, 0, 128, 1)
    SEGB_ROWS_CASE(1, 2, 1, 128, 1) SEGB_ROWS_CASE(2, 1, 0, 128, 1) SEGB_ROWS_CASE(2, 1, 1, 128, 1)
    SEGB_ROWS_CASE(2, 2, 0, 128, 1) SEGB_ROWS_CASE(2, 2, 1, 128, 1) SEGB_ROWS_CASE(3, 1, 0, 128, 1)
    SEGB_ROWS_CASE(3, 1, 1, 128, 1) SEGB_ROWS_CASE(3, 2, 0, 128, 1) SEGB_ROWS_CASE(3, 2, 1, 128, 1)
    SEGB_ROWS_CASE(2, 2, 0, 128, 2) SEGB_ROWS_CASE(2, 1, 0, 64, 1) SEGB_ROWS_CASE(2, 1, 0, 64, 2)
    SEGB_ROWS_CASE(2, 2, 0, 64, 1) SEGB_ROWS_CASE(2, 2, 0, 64, 2) SEGB_ROWS_CASE(2, 2, 1, 64, 2)
    SEGB_ROWS_CASE(2, 1, 0, 64, 3) SEGB_ROWS_CASE(2, 2, 0, 64, 3) SEGB_ROWS_CASE(2, 1, 1, 64, 3)
    SEGB_ROWS_CASE(2, 2, 1, 64, 3) SEGB_ROWS_CASE(2, 1, 0, 128, 4) SEGB_ROWS_CASE(2, 1, 1, 128, 4)
    SEGB_ROWS_CASE(2, 2, 0, 128, 4) SEGB_ROWS_CASE(2, 2, 1, 128, 4) SEGB_ROWS_CASE(2, 1, 0, 128, 5)
    SEGB_ROWS_CASE(2, 1, 1, 128, 5) SEGB_ROWS_CASE(2, 2, 0, 128, 5) SEGB_ROWS_CASE(2, 2, 1, 128, 5)
    { rc = fail(SEGB_ERR_UNSUPPORTED, "row-streaming implicit GEMM: variant not instantiated"); }
#undef SEGB_ROWS_CASE
    if (rc) return rc;
    note_launch();
    return check_launch("igemm_rows_kernel");
}

}  // namespace segb

// debug hook (not part of the ABI header): role cycle counters of CTA 0 of the last K3b launch
extern "C" int segb_debug_rows_profile(unsigned long long *out) {
    cudaDeviceSynchronize();
    if (!segb::g_rows_prof_buf) return 1;
    cudaMemcpy(out, segb::g_rows_prof_buf, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    return 0;
}
