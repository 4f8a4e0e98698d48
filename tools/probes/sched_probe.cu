// Probe (not part of the library): K3b's ebgan_l7 MMA schedule (n = 4, P = 2, 128-position
// tiles, 64 channels: 9 shared windows per k-step, N = 256 / 4 x 128 / 4 x 64) issued back to
// back by one warp per SM, with optional background traffic from other warps, to find what
// slows the schedule down inside the kernel:
//   bit 1: 4 warps read the other TMEM buffer (tcgen05.ld 32x32b.x8 + wait, as the epilogue)
//   bit 2: 4 warps store 16 B per lane into shared memory (as the row loaders' transposes)
//   bit 4: 4 warps issue 4-byte-per-lane global stores (as the epilogue, 128 B per instruction)
//   bit 8: the 4 loader warps also issue 128-bit global loads (as the row loaders)
//   bit 16: commit each tile to an mbarrier and wait for it before the next tile (no overlap)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2502_20493_b200/csrc \
//        tools/probes/sched_probe.cu -o tools/probes/bin/sched_probe
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace segb;

struct G { int du, dc, c0, nc, b0; };
// the make_schedule<2, 0, -1> order of igemm_rows_sm100.cu: full window first, then the rest
// (11 MMAs per k-step: N = 256, 2 x 128, 8 x 64)
__constant__ G kSched[11] = {
    {1, 1, 0, 4, 0},                                    // centre: all four classes
    {0, 0, 0, 1, 4}, {0, 1, 0, 2, 5}, {0, 2, 1, 1, 7},  // row window 0 (classes r = 0)
    {1, 0, 0, 1, 8}, {1, 0, 2, 1, 9},                   // column window 0 (classes s = 0)
    {1, 2, 1, 1, 10}, {1, 2, 3, 1, 11},
    {2, 0, 2, 1, 12}, {2, 1, 2, 2, 13}, {2, 2, 3, 1, 15}};

// TMEM class order [0, 1, 3, 2]: three column/row windows become N = 128 (10 MMAs: 256, 3 x 128, 6 x 64)
__constant__ G kSched2[10] = {
    {1, 1, 0, 4, 0}, {0, 0, 0, 1, 4}, {0, 1, 0, 2, 5}, {0, 2, 1, 1, 7}, {1, 0, 0, 1, 8}, {1, 0, 3, 1, 9},
    {1, 2, 1, 2, 10}, {2, 0, 3, 1, 12}, {2, 1, 2, 2, 13}, {2, 2, 2, 1, 15}};

constexpr int kSlot = 17408, kRing = 5, kBTile = 8192;

__global__ void __launch_bounds__(320, 1) sched(int tiles, int mode, int nsched, long long *out, uint32_t *gbuf,
                                                const uint4 *gin) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sB = smem;                 // 16 B tiles of 64 rows x 128 B
    uint8_t *sRing = smem + 16 * kBTile;  // 5 slots
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    __shared__ volatile int done;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < (16 * kBTile + kRing * kSlot) / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); done = 0; }
    fence_proxy_async_smem();
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 1) {
        const uint32_t leader = elect_one();
        const uint64_t dA0 = desc_k_sw128(smem_u32(sRing)), dB0 = desc_k_sw128(smem_u32(sB));
        const uint32_t S16 = kSlot >> 4, B16 = kBTile >> 4;
        long long t0 = clock64();
        uint32_t ph = 0;
        for (int t = 0; t < tiles; ++t) {
            const uint32_t d0 = tmem + (t & 1) * 256;
            const uint32_t sq = t % kRing;
#pragma unroll
            for (int gi = 0; gi < 11; ++gi) {
                if (gi >= nsched || ((mode & 32) && gi >= 10)) break;
                const G g = (mode & 32) ? kSched2[gi] : kSched[gi];
                const uint32_t sl = sq + g.du >= kRing ? sq + g.du - kRing : sq + g.du;
                const uint32_t arow = sl * S16 + g.dc * 8;
                const uint32_t idesc = idesc_bf16_m(128, g.nc * 64);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    tc_mma_pred(d0 + g.c0 * 64, dA0 + arow + kk * 2, dB0 + g.b0 * B16 + kk * 2, idesc,
                                (gi == 0 && kk == 0) ? 0u : 1u, leader);
            }
            if (mode & 16) {
                if (leader) tc_commit(&bar);
                __syncwarp();
                mbar_wait(&bar, ph);
                ph ^= 1;
            }
        }
        if (!(mode & 16)) {
            if (leader) tc_commit(&bar);
            __syncwarp();
            mbar_wait(&bar, 0);
        }
        long long t1 = clock64();
        if (lane == 0) { out[blockIdx.x] = t1 - t0; done = 1; }
    } else if (warp >= 2 && warp <= 5) {  // "epilogue" warps
        const int q = warp - 2;
        uint32_t *gp = gbuf + ((size_t)blockIdx.x * 4 + q) * (1 << 20) + lane;
        int it = 0;
        while (!done) {
            if (mode & 1) {
                uint32_t v[8];
#pragma unroll 1
                for (int c = 0; c < 256; c += 8) {
                    tmem_ld8(tmem + ((uint32_t)(q * 32) << 16) + 256 * ((it & 1) ^ 1) + c, v);
                    tmem_wait_ld();
                    if (mode & 4) {
                        gp[(it * 64 + c / 8 * 2) % (1 << 20) & ~31] = v[0] ^ v[3];
                        gp[(it * 64 + c / 8 * 2 + 32) % (1 << 20) & ~31] = v[5] ^ v[7];
                    }
                }
            } else if (mode & 4) {
#pragma unroll 4
                for (int c = 0; c < 64; ++c) gp[((it * 64 + c) * 32) % (1 << 20)] = c;
            } else {
                break;
            }
            ++it;
        }
    } else if (warp >= 6) {  // "loader" warps
        const int tt = threadIdx.x - 192;
        int it = 0;
        uint4 r = make_uint4(0, 0, 0, 0);
        while (!done) {
            if (mode & 8) r = __ldg(gin + (((size_t)blockIdx.x * 128 + tt) + (size_t)it * 148 * 128) % (1 << 24));
            if (mode & 2) {
                const uint32_t dst = smem_u32(sRing + ((it + 3) % kRing) * kSlot);
#pragma unroll
                for (int w = 0; w < 8; ++w) {
                    const int rho = (tt >> 3) * 8 + w;
                    const uint32_t addr = dst + rho * 128 + (((tt & 7) ^ (rho & 7)) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r.x), "r"(r.y), "r"(r.z),
                                 "r"(r.w)
                                 : "memory");
                }
            } else if (!(mode & 8)) {
                break;
            }
            ++it;
        }
        if (r.x == 12345) gbuf[0] = r.y;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
    long long *d;
    uint32_t *gbuf;
    uint4 *gin;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaMalloc(&gbuf, (size_t)148 * 4 * (1 << 20) * 4);
    cudaMalloc(&gin, (size_t)(1 << 24) * 16);
    cudaMemset(gin, 0, (size_t)(1 << 24) * 16);
    const int smem = 16 * kBTile + kRing * kSlot + 1024;
    cudaFuncSetAttribute(sched, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int tiles = 221;
    struct Case { int mode, nsched; const char *what; } cases[] = {
        {0, 11, "schedule alone"},
        {16, 11, "schedule, commit+wait per tile"},
        {1, 11, "+ TMEM reads (4 warps)"},
        {2, 11, "+ smem stores (4 warps)"},
        {4, 11, "+ global stores (4 warps)"},
        {8, 11, "+ global loads (4 warps)"},
        {1 | 4, 11, "+ TMEM reads feeding global stores"},
        {1 | 4 | 2 | 8, 11, "+ everything"},
        {2 | 8, 11, "+ loads and smem stores"},
        {32, 11, "class order 0,1,3,2 (10 MMAs)"},
        {32 | 1 | 4 | 2 | 8, 11, "class order 0,1,3,2 + everything"},
        {0, 1, "centre window only (N=256)"},
        {0, 4, "centre + row window 0"}, {0, 3, "centre + 2 row-0 windows"},
    };
    for (auto c : cases) {
        for (int rep = 0; rep < 2; ++rep) {
            sched<<<148, 320, smem>>>(tiles, c.mode, c.nsched, d, gbuf, gin);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 148; ++i) avg += h[i];
            avg /= 148;
            if (rep == 1)
                printf("%-44s mode %2d: %7.0f cycles/tile (%s)\n", c.what, c.mode, avg / tiles,
                       e == cudaSuccess ? "ok" : cudaGetErrorString(e));
        }
    }
    return 0;
}
