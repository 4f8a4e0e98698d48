// Probe (not part of the library): tcgen05.mma issue rate for the shapes K3b uses.
// One CTA per SM issues `iters` MMAs (SS operands, SWIZZLE_128B K-major tiles) in a
// given pattern and reports cycles per MMA:
//   same-D chains (every MMA accumulates into the previous one's D) vs. rotating over
//   `nd` independent accumulators, for N = 64 / 128 / 256, M = 128 (cta_group::1) and
//   M = 64.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2502_20493_b200/csrc \
//        tools/probes/mma_rate_probe.cu -o tools/probes/bin/mma_rate_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace segb;

__global__ void __launch_bounds__(128, 1) rate(int m, int n, int nd, int arows_shift, int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;               // 8 A tiles of 128 rows x 128 B (distinct windows)
    uint8_t *sB = smem + 8 * 16384;   // B: 256 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < (8 * 16384 + 32768) / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    fence_proxy_async_smem();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        const uint32_t leader = elect_one();
        const uint32_t idesc = idesc_bf16_m(m, n);
        const uint64_t dA = desc_k_sw128(smem_u32(sA)), dB = desc_k_sw128(smem_u32(sB));
        const int dstep = 512 / nd;  // TMEM column stride between accumulators
        long long t0 = clock64();
        if (arows_shift < 0) {  // lean loop: 8 MMAs per iteration, descriptors precomputed;
                                // shift -1: 1024-aligned A tiles, -2: A tiles shifted by j % 3 rows
            uint64_t as[8];
            uint32_t ds[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                as[j] = dA + (uint64_t)((j * 16384 + (arows_shift == -2 ? (j % 3) * 128 : 0)) >> 4) + (j & 3) * 2;
                ds[j] = tmem + (j % nd) * dstep;
            }
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) tc_mma_pred(ds[j], as[j], dB + (j & 3) * 2, idesc, 1u, leader);
            }
        } else {
            for (int i = 0; i < iters; ++i) {
                const int d = i % nd;
                // A window: rotate over 8 tiles, optionally shifted by rows (as K3b's windows)
                const uint64_t a = dA + (uint64_t)(((i % 8) * 16384 + (i % 3) * arows_shift * 128) >> 4) + (i & 3) * 2;
                tc_mma_pred(tmem + d * dstep, a, dB + (i & 3) * 2, idesc, i >= nd, leader);
            }
        }
        if (leader) tc_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    const int smem = 8 * 16384 + 32768 + 1024;
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 4096;
    struct Case { int m, n, nd, shift; } cases[] = {
        {128, 64, 1, -1}, {128, 64, 4, -1}, {128, 128, 1, -1}, {128, 128, 4, -1}, {128, 32, 1, -1}, {128, 16, 1, -1},
        {64, 64, 1, -1}, {64, 128, 2, -1}, {128, 192, 1, -1},
        {128, 64, 1, -2}, {128, 128, 1, -2}, {128, 256, 1, -2}, {64, 64, 1, -2}, {64, 128, 1, -2},
        {128, 64, 1, 0}, {128, 64, 2, 0}, {128, 64, 4, 0}, {128, 64, 8, 0}, {128, 64, 4, 1},
        {128, 128, 1, 0}, {128, 128, 2, 0}, {128, 128, 4, 0},
        {128, 256, 1, 0}, {128, 256, 2, 0},
        {64, 64, 1, 0}, {64, 64, 4, 0}, {64, 128, 1, 0}, {64, 128, 4, 0}, {64, 256, 2, 0},
    };
    for (auto c : cases) {
        for (int grid : {1, 148}) {
            rate<<<grid, 128, smem>>>(c.m, c.n, c.nd, c.shift, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < grid; ++i) avg += h[i];
            avg /= grid;
            const double floor_cyc = (c.m < 128 ? 128 : c.m) * c.n / 256.0;
            printf("M=%3d N=%3d accumulators=%d shift=%d grid=%3d: %7.1f cycles/MMA (floor %5.1f) %s\n", c.m, c.n,
                   c.nd, c.shift, grid, avg / iters, floor_cyc, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
