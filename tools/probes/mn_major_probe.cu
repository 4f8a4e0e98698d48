// Probe (not part of the library): UMMA descriptor fields for an MN-major SWIZZLE_128B A
// operand laid out the way a TMA box {64 positions, 64 channels} of an NCHW tensor lands
// in shared memory: box h (positions 64h..64h+63) at 8192 h, channel k's 128-byte row at
// 128 k, 16-byte chunk c of that row at chunk c ^ (k & 7).
// A[m][k] = m (k = 0, 16), 1 (k = 1, 17); B[n][k] = 1 (k = 0, 16), 1024 n (k = 1, 17), so two
// K=16 MMAs (the second starting 2 channel atoms = 2048 B further) give D = 2 (m + 1024 n).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2502_20493_b200/csrc \
//        tools/probes/mn_major_probe.cu -o tools/probes/bin/mn_major_probe
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace segb;

constexpr int N = 16;

__device__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}

__global__ void __launch_bounds__(128, 1) probe(int variant, float *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;          // 2 boxes x 8 KB
    uint8_t *sB = smem + 16384;  // N rows x 128 B, K-major SW128
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int i = tid; i < 128 * 64; i += 128) {
        const int m = i / 64, k = i % 64;
        float a = 0.f;
        if (k == 0 || k == 16) a = (float)m;
        if (k == 1 || k == 17) a = 1.f;
        const int h = m / 64, mm = m % 64;
        const int off = h * 8192 + k * 128 + (((mm / 8) ^ (k & 7)) << 4) + (mm % 8) * 2;
        *reinterpret_cast<__nv_bfloat16 *>(sA + off) = __float2bfloat16(a);
    }
    for (int i = tid; i < N * 64; i += 128) {
        const int n = i / 64, k = i % 64;
        float b = 0.f;
        if (k == 0 || k == 16) b = 1.f;
        if (k == 1 || k == 17) b = 1024.f * n;
        const int off = n * 128 + (((k / 8) ^ (n & 7)) << 4) + (k % 8) * 2;
        *reinterpret_cast<__nv_bfloat16 *>(sB + off) = __float2bfloat16(b);
    }
    if (tid == 0) mbar_init(&bar, 1);
    fence_proxy_async_smem();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                     "r"(32));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0 && elect_one()) {
        const uint32_t idesc = idesc_bf16_m(128, N) | (1u << 15);  // A MN-major
        const uint32_t lbo = variant == 0 ? 8192 : 1024, sbo = variant == 0 ? 1024 : 8192;
        for (int kk = 0; kk < 2; ++kk)
            tc_mma(tmem, desc_mn(smem_u32(sA) + kk * 2048, lbo, sbo), desc_k_sw128(smem_u32(sB) + kk * 32), idesc,
                   kk);
        tc_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
    tmem_wait_ld();
    for (int j = 0; j < N; ++j) out[(warp * 32 + lane) * N + j] = __uint_as_float(v[j]);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
    float *d;
    cudaMalloc(&d, 128 * N * sizeof(float));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int variant = 0; variant < 2; ++variant) {
        cudaMemset(d, 0, 128 * N * sizeof(float));
        probe<<<1, 128, 32768>>>(variant, d);
        cudaError_t e = cudaDeviceSynchronize();
        static float h[128 * N];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < N; ++n)
                if (h[m * N + n] != 2.f * (m + 1024.f * n)) ++bad;
        printf("variant %d (%s): %s, mismatches %d / %d; D[5][3]=%.0f D[100][7]=%.0f (expect %.0f, %.0f)\n", variant,
               variant == 0 ? "LBO=8192 SBO=1024" : "LBO=1024 SBO=8192", cudaGetErrorString(e), bad, 128 * N,
               h[5 * N + 3], h[100 * N + 7], 2.f * (5 + 1024 * 3), 2.f * (100 + 1024 * 7));
    }
    return 0;
}
