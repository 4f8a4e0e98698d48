// Probe (not part of the library): tcgen05.mma kind::f16 (fp16 operands) issue rate per shape,
// cta_group::1, one CTA per SM on every SM, operands resident in shared memory, back-to-back
// MMAs into two alternating accumulators. Shows how much of the N = 256 peak the narrow shapes
// the rows kernel issues (M = 64 / 128 per SM, N = 32..128) can reach.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I paper_2502_20493_b200/csrc \
//        tools/probes/mma_shape_probe.cu -o tools/probes/bin/mma_shape_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace segb;

__global__ void __launch_bounds__(128, 1) mma_shape(uint32_t idesc, int iters, long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem, *sB = smem + 65536;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < (65536 + 32768) / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
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
        const uint32_t aLo = desc_lo_sw128(smem_u32(sA)), bLo = desc_lo_sw128(smem_u32(sB));
        const long long c0 = clock64();
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                tc_mma_lo<1, false>(tmem + (j & 1) * 256, aLo + (j & 3) * 1024 + (j & 3) * 2, bLo + (j & 3) * 2,
                                    idesc, 1u, leader);
        }
        if (leader) tc_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// the same through a 2-CTA cluster: the leader issues tcgen05.mma.cta_group::2 (M = 128: 64 rows
// per SM, or M = 256: 128 per SM; B split N/2 per CTA), the commit arrives at both CTAs
__global__ void __launch_bounds__(128, 1) mma_shape_pair(uint32_t idesc, int iters, long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem, *sB = smem + 65536;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x; i < (65536 + 32768) / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async_smem();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        const long long c0 = clock64();
        if (rank == 0) {
            const uint32_t leader = elect_one();
            const uint32_t aLo = desc_lo_sw128(smem_u32(sA)), bLo = desc_lo_sw128(smem_u32(sB));
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    tc_mma_lo<2, false>(tmem + (j & 1) * 256, aLo + (j & 3) * 1024 + (j & 3) * 2, bLo + (j & 3) * 2,
                                        idesc, 1u, leader);
            }
            tc_commit_2sm_mc_pred(&bar, 3, leader);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *dc;
    cudaMalloc(&dc, sms * sizeof(long long));
    const int smem = 65536 + 32768 + 1024;
    cudaFuncSetAttribute(mma_shape, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int ms[2] = {128, 64}, ns[5] = {256, 128, 64, 32, 16};
    printf("{\"unit\": \"SM cycles per MMA (K = 16 fp16) and fp16 MACs per SM cycle\"");
    for (int m : ms)
        for (int n : ns) {
            const uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
            const int iters = 1 << 15;
            double best = 1e30;
            for (int rep = 0; rep < 3; ++rep) {
                mma_shape<<<sms, 128, smem>>>(idesc, iters, dc);
                if (cudaDeviceSynchronize() != cudaSuccess) { printf(", \"error\": 1}\n"); return 1; }
                long long hc[256];
                cudaMemcpy(hc, dc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
                double c = 0;
                for (int i = 0; i < sms; ++i) c += hc[i];
                c /= sms * (double)iters;
                if (c < best) best = c;
            }
            printf(", \"M%d_N%d\": {\"cycles\": %.2f, \"macs_per_cycle\": %.0f}", m, n, best, m * n * 16.0 / best);
        }
    cudaFuncSetAttribute(mma_shape_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int pms[2] = {256, 128}, pns[5] = {256, 128, 64, 32, 16};
    for (int m : pms)
        for (int n : pns) {
            const uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
            const int iters = 1 << 15;
            double best = 1e30;
            for (int rep = 0; rep < 3; ++rep) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(sms / 2 * 2);
                cfg.blockDim = dim3(128);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = 2;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, mma_shape_pair, idesc, iters, dc);
                if (cudaDeviceSynchronize() != cudaSuccess) { printf(", \"error_pair\": 1}\n"); return 1; }
                long long hc[256];
                cudaMemcpy(hc, dc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
                double c = 0;
                for (int i = 0; i < sms; ++i) c += hc[i];
                c /= sms * (double)iters;
                if (c < best) best = c;
            }
            // per SM: M/2 rows x N columns x 16
            printf(", \"pair_M%d_N%d\": {\"cycles\": %.2f, \"macs_per_sm_cycle\": %.0f}", m, n, best,
                   m / 2 * n * 16.0 / best);
        }
    printf("}\n");
    return 0;
}
