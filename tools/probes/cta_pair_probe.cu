// Probe (not part of the library): where does tcgen05.mma.cta_group::2 put its rows and
// columns? A CTA pair (cluster of 2) holds A rows [r*MC, (r+1)*MC) and B columns
// [r*N/2, (r+1)*N/2) in its own shared memory at identical offsets; the leader issues one
// M = 2*MC MMA with A[m][0] = m, A[m][1] = 1, B[n][0] = 1, B[n][1] = 1024*n, so
// D[m][n] = m + 1024 n. Every warp of both CTAs then dumps its TMEM lane quarter.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2502_20493_b200/csrc \
//        tools/probes/cta_pair_probe.cu -o /tmp/cta_pair_probe && /tmp/cta_pair_probe
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace segb;

constexpr int N = 64;  // MMA N (each CTA holds N/2 B rows)

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float *out) {
    __shared__ __align__(1024) uint8_t sA[128 * 128];
    __shared__ __align__(1024) uint8_t sB[128 * 128];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t rank = cluster_rank();
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    // SW128 K-major tiles: row r, 16-byte chunk c at r*128 + ((c ^ (r & 7)) << 4)
    for (int i = tid; i < 128 * 64; i += 128) {
        const int r = i / 64, k = i % 64;
        const int off = r * 128 + (((k / 8) ^ (r & 7)) << 4) + (k % 8) * 2;
        float a = 0.f, b = 0.f;
        if (r < MC) a = k == 0 ? (float)(rank * MC + r) : (k == 1 ? 1.f : 0.f);
        if (r < N / 2) b = k == 0 ? 1.f : (k == 1 ? 1024.f * (rank * (N / 2) + r) : 0.f);
        *reinterpret_cast<__nv_bfloat16 *>(sA + off) = __float2bfloat16(a);
        *reinterpret_cast<__nv_bfloat16 *>(sB + off) = __float2bfloat16(b);
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async_smem();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                     "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (rank == 0 && warp == 0 && elect_one()) {
        const uint32_t idesc = idesc_bf16_m(2 * MC, N);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(desc_k_sw128(smem_u32(sA))), "l"(desc_k_sw128(smem_u32(sB))), "r"(idesc));
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3)
            : "memory");
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
        tmem_wait_ld();
        for (int j = 0; j < 8; ++j) out[((rank * 128) + warp * 32 + lane) * N + c0 + j] = __uint_as_float(v[j]);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

template <int MC>
static void run() {
    float *d;
    cudaMalloc(&d, 2 * 128 * N * sizeof(float));
    cudaMemset(d, 0xff, 2 * 128 * N * sizeof(float));
    probe<MC><<<2, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    printf("== M = %d (MC = %d per CTA): %s\n", 2 * MC, MC, cudaGetErrorString(e));
    static float h[2 * 128 * N];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int r = 0; r < 2; ++r)
        for (int lane = 0; lane < 128; lane += (lane % 16 == 15 ? 1 : 15)) {
            const float *p = h + (r * 128 + lane) * N;
            printf("cta %d lane %3d: col0 -> m %.0f n %.0f | col31 -> m %.0f n %.0f | col32 -> m %.0f n %.0f | col63 -> m %.0f n %.0f\n", r,
                   lane, fmodf(p[0], 1024.f), floorf(p[0] / 1024.f), fmodf(p[31], 1024.f), floorf(p[31] / 1024.f),
                   fmodf(p[32], 1024.f), floorf(p[32] / 1024.f), fmodf(p[63], 1024.f), floorf(p[63] / 1024.f));
        }
    cudaFree(d);
}

int main() {
    run<128>();
    run<64>();
    return 0;
}
