// Probe (not part of the library): latencies of the handshakes K3b's pipeline is made of --
//   (1) tcgen05.commit -> mbarrier completion seen by the committing warp (no MMA in flight,
//       and after one M=128 N=256 MMA);
//   (2) fence.proxy.async.shared::cta after 128 threads stored 16 KB to shared memory;
//   (3) a ping-pong of mbarrier arrive / wait between two warps of a CTA, and between two CTAs
//       of a cluster (remote arrive, cluster-scope wait).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2502_20493_b200/csrc \
//        tools/probes/sync_latency_probe.cu -o tools/probes/bin/sync_latency_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace segb;

constexpr int kIters = 256;

__global__ void __launch_bounds__(256, 1) probe_commit_fence(long long *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[4];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        const uint32_t leader = elect_one();
        // (1a) commit with nothing in flight
        uint32_t ph = 0;
        long long t0 = clock64();
        for (int i = 0; i < kIters; ++i) {
            tc_commit_pred(&bar[0], leader);
            __syncwarp();
            mbar_wait(&bar[0], ph);
            ph ^= 1;
        }
        long long t1 = clock64();
        // (1b) one MMA (M=128, N=256, K=16) then commit
        const uint64_t dA = desc_k_sw128(smem_u32(smem)), dB = desc_k_sw128(smem_u32(smem + 16384));
        ph = 0;
        long long t2 = clock64();
        for (int i = 0; i < kIters; ++i) {
            tc_mma_pred(tmem, dA, dB, idesc_bf16_m(128, 256), 0u, leader);
            tc_commit_pred(&bar[1], leader);
            __syncwarp();
            mbar_wait(&bar[1], ph);
            ph ^= 1;
        }
        long long t3 = clock64();
        if (lane == 0) {
            out[0] = (t1 - t0) / kIters;
            out[1] = (t3 - t2) / kIters;
        }
    } else if (warp >= 4) {  // (2) 128 threads store 16 KB, fence.proxy.async, named barrier
        const int tt = threadIdx.x - 128;
        long long acc = 0;
        for (int i = 0; i < kIters; ++i) {
            for (int k = 0; k < 8; ++k)
                asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(smem_u32(smem + 32768 + (k * 128 + tt) * 16)),
                             "r"(i)
                             : "memory");
            long long a = clock64();
            fence_proxy_async_smem();
            long long b = clock64();
            acc += b - a;
        }
        if (tt == 0) out[2] = acc / kIters;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// (3) ping-pong: warp 0 arrives on A and waits B; warp 1 (or the peer CTA's warp 0) waits A and
// arrives on B. Reports cycles per round trip.
__global__ void __launch_bounds__(64, 1) probe_pingpong(long long *out, int remote) {
    __shared__ uint64_t bar[2];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = remote ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (remote) cluster_sync_all();
    const bool ping = remote ? (rank == 0 && warp == 0) : warp == 0;
    const bool pong = remote ? (rank == 1 && warp == 0) : warp == 1;
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
        if (ping) {
            if (lane == 0) {
                if (remote) mbar_arrive_cluster(mapa_rank(&bar[0], 1));
                else mbar_arrive(&bar[0]);
            }
            if (remote) mbar_wait_cluster(&bar[1], ph);
            else mbar_wait(&bar[1], ph);
        } else if (pong) {
            if (remote) mbar_wait_cluster(&bar[0], ph);
            else mbar_wait(&bar[0], ph);
            if (lane == 0) {
                if (remote) mbar_arrive_cluster(mapa_rank(&bar[1], 0));
                else mbar_arrive(&bar[1]);
            }
        }
        ph ^= 1;
    }
    long long t1 = clock64();
    if (ping && lane == 0) out[remote ? 4 : 3] = (t1 - t0) / kIters;
    __syncthreads();
    if (remote) cluster_sync_all();
}

int main() {
    long long *d, h[8] = {0};
    cudaMalloc(&d, sizeof(h));
    cudaMemset(d, 0, sizeof(h));
    cudaFuncSetAttribute(probe_commit_fence, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    probe_commit_fence<<<1, 256, 65536 + 1024>>>(d);
    printf("commit/fence: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    probe_pingpong<<<1, 64>>>(d, 0);
    printf("local ping-pong: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(64);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, probe_pingpong, d, 1);
    printf("cluster ping-pong: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("tcgen05.commit -> mbarrier, nothing in flight: %lld cycles\n", h[0]);
    printf("MMA (128x256x16) + commit -> mbarrier:       %lld cycles\n", h[1]);
    printf("fence.proxy.async after 16 KB of st.shared:  %lld cycles\n", h[2]);
    printf("mbarrier ping-pong, two warps of a CTA:       %lld cycles per round trip\n", h[3]);
    printf("mbarrier ping-pong, two CTAs of a cluster:    %lld cycles per round trip\n", h[4]);
    return 0;
}
