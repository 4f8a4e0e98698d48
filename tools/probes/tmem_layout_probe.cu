// Probe (not part of the library): register layout of tcgen05.ld.16x256b. TMEM is filled with
// tcgen05.st.32x32b (thread t -> lane t, register j -> column j) with value lane * 1000 + col,
// then read back with .16x256b.x2 at lane 0 / column 0 of warp 0's quarter; prints, for each
// thread and register, the (lane, column) it received.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2502_20493_b200/csrc \
//        tools/probes/tmem_layout_probe.cu -o tools/probes/bin/tmem_layout_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace segb;

__global__ void probe(uint32_t *out) {
    __shared__ uint32_t tslot;
    const int t = threadIdx.x;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = t * 1000 + j;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(tmem),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem));
    tmem_wait_ld();
    for (int j = 0; j < 8; ++j) out[t * 8 + j] = r[j];
    uint32_t s[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]), "=r"(s[7])
                 : "r"(tmem + (16u << 16)));
    tmem_wait_ld();
    for (int j = 0; j < 8; ++j) out[256 + t * 8 + j] = s[j];
    tc_fence_before();
    __syncthreads();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
    uint32_t *d, h[512];
    cudaMalloc(&d, sizeof(h));
    probe<<<1, 32>>>(d);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int part = 0; part < 2; ++part) {
        printf("ld 16x256b.x2 at lane offset %d:\n", part * 16);
        for (int t = 0; t < 32; ++t) {
            printf("t%2d:", t);
            for (int j = 0; j < 8; ++j) printf(" (%2u,%2u)", h[part * 256 + t * 8 + j] / 1000, h[part * 256 + t * 8 + j] % 1000);
            printf("\n");
        }
    }
    return 0;
}
