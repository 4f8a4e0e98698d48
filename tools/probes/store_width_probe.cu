// Probe (not part of the library): HBM write bandwidth by store width (4 / 8 / 16 B per lane)
// and by warps per SM, with one persistent CTA per SM -- the shape of K3b's epilogue (4 warps
// per SM storing 4-byte bf16x2 pairs, 128 B per warp instruction).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probes/store_width_probe.cu -o tools/probes/bin/store_width_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void k_store(T *y, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    T v;
    memset(&v, 0, sizeof(T));
#pragma unroll 8
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) y[i] = v;
}

int main() {
    const size_t bytes = (size_t)2150 << 20;
    void *y;
    cudaMalloc(&y, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char *name, auto launch) {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it && ms < best) best = ms;
        }
        printf("%-34s %7.3f ms %7.0f GB/s (%s)\n", name, best, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    for (int warps : {4, 8, 16, 32}) {
        char nm[64];
        const int blk = warps * 32;
        snprintf(nm, sizeof nm, "4 B/lane, %2d warps/SM", warps);
        run(nm, [&] { k_store<uint32_t><<<148, blk>>>((uint32_t *)y, bytes / 4); });
        snprintf(nm, sizeof nm, "8 B/lane, %2d warps/SM", warps);
        run(nm, [&] { k_store<uint2><<<148, blk>>>((uint2 *)y, bytes / 8); });
        snprintf(nm, sizeof nm, "16 B/lane, %2d warps/SM", warps);
        run(nm, [&] { k_store<uint4><<<148, blk>>>((uint4 *)y, bytes / 16); });
    }
    return 0;
}
