// Probe (not part of the library): achievable HBM bandwidth for EB-GAN l7's traffic mix
// (read 0.54 GB, write 2.15 GB: 1 byte read per 4 written) with plain 128-bit streaming
// kernels, next to pure read, pure write and 1:1 copy, all on 1 GiB-class buffers.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probes/mix_bw_probe.cu -o tools/probes/bin/mix_bw_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write(uint4 *y, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        y[i] = make_uint4((uint32_t)i, 1, 2, 3);
}
__global__ void k_read(const uint4 *x, size_t n, uint32_t *sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldg(x + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678) *sink = acc;
}
__global__ void k_copy(const uint4 *x, uint4 *y, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        y[i] = __ldg(x + i);
}
// read one vector, write `R` vectors (y is R x larger), all coalesced
template <int R>
__global__ void k_mix(const uint4 *x, uint4 *y, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldg(x + i);
#pragma unroll
        for (int r = 0; r < R; ++r) y[(size_t)r * n + i] = make_uint4(v.x + r, v.y, v.z, v.w);
    }
}

int main() {
    const size_t nx = (size_t)537 << 20 >> 4;  // 0.54 GB of uint4
    uint4 *x, *y;
    uint32_t *sink;
    cudaMalloc(&x, nx * 16);
    cudaMalloc(&y, 4 * nx * 16);
    cudaMalloc(&sink, 4);
    cudaMemset(x, 1, nx * 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto time = [&](const char *what, double bytes, auto launch) {
        float best = 1e9;
        for (int it = 0; it < 8; ++it) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it > 0 && ms < best) best = ms;
        }
        printf("%-40s %8.3f ms  %7.0f GB/s  (%s)\n", what, best, bytes / best / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int bpsm : {4, 8, 16}) {
        const int grid = sms * bpsm, blk = 512;
        printf("grid %d x %d\n", grid, blk);
        time("write 2.15 GB", 4.0 * nx * 16, [&] { k_write<<<grid, blk>>>(y, 4 * nx); });
        time("read 0.54 GB", 1.0 * nx * 16, [&] { k_read<<<grid, blk>>>(x, nx, sink); });
        time("read 2.15 GB", 4.0 * nx * 16, [&] { k_read<<<grid, blk>>>(y, 4 * nx, sink); });
        time("copy 0.54 GB -> 0.54 GB", 2.0 * nx * 16, [&] { k_copy<<<grid, blk>>>(x, y, nx); });
        time("mix 1:4 (0.54 GB read, 2.15 GB write)", 5.0 * nx * 16, [&] { k_mix<4><<<grid, blk>>>(x, y, nx); });
        time("mix 1:2", 3.0 * nx * 16, [&] { k_mix<2><<<grid, blk>>>(x, y, nx); });
    }
    return 0;
}
