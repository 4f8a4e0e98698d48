// Probe (not part of the library): tcgen05.ld read throughput per SM by load shape, loads in
// flight per wait, and number of reading warps (one CTA per SM, 512 TMEM columns, every
// warp reads its own lane quarter, columns rotate over the allocation).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2502_20493_b200/csrc \
//        tools/probes/tmem_ld_probe.cu -o tools/probes/bin/tmem_ld_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace segb;

template <int X>
__device__ __forceinline__ void ld32x32b(uint32_t taddr, uint32_t *v);
template <>
__device__ __forceinline__ void ld32x32b<8>(uint32_t taddr, uint32_t *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
template <>
__device__ __forceinline__ void ld32x32b<16>(uint32_t taddr, uint32_t *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
template <>
__device__ __forceinline__ void ld32x32b<32>(uint32_t taddr, uint32_t *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
// 16 lanes x 256 bit (x2: two such blocks): lanes [0,16) of the warp's quarter, 8 columns each
template <int X>
__device__ __forceinline__ void ld16x256b(uint32_t taddr, uint32_t *v);
template <>
__device__ __forceinline__ void ld16x256b<2>(uint32_t taddr, uint32_t *v) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
template <>
__device__ __forceinline__ void ld16x256b<4>(uint32_t taddr, uint32_t *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

// SHAPE 0: 32x32b.xX (X regs, 32 lanes x X columns = 128 X bytes); SHAPE 1: 16x256b.x(X/8)
// DEPTH loads issued per tcgen05.wait::ld
template <int SHAPE, int X, int DEPTH>
__global__ void __launch_bounds__(512, 1) tmem_rd(int iters, int nwarps, long long *out, uint32_t *sink) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    uint32_t acc = 0;
    long long t0 = clock64();
    if (warp < nwarps) {
        const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        uint32_t v[DEPTH][X];
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
                const uint32_t col = ((i * DEPTH + d) * X + (warp >> 2) * 256) & 511;
                if (SHAPE == 0) ld32x32b<X>(base + col, v[d]);
                else ld16x256b<X / 8>(base + col, v[d]);
            }
            tmem_wait_ld();
#pragma unroll
            for (int d = 0; d < DEPTH; ++d)
#pragma unroll
                for (int k = 0; k < X; ++k) acc += v[d][k];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345) *sink = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int SHAPE, int X, int DEPTH>
void run(const char *name, int nwarps, long long *d, uint32_t *sink) {
    const int iters = 2048;
    tmem_rd<SHAPE, X, DEPTH><<<148, 512>>>(iters, nwarps, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    tmem_rd<SHAPE, X, DEPTH><<<148, 512>>>(iters, nwarps, d, sink);
    e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    // bytes per load per warp: 32x32b.xX = 32 lanes * 4 B * X; 16x256b.x(X/8) = 16 lanes * 32 B * X/8
    const double bytes_per_ld = SHAPE == 0 ? 128.0 * X : 64.0 * X;
    const double bytes = bytes_per_ld * DEPTH * iters * nwarps;
    printf("%-14s x%-2d depth %d warps %2d: %6.1f B/cycle/SM (%s)\n", name, X, DEPTH, nwarps, bytes / avg,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
}

int main() {
    long long *d;
    uint32_t *sink;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaMalloc(&sink, 4);
    for (int nw : {4, 8, 16}) {
        run<0, 8, 1>("32x32b", nw, d, sink);
        run<0, 8, 4>("32x32b", nw, d, sink);
        run<0, 16, 1>("32x32b", nw, d, sink);
        run<0, 16, 2>("32x32b", nw, d, sink);
        run<0, 32, 1>("32x32b", nw, d, sink);
        run<0, 32, 2>("32x32b", nw, d, sink);
        run<1, 16, 1>("16x256b", nw, d, sink);
        run<1, 16, 2>("16x256b", nw, d, sink);
    }
    return 0;
}
