// Probe (not part of the library): HBM write bandwidth of plain coalesced stores, the ceiling of
// an epilogue that writes 4.24 GB of fp32 (ebgan_l7 at batch 256) with and without a concurrent
// 1.07 GB read stream, for 8-byte and 16-byte per-lane stores and a few grid shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probes/store_probe.cu -o tools/probes/bin/store_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int VEC>
__global__ void write_k(float *y, long long n, const float *x, long long nx, float s) {
    const long long stride = (long long)gridDim.x * blockDim.x * VEC;
    float acc = 0.f;
    long long rx = (long long)(blockIdx.x * blockDim.x + threadIdx.x) * 4;
    const long long xstride = (long long)gridDim.x * blockDim.x * 4;
    int k = 0;
    for (long long i = (long long)(blockIdx.x * blockDim.x + threadIdx.x) * VEC; i < n; i += stride, ++k) {
        if (x && (k & 3) == 0 && rx < nx) {  // one 16-byte read per four 16-byte writes
            float4 v = __ldg(reinterpret_cast<const float4 *>(x + rx));
            acc += v.x + v.w;
            rx += xstride;
        }
        if constexpr (VEC == 2) *reinterpret_cast<float2 *>(y + i) = make_float2(s + acc, s);
        else *reinterpret_cast<float4 *>(y + i) = make_float4(s + acc, s, s, s);
    }
}

int main() {
    const long long n = 4240ll * 1000 * 1000 / 4, nx = 1070ll * 1000 * 1000 / 4;
    float *y, *x;
    cudaMalloc(&y, n * 4);
    cudaMalloc(&x, nx * 4);
    cudaMemset(x, 0, nx * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("{\"bytes_written\": %lld", n * 4);
    for (int mixed = 0; mixed < 2; ++mixed)
        for (int vec = 2; vec <= 4; vec += 2)
            for (int bpsm : {-4, -8, -16, 1, 2, 4, 8}) {
                // bpsm < 0: one block of -bpsm warps per SM
                const int blocks = bpsm < 0 ? sms : sms * bpsm, threads = bpsm < 0 ? -bpsm * 32 : 256;
                float best = 1e9;
                for (int rep = 0; rep < 4; ++rep) {
                    cudaEventRecord(e0);
                    if (vec == 2) write_k<2><<<blocks, threads>>>(y, n, mixed ? x : nullptr, nx, 1.f);
                    else write_k<4><<<blocks, threads>>>(y, n, mixed ? x : nullptr, nx, 1.f);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                const double bytes = n * 4.0 + (mixed ? nx * 4.0 : 0);
                printf(", \"%s_v%d_%s%d\": {\"ms\": %.3f, \"GBs\": %.0f}", mixed ? "rw" : "w", vec, bpsm < 0 ? "warps" : "b", bpsm < 0 ? -bpsm : bpsm, best,
                       bytes / best / 1e6);
            }
    printf("}\n");
    return 0;
}
