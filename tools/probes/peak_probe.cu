// Probe (not part of the library): the compute peaks the bench's rooflines divide by, measured
// on this B200 instead of derived from datasheets ("measure the FFMA and kind::tf32
// peaks on the box").
//   - tcgen05.mma issue-rate peaks: kind::f16 (bf16 and fp16 operands) and kind::tf32, M = 128
//     (cta_group::1) with N = 256 and independent accumulators, one CTA per SM, all 148 SMs,
//     K-major SWIZZLE_128B operands already in shared memory (no memory traffic): the hardware
//     ceiling of the MMA kinds the fp32 paths use;
//   - FFMA: 148 x 4 warps x independent FMA chains.
// Each number is FLOP / (device time of the launch), CUDA events, best of 5, with the SM clock
// read by clock64 / globaltimer over the same launch (so a power-capped clock shows up).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I paper_2502_20493_b200/csrc \
//        tools/probes/peak_probe.cu -o tools/probes/bin/peak_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace segb;

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// kind: 0 = bf16 (kind::f16), 1 = fp16 (kind::f16), 2 = tf32 (kind::tf32)
__global__ void __launch_bounds__(128, 1) mma_peak(int kind, int iters, long long *cyc, unsigned long long *ns) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;          // 4 A tiles of 128 rows x 128 B
    uint8_t *sB = smem + 65536;  // B: 256 rows x 128 B
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
        const int N = 256;
        uint32_t idesc;
        if (kind == 2) idesc = idesc_tf32(N);
        else if (kind == 1) idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        else idesc = idesc_bf16(N);
        const uint32_t aLo = desc_lo_sw128(smem_u32(sA)), bLo = desc_lo_sw128(smem_u32(sB));
        const long long c0 = clock64();
        const uint64_t g0 = gtimer();
        if (kind == 2) {
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    tc_mma_lo<1, true>(tmem + (j & 1) * 256, aLo + (j & 3) * 1024 + (j & 3) * 2, bLo + (j & 3) * 2,
                                       idesc, 1u, leader);
            }
        } else {
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    tc_mma_lo<1, false>(tmem + (j & 1) * 256, aLo + (j & 3) * 1024 + (j & 3) * 2, bLo + (j & 3) * 2,
                                        idesc, 1u, leader);
            }
        }
        if (leader) tc_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        const long long c1 = clock64();
        const uint64_t g1 = gtimer();
        if (threadIdx.x == 0) {
            cyc[blockIdx.x] = c1 - c0;
            ns[blockIdx.x] = g1 - g0;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// FFMA with all three operands in registers (the direct kernel's x * w + acc), and its packed
// FFMA2 form (two fp32 FMAs per lane per instruction, sm_100)
__global__ void __launch_bounds__(256) ffma_reg_peak(int iters, const float *bw, float *out) {
    float a[16];
    const float b = bw[threadIdx.x & 7], c = bw[8 + (threadIdx.x & 7)];
    float bb[16], cr[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) { a[k] = threadIdx.x * 1e-7f + k; bb[k] = b + k * 1e-9f; cr[k] = c - k * 1e-9f; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = fmaf(bb[k], a[k], cr[k]);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += a[k];
    if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) ffma2_peak(int iters, const float *bw, float *out) {
    float2 a[8], bb[8];
    const float b = bw[threadIdx.x & 7], c = bw[8 + (threadIdx.x & 7)];
    const float2 cc = make_float2(c, c);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        a[k] = make_float2(threadIdx.x * 1e-7f + k, k + 0.5f);
        bb[k] = make_float2(b + k * 1e-9f, b - k * 1e-9f);
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __ffma2_rn(bb[k], a[k], cc);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k].x + a[k].y;
    if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) ffma_peak(int iters, float *out) {
    float a[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = threadIdx.x * 1e-7f + k;
    const float b = 0.9999f, c = 1e-6f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = fmaf(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += a[k];
    if (s == 12345.f) out[threadIdx.x] = s;  // never true; keeps the chains alive
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *dc;
    unsigned long long *dn;
    float *df;
    cudaMalloc(&dc, sms * sizeof(long long));
    cudaMalloc(&dn, sms * sizeof(unsigned long long));
    cudaMalloc(&df, 1024 * sizeof(float));
    const int smem = 65536 + 32768 + 1024;
    cudaFuncSetAttribute(mma_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[3] = {"bf16 kind::f16", "fp16 kind::f16", "tf32 kind::tf32"};
    printf("{\"sms\": %d", sms);
    for (int kind = 0; kind < 3; ++kind) {
        const int iters = 1 << 16;
        double best = 0, best_mhz = 0, best_cyc_per = 0;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            mma_peak<<<sms, 128, smem>>>(kind, iters, dc, dn);
            cudaEventRecord(e1);
            cudaError_t err = cudaEventSynchronize(e1);
            if (err != cudaSuccess) {
                printf(", \"error\": \"%s\"}\n", cudaGetErrorString(err));
                return 1;
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            long long hc[256];
            unsigned long long hn[256];
            cudaMemcpy(hc, dc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
            cudaMemcpy(hn, dn, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
            double cyc = 0, nsec = 0;
            for (int i = 0; i < sms; ++i) { cyc += hc[i]; nsec += hn[i]; }
            cyc /= sms;
            nsec /= sms;
            // per MMA: M=128, N=256, K = 32 B of K (16 bf16/fp16 or 8 tf32 elements)
            const double kel = kind == 2 ? 8 : 16;
            const double flop = 2.0 * 128 * 256 * kel * iters * sms;
            const double tf = flop / (ms * 1e-3) / 1e12;
            if (tf > best) { best = tf; best_mhz = cyc / nsec * 1e3; best_cyc_per = cyc / iters; }
        }
        printf(", \"%s\": {\"tflops\": %.1f, \"cycles_per_mma_n256\": %.2f, \"sm_mhz\": %.0f}", names[kind], best,
               best_cyc_per, best_mhz);
    }
    {
        const int iters = 1 << 14, blocks = sms * 8;
        double best = 0;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            ffma_peak<<<blocks, 256>>>(iters, df);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flop = 2.0 * 16 * iters * 256.0 * blocks;
            const double tf = flop / (ms * 1e-3) / 1e12;
            if (tf > best) best = tf;
        }
        printf(", \"ffma\": {\"tflops\": %.1f}", best);
    }
    {  // register-operand FFMA and FFMA2
        float hb[16];
        for (int i = 0; i < 16; ++i) hb[i] = 0.999f + i * 1e-6f;
        float *dbw;
        cudaMalloc(&dbw, sizeof hb);
        cudaMemcpy(dbw, hb, sizeof hb, cudaMemcpyHostToDevice);
        const int iters = 1 << 14, blocks = sms * 8;
        for (int v = 0; v < 2; ++v) {
            double best = 0;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(e0);
                if (v == 0) ffma_reg_peak<<<blocks, 256>>>(iters, dbw, df);
                else ffma2_peak<<<blocks, 256>>>(iters, dbw, df);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                const double flop = 2.0 * 16 * iters * 256.0 * blocks;
                const double tf = flop / (ms * 1e-3) / 1e12;
                if (tf > best) best = tf;
            }
            printf(", \"%s\": {\"tflops\": %.1f}", v == 0 ? "ffma_reg" : "ffma2_reg", best);
        }
    }
    printf("}\n");
    return 0;
}
