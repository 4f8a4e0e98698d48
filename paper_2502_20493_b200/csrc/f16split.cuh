// 3xFP16: fp32 operands on the kind::f16 tensor-core path at the fp16 rate (twice kind::tf32's).
//
// A tensor is scaled by a power of two 2^k chosen from its largest magnitude so that every
// scaled value lies below 2^15 (fp16's largest finite value is 65504), then split
//     v * 2^k = hi + lo,   hi = fp16(v * 2^k),   lo = fp16(v * 2^k - hi)
// (the subtraction is exact in fp32). hi and lo carry 11 significant bits each, so hi + lo holds
// ~22 bits: the same precision as 3xTF32's tf32 hi/lo pair (tf32 and fp16 both have 10 stored
// mantissa bits), while the power-of-two scale gives fp16 the exponent range it lacks. A product
// is hi_a*hi_b + hi_a*lo_b + lo_a*hi_b (the dropped lo_a*lo_b is ~2^-22 relative); the products of
// 11-bit operands are exact in the fp32 accumulator, and the result is multiplied back by
// 2^-(k_a + k_b), which is exact. Values below 2^-24 of the tensor's maximum lose their low bits
// (fp16 subnormals): an absolute error of at most ~2^-39 x max|v| x max|w| per product.
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"

namespace segb {

#ifndef SEGB_ABSMAX_BPS
#define SEGB_ABSMAX_BPS 8  // measured: 8 vs 4 blocks per SM, ebgan_l5..l7 fp32 0.7-1 % faster
#endif
constexpr int kAbsmaxBlocks = SEGB_ABSMAX_BPS * 148;  // partial maxima written by absmax_partials_kernel (blocks per SM x 148)
constexpr int kAbsmaxBytes = (kAbsmaxBlocks * 4 + 255) / 256 * 256;

// exponent k with max|v| * 2^k < 2^15; 0 for an all-zero or non-finite maximum
__host__ __device__ inline int f16_scale_exp(float maxabs) {
    if (!(maxabs > 0.f) || maxabs > 3.0e38f) return 0;
    int e;
    frexpf(maxabs, &e);  // maxabs = m * 2^e, m in [0.5, 1)
    const int k = 15 - e;
    return k < -120 ? -120 : (k > 120 ? 120 : k);
}

__device__ __forceinline__ void split_f16(float v, __half &hi, __half &lo) {
    hi = __float2half_rn(v);
    lo = __float2half_rn(v - __half2float(hi));
}

// the same split for two values at once, packed (a in the low half): two paired conversions
// (cvt.rn.f16x2.f32) instead of four scalar ones and the packing; bitwise split_f16's halves
__device__ __forceinline__ void split_f16x2(float a, float b, uint32_t &hi, uint32_t &lo) {
    const __half2 h = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
    hi = *reinterpret_cast<const uint32_t *>(&h);
    lo = *reinterpret_cast<const uint32_t *>(&l);
}

__device__ __forceinline__ uint32_t pack_h2(__half a, __half b) {
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

// max over the kAbsmaxBlocks partial maxima (fmaxf: a NaN partial is ignored, so NaN inputs keep
// a finite scale and propagate through the products as NaN)
__device__ __forceinline__ float reduce_partials(const float *__restrict__ partials) {
    float m = 0.f;
    for (int i = 0; i < kAbsmaxBlocks; ++i) m = fmaxf(m, __ldg(partials + i));
    return m;
}

template <typename T> __device__ __forceinline__ float absf_of(T v) { return fabsf((float)v); }
template <> __device__ __forceinline__ float absf_of<__nv_bfloat16>(__nv_bfloat16 v) {
    return fabsf(__bfloat162float(v));
}

// per-block max |v| over a grid-strided range; exactly kAbsmaxBlocks blocks
template <typename T>
__global__ void __launch_bounds__(256) absmax_partials_kernel(const T *__restrict__ v, int64_t count,
                                                              float *__restrict__ partials) {
    float m = 0.f;
    if constexpr (sizeof(T) == 4) {
        const int64_t n4 = count / 4;
        const float4 *v4 = reinterpret_cast<const float4 *>(v);
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        for (; i + 3 * stride < n4; i += 4 * stride) {  // four 16-byte loads in flight per thread
            float4 a = __ldg(v4 + i), b = __ldg(v4 + i + stride), c = __ldg(v4 + i + 2 * stride),
                   d = __ldg(v4 + i + 3 * stride);
            m = fmaxf(m, fmaxf(fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))),
                               fmaxf(fmaxf(fabsf(b.x), fabsf(b.y)), fmaxf(fabsf(b.z), fabsf(b.w)))));
            m = fmaxf(m, fmaxf(fmaxf(fmaxf(fabsf(c.x), fabsf(c.y)), fmaxf(fabsf(c.z), fabsf(c.w))),
                               fmaxf(fmaxf(fabsf(d.x), fabsf(d.y)), fmaxf(fabsf(d.z), fabsf(d.w)))));
        }
        for (; i < n4; i += stride) {
            float4 a = __ldg(v4 + i);
            m = fmaxf(m, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
        }
        for (int64_t j = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count; j += stride)
            m = fmaxf(m, absf_of(v[j]));
    } else {
        for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x)
            m = fmaxf(m, absf_of(v[j]));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    __shared__ float wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, wm[w]);
        partials[blockIdx.x] = m;
    }
}

// host launcher: partials[kAbsmaxBlocks] = per-block max |v| (dtype: SEGB_F32 / F64 / BF16)
int run_absmax_partials(const void *v, int dtype, int64_t count, float *partials, cudaStream_t st);

}  // namespace segb
