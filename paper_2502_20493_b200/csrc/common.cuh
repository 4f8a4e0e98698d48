// Shared helpers of the segb200 library: error state, dtype traits, launch counter.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/segb200.h"

namespace segb {

// thread-local last-error message (segb_last_error)
void set_error(const char *fmt, ...);
int fail(int code, const char *fmt, ...);
void note_launch(int n = 1);

// returns SEGB_ERR_CUDA with a message if the last launch failed
int check_launch(const char *what);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline size_t dtype_size(int dt) {
    switch (dt) {
        case SEGB_F32: return 4;
        case SEGB_F64: return 8;
        case SEGB_BF16: return 2;
        default: return 0;
    }
}

// Sub-kernel side for a parity (segregation.py:53-58): ceil(n/2) for 0, floor(n/2) for 1.
__host__ __device__ inline int sub_len(int n, int parity) { return parity == 0 ? (n + 1) / 2 : n / 2; }

// Offset of class c = 2r + s inside an n*n class-packed tap vector [k00|k01|k10|k11].
__host__ __device__ inline int class_offset(int n, int c) {
    const int a = (n + 1) / 2, b = n / 2;
    switch (c) {
        case 0: return 0;
        case 1: return a * a;
        case 2: return a * a + a * b;
        default: return a * a + 2 * a * b;
    }
}

// element load/store conversions
__device__ __forceinline__ float ld_as_float(const float *p) { return __ldg(p); }
__device__ __forceinline__ float ld_as_float(const __nv_bfloat16 *p) { return __bfloat162float(*p); }
__device__ __forceinline__ double ld_as_double(const double *p) { return __ldg(p); }

template <typename T> __device__ __forceinline__ T from_float(float v);
template <> __device__ __forceinline__ float from_float<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_float<__nv_bfloat16>(float v) {
    return __float2bfloat16_rn(v);
}

__device__ __forceinline__ float round_bf16(float v) {
    return __bfloat162float(__float2bfloat16_rn(v));
}

}  // namespace segb
