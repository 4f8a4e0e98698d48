// K1 -- device-side kernel segregation, once per weight tensor.
//
// Reference: segregation.py:61-70 (segregate_kernel: k_rs = K[r::2, s::2]),
// segregation.py:73-88 (merge_subkernels) and the per-class weight layout of
// PreparedLayer.__init__, engines.py:236-244. All copies are bit-exact
// permutations (plus an optional round-to-nearest-even cast to bf16).
#include "common.cuh"
#include "f16split.cuh"
#include "kernels.cuh"

namespace segb {

// class of tap (i, j) of an n x n kernel and its index inside the packed vector
__device__ __forceinline__ int packed_index(int n, int i, int j) {
    const int r = i & 1, s = j & 1, u = i >> 1, v = j >> 1;
    return class_offset(n, 2 * r + s) + u * sub_len(n, s) + v;
}

// inverse: packed index k -> (i, j)
__device__ __forceinline__ void unpack_index(int n, int k, int &i, int &j) {
    int c = 3;
    while (c > 0 && k < class_offset(n, c)) --c;
    const int r = c >> 1, s = c & 1, cols = sub_len(n, s);
    const int rem = k - class_offset(n, c);
    i = 2 * (rem / cols) + r;
    j = 2 * (rem % cols) + s;
}

template <typename T>
__global__ void segregate_kernel_k(const T *__restrict__ kern, T *__restrict__ subs, int64_t count, int n) {
    const int64_t total = count * n * n;
    const int n2 = n * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / n2;
        const int ij = (int)(e - k * n2), i = ij / n, j = ij % n;
        const int r = i & 1, s = j & 1, rows = sub_len(n, r), cols = sub_len(n, s);
        const int64_t dst = count * class_offset(n, 2 * r + s) + k * rows * cols + (i >> 1) * cols + (j >> 1);
        subs[dst] = kern[e];
    }
}

template <typename T>
__global__ void merge_kernel_k(const T *__restrict__ subs, T *__restrict__ kern, int64_t count, int n) {
    const int64_t total = count * n * n;
    const int n2 = n * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / n2;
        const int ij = (int)(e - k * n2), i = ij / n, j = ij % n;
        const int r = i & 1, s = j & 1, rows = sub_len(n, r), cols = sub_len(n, s);
        const int64_t src = count * class_offset(n, 2 * r + s) + k * rows * cols + (i >> 1) * cols + (j >> 1);
        kern[e] = subs[src];
    }
}

template <typename TS> __device__ __forceinline__ double to_f64(TS v) { return (double)v; }
template <> __device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 v) {
    return (double)__bfloat162float(v);
}

// Direct-kernel layout (K2): dst[(co * c_in + ci) * n2p + k] where k is the
// class-packed tap index (packed=1) or the raw u * n + v index (packed=0,
// reference engine); k >= n*n is zero padding. mode: 0 fp32, 1 fp64,
// 2 fp32 holding bf16-rounded values.
template <typename TS>
__global__ void prep_direct_kernel(const TS *__restrict__ bank, void *dst, int c_in, int c_out, int n,
                                   int n2p, int packed, int mode) {
    const int64_t total = (int64_t)c_out * c_in * n2p;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e % n2p);
        const int64_t cc = e / n2p;
        const int ci = (int)(cc % c_in), co = (int)(cc / c_in);
        double v = 0.0;
        if (k < n * n) {
            int i, j;
            if (packed) unpack_index(n, k, i, j);
            else { i = k / n; j = k % n; }
            v = to_f64(bank[(((int64_t)ci * c_out + co) * n + i) * n + j]);
        }
        if (mode == 1) reinterpret_cast<double *>(dst)[e] = v;
        else if (mode == 0) reinterpret_cast<float *>(dst)[e] = (float)v;
        else reinterpret_cast<float *>(dst)[e] = round_bf16((float)v);
    }
}

// Implicit-GEMM layout (K3): per class c and sub-kernel tap (u, v), a K-major
// [c_out_pad][c_in_pad] bf16 matrix: dst[((tapbase(c) + u*C + v) * c_out_pad + co) * c_in_pad + ci]
// = bf16(K[ci, co, 2u + r, 2v + s]); tap bases follow the class-packed order; the padding
// rows/columns are zero.
template <typename TS>
__global__ void prep_gemm_kernel(const TS *__restrict__ bank, __nv_bfloat16 *dst, int c_in, int c_in_pad,
                                 int c_out, int c_out_pad, int n) {
    const int64_t total = (int64_t)n * n * c_out_pad * c_in_pad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int ci = (int)(e % c_in_pad);
        const int64_t rest = e / c_in_pad;
        const int co = (int)(rest % c_out_pad);
        const int k = (int)(rest / c_out_pad);  // class-packed tap index
        float v = 0.f;
        if (ci < c_in && co < c_out) {
            int i, j;
            unpack_index(n, k, i, j);
            v = (float)to_f64(bank[(((int64_t)ci * c_out + co) * n + i) * n + j]);
        }
        dst[e] = __float2bfloat16_rn(v);
    }
}

// 3xTF32 operand split: hi = x rounded to TF32 (10-bit mantissa, round-to-nearest),
// lo = TF32(x - hi); x ~= hi + lo to ~2^-22 relative.
__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// [tap][c_out_pad][c_in_pad] fp32 hi and lo planes for kind::tf32 (see prep_gemm_kernel)
template <typename TS>
__global__ void prep_gemm_tf32_kernel(const TS *__restrict__ bank, float *hi, float *lo, int c_in, int c_in_pad,
                                      int c_out, int c_out_pad, int n) {
    const int64_t total = (int64_t)n * n * c_out_pad * c_in_pad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int ci = (int)(e % c_in_pad);
        const int64_t rest = e / c_in_pad;
        const int co = (int)(rest % c_out_pad);
        const int k = (int)(rest / c_out_pad);
        float v = 0.f;
        if (ci < c_in && co < c_out) {
            int i, j;
            unpack_index(n, k, i, j);
            v = (float)to_f64(bank[(((int64_t)ci * c_out + co) * n + i) * n + j]);
        }
        const float h = tf32_rn(v);
        hi[e] = h;
        lo[e] = tf32_rn(v - h);
    }
}

// [tap][c_out_pad][c_in_pad] fp16 hi and lo planes for 3xFP16 (f16split.cuh): the bank scaled
// by 2^k_w (k_w from the bank's largest magnitude, reduced into `partials` beforehand) and split
template <typename TS>
__global__ void prep_gemm_f16x2_kernel(const TS *__restrict__ bank, __half *hi, __half *lo, int c_in, int c_in_pad,
                                       int c_out, int c_out_pad, int n, const float *__restrict__ partials) {
    __shared__ float scale;
    if (threadIdx.x == 0) scale = ldexpf(1.f, f16_scale_exp(reduce_partials(partials)));
    __syncthreads();
    const int64_t total = (int64_t)n * n * c_out_pad * c_in_pad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int ci = (int)(e % c_in_pad);
        const int64_t rest = e / c_in_pad;
        const int co = (int)(rest % c_out_pad);
        const int k = (int)(rest / c_out_pad);
        float v = 0.f;
        if (ci < c_in && co < c_out) {
            int i, j;
            unpack_index(n, k, i, j);
            v = (float)to_f64(bank[(((int64_t)ci * c_out + co) * n + i) * n + j]);
        }
        __half h, l;
        split_f16(v * scale, h, l);
        hi[e] = h;
        lo[e] = l;
    }
}

static unsigned grid_for(int64_t total) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 148 * 32));
}

int run_segregate(const void *kern, int dtype, int64_t count, int n, void *subs, bool merge, cudaStream_t st) {
    const int64_t total = count * n * n;
    if (total == 0) return SEGB_OK;
    const unsigned g = grid_for(total);
    switch (dtype_size(dtype)) {
        case 2:
            if (merge) merge_kernel_k<uint16_t><<<g, 256, 0, st>>>((const uint16_t *)kern, (uint16_t *)subs, count, n);
            else segregate_kernel_k<uint16_t><<<g, 256, 0, st>>>((const uint16_t *)kern, (uint16_t *)subs, count, n);
            break;
        case 4:
            if (merge) merge_kernel_k<uint32_t><<<g, 256, 0, st>>>((const uint32_t *)kern, (uint32_t *)subs, count, n);
            else segregate_kernel_k<uint32_t><<<g, 256, 0, st>>>((const uint32_t *)kern, (uint32_t *)subs, count, n);
            break;
        case 8:
            if (merge) merge_kernel_k<uint64_t><<<g, 256, 0, st>>>((const uint64_t *)kern, (uint64_t *)subs, count, n);
            else segregate_kernel_k<uint64_t><<<g, 256, 0, st>>>((const uint64_t *)kern, (uint64_t *)subs, count, n);
            break;
        default: return fail(SEGB_ERR_VALUE, "unknown dtype %d", dtype);
    }
    note_launch();
    return check_launch(merge ? "merge_kernel" : "segregate_kernel");
}

int run_prep_direct(const void *bank, int bank_dtype, int c_in, int c_out, int n, int n2p, bool packed,
                    int mode, void *dst, cudaStream_t st) {
    const int64_t total = (int64_t)c_out * c_in * n2p;
    const unsigned g = grid_for(total);
    switch (bank_dtype) {
        case SEGB_F32:
            prep_direct_kernel<float><<<g, 256, 0, st>>>((const float *)bank, dst, c_in, c_out, n, n2p, packed, mode);
            break;
        case SEGB_F64:
            prep_direct_kernel<double><<<g, 256, 0, st>>>((const double *)bank, dst, c_in, c_out, n, n2p, packed, mode);
            break;
        case SEGB_BF16:
            prep_direct_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16 *)bank, dst, c_in, c_out, n,
                                                                 n2p, packed, mode);
            break;
        default: return fail(SEGB_ERR_VALUE, "unknown bank dtype %d", bank_dtype);
    }
    note_launch();
    return check_launch("prep_direct_kernel");
}

int run_prep_gemm(const void *bank, int bank_dtype, int c_in, int c_in_pad, int c_out, int c_out_pad, int n,
                  void *dst, cudaStream_t st) {
    const int64_t total = (int64_t)n * n * c_out_pad * c_in_pad;
    const unsigned g = grid_for(total);
    __nv_bfloat16 *d = (__nv_bfloat16 *)dst;
    switch (bank_dtype) {
        case SEGB_F32: prep_gemm_kernel<float><<<g, 256, 0, st>>>((const float *)bank, d, c_in, c_in_pad, c_out, c_out_pad, n); break;
        case SEGB_F64: prep_gemm_kernel<double><<<g, 256, 0, st>>>((const double *)bank, d, c_in, c_in_pad, c_out, c_out_pad, n); break;
        case SEGB_BF16:
            prep_gemm_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16 *)bank, d, c_in, c_in_pad, c_out, c_out_pad, n);
            break;
        default: return fail(SEGB_ERR_VALUE, "unknown bank dtype %d", bank_dtype);
    }
    note_launch();
    return check_launch("prep_gemm_kernel");
}

}  // namespace segb

namespace segb {
int run_prep_gemm_tf32(const void *bank, int bank_dtype, int c_in, int c_in_pad, int c_out, int c_out_pad, int n,
                       void *hi, void *lo, cudaStream_t st) {
    const int64_t total = (int64_t)n * n * c_out_pad * c_in_pad;
    const unsigned g = grid_for(total);
    float *h = (float *)hi, *l = (float *)lo;
    switch (bank_dtype) {
        case SEGB_F32:
            prep_gemm_tf32_kernel<float><<<g, 256, 0, st>>>((const float *)bank, h, l, c_in, c_in_pad, c_out, c_out_pad, n);
            break;
        case SEGB_F64:
            prep_gemm_tf32_kernel<double><<<g, 256, 0, st>>>((const double *)bank, h, l, c_in, c_in_pad, c_out, c_out_pad, n);
            break;
        case SEGB_BF16:
            prep_gemm_tf32_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16 *)bank, h, l, c_in, c_in_pad,
                                                                    c_out, c_out_pad, n);
            break;
        default: return fail(SEGB_ERR_VALUE, "unknown bank dtype %d", bank_dtype);
    }
    note_launch();
    return check_launch("prep_gemm_tf32_kernel");
}
}  // namespace segb

namespace segb {
int run_absmax_partials(const void *v, int dtype, int64_t count, float *partials, cudaStream_t st) {
    switch (dtype) {
        case SEGB_F32: absmax_partials_kernel<float><<<kAbsmaxBlocks, 256, 0, st>>>((const float *)v, count, partials); break;
        case SEGB_F64: absmax_partials_kernel<double><<<kAbsmaxBlocks, 256, 0, st>>>((const double *)v, count, partials); break;
        case SEGB_BF16:
            absmax_partials_kernel<__nv_bfloat16><<<kAbsmaxBlocks, 256, 0, st>>>((const __nv_bfloat16 *)v, count, partials);
            break;
        default: return fail(SEGB_ERR_VALUE, "unknown dtype %d", dtype);
    }
    note_launch();
    return check_launch("absmax_partials_kernel");
}

int run_prep_gemm_f16x2(const void *bank, int bank_dtype, int c_in, int c_in_pad, int c_out, int c_out_pad, int n,
                        void *hi, void *lo, float *partials, cudaStream_t st) {
    if (int rc = run_absmax_partials(bank, bank_dtype, (int64_t)c_in * c_out * n * n, partials, st)) return rc;
    const int64_t total = (int64_t)n * n * c_out_pad * c_in_pad;
    const unsigned g = grid_for(total);
    __half *h = (__half *)hi, *l = (__half *)lo;
    switch (bank_dtype) {
        case SEGB_F32:
            prep_gemm_f16x2_kernel<float><<<g, 256, 0, st>>>((const float *)bank, h, l, c_in, c_in_pad, c_out,
                                                             c_out_pad, n, partials);
            break;
        case SEGB_F64:
            prep_gemm_f16x2_kernel<double><<<g, 256, 0, st>>>((const double *)bank, h, l, c_in, c_in_pad, c_out,
                                                              c_out_pad, n, partials);
            break;
        case SEGB_BF16:
            prep_gemm_f16x2_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16 *)bank, h, l, c_in, c_in_pad,
                                                                     c_out, c_out_pad, n, partials);
            break;
        default: return fail(SEGB_ERR_VALUE, "unknown bank dtype %d", bank_dtype);
    }
    note_launch();
    return check_launch("prep_gemm_f16x2_kernel");
}
}  // namespace segb
