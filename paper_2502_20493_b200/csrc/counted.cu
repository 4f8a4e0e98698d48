// The instrumented scalar engines on the device (engines.py:353-406 of the reference:
// transpose_conv_reference_counted / transpose_conv_segregated_counted).
//
// The reference runs these as plain-Python loops over one feature map: fp64 accumulation in
// (u, v) order, one `acc += x * w` per tap (a rounded multiply, then a rounded add: no fused
// multiply-add), a mults counter bumped per product and a writes counter per stored output.
// Here one thread owns one output element and does exactly that; the counters are the number
// of multiplications the threads executed and the number of stores they issued, summed with
// one atomic per warp, so they are measured by the kernel rather than derived from a formula.
#include "common.cuh"

namespace segb {
namespace {

__device__ __forceinline__ double load_f64(const void *p, int dt, int64_t i) {
    return dt == SEGB_F64 ? static_cast<const double *>(p)[i] : (double)static_cast<const float *>(p)[i];
}

// engine 1 (segregated, engines.py:379-406): r = (x + swap) % 2, base = (x + r) / 2, taps
// K[2u + r, 2v + s] of the class sub-kernel (segregation.py:61-70), input zero-padded by P / 2.
// engine 0 (reference, engines.py:353-376): the bed-of-nails upsampled map padded by P,
// correlated with all n x n taps (zeros included, as the reference counts them).
__global__ void counted_kernel(const void *__restrict__ fmap, int fdt, int h, int w, const void *__restrict__ kern,
                               int kdt, int n, int pad, int engine, int out_h, int out_w, double *__restrict__ out,
                               unsigned long long *__restrict__ counters) {
    const int64_t total = (int64_t)out_h * out_w;
    unsigned long long mults = 0, writes = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(e / out_w), y = (int)(e % out_w);
        double acc = 0.0;
        if (engine == SEGB_ENGINE_SEGREGATED) {
            const int p = pad / 2, swap = pad & 1;
            const int r = (x + swap) % 2, s = (y + swap) % 2;
            const int bx = (x + r) / 2, by = (y + s) / 2;
            const int R = sub_len(n, r), C = sub_len(n, s);
            for (int u = 0; u < R; ++u) {
                const int i = bx + u - p;
                for (int v = 0; v < C; ++v) {
                    const int j = by + v - p;
                    const double xv = (i >= 0 && i < h && j >= 0 && j < w) ? load_f64(fmap, fdt, (int64_t)i * w + j) : 0.0;
                    const double kv = load_f64(kern, kdt, (2 * u + r) * n + 2 * v + s);
                    acc = __dadd_rn(acc, __dmul_rn(xv, kv));
                    ++mults;
                }
            }
        } else {
            const int uh = 2 * h - 1, uw = 2 * w - 1;  // upsampled extent (tensors.py:85-95)
            for (int u = 0; u < n; ++u) {
                const int i = x + u - pad;  // row of the upsampled map
                for (int v = 0; v < n; ++v) {
                    const int j = y + v - pad;
                    double xv = 0.0;
                    if (i >= 0 && i < uh && j >= 0 && j < uw && !(i & 1) && !(j & 1))
                        xv = load_f64(fmap, fdt, (int64_t)(i / 2) * w + j / 2);
                    const double kv = load_f64(kern, kdt, u * n + v);
                    acc = __dadd_rn(acc, __dmul_rn(xv, kv));
                    ++mults;
                }
            }
        }
        out[e] = acc;
        ++writes;
    }
    // one atomic per warp and counter
    for (int o = 16; o > 0; o >>= 1) {
        mults += __shfl_down_sync(0xFFFFFFFFu, mults, o);
        writes += __shfl_down_sync(0xFFFFFFFFu, writes, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (mults) atomicAdd(&counters[0], mults);
        if (writes) atomicAdd(&counters[1], writes);
    }
}

}  // namespace
}  // namespace segb

using namespace segb;

extern "C" int segb_counted_forward(const void *fmap, int fmap_dtype, int in_h, int in_w, const void *kernel,
                                    int kernel_dtype, int kernel_n, int pad, int engine, double *out,
                                    unsigned long long *counters, void *stream) {
    if ((fmap_dtype != SEGB_F32 && fmap_dtype != SEGB_F64) || (kernel_dtype != SEGB_F32 && kernel_dtype != SEGB_F64))
        return fail(SEGB_ERR_VALUE, "counted engines take f32 or f64 tensors (got %d / %d)", fmap_dtype, kernel_dtype);
    if (engine != SEGB_ENGINE_REFERENCE && engine != SEGB_ENGINE_SEGREGATED)
        return fail(SEGB_ERR_VALUE, "unknown engine %d", engine);
    int oh, ow;
    if (int rc = segb_output_dims(in_h, in_w, kernel_n, pad, &oh, &ow)) return rc;
    if (!fmap || !kernel || !out || !counters) return fail(SEGB_ERR_VALUE, "null tensor");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return fail(SEGB_ERR_CUDA, "counter reset: %s", cudaGetErrorString(e));
    const int64_t total = (int64_t)oh * ow;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 148 * 16));
    counted_kernel<<<grid, 256, 0, st>>>(fmap, fmap_dtype, in_h, in_w, kernel, kernel_dtype, kernel_n, pad, engine,
                                        oh, ow, out, counters);
    note_launch();
    return check_launch("counted_kernel");
}
