// Dataset-style inputs straight to the device. The reference decodes a
// binary P6 PPM into a (3, H, W) float32 tensor in [0, 1] on the host
// (tensor_io.py:27-52: pixels.transpose(2, 0, 1).astype(float32) / float32(255)). Here only the
// raw interleaved u8 payload crosses PCIe (a quarter of the fp32 bytes) and one kernel
// deinterleaves HWC -> CHW and scales, with the same IEEE fp32 division (no fast math), so the
// device tensor is bitwise the reference's.
#include "common.cuh"
#include "kernels.cuh"

namespace segb {

// one thread per output element, output-major so stores are coalesced; the u8 reads of a
// warp span 32 consecutive pixels of one channel (3-byte stride, same cache lines)
template <typename T>
__global__ void u8_hwc_to_chw_kernel(const uint8_t *src, T *dst, int64_t images, int hw, int c) {
    const int64_t total = images * (int64_t)c * hw;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / ((int64_t)c * hw);
        const int rem = (int)(i - b * c * (int64_t)hw);
        const int ch = rem / hw, p = rem - ch * hw;
        const float v = (float)src[(b * hw + p) * c + ch] / 255.0f;
        if constexpr (sizeof(T) == 4) dst[i] = v;
        else if constexpr (sizeof(T) == 8) dst[i] = (double)v;
        else dst[i] = __float2bfloat16_rn(v);
    }
}

int run_u8_hwc_to_chw(const void *src, int64_t images, int height, int width, int channels, void *dst,
                      int dst_dtype, cudaStream_t st) {
    const int64_t total = images * (int64_t)channels * height * width;
    if (total <= 0) return SEGB_OK;
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 32);
    const int hw = height * width;
    const uint8_t *s = (const uint8_t *)src;
    if (dst_dtype == SEGB_F32) u8_hwc_to_chw_kernel<float><<<g, 256, 0, st>>>(s, (float *)dst, images, hw, channels);
    else if (dst_dtype == SEGB_F64) u8_hwc_to_chw_kernel<double><<<g, 256, 0, st>>>(s, (double *)dst, images, hw, channels);
    else u8_hwc_to_chw_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(s, (__nv_bfloat16 *)dst, images, hw, channels);
    note_launch();
    return check_launch("u8_hwc_to_chw_kernel");
}

}  // namespace segb

extern "C" int segb_u8_hwc_to_chw(const void *src, int64_t images, int height, int width, int channels, void *dst,
                                  int dst_dtype, void *stream) {
    using namespace segb;
    if (images < 0 || height < 1 || width < 1 || channels < 1)
        return fail(SEGB_ERR_SHAPE, "image batch dims must be >= 1, got %lldx%dx%dx%d", (long long)images, height,
                    width, channels);
    if (dst_dtype != SEGB_F32 && dst_dtype != SEGB_F64 && dst_dtype != SEGB_BF16)
        return fail(SEGB_ERR_VALUE, "unknown dtype %d", dst_dtype);
    if (images > 0 && (!src || !dst)) return fail(SEGB_ERR_VALUE, "null tensor");
    return run_u8_hwc_to_chw(src, images, height, width, channels, dst, dst_dtype, (cudaStream_t)stream);
}
