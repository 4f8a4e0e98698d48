// Host-side launchers of the segb200 kernels (internal to the library).
#pragma once

#include "common.cuh"

namespace segb {

// K1 (segregate.cu)
int run_segregate(const void *kern, int dtype, int64_t count, int n, void *subs, bool merge, cudaStream_t st);
int run_prep_direct(const void *bank, int bank_dtype, int c_in, int c_out, int n, int n2p, bool packed,
                    int mode, void *dst, cudaStream_t st);
int run_prep_gemm(const void *bank, int bank_dtype, int c_in, int c_in_pad, int c_out, int c_out_pad, int n,
                  void *dst, cudaStream_t st);

int run_prep_gemm_tf32(const void *bank, int bank_dtype, int c_in, int c_in_pad, int c_out, int c_out_pad, int n,
                       void *hi, void *lo, cudaStream_t st);

// 3xFP16 weights (f16split.cuh): absmax of the bank into partials[kAbsmaxBlocks], then the scaled
// fp16 hi / lo planes in the K3 layout
int run_prep_gemm_f16x2(const void *bank, int bank_dtype, int c_in, int c_in_pad, int c_out, int c_out_pad, int n,
                        void *hi, void *lo, float *partials, cudaStream_t st);

// synthetic inputs (synth.cu)
int run_unit_floats(void *out, int dtype, int64_t count, uint64_t seed, cudaStream_t st);

// dataset images (image_io.cu)
int run_u8_hwc_to_chw(const void *src, int64_t images, int height, int width, int channels, void *dst,
                      int dst_dtype, cudaStream_t st);

}  // namespace segb
