// K3 interface: per-parity-class implicit GEMM on tcgen05/TMEM (igemm_sm100.cu).
#pragma once

#include "common.cuh"

namespace segb {

struct IgemmShape {
    int64_t batch;
    int c_in, c_out, h, w, n, pad, x_dtype, y_dtype, c_in_pad, c_out_pad, c_in_pad32;
    int compute;  // SEGB_BF16 (kind::f16) or SEGB_F32 (3xFP16 on kind::f16, or 3xTF32 on kind::tf32)
    int f16x3;    // fp32 compute as 3xFP16 (weights: scaled fp16 hi / lo planes)
    int w_exp;    // 3xFP16: the weight planes' scale exponent k_w
};

bool igemm_available();
bool igemm_supported(const IgemmShape &s);
const char *igemm_kernel_name(const IgemmShape &s);  // the kernel family run_igemm picks
// workspace (bytes) run_igemm needs for this shape: K3's NHWC operand copy or K3c's tap products
int64_t igemm_workspace_bytes(const IgemmShape &s);
int run_igemm(const IgemmShape &s, const void *x, const void *wg, const void *wg_lo, void *y, void *ws,
              int64_t ws_bytes, cudaStream_t st);

// K3c: input-stationary scatter GEMM + gather for narrow outputs (igemm_scatter_sm100.cu)
bool igemm_scatter_supported(const IgemmShape &s);
int scatter_weight_rows(int c_out, int n);
int run_prep_scatter(const void *bank, int bank_dtype, int c_in, int c_in_pad, int c_out, int n, void *dst,
                     cudaStream_t st);
int64_t igemm_scatter_workspace_bytes(const IgemmShape &s);
int run_igemm_scatter(const IgemmShape &s, const void *x, const void *wz, void *y, void *ws, int64_t ws_bytes,
                      cudaStream_t st);

// K3p: class-pair tiles as 2-SM CTA pairs over K3's operands (igemm_cp_sm100.cu)
bool igemm_cp_supported(const IgemmShape &s);
int run_igemm_cp_core(const IgemmShape &s, const void *x_nhwc, const void *wg, void *y, cudaStream_t st);

// K3b: row-streaming variant for wide class grids (igemm_rows_sm100.cu)
bool igemm_rows_supported(const IgemmShape &s);
int igemm_rows_variant(const IgemmShape &s);  // its CTA split (3 / 4: 2-SM pairs), 0 if unsupported
int64_t igemm_rows_workspace_bytes(const IgemmShape &s);  // 3xFP16: the input's absmax partials
int run_igemm_rows(const IgemmShape &s, const void *x, const void *wg, const void *wg_lo, void *y, void *ws,
                   int64_t ws_bytes, cudaStream_t st);

}  // namespace segb
