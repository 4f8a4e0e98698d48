// K2 instantiations for bf16 compute: operands rounded to bf16 (weights by K1,
// fp32 activations on load), exact products, fp32 accumulation -- the same
// arithmetic contract as the tcgen05 kind::f16 path, so both paths agree.
#include "direct_impl.cuh"

namespace segb {
int launch_direct_bf16(const DirectArgs &a, int x_dtype, int y_dtype, bool ref_engine, cudaStream_t st) {
    if (x_dtype == SEGB_BF16 && y_dtype == SEGB_BF16)
        return launch_direct_typed<__nv_bfloat16, float, __nv_bfloat16, false>(a, ref_engine, st);
    if (x_dtype == SEGB_BF16 && y_dtype == SEGB_F32)
        return launch_direct_typed<__nv_bfloat16, float, float, false>(a, ref_engine, st);
    if (x_dtype == SEGB_F32 && y_dtype == SEGB_BF16)
        return launch_direct_typed<float, float, __nv_bfloat16, true>(a, ref_engine, st);
    if (x_dtype == SEGB_F32 && y_dtype == SEGB_F32)
        return launch_direct_typed<float, float, float, true>(a, ref_engine, st);
    return fail(SEGB_ERR_VALUE, "bf16 compute supports x/y dtypes f32 or bf16 (got %d/%d)", x_dtype, y_dtype);
}
}  // namespace segb
