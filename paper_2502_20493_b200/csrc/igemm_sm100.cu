// K3 placeholder (filled in by the tcgen05 implementation).
#include "igemm.cuh"

namespace segb {
bool igemm_available() { return false; }
bool igemm_supported(const IgemmShape &) { return false; }
int run_igemm(const IgemmShape &, const void *, const void *, void *, cudaStream_t) {
    return fail(SEGB_ERR_UNSUPPORTED, "implicit GEMM not built");
}
}  // namespace segb
