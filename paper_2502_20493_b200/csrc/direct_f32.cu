// K2 instantiations: fp32 in / fp32 compute / fp32 out (the reference's working precision).
#include "direct_impl.cuh"

namespace segb {
int launch_direct_f32(const DirectArgs &a, bool ref_engine, cudaStream_t st) {
    return launch_direct_typed<float, float, float, false>(a, ref_engine, st);
}
}  // namespace segb
