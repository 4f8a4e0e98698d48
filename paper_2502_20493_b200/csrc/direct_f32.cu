// K2 instantiations: fp32 in / fp32 compute / fp32 out (the reference's working precision), and
// the paired FFMA2 kernel K2p for the low-channel layers (direct_pair.cuh).
#include "direct_pair.cuh"

namespace segb {
int launch_direct_f32(const DirectArgs &a, bool ref_engine, cudaStream_t st) {
    return launch_direct_typed<float, float, float, false>(a, ref_engine, st);
}
int launch_direct_pair_f32(const DirectArgs &a, const float *w_host, cudaStream_t st) {
    return launch_direct_pair<float>(a, w_host, st);
}
int launch_direct_pair_wsm(const DirectArgs &a, cudaStream_t st) { return launch_direct_pair_wsm_impl(a, st); }
}  // namespace segb
