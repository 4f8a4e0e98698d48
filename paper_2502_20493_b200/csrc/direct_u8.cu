// K2 instantiations: the dataset path's interleaved u8 image payload (B, H, W, C) decoded on load
// (float32(u8) / 255, tensor_io.py:52) / fp32 compute / fp32 out (fused), on
// K2 and on the paired FFMA2 kernel K2p (direct_pair.cuh).
#include "direct_pair.cuh"

namespace segb {
int launch_direct_u8(const DirectArgs &a, bool ref_engine, cudaStream_t st) {
    return launch_direct_typed<uint8_t, float, float, false>(a, ref_engine, st);
}
int launch_direct_pair_u8(const DirectArgs &a, const float *w_host, cudaStream_t st) {
    return launch_direct_pair<uint8_t>(a, w_host, st);
}
}  // namespace segb
