// K2 instantiations: the dataset path's interleaved u8 image payload (B, H, W, C) decoded on load
// (float32(u8) / 255, tensor_io.py:52) / fp32 compute / fp32 out (fused).
#include "direct_impl.cuh"

namespace segb {
int launch_direct_u8(const DirectArgs &a, bool ref_engine, cudaStream_t st) {
    return launch_direct_typed<uint8_t, float, float, false>(a, ref_engine, st);
}
}  // namespace segb
