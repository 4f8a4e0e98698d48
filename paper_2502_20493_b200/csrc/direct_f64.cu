// K2 instantiations: fp64 in / compute / out (the reference's oracle-grade mode).
#include "direct_impl.cuh"

namespace segb {
int launch_direct_f64(const DirectArgs &a, bool ref_engine, cudaStream_t st) {
    return launch_direct_typed<double, double, double, false>(a, ref_engine, st);
}
}  // namespace segb
