// Device-side synthetic inputs with the reference's exact bits.
// synth.py:20-39: element i = float32(float64(splitmix64(seed + i)) * 2^-64):
// u64 -> f64 round-to-nearest, exact scaling, f64 -> f32 round-to-nearest
// (numpy's astype chain), optionally rounded on to bf16.
#include "common.cuh"
#include "kernels.cuh"

namespace segb {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void unit_floats_kernel(T *out, int64_t count, uint64_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = __ull2double_rn(splitmix64(seed + (uint64_t)i)) * 0x1p-64;
        const float f = __double2float_rn(d);
        if constexpr (sizeof(T) == 4) out[i] = f;
        else out[i] = __float2bfloat16_rn(f);
    }
}

int run_unit_floats(void *out, int dtype, int64_t count, uint64_t seed, cudaStream_t st) {
    if (count <= 0) return SEGB_OK;
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(count, 256), 148 * 64);
    if (dtype == SEGB_F32) unit_floats_kernel<float><<<g, 256, 0, st>>>((float *)out, count, seed);
    else if (dtype == SEGB_BF16) unit_floats_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((__nv_bfloat16 *)out, count, seed);
    else return fail(SEGB_ERR_VALUE, "unit_floats supports f32 or bf16 (got %d)", dtype);
    note_launch();
    return check_launch("unit_floats_kernel");
}

}  // namespace segb
