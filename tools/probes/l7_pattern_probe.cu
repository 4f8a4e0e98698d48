// Probe (not part of the library): HBM bandwidth with EB-GAN l7's access pattern and no
// compute: per tile (b, i) read input row i of 64 channel planes (64 x 256 B, NCHW 256x64x128x128
// bf16) and write output rows 2i, 2i+1 of 64 planes (128 x 512 B, NCHW 256x64x256x256), tiles
// split in contiguous ranges over one CTA per SM like K3b, vs the same bytes streamed
// sequentially. Shows how much of l7's gap to the streaming mix floor is the access pattern.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probes/l7_pattern_probe.cu -o tools/probes/bin/l7_pattern_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int B = 256, C = 64, H = 128, W = 128, OH = 256, OW = 256;

// warps/CTA = nw; each tile: warps split the 64 read rows (16 B per lane: 256 B = 16 lanes) and the
// 128 write rows (512 B = 32 lanes x 16 B)
__global__ void pattern(const uint4 *x, uint4 *y, int tiles_per_cta, int nw) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int t0 = blockIdx.x * tiles_per_cta, t1 = min(B * H, t0 + tiles_per_cta);
    uint32_t acc = 0;
    for (int t = t0; t < t1; ++t) {
        const int b = t / H, i = t % H;
        // reads: 64 planes x 16 uint4; lane pair-of-halves: 2 planes per warp instruction
        for (int r = warp * 2 + (lane >> 4); r < C; r += nw * 2) {
            const uint4 v = __ldg(x + (((size_t)(b * C + r) * H + i) * W) / 8 + (lane & 15));
            acc ^= v.x ^ v.w;
        }
        // writes: 64 planes x 2 rows x 32 uint4
        for (int r = warp; r < 2 * C; r += nw) {
            const int c = r >> 1, row = 2 * i + (r & 1);
            y[(((size_t)(b * C + c) * OH + row) * OW) / 8 + lane] = make_uint4(acc, t, r, lane);
        }
    }
    if (acc == 0x1234567) y[0] = make_uint4(1, 2, 3, 4);
}

__global__ void streaming(const uint4 *x, uint4 *y, size_t nx) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < nx; k += (size_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldg(x + k);
#pragma unroll
        for (int r = 0; r < 4; ++r) y[r * nx + k] = make_uint4(v.x + r, v.y, v.z, v.w);
    }
}

int main() {
    const size_t nx = (size_t)B * C * H * W / 8, ny = (size_t)B * C * OH * OW / 8;
    uint4 *x, *y;
    cudaMalloc(&x, nx * 16);
    cudaMalloc(&y, ny * 16);
    cudaMemset(x, 1, nx * 16);
    cudaEvent_t a, e;
    cudaEventCreate(&a);
    cudaEventCreate(&e);
    auto run = [&](const char *name, auto launch) {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(e);
            cudaEventSynchronize(e);
            float ms;
            cudaEventElapsedTime(&ms, a, e);
            if (it && ms < best) best = ms;
        }
        printf("%-46s %7.3f ms %7.0f GB/s (%s)\n", name, best, (nx + ny) * 16 / best / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    run("streaming 1:4 (2368 x 512 threads)", [&] { streaming<<<2368, 512>>>(x, y, nx); });
    for (int nw : {4, 8, 16, 32}) {
        char nm[80];
        const int tpc = (B * H + 147) / 148;
        snprintf(nm, sizeof nm, "l7 pattern, 148 CTAs x %d warps, contiguous", nw);
        run(nm, [&] { pattern<<<148, nw * 32>>>(x, y, tpc, nw); });
    }
    return 0;
}
