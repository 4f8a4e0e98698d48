// The C ABI (include/segb200.h): validation with the reference's error
// taxonomy, the prepared-layer object, and kernel dispatch.
#include <mutex>
#include <vector>

#include "common.cuh"
#include "direct_impl.cuh"
#include "f16split.cuh"
#include "igemm.cuh"
#include "kernels.cuh"

namespace segb {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
}

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SEGB_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return SEGB_OK;
}

// engines.py:70-86: TransposeConvSpec.__post_init__ (stride is fixed at 2 here)
static int check_spec(int in_h, int in_w, int n, int pad, int c_in, int c_out, int *oh, int *ow) {
    if (in_h < 1 || in_w < 1) return fail(SEGB_ERR_SPEC, "input dims must be >= 1, got %dx%d", in_h, in_w);
    if (n < 2) return fail(SEGB_ERR_SPEC, "kernel side must be >= 2, got %d", n);
    if (pad < 0) return fail(SEGB_ERR_SPEC, "padding must be >= 0, got %d", pad);
    if (c_in < 1 || c_out < 1) return fail(SEGB_ERR_SPEC, "channel counts must be >= 1, got %d->%d", c_in, c_out);
    const int h = 2 * in_h + 2 * pad - n, w = 2 * in_w + 2 * pad - n;
    if (h < 1 || w < 1)
        return fail(SEGB_ERR_SPEC, "output dims %dx%d are not >= 1 (input %dx%d, kernel %d, pad %d)", h, w, in_h,
                    in_w, n, pad);
    if (oh) *oh = h;
    if (ow) *ow = w;
    return SEGB_OK;
}

static bool valid_dtype(int dt) { return dt == SEGB_F32 || dt == SEGB_F64 || dt == SEGB_BF16; }

}  // namespace segb

using namespace segb;

struct segb_layer {
    int c_in, c_out, n, pad, engine, compute;
    int device = 0;        // the CUDA device the layer was prepared on (every call runs there)
    void *bank = nullptr;  // owned device copy of the bank (c_in, c_out, n, n)
    int bank_dtype;
    std::mutex mu;
    void *wd[3] = {nullptr, nullptr, nullptr};  // K2 weights per compute dtype (F32, F64, BF16)
    int n2p = 0;
    void *wg = nullptr;  // K3 weights (bf16, class/tap-major, K-major)
    void *wt = nullptr;  // K3 3xTF32 weights: fp32 hi plane followed by the lo plane
    void *wf = nullptr;  // K3 3xFP16 weights: fp16 hi plane, lo plane, then the bank's absmax partials
    int f16_wexp = 0;    // their scale exponent k_w (weights were multiplied by 2^k_w)
    int c_in_pad = 0, c_out_pad = 0, c_in_pad32 = 0;  // zero-padded GEMM operand extents
    void *wz = nullptr;  // K3c weights (bf16, (kx, ky, co) rows x 64-padded c_in, K-major)
    void *ws = nullptr;  // workspace reserved by segb_layer_reserve_workspace (segb_forward)
    int64_t ws_bytes = 0;
    std::vector<float> w_pair;  // K2p: host copy of the fp32 K2 weights (a kernel parameter), or empty
};

namespace segb {

// Runs a call on the layer's device and restores the caller's current device afterwards, so a
// layer prepared on cuda:1 works while cuda:0 is current (allocations, launches and tensor maps
// all follow the current device).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Builds one weight layout (K1) into *slot unless it exists. Called eagerly by segb_prepare for
// every layout the dispatcher can select for the layer's own compute dtype; a forward that
// overrides the compute dtype may build a missing layout here, but never inside a CUDA-graph
// capture (the build would only be recorded while the layout is already marked as built), and a
// lazy build is synchronous so no other stream can read the layout before it exists.
template <typename Build>
static int ensure_layout(segb_layer *L, void **slot, size_t bytes, bool lazy, cudaStream_t st, const char *what,
                         Build build) {
    std::lock_guard<std::mutex> g(L->mu);
    if (*slot) return SEGB_OK;
    if (lazy) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
            return fail(SEGB_ERR_VALUE,
                        "%s weights were not prepared for this compute dtype; run one forward outside the CUDA "
                        "graph capture (or prepare the layer with this compute dtype) first", what);
    }
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return fail(SEGB_ERR_CUDA, "cudaMalloc(%zu) for %s weights: %s", bytes, what, cudaGetErrorString(e));
    if (int rc = build(p)) {
        cudaFree(p);
        return rc;
    }
    if (lazy) {
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            cudaFree(p);
            return fail(SEGB_ERR_CUDA, "%s weight build: %s", what, cudaGetErrorString(e));
        }
    }
    *slot = p;
    return SEGB_OK;
}

// K2 weights for a compute dtype
static int ensure_direct_weights(segb_layer *L, int compute, bool lazy, cudaStream_t st, const void **out) {
    const size_t elt = compute == SEGB_F64 ? 8 : 4;
    const size_t bytes = elt * (size_t)L->c_out * L->c_in * L->n2p;
    int rc = ensure_layout(L, &L->wd[compute], bytes, lazy, st, "direct-kernel", [&](void *p) {
        const int mode = compute == SEGB_F64 ? 1 : (compute == SEGB_BF16 ? 2 : 0);
        const bool packed = L->engine == SEGB_ENGINE_SEGREGATED;
        return run_prep_direct(L->bank, L->bank_dtype, L->c_in, L->c_out, L->n, L->n2p, packed, mode, p, st);
    });
    if (!rc && out) *out = L->wd[compute];
    return rc;
}

static int ensure_gemm_weights(segb_layer *L, bool lazy, cudaStream_t st) {
    const size_t bytes = 2ull * L->n * L->n * L->c_out_pad * L->c_in_pad;
    return ensure_layout(L, &L->wg, bytes, lazy, st, "bf16 implicit-GEMM", [&](void *p) {
        return run_prep_gemm(L->bank, L->bank_dtype, L->c_in, L->c_in_pad, L->c_out, L->c_out_pad, L->n, p, st);
    });
}

static int ensure_scatter_weights(segb_layer *L, bool lazy, cudaStream_t st) {
    const int c_in_pad = (int)ceil_div(L->c_in, 64) * 64;
    const size_t bytes = 2ull * scatter_weight_rows(L->c_out, L->n) * c_in_pad;
    return ensure_layout(L, &L->wz, bytes, lazy, st, "scatter-GEMM", [&](void *p) {
        return run_prep_scatter(L->bank, L->bank_dtype, L->c_in, c_in_pad, L->c_out, L->n, p, st);
    });
}

static size_t tf32_plane(const segb_layer *L) { return (size_t)L->n * L->n * L->c_out_pad * L->c_in_pad32; }

static int ensure_tf32_weights(segb_layer *L, bool lazy, cudaStream_t st) {
    const size_t plane = tf32_plane(L);
    return ensure_layout(L, &L->wt, 2 * 4 * plane, lazy, st, "3xTF32 implicit-GEMM", [&](void *p) {
        return run_prep_gemm_tf32(L->bank, L->bank_dtype, L->c_in, L->c_in_pad32, L->c_out, L->c_out_pad, L->n, p,
                                  (char *)p + 4 * plane, st);
    });
}

static size_t f16_plane(const segb_layer *L) { return (size_t)L->n * L->n * L->c_out_pad * L->c_in_pad; }

// 3xFP16 weights; the scale exponent is read back once (prepare is synchronous on its stream)
static int ensure_f16x3_weights(segb_layer *L, bool lazy, cudaStream_t st) {
    const size_t plane = f16_plane(L);
    const size_t bytes = 2 * 2 * plane + kAbsmaxBytes;
    int rc = ensure_layout(L, &L->wf, bytes, lazy, st, "3xFP16 implicit-GEMM", [&](void *p) -> int {
        float *partials = (float *)((char *)p + 4 * plane);
        int r = run_prep_gemm_f16x2(L->bank, L->bank_dtype, L->c_in, L->c_in_pad, L->c_out, L->c_out_pad, L->n, p,
                                    (char *)p + 2 * plane, partials, st);
        if (r) return r;
        float hp[kAbsmaxBlocks];
        cudaError_t e = cudaMemcpyAsync(hp, partials, sizeof hp, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail(SEGB_ERR_CUDA, "3xFP16 weight scale: %s", cudaGetErrorString(e));
        float m = 0.f;
        for (float v : hp) m = std::max(m, v);
        L->f16_wexp = f16_scale_exp(m);
        return (int)SEGB_OK;
    });
    return rc;
}

// fp32 tensor-core mode: 3xFP16 unless SEGB200_FP32_TC=tf32x3 (A/B switch, read at prepare)
static bool want_tf32x3() {
    const char *e = getenv("SEGB200_FP32_TC");
    return e && std::string(e) == "tf32x3";
}

// weight-only conditions under which the dispatcher can pick each tensor-core path (the shape
// conditions of igemm_supported that do not depend on the input)
static bool may_use_gemm_bf16(const segb_layer *L) {
    return L->engine == SEGB_ENGINE_SEGREGATED && L->c_in >= 16 && igemm_available();
}
static bool may_use_scatter(const segb_layer *L) {
    return L->engine == SEGB_ENGINE_SEGREGATED && L->c_in >= 64 && L->c_in <= 256 &&
           L->n * L->n * L->c_out <= 256 && L->n <= 8 && 4 * L->c_out <= L->c_in && igemm_available();
}
static bool may_use_f16x3(const segb_layer *L) {
    return L->engine == SEGB_ENGINE_SEGREGATED && L->n % 2 == 0 && L->c_in >= 64 && L->c_in % 8 == 0 &&
           igemm_available();
}
static bool may_use_tf32(const segb_layer *L) {
    return L->engine == SEGB_ENGINE_SEGREGATED && L->n % 2 == 0 && L->c_in >= 32 && L->c_in % 4 == 0 &&
           L->c_out >= 16 && igemm_available();
}

}  // namespace segb

// tensor cores for bf16 (kind::f16) and for fp32 as 3xTF32 (kind::tf32)
static bool igemm_ok(const segb_layer *L, int x_dtype, int64_t batch, int in_h, int in_w, int compute,
                     int y_dtype) {
    if (L->engine != SEGB_ENGINE_SEGREGATED || (compute != SEGB_BF16 && compute != SEGB_F32)) return false;
    IgemmShape s{};
    s.batch = batch; s.c_in = L->c_in; s.c_out = L->c_out; s.h = in_h; s.w = in_w; s.n = L->n; s.pad = L->pad;
    s.x_dtype = x_dtype; s.y_dtype = y_dtype; s.compute = compute;
    s.f16x3 = compute == SEGB_F32 && L->wf != nullptr;
    if (compute == SEGB_F32 && L->c_out < 16) {
        // narrow fp32 outputs (dcgan_l5): the tensor cores pad N to 32 and re-read the input per
        // class and tap, the direct kernel streams it once; the direct kernel wins whenever it has
        // blocks enough to fill the GPU (measured: 97 us vs 127 us at batch 64, 141 vs 436 at 256),
        // the tensor-core kernel at small batches (34 vs 101 us at batch 1: 2 direct blocks)
        const int oh = 2 * in_h + 2 * L->pad - L->n, ow = 2 * in_w + 2 * L->pad - L->n, swap = L->pad & 1;
        const int64_t nqr = (oh - 1 + swap) / 2 + 1, nqc = (ow - 1 + swap) / 2 + 1;
        const int cob = std::min(L->c_out, 4), rq = L->n <= 5 ? 4 : 2, cq = (L->n <= 5 && cob <= 2) ? 2 : 1;
        const int64_t blocks = ceil_div(nqc, 32 * cq) * ceil_div(L->c_out, cob) * ceil_div(nqr, 4 * rq) * batch;
        if (blocks >= 64) return false;
    }
    return igemm_supported(s);
}

extern "C" {

int segb_abi_version(void) { return SEGB_ABI_VERSION; }

const char *segb_last_error(void) { return g_err.c_str(); }

int64_t segb_launch_count(void) { return g_launches.load(); }

int segb_output_dims(int in_h, int in_w, int kernel_n, int pad, int *out_h, int *out_w) {
    return check_spec(in_h, in_w, kernel_n, pad, 1, 1, out_h, out_w);
}

int segb_effective_padding(int pad, int *eff_pad, int *swap) {
    if (pad < 0) return fail(SEGB_ERR_VALUE, "padding must be >= 0, got %d", pad);
    if (eff_pad) *eff_pad = pad / 2;
    if (swap) *swap = pad % 2;
    return SEGB_OK;
}

int segb_subkernel_dims(int kernel_n, int r, int s, int *rows, int *cols) {
    if (kernel_n < 2) return fail(SEGB_ERR_SHAPE, "kernel side must be >= 2, got %d", kernel_n);
    if ((r & ~1) || (s & ~1)) return fail(SEGB_ERR_VALUE, "parities must be 0 or 1, got (%d,%d)", r, s);
    if (rows) *rows = sub_len(kernel_n, r);
    if (cols) *cols = sub_len(kernel_n, s);
    return SEGB_OK;
}

int64_t segb_mult_count_segregated(int in_h, int in_w, int n, int pad, int c_in, int c_out) {
    int oh, ow;
    if (check_spec(in_h, in_w, n, pad, c_in, c_out, &oh, &ow)) return -1;
    const int swap = pad & 1;
    int64_t total = 0;
    for (int r = 0; r < 2; ++r) {
        const int st_r = (r + swap) % 2;
        const int64_t rows = std::max(0, (oh - st_r + 1) / 2);
        for (int s = 0; s < 2; ++s) {
            const int st_s = (s + swap) % 2;
            const int64_t cols = std::max(0, (ow - st_s + 1) / 2);
            total += rows * cols * sub_len(n, r) * sub_len(n, s);
        }
    }
    return total * c_in * c_out;
}

int segb_segregate(const void *kern, int dtype, int64_t count, int n, void *subs, void *stream) {
    if (!valid_dtype(dtype)) return fail(SEGB_ERR_VALUE, "unknown dtype %d", dtype);
    if (n < 2) return fail(SEGB_ERR_SHAPE, "kernel side must be >= 2, got %d", n);
    if (count < 0 || (count > 0 && (!kern || !subs))) return fail(SEGB_ERR_VALUE, "null tensor");
    return run_segregate(kern, dtype, count, n, subs, false, (cudaStream_t)stream);
}

int segb_merge(const void *subs, int dtype, int64_t count, int n, void *kern, void *stream) {
    if (!valid_dtype(dtype)) return fail(SEGB_ERR_VALUE, "unknown dtype %d", dtype);
    if (n < 2) return fail(SEGB_ERR_SHAPE, "kernel side must be >= 2, got %d", n);
    if (count < 0 || (count > 0 && (!kern || !subs))) return fail(SEGB_ERR_VALUE, "null tensor");
    return run_segregate(subs, dtype, count, n, kern, true, (cudaStream_t)stream);
}

int segb_prepare(const void *bank, int bank_dtype, int c_in, int c_out, int n, int pad, int engine,
                 int compute, void *stream, segb_layer **out) {
    if (!out) return fail(SEGB_ERR_VALUE, "null output handle");
    *out = nullptr;
    // engines.py:213-225 validation order: bank shape, kernel side, dtype, pad, engine
    if (c_in < 1 || c_out < 1) return fail(SEGB_ERR_SHAPE, "kernel bank must have c_in, c_out >= 1");
    if (n < 2) return fail(SEGB_ERR_SHAPE, "kernel side must be >= 2, got %d", n);
    if (!valid_dtype(bank_dtype)) return fail(SEGB_ERR_SHAPE, "kernel bank must hold floats (dtype %d)", bank_dtype);
    if (pad < 0) return fail(SEGB_ERR_SPEC, "padding must be >= 0, got %d", pad);
    if (engine != SEGB_ENGINE_REFERENCE && engine != SEGB_ENGINE_SEGREGATED)
        return fail(SEGB_ERR_VALUE, "unknown engine %d, expected one of ('reference', 'segregated')", engine);
    if (!valid_dtype(compute)) return fail(SEGB_ERR_VALUE, "unknown compute dtype %d", compute);
    if (!bank) return fail(SEGB_ERR_VALUE, "null bank");
    cudaStream_t st = (cudaStream_t)stream;
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, bank) != cudaSuccess || pa.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        return fail(SEGB_ERR_VALUE, "bank must be a device pointer");
    }
    DeviceGuard dg(pa.device);
    segb_layer *L = new segb_layer();
    L->c_in = c_in; L->c_out = c_out; L->n = n; L->pad = pad; L->engine = engine; L->compute = compute;
    L->bank_dtype = bank_dtype;
    L->device = pa.device;
    L->n2p = (n * n + 3) / 4 * 4;
    L->c_in_pad = (int)ceil_div(c_in, 64) * 64;
    L->c_out_pad = (int)ceil_div(c_out, 32) * 32;
    L->c_in_pad32 = (int)ceil_div(c_in, 32) * 32;
    const size_t bytes = dtype_size(bank_dtype) * (size_t)c_in * c_out * n * n;
    cudaError_t e = cudaMalloc(&L->bank, bytes);
    if (e == cudaSuccess) e = cudaMemcpyAsync(L->bank, bank, bytes, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) {
        segb_release(L);
        return fail(SEGB_ERR_CUDA, "bank copy: %s", cudaGetErrorString(e));
    }
    // every layout the dispatcher can select for this compute dtype is built here, so forward
    // never allocates (and is capturable into a CUDA graph from its first call)
    int rc = ensure_direct_weights(L, compute, false, st, nullptr);
    if (!rc && compute == SEGB_BF16 && may_use_gemm_bf16(L)) rc = ensure_gemm_weights(L, false, st);
    if (!rc && compute == SEGB_BF16 && may_use_scatter(L)) rc = ensure_scatter_weights(L, false, st);
    if (!rc && compute == SEGB_F32 && may_use_f16x3(L) && !want_tf32x3()) rc = ensure_f16x3_weights(L, false, st);
    if (!rc && compute == SEGB_F32 && may_use_tf32(L) && !L->wf) rc = ensure_tf32_weights(L, false, st);
    if (!rc && compute == SEGB_F32 && engine == SEGB_ENGINE_SEGREGATED && direct_pair_ok(c_in, c_out, n, L->n2p)) {
        // K2p takes its (few) weights as a kernel parameter: one host copy, made here
        L->w_pair.resize((size_t)c_in * c_out * L->n2p);
        cudaError_t e2 = cudaMemcpyAsync(L->w_pair.data(), L->wd[SEGB_F32], L->w_pair.size() * sizeof(float),
                                         cudaMemcpyDeviceToHost, st);
        if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(st);
        if (e2 != cudaSuccess) rc = fail(SEGB_ERR_CUDA, "paired direct-kernel weights: %s", cudaGetErrorString(e2));
    }
    if (rc) {
        segb_release(L);
        return rc;
    }
    *out = L;
    return SEGB_OK;
}

int segb_layer_info(const segb_layer *L, int *c_in, int *c_out, int *n, int *pad, int *engine, int *compute) {
    if (!L) return fail(SEGB_ERR_VALUE, "null layer");
    if (c_in) *c_in = L->c_in;
    if (c_out) *c_out = L->c_out;
    if (n) *n = L->n;
    if (pad) *pad = L->pad;
    if (engine) *engine = L->engine;
    if (compute) *compute = L->compute;
    return SEGB_OK;
}

int segb_select_path(const segb_layer *L, int x_dtype, int64_t batch, int in_h, int in_w, int compute) {
    if (!L) return fail(SEGB_ERR_VALUE, "null layer");
    if (compute < 0) compute = L->compute;
    const int y_dtype = compute == SEGB_F32 ? SEGB_F32 : SEGB_BF16;
    return igemm_ok(L, x_dtype, batch, in_h, in_w, compute, y_dtype) ? SEGB_PATH_IGEMM : SEGB_PATH_DIRECT;
}

// the resolved plan of one forward call: the kernel family and the workspace it needs
struct FwdPlan {
    int path, oh, ow, compute;
    IgemmShape s;
    int64_t ws_bytes;
};

static int plan_forward(const segb_layer *L, int x_dtype, int64_t batch, int in_h, int in_w, int y_dtype,
                        int compute, int path, FwdPlan &pl) {
    if (!L) return fail(SEGB_ERR_VALUE, "null layer");
    if (batch < 1) return fail(SEGB_ERR_SHAPE, "batch must be >= 1, got %lld", (long long)batch);
    if (int rc = check_spec(in_h, in_w, L->n, L->pad, L->c_in, L->c_out, &pl.oh, &pl.ow)) return rc;
    if (compute < 0) compute = L->compute;
    if (x_dtype == SEGB_U8_HWC) {  // the fused dataset-image path: K2, fp32
        if (compute != SEGB_F32 || y_dtype != SEGB_F32)
            return fail(SEGB_ERR_VALUE, "u8 image input computes in fp32 into f32 y (compute %d, y %d)", compute,
                        y_dtype);
        if (path == SEGB_PATH_IGEMM) return fail(SEGB_ERR_UNSUPPORTED, "u8 image input runs on the direct kernel");
        path = SEGB_PATH_DIRECT;
    } else if (!valid_dtype(x_dtype)) {
        return fail(SEGB_ERR_VALUE, "unknown x dtype %d", x_dtype);
    }
    if (!valid_dtype(compute) || !valid_dtype(y_dtype))
        return fail(SEGB_ERR_VALUE, "unknown dtype (x %d, y %d, compute %d)", x_dtype, y_dtype, compute);
    if (path == SEGB_PATH_AUTO)
        path = igemm_ok(L, x_dtype, batch, in_h, in_w, compute, y_dtype) ? SEGB_PATH_IGEMM : SEGB_PATH_DIRECT;
    if (path != SEGB_PATH_IGEMM && path != SEGB_PATH_DIRECT) return fail(SEGB_ERR_VALUE, "unknown path %d", path);
    pl.path = path;
    pl.compute = compute;
    pl.ws_bytes = 0;
    if (path == SEGB_PATH_IGEMM) {
        if (!igemm_ok(L, x_dtype, batch, in_h, in_w, compute, y_dtype))
            return fail(SEGB_ERR_UNSUPPORTED, "implicit-GEMM path not eligible for this layer/shape/dtype");
        IgemmShape &s = pl.s;
        s = IgemmShape{};
        s.batch = batch; s.c_in = L->c_in; s.c_out = L->c_out; s.h = in_h; s.w = in_w; s.n = L->n; s.pad = L->pad;
        s.x_dtype = x_dtype; s.y_dtype = y_dtype; s.compute = compute;
        s.c_out_pad = L->c_out_pad;
        s.c_in_pad = L->c_in_pad;
        s.c_in_pad32 = L->c_in_pad32;
        if (compute == SEGB_F32 && L->wf) {
            s.f16x3 = 1;
            s.w_exp = L->f16_wexp;
        }
        pl.ws_bytes = igemm_workspace_bytes(s);
    }
    return SEGB_OK;
}

// K2p for the direct path: fp32 compute on f32 / u8-image x into f32 y, the layer's host weight
// copy made at prepare (SEGB200_DIRECT_PAIR=0 keeps K2, for A/B runs and the bitwise test)
static bool use_direct_pair(const segb_layer *L, int x_dtype, int y_dtype, int compute, int in_w) {
    if (L->w_pair.empty() || compute != SEGB_F32 || y_dtype != SEGB_F32) return false;
    if (x_dtype != SEGB_F32 && x_dtype != SEGB_U8_HWC) return false;
    if (!direct_pair_n_ok(L->n, x_dtype == SEGB_F32, in_w)) return false;
    const char *e = getenv("SEGB200_DIRECT_PAIR");
    return !(e && !atoi(e));
}

// K2p with shared-memory weights: segregated fp32 layers whose weights exceed the parameter
static bool use_direct_pair_wsm(const segb_layer *L, int x_dtype, int y_dtype, int compute, int in_w) {
    if (L->engine != SEGB_ENGINE_SEGREGATED || compute != SEGB_F32 || x_dtype != SEGB_F32 || y_dtype != SEGB_F32)
        return false;
    const char *e = getenv("SEGB200_DIRECT_PAIR");
    if (e && !atoi(e)) return false;
    return direct_pair_wsm_ok(L->c_in, L->c_out, L->n, L->n2p, in_w);
}

static int forward_impl(segb_layer *L, const void *x, int x_dtype, int64_t batch, int in_h, int in_w, void *y,
                        int y_dtype, int compute, int path, void *ws, int64_t ws_bytes, cudaStream_t st) {
    FwdPlan pl;
    if (int rc = plan_forward(L, x_dtype, batch, in_h, in_w, y_dtype, compute, path, pl)) return rc;
    if (!x || !y) return fail(SEGB_ERR_VALUE, "null tensor");
    if (pl.ws_bytes > 0 && (!ws || ws_bytes < pl.ws_bytes))
        return fail(SEGB_ERR_VALUE,
                    "this forward needs a workspace of %lld bytes (segb_forward_workspace_bytes), got %lld",
                    (long long)pl.ws_bytes, (long long)(ws ? ws_bytes : 0));
    DeviceGuard dg(L->device);
    compute = pl.compute;
    const int oh = pl.oh, ow = pl.ow;
    if (pl.path == SEGB_PATH_IGEMM) {
        IgemmShape &s = pl.s;
        if (compute == SEGB_F32 && s.f16x3) return run_igemm(s, x, L->wf, (const char *)L->wf + 2 * f16_plane(L), y, ws,
                                                             ws_bytes, st);
        if (compute == SEGB_F32) {
            if (int rc = ensure_tf32_weights(L, true, st)) return rc;
            return run_igemm(s, x, L->wt, (const char *)L->wt + 4 * tf32_plane(L), y, ws, ws_bytes, st);
        }
        if (igemm_scatter_supported(s)) {
            if (int rc = ensure_scatter_weights(L, true, st)) return rc;
            return run_igemm_scatter(s, x, L->wz, y, ws, ws_bytes, st);
        }
        if (int rc = ensure_gemm_weights(L, true, st)) return rc;
        return run_igemm(s, x, L->wg, nullptr, y, ws, ws_bytes, st);
    }
    const void *w;
    if (int rc = ensure_direct_weights(L, compute, true, st, &w)) return rc;
    DirectArgs a{};
    a.x = x; a.y = y; a.w = w; a.batch = batch; a.b0 = 0;
    a.c_in = L->c_in; a.c_out = L->c_out; a.h = in_h; a.w_in = in_w; a.oh = oh; a.ow = ow; a.n = L->n;
    a.p = L->pad / 2; a.swap = L->pad & 1; a.n2p = L->n2p;
    a.nqr = (oh - 1 + a.swap) / 2 + 1;
    a.nqc = (ow - 1 + a.swap) / 2 + 1;
    const bool ref = L->engine == SEGB_ENGINE_REFERENCE;
    if (ref) a.p = L->pad;  // the reference engine pads the upsampled map by P
    if (use_direct_pair(L, x_dtype, y_dtype, compute, in_w))
        return x_dtype == SEGB_U8_HWC ? launch_direct_pair_u8(a, L->w_pair.data(), st)
                                      : launch_direct_pair_f32(a, L->w_pair.data(), st);
    if (use_direct_pair_wsm(L, x_dtype, y_dtype, compute, in_w)) return launch_direct_pair_wsm(a, st);
    if (x_dtype == SEGB_U8_HWC) return launch_direct_u8(a, ref, st);
    switch (compute) {
        case SEGB_F32:
            if (x_dtype != SEGB_F32 || y_dtype != SEGB_F32)
                return fail(SEGB_ERR_VALUE, "fp32 compute needs f32 x and y (got %d/%d)", x_dtype, y_dtype);
            return launch_direct_f32(a, ref, st);
        case SEGB_F64:
            if (x_dtype != SEGB_F64 || y_dtype != SEGB_F64)
                return fail(SEGB_ERR_VALUE, "fp64 compute needs f64 x and y (got %d/%d)", x_dtype, y_dtype);
            return launch_direct_f64(a, ref, st);
        default: return launch_direct_bf16(a, x_dtype, y_dtype, ref, st);
    }
}

int segb_describe_path(const segb_layer *L, int x_dtype, int64_t batch, int in_h, int in_w, int y_dtype,
                       int compute, int path, char *buf, int buf_len) {
    FwdPlan pl;
    if (int rc = plan_forward(L, x_dtype, batch, in_h, in_w, y_dtype, compute, path, pl)) return rc;
    const char *name = "K2 direct (fp32 FFMA)";
    if (pl.path == SEGB_PATH_IGEMM) name = igemm_kernel_name(pl.s);
    else if (use_direct_pair(L, x_dtype, y_dtype, pl.compute, in_w))
        name = x_dtype == SEGB_U8_HWC ? "K2p direct (u8 image decoded on load, fp32 FFMA2, two samples per thread)"
               : (in_w % 4 == 0 && direct_pair_tma_enabled())
                   ? "K2p direct (fp32 FFMA2, two samples per thread, TMA-staged input tiles)"
                   : "K2p direct (fp32 FFMA2, two samples per thread)";
    else if (pl.path == SEGB_PATH_DIRECT && use_direct_pair_wsm(L, x_dtype, y_dtype, pl.compute, in_w))
        name = "K2p direct (fp32 FFMA2, two samples per thread, TMA-staged input tiles, weights in shared memory)";
    else if (x_dtype == SEGB_U8_HWC) name = "K2 direct (u8 image decoded on load, fp32 FFMA)";
    else if (pl.compute == SEGB_F64) name = "K2 direct (fp64)";
    else if (pl.compute == SEGB_BF16) name = "K2 direct (bf16 operands, fp32 FFMA)";
    if (buf && buf_len > 0) snprintf(buf, (size_t)buf_len, "%s", name);
    return SEGB_OK;
}

int segb_forward_workspace_bytes(const segb_layer *L, int x_dtype, int64_t batch, int in_h, int in_w, int y_dtype,
                                 int compute, int path, int64_t *bytes) {
    FwdPlan pl;
    if (int rc = plan_forward(L, x_dtype, batch, in_h, in_w, y_dtype, compute, path, pl)) return rc;
    if (bytes) *bytes = pl.ws_bytes;
    return SEGB_OK;
}

int segb_forward_ws(const segb_layer *L, const void *x, int x_dtype, int64_t batch, int in_h, int in_w, void *y,
                    int y_dtype, int compute, int path, void *workspace, int64_t workspace_bytes, void *stream) {
    return forward_impl(const_cast<segb_layer *>(L), x, x_dtype, batch, in_h, in_w, y, y_dtype, compute, path,
                        workspace, workspace_bytes, (cudaStream_t)stream);
}

int segb_forward(const segb_layer *Lc, const void *x, int x_dtype, int64_t batch, int in_h, int in_w, void *y,
                 int y_dtype, int compute, int path, void *stream) {
    segb_layer *L = const_cast<segb_layer *>(Lc);
    if (!L) return fail(SEGB_ERR_VALUE, "null layer");
    return forward_impl(L, x, x_dtype, batch, in_h, in_w, y, y_dtype, compute, path, L->ws, L->ws_bytes,
                        (cudaStream_t)stream);
}

int segb_layer_reserve_workspace(segb_layer *L, int64_t bytes) {
    if (!L) return fail(SEGB_ERR_VALUE, "null layer");
    if (bytes < 0) return fail(SEGB_ERR_VALUE, "workspace bytes must be >= 0, got %lld", (long long)bytes);
    std::lock_guard<std::mutex> g(L->mu);
    if (bytes <= L->ws_bytes) return SEGB_OK;
    DeviceGuard dg(L->device);
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)bytes);
    if (e != cudaSuccess)
        return fail(SEGB_ERR_CUDA, "cudaMalloc(%lld) for the workspace: %s", (long long)bytes, cudaGetErrorString(e));
    if (L->ws) {
        cudaDeviceSynchronize();  // queued forwards may still read the old buffer
        cudaFree(L->ws);
    }
    L->ws = p;
    L->ws_bytes = bytes;
    return SEGB_OK;
}

// ---------------------------------------------------------------- layer stacks
// the GAN_SUITE generator stacks (bench.py:124-139 of the reference) run
// device-resident. The reference has no stack call: a user chains layer_forward (engines.py:
// 163-172) per layer through host arrays. Here layer i's output is layer i+1's input in the
// caller's workspace (two ping-pong buffers of the largest intermediate, inter_dtype), so
// nothing crosses PCIe between layers and the whole chain is one stream-ordered launch
// sequence (capturable as one CUDA graph).

// Plans a chain: per layer its input/output dims and dtypes; returns the largest intermediate
// (elements) and the largest per-layer forward workspace (bytes).
static int stack_plan(const segb_layer *const *layers, int count, int64_t batch, int in_h, int in_w, int x_dtype,
                      int y_dtype, int inter_dtype, int64_t *inter_elems, int64_t *fwd_ws) {
    if (!layers || count < 1) return fail(SEGB_ERR_VALUE, "a stack needs at least one layer");
    if (batch < 1) return fail(SEGB_ERR_SHAPE, "batch must be >= 1, got %lld", (long long)batch);
    if (!valid_dtype(inter_dtype)) return fail(SEGB_ERR_VALUE, "unknown intermediate dtype %d", inter_dtype);
    int h = in_h, w = in_w, dt = x_dtype;
    int64_t most = 0, ws = 0;
    for (int i = 0; i < count; ++i) {
        const segb_layer *L = layers[i];
        if (!L) return fail(SEGB_ERR_VALUE, "null layer %d in the stack", i);
        if (i > 0 && layers[i - 1]->c_out != L->c_in)
            return fail(SEGB_ERR_SHAPE, "stack layer %d expects %d input channels, layer %d produces %d", i, L->c_in,
                        i - 1, layers[i - 1]->c_out);
        int oh, ow;
        if (int rc = check_spec(h, w, L->n, L->pad, L->c_in, L->c_out, &oh, &ow)) return rc;
        const int odt = i + 1 < count ? inter_dtype : y_dtype;
        if (i + 1 < count) most = std::max<int64_t>(most, batch * L->c_out * (int64_t)oh * ow);
        FwdPlan pl;
        if (valid_dtype(dt) && valid_dtype(odt)) {
            if (int rc = plan_forward(L, dt, batch, h, w, odt, -1, SEGB_PATH_AUTO, pl)) return rc;
            ws = std::max(ws, pl.ws_bytes);
        }
        h = oh;
        w = ow;
        dt = odt;
    }
    if (inter_elems) *inter_elems = most;
    if (fwd_ws) *fwd_ws = ws;
    return SEGB_OK;
}

static int64_t align256(int64_t b) { return (b + 255) / 256 * 256; }

int segb_stack_workspace_bytes2(const segb_layer *const *layers, int count, int64_t batch, int in_h, int in_w,
                                int x_dtype, int y_dtype, int inter_dtype, int64_t *bytes) {
    int64_t most = 0, fws = 0;
    if (int rc = stack_plan(layers, count, batch, in_h, in_w, x_dtype, y_dtype, inter_dtype, &most, &fws)) return rc;
    const int64_t one = align256(most * (int64_t)dtype_size(inter_dtype));
    if (bytes) *bytes = (count > 2 ? 2 * one : one) + align256(fws);
    return SEGB_OK;
}

int segb_stack_workspace_bytes(const segb_layer *const *layers, int count, int64_t batch, int in_h, int in_w,
                               int inter_dtype, int64_t *bytes) {
    // without the end dtypes: the intermediates' dtype stands in for both (the bf16 stacks)
    return segb_stack_workspace_bytes2(layers, count, batch, in_h, in_w, inter_dtype, inter_dtype, inter_dtype,
                                       bytes);
}

int segb_stack_forward(const segb_layer *const *layers, int count, const void *x, int x_dtype, int64_t batch,
                       int in_h, int in_w, void *y, int y_dtype, int inter_dtype, void *workspace,
                       int64_t workspace_bytes, void *stream) {
    int64_t most = 0, fws = 0;
    if (int rc = stack_plan(layers, count, batch, in_h, in_w, x_dtype, y_dtype, inter_dtype, &most, &fws)) return rc;
    const int64_t one = align256(most * (int64_t)dtype_size(inter_dtype));
    const int64_t inter = count > 2 ? 2 * one : one;
    const int64_t need = inter + align256(fws);
    if (!x || !y) return fail(SEGB_ERR_VALUE, "null tensor");
    if (need > 0 && (!workspace || workspace_bytes < need))
        return fail(SEGB_ERR_VALUE, "stack workspace of %lld bytes needed, got %lld", (long long)need,
                    (long long)workspace_bytes);
    void *fwd_ws = fws > 0 ? (char *)workspace + inter : nullptr;
    const void *cur = x;
    int cur_dt = x_dtype, h = in_h, w = in_w;
    for (int i = 0; i < count; ++i) {
        const bool last = i + 1 == count;
        void *dst = last ? y : (char *)workspace + (i % 2) * one;
        const int dst_dt = last ? y_dtype : inter_dtype;
        if (int rc = forward_impl(const_cast<segb_layer *>(layers[i]), cur, cur_dt, batch, h, w, dst, dst_dt, -1,
                                  SEGB_PATH_AUTO, fwd_ws, fws, (cudaStream_t)stream))
            return rc;
        h = 2 * h + 2 * layers[i]->pad - layers[i]->n;
        w = 2 * w + 2 * layers[i]->pad - layers[i]->n;
        cur = dst;
        cur_dt = dst_dt;
    }
    return SEGB_OK;
}

int segb_release(segb_layer *L) {
    if (!L) return SEGB_OK;
    cudaFree(L->bank);
    for (void *p : L->wd) cudaFree(p);
    cudaFree(L->wg);
    cudaFree(L->wt);
    cudaFree(L->wz);
    cudaFree(L->wf);
    cudaFree(L->ws);
    delete L;
    return SEGB_OK;
}

int segb_unit_floats(void *out, int dtype, int64_t count, uint64_t seed, void *stream) {
    if (count < 0) return fail(SEGB_ERR_VALUE, "count must be >= 0, got %lld", (long long)count);
    if (count > 0 && !out) return fail(SEGB_ERR_VALUE, "null tensor");
    return run_unit_floats(out, dtype, count, seed, (cudaStream_t)stream);
}

}  // extern "C"
