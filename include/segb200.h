/*
 * segb200 -- C ABI of the B200-native unified kernel-segregated stride-2
 * transpose convolution (arXiv 2502.20493).
 *
 * This is the drop-in boundary for the reference package `segconv`
 * (/root/reference/pkg/src/segconv). The reference has no FFI; its operator
 * API is Python. Each entry point below replaces one reference interface,
 * cited as file:line relative to /root/reference/pkg/src/segconv/. The host
 * mirror of that Python API (paper_2502_20493_b200/engines.py) binds these
 * symbols through ctypes; INTEGRATION.md shows the binding a maintainer would
 * add to the reference itself.
 *
 * Conventions
 *   - plain pointers and sizes; no torch types. Tensor pointers passed to
 *     segb_prepare / segb_forward / segb_segregate / segb_merge /
 *     segb_unit_floats are DEVICE pointers owned by the caller.
 *   - activations are batched NCHW: x (batch, c_in, in_h, in_w),
 *     y (batch, c_out, out_h, out_w), contiguous. The reference's per-sample
 *     CHW tensor is batch = 1 (batch is a map over samples).
 *   - the weight bank is (c_in, c_out, n, n) contiguous, the reference's
 *     layout (engines.py:213-217), used unflipped in correlation form.
 *   - every function returns SEGB_OK (0) or an error code; the message is in
 *     segb_last_error() (thread-local). Codes map to the reference's
 *     exceptions: SEGB_ERR_SPEC -> SpecError (engines.py:54),
 *     SEGB_ERR_SHAPE -> ShapeError (tensors.py:26), SEGB_ERR_VALUE ->
 *     ValueError (engines.py:224-225,251-252), SEGB_ERR_CUDA -> RuntimeError.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream). Launches are
 *     asynchronous. segb_forward / segb_forward_ws / segb_stack_forward never
 *     allocate: the scratch a forward needs (K3's channels-last operand copy,
 *     K3c's tap products; K2 and K3b need none) is a caller-provided workspace
 *     sized by segb_forward_workspace_bytes, or the layer's own buffer reserved
 *     ahead of time with segb_layer_reserve_workspace. segb_prepare builds every
 *     weight layout the dispatcher can select for the layer's compute dtype, so
 *     a forward is capturable into a CUDA graph from its first call.
 *   - calls run on the device the layer was prepared on (the bank pointer's
 *     device), whatever device is current; the current device is restored.
 *   - results are deterministic: fixed accumulation order, no atomics, no
 *     split-K, so outputs are bitwise identical across runs and GPU counts.
 */
#ifndef SEGB200_H
#define SEGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEGB_ABI_VERSION 2

enum segb_status {
    SEGB_OK = 0,
    SEGB_ERR_SPEC = 1,
    SEGB_ERR_SHAPE = 2,
    SEGB_ERR_VALUE = 3,
    SEGB_ERR_CUDA = 4,
    SEGB_ERR_UNSUPPORTED = 5
};

enum segb_dtype {
    SEGB_F32 = 0,
    SEGB_F64 = 1,
    SEGB_BF16 = 2,
    /* x only: the interleaved u8 image payload (batch, in_h, in_w, c_in) of binary P6 PPMs,
     * decoded in the direct kernel's loads as float32(u8) / 255 with IEEE division -- bitwise
     * the reference's parse_ppm values (tensor_io.py:27-52); fp32 compute, f32 y */
    SEGB_U8_HWC = 3
};

/* engines.py:44-46 ENGINE_REFERENCE / ENGINE_SEGREGATED */
enum segb_engine { SEGB_ENGINE_REFERENCE = 0, SEGB_ENGINE_SEGREGATED = 1 };

/* kernel selection for segb_forward */
enum segb_path {
    SEGB_PATH_AUTO = 0,   /* direct for low-channel layers, igemm where eligible */
    SEGB_PATH_DIRECT = 1, /* K2: CUDA-core unified kernel, any shape/dtype       */
    SEGB_PATH_IGEMM = 2   /* K3: tcgen05/TMEM implicit GEMM per parity class     */
};

typedef struct segb_layer segb_layer;

int segb_abi_version(void);
const char *segb_last_error(void);

/* engines.py:70-96 (TransposeConvSpec.__post_init__ + output_dims).
 * SEGB_ERR_SPEC for stride != 2 (not expressible here), in dims < 1,
 * kernel_n < 2, pad < 0, or an output dim < 1. */
int segb_output_dims(int in_h, int in_w, int kernel_n, int pad, int *out_h, int *out_w);

/* segregation.py:91-96 effective_padding: pad -> (pad / 2, pad odd).
 * SEGB_ERR_VALUE for pad < 0 (the reference raises ValueError there). */
int segb_effective_padding(int pad, int *eff_pad, int *swap);

/* segregation.py:53-58 subkernel_dims */
int segb_subkernel_dims(int kernel_n, int row_parity, int col_parity, int *rows, int *cols);

/* analysis.py:46-57 mult_count_segregated: useful MACs of one sample.
 * Returns -1 (and sets the error) on an invalid spec. */
int64_t segb_mult_count_segregated(int in_h, int in_w, int kernel_n, int pad, int c_in,
                                   int c_out);

/* K1, segregation.py:61-70 segregate_kernel, batched over `count` kernels:
 * kern (count, n, n) -> subs = [k00 | k01 | k10 | k11], block (r,s) of shape
 * (count, R(r), R(s)) with k_rs[u, v] = K[2u + r, 2v + s]. Bit-exact copy.
 * dtype applies to both arrays (SEGB_F32 / SEGB_F64 / SEGB_BF16). */
int segb_segregate(const void *kern, int dtype, int64_t count, int kernel_n, void *subs,
                   void *stream);

/* K1 inverse, segregation.py:73-88 merge_subkernels (same packed layout). */
int segb_merge(const void *subs, int dtype, int64_t count, int kernel_n, void *kern,
               void *stream);

/* engines.py:153-160 prepare_layer + engines.py:213-244 PreparedLayer.__init__.
 * bank: device pointer to (c_in, c_out, n, n) of bank_dtype; copied, so the
 * caller may free it afterwards. compute_dtype: SEGB_F32 (fp32 FFMA,
 * the reference's working precision), SEGB_F64 (oracle-grade), SEGB_BF16
 * (bf16 operands, fp32 accumulation, tensor cores where eligible).
 * Runs K1 once (the parity split + operand layout), on `stream`. */
int segb_prepare(const void *bank, int bank_dtype, int c_in, int c_out, int kernel_n, int pad,
                 int engine, int compute_dtype, void *stream, segb_layer **out);

int segb_layer_info(const segb_layer *layer, int *c_in, int *c_out, int *kernel_n, int *pad,
                    int *engine, int *compute_dtype);

/* engines.py:246-256 PreparedLayer.forward -> _forward_segregated :271-291.
 * x: device (batch, c_in, in_h, in_w) of x_dtype; y: device
 * (batch, c_out, out_h, out_w) of y_dtype, sized by segb_output_dims.
 * compute_dtype: as segb_prepare, or -1 for the layer's own. Every output
 * element is written exactly once. */
int segb_forward(const segb_layer *layer, const void *x, int x_dtype, int64_t batch, int in_h,
                 int in_w, void *y, int y_dtype, int compute_dtype, int path, void *stream);

/* bytes of workspace segb_forward_ws needs for this call (0 for K2 and K3b);
 * the same planning as segb_forward, so it fails with the same codes. */
int segb_forward_workspace_bytes(const segb_layer *layer, int x_dtype, int64_t batch, int in_h, int in_w,
                                 int y_dtype, int compute_dtype, int path, int64_t *bytes);

/* segb_forward with a caller-owned device workspace of workspace_bytes bytes
 * (SEGB_ERR_VALUE if smaller than segb_forward_workspace_bytes). Reentrant:
 * concurrent calls on different streams each pass their own workspace. */
int segb_forward_ws(const segb_layer *layer, const void *x, int x_dtype, int64_t batch, int in_h, int in_w,
                    void *y, int y_dtype, int compute_dtype, int path, void *workspace,
                    int64_t workspace_bytes, void *stream);

/* grows the layer-owned workspace that segb_forward uses to at least `bytes`
 * (the only allocation outside segb_prepare; shared by all segb_forward calls
 * on this layer, so concurrent streams should use segb_forward_ws instead). */
int segb_layer_reserve_workspace(segb_layer *layer, int64_t bytes);

/* the kernel family (and operand mode) this call runs, as text, e.g.
 * "K3 implicit GEMM (3xFP16)" or "K3b row-streaming GEMM (bf16)" */
int segb_describe_path(const segb_layer *layer, int x_dtype, int64_t batch, int in_h, int in_w, int y_dtype,
                       int compute_dtype, int path, char *buf, int buf_len);

/* which kernel SEGB_PATH_AUTO picks for this call (SEGB_PATH_DIRECT/IGEMM) */
int segb_select_path(const segb_layer *layer, int x_dtype, int64_t batch, int in_h, int in_w,
                     int compute_dtype);

int segb_release(segb_layer *layer);

/* Layer stacks (the reference's GAN_SUITE generator stacks,
 * bench.py:124-139, which a reference user runs as one layer_forward per layer,
 * engines.py:163-172, through host arrays). layers[0..count) are chained: layer
 * i's output (batch, c_out_i, h_i, w_i) is layer i+1's input, so c_out_i must
 * equal c_in_{i+1} (SEGB_ERR_SHAPE otherwise). Intermediates live in the
 * caller's device workspace in inter_dtype (two ping-pong buffers; the size is
 * segb_stack_workspace_bytes); each layer runs with its own compute dtype and
 * the kernel segb_forward's SEGB_PATH_AUTO picks. Nothing is copied to the
 * host between layers; all launches go to `stream` (capturable as one graph). */
int segb_stack_workspace_bytes(const segb_layer *const *layers, int count, int64_t batch, int in_h,
                               int in_w, int inter_dtype, int64_t *bytes);
/* the same with the stack's input and output dtypes (the workspace also holds
 * the largest per-layer forward workspace, which depends on them) */
int segb_stack_workspace_bytes2(const segb_layer *const *layers, int count, int64_t batch, int in_h,
                                int in_w, int x_dtype, int y_dtype, int inter_dtype, int64_t *bytes);
int segb_stack_forward(const segb_layer *const *layers, int count, const void *x, int x_dtype,
                       int64_t batch, int in_h, int in_w, void *y, int y_dtype, int inter_dtype,
                       void *workspace, int64_t workspace_bytes, void *stream);

/* synth.py:28-39 unit_floats on device: out[i] = float32(float64(
 * splitmix64(seed + i)) * 2^-64), optionally rounded on to bf16. */
int segb_unit_floats(void *out, int dtype, int64_t count, uint64_t seed, void *stream);

/* Dataset images to the device (tensor_io.py:27-52 parse_ppm).
 * src: device (images, height, width, channels) u8, the interleaved PPM payload;
 * dst: device (images, channels, height, width) of dst_dtype with
 * dst = float32(src) / float32(255) (IEEE fp32 division, bitwise the reference's
 * decode; bf16 rounds that value, f64 widens it). */
int segb_u8_hwc_to_chw(const void *src, int64_t images, int height, int width, int channels, void *dst,
                       int dst_dtype, void *stream);

/* number of kernels this library has launched since load (evidence counter) */
int64_t segb_launch_count(void);

/* engines.py:353-406 transpose_conv_reference_counted / _segregated_counted:
 * the instrumented scalar engines on one feature map (in_h, in_w), device
 * pointers. kernel is the merged (n, n) kernel (merge_subkernels of the
 * SubKernelSet for the segregated engine, segregation.py:73-88). out: (out_h,
 * out_w) f64, computed as the reference's Python loops do (fp64, one rounded
 * multiply and one rounded add per tap, (u, v) order); counters[0] = mults,
 * counters[1] = writes, as executed by the kernel (device u64[2], reset here). */
int segb_counted_forward(const void *fmap, int fmap_dtype, int in_h, int in_w, const void *kernel,
                         int kernel_dtype, int kernel_n, int pad, int engine, double *out,
                         unsigned long long *counters, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SEGB200_H */
