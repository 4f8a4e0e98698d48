/* CPU oracle, plain C restatement of the unified segregated rule.
 *
 * TEST INFRASTRUCTURE ONLY -- a checker for the CUDA path, never the product.
 * Follows the reference's literal per-element statement of Alg. 2 + the
 * odd-padding swap, /root/reference/pkg/src/segconv/engines.py:379-406
 * (`transpose_conv_segregated_counted`), extended over channels as
 * engines.py:163-172 (`layer_forward`: out[co] = sum_ci tconv(x[ci], bank[ci, co]),
 * ascending ci, no bias) and over a leading batch dimension (SPEC.md:253:
 * batch is an independent map over samples).
 *
 *   r = (x + swap) & 1, s = (y + swap) & 1, p = P / 2, swap = P & 1
 *   out[b,co,x,y] = sum_ci sum_{u<R(r)} sum_{v<R(s)}
 *                   X[b,ci,(x+r)/2+u-p,(y+s)/2+v-p] * K[ci,co,2u+r,2v+s]
 *   with X = 0 outside [0,H)x[0,W) (the floor(P/2) zero ring, engines.py:273-275).
 *
 * Accumulates in double. Parity pinned against the reference's own outputs in
 * tests/golden (see tests/test_oracle.py).
 */
#include <stdint.h>

static inline int sub_len(int n, int parity) { return parity == 0 ? (n + 1) / 2 : n / 2; }

static void forward_one(const double *x, const double *bank, double *out, int c_in, int c_out,
                        int h, int w, int n, int pad) {
    const int oh = 2 * h + 2 * pad - n, ow = 2 * w + 2 * pad - n;
    const int p = pad / 2, swap = pad & 1;
    for (int co = 0; co < c_out; ++co)
        for (int xx = 0; xx < oh; ++xx) {
            const int r = (xx + swap) & 1, bx = (xx + r) / 2, R = sub_len(n, r);
            for (int yy = 0; yy < ow; ++yy) {
                const int s = (yy + swap) & 1, by = (yy + s) / 2, C = sub_len(n, s);
                double acc = 0.0;
                for (int ci = 0; ci < c_in; ++ci) {
                    const double *xc = x + (int64_t)ci * h * w;
                    const double *kc = bank + ((int64_t)ci * c_out + co) * n * n;
                    for (int u = 0; u < R; ++u) {
                        const int ii = bx + u - p;
                        if (ii < 0 || ii >= h) continue;
                        for (int v = 0; v < C; ++v) {
                            const int jj = by + v - p;
                            if (jj < 0 || jj >= w) continue;
                            acc += xc[(int64_t)ii * w + jj] * kc[(2 * u + r) * n + 2 * v + s];
                        }
                    }
                }
                out[((int64_t)co * oh + xx) * ow + yy] = acc;
            }
        }
}

/* x: (batch, c_in, h, w) fp64; bank: (c_in, c_out, n, n) fp64; out: (batch, c_out, oh, ow). */
int oracle_forward_f64(const double *x, const double *bank, double *out, int64_t batch, int c_in,
                       int c_out, int h, int w, int n, int pad) {
    if (n < 2 || pad < 0 || h < 1 || w < 1 || c_in < 1 || c_out < 1) return 1;
    const int oh = 2 * h + 2 * pad - n, ow = 2 * w + 2 * pad - n;
    if (oh < 1 || ow < 1) return 1;
    for (int64_t b = 0; b < batch; ++b)
        forward_one(x + b * (int64_t)c_in * h * w, bank, out + b * (int64_t)c_out * oh * ow, c_in,
                    c_out, h, w, n, pad);
    return 0;
}

/* analysis.py:46-57: useful MACs per sample. */
int64_t oracle_mult_count(int h, int w, int n, int pad, int c_in, int c_out) {
    const int oh = 2 * h + 2 * pad - n, ow = 2 * w + 2 * pad - n, swap = pad & 1;
    int64_t total = 0;
    for (int r = 0; r < 2; ++r) {
        const int st_r = (r + swap) % 2, rows = (oh - st_r + 1) / 2 > 0 ? (oh - st_r + 1) / 2 : 0;
        for (int s = 0; s < 2; ++s) {
            const int st_s = (s + swap) % 2, cols = (ow - st_s + 1) / 2 > 0 ? (ow - st_s + 1) / 2 : 0;
            total += (int64_t)rows * cols * sub_len(n, r) * sub_len(n, s);
        }
    }
    return total * c_in * c_out;
}
