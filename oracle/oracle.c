/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the forward convolution of
 * Shi & Chu, "Speeding up Convolutional Neural Networks By Exploiting the
 * Sparsity of Rectifier Units" (arXiv 1704.07724; /root/reference/PAPER.md).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  The product (libsparseconv.so and
 * paper_1704_07724_b200/) never links, imports or calls it, and it shares no
 * code, header or table with the CUDA path.
 *
 * Functions:
 *   oracle_conv_fp64  -- the definition, PAPER.md:68-72 (Sec. 3, Eq. 1) with the
 *                        stride T and padding P of Table 1,
 *                        plus batch, bias and groups (readings R2-R4).
 *                        Accumulates in double, loop order n,k,y,x | c,r,t.
 *                        Also returns mass = sum |in|*|W| over the receptive
 *                        field (the tolerance scale of the north star).
 *   oracle_compact_lists -- ISC step 1, PAPER.md:123 (Sec. 4): "skip all the
 *                        zero elements of the input data, and store the
 *                        non-zero values in a vector with their column and row
 *                        information": per (image, channel, row tile) the
 *                        nonzero values with their (row, column), row-major.
 *                        The kernel's own stream format (stage-2 instruction
 *                        stream, R9) is derived from these lists by
 *                        a test-side adapter (tests/r9_adapter.py), not here.
 *   oracle_conv_backward_fp64 -- SURVEY 8f row f4: the gradients of Eq. 1
 *                        (chain rule) for training, where the paper measures
 *                        the sparsity (Sec. 1; Sec. 3);
 *                        the input-gradient is taken through the producing
 *                        ReLU (Eq. 2), R19-R20.
 *
 * Build: gcc -O2 -fopenmp -fPIC -shared (no -ffast-math: rounding and IEEE
 * zero tests must be exact).
 */
#include <stdint.h>
#include <string.h>
#include <math.h>

/* Output extent, R1: floor((H + 2P - R)/T) + 1 (PAPER.md:37 garbled). */
static int64_t out_extent(int64_t in, int64_t pad, int64_t k, int64_t stride) {
    return (in + 2 * pad - k) / stride + 1;
}

/*
 * out[n,k,y,x] = bias[k] + sum_{c in group(k)} sum_{r<R} sum_{t<S}
 *                in[n, c, y*T + r - P, x*T + t - P] * W[k, c - g*Cg, r, t]
 * with reads outside [0,H)x[0,W) equal to zero (virtual padding).
 *
 * in   : float [N][C][H][W]
 * w    : float [K][C/G][R][S]
 * bias : float [K] or NULL (zero bias)
 * out  : double [N][K][Ho][Wo]
 * mass : double [N][K][Ho][Wo] or NULL; sum of |in|*|W| over the same terms.
 * Returns 0, or -1 on invalid shape.
 */
int oracle_conv_fp64(const float *in, const float *w, const float *bias,
                     int64_t N, int64_t C, int64_t H, int64_t W,
                     int64_t K, int64_t R, int64_t S,
                     int64_t stride, int64_t pad, int64_t groups,
                     double *out, double *mass)
{
    if (N < 1 || C < 1 || H < 1 || W < 1 || K < 1 || R < 1 || S < 1 ||
        stride < 1 || pad < 0 || groups < 1 || C % groups || K % groups)
        return -1;
    if (R > H + 2 * pad || S > W + 2 * pad) return -1;
    const int64_t Ho = out_extent(H, pad, R, stride);
    const int64_t Wo = out_extent(W, pad, S, stride);
    const int64_t Cg = C / groups, Kg = K / groups;

    #pragma omp parallel for collapse(2) schedule(static)
    for (int64_t n = 0; n < N; ++n) {
        for (int64_t k = 0; k < K; ++k) {
            const int64_t g = k / Kg;
            for (int64_t y = 0; y < Ho; ++y) {
                for (int64_t x = 0; x < Wo; ++x) {
                    double acc = bias ? (double)bias[k] : 0.0;
                    double m = 0.0;
                    for (int64_t cl = 0; cl < Cg; ++cl) {
                        const int64_t c = g * Cg + cl;
                        for (int64_t r = 0; r < R; ++r) {
                            const int64_t i = y * stride + r - pad;
                            if (i < 0 || i >= H) continue;
                            for (int64_t t = 0; t < S; ++t) {
                                const int64_t j = x * stride + t - pad;
                                if (j < 0 || j >= W) continue;
                                const double v = (double)in[((n * C + c) * H + i) * W + j];
                                const double wt = (double)w[((k * Cg + cl) * R + r) * S + t];
                                acc += v * wt;
                                m += fabs(v) * fabs(wt);
                            }
                        }
                    }
                    const int64_t o = ((n * K + k) * Ho + y) * Wo + x;
                    out[o] = acc;
                    if (mass) mass[o] = m;
                }
            }
        }
    }
    return 0;
}

/*
 * ISC step 1, PAPER.md:123 (Sec. 4, "Inverse Sparse Convolution"): "we skip all
 * the zero elements of the input data, and store the non-zero values in a
 * vector with their column and row information".
 *
 * One vector (list) per (image n, channel c, row tile t), the tile being input
 * rows [t*TH, min((t+1)*TH, H)) of the plane (TH = H gives one
 * list per plane).  A plain row-major scan of the plane: for every element
 * x = in[n,c,i,j] with x != 0.0f (IEEE compare: -0.0 is zero; subnormals, NaN
 * and Inf are nonzero -- DESIGN.md R7), in ascending (i, j):
 *     values[l][k] = bit copy of x,  rows[l][k] = i,  cols[l][k] = j
 * and counts[l] = number of such elements, l = (n*C + c)*tiles + t.  Every list
 * has TH*W slots; slots at or beyond counts[l] are not written.
 * values: u32 [N][C][tiles][TH*W]; rows, cols: i32 same; counts: u32 [N][C][tiles].
 * Returns 0, or -1 on invalid arguments.
 */
int oracle_compact_lists(const float *in, int64_t N, int64_t C, int64_t H, int64_t W, int64_t TH,
                         uint32_t *values, int32_t *rows, int32_t *cols, uint32_t *counts)
{
    if (N < 1 || C < 1 || H < 1 || W < 1 || TH < 1) return -1;
    const int64_t tiles = (H + TH - 1) / TH, slots = TH * W;
    #pragma omp parallel for collapse(2) schedule(static)
    for (int64_t n = 0; n < N; ++n) {
        for (int64_t c = 0; c < C; ++c) {
            for (int64_t t = 0; t < tiles; ++t) {
                const int64_t l = (n * C + c) * tiles + t;
                uint32_t k = 0;
                for (int64_t i = t * TH; i < (t + 1) * TH && i < H; ++i) {
                    for (int64_t j = 0; j < W; ++j) {
                        const float x = in[((n * C + c) * H + i) * W + j];
                        if (x != 0.0f) {
                            uint32_t bits;
                            memcpy(&bits, &x, sizeof bits);
                            values[l * slots + k] = bits;
                            rows[l * slots + k] = (int32_t)i;
                            cols[l * slots + k] = (int32_t)j;
                            ++k;
                        }
                    }
                }
                counts[l] = k;
            }
        }
    }
    return 0;
}

/*
 * Backward of Eq. 1 (R19, R20).  With out = conv(in, W) + bias and
 * the upstream gradient dout = dL/dout [N][K][Ho][Wo]:
 *
 *   dw[k][cl][r][t] = sum_{n,y,x} in[n, g*Cg+cl, y*T+r-P, x*T+t-P] * dout[n,k,y,x]
 *                     (g = k / Kg; reads outside the plane are zero)
 *   dbias[k]        = sum_{n,y,x} dout[n,k,y,x]
 *   dz[n][c][i][j]  = [in[n,c,i,j] != 0] *
 *                     sum_{k in group(c)} sum_{r,t : y = (i+P-r)/T, x = (j+P-t)/T
 *                                          integral and in range} W[k][cl][r][t] * dout[n,k,y,x]
 *
 * dz is dL/dz for in = ReLU(z) (Eq. 2: the derivative is 1 where the ReLU
 * output is positive, 0 elsewhere; for a ReLU output in != 0 <=> in > 0).
 * Accumulation in double; the loop orders are the definitions' (k,cl,r,t |
 * n,y,x) and (n,c,i,j | k,r,t).  dw_mass / dz_mass (nullable) are the sums of
 * the absolute values of the same products (tolerance scales).
 * in, dout: float; w: float [K][Cg][R][S]; outputs double.
 * Returns 0, or -1 on invalid shape.
 */
int oracle_conv_backward_fp64(const float *in, const float *w, const float *dout,
                              int64_t N, int64_t C, int64_t H, int64_t W,
                              int64_t K, int64_t R, int64_t S,
                              int64_t stride, int64_t pad, int64_t groups,
                              double *dw, double *dw_mass, double *dbias,
                              double *dz, double *dz_mass)
{
    if (N < 1 || C < 1 || H < 1 || W < 1 || K < 1 || R < 1 || S < 1 ||
        stride < 1 || pad < 0 || groups < 1 || C % groups || K % groups)
        return -1;
    if (R > H + 2 * pad || S > W + 2 * pad) return -1;
    const int64_t Ho = out_extent(H, pad, R, stride);
    const int64_t Wo = out_extent(W, pad, S, stride);
    const int64_t Cg = C / groups, Kg = K / groups;
    const int64_t T = stride, P = pad;

    if (dw) {
        #pragma omp parallel for collapse(2) schedule(static)
        for (int64_t k = 0; k < K; ++k) {
            for (int64_t cl = 0; cl < Cg; ++cl) {
                const int64_t c = (k / Kg) * Cg + cl;
                for (int64_t r = 0; r < R; ++r) {
                    for (int64_t t = 0; t < S; ++t) {
                        double acc = 0.0, m = 0.0;
                        for (int64_t n = 0; n < N; ++n) {
                            for (int64_t y = 0; y < Ho; ++y) {
                                const int64_t i = y * T + r - P;
                                if (i < 0 || i >= H) continue;
                                for (int64_t x = 0; x < Wo; ++x) {
                                    const int64_t j = x * T + t - P;
                                    if (j < 0 || j >= W) continue;
                                    const double v = (double)in[((n * C + c) * H + i) * W + j];
                                    const double d = (double)dout[((n * K + k) * Ho + y) * Wo + x];
                                    acc += v * d;
                                    m += fabs(v) * fabs(d);
                                }
                            }
                        }
                        const int64_t o = ((k * Cg + cl) * R + r) * S + t;
                        dw[o] = acc;
                        if (dw_mass) dw_mass[o] = m;
                    }
                }
            }
        }
    }
    if (dbias) {
        for (int64_t k = 0; k < K; ++k) {
            double acc = 0.0;
            for (int64_t n = 0; n < N; ++n)
                for (int64_t y = 0; y < Ho; ++y)
                    for (int64_t x = 0; x < Wo; ++x)
                        acc += (double)dout[((n * K + k) * Ho + y) * Wo + x];
            dbias[k] = acc;
        }
    }
    if (dz) {
        #pragma omp parallel for collapse(2) schedule(static)
        for (int64_t n = 0; n < N; ++n) {
            for (int64_t c = 0; c < C; ++c) {
                const int64_t g = c / Cg, cl = c - g * Cg;
                for (int64_t i = 0; i < H; ++i) {
                    for (int64_t j = 0; j < W; ++j) {
                        const int64_t o = ((n * C + c) * H + i) * W + j;
                        double acc = 0.0, m = 0.0;
                        if (in[o] != 0.0f) {
                            for (int64_t k = g * Kg; k < (g + 1) * Kg; ++k) {
                                for (int64_t r = 0; r < R; ++r) {
                                    const int64_t yT = i + P - r;
                                    if (yT < 0 || yT % T) continue;
                                    const int64_t y = yT / T;
                                    if (y >= Ho) continue;
                                    for (int64_t t = 0; t < S; ++t) {
                                        const int64_t xT = j + P - t;
                                        if (xT < 0 || xT % T) continue;
                                        const int64_t x = xT / T;
                                        if (x >= Wo) continue;
                                        const double wt = (double)w[((k * Cg + cl) * R + r) * S + t];
                                        const double d = (double)dout[((n * K + k) * Ho + y) * Wo + x];
                                        acc += wt * d;
                                        m += fabs(wt) * fabs(d);
                                    }
                                }
                            }
                        }
                        dz[o] = acc;
                        if (dz_mass) dz_mass[o] = m;
                    }
                }
            }
        }
    }
    return 0;
}
