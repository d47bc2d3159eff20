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
 *   oracle_compact    -- ISC step 1, PAPER.md:123 (Sec. 4): "skip all the zero
 *                        elements of the input data, and store the non-zero
 *                        values in a vector with their column and row
 *                        information", in the list format of DESIGN.md R9.
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
 * ISC step 1 in the list format of DESIGN.md R9.
 *
 * A list covers TH consecutive input rows of one (n, c) plane:
 *   list id  = (n*C + c) * tiles + tile,  tiles = ceil(H / TH)
 *   entries  = every element x of those rows with x != 0.0f (IEEE compare:
 *              -0.0 is zero, subnormals/NaN/Inf are nonzero), in ascending
 *              row-major scan order
 *   value    = bit copy of x
 *   idx      = (row - tile*TH) * W + col, stored as u8 (idx_bytes == 1) or
 *              u16 (idx_bytes == 2)
 *   count    = number of entries
 * values/idx are [num_lists][cap]; entries beyond count are not written.
 * Returns 0, or -1 on invalid arguments.
 */
int oracle_compact(const float *in, int64_t N, int64_t C, int64_t H, int64_t W,
                   int64_t TH, int64_t idx_bytes, int64_t cap,
                   float *values, void *idx, uint32_t *counts)
{
    if (N < 1 || C < 1 || H < 1 || W < 1 || TH < 1 || TH > H) return -1;
    if (idx_bytes != 1 && idx_bytes != 2) return -1;
    if (TH * W > (idx_bytes == 1 ? 256 : 65536) || cap < TH * W) return -1;
    const int64_t tiles = (H + TH - 1) / TH;
    #pragma omp parallel for schedule(static)
    for (int64_t plane = 0; plane < N * C; ++plane) {
        for (int64_t tile = 0; tile < tiles; ++tile) {
            const int64_t list = plane * tiles + tile;
            uint32_t cnt = 0;
            for (int64_t i = tile * TH; i < H && i < (tile + 1) * TH; ++i) {
                for (int64_t j = 0; j < W; ++j) {
                    const float x = in[(plane * H + i) * W + j];
                    if (x != 0.0f) {
                        const int64_t local = (i - tile * TH) * W + j;
                        memcpy(&values[list * cap + cnt], &x, sizeof(float));
                        if (idx_bytes == 1)
                            ((uint8_t *)idx)[list * cap + cnt] = (uint8_t)local;
                        else
                            ((uint16_t *)idx)[list * cap + cnt] = (uint16_t)local;
                        ++cnt;
                    }
                }
            }
            counts[list] = cnt;
        }
    }
    return 0;
}
