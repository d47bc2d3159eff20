// Stage 2, generic variant: output-stationary sparse-gather convolution for
// ANY stride / padding / kernel size / groups (e.g. the T=2 LeNet row and the
// 1x1 rows of Table 2).  Correct first, simple on purpose;
// the shape-specialised register-tile kernels live in gather_fast_*.
//
// Input: the stage-1 tile streams with ONE tile per image (TY = H_out), so an
// entry's code is (i + P)*W + j.  For output row y and column block x0:
//   out[n,k,y,x] = bias[k] + sum over stream entries (c, i, j, v) with
//                  r = i + P - y*T in [0,R), t = j + P - x*T in [0,S) of
//                  v * wpack[g][kb][cl][r][t][j']   (k = kbw*kb + j', pack.cu)
// i.e. exactly Eq. 1 with the zero terms skipped.
//
// Mapping: one warp per (n, group, 32-channel slice, output row y, 32-column
// block); lane = output channel.  Accumulators live in a per-warp shared
// tile acc[x][lane] (each lane owns its column: no atomics; order channel,
// entry (ascending), tap t ascending -> deterministic).  The entry stream is
// warp-uniform (broadcast loads).  Epilogue: + bias (+ ReLU, Eq. 2), rows of
// 32 consecutive x.
#include "sc_internal.h"

namespace sc {

__global__ void __launch_bounds__(256) gather_generic_kernel(
    const uint2* __restrict__ entries, const uint32_t* __restrict__ offs, const float* __restrict__ wpack,
    const float* __restrict__ bias, float* __restrict__ out, int64_t total_warps, int64_t C, int64_t H, int64_t W,
    int64_t K, int64_t R, int64_t S, int64_t T, int64_t P, int64_t Cg, int64_t Kg, int64_t Kg_pad, int64_t kbw,
    int64_t Ho, int64_t Wo, int64_t cap, int relu, Gate gate) {
    if (gate_closed(gate)) return;
    __shared__ float acc_s[8][32][33];
    const unsigned lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    int64_t wid = (int64_t)blockIdx.x * 8 + wib;
    if (wid >= total_warps) return;
    const int64_t xblocks = (Wo + 31) / 32, kq32 = Kg_pad / 32, kblocks = Kg_pad / kbw, G = K / Kg;
    const int64_t xb = wid % xblocks; wid /= xblocks;
    const int64_t y = wid % Ho; wid /= Ho;
    const int64_t kq = wid % kq32; wid /= kq32;   // 32-channel slice: k = 32*kq + lane
    const int64_t kb = kq / (kbw / 32), khalf = kq % (kbw / 32);
    const int64_t g = wid % G;
    const int64_t n = wid / G;
    const int64_t x0 = xb * 32;
    float(*acc)[33] = acc_s[wib];
#pragma unroll 4
    for (int x = 0; x < 32; ++x) acc[x][lane] = 0.0f;

    const uint2* st = entries + n * cap;            // tile 0 of image n
    const uint32_t* of = offs + n * (C + 1);
    const int64_t wrow0 = y * T;                     // window row of tap r = 0 (window starts at input row -P)
    for (int64_t cl = 0; cl < Cg; ++cl) {
        const int64_t c = g * Cg + cl;
        const float* wc = wpack + ((g * kblocks + kb) * Cg + cl) * R * S * kbw + khalf * 32 + lane;
        const uint32_t a = of[c] + 1, b = of[c + 1];  // skip the channel marker
        for (uint32_t e = a; e < b; ++e) {
            const uint2 en = st[e];
            const int64_t wi = (int64_t)en.y / W;
            const int64_t r = wi - wrow0;
            if (r < 0) continue;
            if (r >= R) break;  // entries ascend in (row, column)
            const int64_t j = (int64_t)en.y - wi * W;
            const float v = __uint_as_float(en.x);
            for (int64_t t = 0; t < S; ++t) {
                const int64_t num = j + P - t;
                if (num < 0) break;
                if (num % T) continue;
                const int64_t xo = num / T;
                if (xo < x0 || xo >= x0 + 32 || xo >= Wo) continue;
                acc[xo - x0][lane] = fmaf(v, wc[(r * S + t) * kbw], acc[xo - x0][lane]);
            }
        }
    }
    __syncwarp();
    const int64_t x = x0 + lane;
    for (int kk = 0; kk < 32; ++kk) {
        const int64_t k = kq * 32 + kk;
        if (k >= Kg) break;
        const int64_t kglob = g * Kg + k;
        if (x < Wo) {
            float o = acc[lane][kk] + bias[kglob];
            if (relu) o = fmaxf(o, 0.0f);
            out[((n * K + kglob) * Ho + y) * Wo + x] = o;
        }
    }
}

cudaError_t launch_gather_generic(const Geometry& g, int64_t n, const uint2* entries, const uint32_t* offs,
                                  const float* wpack, const float* bias, float* out, cudaStream_t st,
                                  Gate gate) {
    if (g.tiles != 1) return cudaErrorInvalidValue;  // generic path runs on one tile per image
    const int64_t total_warps = n * g.G * (g.Kg_pad / 32) * g.Ho * ((g.Wo + 31) / 32);
    const int64_t blocks = (total_warps + 7) / 8;
    gather_generic_kernel<<<(unsigned)blocks, 256, 0, st>>>(entries, offs, wpack, bias, out, total_warps, g.C, g.H,
                                                            g.W, g.K, g.R, g.S, g.T, g.P, g.Cg, g.Kg, g.Kg_pad,
                                                            g.kbw, g.Ho, g.Wo, g.cap, g.relu ? 1 : 0, gate);
    return cudaGetLastError();
}

}  // namespace sc
