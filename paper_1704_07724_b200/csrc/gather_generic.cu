// Stage 2, generic variant: output-stationary sparse-gather convolution for
// ANY stride / padding / kernel size / groups (e.g. the T=2 LeNet row and the
// 1x1 rows of Table 2).  Correct first, simple on purpose;
// the shape-specialised register-tile kernels live in gather_fast.cu.
//
// out[n,k,y,x] = bias[k] + sum over nonzero inputs (c,i,j) of the lists whose
// receptive-field tap (r,t) = (i + P - y*T, j + P - x*T) is inside R x S of
//   v * wpack[g][kb][cl][r][t][j]   (k = kbw*kb + j, pack.cu)
// i.e. exactly Eq. 1 with the zero terms skipped.
//
// Mapping: one warp per (n, group, 32-channel block, output row y, 32-column
// block); lane = output channel.  Accumulators live in a per-warp shared
// tile acc[x][lane] (each lane owns its column: no atomics, fixed order:
// channel, entry (ascending scan order), tap t ascending -> deterministic).
// The nonzero stream is warp-uniform (broadcast loads).  The epilogue adds the
// bias (and the optional ReLU, Eq. 2) and stores rows of 32 consecutive x.
#include "sc_internal.h"

namespace sc {

template <typename IdxT>
__global__ void __launch_bounds__(256) gather_generic_kernel(
    const float* __restrict__ values, const IdxT* __restrict__ idx, const uint32_t* __restrict__ counts,
    const float* __restrict__ wpack, const float* __restrict__ bias, float* __restrict__ out,
    int64_t total_warps, int64_t C, int64_t H, int64_t W, int64_t K, int64_t R, int64_t S, int64_t T,
    int64_t P, int64_t Cg, int64_t Kg, int64_t Kg_pad, int64_t kbw, int64_t Ho, int64_t Wo, int64_t th,
    int64_t tiles, int64_t cap, int relu) {
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

    const int64_t i_lo = y * T - P;            // input row of tap r = 0
    const int64_t r_lo = i_lo < 0 ? -i_lo : 0;
    const int64_t i_first = i_lo + r_lo;        // first in-range input row
    const int64_t i_last = (i_lo + R - 1 < H - 1) ? i_lo + R - 1 : H - 1;
    if (i_first <= i_last) {
        const int64_t tile_lo = i_first / th, tile_hi = i_last / th;
        for (int64_t cl = 0; cl < Cg; ++cl) {
            const int64_t c = g * Cg + cl;
            const float* wc = wpack + ((g * kblocks + kb) * Cg + cl) * R * S * kbw + khalf * 32 + lane;
            for (int64_t tile = tile_lo; tile <= tile_hi; ++tile) {
                const int64_t list = (n * C + c) * tiles + tile;
                const uint32_t cnt = counts[list];
                const float* lv = values + list * cap;
                const IdxT* li = idx + list * cap;
                for (uint32_t e = 0; e < cnt; ++e) {
                    const int64_t loc = (int64_t)li[e];
                    const int64_t i = tile * th + loc / W;
                    const int64_t r = i - i_lo;
                    if (r < 0) continue;
                    if (r >= R) break;  // entries ascend in scan order
                    const int64_t j = loc - (loc / W) * W;
                    const float v = lv[e];
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

cudaError_t launch_gather_generic(const Geometry& g, int64_t n, const float* values, const void* idx,
                                  const uint32_t* counts, const float* wpack, const float* bias,
                                  float* out, cudaStream_t st) {
    const int64_t total_warps = n * g.G * (g.Kg_pad / 32) * g.Ho * ((g.Wo + 31) / 32);
    const int64_t blocks = (total_warps + 7) / 8;
    if (g.idx_bytes == 1)
        gather_generic_kernel<uint8_t><<<(unsigned)blocks, 256, 0, st>>>(
            values, (const uint8_t*)idx, counts, wpack, bias, out, total_warps, g.C, g.H, g.W, g.K, g.R,
            g.S, g.T, g.P, g.Cg, g.Kg, g.Kg_pad, g.kbw, g.Ho, g.Wo, g.th, g.tiles, g.cap, g.relu ? 1 : 0);
    else
        gather_generic_kernel<uint16_t><<<(unsigned)blocks, 256, 0, st>>>(
            values, (const uint16_t*)idx, counts, wpack, bias, out, total_warps, g.C, g.H, g.W, g.K, g.R,
            g.S, g.T, g.P, g.Cg, g.Kg, g.Kg_pad, g.kbw, g.Ho, g.Wo, g.th, g.tiles, g.cap, g.relu ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace sc
