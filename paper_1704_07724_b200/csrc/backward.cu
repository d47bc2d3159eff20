// Backward pass with sparse activations (the paper measures
// the ReLU sparsity during training; definitions DESIGN.md
// R19-R20, oracle/oracle.c oracle_conv_backward_fp64):
//
//   dW[k,c,r,t] = sum_{n,y,x} in[n,c,yT+r-P,xT+t-P] * dout[n,k,y,x]   (wgrad)
//   dz[n,c,i,j] = [in != 0] * sum_{k,r,t} W[k,c,r,t] * dout[n,k,y,x]    (dgrad through the ReLU)
//   dbias[k]    = sum_{n,y,x} dout[n,k,y,x]
//
// Both sums only run over the nonzero inputs: every term of wgrad carries a
// factor in[...], and dgrad is needed only where the ReLU derivative is 1.
// The nonzeros come from the plane-major stage-1 lists (plist/prow of
// compact.cu, one (bits, flat index) list per (image, channel) plane, row
// prefix for band ranges).
//
// Kernel structure (bwd_kernel<R,S,KL,T,WGRAD>): one CTA = 16 warps; warp w
// owns one input channel; lane l covers the output channels
// k = kc*KC + l + 32q (q < KL) of a KC = 32*KL chunk.  The CTA walks a sequence of
// tiles (image n, k-chunk kc, band of BY output rows); each tile is
// dout[n][kc*KC..+KC][band] staged into shared memory as [k][pixels | 1]
// (odd row stride: conflict-free staging stores and per-tap loads).  Per nonzero (v, i, j) of the warp's plane whose
// taps reach the band, per tap (r, t) with y = (i+P-r)/T, x = (j+P-t)/T
// integral and in the band (two bit masks per nonzero, R + S bits): KL shared
// loads d[q] at constant offsets from the nonzero's base address (T = 1) and
//   wgrad: acc[r][t][q] += v * d[q]           (registers, across all tiles)
//   dgrad: part += W[r][t][q] * d[q]          (W in registers per (c, kc)),
//          then a warp sum and one read-modify-write of dz by lane 0
// The branch per tap is warp-uniform (all lanes share the nonzero).
// wgrad: grid (split of images, cblock, kc, group); partial dW per split into
// a workspace, summed in split order by bwd_reduce_kernel (deterministic).
// dgrad: grid (split of images, cblock, group); tiles walk (kc, n, band); per
// (n, kc) the warp accumulates its channel's plane in shared memory and then
// stores it (kc = 0) or adds it (kc > 0, in k-chunk order) to dz.
#include <cuda_runtime.h>

#include "sc_internal.h"

namespace sc {
namespace bwd {

constexpr int kWarps = 16;               // compute warps (one input channel each)
constexpr int kThreads = kWarps * 32;
constexpr int kBlock = kThreads + 32;    // + one producer warp (TMA issue in bulk mode)

struct Args {
    const uint2* plist;     // [N*C][H*W] (bits, i*W + j), row-major order
    const uint32_t* prow;   // [N*C][H+1] nonzeros before row r
    const float* dout;      // [N][K][Ho][Wo]
    const float* wpack;     // forward packed weights [G][kblocks][Cg][R][S][kbw]
    float* ws;              // wgrad partials [splits][K][Cg][R][S]
    float* dz;              // [N][C][H][W]
    int n, C, H, W, K, Cg, Kg, Ho, Wo, T, P;
    int kbw, fkblocks;      // forward weight packing
    uint32_t wmagic;        // floor(2^32 / W) + 1: i = umulhi(i*W + j, wmagic) for i*W + j < 2^32 / W
    int KC, kchunks, cblocks, BY, bands, splits, ipc;  // ipc: images per split
    int bulk;               // whole-plane tiles by one TMA bulk copy, double buffered (see bwd_geometry)
    int tile_floats;        // shared memory: tiles, then (dgrad) one H*W dz plane per warp, then 2 mbarriers
};

template <bool B>
struct bool_const {
    static constexpr bool value = B;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// One bulk copy of `bytes` (multiple of 16, 16-byte aligned ends) completing on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Stage dout[n][g*Kg + kc*KC + k][y0 .. y0+rows)[0..Wo) (k >= Kg -> 0) as
// tile[k*PS + pixel], PS = pixels rounded up to odd: the hot loop's loads
// (lanes over consecutive k at one pixel) hit 32 distinct banks, and the
// staging stores (lanes over consecutive pixels of one k row) too.  Global
// reads are coalesced; RB x MB independent loads in flight per thread.
template <int KL>
__device__ __forceinline__ void stage(const Args& a, float* tile, int n, int g, int kc, int y0, int rows, int PS) {
    constexpr int KC = 32 * KL, RB = KC / kWarps < 2 ? KC / kWarps : 2, MB = 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pix = rows * a.Wo;
    const int pblocks = (pix + 31) >> 5;
    const int64_t HoWo = (int64_t)a.Ho * a.Wo;
    const float* base = a.dout + ((int64_t)n * a.K + (int64_t)g * a.Kg + (int64_t)kc * KC) * HoWo + (int64_t)y0 * a.Wo;
    const int kvalid = a.Kg - kc * KC;  // k < kvalid are real filters
    for (int k0 = warp; k0 < KC; k0 += RB * kWarps) {
        for (int m0 = 0; m0 < pblocks; m0 += MB) {
            float v[RB][MB];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) {
                const int k = k0 + rb * kWarps;
                const float* src = base + (int64_t)k * HoWo;
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    const int p = (m0 + mb) * 32 + lane;
                    v[rb][mb] = (k < kvalid && p < pix) ? __ldg(src + p) : 0.f;
                }
            }
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) {
                const int k = k0 + rb * kWarps;
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    const int p = (m0 + mb) * 32 + lane;
                    if (p < pix) tile[k * PS + p] = v[rb][mb];
                }
            }
        }
    }
}

template <int R, int S, int KL, int T, bool WGRAD>
__global__ void __launch_bounds__(kBlock, 1) bwd_kernel(const Args a) {
    extern __shared__ __align__(16) float smem[];
    constexpr int KC = 32 * KL;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int HoWo = a.Ho * a.Wo;
    float* dzbuf = smem + a.tile_floats + warp * a.H * a.W;  // dgrad: this warp's dz plane of the current image
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.tile_floats + kWarps * a.H * a.W + 2);
    full = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(full) + 15) & ~(uintptr_t)15);
    uint64_t* empty = full + 2;  // bulk mode: buffer b released by all compute warps
    // block -> (split, cblock, kc (wgrad), group)
    int b = blockIdx.x;
    const int split = b % a.splits;
    b /= a.splits;
    const int cb = b % a.cblocks;
    b /= a.cblocks;
    int kc_fixed = 0;
    if constexpr (WGRAD) {
        kc_fixed = b % a.kchunks;
        b /= a.kchunks;
    }
    const int g = b;
    const bool producer = warp == kWarps;
    const int cl = cb * kWarps + warp;  // channel in group
    const bool active = !producer && cl < a.Cg;
    const int c = g * a.Cg + cl;
    const int n0 = split * a.ipc;
    const int n1 = min(a.n, n0 + a.ipc);
    if (n0 >= n1) return;
    const int per_img = WGRAD ? a.bands : a.kchunks * a.bands;
    const int ntiles = (n1 - n0) * per_img;
    const int HW = a.H * a.W;

    float acc[R * S][KL];
    float wr[R * S][KL];
#pragma unroll
    for (int u = 0; u < R * S; ++u)
#pragma unroll
        for (int q = 0; q < KL; ++q) acc[u][q] = 0.f;
    int wr_kc = -1;

    // bulk mode: tile `it` (image n, chunk kc) is dout[n][g*Kg + kc*KC ..][all pixels], contiguous
    // tile order: wgrad (image, band); dgrad (k-chunk, image, band) -- k-chunk major, so a warp
    // reloads its channel's weights once per k-chunk, not once per tile
    auto decode = [&](int it, int& n, int& kc, int& band) {
        if constexpr (WGRAD) {
            n = n0 + it / a.bands;
            kc = kc_fixed;
            band = it - (it / a.bands) * a.bands;
        } else {
            const int per_kc = (n1 - n0) * a.bands;
            kc = it / per_kc;
            const int rem = it - kc * per_kc;
            n = n0 + rem / a.bands;
            band = rem - (rem / a.bands) * a.bands;
        }
    };
    auto issue = [&](int it) {
        int n, kc, band;
        decode(it, n, kc, band);
        const int rows = min(KC, a.Kg - kc * KC);
        const float* src = a.dout + ((int64_t)n * a.K + (int64_t)g * a.Kg + (int64_t)kc * KC) * HoWo;
        bulk_g2s(smem + (it & 1) * KC * HoWo, src, (unsigned)(rows * HoWo * 4), full + (it & 1));
    };
    if (a.bulk) {
        // the buffers start zeroed: rows of padding filters (k >= Kg, never copied) read as 0
        // or as an earlier tile's finite dout values, which meet only zero weights (dgrad) or
        // accumulators that are never written out (wgrad)
        for (int e = threadIdx.x; e < 2 * KC * HoWo; e += kBlock) smem[e] = 0.f;
        if (threadIdx.x == 0) {
            mbar_init(full, 1);
            mbar_init(full + 1, 1);
            mbar_init(empty, kWarps);
            mbar_init(empty + 1, kWarps);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (producer) {  // tile it+2 refills buffer it&1 once all compute warps released tile it
            if (lane == 0)
                for (int it = 0; it < ntiles; ++it) {
                    if (it >= 2) mbar_wait(empty + (it & 1), (unsigned)(((it >> 1) - 1) & 1));
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(it);
                }
            return;
        }
    }
    for (int it = 0; it < ntiles; ++it) {
        int n, kc, band;
        decode(it, n, kc, band);
        const int y0 = band * a.BY, y1 = min(a.Ho, y0 + a.BY);
        int PS;
        float* tile;
        if (a.bulk) {
            PS = HoWo;  // odd (bwd_geometry)
            tile = smem + (it & 1) * KC * HoWo;
            if (it >= 1) {  // done with tile it-1: the producer may refill its buffer with tile it+1
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + ((it - 1) & 1));
            }
            mbar_wait(full + (it & 1), (unsigned)((it >> 1) & 1));
        } else {
            if (it > 0) __syncthreads();  // everyone is done with the previous tile
            PS = ((y1 - y0) * a.Wo) | 1;  // odd k-row stride of this tile
            tile = smem;
            if (!producer) stage<KL>(a, tile, n, g, kc, y0, y1 - y0, PS);
            __syncthreads();
        }
        if (!active) continue;
        const int64_t plane = (int64_t)n * a.C + c;
        if constexpr (!WGRAD) {
            if (band == 0) {  // first band of (image, k-chunk): this chunk's partial plane starts at zero
                for (int e = lane; e < HW; e += 32) dzbuf[e] = 0.f;
                __syncwarp();
            }
            if (kc != wr_kc) {  // W[k][cl][r][t] for this lane's k, from the forward packing
                wr_kc = kc;
#pragma unroll
                for (int q = 0; q < KL; ++q) {
                    const int kl = kc * KC + lane + 32 * q;
                    const bool ok = kl < a.Kg;
                    const int kb = ok ? kl / a.kbw : 0, kx = ok ? kl - kb * a.kbw : 0;
                    // position of filter kx inside a packed k-block (pack.cu: KL=3 blocks store the
                    // pair (3l, 3l+1) at 2l and the single 3l+2 at 64 + l)
                    const int kk = a.kbw == 96 ? (kx % 3 < 2 ? 2 * (kx / 3) + kx % 3 : 64 + kx / 3) : kx;
                    const float* wp = a.wpack + (((int64_t)g * a.fkblocks + kb) * a.Cg + cl) * (R * S) * a.kbw + kk;
#pragma unroll
                    for (int u = 0; u < R * S; ++u) wr[u][q] = ok ? __ldg(wp + u * a.kbw) : 0.f;
                }
            }
        }
        // input rows whose taps reach output rows [y0, y1)
        const int ilo = max(0, y0 * T - a.P), ihi = min(a.H - 1, (y1 - 1) * T - a.P + R - 1);
        if (ilo <= ihi) {
        const uint32_t* pr = a.prow + plane * (a.H + 1);
        const uint32_t e0 = __ldg(pr + ilo), e1 = __ldg(pr + ihi + 1);
        const uint2* lst = a.plist + plane * HW;
        uint2 mine = make_uint2(0u, 0u);  // entries e0+32m+lane, fetched 32 at a time (one coalesced load)
        for (uint32_t e = e0; e < e1; ++e) {
            const uint32_t sl = (e - e0) & 31u;
            if (sl == 0) {
                const uint32_t ee = e + lane;
                mine = ee < e1 ? __ldg(lst + ee) : make_uint2(0u, 0u);
            }
            uint2 en;
            en.x = __shfl_sync(0xffffffffu, mine.x, (int)sl);
            en.y = __shfl_sync(0xffffffffu, mine.y, (int)sl);
            const float v = __uint_as_float(en.x);
            const int i = (int)__umulhi(en.y, a.wmagic), j = (int)en.y - i * a.W;
            // taps reaching the band: y = (i+P-r)/T in [y0, y1), x = (j+P-t)/T in [0, Wo), integral
            const int ip = i + a.P, jp = j + a.P;
            const int rlo = max(0, ip - T * (y1 - 1)), rhi = min(R - 1, ip - T * y0);
            const int tlo = max(0, jp - T * (a.Wo - 1)), thi = min(S - 1, jp);
            uint32_t rmask = rlo <= rhi ? (2u << rhi) - (1u << rlo) : 0u;
            uint32_t tmask = tlo <= thi ? (2u << thi) - (1u << tlo) : 0u;
            if constexpr (T == 2) {
                rmask &= (ip & 1) ? 0xAAAAAAAAu : 0x55555555u;
                tmask &= (jp & 1) ? 0xAAAAAAAAu : 0x55555555u;
            }
            // lane reads k = lane + 32q at tile[k*PS + pixel]; T == 1: tap (r, t) is pixel
            // (ip - y0 - r)*Wo + (jp - t)
            const float* abase = tile + lane * PS + (ip - y0) * a.Wo + jp;
            float part = 0.f;
            // interior nonzeros (every tap reaches the band and the plane) take an unpredicated copy
            // of the tap loop; the others a branch-free one where a tap outside loads nothing and
            // adds v*0 or W*0 -- in both, all taps' loads can be issued ahead of the FMAs
            auto taps = [&](auto all) {
                constexpr bool kAll = decltype(all)::value;
#pragma unroll
                for (int r = 0; r < R; ++r) {
#pragma unroll
                    for (int t = 0; t < S; ++t) {
                        const bool ok = kAll || ((rmask >> r) & (tmask >> t) & 1u) != 0u;
                        const float* src;
                        if constexpr (T == 1)
                            src = abase - r * a.Wo - t;
                        else
                            src = tile + lane * PS + ((ip - r) / T - y0) * a.Wo + (jp - t) / T;
                        float d[KL];
#pragma unroll
                        for (int q = 0; q < KL; ++q) d[q] = ok ? src[32 * q * PS] : 0.f;
#pragma unroll
                        for (int q = 0; q < KL; ++q) {
                            if constexpr (WGRAD)
                                acc[r * S + t][q] = fmaf(v, d[q], acc[r * S + t][q]);
                            else
                                part = fmaf(wr[r * S + t][q], d[q], part);
                        }
                    }
                }
            };
            if (T == 1 && rmask == (1u << R) - 1u && tmask == (1u << S) - 1u)
                taps(bool_const<true>{});
            else
                taps(bool_const<false>{});
            if constexpr (!WGRAD) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                if (lane == 0) dzbuf[en.y] += part;
            }
        }
        }
        if constexpr (!WGRAD) {
            if (band == a.bands - 1) {  // last band: store (first k-chunk) or add (later ones, in order)
                __syncwarp();
                float* dzp = a.dz + plane * HW;
                if (kc == 0)
                    for (int e = lane; e < HW; e += 32) dzp[e] = dzbuf[e];
                else
                    for (int e = lane; e < HW; e += 32) dzp[e] += dzbuf[e];
            }
        }
    }
    if constexpr (WGRAD) {
        if (active) {
#pragma unroll
            for (int q = 0; q < KL; ++q) {
                const int kl = kc_fixed * KC + lane + 32 * q;
                if (kl >= a.Kg) continue;
                float* dst = a.ws + (((int64_t)split * a.K + (int64_t)g * a.Kg + kl) * a.Cg + cl) * (R * S);
#pragma unroll
                for (int u = 0; u < R * S; ++u) dst[u] = acc[u][q];
            }
        }
    }
}

// dw[i] = sum over splits (in split order) of ws[split][i]; i over K*Cg*R*S.
__global__ void bwd_reduce_kernel(const float* __restrict__ ws, int splits, int64_t count, float* __restrict__ dw) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int sp = 0; sp < splits; ++sp) s += __ldg(ws + sp * count + i);
        dw[i] = s;
    }
}

// dbias[k] = sum_{n, p} dout[n][k][p]: one CTA per k, lanes over pixels, fixed order.
__global__ void __launch_bounds__(256) bwd_dbias_kernel(const float* __restrict__ dout, int n, int K, int HW,
                                                        float* __restrict__ dbias) {
    __shared__ float part[8];
    const int k = blockIdx.x;
    float s = 0.f;
    for (int img = threadIdx.x >> 5; img < n; img += 8) {
        const float* p = dout + ((int64_t)img * K + k) * HW;
        for (int e = threadIdx.x & 31; e < HW; e += 32) s += __ldg(p + e);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += part[w];
        dbias[k] = t;
    }
}

template <int R, int S, int KL>
cudaError_t launch_rs(const Args& a, int G, bool wgrad, size_t smem, cudaStream_t st) {
    auto kern = a.T == 1 ? (wgrad ? bwd_kernel<R, S, KL, 1, true> : bwd_kernel<R, S, KL, 1, false>)
                         : (wgrad ? bwd_kernel<R, S, KL, 2, true> : bwd_kernel<R, S, KL, 2, false>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = (int64_t)a.splits * a.cblocks * (wgrad ? a.kchunks : 1) * G;
    kern<<<(unsigned)grid, kBlock, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace bwd

// Image splits for a launch of `per` CTAs per split: the count (<= min(n, smax))
// whose grid fills its last wave of 148 one-CTA-per-SM blocks best, fewest first.
static int64_t pick_splits(int64_t per, int64_t n, int64_t smax) {
    const int64_t lim = n < smax ? n : smax;
    int64_t best = 1;
    double best_eff = -1.0;
    for (int64_t sp = 1; sp <= lim; ++sp) {
        const int64_t ctas = per * sp, waves = (ctas + 147) / 148;
        const double eff = (double)ctas / (double)(waves * 148);
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = sp;
        }
    }
    return best;
}

// Geometry of the backward kernels; supported == false -> SC_ERR_UNSUPPORTED.
void backward_geometry(const Geometry& g, BwdGeom* b) {
    *b = BwdGeom{};
    const int64_t rs = g.R * g.S;
    b->supported = compact_uses_counts(g) && g.T <= 2 &&
                   ((g.R == 1 && g.S == 1) || (g.R == 3 && g.S == 3) || (g.R == 5 && g.S == 5));
    if (!b->supported) return;
    const int64_t klmax = rs <= 9 ? 4 : 2;
    int64_t kl = (g.Kg + 31) / 32;
    kl = kl >= 4 ? 4 : kl >= 2 ? 2 : 1;
    if (kl > klmax) kl = klmax;
    if (kl == 3) kl = 4;
    b->kl = kl;
    b->kc = 32 * kl;
    b->kchunks = (g.Kg + b->kc - 1) / b->kc;
    b->cblocks = (g.Cg + bwd::kWarps - 1) / bwd::kWarps;
    // one tile within 220 KB less the dgrad planes (16 x H*W floats): kc rows of (by*Wo | 1) floats
    const int64_t planes_bytes = (int64_t)bwd::kWarps * g.H * g.W * 4 + 64;
    const int64_t budget = 220 * 1024 - planes_bytes;
    int64_t by = g.Ho;
    while (by > 1 && b->kc * ((by * g.Wo) | 1) * 4 > budget) --by;
    b->by = by;
    b->bands = (g.Ho + by - 1) / by;
    b->tile_floats = b->kc * ((by * g.Wo) | 1);
    // whole-plane tiles with an odd pixel count whose k rows start 16-byte aligned for every
    // (n, group, chunk) and whose copy sizes are multiples of 16 bytes: one bulk copy per tile
    const int64_t howo = g.Ho * g.Wo;
    b->bulk = (howo & 1) && g.K % 4 == 0 && g.Kg % 4 == 0 && 2 * b->kc * howo * 4 <= budget;
    if (b->bulk) {
        b->by = g.Ho;
        b->bands = 1;
        b->tile_floats = 2 * b->kc * howo;
    }
    b->smem = (size_t)b->tile_floats * sizeof(float) + (size_t)planes_bytes;
    if (b->smem > 227 * 1024) {
        b->supported = false;
        return;
    }
    // at most about two waves of 1-CTA-per-SM blocks (bounds the wgrad workspace)
    const int64_t per_split_w = g.G * b->cblocks * b->kchunks;
    b->splits_w = (296 + per_split_w - 1) / per_split_w;
    if (b->splits_w > g.N) b->splits_w = g.N;
    const int64_t per_split_d = g.G * b->cblocks;
    b->splits_d = (296 + per_split_d - 1) / per_split_d;
    if (b->splits_d > g.N) b->splits_d = g.N;
}

cudaError_t launch_backward(const Geometry& g, const BwdGeom& b, int64_t n, const uint2* plist, const uint32_t* prow,
                            const float* dout, const float* wpack, float* ws, float* dw, float* dbias, float* dz,
                            cudaStream_t st) {
    using namespace bwd;
    if (!b.supported) return cudaErrorNotSupported;
    Args a;
    a.plist = plist; a.prow = prow; a.dout = dout; a.wpack = wpack; a.ws = ws; a.dz = dz;
    a.n = (int)n; a.C = (int)g.C; a.H = (int)g.H; a.W = (int)g.W; a.K = (int)g.K; a.Cg = (int)g.Cg;
    a.Kg = (int)g.Kg; a.Ho = (int)g.Ho; a.Wo = (int)g.Wo; a.T = (int)g.T; a.P = (int)g.P;
    a.kbw = (int)g.kbw; a.fkblocks = (int)g.kblocks;
    a.wmagic = (uint32_t)((1ull << 32) / (uint64_t)g.W + 1);
    a.KC = (int)b.kc; a.kchunks = (int)b.kchunks; a.cblocks = (int)b.cblocks; a.BY = (int)b.by;
    a.bands = (int)b.bands;
    a.bulk = b.bulk ? 1 : 0;
    a.tile_floats = (int)b.tile_floats;
    cudaError_t e = cudaSuccess;
    auto run = [&](bool wgrad) -> cudaError_t {
        const int64_t per = g.G * b.cblocks * (wgrad ? b.kchunks : 1);
        a.splits = (int)pick_splits(per, n, wgrad ? b.splits_w : b.splits_d);
        a.ipc = (int)((n + a.splits - 1) / a.splits);
        const int G = (int)g.G;
        if (g.R == 1) {
            if (b.kl == 1) return launch_rs<1, 1, 1>(a, G, wgrad, b.smem, st);
            if (b.kl == 2) return launch_rs<1, 1, 2>(a, G, wgrad, b.smem, st);
            return launch_rs<1, 1, 4>(a, G, wgrad, b.smem, st);
        }
        if (g.R == 3) {
            if (b.kl == 1) return launch_rs<3, 3, 1>(a, G, wgrad, b.smem, st);
            if (b.kl == 2) return launch_rs<3, 3, 2>(a, G, wgrad, b.smem, st);
            return launch_rs<3, 3, 4>(a, G, wgrad, b.smem, st);
        }
        if (b.kl == 1) return launch_rs<5, 5, 1>(a, G, wgrad, b.smem, st);
        return launch_rs<5, 5, 2>(a, G, wgrad, b.smem, st);
    };
    if (dw) {
        if ((e = run(true)) != cudaSuccess) return e;
        const int64_t count = g.K * g.Cg * g.R * g.S;
        bwd_reduce_kernel<<<148 * 4, 256, 0, st>>>(ws, a.splits, count, dw);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (dbias) {
        bwd_dbias_kernel<<<(unsigned)g.K, 256, 0, st>>>(dout, (int)n, (int)g.K, (int)(g.Ho * g.Wo), dbias);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (dz) {
        if ((e = run(false)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace sc
