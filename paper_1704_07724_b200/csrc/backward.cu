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
// Kernel structure (bwd_kernel<R,S,KL,T,WGRAD>): one CTA = 16 warps + a producer
// warp; warp w owns one input channel; lane l covers the KL consecutive output
// channels k = kc*KC + KL*l + q (q < KL) of a KC = 32*KL chunk.  dout is first
// rewritten once (bwd_transpose_kernel) as doutT[n][g][kc][pixel][KC], so a band of
// BY output rows of one (image, chunk) is one contiguous run, moved into shared
// memory by bulk copies (two buffers on mbarriers, or one when every CTA has a
// single tile), and a lane's KL filters of one pixel are one 32/64/128-bit load.
// Per nonzero (v, i, j) of the warp's plane whose taps reach the band, per tap
// (r, t) with y = (i+P-r)/T, x = (j+P-t)/T integral and in the band (two bit masks
// per nonzero, R + S bits): one vector load d[0..KL) and
//   wgrad: acc[r][t][q] += v * d[q]           (FFMA2 on filter pairs, registers across all tiles)
//   dgrad: part_r += W[r][t][q] * d[q]        (FFMA2, W in registers per (c, kc), one chain per r)
// then (dgrad) the lane partials of 16 nonzeros are summed through a small shared
// transpose buffer (one lane per nonzero, lanes in order) into the warp's dz plane.
// The branch per tap is warp-uniform (all lanes share the nonzero).
// wgrad: grid (split of images, cblock, kc, group); partial dW per split into
// a workspace, summed in split order by bwd_reduce_kernel (deterministic).
// dgrad: grid (split of images, cblock, group); tiles walk (kc, n, band); per
// (n, kc) the warp accumulates its channel's plane in shared memory and then
// stores it (kc = 0) or adds it (kc > 0, in k-chunk order) to dz; with one chunk and
// one band ("direct") the sums go straight to dz.
#include <cuda_runtime.h>

#include "sc_internal.h"

namespace sc {
namespace bwd {

constexpr int kWarps = 16;               // compute warps (one input channel each)
constexpr int kThreads = kWarps * 32;
constexpr int kBlock = kThreads + 32;    // + one producer warp (TMA issue of the dout bands)
constexpr int kRed = 32 * 17;            // dgrad reduction buffer per warp (floats): 32 lanes x 16 slots, odd stride

struct Args {
    const uint2* plist;     // [N*C][H*W] (bits, i*W + j), row-major order
    const uint32_t* prow;   // [N*C][H+1] nonzeros before row r
    const float* doutT;     // [N][G][kchunks][Ho*Wo][KC]: dout with the chunk's filters contiguous (0 past Kg)
    const float* wpack;     // forward packed weights [G][kblocks][Cg][R][S][kbw]
    float* ws;              // wgrad partials [splits][K][Cg][R][S]
    float* dz;              // [N][C][H][W]
    int n, C, H, W, K, Cg, Kg, Ho, Wo, T, P, G;
    int kbw, fkblocks;      // forward weight packing
    uint32_t wmagic;        // floor(2^32 / W) + 1: i = umulhi(i*W + j, wmagic) for i*W + j < 2^32 / W
    int KC, kchunks, cblocks, BY, bands, splits, ipc;  // ipc: images per split
    int buf_floats;         // one band buffer: BY*Wo*KC floats (two, double buffered)
    int direct;             // dgrad with one k-chunk and one band: sums stored straight to dz
    int nbuf;               // band buffers: 2 (double buffered), 1 when every CTA has a single tile
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
// A bulk copy of `bytes` (multiple of 16, 16-byte aligned ends) completing on `bar` (whose
// expected transaction count the caller has raised).
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// doutT[n][g][kc][p][kk] = dout[n][g*Kg + kc*KC + kk][p] (0 for kc*KC + kk >= Kg).  One CTA per
// (32-pixel block, chunk, group, image): coalesced reads along pixels, writes along filters,
// through a [KC][33] shared tile (both sides conflict-free).
template <int KC>
__global__ void __launch_bounds__(256) bwd_transpose_kernel(const float* __restrict__ dout, float* __restrict__ doutT,
                                                            int K, int Kg, int G, int kchunks, int HoWo) {
    __shared__ float t[KC][33];
    int b = blockIdx.x;
    const int pblocks = (HoWo + 31) >> 5;
    const int pb = b % pblocks;
    b /= pblocks;
    const int kc = b % kchunks;
    b /= kchunks;
    const int g = b % G, img = b / G;
    const int p0 = pb * 32, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float* src = dout + ((int64_t)img * K + (int64_t)g * Kg + (int64_t)kc * KC) * HoWo + p0;
    const int kvalid = Kg - kc * KC;
    for (int kk = warp; kk < KC; kk += 8)
        t[kk][lane] = (kk < kvalid && p0 + lane < HoWo) ? __ldg(src + (int64_t)kk * HoWo + lane) : 0.f;
    __syncthreads();
    float* dst = doutT + ((((int64_t)img * G + g) * kchunks + kc) * HoWo + p0) * KC;
    const int np = min(32, HoWo - p0);
    for (int e = threadIdx.x; e < np * KC; e += 256) dst[e] = t[e % KC][e / KC];
}

// The lane's KL consecutive filters of one pixel: one 32/64/128-bit shared load (zeros when !ok).
template <int KL>
__device__ __forceinline__ void load_k(const float* src, bool ok, float (&d)[KL]) {
    if constexpr (KL == 4) {
        const float4 v = ok ? *reinterpret_cast<const float4*>(src) : make_float4(0.f, 0.f, 0.f, 0.f);
        d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    } else if constexpr (KL == 2) {
        const float2 v = ok ? *reinterpret_cast<const float2*>(src) : make_float2(0.f, 0.f);
        d[0] = v.x; d[1] = v.y;
    } else {
        d[0] = ok ? *src : 0.f;
    }
}

template <int R, int S, int KL, int T, bool WGRAD>
__global__ void __launch_bounds__(kBlock, 1) bwd_kernel(const Args a) {
    extern __shared__ __align__(16) float smem[];
    constexpr int KC = 32 * KL;
    static_assert(KL == 1 || KL == 2 || KL == 4, "KL");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int HoWo = a.Ho * a.Wo;
    // dgrad only: the dz planes (none in direct mode: one k-chunk and one band, every nonzero's
    // sum is final and goes straight to dz) and the reduction buffers follow the band buffers
    const int planes = a.direct ? 0 : kWarps * a.H * a.W;
    float* dzbuf = smem + a.nbuf * a.buf_floats + warp * a.H * a.W;  // dgrad: this warp's dz plane of the current image
    // dgrad: lane partials of up to 16 nonzeros, red[lane*17 + slot], summed per nonzero by one lane
    float* red = smem + a.nbuf * a.buf_floats + planes + warp * kRed;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.nbuf * a.buf_floats + (WGRAD ? 0 : planes + kWarps * kRed) + 2);
    full = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(full) + 15) & ~(uintptr_t)15);
    uint64_t* empty = full + 2;  // buffer b released by all compute warps
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

    // lane l covers filters kc*KC + KL*l + q (q < KL): pairs (q, q+1) are f32x2 operands
    float acc[R * S][KL];
    float wr[R * S][KL];
#pragma unroll
    for (int u = 0; u < R * S; ++u)
#pragma unroll
        for (int q = 0; q < KL; ++q) acc[u][q] = 0.f;
    int wr_kc = -1;

    // tile `it` = dout band (image n, chunk kc, rows [band*BY, +BY)), one contiguous run of doutT;
    // order: wgrad (image, band); dgrad (k-chunk, image, band) -- k-chunk major, so a warp
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
                const int bf = it % a.nbuf;
                if (it >= a.nbuf) mbar_wait(empty + bf, (unsigned)((it / a.nbuf - 1) & 1));
                int n, kc, band;
                decode(it, n, kc, band);
                const int y0 = band * a.BY, rows = min(a.BY, a.Ho - y0);
                const float* src =
                    a.doutT + ((((int64_t)n * a.G + g) * a.kchunks + kc) * HoWo + (int64_t)y0 * a.Wo) * KC;
                // the band in eight bulk copies (more requests in flight than one long copy)
                const unsigned bytes = (unsigned)(rows * a.Wo * KC * 4);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + bf)),
                             "r"(bytes)
                             : "memory");
                const unsigned part = ((bytes / 8u) + 15u) & ~15u;
                for (unsigned off = 0; off < bytes; off += part)
                    bulk_copy(reinterpret_cast<char*>(smem + bf * a.buf_floats) + off,
                              reinterpret_cast<const char*>(src) + off, bytes - off < part ? bytes - off : part,
                              full + bf);
            }
        return;
    }
    // per-tile list metadata (the plane's entry range over the band's input rows and its first 32
    // entries) is loaded one tile ahead, so the global-load latency overlaps the previous tile
    auto rows_of = [&](int band, int& ilo, int& ihi) {
        const int y0 = band * a.BY, y1 = min(a.Ho, y0 + a.BY);
        ilo = max(0, y0 * T - a.P);
        ihi = min(a.H - 1, (y1 - 1) * T - a.P + R - 1);
    };
    uint32_t pe0 = 0, pe1 = 0;
    uint2 pm = make_uint2(0u, 0u);
    auto fetch = [&](int it) {
        int n, kc, band, ilo, ihi;
        decode(it, n, kc, band);
        rows_of(band, ilo, ihi);
        const int64_t plane = (int64_t)n * a.C + c;
        if (ilo <= ihi) {
            const uint32_t* pr = a.prow + plane * (a.H + 1);
            pe0 = __ldg(pr + ilo);
            pe1 = __ldg(pr + ihi + 1);
            // entries 0..31 of the plane (prow[plane][0] == 0): the first batch when ilo == 0
            if (ilo == 0 && lane < HW) pm = __ldg(a.plist + plane * HW + lane);
        } else {
            pe0 = pe1 = 0;
        }
    };
    if (active && ntiles > 0) fetch(0);
    for (int it = 0; it < ntiles; ++it) {
        int n, kc, band;
        decode(it, n, kc, band);
        const int y0 = band * a.BY, y1 = min(a.Ho, y0 + a.BY);
        const int bf = it % a.nbuf;
        const float* tile = smem + bf * a.buf_floats;  // [pixel of the band][KC]
        const uint32_t ce0 = pe0, ce1 = pe1;
        const uint2 cm = pm;
        if (active && it + 1 < ntiles) fetch(it + 1);
        if (it >= 1) {  // done with tile it-1: the producer may refill its buffer
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + ((it - 1) % a.nbuf));
        }
        mbar_wait(full + bf, (unsigned)((it / a.nbuf) & 1));
        if (!active) continue;
        const int64_t plane = (int64_t)n * a.C + c;
        if constexpr (!WGRAD) {
            if (a.direct) {  // zeros where the input is zero; the nonzeros' sums overwrite the rest
                float* dzp = a.dz + plane * HW;
                for (int e = lane; e < HW; e += 32) dzp[e] = 0.f;
                __syncwarp();
            } else if (band == 0) {  // first band of (image, k-chunk): this chunk's partial plane starts at zero
                for (int e = lane; e < HW; e += 32) dzbuf[e] = 0.f;
                __syncwarp();
            }
            if (kc != wr_kc) {  // W[k][cl][r][t] for this lane's k, from the forward packing
                wr_kc = kc;
#pragma unroll
                for (int q = 0; q < KL; ++q) {
                    const int kl = kc * KC + KL * lane + q;
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
        // dgrad, last band of a later k-chunk: the plane's earlier partial sums, loaded now (added at
        // the end of the tile); planes of <= 256 elements only
        float dzp_pre[8];
        if constexpr (!WGRAD) {
            if (band == a.bands - 1 && kc > 0 && HW <= 256) {
                const float* dzp = a.dz + plane * HW;
#pragma unroll
                for (int m = 0; m < 8; ++m) dzp_pre[m] = lane + 32 * m < HW ? dzp[lane + 32 * m] : 0.f;
            }
        }
        // input rows whose taps reach output rows [y0, y1)
        int ilo, ihi;
        rows_of(band, ilo, ihi);
        if (ilo <= ihi) {
        const uint32_t e0 = ce0, e1 = ce1;
        const uint2* lst = a.plist + plane * HW;
        // entries e0+32m+lane, fetched 32 at a time (one coalesced load; the first batch prefetched
        // when e0 == 0); lanes past e1 hold entries that are never read
        uint2 mine = cm;
        for (uint32_t e = e0; e < e1; ++e) {
            const uint32_t sl = (e - e0) & 31u;
            if (sl == 0 && (e != 0 || ilo != 0)) {
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
            // lane reads filters KL*lane.. at tile[pixel*KC + KL*lane]; T == 1: tap (r, t) is pixel
            // (ip - y0 - r)*Wo + (jp - t)
            const float* abase = tile + ((ip - y0) * a.Wo + jp) * KC + KL * lane;
            // dgrad partials: one chain per filter row (a single accumulator would make the
            // R*S*KL/2 FMAs of a nonzero one dependent chain)
            float2 part2[R];
            float part1[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                part2[r] = make_float2(0.f, 0.f);
                part1[r] = 0.f;
            }
            const float2 vv = make_float2(v, v);
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
                            src = abase - (r * a.Wo + t) * KC;
                        else
                            src = tile + (((ip - r) / T - y0) * a.Wo + (jp - t) / T) * KC + KL * lane;
                        float d[KL];
                        load_k<KL>(src, ok, d);
                        const int u = r * S + t;
                        if constexpr (KL == 1) {
                            if constexpr (WGRAD)
                                acc[u][0] = fmaf(v, d[0], acc[u][0]);
                            else
                                part1[r] = fmaf(wr[u][0], d[0], part1[r]);
                        } else {
#pragma unroll
                            for (int q = 0; q < KL; q += 2) {
                                const float2 dd = make_float2(d[q], d[q + 1]);
                                if constexpr (WGRAD) {
                                    const float2 o = __ffma2_rn(dd, vv, make_float2(acc[u][q], acc[u][q + 1]));
                                    acc[u][q] = o.x;
                                    acc[u][q + 1] = o.y;
                                } else {
                                    part2[r] = __ffma2_rn(make_float2(wr[u][q], wr[u][q + 1]), dd, part2[r]);
                                }
                            }
                        }
                    }
                }
            };
            if (T == 1 && rmask == (1u << R) - 1u && tmask == (1u << S) - 1u)
                taps(bool_const<true>{});
            else
                taps(bool_const<false>{});
            if constexpr (!WGRAD) {
                // sum over the lanes (filters) without a shuffle chain per nonzero: 16 nonzeros'
                // lane partials go to red[lane][slot]; then lane q sums slot q's column (32 rows, in
                // lane order) and adds it to dz at that nonzero's position
                const uint32_t slot = (e - e0) & 15u;
                float part = 0.f;
#pragma unroll
                for (int r = 0; r < R; ++r) part += KL == 1 ? part1[r] : part2[r].x + part2[r].y;
                red[lane * 17 + slot] = part;
                if (slot == 15u || e + 1 == e1) {
                    const uint32_t pos = __shfl_sync(0xffffffffu, mine.y, (int)(((e - e0) & 16u) + (lane & 15)));
                    __syncwarp();
                    if ((uint32_t)lane <= slot) {
                        float sum = 0.f;
#pragma unroll 8
                        for (int r = 0; r < 32; ++r) sum += red[r * 17 + lane];
                        if (a.direct)
                            a.dz[plane * HW + pos] = sum;
                        else
                            dzbuf[pos] += sum;
                    }
                    __syncwarp();
                }
            }
        }
        }
        if constexpr (!WGRAD) {
            if (!a.direct && band == a.bands - 1) {  // last band: store (first k-chunk) or add (later ones, in order)
                __syncwarp();
                float* dzp = a.dz + plane * HW;
                if (kc == 0) {
                    for (int e = lane; e < HW; e += 32) dzp[e] = dzbuf[e];
                } else if (HW <= 256) {
#pragma unroll
                    for (int m = 0; m < 8; ++m)
                        if (lane + 32 * m < HW) dzp[lane + 32 * m] = dzp_pre[m] + dzbuf[lane + 32 * m];
                } else {
                    for (int e = lane; e < HW; e += 32) dzp[e] += dzbuf[e];
                }
            }
        }
    }
    if constexpr (WGRAD) {
        if (active) {
#pragma unroll
            for (int q = 0; q < KL; ++q) {
                const int kl = kc_fixed * KC + KL * lane + q;
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
    b->kl = kl;
    b->kc = 32 * kl;
    b->kchunks = (g.Kg + b->kc - 1) / b->kc;
    b->cblocks = (g.Cg + bwd::kWarps - 1) / bwd::kWarps;
    // two band buffers of by output rows x kc filters within 220 KB; dgrad (index 1) less its
    // dz planes and reduction buffers (16 x (H*W + kRed) floats)
    // image splits (below) reach one image per CTA when the grid has <= 2 waves per image split;
    // then each CTA has a single tile per k-chunk and band, and one buffer suffices
    const int64_t cb16 = (g.Cg + bwd::kWarps - 1) / bwd::kWarps;
    for (int d = 0; d < 2; ++d) {
        const bool one_img = g.G * cb16 * (d ? 1 : b->kchunks) * g.N <= 296;
        const bool one_tile = one_img && (d == 0 || b->kchunks == 1);
        const int64_t plane_bytes = g.Ho * g.Wo * b->kc * 4;
        b->nbuf[d] = one_tile ? 1 : 2;
        // dgrad with one k-chunk: no dz planes if the whole plane then fits one band ("direct")
        b->direct = d == 1 && b->kchunks == 1 &&
                    b->nbuf[1] * plane_bytes <= 220 * 1024 - 64 - bwd::kWarps * bwd::kRed * 4;
        const int64_t extra = d ? (int64_t)bwd::kWarps * ((b->direct ? 0 : g.H * g.W) + bwd::kRed) * 4 : 0;
        const int64_t budget = 220 * 1024 - 64 - extra;
        int64_t by = g.Ho;
        while (by > 1 && b->nbuf[d] * by * g.Wo * b->kc * 4 > budget) --by;
        b->by[d] = by;
        b->bands[d] = (g.Ho + by - 1) / by;
        if (b->bands[d] > 1) b->nbuf[d] = 2;  // several tiles per CTA: double buffer (re-fit)
        while (by > 1 && b->nbuf[d] * by * g.Wo * b->kc * 4 > budget) --by;
        b->by[d] = by;
        b->bands[d] = (g.Ho + by - 1) / by;
        b->buf_floats[d] = by * g.Wo * b->kc;
        b->smem[d] = (size_t)(b->nbuf[d] * b->buf_floats[d]) * sizeof(float) + (size_t)(extra + 64);
        if (b->smem[d] > 227 * 1024) {
            b->supported = false;
            return;
        }
    }
    b->doutT_floats = g.N * g.G * b->kchunks * g.Ho * g.Wo * b->kc;
    // at most about two waves of 1-CTA-per-SM blocks (bounds the wgrad workspace)
    const int64_t per_split_w = g.G * b->cblocks * b->kchunks;
    b->splits_w = (296 + per_split_w - 1) / per_split_w;
    if (b->splits_w > g.N) b->splits_w = g.N;
    const int64_t per_split_d = g.G * b->cblocks;
    b->splits_d = (296 + per_split_d - 1) / per_split_d;
    if (b->splits_d > g.N) b->splits_d = g.N;
}

cudaError_t launch_backward(const Geometry& g, const BwdGeom& b, int64_t n, const uint2* plist, const uint32_t* prow,
                            const float* dout, const float* wpack, float* ws, float* doutT, float* dw, float* dbias,
                            float* dz, cudaStream_t st, cudaStream_t st2, cudaEvent_t ev_fork, cudaEvent_t ev_join) {
    using namespace bwd;
    if (!b.supported) return cudaErrorNotSupported;
    Args a;
    a.plist = plist; a.prow = prow; a.doutT = doutT; a.wpack = wpack; a.ws = ws; a.dz = dz;
    a.n = (int)n; a.C = (int)g.C; a.H = (int)g.H; a.W = (int)g.W; a.K = (int)g.K; a.Cg = (int)g.Cg;
    a.Kg = (int)g.Kg; a.Ho = (int)g.Ho; a.Wo = (int)g.Wo; a.T = (int)g.T; a.P = (int)g.P; a.G = (int)g.G;
    a.kbw = (int)g.kbw; a.fkblocks = (int)g.kblocks;
    a.wmagic = (uint32_t)((1ull << 32) / (uint64_t)g.W + 1);
    a.KC = (int)b.kc; a.kchunks = (int)b.kchunks; a.cblocks = (int)b.cblocks;
    cudaError_t e = cudaSuccess;
    if (dw || dz) {  // dout with each chunk's filters contiguous per pixel (vector loads per tap)
        const int howo = (int)(g.Ho * g.Wo);
        const int64_t grid = (int64_t)((howo + 31) / 32) * b.kchunks * g.G * n;
        if (b.kc == 128)
            bwd_transpose_kernel<128><<<(unsigned)grid, 256, 0, st>>>(dout, doutT, (int)g.K, (int)g.Kg, (int)g.G,
                                                                     (int)b.kchunks, howo);
        else if (b.kc == 64)
            bwd_transpose_kernel<64><<<(unsigned)grid, 256, 0, st>>>(dout, doutT, (int)g.K, (int)g.Kg, (int)g.G,
                                                                    (int)b.kchunks, howo);
        else
            bwd_transpose_kernel<32><<<(unsigned)grid, 256, 0, st>>>(dout, doutT, (int)g.K, (int)g.Kg, (int)g.G,
                                                                    (int)b.kchunks, howo);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    auto run = [&](bool wgrad, cudaStream_t rs) -> cudaError_t {
        const int d = wgrad ? 0 : 1;
        a.BY = (int)b.by[d];
        a.bands = (int)b.bands[d];
        a.buf_floats = (int)b.buf_floats[d];
        a.direct = (!wgrad && b.direct) ? 1 : 0;
        a.nbuf = (int)b.nbuf[d];
        const size_t smem = b.smem[d];
        const int64_t per = g.G * b.cblocks * (wgrad ? b.kchunks : 1);
        a.splits = (int)pick_splits(per, n, wgrad ? b.splits_w : b.splits_d);
        a.ipc = (int)((n + a.splits - 1) / a.splits);
        const int G = (int)g.G;
        if (g.R == 1) {
            if (b.kl == 1) return launch_rs<1, 1, 1>(a, G, wgrad, smem, rs);
            if (b.kl == 2) return launch_rs<1, 1, 2>(a, G, wgrad, smem, rs);
            return launch_rs<1, 1, 4>(a, G, wgrad, smem, rs);
        }
        if (g.R == 3) {
            if (b.kl == 1) return launch_rs<3, 3, 1>(a, G, wgrad, smem, rs);
            if (b.kl == 2) return launch_rs<3, 3, 2>(a, G, wgrad, smem, rs);
            return launch_rs<3, 3, 4>(a, G, wgrad, smem, rs);
        }
        if (b.kl == 1) return launch_rs<5, 5, 1>(a, G, wgrad, smem, rs);
        return launch_rs<5, 5, 2>(a, G, wgrad, smem, rs);
    };
    // dgrad and dbias are independent of wgrad: with a second stream they run beside it (each
    // kernel's last wave overlaps the other's), joined back into st at the end
    const bool two = st2 && ev_fork && ev_join && dw && (dz || dbias);
    cudaStream_t sd = two ? st2 : st;
    if (two && ((e = cudaEventRecord(ev_fork, st)) != cudaSuccess || (e = cudaStreamWaitEvent(st2, ev_fork, 0)) != cudaSuccess))
        return e;
    if (dz) {  // run() fills the launch-specific fields of `a`; the launch copies them
        if ((e = run(false, sd)) != cudaSuccess) return e;
    }
    if (dw) {
        if ((e = run(true, st)) != cudaSuccess) return e;
        const int64_t count = g.K * g.Cg * g.R * g.S;
        bwd_reduce_kernel<<<148 * 4, 256, 0, st>>>(ws, a.splits, count, dw);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (dbias) {
        bwd_dbias_kernel<<<(unsigned)g.K, 256, 0, sd>>>(dout, (int)n, (int)g.K, (int)(g.Ho * g.Wo), dbias);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (two && ((e = cudaEventRecord(ev_join, st2)) != cudaSuccess || (e = cudaStreamWaitEvent(st, ev_join, 0)) != cudaSuccess))
        return e;
    return cudaSuccess;
}

}  // namespace sc
