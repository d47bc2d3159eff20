// Stage 2, shape-specialised: output-stationary sparse-gather convolution
// with the output tile in registers.
//
// Computes, for stride 1 (ISC steps 2-3; Eq. 1 P:68-72 with the
// zero terms skipped):
//   out[n,k,y,x] = bias[k] + sum_{c in group, nonzero in[n,c,i,j]} in * W[k,c,i+P-y,j+P-x]
//
// Mapping:
//  * CTA = 8 warps sharing one (group g, 32-output-channel block kb).  The
//    packed weight slice wpack[g][kb][c0:c0+CH][R][S][32] of CH input channels
//    is ONE contiguous run and is streamed through a STAGES-deep shared-memory
//    ring by 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx);
//    warp 0 lane 0 refills a stage once all 8 warps released it (empty
//    mbarrier, 8 arrivals).
//  * warp = one unit (image n, output rows [y0, y0+TY)); lane = output channel
//    k = 32*kb + lane ("4 floats of weights ... at one time", becomes
//    32 lanes).  The warp's tile acc[TY][NP] (pairs of adjacent x) lives in
//    registers for the whole reduction over input channels.
//  * per input channel: the lane's R*S weights come from shared memory (one
//    conflict-free LDS per tap) and are arranged as pairs (W[r][u], W[r][u-1]);
//    the channel's nonzero lists (stage-1 output, warp-uniform) are staged 32
//    entries at a time into a per-warp shared buffer, keeping only entries
//    inside the tile's input window, then each entry is one indirect branch
//    (switch -> BRX) into generated code that applies FFMA2 to exactly the
//    accumulators the entry reaches (tools/gen_gather.py).
//  * epilogue (ISC step 3, "transpose temporary results"): registers ->
//    per-warp shared buffer [k][x] -> contiguous NCHW row runs, + bias, optional
//    ReLU (Eq. 2).  One global write per output, no atomics; accumulation order
//    (channel, entry) is fixed, so results are deterministic.
#pragma once
#include "sc_internal.h"

namespace sc {
namespace fast {

#include "gather_variants.inc"

constexpr int NW = 8;          // warps per CTA
constexpr int kLookahead = 2;  // list segments whose first 32 entries are prefetched

struct Args {
    const float* values;
    const void* idx;
    const uint32_t* counts;
    const float* wpack;
    const float* bias;
    float* out;
    int n, C, H, K, Cg, Kg, kblocks, Ho, th, tiles, cap, relu;
    int ytiles, units, ctas_per_kb;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <class V>
struct Smem {
    static constexpr int kStageFloats = V::CH * V::R * V::S * 32;
    static constexpr int kER = (96 / V::WO) > 0 ? (96 / V::WO < V::TY ? 96 / V::WO : V::TY) : 1;  // epilogue rows
    static constexpr int kEpiStride = (kER * V::WO) | 1;                                        // odd: no conflicts
    static constexpr size_t ring = sizeof(float) * V::STAGES * kStageFloats;
    static constexpr size_t bars = 16 * V::STAGES;
    static constexpr size_t ent = sizeof(uint2) * NW * 32;
    static constexpr size_t epi = sizeof(float) * NW * 32 * kEpiStride;
    static constexpr size_t total = ring + bars + ent + epi;
};

template <class V, typename IdxT>
__global__ void __launch_bounds__(NW * 32, 1) gather_fast_kernel(const Args a) {
    using SM = Smem<V>;
    constexpr int R = V::R, S = V::S, RS = R * S, TY = V::TY, NP = V::NP, WO = V::WO, W = V::W;
    constexpr int CH = V::CH, STAGES = V::STAGES;
    extern __shared__ __align__(128) unsigned char smem[];
    float* ring = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::ring);
    uint64_t* empty = full + STAGES;
    uint2* ent_all = reinterpret_cast<uint2*>(smem + SM::ring + SM::bars);
    float* epi_all = reinterpret_cast<float*>(smem + SM::ring + SM::bars + SM::ent);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cb = blockIdx.x % a.ctas_per_kb;
    const int gkb = blockIdx.x / a.ctas_per_kb;  // g * kblocks + kb
    const int kb = gkb % a.kblocks, g = gkb / a.kblocks;
    const int unit = cb * NW + warp;
    const bool active = unit < a.units;
    const int n = active ? unit / a.ytiles : 0;
    const int y0 = active ? (unit % a.ytiles) * TY : 0;
    const int nchunks = (a.Cg + CH - 1) / CH;
    const float* wsrc = a.wpack + (size_t)gkb * a.Cg * RS * 32;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q < STAGES && q < nchunks; ++q) {
            const int chs = (a.Cg - q * CH) < CH ? (a.Cg - q * CH) : CH;
            const unsigned bytes = (unsigned)(chs * RS * 32 * sizeof(float));
            mbar_expect_tx(&full[q], bytes);
            tma_bulk_g2s(ring + q * SM::kStageFloats, wsrc + (size_t)q * CH * RS * 32, bytes, &full[q]);
        }
    }

    // Lists overlapping the input window rows [y0 - P, y0 + TY - 1 + R - 1 - P].
    int i_lo = y0 - V::P, i_hi = y0 + TY + R - 2 - V::P;
    i_lo = i_lo < 0 ? 0 : i_lo;
    i_hi = i_hi > a.H - 1 ? a.H - 1 : i_hi;
    const int tl_lo = i_lo / a.th, nl = i_hi / a.th - tl_lo + 1;  // lists per channel (1..3)

    // f32x2 accumulators as 64-bit patterns: x (= output column 2m) in the low word
    unsigned long long acc[TY][NP];
#pragma unroll
    for (int ty = 0; ty < TY; ++ty)
#pragma unroll
        for (int m = 0; m < NP; ++m) acc[ty][m] = 0ull;

    uint2* ent = ent_all + warp * 32;
    const float* vbase = a.values;
    const IdxT* ibase = reinterpret_cast<const IdxT*>(a.idx);

    // Segment = (channel cl, list tl_lo + l); global order s = cl * nl + l.
    const int nseg = a.Cg * nl;
    auto seg_list = [&](int s) -> int {
        const int cl = s / nl, l = s - cl * nl;
        return (n * a.C + g * a.Cg + cl) * a.tiles + tl_lo + l;
    };
    // prefetch ring: counts and first 32 entries of segments s .. s+kLookahead
    uint32_t pc[kLookahead + 1];
    float pv[kLookahead + 1];
    int pi[kLookahead + 1];
    auto issue = [&](int s, int slot) {
        if (active && s < nseg) {
            const int list = seg_list(s);
            const uint32_t cnt = __ldg(&a.counts[list]);
            pc[slot] = cnt;
            pv[slot] = (lane < (int)cnt) ? __ldg(&vbase[(size_t)list * a.cap + lane]) : 0.f;
            pi[slot] = (lane < (int)cnt) ? (int)__ldg(&ibase[(size_t)list * a.cap + lane]) : 0;
        } else {
            pc[slot] = 0;
            pv[slot] = 0.f;
            pi[slot] = 0;
        }
    };
#pragma unroll
    for (int d = 0; d <= kLookahead; ++d) issue(d, d);

    int s = 0;  // next segment to process
#pragma unroll 1
    for (int ch = 0; ch < nchunks; ++ch) {
        const int st = ch % STAGES;
        mbar_wait(&full[st], (ch / STAGES) & 1);
        const float* wst = ring + st * SM::kStageFloats;
        const int cc_n = (a.Cg - ch * CH) < CH ? (a.Cg - ch * CH) : CH;
        if (active) {
#pragma unroll 1
            for (int cc = 0; cc < cc_n; ++cc) {
                // wp[r][u] = (W[r][u], W[r][u-1]) with W[r][-1] = W[r][S] = 0
                unsigned long long wp[R][S + 1];
                {
                    unsigned w[R][S];
#pragma unroll
                    for (int r = 0; r < R; ++r)
#pragma unroll
                        for (int t = 0; t < S; ++t) w[r][t] = __float_as_uint(wst[(cc * RS + r * S + t) * 32 + lane]);
#pragma unroll
                    for (int r = 0; r < R; ++r)
#pragma unroll
                        for (int u = 0; u <= S; ++u)
                            wp[r][u] = (u < S ? (unsigned long long)w[r][u] : 0ull) |
                                       ((u >= 1 ? (unsigned long long)w[r][u - 1] : 0ull) << 32);
                }
#pragma unroll 1
                for (int l = 0; l < nl; ++l, ++s) {
                    // rotate the prefetch ring: slot 0 is segment s
                    const uint32_t cnt = pc[0];
                    float v0 = pv[0];
                    int i0 = pi[0];
#pragma unroll
                    for (int d = 0; d < kLookahead; ++d) {
                        pc[d] = pc[d + 1];
                        pv[d] = pv[d + 1];
                        pi[d] = pi[d + 1];
                    }
                    issue(s + kLookahead + 1, kLookahead);
                    const int list = seg_list(s);
                    const int off = ((tl_lo + l) * a.th - (y0 - V::P)) * W;
#pragma unroll 1
                    for (uint32_t e0 = 0; e0 < cnt; e0 += 32) {
                        if (e0 > 0) {  // long list (dense input): synchronous loads
                            const bool ok = e0 + lane < cnt;
                            v0 = ok ? vbase[(size_t)list * a.cap + e0 + lane] : 0.f;
                            i0 = ok ? (int)ibase[(size_t)list * a.cap + e0 + lane] : 0;
                        }
                        const int cs = i0 + off;
                        const bool inwin = (e0 + lane < cnt) && cs >= 0 && cs < V::NCASES;
                        const unsigned bal = __ballot_sync(0xffffffffu, inwin);
                        const int rank = __popc(bal & ((1u << lane) - 1u));
                        if (inwin) ent[rank] = make_uint2(__float_as_uint(v0), (unsigned)cs);
                        __syncwarp();
                        const int nin = __popc(bal);
                        uint2 nxt = ent[0];  // software-pipelined: next entry loads during this case
#pragma unroll 1
                        for (int e = 0; e < nin; ++e) {
                            const uint2 t = nxt;
                            nxt = ent[(e + 1) & 31];
                            V::apply(acc, wp, __uint_as_float(t.x), (int)t.y);
                        }
                        __syncwarp();
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (threadIdx.x == 0 && ch >= 1) {
            const int q = ch - 1 + STAGES;
            if (q < nchunks) {
                const int qs = (ch - 1) % STAGES;
                mbar_wait(&empty[qs], ((ch - 1) / STAGES) & 1);
                const int chs = (a.Cg - q * CH) < CH ? (a.Cg - q * CH) : CH;
                const unsigned bytes = (unsigned)(chs * RS * 32 * sizeof(float));
                mbar_expect_tx(&full[qs], bytes);
                tma_bulk_g2s(ring + qs * SM::kStageFloats, wsrc + (size_t)q * CH * RS * 32, bytes, &full[qs]);
            }
        }
    }

    if (!active) return;
    // Epilogue: registers -> smem [k][rows*WO] -> contiguous NCHW runs.
    constexpr int ER = SM::kER, ES = SM::kEpiStride;
    float* epi = epi_all + warp * 32 * ES;
    const int kloc = kb * 32;
#pragma unroll
    for (int r0 = 0; r0 < TY; r0 += ER) {
#pragma unroll
        for (int rr = 0; rr < ER; ++rr) {
            if (r0 + rr < TY) {
#pragma unroll
                for (int m = 0; m < NP; ++m) {
                    epi[lane * ES + rr * WO + 2 * m] = __uint_as_float((unsigned)acc[r0 + rr][m]);
                    if (2 * m + 1 < WO)
                        epi[lane * ES + rr * WO + 2 * m + 1] = __uint_as_float((unsigned)(acc[r0 + rr][m] >> 32));
                }
            }
        }
        __syncwarp();
        int rows = TY - r0 < ER ? TY - r0 : ER;
        if (y0 + r0 + rows > a.Ho) rows = a.Ho - (y0 + r0);
        if (rows > 0) {
            const int len = rows * WO;
            for (int kk = 0; kk < 32; ++kk) {
                const int k = kloc + kk;
                if (k >= a.Kg) break;
                const int kglob = g * a.Kg + k;
                const float b = __ldg(&a.bias[kglob]);
                float* dst = a.out + ((size_t)(n * a.K + kglob) * a.Ho + y0 + r0) * WO;
                for (int p = lane; p < len; p += 32) {
                    float o = epi[kk * ES + p] + b;
                    if (a.relu) o = fmaxf(o, 0.f);
                    dst[p] = o;
                }
            }
        }
        __syncwarp();
    }
}

template <class V, typename IdxT>
cudaError_t launch_v(const Geometry& g, int64_t n, const float* values, const void* idx, const uint32_t* counts,
                     const float* wpack, const float* bias, float* out, cudaStream_t st) {
    Args a;
    a.values = values; a.idx = idx; a.counts = counts; a.wpack = wpack; a.bias = bias; a.out = out;
    a.n = (int)n; a.C = (int)g.C; a.H = (int)g.H; a.K = (int)g.K; a.Cg = (int)g.Cg; a.Kg = (int)g.Kg;
    a.kblocks = (int)g.kblocks; a.Ho = (int)g.Ho; a.th = (int)g.th; a.tiles = (int)g.tiles; a.cap = (int)g.cap;
    a.relu = g.relu ? 1 : 0;
    a.ytiles = (int)((g.Ho + V::TY - 1) / V::TY);
    a.units = (int)n * a.ytiles;
    a.ctas_per_kb = (a.units + NW - 1) / NW;
    const size_t smem = Smem<V>::total;
    auto kern = gather_fast_kernel<V, IdxT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = (int64_t)a.ctas_per_kb * g.G * g.kblocks;
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace fast
}  // namespace sc

// Each gather_fast_vN.cu instantiates one variant (parallel compilation: ptxas
// spends minutes on each jump-table kernel).
#define SC_INSTANTIATE_VARIANT(VV)                                                                         \
    namespace sc {                                                                                         \
    namespace fast {                                                                                       \
    cudaError_t launch_##VV(const Geometry& g, int64_t n, const float* values, const void* idx,            \
                            const uint32_t* counts, const float* wpack, const float* bias, float* out,     \
                            cudaStream_t st) {                                                             \
        return launch_v<VV, uint8_t>(g, n, values, idx, counts, wpack, bias, out, st);                    \
    }                                                                                                      \
    }                                                                                                      \
    }
