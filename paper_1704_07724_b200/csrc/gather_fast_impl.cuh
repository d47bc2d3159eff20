// Stage 2, shape-specialised: output-stationary sparse-gather convolution
// with the output tile in registers (template; one .cu per variant).
//
// Computes, for stride 1 (ISC steps 2-3; Eq. 1 P:68-72 with the
// zero terms skipped):
//   out[n,k,y,x] = bias[k] + sum_{c in group, nonzero in[n,c,i,j]} in * W[k,c,i+P-y,j+P-x]
//
// Mapping:
//  * CTA = NW warps sharing one (group g, k-block kb of KBW = 32*KL output
//    channels).  The packed weight slice wpack[g][kb][c0:c0+CH][R][S][KBW] of
//    CH input channels is ONE contiguous run, streamed through a STAGES-deep
//    shared-memory ring by 1-D TMA bulk copies (cp.async.bulk + mbarrier
//    complete_tx); thread 0 refills a stage once all NW warps released it.
//  * warp = one unit (image n, output rows [y0, y0+TY)); lane owns KL output
//    channels (the paper's "4 floats of weights ... at one time", P:123,
//    becomes 32*KL per warp).  The warp's tile acc[TY][NX] (f32x2 pairs) stays
//    in registers for the whole reduction over input channels.
//  * per input channel: the lane's R*S weights come from the ring (conflict-
//    free LDS), the channel's nonzero list (stage-1 output, warp-uniform) is
//    staged 32 entries at a time into a per-warp shared buffer keeping only
//    entries inside the tile's input window; each entry is one indirect,
//    warp-uniform branch (brx.idx.uni) into generated code that applies
//    FFMA2/FFMA to exactly the accumulators the entry reaches
//    (tools/gen_gather.py).
//  * epilogue (ISC step 3, "transpose temporary results"): registers ->
//    per-warp shared buffer [k][pixels] -> contiguous NCHW runs, + bias,
//    optional ReLU (Eq. 2).  One global write per output, no atomics;
//    accumulation order (channel, entry) is fixed -> deterministic.
#pragma once
#include "sc_internal.h"

namespace sc {
namespace fast {

#include "gather_variants.inc"

constexpr int kSegRing = 32;  // list segments in flight per warp (cp.async ring, ~2 chunks)
constexpr int kEntCap = 256;  // entries of the per-warp stream buffer

// One prefetched list segment: count + first 32 values + first 32 u8 indices.
struct __align__(16) SegSlot {
    float v[32];
    uint32_t i4[8];
    uint32_t cnt;
    uint32_t pad[3];
};

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
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <class V>
struct Smem {
    static constexpr int KBW = 32 * V::KL;
    static constexpr int kStageFloats = V::CH * V::R * V::S * KBW;
    // epilogue rows per pass: KBW x (kER*WO) floats per warp ~ 8 KB
    static constexpr int kERraw = (2048 / KBW) / V::WO;
    static constexpr int kER = kERraw < 1 ? 1 : (kERraw > V::TY ? V::TY : kERraw);
    static constexpr int kEpiStride = (kER * V::WO) | 1;                                        // odd
    static constexpr size_t ring = sizeof(float) * V::STAGES * kStageFloats;
    static constexpr size_t bars = 16 * V::STAGES;
    static constexpr size_t ent = sizeof(uint2) * V::NW * kEntCap;
    static constexpr size_t seg = sizeof(SegSlot) * V::NW * kSegRing;
    static constexpr size_t epi = sizeof(float) * V::NW * KBW * kEpiStride;
    static constexpr size_t total = ring + bars + ent + seg + epi;
    static_assert(total <= 227 * 1024, "shared memory budget of one CTA exceeded");
};

template <class V, typename IdxT>
__global__ void __launch_bounds__(V::NW * 32, 1) gather_fast_kernel(const Args a) {
    using SM = Smem<V>;
    constexpr int R = V::R, RS = V::R * V::S, TY = V::TY, NX = V::NX, WO = V::WO, W = V::W;
    constexpr int CH = V::CH, STAGES = V::STAGES, NW = V::NW, KBW = SM::KBW;
    extern __shared__ __align__(128) unsigned char smem[];
    float* ring = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::ring);
    uint64_t* empty = full + STAGES;
    uint2* ent_all = reinterpret_cast<uint2*>(smem + SM::ring + SM::bars);
    SegSlot* seg_all = reinterpret_cast<SegSlot*>(smem + SM::ring + SM::bars + SM::ent);
    float* epi_all = reinterpret_cast<float*>(smem + SM::ring + SM::bars + SM::ent + SM::seg);
    static_assert(sizeof(IdxT) == 1, "register-tile kernels read u8 list indices");

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cb = blockIdx.x % a.ctas_per_kb;
    const int gkb = blockIdx.x / a.ctas_per_kb;  // g * kblocks + kb
    const int kb = gkb % a.kblocks, g = gkb / a.kblocks;
    const int unit = cb * NW + warp;
    const bool active = unit < a.units;
    const int n = active ? unit / a.ytiles : 0;
    const int y0 = active ? (unit % a.ytiles) * TY : 0;
    const int nchunks = (a.Cg + CH - 1) / CH;
    const float* wsrc = a.wpack + (size_t)gkb * a.Cg * RS * KBW;

    // Warps without a unit (last CTA of a k-block) leave right after the
    // barrier set-up; `empty` counts only the active warps of this CTA.
    const int nactive = (a.units - cb * NW) < NW ? (a.units - cb * NW) : NW;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], (unsigned)nactive);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q < STAGES && q < nchunks; ++q) {
            const int chs = (a.Cg - q * CH) < CH ? (a.Cg - q * CH) : CH;
            const unsigned bytes = (unsigned)(chs * RS * KBW * sizeof(float));
            mbar_expect_tx(&full[q], bytes);
            tma_bulk_g2s(ring + q * SM::kStageFloats, wsrc + (size_t)q * CH * RS * KBW, bytes, &full[q]);
        }
    }
    if (!active) return;  // warp 0 is always active (every CTA has >= 1 unit)

    // Lists overlapping the input window rows [y0 - P, y0 + TY - 1 + R - 1 - P].
    int i_lo = y0 - V::P, i_hi = y0 + TY + R - 2 - V::P;
    i_lo = i_lo < 0 ? 0 : i_lo;
    i_hi = i_hi > a.H - 1 ? a.H - 1 : i_hi;
    const int tl_lo = i_lo / a.th, nl = i_hi / a.th - tl_lo + 1;  // lists per channel (1..3)

    unsigned long long acc[TY][NX];  // f32x2 bit patterns, low word = first element
#pragma unroll
    for (int ty = 0; ty < TY; ++ty)
#pragma unroll
        for (int m = 0; m < NX; ++m) acc[ty][m] = 0ull;

    uint2* ent = ent_all + warp * kEntCap;
    const unsigned ent_s = smem_u32(ent);
    const float* vbase = a.values;
    const IdxT* ibase = reinterpret_cast<const IdxT*>(a.idx);
    // list id of channel cl, list l = (n*C + g*Cg + cl)*tiles + tl_lo + l
    const int list0 = (n * a.C + g * a.Cg) * a.tiles + tl_lo;

    // Segment s = (channel s / nl, list s % nl).  A per-warp ring of kSegRing
    // shared-memory slots receives, by cp.async (no registers held while in
    // flight), the count and the first 32 entries of each segment, two weight
    // chunks ahead of use.  The first 32 slots of a list are read regardless
    // of its count (slack is zero-initialised at plan creation and masked).
    const int nseg = a.Cg * nl;
    SegSlot* segring = seg_all + warp * kSegRing;
    const int vlanes = a.cap < 32 ? a.cap : 32;
    auto seg_list = [&](int s) -> int {
        const int cl = nl == 1 ? s : s / nl;
        return list0 + cl * a.tiles + (s - cl * nl);
    };
    auto issue = [&](int s) {
        if (active && s < nseg) {
            SegSlot* sl = segring + (s % kSegRing);
            const size_t list = (size_t)seg_list(s);
            if (lane < vlanes) cp_async4(&sl->v[lane], vbase + list * a.cap + lane);
            if (lane < (vlanes + 3) / 4)
                cp_async4(&sl->i4[lane], reinterpret_cast<const uint8_t*>(ibase) + list * a.cap + 4 * lane);
            if (lane == 31) cp_async4(&sl->cnt, a.counts + list);
        }
        cp_async_commit();
    };
#pragma unroll 1
    for (int d = 0; d < kSegRing; ++d) issue(d);

    unsigned long long wp[V::NWOPS];
#pragma unroll
    for (int i = 0; i < V::NWOPS; ++i) wp[i] = 0ull;
    int s = 0;  // next segment to stage
#pragma unroll 1
    for (int ch = 0; ch < nchunks; ++ch) {
        const int st = ch % STAGES;
        const int cc_n = (a.Cg - ch * CH) < CH ? (a.Cg - ch * CH) : CH;
        const unsigned wlane = smem_u32(ring + st * SM::kStageFloats) + lane * 4 * V::KL;
        if (active) {
            // Stage this chunk's entry stream: per channel a LOADW entry, then
            // its in-window nonzeros (ascending), finally EXIT.
            int base = 0;
#pragma unroll 1
            for (int cc = 0; cc < cc_n; ++cc) {
                if (lane == 0) ent[base] = make_uint2((unsigned)(cc * RS * KBW * 4), (unsigned)V::LOADW);
                ++base;
#pragma unroll 1
                for (int l = 0; l < nl; ++l, ++s) {
                    cp_async_wait<kSegRing - 1>();  // segment s has landed
                    __syncwarp();
                    SegSlot* sl = segring + (s % kSegRing);
                    const uint32_t cnt = sl->cnt;
                    float v0 = sl->v[lane];
                    int i0 = (int)((sl->i4[lane >> 2] >> (8 * (lane & 3))) & 0xffu);
                    __syncwarp();
                    issue(s + kSegRing);  // refill this slot
                    const int off = ((tl_lo + l) * a.th - (y0 - V::P)) * W;
#pragma unroll 1
                    for (uint32_t e0 = 0; e0 < cnt; e0 += 32) {
                        if (e0 > 0) {  // long list (dense input): synchronous loads
                            const int list = seg_list(s);
                            const bool ok = e0 + lane < cnt;
                            v0 = ok ? vbase[(size_t)list * a.cap + e0 + lane] : 0.f;
                            i0 = ok ? (int)ibase[(size_t)list * a.cap + e0 + lane] : 0;
                        }
                        const int cs = i0 + off;
                        const bool inwin = (e0 + lane < cnt) && cs >= 0 && cs < V::NCASES;
                        const unsigned bal = __ballot_sync(0xffffffffu, inwin);
                        if (base + 32 + 2 > kEntCap) {  // stream full: run what we have
                            if (lane == 0) ent[base] = make_uint2(0u, (unsigned)V::EXIT);
                            __syncwarp();
                            mbar_wait(&full[st], (ch / STAGES) & 1);
                            V::run(acc, wp, ent_s, wlane);
                            __syncwarp();
                            base = 0;
                        }
                        const int rank = __popc(bal & ((1u << lane) - 1u));
                        if (inwin) ent[base + rank] = make_uint2(__float_as_uint(v0), (unsigned)cs);
                        base += __popc(bal);
                    }
                }
            }
            if (lane == 0) ent[base] = make_uint2(0u, (unsigned)V::EXIT);
            __syncwarp();
            mbar_wait(&full[st], (ch / STAGES) & 1);  // this chunk's weights have landed
            V::run(acc, wp, ent_s, wlane);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (threadIdx.x == 0 && ch >= 1) {
            const int q = ch - 1 + STAGES;
            if (q < nchunks) {
                const int qs = (ch - 1) % STAGES;
                mbar_wait(&empty[qs], ((ch - 1) / STAGES) & 1);
                const int chs = (a.Cg - q * CH) < CH ? (a.Cg - q * CH) : CH;
                const unsigned bytes = (unsigned)(chs * RS * KBW * sizeof(float));
                mbar_expect_tx(&full[qs], bytes);
                tma_bulk_g2s(ring + qs * SM::kStageFloats, wsrc + (size_t)q * CH * RS * KBW, bytes, &full[qs]);
            }
        }
    }

    if (!active) return;
    // Epilogue: registers -> smem [k][rows*WO] -> contiguous NCHW runs.
    constexpr int ER = SM::kER, ES = SM::kEpiStride;
    float* epi = epi_all + warp * KBW * ES;
    const int kloc = kb * KBW;
#pragma unroll
    for (int r0 = 0; r0 < TY; r0 += ER) {
#pragma unroll
        for (int rr = 0; rr < ER; ++rr) {
            if (r0 + rr < TY) {
#pragma unroll
                for (int m = 0; m < NX; ++m) {
                    const float lo = __uint_as_float((unsigned)acc[r0 + rr][m]);
                    const float hi = __uint_as_float((unsigned)(acc[r0 + rr][m] >> 32));
                    if constexpr (V::KL == 2) {  // (k = 2*lane, 2*lane+1) of pixel x = m
                        epi[(2 * lane) * ES + rr * WO + m] = lo;
                        epi[(2 * lane + 1) * ES + rr * WO + m] = hi;
                    } else {                     // (x = 2m, 2m+1) of channel k = lane
                        epi[lane * ES + rr * WO + 2 * m] = lo;
                        if (2 * m + 1 < WO) epi[lane * ES + rr * WO + 2 * m + 1] = hi;
                    }
                }
            }
        }
        __syncwarp();
        int rows = TY - r0 < ER ? TY - r0 : ER;
        if (y0 + r0 + rows > a.Ho) rows = a.Ho - (y0 + r0);
        if (rows > 0) {
            const int len = rows * WO;
#pragma unroll 1
            for (int kk = 0; kk < KBW; ++kk) {
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
    a.ctas_per_kb = (a.units + V::NW - 1) / V::NW;
    const size_t smem = Smem<V>::total;
    auto kern = gather_fast_kernel<V, IdxT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = (int64_t)a.ctas_per_kb * g.G * g.kblocks;
    kern<<<(unsigned)grid, V::NW * 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace fast
}  // namespace sc

// Each gather_fast_vN.cu instantiates one variant (parallel compilation).
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
