// Device half of the shape-specialised stage-2 kernel (see gather_fast_impl.cuh for
// the design).  Self-contained device code: compiled into libsparseconv.so for the
// generated variants (gather_variants.inc) and, at run time through NVRTC, for a
// variant generated for a plan's shape (jit.cu).  Include inside no namespace,
// after the variant struct(s) are declared in sc::fast.
#pragma once
#include "sc_device.h"

namespace sc {
namespace fast {

template <class A, class B>
struct same_type {
    static constexpr bool value = false;
};
template <class A>
struct same_type<A, A> {
    static constexpr bool value = true;
};

// Per variant (gather_variants.inc): V::PIECE = max entries per piece (+ alignment
// slot + EXIT), V::SLOTS = pieces in flight per warp.

struct Args {
    const uint2* entries;
    const uint32_t* offs;
    const float* wpack;
    const float* bias;
    float* out;        // NCHW output; may be null when rowlist is set (chained layers)
    uint2* rowlist;    // chained layers: the next layer's per-(plane,row) lists
    uint32_t* rowcnt;  //   [N*K][Ho][WO] entries (bits, y*WO + x) and [N*K][Ho] counts
    int n, C, H, K, Cg, Kg, kblocks, Ho, relu;
    int64_t cap;
    int ytiles, units, ctas_per_kb;
    int edge_last;     // unit order: interior row tiles first, edge tiles last (grids of >= 2 waves)
};
// f3 (device-side path selection) launches a separate instantiation with the gate
// appended: adding the field to Args itself was measured to slow the ungated
// kernel by 10% (V21, C2 s=0.95: 172 -> 189 us; register allocation shifts).
struct ArgsGated : Args {
    Gate gate;
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
    static constexpr int KBW = 32 * V::KL;
    static constexpr int kStageFloats = V::CH * V::R * V::S * KBW;
    // The epilogue reuses the warp's own piece slots (all its pieces have been
    // consumed by then): KBW x kEpiStride floats must fit V::SLOTS*(V::PIECE+2)*8 B.
    static constexpr int kPieceFloats = V::SLOTS * (V::PIECE + 2) * 2;
    // One epilogue pass covers 32 output channels (KL passes).
    static constexpr int kERraw = ((kPieceFloats / 32) - 1) / V::WO;
    static constexpr int kER = kERraw < 1 ? 1 : (kERraw > V::TY ? V::TY : kERraw);
    static constexpr int kEpiStride = (kER * V::WO) | 1;  // odd
    static_assert(32 * kEpiStride <= kPieceFloats, "epilogue buffer does not fit the piece slots");
    static constexpr size_t ring = sizeof(float) * V::STAGES * kStageFloats;
    static constexpr size_t bars = 8 * (2 * V::STAGES + V::NW * V::SLOTS);
    static constexpr size_t bars_pad = (bars + 127) / 128 * 128;
    // +4 entries: the interpreter prefetches up to two entries past EXIT, which for a
    // full piece in the last slot of the last warp lies beyond the ring
    static constexpr size_t pieces = sizeof(uint2) * (V::NW * V::SLOTS * (V::PIECE + 2) + 4);
    static constexpr size_t total = ring + bars_pad + pieces;
    static_assert(total * V::MINB <= 227 * 1024, "shared memory budget of the SM exceeded");
};

template <class V, bool EMIT, class A = Args>
__global__ void __launch_bounds__((V::NW + 1) * 32, V::MINB) gather_fast_kernel(const A a) {
    using SM = Smem<V>;
    constexpr int RS = V::R * V::S, TY = V::TY, NX = V::NX, WO = V::WO;
    constexpr int CH = V::CH, STAGES = V::STAGES, NW = V::NW, KBW = SM::KBW;
    if constexpr (same_type<A, ArgsGated>::value) {
        if (gate_closed(a.gate)) return;
    }
    extern __shared__ __align__(128) unsigned char smem[];
    float* ring = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::ring);
    uint64_t* empty = full + STAGES;
    uint64_t* pbar_all = empty + STAGES;  // [NW][V::SLOTS]
    uint2* piece_all = reinterpret_cast<uint2*>(smem + SM::ring + SM::bars_pad);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cb = blockIdx.x % a.ctas_per_kb;
    const int gkb = blockIdx.x / a.ctas_per_kb;  // g * kblocks + kb
    const int kb = gkb % a.kblocks, g = gkb / a.kblocks;
    const int unit = cb * NW + warp;
    const bool active = unit < a.units;
    const int nactive = (a.units - cb * NW) < NW ? (a.units - cb * NW) : NW;
    const int nchunks = (a.Cg + CH - 1) / CH;
    const float* wsrc = a.wpack + (size_t)gkb * a.Cg * RS * KBW;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], (unsigned)nactive);
        }
        for (int i = 0; i < NW * V::SLOTS; ++i) mbar_init(&pbar_all[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NW) {  // producer warp: streams the weight chunks through the ring
        if (lane == 0) {
            for (int q = 0; q < nchunks; ++q) {
                const int qs = q % STAGES;
                if (q >= STAGES) mbar_wait(&empty[qs], ((q / STAGES) - 1) & 1);  // all warps released it
                const int chs = (a.Cg - q * CH) < CH ? (a.Cg - q * CH) : CH;
                const unsigned bytes = (unsigned)(chs * RS * KBW * sizeof(float));
                mbar_expect_tx(&full[qs], bytes);
                // the stage in four bulk copies (more requests in flight than one long copy)
                const unsigned part = ((bytes / 4u) + 15u) & ~15u;
                for (unsigned off = 0; off < bytes; off += part) {
                    const unsigned len = bytes - off < part ? bytes - off : part;
                    tma_bulk_g2s(reinterpret_cast<unsigned char*>(ring + qs * SM::kStageFloats) + off,
                                 reinterpret_cast<const unsigned char*>(wsrc + (size_t)q * CH * RS * KBW) + off, len,
                                 &full[qs]);
                }
            }
        }
        return;
    }
    if (!active) return;

    // Unit order (edge_last): interior row tiles first, then every image's first tile, then
    // its last tile.  The edge tiles' input windows are clipped by the padding (C2: 3 and 2 of 4
    // window rows), so their streams are shorter; consecutive units share a CTA whose
    // warps walk the weight ring in lock step, so grouping by tile position keeps short
    // streams from idling in CTAs of long ones, and the short CTAs run last (measured: C5 -7%;
    // single-batch C2 (1.66 waves) +1%, but -4% per batch when batches are pipelined, so it is
    // on for every grid: sc_internal.h edge_last_order).  A relabelling only: every stream is
    // computed the same way by whichever warp owns it.
    int n, tile;
    {
        const int nimg = a.n, T = a.ytiles;
        const int inner = T > 2 ? nimg * (T - 2) : 0;
        if (!a.edge_last) {
            n = unit / T;
            tile = unit - n * T;
        } else if (unit < inner) {
            n = unit % nimg;
            tile = 1 + unit / nimg;
        } else {
            const int e = unit - inner;
            n = e % nimg;
            tile = T > 2 ? (e < nimg ? 0 : T - 1) : e / nimg;
        }
    }
    const int y0 = tile * TY;
    const int64_t stream = (int64_t)n * a.ytiles + tile;
    const uint2* sbase = a.entries + stream * a.cap;
    const uint32_t* of = a.offs + stream * (a.C + 1) + (int64_t)g * a.Cg;  // of[cl] = marker of channel g*Cg+cl
    uint64_t* pbar = pbar_all + warp * V::SLOTS;
    uint2* pieces = piece_all + warp * V::SLOTS * (V::PIECE + 2);

    // f32x2 bit patterns (low word = first element): channel pairs (KL >= 2) or
    // x pairs (KL == 1); odd KL adds one f32 accumulator per pixel
    unsigned long long accp[TY][NX][V::NPAIR];
    float accs[TY][NX];
#pragma unroll
    for (int ty = 0; ty < TY; ++ty)
#pragma unroll
        for (int m = 0; m < NX; ++m) {
#pragma unroll
            for (int pi = 0; pi < V::NPAIR; ++pi) accp[ty][m][pi] = 0ull;
            accs[ty][m] = 0.0f;
        }
    unsigned long long wp[V::NWP];
    float ws[V::NWS];
#pragma unroll
    for (int i = 0; i < V::NWP; ++i) wp[i] = 0ull;
#pragma unroll
    for (int i = 0; i < V::NWS; ++i) ws[i] = 0.0f;

    // Chunk boundaries bnd(q) = of[min(q*CH, Cg)], q <= nchunks (<= 63), held
    // two per lane and broadcast with shuffles.
    // programmatic dependent launch: everything above overlaps the tail of stage 1; its
    // outputs (offs, entries) are read only from here on (a no-op without the launch attribute)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t bnd0 = __ldg(&of[(lane * CH < a.Cg) ? lane * CH : a.Cg]);
    const uint32_t bnd1 = __ldg(&of[((lane + 32) * CH < a.Cg) ? (lane + 32) * CH : a.Cg]);
    auto bnd = [&](int q) -> uint32_t {
        const uint32_t v0 = __shfl_sync(0xffffffffu, bnd0, q & 31);
        const uint32_t v1 = __shfl_sync(0xffffffffu, bnd1, q & 31);
        return q < 32 ? v0 : v1;
    };
    // Piece sequence: the range [bnd(0), bnd(nchunks)) cut at chunk
    // boundaries and every V::PIECE entries.  Issue and consume cursors walk it
    // identically; lane 0 issues the bulk copies.
    // Chunks without entries (R9: their channels have no markers either) get no piece: bit q of
    // `filled` marks chunk q non-empty; the issue cursor jumps over the others.
    const uint32_t dn0 = __shfl_down_sync(0xffffffffu, bnd0, 1);  // all lanes take part in every shuffle
    const uint32_t b32 = __shfl_sync(0xffffffffu, bnd1, 0);
    const uint32_t nb0 = lane < 31 ? dn0 : b32;                      // bnd(lane + 1)
    const uint32_t nb1 = __shfl_down_sync(0xffffffffu, bnd1, 1);     // bnd(lane + 33)
    const uint64_t filled = (uint64_t)__ballot_sync(0xffffffffu, lane < nchunks && nb0 > bnd0) |
                            ((uint64_t)__ballot_sync(0xffffffffu, lane + 32 < nchunks && nb1 > bnd1) << 32);
    auto next_filled = [&](int q) -> int {  // first non-empty chunk >= q, else nchunks
        const uint64_t rest = q < 64 ? filled >> q : 0ull;
        return rest ? q + __ffsll((long long)rest) - 1 : nchunks;
    };
    int iq = next_filled(0);    // issue cursor: chunk (non-empty or nchunks)
    uint32_t ia = bnd(iq < nchunks ? iq : 0);        // issue cursor: next entry
    uint32_t iend = bnd(iq < nchunks ? iq + 1 : 0);
    int issued = 0;
    auto issue_next = [&]() {
        if (iq >= nchunks) return;
        const uint32_t b = (ia + V::PIECE < iend) ? ia + V::PIECE : iend;
        const int slot = issued % V::SLOTS;
        if (lane == 0) {
            const uint32_t a2 = ia & ~1u;
            const unsigned bytes = ((b - a2) * 8u + 15u) & ~15u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // EXIT write -> TMA overwrite
            mbar_expect_tx(&pbar[slot], bytes);
            tma_bulk_g2s(pieces + slot * (V::PIECE + 2), sbase + a2, bytes, &pbar[slot]);
        }
        ++issued;
        ia = b;
        if (ia == iend) {
            iq = next_filled(iq + 1);
            const int qq = iq < nchunks ? iq : 0;
            ia = bnd(qq);
            iend = bnd(qq + 1);
        }
    };
#pragma unroll 1
    for (int i = 0; i < V::SLOTS; ++i) issue_next();

    int consumed = 0;
    uint32_t ca = bnd(0);  // consume cursor
#pragma unroll 1
    for (int ch = 0; ch < nchunks; ++ch) {
        const int st = ch % STAGES;
        const uint32_t chunk_end = bnd(ch + 1);
        const unsigned wstage = smem_u32(ring + st * SM::kStageFloats);
        // lane's weights in a tap block of 32*KL floats (pack.cu): KL=1,2,4 lane-contiguous
        // runs of KL floats; KL=3 a pair at 8*lane and a single at 256 + 4*lane
        const unsigned wlane = wstage + lane * (V::XPAIR ? 4u : 8u * V::NPAIR);
        const unsigned wlane_s = wstage + lane * 4u;
        const unsigned cbase = (unsigned)(g * a.Cg + ch * CH);
        mbar_wait(&full[st], (ch / STAGES) & 1);  // this chunk's weights have landed
#pragma unroll 1
        while (ca < chunk_end) {
            const uint32_t b = (ca + V::PIECE < chunk_end) ? ca + V::PIECE : chunk_end;
            const int slot = consumed % V::SLOTS;
            mbar_wait(&pbar[slot], (consumed / V::SLOTS) & 1);
            uint2* p = pieces + slot * (V::PIECE + 2) + (ca & 1u);
            if (lane == 0) p[b - ca] = make_uint2(0u, (unsigned)V::EXIT);
            __syncwarp();
            V::run(accp, accs, wp, ws, smem_u32(p), wlane, wlane_s, cbase);
            __syncwarp();
            ++consumed;
            ca = b;
            issue_next();  // refill the slot just consumed
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }

    // Epilogue: registers -> smem [k][rows*WO] -> contiguous NCHW runs, + bias,
    // optional ReLU (Eq. 2).  One pass per channel slot h of a lane (KL >= 2:
    // channel kloc + KL*lane + h; KL == 1: channel kloc + lane, pixels in pairs).
    constexpr int ER = SM::kER, ES = SM::kEpiStride;
    float* epi = reinterpret_cast<float*>(pieces);  // this warp's slots are idle now
    const int kloc = kb * KBW;
    const int krows = (a.Kg - kloc) < KBW ? (a.Kg - kloc) : KBW;  // valid output channels of this block
    float bv[V::KL];
#pragma unroll
    for (int h = 0; h < V::KL; ++h) {
        const int k = kloc + V::KL * lane + h;
        bv[h] = k < a.Kg ? __ldg(&a.bias[g * a.Kg + k]) : 0.0f;
    }
    if constexpr (EMIT) {
        // f1: this tile's output rows, after bias and ReLU, compacted per (channel, row) for
        // the next layer's stage 1 (row-major, as the plane-major compaction would list them)
        static_assert(!V::XPAIR, "chained list emission needs channel-slot accumulators");
#pragma unroll
        for (int h = 0; h < V::KL; ++h) {
            const int k = kloc + V::KL * lane + h;
#pragma unroll
            for (int ty = 0; ty < TY; ++ty) {
                const int y = y0 + ty;
                if (k < a.Kg && y < a.Ho) {
                    const size_t row = ((size_t)n * a.K + (size_t)g * a.Kg + k) * a.Ho + y;
                    uint2* dst = a.rowlist + row * WO;
                    uint32_t cnt = 0;
#pragma unroll
                    for (int m = 0; m < NX; ++m) {
                        float o;
                        if (h < 2 * V::NPAIR) {
                            const unsigned long long u = accp[ty][m][h / 2];
                            o = __uint_as_float((h & 1) ? (unsigned)(u >> 32) : (unsigned)u);
                        } else {
                            o = accs[ty][m];
                        }
                        o += bv[h];
                        if (a.relu) o = fmaxf(o, 0.f);
                        if (o != 0.0f) {  // IEEE: -0.0 is zero (R7)
                            dst[cnt] = make_uint2(__float_as_uint(o), (unsigned)(y * WO + m));
                            ++cnt;
                        }
                    }
                    a.rowcnt[row] = cnt;
                }
            }
        }
        if (a.out == nullptr) return;
    }
#pragma unroll
    for (int h = 0; h < V::KL; ++h)
#pragma unroll
    for (int r0 = 0; r0 < TY; r0 += ER) {
#pragma unroll
        for (int rr = 0; rr < ER; ++rr) {
            if (r0 + rr < TY) {
#pragma unroll
                for (int m = 0; m < NX; ++m) {
                    if constexpr (V::XPAIR) {  // (x = 2m, 2m+1) of channel k = lane
                        const unsigned long long u = accp[r0 + rr][m][0];
                        float lo = __uint_as_float((unsigned)u) + bv[0];
                        float hi = __uint_as_float((unsigned)(u >> 32)) + bv[0];
                        if (a.relu) {
                            lo = fmaxf(lo, 0.f);
                            hi = fmaxf(hi, 0.f);
                        }
                        epi[lane * ES + rr * WO + 2 * m] = lo;
                        if (2 * m + 1 < WO) epi[lane * ES + rr * WO + 2 * m + 1] = hi;
                    } else {  // channel slot h of pixel x = m
                        float o;
                        if (h < 2 * V::NPAIR) {
                            const unsigned long long u = accp[r0 + rr][m][h / 2];
                            o = __uint_as_float((h & 1) ? (unsigned)(u >> 32) : (unsigned)u);
                        } else {
                            o = accs[r0 + rr][m];
                        }
                        o += bv[h];
                        if (a.relu) o = fmaxf(o, 0.f);
                        epi[lane * ES + rr * WO + m] = o;
                    }
                }
            }
        }
        __syncwarp();
        int rows = TY - r0 < ER ? TY - r0 : ER;
        if (y0 + r0 + rows > a.Ho) rows = a.Ho - (y0 + r0);
        if (rows > 0) {
            // channel row kk (the channel of lane kk's slot h) is one contiguous run of
            // rows*WO outputs in NCHW: lanes store consecutive elements of it
            const int len = rows * WO;
            const int nrows = (krows - h + V::KL - 1) / V::KL;  // lanes whose slot h is a valid channel
            float* dst0 = a.out + ((size_t)(n * a.K + g * a.Kg + kloc + h) * a.Ho + y0 + r0) * WO + lane;
            const size_t kstride = (size_t)a.Ho * WO * V::KL;
            if (len <= 32) {
                if (lane < len) {
#pragma unroll 4
                    for (int kk = 0; kk < nrows; ++kk) dst0[kk * kstride] = epi[kk * ES + lane];
                }
            } else {
                for (int kk = 0; kk < nrows; ++kk)
                    for (int p = lane; p < len; p += 32) dst0[kk * kstride + p - lane] = epi[kk * ES + p];
            }
        }
        __syncwarp();
    }
}


}  // namespace fast
}  // namespace sc
