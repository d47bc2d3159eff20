// Stage 1 of the sparse path: on-the-fly nonzero compaction into tile streams.
//
// ISC step 1: "we skip all the zero elements of the input data,
// and store the non-zero values in a vector with their column and row
// information".  Output format: reading R9 (include/sparse_conv.h,
// DESIGN.md): one stream per (image n, output row-tile t) holding, for every
// input channel c in order, a marker (c, NWIN) followed by the channel's
// nonzeros inside the tile's input window as (value bits, window position),
// ascending; offs[n][t][c] = index of channel c's marker, offs[..][C] = length.
// The stream is exactly the instruction stream the stage-2 interpreter runs.
//
// Design: one CTA per stream, one pass over the data.
// The window rows of one channel are a single contiguous run of the NCHW
// array (`seg` floats).  Channels are processed in rounds of NW*RCH (warp w
// owns channels w, w+NW, ...).  In a round every lane issues all its loads
// at once (RCH channels x KV coalesced 4-byte loads, lanes over the run), so
// one HBM/L2 round trip covers the round; __ballot_sync masks of the loaded
// values give the per-channel counts, a block scan of (1 + count) gives every
// channel's marker index (-> offs), and the same masks place each nonzero at
// its rank (__popc of the lower lanes) -- values are written from registers,
// nothing is re-read.  Runs longer than 32*KV floats are handled in blocks
// (counted first, re-loaded for the emit).
#include "sc_internal.h"

namespace sc {

namespace {
constexpr int kRegs = 16;  // RCH * KV: values held per lane per round
}  // namespace

template <int KV>
__global__ void __launch_bounds__(512) compact_streams_kernel(const float* __restrict__ in, int C, int H, int W,
                                                               int TY, int tiles, int T, int P, int NWR, int NWIN,
                                                               int64_t cap, uint2* __restrict__ entries,
                                                               uint32_t* __restrict__ offs) {
    constexpr int RCH = kRegs / KV;  // channels per warp per round
    constexpr int BLK = 32 * KV;     // floats per load block
    __shared__ uint32_t start_s[32 * RCH];
    __shared__ uint32_t wsum_s[33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int stream = blockIdx.x;
    const int n = stream / tiles, t = stream - n * tiles;
    const int i_lo = t * TY * T - P;
    const int r0 = i_lo < 0 ? 0 : i_lo;
    const int r1 = (i_lo + NWR < H) ? i_lo + NWR : H;
    const int seg = r1 > r0 ? (r1 - r0) * W : 0;        // window rows: one contiguous run per plane
    const unsigned shift = (unsigned)((r0 - i_lo) * W);  // window position of the run's first element
    const unsigned lt = (1u << lane) - 1u;
    const float* img = in + (int64_t)n * C * H * W + (int64_t)r0 * W;
    uint2* st = entries + (int64_t)stream * cap;
    uint32_t* of = offs + (int64_t)stream * (C + 1);
    const int per_round = nw * RCH;

    uint32_t base = 0;
    for (int cb = 0; cb < C; cb += per_round) {
        const int nround = (C - cb) < per_round ? (C - cb) : per_round;
        // ---- loads of the first block of every owned channel, all in flight
        float v[RCH][KV];
#pragma unroll
        for (int q = 0; q < RCH; ++q) {
            const int ch = warp + q * nw;
            const float* src = img + (int64_t)(cb + ch) * H * W;
#pragma unroll
            for (int u = 0; u < KV; ++u) {
                const int off = 32 * u + lane;
                v[q][u] = (ch < nround && off < seg) ? __ldg(src + off) : 0.0f;
            }
        }
        // ---- counts (ballot masks of the first block are kept for the emit)
        unsigned bal[RCH][KV];
#pragma unroll
        for (int q = 0; q < RCH; ++q) {
            const int ch = warp + q * nw;
            uint32_t cnt = 0;
#pragma unroll
            for (int u = 0; u < KV; ++u) {
                bal[q][u] = __ballot_sync(0xffffffffu, v[q][u] != 0.0f);  // IEEE: -0.0 is zero
                cnt += __popc(bal[q][u]);
            }
            if (seg > BLK && ch < nround) {  // long runs: count the remaining blocks
                const float* src = img + (int64_t)(cb + ch) * H * W;
                for (int o0 = BLK; o0 < seg; o0 += 32) {
                    const float x = o0 + lane < seg ? __ldg(src + o0 + lane) : 0.0f;
                    cnt += __popc(__ballot_sync(0xffffffffu, x != 0.0f));
                }
            }
            if (lane == 0 && ch < nround) start_s[ch] = 1u + cnt;
        }
        __syncthreads();
        // ---- block-wide exclusive scan of (1 + count) over the round's channels;
        // thread i owns channels RCH*i .. RCH*i + RCH-1 of the round
        {
            uint32_t a[RCH];
            uint32_t mine = 0;
#pragma unroll
            for (int q = 0; q < RCH; ++q) {
                const int i = RCH * (int)threadIdx.x + q;
                a[q] = i < nround ? start_s[i] : 0u;
                mine += a[q];
            }
            uint32_t incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            if (lane == 31) wsum_s[warp] = incl;
            __syncthreads();
            if (warp == 0) {
                const uint32_t x = lane < nw ? wsum_s[lane] : 0u;
                uint32_t xi = x;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t u = __shfl_up_sync(0xffffffffu, xi, o);
                    if (lane >= o) xi += u;
                }
                wsum_s[lane] = xi - x;  // exclusive warp offsets
                if (lane == 31) wsum_s[32] = xi;  // round total
            }
            __syncthreads();
            uint32_t excl = base + wsum_s[warp] + incl - mine;
#pragma unroll
            for (int q = 0; q < RCH; ++q) {
                const int i = RCH * (int)threadIdx.x + q;
                if (i < nround) {
                    start_s[i] = excl;
                    of[cb + i] = excl;
                }
                excl += a[q];
            }
            __syncthreads();
        }
        // ---- emit: marker + entries at their ranks (first block from registers)
#pragma unroll
        for (int q = 0; q < RCH; ++q) {
            const int ch = warp + q * nw;
            if (ch < nround) {
                uint32_t pos = start_s[ch];
                if (lane == 0) st[pos] = make_uint2((unsigned)(cb + ch), (unsigned)NWIN);
                ++pos;
#pragma unroll
                for (int u = 0; u < KV; ++u) {
                    if (v[q][u] != 0.0f)
                        st[pos + __popc(bal[q][u] & lt)] =
                            make_uint2(__float_as_uint(v[q][u]), shift + (unsigned)(32 * u + lane));
                    pos += __popc(bal[q][u]);
                }
                if (seg > BLK) {
                    const float* src = img + (int64_t)(cb + ch) * H * W;
                    for (int o0 = BLK; o0 < seg; o0 += 32) {
                        const float x = o0 + lane < seg ? __ldg(src + o0 + lane) : 0.0f;
                        const unsigned b = __ballot_sync(0xffffffffu, x != 0.0f);
                        if (x != 0.0f)
                            st[pos + __popc(b & lt)] = make_uint2(__float_as_uint(x), shift + (unsigned)(o0 + lane));
                        pos += __popc(b);
                    }
                }
            }
        }
        base += wsum_s[32];
        __syncthreads();  // start_s / wsum_s are reused by the next round
    }
    if (threadIdx.x == 0) of[C] = base;
}

cudaError_t launch_compact(const Geometry& g, int64_t n, const float* in, uint2* entries, uint32_t* offs,
                           cudaStream_t st) {
    const int64_t rows = g.nwr < g.H ? g.nwr : g.H;
    const int64_t seg = rows * g.W;
    const int kv = seg <= 32 ? 1 : seg <= 64 ? 2 : seg <= 128 ? 4 : 8;
    const int rch = kRegs / kv;
    // enough warps for every channel in one round, at most 16 (several CTAs per SM overlap
    // one CTA's scan with another's loads)
    int64_t warps = (g.C + rch - 1) / rch;
    if (warps > 16) warps = 16;
    if (warps < 2) warps = 2;
    const unsigned threads = (unsigned)(32 * warps);
    const unsigned grid = (unsigned)(n * g.tiles);
#define SC_LAUNCH_KV(K)                                                                                            \
    compact_streams_kernel<K><<<grid, threads, 0, st>>>(in, (int)g.C, (int)g.H, (int)g.W, (int)g.ty,               \
                                                        (int)g.tiles, (int)g.T, (int)g.P, (int)g.nwr, (int)g.nwin, \
                                                        g.cap, entries, offs)
    if (kv == 1) SC_LAUNCH_KV(1);
    else if (kv == 2) SC_LAUNCH_KV(2);
    else if (kv == 4) SC_LAUNCH_KV(4);
    else SC_LAUNCH_KV(8);
#undef SC_LAUNCH_KV
    return cudaGetLastError();
}

}  // namespace sc
