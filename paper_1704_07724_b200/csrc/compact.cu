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

static cudaError_t launch_compact_streamwise(const Geometry& g, int64_t n, const float* in, uint2* entries,
                                            uint32_t* offs, cudaStream_t st) {
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

// ---------------------------------------------------------------------------
// Plane-major path (planes of up to kMaxPlane elements): every plane is read
// once per kernel instead of once per tile window.
//  count: one warp per (image, channel) plane: compacts the plane (ballot
//         ranks, row-major = stream order) into plist[plane] as (bits, flat
//         index), the exclusive row prefix prow[plane][0..H] (shared atomics +
//         shuffle scan), and each tile's window count cnt[n][t][c] =
//         prow[r1] - prow[r0].
//  emit:  one CTA per (image, chunk of 32 channels).  Warp w scans tiles
//         w, w+NW, ...: the chunk's stream base is 1 + count summed over the
//         channels before it, a shuffle scan over the chunk's channels gives
//         each marker index (-> offs).  Then every (channel, tile) gets its
//         marker and the contiguous run plist[prow[r0] .. prow[r1]) of the
//         plane, positions re-coded relative to the window.
// ---------------------------------------------------------------------------
namespace {
constexpr int kMaxPlane = 2048;   // elements per plane on the plane-major path (list: 16 KB/warp)
constexpr int kPlaneWarps = 8;
constexpr int kPlaneChunk = 32;   // channels per emit CTA
constexpr int kMaxTiles = 64;

// floor(e / W) for 0 <= e < 2^32 / W: magic = floor(2^32 / W) + 1
__device__ __forceinline__ unsigned div_w(unsigned e, unsigned magic) { return __umulhi(e, magic); }
}  // namespace

__global__ void __launch_bounds__(kPlaneWarps * 32) compact_plane_count_kernel(
    const float* __restrict__ in, int planes, int C, int H, int W, unsigned magic, int TYT, int P, int NWR,
    int tiles, uint32_t* __restrict__ cnt, uint2* __restrict__ plist, uint32_t* __restrict__ prow) {
    extern __shared__ uint32_t rows_s[];  // [kPlaneWarps][H + 1]: nonzeros per row, then prefix
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int plane = blockIdx.x * kPlaneWarps + warp;
    if (plane >= planes) return;
    uint32_t* rc = rows_s + warp * (H + 1);
    for (int r = lane; r <= H; r += 32) rc[r] = 0u;
    __syncwarp();
    const int HW = H * W;
    const float* src = in + (int64_t)plane * HW;
    uint2* lst = plist + (int64_t)plane * HW;
    const unsigned lt = (1u << lane) - 1u;
    uint32_t total = 0;
    for (int e0 = 0; e0 < HW; e0 += 128) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + 32 * u + lane;
            v[u] = e < HW ? __ldg(src + e) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned bal = __ballot_sync(0xffffffffu, v[u] != 0.0f);  // IEEE: -0.0 is zero
            if (v[u] != 0.0f) {
                const unsigned e = (unsigned)(e0 + 32 * u + lane);
                lst[total + __popc(bal & lt)] = make_uint2(__float_as_uint(v[u]), e);  // row-major = stream order
                atomicAdd(&rc[div_w(e, magic) + 1], 1u);
            }
            total += __popc(bal);
        }
    }
    __syncwarp();
    // rc[r] = nonzeros in rows < r (exclusive prefix over H + 1 entries) -> prow
    uint32_t carry = 0;
    for (int r0 = 0; r0 <= H; r0 += 32) {
        const int r = r0 + lane;
        uint32_t x = r <= H ? rc[r] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += u;
        }
        x += carry;
        if (r <= H) {
            rc[r] = x;
            prow[(int64_t)plane * (H + 1) + r] = x;
        }
        carry = __shfl_sync(0xffffffffu, x, 31);
    }
    __syncwarp();
    const int n = plane / C, c = plane - (plane / C) * C;
    for (int t = lane; t < tiles; t += 32) {  // window rows of tile t: [t*TYT - P, + NWR) within the plane
        const int lo = t * TYT - P;
        const int r0 = lo < 0 ? 0 : lo, r1 = (lo + NWR < H) ? lo + NWR : H;
        cnt[((int64_t)n * tiles + t) * C + c] = r1 > r0 ? rc[r1] - rc[r0] : 0u;
    }
}

__global__ void __launch_bounds__(kPlaneWarps * 32) compact_plane_emit_kernel(
    const uint2* __restrict__ plist, const uint32_t* __restrict__ prow, const uint32_t* __restrict__ cnt, int C,
    int H, int W, int TYT, int P, int NWR, int NWIN, int tiles, int64_t cap, int chunks, uint2* __restrict__ entries,
    uint32_t* __restrict__ offs) {
    __shared__ uint32_t start_s[kMaxTiles][kPlaneChunk];
    __shared__ int2 trow_s[kMaxTiles];  // window rows [r0, r1) of tile t within the plane
    __shared__ uint2* tst_s[kMaxTiles];  // stream base of tile t
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int chunk = blockIdx.x % chunks;
    const int n = blockIdx.x / chunks;
    const int c0 = chunk * kPlaneChunk;
    const int nch = (C - c0) < kPlaneChunk ? (C - c0) : kPlaneChunk;
    const int HW = H * W;
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
        const int i_lo = t * TYT - P;
        trow_s[t] = make_int2(i_lo < 0 ? 0 : i_lo, (i_lo + NWR < H) ? i_lo + NWR : H);
        tst_s[t] = entries + ((int64_t)n * tiles + t) * cap;
    }
    // ---- stream offsets of this chunk's channels in every tile stream
    for (int t = warp; t < tiles; t += kPlaneWarps) {
        const uint32_t* cs = cnt + ((int64_t)n * tiles + t) * C;
        uint32_t base = 0;
        for (int c = lane; c < c0; c += 32) base += 1u + cs[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) base += __shfl_xor_sync(0xffffffffu, base, o);
        const uint32_t v = lane < nch ? 1u + cs[c0 + lane] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        const uint32_t start = base + incl - v;
        start_s[t][lane] = start;
        uint32_t* of = offs + ((int64_t)n * tiles + t) * (C + 1);
        if (lane < nch) of[c0 + lane] = start;
        if (lane == nch - 1 && c0 + nch == C) of[C] = start + v;
    }
    __syncthreads();
    // ---- every (channel, tile): marker + the run of the plane's list inside the window rows.
    // The plane's row prefix (lanes over rows) and its list (lanes over entries,
    // 32 per register block) are loaded once; the runs are assembled with shuffles.
    for (int ch = warp; ch < nch; ch += kPlaneWarps) {
        const int plane = n * C + c0 + ch;
        const uint2* lst = plist + (int64_t)plane * HW;
        const uint32_t* pr = prow + (int64_t)plane * (H + 1);
        const uint32_t pv = lane <= H ? __ldg(pr + lane) : 0u;  // lane r: nonzeros in rows < r (H < 32)
        const uint32_t total = H < 32 ? __shfl_sync(0xffffffffu, pv, H) : __ldg(pr + H);
        for (uint32_t k0 = 0; k0 < total || k0 == 0; k0 += 32) {  // list block [k0, k0 + 32)
            const uint2 en = k0 + lane < total ? __ldg(lst + k0 + lane) : make_uint2(0u, 0u);
            for (int t = 0; t < tiles; ++t) {
                const int2 rr = trow_s[t];
                uint2* st = tst_s[t];
                const uint32_t pos = start_s[t][ch] + 1;
                if (k0 == 0 && lane == 0) st[pos - 1] = make_uint2((unsigned)(c0 + ch), (unsigned)NWIN);
                // run [a, b) of the list (row prefix values at the window rows)
                const uint32_t a = H < 32 ? __shfl_sync(0xffffffffu, pv, rr.x) : __ldg(pr + rr.x);
                const uint32_t b = H < 32 ? __shfl_sync(0xffffffffu, pv, rr.y) : __ldg(pr + rr.y);
                const unsigned shift = (unsigned)((t * TYT - P) * W);  // code = flat index - i_lo*W
                // block k0 covers list indices [k0, k0+32): lane l writes entry k0 + l if inside the run
                const uint32_t k = k0 + lane;
                if (k >= a && k < b) st[pos + (k - a)] = make_uint2(en.x, en.y - shift);
            }
            if (total == 0) break;
        }
    }
}

cudaError_t launch_compact(const Geometry& g, int64_t n, const float* in, uint32_t* cnt, uint2* plist,
                           uint32_t* prow, uint2* entries, uint32_t* offs, cudaStream_t st) {
    if (!compact_uses_counts(g) || cnt == nullptr || plist == nullptr || prow == nullptr)
        return launch_compact_streamwise(g, n, in, entries, offs, st);
    const unsigned magic = (unsigned)((0x100000000ull / (uint64_t)g.W) + 1ull);
    const int TYT = (int)(g.ty * g.T);
    const int planes = (int)(n * g.C);
    compact_plane_count_kernel<<<(unsigned)((planes + kPlaneWarps - 1) / kPlaneWarps), kPlaneWarps * 32,
                                 sizeof(uint32_t) * kPlaneWarps * (g.H + 1), st>>>(
        in, planes, (int)g.C, (int)g.H, (int)g.W, magic, TYT, (int)g.P, (int)g.nwr, (int)g.tiles, cnt, plist, prow);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int chunks = (int)((g.C + kPlaneChunk - 1) / kPlaneChunk);
    compact_plane_emit_kernel<<<(unsigned)(n * chunks), kPlaneWarps * 32, 0, st>>>(
        plist, prow, cnt, (int)g.C, (int)g.H, (int)g.W, TYT, (int)g.P, (int)g.nwr, (int)g.nwin, (int)g.tiles, g.cap,
        chunks, entries, offs);
    return cudaGetLastError();
}

bool compact_uses_counts(const Geometry& g) {
    return g.H * g.W <= kMaxPlane && g.tiles <= kMaxTiles && g.H + 1 <= 1024;
}

}  // namespace sc
