// Stage 1 of the sparse path: on-the-fly nonzero compaction into tile streams.
//
// ISC step 1: "we skip all the zero elements of the input data,
// and store the non-zero values in a vector with their column and row
// information".  Output format: reading R9 (include/sparse_conv.h,
// DESIGN.md): one stream per (image n, output row-tile t) holding, for every
// input channel c in order that has a nonzero inside the tile's input window, a
// marker (c, NWIN + mask) followed by those nonzeros as (value bits, window
// position), ascending; offs[n][t][c] = index of channel c's marker (channels
// without entries have none: offs[c] == offs[c+1]), offs[..][C] = length;
// bit r of mask = filter row r is reached by one of the channel's entries.
// The stream is exactly the instruction stream the stage-2 interpreter runs.
//
// Design: one CTA per stream, one pass over the data.
// The window rows of one channel are a single contiguous run of the NCHW
// array (`seg` floats).  Channels are processed in rounds of NW*RCH (warp w
// owns channels w, w+NW, ...).  In a round every lane issues all its loads
// at once (RCH channels x KV coalesced 4-byte loads, lanes over the run), so
// one HBM/L2 round trip covers the round; __ballot_sync masks of the loaded
// values give the per-channel counts, a block scan of (count ? 1 + count : 0) gives every
// channel's marker index (-> offs), and the same masks place each nonzero at
// its rank (__popc of the lower lanes) -- values are written from registers,
// nothing is re-read.  Runs longer than 32*KV floats are handled in blocks
// (counted first, re-loaded for the emit).
#include "sc_internal.h"

namespace sc {

namespace {
constexpr int kRegs = 16;  // RCH * KV: values held per lane per round

// Marker mask bits (R9) of one entry at window row wi: filter row r is reached
// iff wi - r = ty*T for a tile row 0 <= ty < TY.
__device__ __forceinline__ unsigned tap_rows(unsigned wi, int R, int T, int TY) {
    unsigned m = 0;
    for (int r = 0; r < R && r < 32; ++r) {
        const int d = (int)wi - r;
        if (d >= 0 && d % T == 0 && d / T < TY) m |= 1u << r;
    }
    return m;
}
}  // namespace

template <int KV>
__global__ void __launch_bounds__(512) compact_streams_kernel(const float* __restrict__ in, int C, int H, int W,
                                                               int TY, int tiles, int T, int P, int NWR, int NWIN,
                                                               int64_t cap, uint2* __restrict__ entries,
                                                               uint32_t* __restrict__ offs, Gate gate) {
    if (gate_closed(gate)) return;
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
    const int R = NWR - (TY - 1) * T;  // filter rows

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
            if (lane == 0 && ch < nround) start_s[ch] = cnt ? 1u + cnt : 0u;  // no entry: no marker (R9)
        }
        __syncthreads();
        // ---- block-wide exclusive scan of (count ? 1 + count : 0) over the round's channels;
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
                const uint32_t pos0 = start_s[ch];
                uint32_t pos = pos0 + 1;
                unsigned mask = 0;  // filter rows reached by this channel's entries (R9 marker)
#pragma unroll
                for (int u = 0; u < KV; ++u) {
                    if (v[q][u] != 0.0f) {
                        const unsigned code = shift + (unsigned)(32 * u + lane);
                        st[pos + __popc(bal[q][u] & lt)] = make_uint2(__float_as_uint(v[q][u]), code);
                        mask |= tap_rows(code / (unsigned)W, R, T, TY);
                    }
                    pos += __popc(bal[q][u]);
                }
                if (seg > BLK) {
                    const float* src = img + (int64_t)(cb + ch) * H * W;
                    for (int o0 = BLK; o0 < seg; o0 += 32) {
                        const float x = o0 + lane < seg ? __ldg(src + o0 + lane) : 0.0f;
                        const unsigned b = __ballot_sync(0xffffffffu, x != 0.0f);
                        if (x != 0.0f) {
                            const unsigned code = shift + (unsigned)(o0 + lane);
                            st[pos + __popc(b & lt)] = make_uint2(__float_as_uint(x), code);
                            mask |= tap_rows(code / (unsigned)W, R, T, TY);
                        }
                        pos += __popc(b);
                    }
                }
                mask = __reduce_or_sync(0xffffffffu, mask);
                if (lane == 0 && pos != pos0 + 1) st[pos0] = make_uint2((unsigned)(cb + ch), (unsigned)NWIN + mask);
            }
        }
        base += wsum_s[32];
        __syncthreads();  // start_s / wsum_s are reused by the next round
    }
    if (threadIdx.x == 0) of[C] = base;
}

static cudaError_t launch_compact_streamwise(const Geometry& g, int64_t n, const float* in, uint2* entries,
                                            uint32_t* offs, cudaStream_t st, Gate gate) {
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
                                                        g.cap, entries, offs, gate)
    if (kv == 1) SC_LAUNCH_KV(1);
    else if (kv == 2) SC_LAUNCH_KV(2);
    else if (kv == 4) SC_LAUNCH_KV(4);
    else SC_LAUNCH_KV(8);
#undef SC_LAUNCH_KV
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Plane-major path (planes of up to 32*kMaxSlots elements and at most 31 rows):
// every plane is read once from HBM and compacted once.
//  count: one warp per (image, channel) plane.  All loads of the plane are in
//         flight at once (lanes over the flat plane, NSLOT slots of 32); the
//         slot ballots stay in registers and give (a) each nonzero's rank ->
//         plist[plane] = (bits, flat index) in row-major order (= the stream
//         order), (b) the exclusive row prefix prow[plane][r] = nonzeros
//         before row r (lane r: popc of the ballot bits below r*W), and (c)
//         each tile's window count cnt[n][t][c] = prow[r1] - prow[r0].
//  emit:  one CTA per (image, chunk of 8/16/32 channels).  Warp w scans tiles
//         w, w+NW, ...: the chunk's stream base is (count ? 1 + count : 0) summed over the
//         channels before it, a shuffle scan over the chunk's channels gives
//         each marker index (-> offs).  Then, per plane, lanes over tiles write the
//         markers and lanes over the plane's list entries write each entry into every
//         tile stream whose window holds its row.
// ---------------------------------------------------------------------------
namespace {
constexpr int kMaxSlots = 32;     // plane elements / 32 on the plane-major path
constexpr int kPlaneWarps = 8;
constexpr int kMaxTiles = 32;     // tiles per image on the plane-major path
}  // namespace

template <int NSLOT, int IMG>
__global__ void __launch_bounds__(kPlaneWarps * 32, NSLOT >= 16 ? 4 : 0) compact_plane_count_kernel(
    const float* __restrict__ in, int nimg, int C, int H, int W, int TYT, int P, int NWR, int tiles,
    uint32_t* __restrict__ cnt, uint2* __restrict__ plist, uint32_t* __restrict__ prow, Gate gate) {
    // the emit kernel (a programmatic dependent on the forward path) may be scheduled once every
    // CTA of this grid is resident; it waits for this grid's completion before reading
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (gate_closed(gate)) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // grid (channel blocks, images): no division to split a plane index
    const int c = blockIdx.x * kPlaneWarps + warp;
    if (c >= C) return;
    const int HW = H * W;
    // IMG images per iteration: the loads of all of them are issued first (small planes: more
    // bytes in flight per warp)
    for (int n0 = blockIdx.y * IMG; n0 < nimg; n0 += gridDim.y * IMG) {
    float vv[IMG][NSLOT];
#pragma unroll
    for (int i = 0; i < IMG; ++i) {
        const float* src = in + (int64_t)((n0 + i) * C + c) * HW;
#pragma unroll
        for (int u = 0; u < NSLOT; ++u) {
            const int e = 32 * u + lane;
            vv[i][u] = (e < HW && n0 + i < nimg) ? __ldg(src + e) : 0.0f;
        }
    }
#pragma unroll
    for (int i = 0; i < IMG; ++i) {
    const int n = n0 + i;
    if (n >= nimg) break;
    const int plane = n * C + c;
    float (&v)[NSLOT] = vv[i];
    const unsigned lt = (1u << lane) - 1u;
    uint2* lst = plist + (int64_t)plane * HW;
    // lane r <= H: nonzeros before element r*W (the first element of row r), accumulated slot by
    // slot (branch-free: slots below sb whole, slot sb below element eb) so no slot's ballot
    // stays live past its own iteration
    const int eb = lane * W;
    const int sb = eb >> 5;
    const unsigned mb = (1u << (eb & 31)) - 1u;
    uint32_t pre = 0;
    uint32_t total = 0;
#pragma unroll
    for (int u = 0; u < NSLOT; ++u) {
        const bool nz = v[u] != 0.0f;  // IEEE: -0.0 is zero
        const unsigned bal = __ballot_sync(0xffffffffu, nz);
        if (bal != 0u) {  // warp-uniform: slots without a nonzero store nothing
            // predicated store (no branch / reconvergence per lane)
            const uint2* dst = lst + total + __popc(bal & lt);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t@p st.global.v2.u32 [%0], {%1, %2};\n\t}" ::"l"(dst),
                "r"(__float_as_uint(v[u])), "r"(32u * u + lane), "r"((unsigned)nz)
                : "memory");
        }
        const unsigned m = u < sb ? 0xffffffffu : (u == sb ? mb : 0u);
        pre += __popc(bal & m);
        total += __popc(bal);
    }
    if (lane > H) pre = total;
    if (lane <= H) prow[(int64_t)plane * (H + 1) + lane] = pre;
    // lane t: tile t's window rows [t*TYT - P, + NWR) clipped to the plane
    const int lo = lane * TYT - P;
    const int r0 = lo < 0 ? 0 : (lo > H ? H : lo), r1 = (lo + NWR < H) ? (lo + NWR < 0 ? 0 : lo + NWR) : H;
    const uint32_t p0 = __shfl_sync(0xffffffffu, pre, r0), p1 = __shfl_sync(0xffffffffu, pre, r1);
    if (lane < tiles) cnt[((int64_t)n * tiles + lane) * C + c] = r1 > r0 ? p1 - p0 : 0u;
    }
    }
}

// FROM_ROWS (chained layers, f1): the plane lists come from the producing gather as
// per-(plane, row) slots rows[plane*H + r][0..W) with counts rcnt[plane*H + r]
// (entries (bits, flat index)); each warp derives the plane's row prefix from the counts
// and finds an entry's row by a search over that prefix.
template <bool FROM_ROWS, int kPlaneChunk>
__global__ void __launch_bounds__(kPlaneWarps * 32) compact_plane_emit_kernel(
    const uint2* __restrict__ plist, const uint32_t* __restrict__ prow, const uint32_t* __restrict__ cnt, int C,
    int H, int W, int TY, int T, int P, int NWR, int NWIN, int tiles, int64_t cap, int chunks, uint2* __restrict__ entries,
    uint32_t* __restrict__ offs, Gate gate) {
    // let stage 2 (a programmatic dependent) start its prologue; it waits for this grid's
    // completion before it reads the streams
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (gate_closed(gate)) return;
    // launched as a programmatic dependent of the count kernel (FROM_ROWS: of the tile-count
    // kernel, or plainly): its lists are read only from here on (a no-op without the attribute)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ uint32_t start_s[kMaxTiles][kPlaneChunk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int chunk = blockIdx.x % chunks;
    const int n = blockIdx.x / chunks;
    const int c0 = chunk * kPlaneChunk;
    const int nch = (C - c0) < kPlaneChunk ? (C - c0) : kPlaneChunk;
    const int HW = H * W;
    // Issue this warp's plane loads (row prefix: lane r = nonzeros before row r;
    // the first 32 list entries) before the offset phase so their latency overlaps it.
    constexpr int kPerWarp = kPlaneChunk / kPlaneWarps;
    uint32_t pv[kPerWarp];
    uint2 en0[kPerWarp];
#pragma unroll
    for (int q = 0; q < kPerWarp; ++q) {
        const int ch = warp + q * kPlaneWarps;
        const int plane = n * C + c0 + ch;
        if constexpr (FROM_ROWS) {
            // prow / plist hold the row counts rcnt[plane*H + r] and the row slots
            const uint32_t rc = (ch < nch && lane < H) ? __ldg(prow + (int64_t)plane * H + lane) : 0u;
            uint32_t incl = rc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            pv[q] = incl - rc;  // lane r <= H: nonzeros before row r (lane H: the total)
            en0[q] = make_uint2(0u, 0u);
        } else {
            pv[q] = (ch < nch && lane <= H) ? __ldg(prow + (int64_t)plane * (H + 1) + lane) : 0u;
            // lanes past a small plane (HW < 32) load nothing: the last plane ends the allocation
            en0[q] = (ch < nch && lane < HW) ? __ldg(plist + (int64_t)plane * HW + lane) : make_uint2(0u, 0u);
        }
    }
    // ---- stream offsets of this chunk's channels in every tile stream
    for (int t = warp; t < tiles; t += kPlaneWarps) {
        const uint32_t* cs = cnt + ((int64_t)n * tiles + t) * C;
        uint32_t base = 0;
        for (int c = lane; c < c0; c += 32) base += cs[c] ? 1u + cs[c] : 0u;  // marker only with entries (R9)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) base += __shfl_xor_sync(0xffffffffu, base, o);
        const uint32_t cv = lane < nch ? cs[c0 + lane] : 0u;
        const uint32_t v = cv ? 1u + cv : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        const uint32_t start = base + incl - v;
        if (lane < kPlaneChunk) start_s[t][lane] = start;
        uint32_t* of = offs + ((int64_t)n * tiles + t) * (C + 1);
        if (lane < nch) of[c0 + lane] = start;
        if (lane == nch - 1 && c0 + nch == C) of[C] = start + v;
    }
    __syncthreads();
    const int TYT = TY * T;
    const int R = NWR - (TY - 1) * T;  // filter rows
    // lane t: tile t's window rows, stream base and position shift
    const int lo = lane * TYT - P;
    const int r0 = lo < 0 ? 0 : (lo > H ? H : lo), r1 = (lo + NWR < H) ? (lo + NWR < 0 ? 0 : lo + NWR) : H;
    const unsigned shift_t = (unsigned)(lo * W);  // code = flat index - i_lo*W
    uint2* st_t = entries + ((int64_t)n * tiles + (lane < tiles ? lane : 0)) * cap;
    {
        // Lanes over the plane's list entries: entry k (row i) goes to every tile whose window
        // holds row i, at that tile's marker index + 1 + (k - first list entry of the window);
        // lanes over tiles write the markers.  Plane lists: row i of an entry from its flat
        // index through a float reciprocal (exact: the quotient's fraction stays >= 0.5/W from
        // an integer).  Row slots (FROM_ROWS): row i = the last row whose prefix is <= k (a
        // five-step shuffle search), the entry at slot k - prefix(i) of that row.
        // Lane r < H: the first tile whose window holds row r, and the last.
        const int num = lane + P - NWR;
        const int tl_r = num < 0 ? 0 : num / TYT + 1;
        const int th_r0 = (lane + P) / TYT;
        const int th_r = th_r0 < tiles - 1 ? th_r0 : tiles - 1;
        const int span = (NWR + TYT - 1) / TYT;  // tiles holding one row, at most
        const float invW = 1.0f / (float)W;
#pragma unroll
        for (int q = 0; q < kPerWarp; ++q) {
            const int ch = warp + q * kPlaneWarps;
            if (ch >= nch) break;
            const int plane = n * C + c0 + ch;
            const uint2* lst = plist + (int64_t)plane * HW;
            const uint32_t pre = pv[q];
            const uint32_t a = __shfl_sync(0xffffffffu, pre, r0), b = __shfl_sync(0xffffffffu, pre, r1);
            const uint32_t cnt_t = (lane < tiles && r1 > r0) ? b - a : 0u;
            const uint32_t pos_t = lane < tiles ? start_s[lane][ch] : 0u;
            const uint32_t pnext = __shfl_down_sync(0xffffffffu, pre, 1);
            const unsigned rowbits = __ballot_sync(0xffffffffu, lane < H && pnext > pre);
            unsigned mask_t = 0;
            const uint64_t rb64 = (uint64_t)rowbits << 32;
            for (int ty = 0; ty < TY; ++ty) {
                const int sh = 32 + lo + ty * T;
                if (sh < 64) mask_t |= (unsigned)(rb64 >> sh);
            }
            mask_t &= (1u << R) - 1u;
            if (cnt_t > 0) st_t[pos_t] = make_uint2((unsigned)(c0 + ch), (unsigned)NWIN + mask_t);
            const uint32_t total = __shfl_sync(0xffffffffu, pre, H);
            for (uint32_t k0 = 0; k0 < total; k0 += 32) {
                const uint32_t k = k0 + lane;
                const bool live = k < total;
                uint2 e = en0[q];
                int i = 0;
                if constexpr (FROM_ROWS) {
#pragma unroll
                    for (int st = 16; st > 0; st >>= 1) {  // last row i < H with prefix(i) <= k
                        const uint32_t pv_s = __shfl_sync(0xffffffffu, pre, (i + st) & 31);
                        if (i + st < H && pv_s <= k) i += st;
                    }
                    const uint32_t pr = __shfl_sync(0xffffffffu, pre, i);
                    if (live) e = __ldg(plist + ((int64_t)plane * H + i) * W + (k - pr));
                } else {
                    if (k0 > 0 && live) e = __ldg(lst + k);
                    i = live ? __float2int_rz(((float)e.y + 0.5f) * invW) : 0;
                }
                const int tl = __shfl_sync(0xffffffffu, tl_r, i);
                const int th = __shfl_sync(0xffffffffu, th_r, i);
                for (int j = 0; j < span; ++j) {
                    const int t = tl + j <= th ? tl + j : th;  // every lane takes part in the shuffles
                    const uint32_t at = __shfl_sync(0xffffffffu, a, t);
                    const uint32_t pt = __shfl_sync(0xffffffffu, pos_t, t);
                    const unsigned sh = __shfl_sync(0xffffffffu, shift_t, t);
                    if (live && tl + j <= th)
                        entries[((int64_t)n * tiles + t) * cap + pt + 1 + (k - at)] = make_uint2(e.x, e.y - sh);
                }
            }
        }
    }
}

cudaError_t launch_plane_lists(const Geometry& g, int64_t n, const float* in, uint32_t* cnt, uint2* plist,
                               uint32_t* prow, cudaStream_t st, Gate gate) {
    if (!compact_uses_counts(g) || cnt == nullptr || plist == nullptr || prow == nullptr)
        return cudaErrorNotSupported;
    const int TYT = (int)(g.ty * g.T);
    // images in the grid's y dimension (the kernel loops over the rest); under the device-side gate
    // (forward_auto) a quarter as many CTAs, so a skipped launch is cheap
    const int64_t ymax = gate.flag ? 32 : 65535;
    const int64_t slots0 = (g.H * g.W + 31) / 32;
    const int img = slots0 <= 8 ? 2 : 1;  // planes of <= 256 elements: two images per warp iteration
    const int64_t ny = (n + img - 1) / img;
    const dim3 cgrid((unsigned)((g.C + kPlaneWarps - 1) / kPlaneWarps), (unsigned)(ny < ymax ? ny : ymax));
    // the smallest instantiated slot count covering the plane (loads of 32 elements)
    const int64_t slots = (g.H * g.W + 31) / 32;
#define SC_COUNT(NS)                                                                                             \
    compact_plane_count_kernel<NS, (NS <= 8 ? 2 : 1)><<<cgrid, kPlaneWarps * 32, 0, st>>>(in, (int)n, (int)g.C, (int)g.H, (int)g.W,  \
                                                                       TYT, (int)g.P, (int)g.nwr, (int)g.tiles,   \
                                                                       cnt, plist, prow, gate)
    if (slots <= 2) SC_COUNT(2);
    else if (slots <= 4) SC_COUNT(4);
    else if (slots <= 6) SC_COUNT(6);
    else if (slots <= 8) SC_COUNT(8);
    else if (slots <= 16) SC_COUNT(16);
    else if (slots <= 25) SC_COUNT(25);
    else SC_COUNT(kMaxSlots);
#undef SC_COUNT
    return cudaGetLastError();
}

// Channels per emit CTA: 32 (measured best on C2: 1024 CTAs), 16 when 32 would leave fewer
// than four CTAs per SM (C4a / C3: 384 -> 768 CTAs, compaction 31 -> 30 and 32 -> 30 us).
// ... and 8 channels when 16 would leave fewer than two CTAs per SM (few channels per image: C1, C4b)
static int emit_chunk(const Geometry& g, int64_t n) {
    if (n * ((g.C + 31) / 32) >= 4 * 148) return 32;
    return n * ((g.C + 15) / 16) >= 2 * 148 ? 16 : 8;
}

cudaError_t launch_compact(const Geometry& g, int64_t n, const float* in, uint32_t* cnt, uint2* plist,
                           uint32_t* prow, uint2* entries, uint32_t* offs, cudaStream_t st, Gate gate) {
    if (!compact_uses_counts(g) || cnt == nullptr || plist == nullptr || prow == nullptr)
        return launch_compact_streamwise(g, n, in, entries, offs, st, gate);
    cudaError_t e = launch_plane_lists(g, n, in, cnt, plist, prow, st, gate);
    if (e != cudaSuccess) return e;
    const int ch = emit_chunk(g, n);
    const int chunks = (int)((g.C + ch - 1) / ch);
    // a programmatic dependent of the count kernel: its launch and CTA placement overlap the
    // count kernel's last wave
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n * chunks));
    cfg.blockDim = dim3(kPlaneWarps * 32);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const uint2* cplist = plist;
    const uint32_t* cprow = prow;
    const uint32_t* ccnt = cnt;
    if (ch == 8)
        return cudaLaunchKernelEx(&cfg, compact_plane_emit_kernel<false, 8>, cplist, cprow, ccnt, (int)g.C, (int)g.H,
                                  (int)g.W, (int)g.ty, (int)g.T, (int)g.P, (int)g.nwr, (int)g.nwin, (int)g.tiles, g.cap,
                                  chunks, entries, offs, gate);
    if (ch == 32)
        return cudaLaunchKernelEx(&cfg, compact_plane_emit_kernel<false, 32>, cplist, cprow, ccnt, (int)g.C, (int)g.H,
                                  (int)g.W, (int)g.ty, (int)g.T, (int)g.P, (int)g.nwr, (int)g.nwin, (int)g.tiles, g.cap,
                                  chunks, entries, offs, gate);
    return cudaLaunchKernelEx(&cfg, compact_plane_emit_kernel<false, 16>, cplist, cprow, ccnt, (int)g.C, (int)g.H,
                              (int)g.W, (int)g.ty, (int)g.T, (int)g.P, (int)g.nwr, (int)g.nwin, (int)g.tiles, g.cap,
                              chunks, entries, offs, gate);
}

// cnt[n][t][c] = row counts summed over tile t's window rows (chained consumers)
__global__ void compact_rows_tilecount_kernel(const uint32_t* __restrict__ rcnt, int64_t planes, int C, int H,
                                              int TYT, int P, int NWR, int tiles, uint32_t* __restrict__ cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= planes * tiles) return;
    const int64_t plane = i / tiles;
    const int t = (int)(i - plane * tiles);
    const int lo = t * TYT - P;
    const int r0 = lo < 0 ? 0 : lo, r1 = (lo + NWR < H) ? lo + NWR : H;
    uint32_t acc = 0;
    for (int r = r0; r < r1; ++r) acc += __ldg(rcnt + plane * H + r);
    const int64_t n = plane / C;
    cnt[(n * tiles + t) * C + (plane - n * C)] = acc;
}

cudaError_t launch_compact_from_rows(const Geometry& g, int64_t n, uint32_t* cnt, const uint2* rows,
                                     const uint32_t* rcnt, uint2* entries, uint32_t* offs, cudaStream_t st) {
    if (!compact_uses_counts(g)) return cudaErrorNotSupported;
    const int TYT = (int)(g.ty * g.T);
    const int64_t planes = n * g.C;
    compact_rows_tilecount_kernel<<<(unsigned)((planes * g.tiles + 255) / 256), 256, 0, st>>>(
        rcnt, planes, (int)g.C, (int)g.H, TYT, (int)g.P, (int)g.nwr, (int)g.tiles, cnt);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int ch = emit_chunk(g, n);
    const int chunks = (int)((g.C + ch - 1) / ch);
    auto kern = ch == 32 ? compact_plane_emit_kernel<true, 32>
                         : (ch == 16 ? compact_plane_emit_kernel<true, 16> : compact_plane_emit_kernel<true, 8>);
    kern<<<(unsigned)(n * chunks), kPlaneWarps * 32, 0, st>>>(
        rows, rcnt, cnt, (int)g.C, (int)g.H, (int)g.W, (int)g.ty, (int)g.T, (int)g.P, (int)g.nwr, (int)g.nwin,
        (int)g.tiles, g.cap, chunks, entries, offs, Gate{});
    return cudaGetLastError();
}

bool compact_uses_counts(const Geometry& g) {
    return g.H * g.W <= 32 * kMaxSlots && g.tiles <= kMaxTiles && g.H <= 31;
}

}  // namespace sc
