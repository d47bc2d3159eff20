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
// Design: one CTA of 8 warps per stream.
//  pass 1: warp w counts the nonzeros of channels w, w+8, ... inside the
//          window (a contiguous run of the flat NCHW array, generally not
//          16-byte aligned: 16-byte-aligned LDG.128 over the covering float4s,
//          masked head/tail, __ballot_sync + __popc);
//  scan:   warp 0 turns the per-channel sizes (1 + count) into offsets
//          (shuffle scan), written to global;
//  pass 2: the same warps re-read their channels (L1/L2 hits) and write the
//          marker and the entries at their ranks.
// HBM traffic: the input once (+ the halo rows shared by neighbouring tiles)
// and 8 bytes per written entry.
#include "sc_internal.h"

namespace sc {

namespace {

__device__ __forceinline__ float4 ld_f4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// The covering float4 of element e0 (multiple of 4), zero outside [lo, hi)
// and beyond the tensor end.
__device__ __forceinline__ float4 load_chunk(const float* __restrict__ in, int64_t e0, int64_t hi, int64_t total) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e0 < hi) {
        if (e0 + 3 < total) {
            v = ld_f4(in + e0);
        } else {
            v.x = in[e0];
            if (e0 + 1 < total) v.y = in[e0 + 1];
            if (e0 + 2 < total) v.z = in[e0 + 2];
        }
    }
    return v;
}

__device__ __forceinline__ unsigned nz_mask(float4 v, int64_t e0, int64_t lo, int64_t hi) {
    const float q[4] = {v.x, v.y, v.z, v.w};
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (e0 + j >= lo && e0 + j < hi && q[j] != 0.0f) m |= 1u << j;  // IEEE: -0.0 is zero
    return m;
}

}  // namespace

__global__ void __launch_bounds__(256) compact_streams_kernel(const float* __restrict__ in, int C, int H, int W,
                                                              int TY, int tiles, int T, int P, int NWR, int NWIN,
                                                              int64_t cap, int64_t total,
                                                              uint2* __restrict__ entries,
                                                              uint32_t* __restrict__ offs) {
    extern __shared__ uint32_t cnt_s[];  // [C + 1]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int stream = blockIdx.x;
    const int n = stream / tiles, t = stream - n * tiles;
    const int i_lo = t * TY * T - P;
    const int r0 = i_lo < 0 ? 0 : i_lo;
    const int r1 = (i_lo + NWR < H) ? i_lo + NWR : H;
    const int64_t seg = r1 > r0 ? (int64_t)(r1 - r0) * W : 0;
    const unsigned lt = (1u << lane) - 1u;

    // ---- pass 1: per-channel window counts
    for (int c = warp; c < C; c += 8) {
        const int64_t plane = ((int64_t)n * C + c) * H * W;
        const int64_t lo = plane + (int64_t)r0 * W, hi = lo + seg;
        unsigned cnt = 0;
        for (int64_t b = lo & ~(int64_t)3; b < hi; b += 256) {  // two float4 per lane in flight
            const float4 v0 = load_chunk(in, b + 4 * lane, hi, total);
            const float4 v1 = load_chunk(in, b + 128 + 4 * lane, hi, total);
            cnt += __popc(nz_mask(v0, b + 4 * lane, lo, hi)) + __popc(nz_mask(v1, b + 128 + 4 * lane, lo, hi));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) cnt_s[c] = cnt;
    }
    __syncthreads();
    // ---- exclusive scan of (1 + count): marker + entries per channel
    if (warp == 0) {
        uint32_t running = 0;
        for (int base = 0; base < C; base += 32) {
            const int c = base + lane;
            const uint32_t v = c < C ? 1u + cnt_s[c] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            if (c < C) cnt_s[c] = running + incl - v;
            running += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) cnt_s[C] = running;
    }
    __syncthreads();
    uint32_t* of = offs + (int64_t)stream * (C + 1);
    for (int c = threadIdx.x; c <= C; c += blockDim.x) of[c] = cnt_s[c];
    // ---- pass 2: marker + entries
    uint2* st = entries + (int64_t)stream * cap;
    for (int c = warp; c < C; c += 8) {
        const int64_t plane = ((int64_t)n * C + c) * H * W;
        const int64_t lo = plane + (int64_t)r0 * W, hi = lo + seg;
        const int64_t code0 = plane + (int64_t)i_lo * W;  // code = e - code0 = (i - i_lo)*W + j
        uint32_t pos = cnt_s[c];
        if (lane == 0) st[pos] = make_uint2((unsigned)c, (unsigned)NWIN);
        ++pos;
        for (int64_t b = lo & ~(int64_t)3; b < hi; b += 128) {
            const int64_t e0 = b + 4 * lane;
            const float4 v = load_chunk(in, e0, hi, total);
            const unsigned m = nz_mask(v, e0, lo, hi);
            const float q[4] = {v.x, v.y, v.z, v.w};
            unsigned before = 0, tot = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const unsigned bal = __ballot_sync(0xffffffffu, (m >> j) & 1u);
                before += __popc(bal & lt);
                tot += __popc(bal);
            }
            uint32_t p = pos + before;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if ((m >> j) & 1u) {
                    st[p] = make_uint2(__float_as_uint(q[j]), (unsigned)(e0 + j - code0));
                    ++p;
                }
            }
            pos += tot;
        }
    }
}

cudaError_t launch_compact(const Geometry& g, int64_t n, const float* in, uint2* entries, uint32_t* offs,
                           cudaStream_t st) {
    const int64_t streams = n * g.tiles;
    const size_t smem = sizeof(uint32_t) * (g.C + 1);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(compact_streams_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    compact_streams_kernel<<<(unsigned)streams, 256, smem, st>>>(
        in, (int)g.C, (int)g.H, (int)g.W, (int)g.ty, (int)g.tiles, (int)g.T, (int)g.P, (int)g.nwr, (int)g.nwin,
        g.cap, n * g.C * g.H * g.W, entries, offs);
    return cudaGetLastError();
}

}  // namespace sc
