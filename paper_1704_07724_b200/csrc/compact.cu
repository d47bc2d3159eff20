// Stage 1 of the sparse path: on-the-fly nonzero compaction.
//
// ISC step 1: "we skip all the zero elements of the input data,
// and store the non-zero values in a vector with their column and row
// information".  List format: reading R9 (include/sparse_conv.h).
//
// Design: one warp per list.  A list is a contiguous
// segment [start, start+len) of the flat NCHW array (TH whole rows of one
// plane), generally not 16-byte aligned (e.g. 13x13 planes are 676 B).  The
// warp reads the 16-byte-aligned float4s that cover the segment with
// ld.global.nc.L1::no_allocate.v4 (LDG.E.128), masks the head/tail, and ranks
// the nonzeros in scan order with four __ballot_sync + __popc per chunk.  All
// of a short list's chunks are loaded before any is ranked, so every warp keeps
// up to three 16-byte loads in flight.  The kernel is HBM-bound: it reads the
// input once and writes nnz*(4 + idx) bytes plus one u32 count per list.
#include "sc_internal.h"

namespace sc {

__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}

template <typename IdxT>
__device__ __forceinline__ void rank_and_store(const float4 v, int64_t e0, int64_t start, int64_t end,
                                               unsigned lane, uint32_t& base, float* __restrict__ vals,
                                               IdxT* __restrict__ idx) {
    const float q[4] = {v.x, v.y, v.z, v.w};
    bool nz[4];
    unsigned before = 0, total = 0;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t e = e0 + j;
        nz[j] = (e >= start) && (e < end) && (q[j] != 0.0f);   // IEEE: -0.0 is zero
        const unsigned b = __ballot_sync(0xffffffffu, nz[j]);
        before += __popc(b & lt);
        total += __popc(b);
    }
    uint32_t rank = base + before;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (nz[j]) {
            vals[rank] = q[j];
            idx[rank] = (IdxT)(e0 + j - start);
            ++rank;
        }
    }
    base += total;
}

__device__ __forceinline__ float4 load_chunk(const float* __restrict__ in, int64_t e0, int64_t end,
                                             int64_t total_elems) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e0 < end) {
        if (e0 + 3 < total_elems) {
            v = ld_stream_f4(in + e0);
        } else {  // the very end of the tensor: scalar loads inside bounds only
            v.x = in[e0];
            if (e0 + 1 < total_elems) v.y = in[e0 + 1];
            if (e0 + 2 < total_elems) v.z = in[e0 + 2];
        }
    }
    return v;
}

// MAXC > 0: lists span at most MAXC 128-float chunks (TH*W <= 256 -> 3);
// MAXC == 0: generic loop for long rows (u16 indices).
template <typename IdxT, int MAXC>
__global__ void __launch_bounds__(256) compact_kernel(const float* __restrict__ in, int64_t num_lists,
                                                      int64_t tiles, int64_t H, int64_t W, int64_t TH,
                                                      int64_t cap, int64_t total_elems,
                                                      float* __restrict__ values, IdxT* __restrict__ idx,
                                                      uint32_t* __restrict__ counts) {
    const unsigned lane = threadIdx.x & 31u;
    const int64_t list = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (list >= num_lists) return;
    const int64_t plane = list / tiles, tile = list - plane * tiles;
    const int64_t row0 = tile * TH;
    const int64_t rows = (H - row0 < TH) ? (H - row0) : TH;
    const int64_t start = plane * H * W + row0 * W;
    const int64_t end = start + rows * W;
    const int64_t a0 = start & ~(int64_t)3;
    float* vals = values + list * cap;
    IdxT* ids = idx + list * cap;
    uint32_t base = 0;
    if constexpr (MAXC > 0) {
        float4 v[MAXC];
#pragma unroll
        for (int ch = 0; ch < MAXC; ++ch)
            v[ch] = load_chunk(in, a0 + ch * 128 + 4 * lane, end, total_elems);
#pragma unroll
        for (int ch = 0; ch < MAXC; ++ch) {
            if (a0 + ch * 128 < end)  // warp-uniform
                rank_and_store<IdxT>(v[ch], a0 + ch * 128 + 4 * lane, start, end, lane, base, vals, ids);
        }
    } else {
        for (int64_t b = a0; b < end; b += 128) {
            const float4 v = load_chunk(in, b + 4 * lane, end, total_elems);
            rank_and_store<IdxT>(v, b + 4 * lane, start, end, lane, base, vals, ids);
        }
    }
    if (lane == 0) counts[list] = base;
}

cudaError_t launch_compact(const Geometry& g, int64_t n, const float* in, float* values, void* idx,
                           uint32_t* counts, cudaStream_t st) {
    const int64_t num_lists = n * g.C * g.tiles;
    const int threads = 256, wpb = threads / 32;
    const int64_t blocks = (num_lists + wpb - 1) / wpb;
    const int64_t total = n * g.C * g.H * g.W;
    const bool short_lists = g.th * g.W <= 256;
    if (g.idx_bytes == 1) {
        compact_kernel<uint8_t, 3><<<(unsigned)blocks, threads, 0, st>>>(
            in, num_lists, g.tiles, g.H, g.W, g.th, g.cap, total, values, (uint8_t*)idx, counts);
    } else if (short_lists) {
        compact_kernel<uint16_t, 3><<<(unsigned)blocks, threads, 0, st>>>(
            in, num_lists, g.tiles, g.H, g.W, g.th, g.cap, total, values, (uint16_t*)idx, counts);
    } else {
        compact_kernel<uint16_t, 0><<<(unsigned)blocks, threads, 0, st>>>(
            in, num_lists, g.tiles, g.H, g.W, g.th, g.cap, total, values, (uint16_t*)idx, counts);
    }
    return cudaGetLastError();
}

}  // namespace sc
