// Internal declarations shared by the translation units of libsparseconv.so.
// Nothing here is visible through include/sparse_conv.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>

#include "sc_device.h"
#include "sparse_conv.h"

namespace sc {

// Geometry derived once at plan creation.
struct Geometry {
    int64_t N, C, H, W, K, R, S, T, P, G;
    int64_t Ho, Wo, Cg, Kg;
    int64_t kbw;            // k-block width of the packed weights: 32 * KL of the stage-2 kernel
    int64_t Kg_pad;         // Kg rounded up to kbw
    int64_t kblocks;        // Kg_pad / kbw
    // stage-1 tile streams (reading R9): row-tile height, tiles per image,
    // window rows / positions, capacity (entries) of one stream
    int64_t ty, tiles, nwr, nwin, cap;
    bool relu;
};

// 1x1 convolutions at stride 1 with Kg >= 150 filters: no
// halo, so one-row tiles, and a nonzero costs one interpreter dispatch per k-block of 32*KL
// filters -- KL = the fewest k-blocks among 4, 6, 8 (ties to the narrower) whose one-row tile
// (Wo*KL accumulators + KL weights) fits V21's 140 registers.  0: not such a layer.  Both the
// shipped variants V53-V56 (gather_fast.cu) and run-time generated tilings (jit.cu) follow it.
// Stage-2 unit order (gather_fast_kernel.cuh): interior row tiles first, edge tiles last, so a
// CTA's warps hold streams of similar length.  Round 1 used it for grids of >= 2 waves only
// (single-batch C2, 1.66 waves: +1%); with batches pipelined (sparse_conv_forward_batches) the
// last wave's holes are filled anyway and the balance inside CTAs wins on every grid: C2 158.2 ->
// 152.0 us per batch, C4b 23.5 -> 22.4 (profiles/r2_edge_last_pipelined.txt).  SC_EDGE_LAST
// (measurement knob): 0 = grids of >= 2 waves only, as in round 1.
inline int edge_last_order(bool multi_wave) {
    static const int force = [] {
        const char* v = getenv("SC_EDGE_LAST");
        return v ? atoi(v) : 1;
    }();
    return force ? 1 : (multi_wave ? 1 : 0);
}

inline int wide_1x1_kl(const Geometry& g) {
    if (g.R != 1 || g.S != 1 || g.T != 1 || g.Kg < 150) return 0;
    auto blocks = [&](int64_t k) { return (g.Kg + 32 * k - 1) / (32 * k); };
    int kl = 4;
    for (int k : {6, 8})
        if (blocks(k) < blocks(kl) && g.Wo * k + k <= 140) kl = k;
    return kl;
}

// Dense tcgen05 path geometry (dense_tc.cu): channels-last input with Cp = G*Cgp
// channels (each group's Cg padded to a multiple of 4); K-dim blocks of 32 channels per tap (cb per group); tiles
// of `rows` whole output rows (npix = rows*Wo pixels, UMMA N = nmma).
struct DenseGeom {
    int64_t cp, cgp, cb, kblocks, mtiles, rows, ptiles, npix, nmma;  // cp = G * cgp, cgp = Cg rounded up to 4
    bool supported;
};

// Backward kernels (backward.cu): KC = 32*kl output channels
// per warp pass, kchunks per group, cblocks of 16 channels; per kernel ([0] wgrad,
// [1] dgrad) bands of `by` output rows, two band buffers of buf_floats, smem bytes;
// image splits for wgrad / dgrad; doutT_floats of workspace for the k-contiguous dout.
struct BwdGeom {
    int64_t kl, kc, kchunks, cblocks, splits_w, splits_d, doutT_floats;
    int64_t by[2], bands[2], buf_floats[2], nbuf[2];
    size_t smem[2];
    bool direct;  // dgrad: one k-chunk and one band, sums stored straight to dz (no dz planes)
    bool supported;
};

// ---- kernels (launchers return cudaGetLastError()) -------------------------
cudaError_t launch_pack_weights(const Geometry& g, const float* w, float* wpack, cudaStream_t st);
void dense_geometry(const Geometry& g, DenseGeom* dg);
size_t dense_workspace_floats(const Geometry& g, const DenseGeom& dg);  // packed A
cudaError_t launch_pack_dense(const Geometry& g, const DenseGeom& dg, const float* w, float* wdense,
                              cudaStream_t st);
// Encode the 4-D TMA map (128 bytes) of the plan's NHWC input buffer.
cudaError_t encode_dense_input_map(const Geometry& g, const DenseGeom& dg, float* nhwc, void* map128);
// Stage 1.  The plane-major path (compact_uses_counts) needs workspaces
// cnt [N][tiles][C] u32, plist [N*C][H*W] (bits, index) pairs and
// prow [N*C][H+1] u32; they may be null otherwise.
bool compact_uses_counts(const Geometry& g);
cudaError_t launch_compact(const Geometry& g, int64_t n, const float* in, uint32_t* cnt, uint2* plist,
                           uint32_t* prow, uint2* entries, uint32_t* offs, cudaStream_t st, Gate gate = {});
// Only the plane lists plist/prow (and tile counts cnt) of the plane-major path;
// cudaErrorNotSupported unless compact_uses_counts(g).
cudaError_t launch_plane_lists(const Geometry& g, int64_t n, const float* in, uint32_t* cnt, uint2* plist,
                               uint32_t* prow, cudaStream_t st, Gate gate = {});
// Stage 1 of a chained consumer (f1): the producing gather wrote per-(plane, row)
// lists `rows` [N*C*H][W] and counts `rcnt` [N*C*H]; builds the same R9 streams.
cudaError_t launch_compact_from_rows(const Geometry& g, int64_t n, uint32_t* cnt, const uint2* rows,
                                     const uint32_t* rcnt, uint2* entries, uint32_t* offs, cudaStream_t st);
cudaError_t launch_gather_generic(const Geometry& g, int64_t n, const uint2* entries, const uint32_t* offs,
                                  const float* wpack, const float* bias, float* out, cudaStream_t st,
                                  Gate gate = {});

// Shape-specialised stage-2 kernels (gather_fast.cu).  `select` returns a
// variant id > 0 (and its lanes-per-channel KL and tile height TY) if one
// applies to the geometry, else 0.
int gather_fast_select(const Geometry& g, int force, const char** name, int* kl, int* ty);
bool gather_fast_can_emit(int variant);  // the variant can emit chained lists (KL >= 2)
// rowlist/rowcnt non-null: also emit the next layer's per-(plane,row) lists (f1; KL >= 2 variants);
// out may then be null.  cudaErrorNotSupported if the variant cannot emit.
cudaError_t launch_gather_fast(int variant, const Geometry& g, int64_t n, const uint2* entries,
                               const uint32_t* offs, const float* wpack, const float* bias, float* out,
                               uint2* rowlist, uint32_t* rowcnt, cudaStream_t st, Gate gate = {});

// Dense tcgen05 TF32 implicit GEMM (dense_tc.cu).
cudaError_t launch_dense_tc(const Geometry& g, const DenseGeom& dg, int64_t n, const float* in, float* nhwc,
                            const void* map128, const float* wdense, const float* bias, float* out, cudaStream_t st,
                            Gate gate = {});

// f3 path selection (select.cu).  sel: 4 x u64 device words (nnz, ticket,
// path flag, last nnz), zero-initialised; the kernel leaves nnz/ticket at 0.
constexpr int kPathSparse = 0;
constexpr int kPathDense = 1;
cudaError_t launch_select_path(const float* in, int64_t elems, unsigned long long thr, unsigned long long* sel,
                               cudaStream_t st);
cudaError_t launch_synth_relu(float* x, int64_t elems, double rho, uint32_t seed, cudaStream_t st);

// Backward (backward.cu).  ws: [splits_w][K][Cg][R][S] floats; doutT: b.doutT_floats
// (rewritten by every call).  dw/dbias/dz nullable.
void backward_geometry(const Geometry& g, BwdGeom* b);
cudaError_t launch_backward(const Geometry& g, const BwdGeom& b, int64_t n, const uint2* plist, const uint32_t* prow,
                            const float* dout, const float* wpack, float* ws, float* doutT, float* dw, float* dbias,
                            float* dz, cudaStream_t st, cudaStream_t st2 = nullptr, cudaEvent_t ev_fork = nullptr,
                            cudaEvent_t ev_join = nullptr);

// Run-time specialised stage 2 (jit.cu): a gather variant generated for the plan's
// shape and compiled through NVRTC when no generated variant matches.
namespace jit {
struct Params {
    int R = 0, S = 0, P = 0, T = 1, W = 0, TY = 1, KL = 1, NW = 11, MINB = 1, CH = 16, STAGES = 2, SLOTS = 3,
        PIECE = 254, id = 1000;
};
bool available();                                 // NVRTC and the driver entry points are loadable
bool choose(const Geometry& g, Params* p);       // false: shape outside the generator's limits
// Why parameter set p cannot run shape g (nullptr: it can): generator, stream-format and
// kernel limits (checked for SC_JIT_FORCE sets and again at launch).
const char* invalid(const Geometry& g, const Params& p);
// Compile (cached per parameter set and device) the ungated and the gated kernel.
cudaError_t compile(const Params& p, int device, void** fn, void** fn_gated, size_t* smem);
cudaError_t launch(void* fn, size_t smem, const Params& p, const Geometry& g, int64_t n, const uint2* entries,
                   const uint32_t* offs, const float* wpack, const float* bias, float* out, cudaStream_t st,
                   Gate gate = {});
const char* last_log();
// Generated source of a variant (tests: must equal tools/gen_gather.py's); returns its length.
size_t variant_source(const Params& p, char* buf, size_t cap);
}  // namespace jit

cudaError_t probe_fma(int kind, double* rate);
cudaError_t launch_flush(void* scratch, size_t bytes, cudaStream_t st);

}  // namespace sc
