// Internal declarations shared by the translation units of libsparseconv.so.
// Nothing here is visible through include/sparse_conv.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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

// Dense tcgen05 path operand geometry.
struct DenseGeom {
    int64_t kdim;        // Cg*R*S
    int64_t kdim_pad;    // rounded up to 32 (one 128-byte TF32 row)
    int64_t m_pad;       // Kg rounded up to 128 (UMMA M)
};

// ---- kernels (launchers return cudaGetLastError()) -------------------------
cudaError_t launch_pack_weights(const Geometry& g, const float* w, float* wpack, cudaStream_t st);
cudaError_t launch_pack_dense(const Geometry& g, const DenseGeom& dg, const float* w, float* wdense,
                              cudaStream_t st);
// Stage 1.  The plane-major path (compact_uses_counts) needs workspaces
// cnt [N][tiles][C] u32, plist [N*C][H*W] (bits, index) pairs and
// prow [N*C][H+1] u32; they may be null otherwise.
bool compact_uses_counts(const Geometry& g);
cudaError_t launch_compact(const Geometry& g, int64_t n, const float* in, uint32_t* cnt, uint2* plist,
                           uint32_t* prow, uint2* entries, uint32_t* offs, cudaStream_t st);
cudaError_t launch_gather_generic(const Geometry& g, int64_t n, const uint2* entries, const uint32_t* offs,
                                  const float* wpack, const float* bias, float* out, cudaStream_t st);

// Shape-specialised stage-2 kernels (gather_fast.cu).  `select` returns a
// variant id > 0 (and its lanes-per-channel KL and tile height TY) if one
// applies to the geometry, else 0.
int gather_fast_select(const Geometry& g, int force, const char** name, int* kl, int* ty);
cudaError_t launch_gather_fast(int variant, const Geometry& g, int64_t n, const uint2* entries,
                               const uint32_t* offs, const float* wpack, const float* bias, float* out,
                               cudaStream_t st);

// Dense tcgen05 TF32 implicit GEMM (dense_tc.cu).
cudaError_t launch_dense_tc(const Geometry& g, const DenseGeom& dg, int64_t n, const float* in,
                            const float* wdense, const float* bias, float* out, cudaStream_t st);

cudaError_t probe_fma(int kind, double* rate);
cudaError_t launch_flush(void* scratch, size_t bytes, cudaStream_t st);

}  // namespace sc
