// Weight packing, run once per plan (not on the hot path).
//
// ISC step 2: "the kernel matrix is stored as column-major
// matrix such that for each non-zero element of inputs, a continious memory
// that stores kernels (say 4 floats of weights: W_{k..k+3,c,i-r,j-s}) can be
// fetched".  On the GPU the contiguous run over k is a warp's 32 lanes:
//
//   wpack[g][cl][r][t][kk] = W[g*Kg + kk][cl][r][t]   (kk < Kg; zero for kk in [Kg, Kg_pad))
//
// so lane kk of a warp reads consecutive 4-byte words (conflict-free shared
// memory, coalesced global memory).
#include "sc_internal.h"

namespace sc {

__global__ void pack_weights_kernel(const float* __restrict__ w, float* __restrict__ wpack,
                                    int64_t G, int64_t Kg, int64_t Kg_pad, int64_t Cg, int64_t RS) {
    const int64_t total = G * Cg * RS * Kg_pad;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t kk = o % Kg_pad;
        const int64_t rest = o / Kg_pad;          // ((g*Cg + cl)*RS + rs)
        const int64_t rs = rest % RS;
        const int64_t gcl = rest / RS;
        const int64_t cl = gcl % Cg;
        const int64_t g = gcl / Cg;
        float v = 0.0f;
        if (kk < Kg) v = w[((g * Kg + kk) * Cg + cl) * RS + rs];
        wpack[o] = v;
    }
}

cudaError_t launch_pack_weights(const Geometry& g, const float* w, float* wpack, cudaStream_t st) {
    const int64_t total = g.G * g.Cg * g.R * g.S * g.Kg_pad;
    const int threads = 256;
    const int64_t blocks = (total + threads - 1) / threads;
    pack_weights_kernel<<<(unsigned)(blocks < 65535 * 16 ? blocks : 65535 * 16), threads, 0, st>>>(
        w, wpack, g.G, g.Kg, g.Kg_pad, g.Cg, g.R * g.S);
    return cudaGetLastError();
}

}  // namespace sc
