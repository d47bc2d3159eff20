// Weight packing, run once per plan (not on the hot path).
//
// ISC step 2: "the kernel matrix is stored as column-major
// matrix such that for each non-zero element of inputs, a continious memory
// that stores kernels (say 4 floats of weights: W_{k..k+3,c,i-r,j-s}) can be
// fetched".  On the GPU the contiguous run over k is a warp's 32 lanes:
//
//   wpack[g][kb][cl][r][t][j] = W[g*Kg + kbw*kb + jj(j)][cl][r][t]   (jj(j) = j for KL != 3)
//   (zero for kbw*kb + j >= Kg; kb < Kg_pad/kbw; kbw = 32*KL of the stage-2 kernel)
//
// so the lanes of a warp read consecutive 4-byte (KL=1) or 8-byte (KL=2)
// words (conflict-free shared memory, coalesced global memory), and the slice
// of CH consecutive input channels for one k-block is ONE contiguous run of
// CH*R*S*kbw*4 bytes -- a single 1-D TMA bulk copy (cp.async.bulk) in the
// gather kernel.
#include "sc_internal.h"

namespace sc {

__global__ void pack_weights_kernel(const float* __restrict__ w, float* __restrict__ wpack,
                                    int64_t G, int64_t Kg, int64_t Kg_pad, int64_t Cg, int64_t RS, int64_t kbw) {
    const int64_t total = G * Cg * RS * Kg_pad;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = o % kbw;
        int64_t rest = o / kbw;                   // ((g*kblocks + kb)*Cg + cl)*RS + rs
        const int64_t rs = rest % RS;
        rest /= RS;
        const int64_t cl = rest % Cg;
        rest /= Cg;
        const int64_t kblocks = Kg_pad / kbw;
        const int64_t kb = rest % kblocks;
        const int64_t g = rest / kblocks;
        // position j of a tap block -> channel offset within the k-block: lane l owns
        // channels KL*l .. KL*l+KL-1; KL=1,2,4 store them contiguously, KL=3 stores
        // the pair (3l, 3l+1) at 2l and the single 3l+2 at 64 + l (8- and 4-byte
        // shared loads without bank conflicts)
        int64_t jj = j;
        if (kbw == 96) jj = j < 64 ? 3 * (j / 2) + (j % 2) : 3 * (j - 64) + 2;
        const int64_t kk = kb * kbw + jj;
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
        w, wpack, g.G, g.Kg, g.Kg_pad, g.Cg, g.R * g.S, g.kbw);
    return cudaGetLastError();
}

}  // namespace sc
