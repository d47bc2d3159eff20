// Device-side sparse <-> dense path selection (the paper's
// regime "speedup ... when the sparsity is not less than 0.9").
//
// select_path_kernel counts the nonzeros of the batch's input (one HBM pass,
// float4 loads, ballot + popc per warp, one atomic per block) and the last
// block to finish writes the path flag: dense iff nnz > thr (thr = the largest
// nonzero count the sparse path is chosen for).  The last block also resets
// the counters, so the launch is re-entrant under CUDA-graph replay.  The flag
// gates the two paths' kernels (sc::Gate), all of which are enqueued: no host
// synchronisation.
//
// synth_relu_kernel writes the calibration input: element i is nonzero with
// probability rho (counter-based hash of (i, seed)), value in (0, 1].
#include <cuda_runtime.h>

#include "sc_internal.h"

namespace sc {

namespace {
constexpr int kSelThreads = 256;

__device__ __forceinline__ uint32_t mix32(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return (uint32_t)x;
}
}  // namespace

__global__ void __launch_bounds__(kSelThreads) select_path_kernel(const float* __restrict__ in, int64_t elems,
                                                                  unsigned long long thr,
                                                                  unsigned long long* __restrict__ sel) {
    // sel[0] = nnz accumulator, sel[1] = finished-block ticket, ((int*)(sel + 2))[0] = path
    __shared__ unsigned wsum[kSelThreads / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n4 = elems >> 2;
    const float4* in4 = reinterpret_cast<const float4*>(in);
    unsigned cnt = 0;
    const int64_t step = (int64_t)gridDim.x * kSelThreads;
    int64_t i = (int64_t)blockIdx.x * kSelThreads + threadIdx.x;
    for (; i + 3 * step < n4; i += 4 * step) {  // four independent 16-byte loads in flight per thread
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(in4 + i + u * step);
#pragma unroll
        for (int u = 0; u < 4; ++u) cnt += (v[u].x != 0.f) + (v[u].y != 0.f) + (v[u].z != 0.f) + (v[u].w != 0.f);
    }
    for (; i < n4; i += step) {
        const float4 v = __ldcs(in4 + i);
        cnt += (v.x != 0.f) + (v.y != 0.f) + (v.z != 0.f) + (v.w != 0.f);
    }
    if (blockIdx.x == 0 && threadIdx.x < (elems & 3)) cnt += in[(n4 << 2) + threadIdx.x] != 0.f;
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) wsum[warp] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < kSelThreads / 32; ++w) s += wsum[w];
        atomicAdd(sel, s);
        __threadfence();
        last = atomicAdd(sel + 1, 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        const unsigned long long nnz = atomicExch(sel, 0ull);
        sel[1] = 0;
        reinterpret_cast<int*>(sel + 2)[0] = nnz > thr ? kPathDense : kPathSparse;
        reinterpret_cast<unsigned long long*>(sel + 3)[0] = nnz;
    }
}

__global__ void synth_relu_kernel(float* __restrict__ x, int64_t elems, uint64_t thr, uint32_t seed) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < elems; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t h = mix32(((uint64_t)seed << 40) ^ (uint64_t)i);
        const uint32_t v = mix32((uint64_t)i * 0x9e3779b97f4a7c15ull + seed);
        x[i] = (uint64_t)h < thr ? (float)((v >> 8) + 1) * (1.0f / 16777216.0f) : 0.f;
    }
}

cudaError_t launch_select_path(const float* in, int64_t elems, unsigned long long thr, unsigned long long* sel,
                               cudaStream_t st) {
    int64_t blocks = (elems / 4 + kSelThreads - 1) / kSelThreads;
    if (blocks > 148 * 4) blocks = 148 * 4;
    if (blocks < 1) blocks = 1;
    select_path_kernel<<<(unsigned)blocks, kSelThreads, 0, st>>>(in, elems, thr, sel);
    return cudaGetLastError();
}

cudaError_t launch_synth_relu(float* x, int64_t elems, double rho, uint32_t seed, cudaStream_t st) {
    const double t = rho <= 0 ? 0.0 : rho >= 1 ? 4294967296.0 : rho * 4294967296.0;
    synth_relu_kernel<<<148 * 4, 256, 0, st>>>(x, elems, (uint64_t)t, seed);
    return cudaGetLastError();
}

}  // namespace sc
