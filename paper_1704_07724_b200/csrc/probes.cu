// Bench utilities: FP32 FMA-pipe probes (roofline denominator evidence) and
// an L2 flush.  Not on the hot path.
//
// The sparse path is bound by FP32 fused multiply-adds on the CUDA cores
// (SURVEY 8d).  Its nominal peak is 148 SMs x 128 FMA/clk x f_max.  These
// probes measure what one SM actually retires per SM clock for
//   kind 0: FFMA  Rd, Ra, Rb, Rc                (1 FMA per lane)
//   kind 1: FFMA2 Rd, Ra.F32x2, Rb.F32, Rc.F32x2 (2 FMAs per lane, scalar bcast)
//   kind 2: kind 1 with ~2 independent ALU-pipe integer ops per FFMA2
// using clock64() around an unrolled loop of independent accumulator chains
// (one CTA of 1024 threads per SM, so every SMSP has 8 warps).
#include "sc_internal.h"

namespace sc {

constexpr int kProbeIters = 4096;

__global__ void __launch_bounds__(1024, 1) probe_ffma_kernel(const float* __restrict__ src, float* dst,
                                                             long long* cycles) {
    float a = src[0], b = src[1];
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = src[2 + i] + threadIdx.x;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < kProbeIters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
    }
    __syncthreads();
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    dst[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <bool kWithInt>
__global__ void __launch_bounds__(1024, 1) probe_ffma2_kernel(const float* __restrict__ src, float* dst,
                                                              long long* cycles) {
    const float v = src[0];
    const float2 vv = make_float2(v, v);
    float2 w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = make_float2(src[2 + 2 * i], src[3 + 2 * i]);
    float2 acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = make_float2(src[1] + threadIdx.x, src[1] - i);
    unsigned ic[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ic[i] = threadIdx.x + 77u * i;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < kProbeIters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            acc[i] = __ffma2_rn(w[i & 3], vv, acc[i]);
            if (kWithInt) ic[i & 7] = (ic[i & 7] ^ (ic[i & 7] >> 3)) + 0x9e37u;  // 8 independent ALU chains
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i].x + acc[i].y;
    if (kWithInt) {
        unsigned u = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) u ^= ic[i];
        s += (float)(u & 1u);
    }
    dst[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

cudaError_t probe_fma(int kind, double* rate) {
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* src = nullptr;
    float* dst = nullptr;
    long long* cyc = nullptr;
    if ((e = cudaMalloc(&src, 64 * sizeof(float))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&dst, (size_t)sms * 1024 * sizeof(float))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&cyc, (size_t)sms * sizeof(long long))) != cudaSuccess) return e;
    float h[64];
    for (int i = 0; i < 64; ++i) h[i] = 1.0f + 1e-7f * i;
    h[0] = 0.999999f;
    cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
    double fma_per_thread = 0;
    for (int rep = 0; rep < 2; ++rep) {  // first launch warms up the clocks
        if (kind == 0) {
            probe_ffma_kernel<<<sms, 1024>>>(src, dst, cyc);
            fma_per_thread = 16.0 * kProbeIters;
        } else if (kind == 1) {
            probe_ffma2_kernel<false><<<sms, 1024>>>(src, dst, cyc);
            fma_per_thread = 32.0 * kProbeIters;
        } else {
            probe_ffma2_kernel<true><<<sms, 1024>>>(src, dst, cyc);
            fma_per_thread = 32.0 * kProbeIters;
        }
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) break;
    }
    if (e == cudaSuccess) {
        long long* hc = new long long[sms];
        cudaMemcpy(hc, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < sms; ++i) mx = hc[i] > mx ? hc[i] : mx;
        delete[] hc;
        *rate = fma_per_thread * 1024.0 / (double)mx;
    }
    cudaFree(src);
    cudaFree(dst);
    cudaFree(cyc);
    return e == cudaSuccess ? cudaGetLastError() : e;
}

__global__ void flush_kernel(int4* p, size_t n16, int salt) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_int4(salt, (int)i, salt, (int)i);
}

cudaError_t launch_flush(void* scratch, size_t bytes, cudaStream_t st) {
    static int salt = 0;
    flush_kernel<<<148 * 8, 512, 0, st>>>((int4*)scratch, bytes / 16, ++salt);
    return cudaGetLastError();
}

}  // namespace sc
