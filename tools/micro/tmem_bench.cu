// Microbenchmark: TMEM load throughput (tcgen05.ld.32x32b) vs shared-memory LDS.128,
// alone and concurrently, per SM (B200).  Question: can the
// stage-2 weight operands come from TMEM so that they stop competing with the
// shared-memory port?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tmem_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

#define LD16(t, r)                                                                                          \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                   "=r"(r[15])                                                                              \
                 : "r"(t))

// mode 0: TMEM only, 1: LDS only, 2: half the warps TMEM, half LDS, 3: every warp both
__global__ void __launch_bounds__(512, 1) k(int mode, int iters, int nwarps, float* out) {
    __shared__ unsigned slot;
    __shared__ __align__(16) float sm[8192];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = (float)i;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tbase = slot + ((unsigned)(32 * (warp & 3)) << 16);
    float acc = 0.f;
    if (warp < nwarps) {
        const bool do_t = mode == 0 || mode == 3 || (mode == 2 && (warp & 4) == 0);
        const bool do_s = mode == 1 || mode == 3 || (mode == 2 && (warp & 4) != 0);
        const unsigned sbase = smem_u32(sm) + lane * 16;
        for (int it = 0; it < iters; ++it) {
            unsigned r[4][16];
            float4 s[8];
            if (do_t) {
#pragma unroll
                for (int j = 0; j < 4; ++j) LD16(tbase + (unsigned)(((it * 4 + j) * 16 + warp * 64) & 511), r[j]);
            }
            if (do_s) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const unsigned a = sbase + (unsigned)((((it * 8 + j) * 512) + warp * 2048) & 32767);
                    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                                 : "=f"(s[j].x), "=f"(s[j].y), "=f"(s[j].z), "=f"(s[j].w)
                                 : "r"(a));
                }
            }
            if (do_t) {
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int q = 0; q < 16; ++q) acc += __uint_as_float(r[j][q]);
            }
            if (do_s) {
#pragma unroll
                for (int j = 0; j < 8; ++j) acc += s[j].x + s[j].y + s[j].z + s[j].w;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    float* o;
    cudaMalloc(&o, 148 * 512 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 4096;
    const char* names[] = {"tmem", "lds", "half/half", "both"};
    for (int mode = 0; mode < 4; ++mode)
        for (int nw : {4, 8, 12, 16}) {
            k<<<148, 512>>>(mode, 16, nw, o);
            cudaEventRecord(a);
            k<<<148, 512>>>(mode, iters, nw, o);
            cudaEventRecord(b);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double cyc = ms * 1e-3 * clk * 1e3;
            int nt = 0, ns = 0;
            for (int w = 0; w < nw; ++w) {
                const bool t = mode == 0 || mode == 3 || (mode == 2 && (w & 4) == 0);
                const bool s = mode == 1 || mode == 3 || (mode == 2 && (w & 4) != 0);
                nt += t; ns += s;
            }
            const double tb = (double)nt * iters * 4 * 16 * 32 * 4, sb = (double)ns * iters * 8 * 512;
            printf("%-9s warps=%2d  %.3f ms  TMEM %.1f B/clk/SM  LDS %.1f B/clk/SM  total %.1f\n", names[mode], nw, ms,
                   tb / cyc, sb / cyc, (tb + sb) / cyc);
        }
    return 0;
}
