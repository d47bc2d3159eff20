// Microbenchmark: global(L2-resident) -> shared copy throughput per SM on B200 for the
// mechanisms the kernels use to stream operands: 1-D bulk copies (cp.async.bulk, one
// thread, mbarrier completion) with 1..8 copies of a stage in flight and 1..4 stages
// outstanding, against LDGSTS (cp.async.cg 16 B by every lane of 1 or 4 warps).
// Question: the gather at s = 0.99 and the backward kernels both move ~32 GB/s
// per SM of bulk copies -- is that a per-SM limit of the copy engine?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_bench bulk_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: bulk copies: `stages` stage buffers of `stage_bytes`, each filled by `parts` bulk copies,
//         all stages kept in flight (refill a stage as soon as it landed)
// mode 1: LDGSTS 16 B per lane by `warps` warps, `stages` commit groups in flight
__global__ void __launch_bounds__(128, 1) k(const char* __restrict__ src, size_t src_bytes, int mode, int stage_bytes,
                                            int parts, int stages, int iters, int warps, unsigned long long* out) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t base = ((size_t)blockIdx.x * 7919 * stage_bytes) % (src_bytes - (size_t)stage_bytes * 64);
    if (threadIdx.x == 0)
        for (int s = 0; s < 8; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    unsigned long long t0 = clock64();
    if (mode == 0) {
        if (threadIdx.x == 0) {
            auto issue = [&](int it) {
                const int s = it % stages;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                             "r"(stage_bytes));
                const int part = stage_bytes / parts;
                const char* g = src + base + (size_t)(it % 64) * stage_bytes;
                for (int p = 0; p < parts; ++p)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(sm + (size_t)s * stage_bytes + p * part)),
                        "l"(g + p * part), "r"(part), "r"(smem_u32(&bar[s]))
                        : "memory");
            };
            for (int it = 0; it < stages && it < iters; ++it) issue(it);
            for (int it = 0; it < iters; ++it) {
                const int s = it % stages;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                        smem_u32(&bar[s])),
                    "r"((unsigned)(it / stages) & 1u)
                    : "memory");
                if (it + stages < iters) issue(it + stages);
            }
        }
    } else if (warp < warps) {
        const int nthr = warps * 32, tid = threadIdx.x;
        for (int it = 0; it < iters; ++it) {
            const int s = it % stages;
            const char* g = src + base + (size_t)(it % 64) * stage_bytes;
            for (int off = tid * 16; off < stage_bytes; off += nthr * 16)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + (size_t)s * stage_bytes + off)),
                             "l"(g + off)
                             : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
            if (it >= stages - 1) asm volatile("cp.async.wait_group %0;" ::"n"(3) : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
    const size_t S = 64ull << 20;  // 64 MB source (L2-resident after the warm-up)
    char* src;
    unsigned long long* out;
    cudaMalloc(&src, S);
    cudaMemset(src, 1, S);
    cudaMalloc(&out, 148 * sizeof(unsigned long long));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    struct Cfg { int mode, stage_kb, parts, stages, warps; };
    const Cfg cfgs[] = {{0, 64, 1, 2, 1}, {0, 64, 4, 2, 1}, {0, 64, 8, 2, 1}, {0, 32, 1, 4, 1}, {0, 32, 4, 4, 1},
                        {0, 16, 1, 8, 1}, {0, 16, 2, 8, 1}, {0, 8, 1, 8, 1},  {0, 72, 4, 2, 1}, {0, 86, 8, 2, 1},
                        {1, 16, 1, 4, 1}, {1, 16, 1, 4, 4}, {1, 32, 1, 4, 4}, {1, 8, 1, 4, 4}};
    for (const Cfg& c : cfgs) {
        const int sb = c.stage_kb * 1024 / 16 * 16;
        const int iters = (int)((64ll << 20) / sb / 4);  // ~16 MB per SM
        const size_t smem = (size_t)sb * c.stages;
        if (smem > 200 * 1024) continue;
        k<<<148, 128, smem>>>(src, S, c.mode, sb, c.parts, c.stages, 8, c.warps, out);
        cudaEventRecord(a);
        k<<<148, 128, smem>>>(src, S, c.mode, sb, c.parts, c.stages, iters, c.warps, out);
        cudaEventRecord(b);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = 148.0 * iters * sb, cyc = ms * 1e-3 * clk * 1e3;
        printf("%-6s stage=%3d KB parts=%d stages=%d warps=%d: %.3f ms  %.2f TB/s total  %.1f B/clk/SM\n",
               c.mode ? "LDGSTS" : "bulk", c.stage_kb, c.parts, c.stages, c.warps, ms, bytes / (ms * 1e-3) / 1e12,
               bytes / 148 / cyc);
    }
    return 0;
}
