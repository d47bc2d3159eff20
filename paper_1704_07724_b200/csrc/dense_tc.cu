// Dense comparison path: the GEMM-mapped convolution of PAPER.md:109-117
// (Fig. 2, M_K x M_I = M_O) as an implicit GEMM on the 5th-generation tensor
// cores (tcgen05.mma kind::tf32, fp32 accumulation in TMEM).
//
//   D[m][p] = sum_kk A[m][kk] * B[kk][p] + bias[m]
//   m  = output channel within group g          (M_K rows, "matrix of kernels")
//   kk = (cl, r, t) flattened = cl*R*S + r*S + t (the R*S*C axis of Fig. 2)
//   p  = (n, y, x) flattened output pixel        (M_I columns; never materialised)
//   B[kk][p] = in[n][g*Cg + cl][y*T + r - P][x*T + t - P]  (0 outside: padding)
//
// Tiles: BM = 128 filters (UMMA M), BN = 128 pixels (UMMA N), BK = 32 (one
// 128-byte swizzle row of TF32).  Operands are K-major, SWIZZLE_128B.
//  * A: pre-packed at plan creation into the exact swizzled shared-memory image
//    of every (g, m-tile, k-block) and rounded to TF32 (cvt.rna); one 16 KB
//    1-D TMA bulk copy per stage (warp 9).
//  * B: im2col on the fly by 8 producer warps: each thread owns one pixel row
//    and four 16-byte chunks per stage, loads 16 input values (coalesced
//    across the warp = consecutive pixels), rounds to TF32 (cvt.rna), stores
//    swizzled with STS.128, fence.proxy.async, arrives on the stage's mbarrier.
//  * MMA: warp 8, one thread: 4 x tcgen05.mma (K=8) per stage, tcgen05.commit
//    frees the stage; the last commit signals the epilogue.
//  * Epilogue: warps 0-3 read their 32 TMEM lanes (tcgen05.ld 32x32b.x32),
//    transpose through shared memory and store pixel-contiguous runs + bias
//    (+ optional ReLU, Eq. 2).
#include "sc_internal.h"

namespace sc {
namespace dense {

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 4;
constexpr int kProducerWarps = 8, kMmaWarp = 8, kALoadWarp = 9, kThreads = 320;
constexpr int kTileBytes = BM * BK * 4;  // 16 KB for A and for B
constexpr uint32_t kTmemCols = 128;

struct Args {
    const float* in;
    const float* adense;  // [G][mtiles][kblocks][128*32] swizzled TF32 image
    const int2* ktab;     // [kblocks*32]: (cl*H*W + r*W + t, r<<16 | t), r = 0x7fff for padding kk
    const float* bias;
    float* out;
    int C, H, W, K, Kg, Cg, T, P, Ho, Wo, HoWo, relu;
    int mtiles, ntiles, kblocks;
    long long ptotal;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05 format):
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major: 1), SBO>>4
// [32,46) = 1024 B between 8-row groups, version 1 [46,48), layout 2 [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
           ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}
// Instruction descriptor: D f32 [4,6)=1, A tf32 [7,10)=2, B tf32 [10,13)=2,
// both K-major, N>>3 at [17,23), M>>4 at [24,29).
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__global__ void __launch_bounds__(kThreads, 1) dense_tc_kernel(const Args a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the swizzle atoms
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    float* sA = reinterpret_cast<float*>(smem);                          // STAGES x 16 KB
    float* sB = reinterpret_cast<float*>(smem + STAGES * kTileBytes);    // STAGES x 16 KB
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * STAGES * kTileBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
    float* epi = reinterpret_cast<float*>(smem + 2 * STAGES * kTileBytes + 256);  // 4 warps x 32 x 33

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int bid = blockIdx.x;
    const int nt = bid % a.ntiles;
    bid /= a.ntiles;
    const int mt = bid % a.mtiles;
    const int g = bid / a.mtiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], kProducerWarps + 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int nk = a.kblocks;

    if (warp < kProducerWarps) {
        // ---- B producers: one pixel row per thread, chunks {c0, c0+2, c0+4, c0+6} ----
        const int t = threadIdx.x;
        const int row = t & (BN - 1);
        const int c0 = t >> 7;  // 0 or 1
        const long long p = (long long)nt * BN + row;
        const bool pvalid = p < a.ptotal;
        int n = 0, y = 0, x = 0;
        if (pvalid) {
            n = (int)(p / a.HoWo);
            const int pix = (int)(p - (long long)n * a.HoWo);
            y = pix / a.Wo;
            x = pix - y * a.Wo;
        }
        const int yb = y * a.T - a.P, xb = x * a.T - a.P;
        const float* pin = a.in + ((long long)n * a.C + (long long)g * a.Cg) * a.H * a.W + (long long)yb * a.W + xb;
        const int swz = row & 7;
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % STAGES;
            mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
            float* dst = sB + s * (kTileBytes / 4) + row * BK;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int ch = c0 + 2 * i;
                float v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int2 e = __ldg(&a.ktab[kb * BK + ch * 4 + q]);
                    const int r = e.y >> 16, tt = e.y & 0xffff;
                    const bool ok = pvalid && (unsigned)(yb + r) < (unsigned)a.H && (unsigned)(xb + tt) < (unsigned)a.W;
                    v[q] = ok ? to_tf32(__ldg(pin + e.x)) : 0.f;
                }
                *reinterpret_cast<float4*>(dst + ((ch ^ swz) << 2)) = make_float4(v[0], v[1], v[2], v[3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
        }
    } else if (warp == kALoadWarp) {
        if (lane == 0) {
            const float* asrc = a.adense + ((long long)g * a.mtiles + mt) * nk * (kTileBytes / 4);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
                mbar_expect_tx(&full[s], kTileBytes);
                tma_bulk_g2s(sA + s * (kTileBytes / 4), asrc + (long long)kb * (kTileBytes / 4), kTileBytes, &full[s]);
            }
        }
    } else if (warp == kMmaWarp) {
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % STAGES;
            mbar_wait(&full[s], (kb / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
                const uint32_t abase = smem_u32(sA + s * (kTileBytes / 4));
                const uint32_t bbase = smem_u32(sB + s * (kTileBytes / 4));
#pragma unroll
                for (int k = 0; k < BK / 8; ++k) {
                    const uint64_t ad = sw128_desc(abase + k * 32);
                    const uint64_t bd = sw128_desc(bbase + k * 32);
                    const uint32_t acc = (kb | k) ? 1u : 0u;
                    asm volatile(
                        "{\n\t.reg .pred p;\n\t"
                        "setp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                        "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc)
                        : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&empty[s]))
                             : "memory");
            }
            __syncwarp();
        }
        if (lane == 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(tmem_full))
                         : "memory");
        __syncwarp();
    }

    // ---- epilogue: warps 0-3 own TMEM lanes 32w..32w+31 (= output channels) ----
    if (warp < 4) {
        mbar_wait(tmem_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float* buf = epi + warp * 32 * 33;
        const int m0 = mt * BM + warp * 32;
        for (int c0 = 0; c0 < BN; c0 += 32) {
            uint32_t r[32];
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                  "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                  "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j) buf[lane * 33 + j] = __uint_as_float(r[j]);  // [m][pixel]
            __syncwarp();
            const long long p = (long long)nt * BN + c0 + lane;
            if (p < a.ptotal) {
                const int n = (int)(p / a.HoWo);
                const int pix = (int)(p - (long long)n * a.HoWo);
                float* dst = a.out + ((long long)n * a.K + (long long)g * a.Kg) * a.HoWo + pix;
#pragma unroll 4
                for (int mm = 0; mm < 32; ++mm) {
                    const int m = m0 + mm;
                    if (m < a.Kg) {
                        float o = buf[mm * 33 + lane] + __ldg(&a.bias[g * a.Kg + m]);
                        if (a.relu) o = fmaxf(o, 0.f);
                        dst[(long long)m * a.HoWo] = o;
                    }
                }
            }
            __syncwarp();
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

// Pack A: adense[g][mt][kb][row][32] in the K-major SWIZZLE_128B image:
// element (row, k) at row*32 + ((k/4) ^ (row%8))*4 + k%4, value
// tf32_rna(W[g*Kg + mt*128 + row][kk = kb*32 + k]) or 0 outside.
__global__ void pack_dense_kernel(const float* __restrict__ w, float* __restrict__ adense, int2* __restrict__ ktab,
                                  int G, int Kg, int mtiles, int kblocks, int kdim, int RS, int S, int H, int W) {
    const long long total = (long long)G * mtiles * kblocks * BM * BK;
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
         o += (long long)gridDim.x * blockDim.x) {
        const int within = (int)(o % (BM * BK));
        long long rest = o / (BM * BK);
        const int kb = (int)(rest % kblocks);
        rest /= kblocks;
        const int mt = (int)(rest % mtiles);
        const int g = (int)(rest / mtiles);
        const int row = within / BK, slot = within % BK;
        const int chunk = (slot >> 2) ^ (row & 7);  // stored chunk -> logical chunk
        const int k = chunk * 4 + (slot & 3);
        const int m = mt * BM + row, kk = kb * BK + k;
        float v = 0.f;
        if (m < Kg && kk < kdim) v = to_tf32(w[((long long)g * Kg + m) * kdim + kk]);
        adense[o] = v;
    }
    // im2col gather table (index metadata, same for every group)
    for (int kk = blockIdx.x * blockDim.x + threadIdx.x; kk < kblocks * BK; kk += gridDim.x * blockDim.x) {
        if (kk < kdim) {
            const int cl = kk / RS, rs = kk - cl * RS, r = rs / S, t = rs - r * S;
            ktab[kk] = make_int2(cl * H * W + r * W + t, (r << 16) | t);
        } else {
            ktab[kk] = make_int2(0, 0x7fff << 16);
        }
    }
}

}  // namespace dense

cudaError_t launch_pack_dense(const Geometry& g, const DenseGeom& dg, const float* w, float* wdense,
                              cudaStream_t st) {
    using namespace dense;
    const int mtiles = (int)(dg.m_pad / BM), kblocks = (int)(dg.kdim_pad / BK);
    int2* ktab = reinterpret_cast<int2*>(wdense + g.G * dg.m_pad * dg.kdim_pad);
    pack_dense_kernel<<<512, 256, 0, st>>>(w, wdense, ktab, (int)g.G, (int)g.Kg, mtiles, kblocks, (int)dg.kdim,
                                            (int)(g.R * g.S), (int)g.S, (int)g.H, (int)g.W);
    return cudaGetLastError();
}

size_t dense_workspace_floats(const Geometry& g, const DenseGeom& dg) {
    return (size_t)(g.G * dg.m_pad * dg.kdim_pad + 2 * dg.kdim_pad);
}

cudaError_t launch_dense_tc(const Geometry& g, const DenseGeom& dg, int64_t n, const float* in, const float* wdense,
                            const float* bias, float* out, cudaStream_t st) {
    using namespace dense;
    Args a;
    a.in = in;
    a.adense = wdense;
    a.ktab = reinterpret_cast<const int2*>(wdense + g.G * dg.m_pad * dg.kdim_pad);
    a.bias = bias;
    a.out = out;
    a.C = (int)g.C; a.H = (int)g.H; a.W = (int)g.W; a.K = (int)g.K; a.Kg = (int)g.Kg; a.Cg = (int)g.Cg;
    a.T = (int)g.T; a.P = (int)g.P; a.Ho = (int)g.Ho; a.Wo = (int)g.Wo; a.HoWo = (int)(g.Ho * g.Wo);
    a.relu = g.relu ? 1 : 0;
    a.mtiles = (int)(dg.m_pad / BM);
    a.kblocks = (int)(dg.kdim_pad / BK);
    a.ptotal = (long long)n * g.Ho * g.Wo;
    a.ntiles = (int)((a.ptotal + BN - 1) / BN);
    const size_t smem = 1024 + 2 * STAGES * kTileBytes + 256 + 4 * 32 * 33 * 4;
    cudaError_t e = cudaFuncSetAttribute(dense_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long grid = (long long)a.ntiles * a.mtiles * g.G;
    dense_tc_kernel<<<(unsigned)grid, kThreads, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace sc
