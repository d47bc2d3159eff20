// Stage 2, shape-specialised: output-stationary sparse-gather convolution
// with the output tile in registers (template; one .cu per variant).
//
// Computes, for stride 1 (ISC steps 2-3; Eq. 1 P:68-72 with the
// zero terms skipped):
//   out[n,k,y,x] = bias[k] + sum_{c in group, nonzero in[n,c,i,j]} in * W[k,c,i+P-y,j+P-x]
//
// Mapping:
//  * CTA = NW warps sharing one (group g, k-block kb of KBW = 32*KL output
//    channels).  The packed weight slice wpack[g][kb][c0:c0+CH][R][S][KBW] of
//    CH input channels is ONE contiguous run, streamed through a STAGES-deep
//    shared-memory ring by 1-D TMA bulk copies (cp.async.bulk + mbarrier
//    complete_tx) issued by a dedicated producer warp (warp NW), which refills
//    a stage once all active compute warps released it (no compute warp ever
//    waits for another except through the ring depth).
//  * warp = one unit = one stage-1 tile stream (image n, output rows
//    [y0, y0+TY)); lane owns KL output channels (the paper's "4 floats of
//    weights ... at one time", becomes 32*KL per warp).  The warp's
//    tile acc[TY][NX] (f32x2 pairs) stays in registers for the whole
//    reduction over input channels.
//  * the unit's stream (per channel: marker, then in-window nonzeros as
//    (value, window position)) is cut into pieces at weight-chunk boundaries
//    and every V::PIECE entries; each piece is bulk-copied (TMA, per-warp
//    mbarrier) into a V::SLOTS-deep per-warp shared ring, terminated with an EXIT
//    entry and run by the generated threaded interpreter (tools/gen_gather.py):
//    one brx.idx.uni per entry into code that applies FFMA2/FFMA to exactly the
//    accumulators the entry reaches; markers reload the lane's weights.
//  * epilogue (ISC step 3, "transpose temporary results"): registers ->
//    per-warp shared buffer [k][pixels] -> contiguous NCHW runs, + bias,
//    optional ReLU (Eq. 2).  One global write per output, no atomics;
//    accumulation order (channel, entry) is fixed -> deterministic.
#pragma once
#include "sc_internal.h"

namespace sc {
namespace fast {

#include "gather_variants.inc"

}  // namespace fast
}  // namespace sc

#include "gather_fast_kernel.cuh"

namespace sc {
namespace fast {

inline int sm_count() {
    static const int sms = [] {
        int d = 0, v = 148;
        if (cudaGetDevice(&d) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess)
            v = 148;
        return v;
    }();
    return sms;
}

template <class V>
cudaError_t launch_v(const Geometry& g, int64_t n, const uint2* entries, const uint32_t* offs, const float* wpack,
                     const float* bias, float* out, uint2* rowlist, uint32_t* rowcnt, cudaStream_t st, Gate gate) {
    if (g.ty != V::TY || g.tiles != (g.Ho + V::TY - 1) / V::TY || (g.Cg + V::CH - 1) / V::CH > 63)
        return cudaErrorInvalidValue;
    ArgsGated ag;
    Args& a = ag;
    a.entries = entries; a.offs = offs; a.wpack = wpack; a.bias = bias; a.out = out;
    a.rowlist = rowlist; a.rowcnt = rowcnt;
    ag.gate = gate;
    a.n = (int)n; a.C = (int)g.C; a.H = (int)g.H; a.K = (int)g.K; a.Cg = (int)g.Cg; a.Kg = (int)g.Kg;
    a.kblocks = (int)g.kblocks; a.Ho = (int)g.Ho; a.relu = g.relu ? 1 : 0;
    a.cap = g.cap;
    a.ytiles = (int)g.tiles;
    a.units = (int)n * a.ytiles;
    a.ctas_per_kb = (a.units + V::NW - 1) / V::NW;
    const size_t smem = Smem<V>::total;
    auto kern = gather_fast_kernel<V, false>;
    if (rowlist != nullptr) {
        if constexpr (V::XPAIR) {
            return cudaErrorNotSupported;
        } else {
            kern = gather_fast_kernel<V, true>;
        }
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = (int64_t)a.ctas_per_kb * g.G * g.kblocks;
    a.edge_last = edge_last_order(grid >= 2LL * sm_count() * V::MINB);
    if (gate.flag != nullptr) {
        if (rowlist != nullptr) return cudaErrorNotSupported;
        auto kg = gather_fast_kernel<V, false, ArgsGated>;
        e = cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        kg<<<(unsigned)grid, (V::NW + 1) * 32, smem, st>>>(ag);
        return cudaGetLastError();
    }
    // launched as a programmatic dependent of stage 1 (the emit kernel releases it early)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((V::NW + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace fast
}  // namespace sc

// Each gather_fast_vN.cu instantiates one variant (parallel compilation).
#define SC_INSTANTIATE_VARIANT(VV)                                                                          \
    namespace sc {                                                                                          \
    namespace fast {                                                                                        \
    cudaError_t launch_##VV(const Geometry& g, int64_t n, const uint2* entries, const uint32_t* offs,       \
                            const float* wpack, const float* bias, float* out, uint2* rowlist,              \
                            uint32_t* rowcnt, cudaStream_t st, Gate gate) {                                 \
        return launch_v<VV>(g, n, entries, offs, wpack, bias, out, rowlist, rowcnt, st, gate);              \
    }                                                                                                       \
    }                                                                                                       \
    }
