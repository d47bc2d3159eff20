// Stage 2 dispatch: pick the shape-specialised register-tile kernel
// (gather_fast_impl.cuh; one translation unit per variant, gather_fast_vN.cu).
#include "sc_internal.h"

namespace sc {
namespace fast {
#include "gather_variants.inc"
template <class V>
bool matches(const Geometry& g) {
    return g.T == V::T && g.R == V::R && g.S == V::S && g.P == V::P && g.W == V::W && g.Wo == V::WO && g.Cg >= 1 &&
           (g.Cg + V::CH - 1) / V::CH <= 63 && g.Kg >= V::KMIN && (V::KMIN == 0 || V::KL == wide_1x1_kl(g));
}
#define SC_DECLARE(VV)                                                                                  \
    cudaError_t launch_##VV(const Geometry& g, int64_t n, const uint2* entries, const uint32_t* offs,   \
                            const float* wpack, const float* bias, float* out, uint2* rowlist,          \
                            uint32_t* rowcnt, cudaStream_t st, Gate gate);
SC_GATHER_VARIANTS(SC_DECLARE)
#undef SC_DECLARE
}  // namespace fast

// force < 0: first matching variant; force == 0: generic; force > 0: that
// variant if it matches the geometry (else generic).
int gather_fast_select(const Geometry& g, int force, const char** name, int* kl, int* ty) {
    using namespace fast;
    *kl = 1;
    *ty = (int)g.Ho;
    if (force == 0) return 0;
#define SC_SELECT(VV)                                       \
    if (matches<VV>(g) && (force < 0 || force == VV::ID)) { \
        if (name) *name = VV::NAME;                         \
        *kl = VV::KL;                                       \
        *ty = VV::TY;                                       \
        return VV::ID;                                      \
    }
    SC_GATHER_VARIANTS(SC_SELECT)
#undef SC_SELECT
    return 0;
}

bool gather_fast_can_emit(int variant) {
    using namespace fast;
#define SC_CAN(VV) \
    if (variant == VV::ID) return !VV::XPAIR;
    SC_GATHER_VARIANTS(SC_CAN)
#undef SC_CAN
    return false;
}

cudaError_t launch_gather_fast(int variant, const Geometry& g, int64_t n, const uint2* entries, const uint32_t* offs,
                               const float* wpack, const float* bias, float* out, uint2* rowlist, uint32_t* rowcnt,
                               cudaStream_t st, Gate gate) {
    using namespace fast;
#define SC_LAUNCH(VV) \
    if (variant == VV::ID) return launch_##VV(g, n, entries, offs, wpack, bias, out, rowlist, rowcnt, st, gate);
    SC_GATHER_VARIANTS(SC_LAUNCH)
#undef SC_LAUNCH
    return cudaErrorInvalidValue;
}

}  // namespace sc
