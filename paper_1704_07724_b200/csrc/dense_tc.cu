// Dense tcgen05 TF32 implicit-GEMM convolution (filled in below).
#include "sc_internal.h"

namespace sc {

cudaError_t launch_pack_dense(const Geometry&, const DenseGeom&, const float*, float*, cudaStream_t) {
    return cudaSuccess;
}

cudaError_t launch_dense_tc(const Geometry&, const DenseGeom&, int64_t, const float*, const float*, const float*,
                            float*, cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace sc
