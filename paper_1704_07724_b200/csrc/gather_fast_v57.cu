// Variant V57 of the register-tile gather kernel (see gather_fast_impl.cuh).
#include "gather_fast_impl.cuh"
SC_INSTANTIATE_VARIANT(V57)
