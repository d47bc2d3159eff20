// Variant V51 of the register-tile gather kernel (see gather_fast_impl.cuh).
#include "gather_fast_impl.cuh"
SC_INSTANTIATE_VARIANT(V51)
