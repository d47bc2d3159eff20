// Device-side declarations shared by the library's kernels and by the kernels
// compiled at run time through NVRTC (jit.cu): no host headers.
#pragma once
#ifdef __CUDACC_RTC__
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned long size_t;
#else
#include <stddef.h>
#include <stdint.h>
#endif

namespace sc {

// Device-side path selection: a kernel launched with a gate
// returns at once unless *flag == run_if (flag null: always runs).  Lets the
// sparse and the dense path both be enqueued (graph-capturable) while only the
// one chosen on the device from the batch's measured density does work.
struct Gate {
    const int* flag = nullptr;
    int run_if = 0;
};
__device__ __forceinline__ bool gate_closed(const Gate& g) { return g.flag != nullptr && *g.flag != g.run_if; }

}  // namespace sc
