"""Microbenchmark: cost of one brx.idx.uni dispatch (LDS entry -> LDC -> BRX ->
case with F FFMA2 -> BRA) vs warps per SMSP and number of cases.
Writes brx_bench.cu (standalone, nvcc -o brx_bench brx_bench.cu)."""
import sys

def kernel(ncases, f):
    nacc = 16
    lines = []
    asm = ["{", ".reg .b64 vv;", ".reg .b32 xc, cc, xn, cn, ep;", "mov.b32 ep, %17;",
           "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;", "LOOP_%=:", "mov.b32 xc, xn;", "mov.b32 cc, cn;",
           "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;", "mov.b64 vv, {xc, xc};"]
    labels = [f"C{i}_%=" for i in range(ncases)] + ["END_%="]
    asm.append("TS_%=: .branchtargets " + ", ".join(labels) + ";")
    asm.append("brx.idx.uni cc, TS_%=;")
    for i in range(ncases):
        asm.append(f"C{i}_%=:")
        for q in range(f):
            a = (i * 3 + q * 5) % nacc
            asm.append(f"fma.rn.f32x2 %{a}, %16, vv, %{a};")
        asm.append("bra.uni LOOP_%=;")
    asm.append("END_%=:")
    asm.append("}")
    body = "\\n\\t".join(asm)
    outs = ", ".join(f'"+l"(acc[{i}])' for i in range(nacc))
    return f'''
extern "C" __global__ void __launch_bounds__(1024, 1) k_{ncases}_{f}(const uint2* __restrict__ g_ent, int n, long long* cyc, float* out, int nwarps_active) {{
  extern __shared__ uint2 ent[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < n + 1; i += blockDim.x) ent[i] = g_ent[i];
  __syncthreads();
  if (warp >= nwarps_active) return;
  unsigned long long acc[{nacc}];
  for (int i = 0; i < {nacc}; ++i) acc[i] = 0ull;
  unsigned long long w = 0x3f8000003f800000ull + lane;
  unsigned s = (unsigned)__cvta_generic_to_shared(ent);
  long long t0 = clock64();
  asm volatile("{body}" : {outs} : "l"(w), "r"(s) : "memory");
  long long t1 = clock64();
  float r = 0; for (int i = 0; i < {nacc}; ++i) r += __uint_as_float((unsigned)acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
}}
'''

def main():
    configs = [(16, 3), (64, 3), (128, 3), (256, 3), (512, 3), (128, 9), (128, 1)]
    src = ['#include <cstdio>', '#include <cstdlib>', '#include <cstdint>', '#include <vector>', '#include <cuda_runtime.h>']
    for nc, f in configs:
        src.append(kernel(nc, f))
    src.append('''
typedef void (*kfn)(const uint2*, int, long long*, float*, int);
int main() {
  const int n = 4096;
  uint2* d_ent; long long* d_cyc; float* d_out;
  cudaMalloc(&d_ent, (n + 1) * 8); cudaMalloc(&d_cyc, 148 * 32 * 8); cudaMalloc(&d_out, 148 * 1024 * 4);
  struct C { int nc, f; kfn k; } cs[] = {''' + ", ".join(f"{{{nc}, {f}, k_{nc}_{f}}}" for nc, f in configs) + '''};
  for (auto& c : cs) {
    std::vector<uint2> h(n + 1);
    srand(1);
    for (int i = 0; i < n; ++i) h[i] = make_uint2(0x3f800000u, (unsigned)(rand() % c.nc));
    h[n] = make_uint2(0, (unsigned)c.nc);
    cudaMemcpy(d_ent, h.data(), (n + 1) * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(c.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 1) * 8);
    for (int wps : {1, 2, 3, 4, 6, 8}) {
      int nw = wps * 4;
      c.k<<<148, 1024, (n + 1) * 8>>>(d_ent, n, d_cyc, d_out, nw);
      c.k<<<148, 1024, (n + 1) * 8>>>(d_ent, n, d_cyc, d_out, nw);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\\n", cudaGetErrorString(e)); return 1; }
      std::vector<long long> cy(148 * 32);
      cudaMemcpy(cy.data(), d_cyc, cy.size() * 8, cudaMemcpyDeviceToHost);
      double mx = 0; for (int i = 0; i < nw; ++i) mx = cy[i] > mx ? cy[i] : mx;
      printf("cases=%4d ffma2/case=%d warps/SMSP=%d  cycles/dispatch/warp=%.1f  per-SMSP=%.1f\\n", c.nc, c.f, wps, mx / n, mx / n / wps);
    }
  }
  return 0;
}
''')
    open(sys.argv[1] if len(sys.argv) > 1 else "brx_bench.cu", "w").write("\n".join(src))

main()
