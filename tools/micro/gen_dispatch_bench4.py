"""Microbenchmark of per-entry dispatch mechanisms for the sparse-gather
interpreter (cycles per dispatch per SMSP vs warps per SMSP):
  brxuni : brx.idx.uni jump table (LDC + BRX)
  brx    : brx.idx (no .uni)
  tree   : binary tree of warp-uniform direct branches on the case index
Each case applies F FFMA2 to a 16-register accumulator set.
Usage: python gen_dispatch_bench.py out.cu && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o b out.cu"""
import sys

NACC = 16


def prologue():
    return ["{", ".reg .b64 vv;", ".reg .b32 xc, cc, xn, cn, ep;", ".reg .pred p;", "mov.b32 ep, %17;",
            "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;", "LOOP_%=:", "mov.b32 xc, xn;",
            "mov.b32 cc, cn;", "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;", "mov.b64 vv, {xc, xc};"]


def body_for(i, f):
    return [f"fma.rn.f32x2 %{(i * 3 + q * 5) % NACC}, %16, vv, %{(i * 3 + q * 5) % NACC};" for q in range(f)]


def asm_brx(nc, f, uni):
    a = prologue()
    labels = [f"C{i}_%=" for i in range(nc)] + ["END_%="]
    a.append("TS_%=: .branchtargets " + ", ".join(labels) + ";")
    a.append(("brx.idx.uni" if uni else "brx.idx") + " cc, TS_%=;")
    for i in range(nc):
        a.append(f"C{i}_%=:")
        a += body_for(i, f)
        a.append("bra.uni LOOP_%=;")
    a += ["END_%=:", "}"]
    return a


def asm_threaded(nc, f):
    """each case ends with the next entry's dispatch (no branch back to a loop head)"""
    a = ["{", ".reg .b64 vv;", ".reg .b32 xc, cc, xn, cn, ep;", "mov.b32 ep, %17;",
         "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;"]
    labels = [f"C{i}_%=" for i in range(nc)] + ["END_%="]
    a.append("TS_%=: .branchtargets " + ", ".join(labels) + ";")
    disp = ["mov.b32 xc, xn;", "mov.b32 cc, cn;", "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
            "mov.b64 vv, {xc, xc};", "brx.idx.uni cc, TS_%=;"]
    a += disp
    for i in range(nc):
        a.append(f"C{i}_%=:")
        a += body_for(i, f)
        a += disp
    a += ["END_%=:", "}"]
    return a


def asm_tree(nc, f):
    a = prologue() + [f"setp.ge.u32 p, cc, {nc};", "@p bra.uni END_%=;"]

    def tree(lo, hi, tag):
        if hi - lo == 1:
            return body_for(lo, f) + ["bra.uni LOOP_%=;"]
        mid = (lo + hi) // 2
        return ([f"setp.ge.u32 p, cc, {mid};", f"@p bra.uni R{tag}_%=;"] + tree(lo, mid, tag + "l") +
                [f"R{tag}_%=:"] + tree(mid, hi, tag + "r"))
    a += tree(0, nc, "x")
    a += ["END_%=:", "}"]
    return a


def kernel(name, asm):
    body = "\\n\\t".join(asm)
    outs = ", ".join(f'"+l"(acc[{i}])' for i in range(NACC))
    return f'''
extern "C" __global__ void __launch_bounds__(1024, 1) {name}(const uint2* __restrict__ g_ent, int n, long long* cyc,
                                                             float* out, int nwarps_active) {{
  extern __shared__ uint2 ent[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < n + 1; i += blockDim.x) ent[i] = g_ent[i];
  __syncthreads();
  if (warp >= nwarps_active) return;
  unsigned long long acc[{NACC}];
  for (int i = 0; i < {NACC}; ++i) acc[i] = 0ull;
  unsigned long long w = 0x3f8000003f800000ull + lane;
  unsigned s = (unsigned)__cvta_generic_to_shared(ent);
  long long t0 = clock64();
  asm volatile("{body}" : {outs} : "l"(w), "r"(s) : "memory");
  long long t1 = clock64();
  float r = 0; for (int i = 0; i < {NACC}; ++i) r += __uint_as_float((unsigned)acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
}}
'''


def main():
    cfgs = [(128, 3)]
    src = ["#include <cstdio>", "#include <cstdlib>", "#include <cstdint>", "#include <vector>",
           "#include <cuda_runtime.h>"]
    entries = []
    for nc, f in cfgs:
        for kind in ("brxuni", "shfl"):
            name = f"k_{kind}_{nc}_{f}"
            asm = asm_brx(nc, f, True)
            if kind == "shfl":
                asm = [x.replace("brx.idx.uni cc, TS_%=;", "shfl.sync.idx.b32 cc, cc, 0, 31, -1; brx.idx.uni cc, TS_%=;") for x in asm]
            src.append(kernel(name, asm))
            entries.append(f'{{{nc}, {f}, {name}, "{kind}"}}')
    src.append("typedef void (*kfn)(const uint2*, int, long long*, float*, int);")
    src.append("struct C { int nc, f; kfn k; const char* name; };")
    src.append("C cs[] = {" + ", ".join(entries) + "};")
    src.append(r'''
int main() {
  const int n = 4096;
  uint2* d_ent; long long* d_cyc; float* d_out;
  cudaMalloc(&d_ent, (n + 1) * 8); cudaMalloc(&d_cyc, 148 * 32 * 8); cudaMalloc(&d_out, 148 * 1024 * 4);
  for (int pat = 0; pat < 1; ++pat)
  for (auto& c : cs) {
    std::vector<uint2> h(n + 1);
    srand(1);
    const char* pn[] = {"random", "constant", "ascending", "runs-of-8"};
    for (int i = 0; i < n; ++i) {
      unsigned cs_ = pat == 0 ? rand() % c.nc : pat == 1 ? 5u : pat == 2 ? (unsigned)(i % c.nc) : (unsigned)((i / 8) * 37 % c.nc);
      h[i] = make_uint2(0x3f800000u, cs_);
    }
    printf("pattern %s\n", pn[pat]);
    h[n] = make_uint2(0, (unsigned)c.nc);
    cudaMemcpy(d_ent, h.data(), (n + 1) * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(c.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 1) * 8);
    for (int wps : {1, 2, 3, 4, 8}) {
      int nw = wps * 4;
      c.k<<<148, 1024, (n + 1) * 8>>>(d_ent, n, d_cyc, d_out, nw);
      c.k<<<148, 1024, (n + 1) * 8>>>(d_ent, n, d_cyc, d_out, nw);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      std::vector<long long> cy(148 * 32);
      cudaMemcpy(cy.data(), d_cyc, cy.size() * 8, cudaMemcpyDeviceToHost);
      double mx = 0; for (int i = 0; i < nw; ++i) mx = cy[i] > mx ? cy[i] : mx;
      printf("%-7s cases=%4d ffma2/case=%d warps/SMSP=%d  cycles/dispatch/warp=%.1f  per-SMSP=%.1f\n", c.name, c.nc,
             c.f, wps, mx / n, mx / n / wps);
    }
  }
  return 0;
}
''')
    open(sys.argv[1], "w").write("\n".join(src))


main()
