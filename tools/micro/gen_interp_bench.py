"""Microbenchmark of the stage-2 interpreter styles on the real case structure
(3x3, pad 1, W=13, KL=2 k-pair FFMA2 accumulators, TY output rows).
Measures lane-FMA/clk/SM for: loop (dispatch at a loop head, bra back),
threaded (each case ends with its own dispatch), threaded2 (2-deep entry
prefetch).  Usage: python gen_interp_bench.py out.cu; nvcc -arch=sm_100a -O3 -o b out.cu; ./b"""
import sys

R, S, P, W = 3, 3, 1, 13
WO = W + 2 * P - S + 1


def cases(TY):
    NWR = TY + R - 1
    out = []
    for wi in range(NWR):
        for j in range(W):
            body = []
            for ty in range(TY):
                r = wi - ty
                if not 0 <= r < R:
                    continue
                for x in range(WO):
                    t = j + P - x
                    if 0 <= t < S:
                        body.append((ty * WO + x, r * S + t))
            out.append(body)
    return out


def gen(style, TY):
    cs = cases(TY)
    nacc = TY * WO
    wbase = nacc
    vop = nacc + 9
    fma = lambda a, w: f"fma.rn.f32x2 %{a}, %{wbase + w}, vv, %{a};"
    a = ["{", ".reg .b64 vv;", ".reg .b32 xc, cc, x1, c1, x2, c2, ep;", ".reg .pred pp;", f"mov.b32 ep, %{vop};"]
    labels = [f"C{i}_%=" for i in range(len(cs))] + ["END_%="]
    if style == "loop":
        a += ["ld.shared.v2.b32 {x1, c1}, [ep];", "add.u32 ep, ep, 8;", "LOOP_%=:", "mov.b32 xc, x1;",
              "mov.b32 cc, c1;", "ld.shared.v2.b32 {x1, c1}, [ep];", "add.u32 ep, ep, 8;", "mov.b64 vv, {xc, xc};",
              "TS_%=: .branchtargets " + ", ".join(labels) + ";", "brx.idx.uni cc, TS_%=;"]
        tail = ["bra.uni LOOP_%=;"]
    elif style == "threaded":
        a += ["ld.shared.v2.b32 {x1, c1}, [ep];", "add.u32 ep, ep, 8;",
              "TS_%=: .branchtargets " + ", ".join(labels) + ";"]
        tail = ["mov.b32 xc, x1;", "mov.b32 cc, c1;", "ld.shared.v2.b32 {x1, c1}, [ep];", "add.u32 ep, ep, 8;",
                "mov.b64 vv, {xc, xc};", "brx.idx.uni cc, TS_%=;"]
        a += tail
    elif style == "shfl":
        a += ["ld.shared.v2.b32 {x1, c1}, [ep];", "add.u32 ep, ep, 8;", "LOOP_%=:", "mov.b32 xc, x1;",
              "shfl.sync.idx.b32 cc, c1, 0, 31, -1;", "ld.shared.v2.b32 {x1, c1}, [ep];", "add.u32 ep, ep, 8;",
              "mov.b64 vv, {xc, xc};",
              "TS_%=: .branchtargets " + ", ".join(labels) + ";", "brx.idx.uni cc, TS_%=;"]
        tail = ["bra.uni LOOP_%=;"]
    elif style == "brxinv":
        # loop-invariant jump index (kernel argument): LDC can leave the loop
        a += ["ld.shared.v2.b32 {x1, c1}, [ep];", "add.u32 ep, ep, 8;", "LOOP_%=:", "mov.b32 xc, x1;",
              "mov.b32 cc, c1;", "ld.shared.v2.b32 {x1, c1}, [ep];", "add.u32 ep, ep, 8;", "mov.b64 vv, {xc, xc};",
              f"setp.ge.u32 pp, cc, {len(cs)};", "@pp bra.uni END_%=;",
              "TS_%=: .branchtargets " + ", ".join(labels) + ";", f"brx.idx.uni %{vop + 1}, TS_%=;"]
        tail = ["bra.uni LOOP_%=;"]
    elif style == "nobrx":
        a += ["ld.shared.v2.b32 {x1, c1}, [ep];", "add.u32 ep, ep, 8;", "LOOP_%=:", "mov.b32 xc, x1;",
              "mov.b32 cc, c1;", "ld.shared.v2.b32 {x1, c1}, [ep];", "add.u32 ep, ep, 8;", "mov.b64 vv, {xc, xc};",
              f"setp.ge.u32 pp, cc, {len(cs)};", "@pp bra.uni END_%=;", f"bra.uni C{len(cs)//2}_%=;"]
        tail = ["bra.uni LOOP_%=;"]
    else:  # threaded2
        a += ["ld.shared.v2.b32 {x1, c1}, [ep];", "ld.shared.v2.b32 {x2, c2}, [ep+8];", "add.u32 ep, ep, 16;",
              "TS_%=: .branchtargets " + ", ".join(labels) + ";"]
        tail = ["mov.b32 xc, x1;", "mov.b32 cc, c1;", "mov.b32 x1, x2;", "mov.b32 c1, c2;",
                "ld.shared.v2.b32 {x2, c2}, [ep];", "add.u32 ep, ep, 8;", "mov.b64 vv, {xc, xc};",
                "brx.idx.uni cc, TS_%=;"]
        a += tail
    for i, b in enumerate(cs):
        a.append(f"C{i}_%=:")
        a += [fma(p, t) for p, t in b]
        a += tail
    a += ["END_%=:", "}"]
    body = "\\n\\t".join(a)
    outs = ", ".join([f'"+l"(acc[{i}])' for i in range(nacc)] + [f'"+l"(w[{i}])' for i in range(9)])
    name = f"k_{style}_ty{TY}"
    NT = {3: 512, 5: 384, 7: 256}[TY]
    nf = sum(len(b) for b in cs)
    src = f'''
extern "C" __global__ void __launch_bounds__({NT}, 1) {name}(const uint2* __restrict__ g_ent, int n, float* out, int nwarps, unsigned fixed) {{
  extern __shared__ uint2 ent[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < n + 2; i += blockDim.x) ent[i] = g_ent[i];
  __syncthreads();
  if (warp >= nwarps) return;
  unsigned long long acc[{nacc}], w[9];
  for (int i = 0; i < {nacc}; ++i) acc[i] = 0ull;
  for (int i = 0; i < 9; ++i) w[i] = 0x3f8000003f800000ull + lane + i;
  unsigned s = (unsigned)__cvta_generic_to_shared(ent);
  for (int rep = 0; rep < 8; ++rep)
  asm volatile("{body}" : {outs} : "r"(s), "r"(fixed) : "memory");
  float r = 0; for (int i = 0; i < {nacc}; ++i) r += __uint_as_float((unsigned)acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}}
'''
    return name, src, len(cs), nf, NT


def main():
    src = ["#include <cstdio>", "#include <cstdlib>", "#include <cstdint>", "#include <cstring>", "#include <vector>",
           "#include <cuda_runtime.h>"]
    ents = []
    for TY in (3, 5, 7):
        for style in ("loop", "shfl", "brxinv", "nobrx"):
            name, s, nc, nf, nt = gen(style, TY)
            src.append(s)
            ents.append(f'{{{nc}, {nf}, {name}, "{name}", {nt}}}')
    src.append("typedef void (*kfn)(const uint2*, int, float*, int, unsigned);")
    src.append("struct C { int nc, nf; kfn k; const char* name; int nt; };")
    src.append("C cs[] = {" + ", ".join(ents) + "};")
    src.append(r'''
int main() {
  const int n = 12000;
  uint2* d_ent; float* d_out;
  cudaMalloc(&d_ent, (n + 2) * 8); cudaMalloc(&d_out, 148 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int pat = 0; pat < 4; ++pat)
  for (auto& c : cs) {
    if (pat != 0 && pat != 1) continue;
    std::vector<uint2> h(n + 2);
    srand(1);
    double fmas = 0;
    // average FFMA2 per case = nf / nc; dispatch counts per warp = n
    for (int i = 0; i < n; ++i) { unsigned q = pat == 0 ? rand() % c.nc : pat == 1 ? c.nc / 2 : pat == 2 ? (c.nc / 2 + (i & 3)) : (unsigned)(i % c.nc); h[i] = make_uint2(0x3f800000u, q); }
    h[n] = make_uint2(0, (unsigned)c.nc); h[n + 1] = h[n];
    cudaMemcpy(d_ent, h.data(), (n + 2) * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(c.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 2) * 8);
    for (int wps : {1, 2, 3, 4}) {
      int nw = wps * 4; if (nw * 32 > c.nt) continue;
      c.k<<<148, c.nt, (n + 2) * 8>>>(d_ent, n, d_out, nw, (unsigned)(c.nc / 2));
      cudaEventRecord(e0);
      c.k<<<148, c.nt, (n + 2) * 8>>>(d_ent, n, d_out, nw, (unsigned)(c.nc / 2));
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double lane_fma = 148.0 * nw * 32 * 8.0 * n * (2.0 * c.nf / c.nc);
      double tflops = 2 * lane_fma / (ms * 1e-3) / 1e12;
      double disp_ns = ms * 1e6 / (8.0 * n);
      printf("pat%d %-16s cases=%4d ffma2/case=%.2f warps/SMSP=%d  %.3f ms  FP32 %.1f TFLOP/s (%.0f%% of 74.4)  ns/dispatch/warp=%.1f\n",
             pat, c.name, c.nc, (double)c.nf / c.nc, wps, ms, tflops, 100 * tflops / 74.4, disp_ns);
    }
  }
  return 0;
}
''')
    open(sys.argv[1], "w").write("\n".join(src))


main()
