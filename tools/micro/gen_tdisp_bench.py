"""Microbenchmark: the stage-2 interpreter with the weights read from TMEM at every
dispatch instead of held in registers (V21 case structure: 3x3, pad 1, W=13, TY=2,
KL=4 as two f32x2 pairs = 104 accumulator registers).

Holding a channel's 9x4 weights in registers costs 36 registers (168 in total: 12
warps per SM); a case that loads its own taps with tcgen05.ld (12-cycle latency,
≥277 B/clk/SM, off the shared-memory port) needs none, so the SM holds 15-16 warps.
Styles (same i.i.d. data as gen_scan_bench.py):
  brx2  -- the shipped structure: marker per non-empty channel loads 9 taps from
           shared memory into registers; one brx.idx per nonzero
  tdisp -- markers only set the channel's TMEM column; every case loads the taps
           it uses (tcgen05.ld.32x32b.x4 per tap), waits, then FMAs
  tdnm  -- as tdisp without markers: the column rides in the entry (code = pos |
           col << 8); the dispatcher masks the position
  solo  -- brx2 where a channel with a single entry in the window is one solo entry
           (its case loads the taps it reaches) plus a data word with the channel,
           instead of marker + entry
  sdnm  -- no markers, every case loads its taps from shared memory
  pair  -- brx2 with the entries loaded two at a time (one LDS.128 every other
           dispatch, selected by a parity predicate): is the entry load on the
           dispatch chain?
Usage: python gen_tdisp_bench.py out.cu [styles,comma,separated] && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o b out.cu && ./b
"""
import sys

R, S, P, W, TY = 3, 3, 1, 13, 2
WO = W
NWR = TY + R - 1
NPOS = NWR * W
NACC = TY * WO * 2  # u64 operands
NWREG = 18          # u64 weight operands (brx2 only)


def case_taps(wi, j):
    """[(tap index r*S+t, [(acc operand, half)])] of window position (wi, j)."""
    out = []
    for r in range(R):
        ty = wi - r
        if not 0 <= ty < TY:
            continue
        for t in range(S):
            x = j + P - t
            if 0 <= x < WO:
                out.append((r * S + t, [((ty * WO + x) * 2 + h, h) for h in range(2)]))
    return out


def gen(style):
    a = ["{", ".reg .b64 vv, wa2, wb2;", ".reg .b32 xc, cc, xn, cn, ep, wa, col, ta, cx;",
         ".reg .b32 " + ", ".join(f"tw{i}" for i in range(24)) + ";"]
    regw = style in ("brx2", "pair", "solo", "solo1")  # weights in registers
    nreg = NACC + (NWREG if regw else 0)
    STREAM, WBASE = nreg, nreg + 1
    labels = [f"C{i}_%=" for i in range(NPOS)] + ["LW_%=", "END_%="]
    if style in ("solo", "solo1"):  # + one case per position for a channel's only entry in the window
        labels += [f"S{i}_%=" for i in range(NPOS)]
    if style == "pair":  # entries loaded two at a time (LDS.128 every other dispatch)
        a += [".reg .b32 x0, c0, x1, c1, par;", ".reg .pred podd;", f"mov.b32 ep, %{STREAM};", "mov.b32 col, 0;",
              "ld.shared.v4.b32 {x0, c0, x1, c1}, [ep];", "add.u32 ep, ep, 16;", "mov.b32 par, 0;",
              "LOOP_%=:", "setp.ne.b32 podd, par, 0;", "selp.b32 xc, x1, x0, podd;", "selp.b32 cc, c1, c0, podd;",
              "@podd ld.shared.v4.b32 {x0, c0, x1, c1}, [ep];", "@podd add.u32 ep, ep, 16;", "xor.b32 par, par, 1;",
              "mov.b64 vv, {xc, xc};"]
    else:
        a += [f"mov.b32 ep, %{STREAM};", "mov.b32 col, 0;", "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
              "LOOP_%=:", "mov.b32 xc, xn;", "mov.b32 cc, cn;", "ld.shared.v2.b32 {xn, cn}, [ep];",
              "add.u32 ep, ep, 8;", "mov.b64 vv, {xc, xc};"]
    if style == "tdnm" or style.startswith("sdnm") or style == "solo1":
        a += ["and.b32 cx, cc, 255;", "TS_%=: .branchtargets " + ", ".join(labels) + ";", "brx.idx.uni cx, TS_%=;"]
    else:
        a += ["TS_%=: .branchtargets " + ", ".join(labels) + ";", "brx.idx.uni cc, TS_%=;"]
    for q in range(NPOS):
        wi, j = divmod(q, W)
        taps = case_taps(wi, j)
        a.append(f"C{q}_%=:")
        if regw:
            for tap, accs in taps:
                for acc, h in accs:
                    a.append(f"fma.rn.f32x2 %{acc}, %{NACC + 2 * tap + h}, vv, %{acc};")
        else:
            if style.startswith("sdnm"):  # weights from shared memory: channel block (c % 16) * 9 taps * 512 B
                a += ["shr.u32 ta, cc, 8;", "and.b32 ta, ta, 15;", f"mad.lo.u32 ta, ta, 4608, %{WBASE};"]
                for i, (tap, _) in enumerate(taps):
                    a.append(f"ld.shared.v4.b32 {{tw{4 * i}, tw{4 * i + 1}, tw{4 * i + 2}, tw{4 * i + 3}}}, [ta+{tap * 512}];")
            else:
                if style == "tdnm":
                    a += ["shr.u32 ta, cc, 8;", f"add.u32 ta, ta, %{WBASE};"]
                else:
                    a += ["mov.b32 ta, col;"]
                for i, (tap, _) in enumerate(taps):
                    a.append(f"tcgen05.ld.sync.aligned.32x32b.x4.b32 {{tw{4 * i}, tw{4 * i + 1}, tw{4 * i + 2}, tw{4 * i + 3}}}, "
                             f"[ta+{tap * 4}];")
                a.append("tcgen05.wait::ld.sync.aligned;")
            for i, (tap, accs) in enumerate(taps):
                a.append(f"mov.b64 wa2, {{tw{4 * i}, tw{4 * i + 1}}};")
                a.append(f"mov.b64 wb2, {{tw{4 * i + 2}, tw{4 * i + 3}}};")
                for acc, h in accs:
                    a.append(f"fma.rn.f32x2 %{acc}, {'wa2' if h == 0 else 'wb2'}, vv, %{acc};")
        a.append("bra.uni LOOP_%=;")
    if style in ("solo", "solo1"):
        # solo: entry (x, SOLO0 + q) followed by a data entry (channel, 0): the channel is the
        # prefetched next entry; load the taps q reaches into the weight registers, skip the
        # data entry (re-prefetch), apply the FMAs.  solo1: one entry (x, SOLO0 + q | c << 8),
        # every dispatch masks the code
        for q in range(NPOS):
            wi, j = divmod(q, W)
            taps = case_taps(wi, j)
            a.append(f"S{q}_%=:")
            if style == "solo":
                a += ["and.b32 wa, xn, 15;", f"mad.lo.u32 wa, wa, 4608, %{WBASE};"]
            else:
                a += ["shr.u32 wa, cc, 8;", "and.b32 wa, wa, 15;", f"mad.lo.u32 wa, wa, 4608, %{WBASE};"]
            for tap, _ in taps:
                a.append(f"ld.shared.v2.b64 {{%{NACC + 2 * tap}, %{NACC + 2 * tap + 1}}}, [wa+{tap * 512}];")
            if style == "solo":
                a += ["ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;"]
            for tap, accs in taps:
                for acc, h in accs:
                    a.append(f"fma.rn.f32x2 %{acc}, %{NACC + 2 * tap + h}, vv, %{acc};")
            a.append("bra.uni LOOP_%=;")
    a.append("LW_%=:")
    if regw:
        a += ["and.b32 wa, xc, 15;", f"mad.lo.u32 wa, wa, 4608, %{WBASE};"]
        for t in range(9):
            a.append(f"ld.shared.v2.b64 {{%{NACC + 2 * t}, %{NACC + 2 * t + 1}}}, [wa+{t * 512}];")
    else:  # channel column (c % 14) * 36
        a += ["rem.u32 wa, xc, 14;", f"mad.lo.u32 col, wa, 36, %{WBASE};"]
    a += ["bra.uni LOOP_%=;", "END_%=:", "}"]
    return "\n\t".join(a), nreg


TMEM_SETUP = r"""
  __shared__ unsigned tslot;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((unsigned)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  wbase = tslot + ((unsigned)(32 * (warp & 3)) << 16);
  if (warp < 4) {  // lane l of quarter q holds channel c's weights at columns (c%14)*36 + tap*4 + k
    for (int col = 0; col < 504; ++col) {
      const int c = col / 36, r = col % 36, tap = r / 4, kk = r % 4;
      unsigned v = sm[(c * 9 + tap) * 128 + lane * 4 + kk];
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(wbase + col), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
"""
TMEM_FREE = r"""
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tslot));
"""


def kernel(style):
    body, nreg = gen(style)
    body = body.replace("\n", "\\n").replace('"', '\\"')
    regw = style in ("brx2", "pair", "solo", "solo1")
    tm = style in ("tdisp", "tdnm")
    outs = ", ".join([f'"+l"(acc[{i}])' for i in range(NACC)] +
                     ([f'"+l"(w[{i}])' for i in range(NWREG)] if regw else []))
    bounds = 384 if (regw or style == "sdnm12") else 512
    wdecl = f"unsigned long long w[{NWREG}]; for (int i = 0; i < {NWREG}; ++i) w[i] = 0ull;" if regw else ""
    return f'''
extern "C" __global__ void __launch_bounds__({bounds}, 1) k_{style}(const unsigned* __restrict__ g_buf, int nwords,
    int soff, float* out, int nwarps, int reps) {{
  extern __shared__ __align__(16) unsigned sm[];
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) sm[i] = g_buf[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  unsigned wbase = base + lane * 16;                             // weights at word 0
  {TMEM_SETUP if tm else ""}
  float r = 0;
  if (warp < nwarps) {{
    unsigned long long acc[{NACC}];
    for (int i = 0; i < {NACC}; ++i) acc[i] = 0ull;
    {wdecl}
    const unsigned stream = base + 4u * (unsigned)soff;
    for (int rep = 0; rep < reps; ++rep)
      asm volatile("{body}" : {outs} : "r"(stream), "r"(wbase) : "memory");
    for (int i = 0; i < {NACC}; ++i) r += __uint_as_float((unsigned)acc[i]) + __uint_as_float((unsigned)(acc[i] >> 32));
  }}
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  {TMEM_FREE if tm else ""}
}}
'''


HOST = r'''
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <random>
#include <cuda_runtime.h>
%KERNELS%
typedef void (*kfn)(const unsigned*, int, int, float*, int, int);
struct K { kfn k; const char* name; int maxw; };
int main(int argc, char** argv) {
  const double rho = argc > 1 ? atof(argv[1]) : 0.05;
  const int nch = 1024, NPOS = %NPOS%, W = 13;
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> U(0.f, 1.f);
  std::vector<unsigned> buf(16 * 9 * 128);   // weights: 16 channels x 9 taps x 128 floats
  for (auto& x : buf) { float f = 1e-3f * U(rng); x = *reinterpret_cast<unsigned*>(&f); }
  std::vector<unsigned> ent, enm, ens;   // with markers / without (TMEM column / channel in the code)
  long nnz = 0, fmas = 0;
  auto nf = [&](int q) { int wi = q / W, j = q % W, c = 0; for (int ty = 0; ty < 2; ++ty) { int r = wi - ty; if (r < 0 || r > 2) continue;
      for (int x = 0; x < W; ++x) { int t = j + 1 - x; if (t >= 0 && t < 3) c += 2; } } return c; };
  std::vector<unsigned> eso, es1;   // solo forms: a channel with one entry -> (x, SOLO0 + q), (c, 0) / (x, SOLO0 + q | c << 8)
  for (int c = 0; c < nch; ++c) {
    int k = 0;
    std::vector<unsigned> cq, cb;
    for (int q = 0; q < NPOS; ++q) if (U(rng) < rho) {
      { float f0 = 0; (void)f0; }
      float f = 1.0f + U(rng); unsigned b = *reinterpret_cast<unsigned*>(&f);
      if (k == 0) { ent.push_back((unsigned)c); ent.push_back((unsigned)NPOS); }
      ent.push_back(b); ent.push_back((unsigned)q);
      enm.push_back(b); enm.push_back((unsigned)q | ((unsigned)((c % 14) * 36) << 8));
      ens.push_back(b); ens.push_back((unsigned)q | ((unsigned)(c % 16) << 8));
      cq.push_back((unsigned)q); cb.push_back(b);
      ++nnz; fmas += nf(q); ++k;
    }
    if (cq.size() == 1) { eso.push_back(cb[0]); eso.push_back((unsigned)(NPOS + 2) + cq[0]); eso.push_back((unsigned)c); eso.push_back(0u);
                          es1.push_back(cb[0]); es1.push_back(((unsigned)(NPOS + 2) + cq[0]) | ((unsigned)(c % 16) << 8)); }
    else if (cq.size() > 1) {
      eso.push_back((unsigned)c); eso.push_back((unsigned)NPOS);
      es1.push_back((unsigned)c); es1.push_back((unsigned)NPOS);
      for (size_t i = 0; i < cq.size(); ++i) { eso.push_back(cb[i]); eso.push_back(cq[i]); es1.push_back(cb[i]); es1.push_back(cq[i]); }
    }
  }
  for (int i = 0; i < 2; ++i) { eso.push_back(0); eso.push_back(NPOS + 1); es1.push_back(0); es1.push_back(NPOS + 1); }
  for (int i = 0; i < 2; ++i) { ent.push_back(0); ent.push_back(NPOS + 1); enm.push_back(0); enm.push_back(NPOS + 1);
                                ens.push_back(0); ens.push_back(NPOS + 1); }
  while (buf.size() % 4) buf.push_back(0);
  const int off_m = (int)buf.size();
  buf.insert(buf.end(), ent.begin(), ent.end());
  const int off_n = (int)buf.size();
  buf.insert(buf.end(), enm.begin(), enm.end());
  const int off_s = (int)buf.size();
  buf.insert(buf.end(), ens.begin(), ens.end());
  const int off_o = (int)buf.size();
  buf.insert(buf.end(), eso.begin(), eso.end());
  const int off_1 = (int)buf.size();
  buf.insert(buf.end(), es1.begin(), es1.end());
  const int nwords = (int)buf.size();
  unsigned* d; float* o;
  cudaMalloc(&d, nwords * 4); cudaMalloc(&o, 148 * 512 * 4);
  cudaMemcpy(d, buf.data(), nwords * 4, cudaMemcpyHostToDevice);
  K ks[] = {%KLIST%};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 8;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("rho=%.3f nch=%d nnz/ch=%.2f ffma2/nz=%.2f smem=%d B\n", rho, nch, (double)nnz / nch, (double)fmas / nnz, nwords * 4);
  for (auto& k : ks) {
    cudaFuncSetAttribute(k.k, cudaFuncAttributeMaxDynamicSharedMemorySize, nwords * 4);
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k.k);
    for (int nw : {4, 8, 11, 12, 14, 15, 16}) {
      if (nw > k.maxw) continue;
      const int so = !strcmp(k.name, "solo1") ? off_1 : !strcmp(k.name, "solo") ? off_o : (!strcmp(k.name, "tdnm") || !strncmp(k.name, "sdnm", 4)) ? (strncmp(k.name, "sdnm", 4) ? off_n : off_s) : off_m;
      k.k<<<148, nw * 32, nwords * 4>>>(d, nwords, so, o, nw, 1);
      cudaEventRecord(e0);
      k.k<<<148, nw * 32, nwords * 4>>>(d, nwords, so, o, nw, reps);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s err %s\n", k.name, cudaGetErrorString(e)); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double lane_fma = 148.0 * nw * 32 * reps * 2.0 * fmas;
      double tf = 2 * lane_fma / (ms * 1e-3) / 1e12;
      double cyc_ch = ms * 1e-3 * clk * 1e3 / (reps * (double)nch);
      printf("%-6s regs=%3d warps/CTA=%2d  %.3f ms  %.1f TFLOP/s (%.1f%% of 74.4)  cycles/channel/warp=%.0f\n", k.name,
             fa.numRegs, nw, ms, tf, 100 * tf / 74.4, cyc_ch);
    }
  }
  return 0;
}
'''


def main():
    styles = sys.argv[2].split(",") if len(sys.argv) > 2 else ["brx2", "tdisp", "tdnm", "pair"]
    src = HOST.replace("%KERNELS%", "\n".join(kernel(s) for s in styles))
    src = src.replace("%KLIST%", ", ".join(f'{{k_{s}, "{s}", {12 if s in ("brx2", "pair", "sdnm12", "solo", "solo1") else 16}}}' for s in styles))
    src = src.replace("%NPOS%", str(NPOS))
    open(sys.argv[1], "w").write(src)


if __name__ == "__main__":
    main()
