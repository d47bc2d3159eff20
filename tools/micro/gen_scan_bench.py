"""Microbenchmark: stage-2 dispatch styles on the V21 case structure
(3x3, pad 1, W=13, TY=2 output rows, KL=4 channels per lane as two f32x2
pairs = 104 accumulator registers, 36 weight registers).

Styles (same data: NCH channels per warp, i.i.d. nonzeros at density RHO
in the 4x13 window of each channel):
  brx   -- the round-1 interpreter: a marker entry per channel (weight load)
           then one brx.idx.uni per nonzero entry
  skip  -- no indirect branch: per channel a 4x16-bit occupancy mask; a
           static scan over the 52 window positions, `@!p bra` over each
           position's FMA block
  ool   -- as skip, but the FMA blocks are out of line (`@p bra` to the
           block, `bra` back): no taken branch for an empty position
  row   -- as skip, with a per-row gate (skip 13 positions of an empty row)
  rowool-- row gate + out-of-line blocks
Usage: python gen_scan_bench.py out.cu && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o b out.cu && ./b
"""
import sys

R, S, P, W, TY = 3, 3, 1, 13, 2
WO = W
NWR = TY + R - 1
NPOS = NWR * W
NACC = TY * WO * 2  # u64 operands
NW = 18             # u64 weight operands (9 taps x 2 pairs)


def case_fmas(wi, j):
    out = []
    for ty in range(TY):
        r = wi - ty
        if not 0 <= r < R:
            continue
        for x in range(WO):
            t = j + P - x
            if 0 <= t < S:
                for h in range(2):
                    out.append(((ty * WO + x) * 2 + h, (r * S + t) * 2 + h))
    return out


def fma(a, w):
    return f"fma.rn.f32x2 %{a}, %{NACC + w}, vv, %{a};"


OPS = NACC + NW  # first input operand index
STREAM, WBASE, NCHO = OPS, OPS + 1, OPS + 2


def load_weights(addr):
    a = []
    for t in range(9):
        a.append(f"ld.shared.v2.b64 {{%{NACC + 2 * t}, %{NACC + 2 * t + 1}}}, [{addr}+{t * 512}];")
    return a



def load_weights_tmem(col_reg):
    regs = ", ".join(f"tw{i}" for i in range(32))
    a = [f"add.u32 ta, %{WBASE}, {col_reg};",
         f"tcgen05.ld.sync.aligned.32x32b.x32.b32 {{{regs}}}, [ta];",
         "add.u32 ta, ta, 32;",
         "tcgen05.ld.sync.aligned.32x32b.x4.b32 {tw32, tw33, tw34, tw35}, [ta];",
         "tcgen05.wait::ld.sync.aligned;"]
    for p in range(18):
        a.append(f"mov.b64 %{NACC + p}, {{tw{2 * p}, tw{2 * p + 1}}};")
    return a

def weights_from(style, xreg):
    if style.startswith("t"):
        return ["rem.u32 wa, %s, 14;" % xreg, "mul.lo.u32 wa, wa, 36;"] + load_weights_tmem("wa")
    return ["and.b32 wa, %s, 15;" % xreg, f"mad.lo.u32 wa, wa, 4608, %{WBASE};"] + load_weights("wa")


def gen(style):
    tm = style.startswith("t") and style != "thr"
    if tm:
        style_t, style = style, style[1:]
    a = ["{", ".reg .b32 ta, " + ", ".join(f"tw{i}" for i in range(36)) + ";" if tm else "", ".reg .b64 vv;", ".reg .b32 xc, cc, xn, cn, ep, mlo, mhi, t, ch, wa, vp, vc, vn, mp;",
         ".reg .pred p, pe;"]

    if style == "thr":
        labels = [f"C{i}_%=" for i in range(NPOS)] + ["LW_%=", "END_%="]
        disp = ["mov.b32 xc, xn;", "mov.b32 cc, cn;", "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
                "mov.b64 vv, {xc, xc};", "brx.idx.uni cc, TS_%=;"]
        a += [f"mov.b32 ep, %{STREAM};", "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
              "TS_%=: .branchtargets " + ", ".join(labels) + ";"] + disp
        for q in range(NPOS):
            wi, j = divmod(q, W)
            a.append(f"C{q}_%=:")
            a += [fma(x, w) for x, w in case_fmas(wi, j)]
            a += disp
        a += ["LW_%=:", "and.b32 wa, xc, 15;", f"mad.lo.u32 wa, wa, 4608, %{WBASE};"] + load_weights("wa")
        a += disp + ["END_%=:", "}"]
        return "\n\t".join(a)

    if style == "fused":
        # per non-empty channel: (c, FUSED + q0) then (bits of its first nonzero, 0) then the
        # remaining nonzeros; the fused case loads the channel's weights and applies q0
        labels = [f"C{i}_%=" for i in range(NPOS)] + ["LW_%=", "END_%="] + [f"F{i}_%=" for i in range(NPOS)]
        a += [".reg .b32 xf;", f"mov.b32 ep, %{STREAM};", "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
              "LOOP_%=:", "mov.b32 xc, xn;", "mov.b32 cc, cn;", "ld.shared.v2.b32 {xn, cn}, [ep];",
              "add.u32 ep, ep, 8;", "mov.b64 vv, {xc, xc};", "TS_%=: .branchtargets " + ", ".join(labels) + ";",
              "brx.idx.uni cc, TS_%=;"]
        for q in range(NPOS):
            wi, j = divmod(q, W)
            a.append(f"C{q}_%=:")
            a += [fma(x, w) for x, w in case_fmas(wi, j)]
            a.append("bra.uni LOOP_%=;")
        for q in range(NPOS):
            wi, j = divmod(q, W)
            a.append(f"F{q}_%=:")
            a += ["mov.b32 xf, xn;", "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;"]
            a += weights_from("t" if tm else "", "xc")
            a += ["mov.b64 vv, {xf, xf};"] + [fma(x, w) for x, w in case_fmas(wi, j)]
            a.append("bra.uni LOOP_%=;")
        a += ["LW_%=:", "bra.uni LOOP_%=;", "END_%=:", "}"]
        return "\n\t".join(a)
    if style in ("brx", "brx2"):
        labels = [f"C{i}_%=" for i in range(NPOS)] + ["LW_%=", "END_%="]
        a += [f"mov.b32 ep, %{STREAM};", "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;", "LOOP_%=:",
              "mov.b32 xc, xn;", "mov.b32 cc, cn;", "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
              "mov.b64 vv, {xc, xc};", "TS_%=: .branchtargets " + ", ".join(labels) + ";",
              "brx.idx.uni cc, TS_%=;"]
        for q in range(NPOS):
            wi, j = divmod(q, W)
            a.append(f"C{q}_%=:")
            a += [fma(x, w) for x, w in case_fmas(wi, j)]
            a.append("bra.uni LOOP_%=;")
        a += ["LW_%=:"] + weights_from("t" if tm else "", "xc")
        a += ["bra.uni LOOP_%=;", "END_%=:", "}"]
        return "\n\t".join(a)
    # scan styles: stream = [nch] uint2 masks (row r at bits 16*(r%2) of word r/2) then values
    a += [f"mov.b32 mp, %{STREAM};", f"mad.lo.u32 vp, %{NCHO}, 8, mp;", "ld.shared.b32 vc, [vp];",
          "ld.shared.b32 vn, [vp+4];", "add.u32 vp, vp, 8;", "mov.b32 ch, 0;",
          "CH_%=:", f"setp.ge.u32 pe, ch, %{NCHO};", "@pe bra.uni END_%=;",
          "ld.shared.v2.b32 {mlo, mhi}, [mp];", "add.u32 mp, mp, 8;",
          "and.b32 wa, ch, 15;", f"mad.lo.u32 wa, wa, 4608, %{WBASE};"] + load_weights("wa")
    ool = []

    def block(q):
        wi, j = divmod(q, W)
        return (["mov.b64 vv, {vc, vc};"] + [fma(x, w) for x, w in case_fmas(wi, j)] +
                ["mov.b32 vc, vn;", "ld.shared.b32 vn, [vp];", "add.u32 vp, vp, 4;"])

    for wi in range(NWR):
        word = "mlo" if wi < 2 else "mhi"
        sh = 16 * (wi % 2)
        if style in ("row", "rowool"):
            a += [f"and.b32 t, {word}, {0x1fff << sh};", "setp.eq.u32 p, t, 0;", f"@p bra.uni RS{wi}_%=;"]
        for j in range(W):
            q = wi * W + j
            a += [f"and.b32 t, {word}, {1 << (sh + j)};"]
            if style in ("skip", "row"):
                a += ["setp.eq.u32 p, t, 0;", f"@p bra.uni S{q}_%=;"] + block(q) + [f"S{q}_%=:"]
            else:
                a += ["setp.ne.u32 p, t, 0;", f"@p bra.uni B{q}_%=;", f"R{q}_%=:"]
                ool += [f"B{q}_%=:"] + block(q) + [f"bra.uni R{q}_%=;"]
        if style in ("row", "rowool"):
            a.append(f"RS{wi}_%=:")
    a += ["add.u32 ch, ch, 1;", "bra.uni CH_%=;"] + ool + ["END_%=:", "}"]
    return "\n\t".join(a)


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
  if (warp < 4) {  // fill: lane l of quarter q holds channel c's weights at columns (c%14)*36 + tap*4 + k
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
    tm = style.startswith("t") and style != "thr"
    body = gen(style).replace("\n", "\\n").replace('"', '\\"')
    outs = ", ".join([f'"+l"(acc[{i}])' for i in range(NACC)] + [f'"+l"(w[{i}])' for i in range(NW)])
    setup = TMEM_SETUP if tm else ""
    free = TMEM_FREE if tm else ""
    sel = 'brx_off' if style in ('brx', 'thr', 'brx2', 'fused', 'tbrx2', 'tfused') else 'nwords_scan(nwords)'
    return f'''
extern "C" __global__ void __launch_bounds__(384, 1) k_{style}(const unsigned* __restrict__ g_buf, int nwords,
    int brx_off, int nch, float* out, int nwarps, int reps) {{
  extern __shared__ __align__(16) unsigned sm[];
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) sm[i] = g_buf[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  unsigned wbase = base + lane * 16;                             // weights at word 0
  {setup}
  float r = 0;
  if (warp < nwarps) {{
    unsigned long long acc[{NACC}], w[{NW}];
    for (int i = 0; i < {NACC}; ++i) acc[i] = 0ull;
    for (int i = 0; i < {NW}; ++i) w[i] = 0ull;
    const unsigned stream = base + 4u * (unsigned)({sel});
    for (int rep = 0; rep < reps; ++rep)
      asm volatile("{body}" : {outs} : "r"(stream), "r"(wbase), "r"(nch) : "memory");
    for (int i = 0; i < {NACC}; ++i) r += __uint_as_float((unsigned)acc[i]) + __uint_as_float((unsigned)(acc[i] >> 32));
  }}
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  {free}
}}
'''


HOST = r'''
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <random>
#include <cuda_runtime.h>
__device__ __forceinline__ int nwords_scan(int) { return 16 * 9 * 128; }
%KERNELS%
typedef void (*kfn)(const unsigned*, int, int, int, float*, int, int);
struct K { kfn k; const char* name; };
int main(int argc, char** argv) {
  const double rho = argc > 1 ? atof(argv[1]) : 0.05;
  const int nch = 1024, NPOS = %NPOS%, W = 13;
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> U(0.f, 1.f);
  // weights: 16 channels x 9 taps x 128 floats (lane l: 4 floats at 16*l)
  std::vector<unsigned> buf(16 * 9 * 128);
  for (auto& x : buf) { float f = 1e-3f * U(rng); x = *reinterpret_cast<unsigned*>(&f); }
  std::vector<unsigned> masks, vals, ent, ent2, fus;
  long nnz = 0, fmas = 0;
  auto nf = [&](int q) { int wi = q / W, j = q % W, c = 0; for (int ty = 0; ty < 2; ++ty) { int r = wi - ty; if (r < 0 || r > 2) continue;
      for (int x = 0; x < W; ++x) { int t = j + 1 - x; if (t >= 0 && t < 3) c += 2; } } return c; };
  for (int c = 0; c < nch; ++c) {
    unsigned m[2] = {0, 0};
    ent.push_back((unsigned)c); ent.push_back((unsigned)NPOS);  // marker (LW)
    int k = 0;
    for (int q = 0; q < NPOS; ++q) if (U(rng) < rho) {
      int wi = q / W, j = q % W; m[wi / 2] |= 1u << (16 * (wi % 2) + j);
      float f = 1.0f + U(rng); unsigned b = *reinterpret_cast<unsigned*>(&f);
      vals.push_back(b); ent.push_back(b); ent.push_back((unsigned)q); ++nnz; fmas += nf(q);
      if (k == 0) { ent2.push_back((unsigned)c); ent2.push_back((unsigned)NPOS);
                    fus.push_back((unsigned)c); fus.push_back((unsigned)(NPOS + 2 + q)); fus.push_back(b); fus.push_back(0u); }
      else { fus.push_back(b); fus.push_back((unsigned)q); }
      ent2.push_back(b); ent2.push_back((unsigned)q);
      ++k;
    }
    masks.push_back(m[0]); masks.push_back(m[1]);
  }
  ent.push_back(0); ent.push_back(NPOS + 1); ent.push_back(0); ent.push_back(NPOS + 1);
  vals.push_back(0); vals.push_back(0); vals.push_back(0);
  const int scan_off = (int)buf.size();
  buf.insert(buf.end(), masks.begin(), masks.end());
  buf.insert(buf.end(), vals.begin(), vals.end());
  while (buf.size() % 4) buf.push_back(0);
  const int brx_off = (int)buf.size();
  buf.insert(buf.end(), ent.begin(), ent.end());
  ent2.push_back(0); ent2.push_back(NPOS + 1); ent2.push_back(0); ent2.push_back(NPOS + 1);
  fus.push_back(0); fus.push_back(NPOS + 1); fus.push_back(0); fus.push_back(NPOS + 1);
  const int brx2_off = (int)buf.size();
  buf.insert(buf.end(), ent2.begin(), ent2.end());
  const int fus_off = (int)buf.size();
  buf.insert(buf.end(), fus.begin(), fus.end());
  const int nwords = (int)buf.size();
  unsigned* d; float* o;
  cudaMalloc(&d, nwords * 4); cudaMalloc(&o, 148 * 384 * 4);
  cudaMemcpy(d, buf.data(), nwords * 4, cudaMemcpyHostToDevice);
  K ks[] = {%KLIST%};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 8;
  printf("rho=%.3f nch=%d nnz/ch=%.2f ffma2/nz=%.2f smem=%d B\n", rho, nch, (double)nnz / nch, (double)fmas / nnz, nwords * 4);
  for (auto& k : ks) {
    cudaFuncSetAttribute(k.k, cudaFuncAttributeMaxDynamicSharedMemorySize, nwords * 4);
    for (int nw : {4, 8, 11, 12}) {
      const int so = (!strcmp(k.name, "brx2") || !strcmp(k.name, "tbrx2")) ? brx2_off :
                     (!strcmp(k.name, "fused") || !strcmp(k.name, "tfused")) ? fus_off : brx_off;
      k.k<<<148, 384, nwords * 4>>>(d, nwords, so, nch, o, nw, 1);
      cudaEventRecord(e0);
      k.k<<<148, 384, nwords * 4>>>(d, nwords, so, nch, o, nw, reps);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s err %s\n", k.name, cudaGetErrorString(e)); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double lane_fma = 148.0 * nw * 32 * reps * 2.0 * fmas;
      double tf = 2 * lane_fma / (ms * 1e-3) / 1e12;
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      double cyc_ch = ms * 1e-3 * clk * 1e3 / (reps * (double)nch);
      printf("%-7s warps/CTA=%2d  %.3f ms  %.1f TFLOP/s (%.1f%% of 74.4)  cycles/channel/warp=%.0f\n", k.name, nw, ms, tf,
             100 * tf / 74.4, cyc_ch);
    }
  }
  return 0;
}
'''


def main():
    styles = ["brx2", "fused", "tbrx2", "tfused"]
    src = HOST.replace("%KERNELS%", "\n".join(kernel(s) for s in styles))
    src = src.replace("%KLIST%", ", ".join(f'{{k_{s}, "{s}"}}' for s in styles)).replace("%NPOS%", str(NPOS))
    open(sys.argv[1], "w").write(src)


main()
