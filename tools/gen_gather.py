"""Generate paper_1704_07724_b200/csrc/gather_variants.inc -- the per-shape
dispatch code of the register-tile sparse-gather kernel (gather_fast_impl.cuh).

Why generated: the kernel keeps a warp's output tile in registers and each
nonzero input lands at a *dynamic* position of the tile's input window.
Register arrays need static indices, so every window position gets its own
block of code naming the exact accumulators it updates (ISC: "calculate the
product I_{c,i,j} x W_{k,c,i-r,j-s} for an output O_{k,i+r,j+s}", PAPER.md:121,
with the inverse index map of reading R6: y = i + P - r, x = j + P - t).  The
blocks are emitted as inline PTX behind ONE `brx.idx.uni` jump table (SASS:
LDC + BRX per nonzero); a C++ `switch` is lowered by the NVVM front end to a
compare tree (~12 branches per nonzero) instead.

Two register-tile forms (KL = output channels per lane):
* KL=2: acc[ty][x] is an f32x2 pair over two adjacent output channels
  (k0, k0+1) of pixel (y0+ty, x); one FFMA2 (fma.rn.f32x2, nonzero value as a
  broadcast scalar) per in-tile tap: acc[ty][x] += v * (W[k0][r][t], W[k0+1][r][t]).
  No lane is wasted; the weight operand is a natural 64-bit shared-memory load.
* KL=1: acc[ty][m] pairs two horizontally adjacent outputs (x = 2m, 2m+1) of
  one output channel.  Where both outputs are in the nonzero's footprint one
  FFMA2 with the weight pair (W[r][u], W[r][u-1]), u = j + P - 2m, updates both;
  where only one is, a single FFMA updates that half.  No zero-padded weights.

Usage: python tools/gen_gather.py  (rewrites the .inc; commit the result).
"""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_1704_07724_b200", "csrc", "gather_variants.inc")

# (id, name, R, S, P, W, TY, KL, NW, MINB, CH, STAGES): stride 1 only.  W = input width.
# NW warps per CTA, MINB CTAs per SM (register budget 65536 / (32*NW*MINB)).
VARIANTS = [
    (1, "r3s3p1_w13_ty7_kl2", 3, 3, 1, 13, 7, 2, 8, 1, 8, 4),      # C2, C5 (AlexNet conv3/4/5)
    (2, "r3s3p1_w28_ty3_kl2", 3, 3, 1, 28, 3, 2, 8, 1, 8, 4),      # C4a (inception-3a 3x3)
    (3, "r5s5p2_w27_ty2_kl2", 5, 5, 2, 27, 2, 2, 8, 1, 4, 4),      # C3 (AlexNet conv2, groups 2)
    (4, "r5s5p2_w28_ty2_kl2", 5, 5, 2, 28, 2, 2, 8, 1, 4, 4),      # C4b (inception-3a 5x5)
    (5, "r5s5p0_w12_ty6_kl2", 5, 5, 0, 12, 6, 2, 8, 1, 4, 4),      # C1 (LeNet conv2)
    (6, "r3s3p1_w13_ty13_kl1", 3, 3, 1, 13, 13, 1, 8, 1, 16, 4),   # C2 alternative (whole plane, 32 k/warp)
    (7, "r3s3p1_w13_ty7_kl1_nw12", 3, 3, 1, 13, 7, 1, 12, 1, 16, 4),  # C2: 3 warps/SMSP
    (8, "r3s3p1_w13_ty4_kl2_nw12", 3, 3, 1, 13, 4, 2, 12, 1, 8, 4),   # C2: 3 warps/SMSP
    (9, "r3s3p1_w13_ty7_kl1_nw8x2", 3, 3, 1, 13, 7, 1, 8, 2, 8, 3),   # C2: 2 CTAs/SM
]

# C2 s=0.95 gather (B200, round 1): V7 232 us, V1 331 us, V8 340 us, V6 393 us, V9 422 us
PRIORITY = [7, 1, 8, 6, 9]


def gen_variant(vid, name, R, S, P, W, TY, KL, NW, MINB, CH, STAGES):
    WO = W + 2 * P - S + 1
    NX = WO if KL == 2 else (WO + 1) // 2          # accumulator columns per row
    NWR = TY + R - 1                                 # window rows
    NCASES = NWR * W
    accs = [(ty, m) for ty in range(TY) for m in range(NX)]
    aop = {a: i for i, a in enumerate(accs)}
    if KL == 2:
        wops = [(r, t) for r in range(R) for t in range(S)]            # f32x2 (k0, k1) per tap
    else:
        assert S >= 2
        wops = [(r, u) for r in range(R) for u in range(1, S)]          # pair (W[r][u], W[r][u-1])
    wop = {w: len(accs) + i for i, w in enumerate(wops)}
    vop = len(accs) + len(wops)

    def scalar(r, t):
        """(operand, half) holding W[r][t] inside the KL=1 weight pairs."""
        if t >= 1:
            return wop[(r, t)], "lo"          # lo of (W[r][t], W[r][t-1])
        return wop[(r, 1)], "hi"              # hi of (W[r][1], W[r][0])

    bodies = []
    n_fma = 0
    for wi in range(NWR):
        for j in range(W):
            body = []
            for ty in range(TY):
                r = wi - ty
                if not (0 <= r < R):
                    continue
                if KL == 2:
                    for x in range(WO):
                        t = j + P - x
                        if 0 <= t < S:
                            a = aop[(ty, x)]
                            body.append(f"fma.rn.f32x2 %{a}, %{wop[(r, t)]}, vv, %{a};")
                else:
                    for m in range(NX):
                        x0, x1 = 2 * m, 2 * m + 1
                        t0, t1 = j + P - x0, j + P - x1
                        in0 = 0 <= t0 < S
                        in1 = 0 <= t1 < S and x1 < WO
                        a = aop[(ty, m)]
                        if in0 and in1:
                            body.append(f"fma.rn.f32x2 %{a}, %{wop[(r, t0)]}, vv, %{a};")
                        elif in0 or in1:
                            t = t0 if in0 else t1
                            half = "l" if in0 else "h"
                            o, wh = scalar(r, t)
                            body.append(f"mov.b64 {{al, ah}}, %{a}; mov.b64 {{wl, wh}}, %{o}; "
                                        f"fma.rn.f32 a{half}, w{wh[0]}, %{vop}, a{half}; mov.b64 %{a}, {{al, ah}};")
            bodies.append(body)
            n_fma += len(body)
    # ---- threaded interpreter over a shared-memory entry stream ----------
    # entry = (x, code): code < NCASES: nonzero with value bits x at window
    # position `code`; code == NCASES: channel marker, x = channel index ->
    # load the lane's weights of channel x from the weight stage;
    # code == NCASES+1: exit.
    # The next entry is loaded before the current one is dispatched.
    LW, EXIT = NCASES, NCASES + 1
    pop = vop   # %pop: stream pointer (u32 smem address)
    wlop = vop + 1   # lane's weight address of the chunk's first channel
    cbop = vop + 2   # global index of the chunk's first channel
    chb = R * S * 32 * KL * 4   # bytes of one channel in the weight stage
    asm = ["{", ".reg .b64 vv;", ".reg .b32 xc, cc, xn, cn, ep, ea;", ".reg .f32 al, ah, wl, wh, vf;",
           f"mov.b32 ep, %{pop};",
           "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
           "LOOP_%=:",
           "mov.b32 xc, xn;", "mov.b32 cc, cn;",
           "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
           "mov.b64 vv, {xc, xc};", "mov.b32 vf, xc;"]
    labels = [f"C{i}_%=" if b else "LOOP_%=" for i, b in enumerate(bodies)] + ["LW_%=", "END_%="]
    asm.append("TS_%=: .branchtargets " + ", ".join(labels) + ";")
    asm.append("brx.idx.uni cc, TS_%=;")
    for i, b in enumerate(bodies):
        if b:
            asm.append(f"C{i}_%=:")
            asm += [x.replace(f"%{vop},", "vf,") for x in b]
            asm.append("bra.uni LOOP_%=;")
    asm.append("LW_%=:")
    asm.append(f"sub.u32 ea, xc, %{cbop};")
    asm.append(f"mad.lo.u32 ea, ea, {chb}, %{wlop};")
    if KL == 2:
        for i in range(len(wops)):
            asm.append(f"ld.shared.b64 %{wop[wops[i]]}, [ea+{i * 256}];")
    else:
        for r in range(R):
            for u in range(1, S):
                # pair (W[r][u], W[r][u-1]); weights of tap (r,t) at byte (r*S+t)*128 + lane*4
                asm.append(f"ld.shared.f32 wl, [ea+{(r * S + u) * 128}]; ld.shared.f32 wh, [ea+{(r * S + u - 1) * 128}]; "
                           f"mov.b64 %{wop[(r, u)]}, {{wl, wh}};")
    asm.append("bra.uni LOOP_%=;")
    asm.append("END_%=:")
    asm.append("}")
    lines = [f"// ---- variant {vid}: {name}  (R={R} S={S} P={P} W={W} WO={WO} TY={TY} KL={KL} NX={NX} NW={NW}); "
             f"{n_fma} FMA instructions over {NCASES} window positions"]
    lines.append(f"struct V{vid} {{")
    for k, v in (("R", R), ("S", S), ("P", P), ("W", W), ("WO", WO), ("NX", NX), ("TY", TY), ("KL", KL),
                 ("NW", NW), ("MINB", MINB), ("NWR", NWR), ("NCASES", NCASES), ("CH", CH), ("STAGES", STAGES), ("ID", vid),
                 ("NWOPS", len(wops))):
        lines.append(f"    static constexpr int {k} = {v};")
    lines.append(f'    static constexpr const char* NAME = "{name}";')
    lines.append(f"    static constexpr int LOADW = {LW}, EXIT = {EXIT};")
    lines.append("    // Run the entry stream at shared address `stream` (see tools/gen_gather.py).")
    lines.append("    // acc[ty][m], wp[i]: f32x2 bit patterns (x in the low word); wlane: shared")
    lines.append("    // address of this lane's weights of channel `cbase` (first channel of the stage).")
    lines.append("    __device__ __forceinline__ static void run(unsigned long long (&acc)[TY][NX], "
                 "unsigned long long (&wp)[NWOPS], const unsigned stream, const unsigned wlane, "
                 "const unsigned cbase) {")
    lines.append("        asm volatile(")
    for a in asm:
        lines.append(f'            "{a}\\n\\t"')
    outs = ", ".join([f'"+l"(acc[{ty}][{m}])' for (ty, m) in accs] + [f'"+l"(wp[{i}])' for i in range(len(wops))])
    ins = '"r"(stream), "r"(wlane), "r"(cbase)'
    lines.append(f"            : {outs}")
    lines.append(f"            : {ins}")
    lines.append('            : "memory");')
    lines.append("    }")
    lines.append("};")
    return "\n".join(lines)


def main():
    parts = ["// GENERATED by tools/gen_gather.py -- do not edit.  See that script for the derivation.",
             "#pragma once", ""]
    for v in VARIANTS:
        parts.append(gen_variant(*v))
        parts.append("")
    # selection order = first match wins: measured fastest first
    order = sorted(VARIANTS, key=lambda v: PRIORITY.index(v[0]) if v[0] in PRIORITY else 100 + v[0])
    parts.append("#define SC_GATHER_VARIANTS(X) \\")
    parts.append(" \\\n".join(f"    X(V{v[0]})" for v in order))
    parts.append("")
    with open(OUT, "w") as f:
        f.write("\n".join(parts))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
