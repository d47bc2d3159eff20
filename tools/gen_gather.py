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
compare tree instead, and a dispatch at the end of every block ("threaded
code") gets one PC-relative jump table per site (constant-cache thrash,
measured 2-4x slower).

Register-tile forms (KL = output channels per lane, lane l owns channels
KL*l .. KL*l+KL-1 of the warp's k-block):
* KL=1 "x-pair": acc[ty][m] pairs two horizontally adjacent outputs
  (x = 2m, 2m+1) of one channel.  Where both outputs are in the nonzero's
  footprint one FFMA2 with the weight pair (W[r][u], W[r][u-1]), u = j+P-2m,
  updates both; where only one is, a single FFMA.
* KL>=2: per output pixel NPAIR = KL/2 f32x2 accumulators over channel pairs
  (k0,k1), (k2,k3) and, for odd KL, one f32 accumulator (k2).  Per in-tile tap:
  NPAIR FFMA2 (nonzero value as broadcast scalar) + one FFMA for odd KL.
  The weights of a tap are one 64-bit (KL=2), one 128-bit (KL=4) or a 64-bit
  + 32-bit pair of shared-memory loads (KL=3, layout of pack.cu).
Every FMA issue slot retires KL lane-FMAs per in-tile tap: the work per
(~8-instruction, ~100-cycle-latency) dispatch grows with KL.

Usage: python tools/gen_gather.py  (rewrites the .inc; commit the result).
"""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_1704_07724_b200", "csrc", "gather_variants.inc")

# (id, name, R, S, P, W, TY, KL, NW, MINB, CH, STAGES): stride 1 only.  W = input width.
# NW compute warps (+1 producer warp) per CTA, MINB CTAs per SM (register budget
# 65536 / (32*(NW+1)*MINB)).
VARIANTS = [
    # k-quads, 3 warps/SMSP, 16-channel weight chunks in a 2-stage ring: measured best of the
    # CH/STAGES/SLOTS/PIECE sweep
    (21, "r3s3p1_w13_ty2_kl4_nw11_ch16s2", 3, 3, 1, 13, 2, 4, 11, 1, 16, 2),   # C2, C5 (AlexNet conv3/4/5)
    (33, "r5s5p2_w27_ty3_kl1_nw11", 5, 5, 2, 27, 3, 1, 11, 1, 16, 2),        # C3: x-pairs
    # round 2: best of whole-forward sweeps (stage 1 depends on the tile height too;
    # profiles/r2_jit_tune_*.txt), replacing V5 / V28 / V29
    (57, "r5s5p0_w12_ty1_kl1_nw7_ch10", 5, 5, 0, 12, 1, 1, 7, 1, 10, 2),     # C1: x-pairs, 7 warps (pipelined batches)
    (51, "r3s3p1_w28_ty2_kl2_nw11_ch32", 3, 3, 1, 28, 2, 2, 11, 1, 32, 2),   # C4a: k-pairs
    (52, "r5s5p2_w28_ty3_kl1_nw11", 5, 5, 2, 28, 3, 1, 11, 1, 16, 2),        # C4b: x-pairs
    # paper Table 2 shapes: stride 2, 1x1, small planes
    # (parameters from tools/jit_tune.py sweeps of run-time generated variants, profiles/r1_jit_tune_t2.txt)
    (40, "r5s5p1t2_w11_ty2_kl2_sl2p126", 5, 5, 1, 11, 2, 2, 11, 1, 16, 2, None, 2, 126, 2),  # LeNet-Conv2 (T=2)
    (41, "r5s5p2_w6_ty1_kl1_s3sl2p126", 5, 5, 2, 6, 1, 1, 11, 1, 16, 3, None, 2, 126),     # AlexNetC-Conv3
    (42, "r3s3p1_w5_ty3_kl2_sl2", 3, 3, 1, 5, 3, 2, 11, 1, 16, 2, None, 2, 254),           # AlexNetI-Conv4
    (43, "r1s1p0_w14_ty2_kl4", 1, 1, 0, 14, 2, 4, 11, 1, 32, 2),                           # Inception4a.2
    (44, "r3s3p1_w14_ty3_kl2_s3sl2", 3, 3, 1, 14, 3, 2, 11, 1, 16, 3, None, 2, 254),       # Inception4e.3
    (45, "r1s1p0_w7_ty2_kl2_sl2", 1, 1, 0, 7, 2, 2, 11, 1, 16, 2, None, 2, 254),           # Inception5a.2
    (46, "r3s3p1_w7_ty2_kl4_p126", 3, 3, 1, 7, 2, 4, 11, 1, 16, 2, None, 3, 126),          # Inception5b.3
    (47, "r5s5p2_w7_ty2_kl2_sl2p126", 5, 5, 2, 7, 2, 2, 11, 1, 16, 2, None, 2, 126),       # Inception5b.5
    # round 2: 1x1 layers with one dispatch per nonzero for all of a k-block of 32*KL >= Kg
    # channels (KL = 6, 8; no halo, so the tile height buys no reuse: TY = 1), 32-channel
    # weight chunks (profiles/r2_t2_kl68_tune.txt), replacing V48 / V49.  KMIN > 0 marks them:
    # they match only where KL is sc_internal.h wide_1x1_kl's choice (fewest k-blocks)
    (53, "r1s1p0_w14_ty1_kl6_ch32sl2_k150", 1, 1, 0, 14, 1, 6, 11, 1, 32, 2, None, 2, 254, 1, 150),  # Inception4a.1
    (54, "r1s1p0_w7_ty1_kl8_ch32s3_k150", 1, 1, 0, 7, 1, 8, 11, 1, 32, 3, None, 3, 254, 1, 150),     # Inception5a.1
    (55, "r1s1p0_w7_ty1_kl6_ch32s3sl2p510_k150", 1, 1, 0, 7, 1, 6, 11, 1, 32, 3, None, 2, 510, 1, 150),  # Inception5a.2
    (56, "r1s1p0_w14_ty1_kl8_ch32sl2_k150", 1, 1, 0, 14, 1, 8, 11, 1, 32, 2, None, 2, 254, 1, 150),  # 14x14, Kg 193-256
]

# Superseded round-1 tilings (slower than the shipped variant of the same shape, DESIGN.md
# "Stage 2") and the V12 ablations (wrong results by design: timing studies only).  Not built
# into libsparseconv.so; any of them can be generated at run time for tuning or tests with
# SC_JIT_FORCE="TY,KL,NW,MINB,CH,STAGES,SLOTS,PIECE" (csrc/jit.cu).
SUPERSEDED = [
    (50, "r5s5p0_w12_ty1_kl1_nw4_ch10", 5, 5, 0, 12, 1, 1, 4, 1, 10, 2),     # C1 until late round 2 (equal single
                                                                               # batch, 8% slower pipelined)
    (48, "r1s1p0_w14_ty3_kl3_sl2_k150", 1, 1, 0, 14, 3, 3, 11, 1, 16, 2, None, 2, 254, 1, 150),  # Inception4a.1 until round 2
    (49, "r1s1p0_w7_ty2_kl4_s3p510_k200", 1, 1, 0, 7, 2, 4, 11, 1, 16, 3, None, 3, 510, 1, 200),  # Inception5a.1 until round 2
    (5, "r5s5p0_w12_ty6_kl2", 5, 5, 0, 12, 6, 2, 7, 1, 4, 4),      # C1 until round 2
    (28, "r3s3p1_w28_ty1_kl4_nw11_ch16s2", 3, 3, 1, 28, 1, 4, 11, 1, 16, 2),   # C4a until round 2
    (29, "r5s5p2_w28_ty4_kl1_nw11", 5, 5, 2, 28, 4, 1, 11, 1, 16, 2),        # C4b until round 2
    (1, "r3s3p1_w13_ty7_kl2", 3, 3, 1, 13, 7, 2, 7, 1, 8, 4),      # C2
    (2, "r3s3p1_w28_ty3_kl2", 3, 3, 1, 28, 3, 2, 7, 1, 8, 4),      # C4a
    (3, "r5s5p2_w27_ty2_kl2", 5, 5, 2, 27, 2, 2, 7, 1, 4, 4),      # C3
    (4, "r5s5p2_w28_ty2_kl2", 5, 5, 2, 28, 2, 2, 7, 1, 4, 4),      # C4b
    (7, "r3s3p1_w13_ty7_kl1_nw11", 3, 3, 1, 13, 7, 1, 11, 1, 16, 4),  # C2: x-pairs
    (10, "r3s3p1_w13_ty3_kl3_nw11", 3, 3, 1, 13, 3, 3, 11, 1, 8, 4),  # C2: k-triples
    (11, "r3s3p1_w13_ty3_kl4_nw7", 3, 3, 1, 13, 3, 4, 7, 1, 8, 3),    # C2: k-quads, 2 warps/SMSP
    (12, "r3s3p1_w13_ty2_kl4_nw11", 3, 3, 1, 13, 2, 4, 11, 1, 8, 3),  # C2: V21 with 8-channel chunks
    (13, "r3s3p1_w13_ty5_kl2_nw11", 3, 3, 1, 13, 5, 2, 11, 1, 8, 4),  # C2: k-pairs
    (14, "r3s3p1_w28_ty1_kl4_nw11", 3, 3, 1, 28, 1, 4, 11, 1, 8, 3),  # C4a: k-quads
    (30, "r5s5p2_w28_ty2_kl1_nw11", 5, 5, 2, 28, 2, 1, 11, 1, 16, 2),  # C4b
]
ABLATIONS = [
    (90, "ablate_v12_noload", 3, 3, 1, 13, 2, 4, 11, 1, 8, 3, "noload"),
    (91, "ablate_v12_nofma", 3, 3, 1, 13, 2, 4, 11, 1, 8, 3, "nofma"),
]

# selection order = first match wins (measured fastest first)
PRIORITY = [21, 51, 52, 33, 57, 53, 54, 55, 56]  # 53-56: Kg >= KMIN and KL = wide_1x1_kl


def gen_variant(vid, name, R, S, P, W, TY, KL, NW, MINB, CH, STAGES, ablate=None, SLOTS=3, PIECE=254, T=1, KMIN=0):
    WO = (W + 2 * P - S) // T + 1
    XPAIR = KL == 1
    assert not (XPAIR and T != 1), "x-pair tiles assume stride 1"
    NX = (WO + 1) // 2 if XPAIR else WO            # accumulator columns per row
    NPAIR = 1 if XPAIR else KL // 2                 # f32x2 accumulators per (ty, m)
    NSING = 0 if XPAIR else KL % 2                  # f32 accumulators per (ty, m)
    NWR = (TY - 1) * T + R                           # window rows (R9)
    NCASES = NWR * W
    ops = []                                         # asm operand list: (constraint, C++ expression)
    accp = {}
    for ty in range(TY):
        for m in range(NX):
            for pi in range(NPAIR):
                accp[(ty, m, pi)] = len(ops)
                ops.append(('"+l"', f"accp[{ty}][{m}][{pi}]"))
    accs = {}
    for ty in range(TY):
        for m in range(NX):
            for si in range(NSING):
                accs[(ty, m)] = len(ops)
                ops.append(('"+f"', f"accs[{ty}][{m}]"))
    if XPAIR:
        assert S >= 2
        wkeys = [(r, u) for r in range(R) for u in range(1, S)]       # pair (W[r][u], W[r][u-1])
    else:
        wkeys = [(r, t) for r in range(R) for t in range(S)]
    wp = {}
    for key in wkeys:
        for pi in range(NPAIR):
            wp[(key, pi)] = len(ops)
            ops.append(('"+l"', f"wp[{len(wp) - 1}]"))
    ws = {}
    for key in wkeys:
        for si in range(NSING):
            ws[key] = len(ops)
            ops.append(('"+f"', f"ws[{len(ws) - 1}]"))
    n_out = len(ops)
    pop, wlop, wsop, cbop = n_out, n_out + 1, n_out + 2, n_out + 3

    def scalar(r, t):
        """(operand, half) holding W[r][t] inside the KL=1 weight pairs."""
        if t >= 1:
            return wp[((r, t), 0)], "lo"          # lo of (W[r][t], W[r][t-1])
        return wp[((r, 1), 0)], "hi"              # hi of (W[r][1], W[r][0])

    bodies = []
    n_fma = 0
    for wi in range(NWR):
        for j in range(W):
            body = []
            for ty in range(TY):
                r = wi - ty * T   # window row wi = ty*T + r (R9)
                if not (0 <= r < R):
                    continue
                if not XPAIR:
                    for x in range(WO):
                        t = j + P - x * T
                        if 0 <= t < S:
                            for pi in range(NPAIR):
                                a = accp[(ty, x, pi)]
                                body.append(f"fma.rn.f32x2 %{a}, %{wp[((r, t), pi)]}, vv, %{a};")
                            if NSING:
                                a = accs[(ty, x)]
                                body.append(f"fma.rn.f32 %{a}, %{ws[(r, t)]}, vf, %{a};")
                else:
                    for m in range(NX):
                        x0, x1 = 2 * m, 2 * m + 1
                        t0, t1 = j + P - x0, j + P - x1
                        in0 = 0 <= t0 < S
                        in1 = 0 <= t1 < S and x1 < WO
                        a = accp[(ty, m, 0)]
                        if in0 and in1:
                            body.append(f"fma.rn.f32x2 %{a}, %{wp[((r, t0), 0)]}, vv, %{a};")
                        elif in0 or in1:
                            t = t0 if in0 else t1
                            half = "l" if in0 else "h"
                            o, wh = scalar(r, t)
                            body.append(f"mov.b64 {{al, ah}}, %{a}; mov.b64 {{wl, wh}}, %{o}; "
                                        f"fma.rn.f32 a{half}, w{wh[0]}, vf, a{half}; mov.b64 %{a}, {{al, ah}};")
            if ablate == "nofma" and body:
                body = ["mov.b32 ea, ea;"]
            bodies.append(body)
            n_fma += len(body)
    # ---- interpreter over a shared-memory entry stream ------------------
    # entry = (x, code): code < NCASES: nonzero with value bits x at window
    # position `code`; code == NCASES: channel marker, x = channel index ->
    # load the lane's weights of channel x from the weight stage;
    # code == NCASES+1: exit.  The next entry is loaded before the current one
    # is dispatched.
    # marker code = NCASES + mask (R9): bit r = filter row r is reached by one of the
    # channel's entries; one marker case per mask loads exactly those rows' weights
    NMASK = 1 << R
    LW, EXIT = NCASES, NCASES + NMASK
    chb = R * S * 32 * KL * 4   # bytes of one channel in the weight stage
    if ablate == "pf2":  # entries prefetched two dispatches ahead
        asm = ["{", ".reg .b64 vv;", ".reg .b32 xc, cc, xn, cn, x2, c2, ep, ea, es;", ".reg .f32 al, ah, wl, wh, vf;",
               f"mov.b32 ep, %{pop};",
               "ld.shared.v2.b32 {xn, cn}, [ep];", "ld.shared.v2.b32 {x2, c2}, [ep+8];", "add.u32 ep, ep, 16;",
               "LOOP_%=:",
               "mov.b32 xc, xn;", "mov.b32 cc, cn;", "mov.b32 xn, x2;", "mov.b32 cn, c2;",
               "ld.shared.v2.b32 {x2, c2}, [ep];", "add.u32 ep, ep, 8;",
               "mov.b64 vv, {xc, xc};", "mov.b32 vf, xc;"]
    else:
        asm = ["{", ".reg .b64 vv;", ".reg .b32 xc, cc, xn, cn, ep, ea, es, mk, mr;", ".reg .pred pm, pr;",
               ".reg .f32 al, ah, wl, wh, vf;",
               f"mov.b32 ep, %{pop};",
               "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
               "LOOP_%=:",
               "mov.b32 xc, xn;", "mov.b32 cc, cn;",
               "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
               "mov.b64 vv, {xc, xc};", "mov.b32 vf, xc;"]
    if ablate == "inline":
        # markers (code >= LOADW) leave through a direct branch before the jump table;
        # only nonzero entries pay the LDC + BRX dispatch
        asm.append(f"setp.ge.u32 pm, cc, {LW};")
        asm.append("@pm bra.uni MK_%=;")
        labels = [f"C{i}_%=" if b else "LOOP_%=" for i, b in enumerate(bodies)]
    else:
        labels = ([f"C{i}_%=" if b else "LOOP_%=" for i, b in enumerate(bodies)] +
                  [f"LW{m}_%=" if m else "LOOP_%=" for m in range(NMASK)] + ["END_%="])
    asm.append("TS_%=: .branchtargets " + ", ".join(labels) + ";")
    asm.append("brx.idx.uni cc, TS_%=;")
    for i, b in enumerate(bodies):
        if b:
            asm.append(f"C{i}_%=:")
            asm += b
            asm.append("bra.uni LOOP_%=;")
    tap_bytes = 32 * KL * 4
    if ablate == "inline":
        # marker: EXIT leaves; otherwise mask = code - LOADW, weights of the masked filter
        # rows loaded with row-predicated shared loads (no jump table)
        asm.append("MK_%=:")
        asm.append(f"setp.ge.u32 pm, cc, {EXIT};")
        asm.append("@pm bra.uni END_%=;")
        asm.append(f"sub.u32 mk, cc, {LW};")
        asm.append(f"sub.u32 ea, xc, %{cbop};")
        if NSING:
            asm.append(f"mad.lo.u32 es, ea, {chb}, %{wsop};")
        asm.append(f"mad.lo.u32 ea, ea, {chb}, %{wlop};")
        for r in range(R):
            asm.append(f"and.b32 mr, mk, {1 << r};")
            asm.append("setp.ne.u32 pr, mr, 0;")
            for i, key in enumerate(wkeys):
                if key[0] != r:
                    continue
                if XPAIR:
                    pass
                elif NPAIR == 1:
                    asm.append(f"@pr ld.shared.b64 %{wp[(key, 0)]}, [ea+{i * tap_bytes}];")
                else:
                    asm.append(f"@pr ld.shared.v2.b64 {{%{wp[(key, 0)]}, %{wp[(key, 1)]}}}, [ea+{i * tap_bytes}];")
                if NSING:
                    asm.append(f"@pr ld.shared.f32 %{ws[key]}, [es+{i * tap_bytes + 256}];")
            if XPAIR:
                for u in range(1, S):
                    asm.append(f"@pr ld.shared.f32 wl, [ea+{(r * S + u) * 128}];")
                    asm.append(f"@pr ld.shared.f32 wh, [ea+{(r * S + u - 1) * 128}];")
                    asm.append(f"@pr mov.b64 %{wp[((r, u), 0)]}, {{wl, wh}};")
        asm.append("bra.uni LOOP_%=;")
    for m in range(1, NMASK if ablate != "inline" else 1):
        asm.append(f"LW{m}_%=:")
        asm.append(f"sub.u32 ea, xc, %{cbop};")
        if NSING:
            asm.append(f"mad.lo.u32 es, ea, {chb}, %{wsop};")
        asm.append(f"mad.lo.u32 ea, ea, {chb}, %{wlop};")
        rows = [r for r in range(R) if (m >> r) & 1]
        if ablate == "noload":
            pass
        elif XPAIR:
            for r in rows:
                for u in range(1, S):
                    # pair (W[r][u], W[r][u-1]); weights of tap (r,t) at byte (r*S+t)*128 + lane*4
                    asm.append(f"ld.shared.f32 wl, [ea+{(r * S + u) * 128}]; ld.shared.f32 wh, [ea+{(r * S + u - 1) * 128}]; "
                               f"mov.b64 %{wp[((r, u), 0)]}, {{wl, wh}};")
        else:
            for i, key in enumerate(wkeys):
                if key[0] not in rows:
                    continue
                # the lane's KL weights of a tap (lane-contiguous, 8*NPAIR bytes per lane, pack.cu):
                # pairs (k0,k1),(k2,k3) per 16-byte load when the lane stride keeps them 16-byte
                # aligned (NPAIR even), else one 8-byte load per pair (KL = 6)
                step = 2 if NPAIR % 2 == 0 else 1
                for pi in range(0, NPAIR, step):
                    off = i * tap_bytes + 8 * pi
                    if step == 2:
                        asm.append(f"ld.shared.v2.b64 {{%{wp[(key, pi)]}, %{wp[(key, pi + 1)]}}}, [ea+{off}];")
                    else:
                        asm.append(f"ld.shared.b64 %{wp[(key, pi)]}, [ea+{off}];")
                if NSING:
                    asm.append(f"ld.shared.f32 %{ws[key]}, [es+{i * tap_bytes + 256}];")
        asm.append("bra.uni LOOP_%=;")
    asm.append("END_%=:")
    asm.append("}")
    lines = [f"// ---- variant {vid}: {name}  (R={R} S={S} P={P} W={W} WO={WO} TY={TY} KL={KL} NX={NX} NW={NW}); "
             f"{n_fma} FMA instructions over {NCASES} window positions"]
    lines.append(f"struct V{vid} {{")
    for k, v in (("R", R), ("S", S), ("P", P), ("T", T), ("W", W), ("WO", WO), ("NX", NX), ("TY", TY), ("KL", KL),
                 ("NW", NW), ("MINB", MINB), ("NWR", NWR), ("NCASES", NCASES), ("CH", CH), ("STAGES", STAGES), ("ID", vid),
                 ("NPAIR", NPAIR), ("NSING", NSING), ("NWP", len(wp)), ("NWS", max(1, len(ws))),
                 ("SLOTS", SLOTS), ("PIECE", PIECE), ("KMIN", KMIN)):
        lines.append(f"    static constexpr int {k} = {v};")
    lines.append(f"    static constexpr bool XPAIR = {'true' if XPAIR else 'false'};")
    lines.append(f'    static constexpr const char* NAME = "{name}";')
    lines.append(f"    static constexpr int LOADW = {LW}, EXIT = {EXIT};  // marker codes LOADW + mask, mask < 2^R")
    lines.append("    // Run the entry stream at shared address `stream` (see tools/gen_gather.py).")
    lines.append("    // accp/wp: f32x2 bit patterns (low word = first element); wlane / wlane_s:")
    lines.append("    // shared address of this lane's paired / single weights of channel `cbase`.")
    lines.append("    __device__ __forceinline__ static void run(unsigned long long (&accp)[TY][NX][NPAIR], "
                 "float (&accs)[TY][NX], unsigned long long (&wp)[NWP], float (&ws)[NWS], const unsigned stream, "
                 "const unsigned wlane, const unsigned wlane_s, const unsigned cbase) {")
    lines.append("        asm volatile(")
    for a in asm:
        lines.append(f'            "{a}\\n\\t"')
    lines.append("            : " + ", ".join(f"{c}({e})" for c, e in ops))
    lines.append('            : "r"(stream), "r"(wlane), "r"(wlane_s), "r"(cbase)')
    lines.append('            : "memory");')
    if not NSING:
        lines.append("        (void)accs; (void)ws;")
    lines.append("    }")
    lines.append("};")
    return "\n".join(lines)


def main():
    parts = ["// GENERATED by tools/gen_gather.py -- do not edit.  See that script for the derivation.",
             "#pragma once", ""]
    for v in VARIANTS:
        parts.append(gen_variant(*v))
        parts.append("")
    order = sorted(VARIANTS, key=lambda v: PRIORITY.index(v[0]) if v[0] in PRIORITY else 100 + v[0])
    parts.append("#define SC_GATHER_VARIANTS(X) \\")
    parts.append(" \\\n".join(f"    X(V{v[0]})" for v in order))
    parts.append("")
    with open(OUT, "w") as f:
        f.write("\n".join(parts))
    print("wrote", OUT)
    # one translation unit per variant (parallel compilation)
    csrc = os.path.dirname(OUT)
    for fn in os.listdir(csrc):
        if fn.startswith("gather_fast_v") and fn.endswith(".cu"):
            os.remove(os.path.join(csrc, fn))
    for v in VARIANTS:
        with open(os.path.join(csrc, f"gather_fast_v{v[0]}.cu"), "w") as f:
            f.write(f"// Variant V{v[0]} of the register-tile gather kernel (see gather_fast_impl.cuh).\n"
                    f"#include \"gather_fast_impl.cuh\"\nSC_INSTANTIATE_VARIANT(V{v[0]})\n")


if __name__ == "__main__":
    main()
