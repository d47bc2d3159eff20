// Run-time specialisation of the stage-2 kernel (NVRTC).
//
// The library ships generated interpreter kernels for the shapes of the
// BASELINE configs and the paper's Table 2 (gather_variants.inc, written by
// tools/gen_gather.py).  For any other shape the plan used to fall back to the
// generic gather kernel (an order of magnitude slower).  This file generates
// the same kind of variant for the plan's shape at plan creation -- a C++ port
// of tools/gen_gather.py:gen_variant (tests/test_jit_cpu.py checks the two
// produce identical code) -- compiles it together with the self-contained
// device code gather_fast_kernel.cuh through NVRTC for sm_100a, and launches
// it through the driver API.  NVRTC is loaded with dlopen; without it (or if a
// compilation fails) the plan keeps the generic kernel.  Compiled kernels are
// cached per parameter set for the life of the process.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "sc_internal.h"
#include "gather_fast_kernel.cuh"  // sc::fast::Args (the kernel's argument block)

namespace sc {
namespace jit {

namespace {
#include "jit_sources.inc"  // kDeviceHeader (sc_device.h), kKernelHeader (gather_fast_kernel.cuh)
}

// ---------------------------------------------------------------------------
// Variant generator: C++ port of tools/gen_gather.py gen_variant (no ablations)
// ---------------------------------------------------------------------------
std::string gen_variant(const Params& p, const std::string& sname, const std::string& name) {
    const int R = p.R, S = p.S, P = p.P, T = p.T, W = p.W, TY = p.TY, KL = p.KL;
    const int WO = (W + 2 * P - S) / T + 1;
    const bool XPAIR = KL == 1;
    const int NX = XPAIR ? (WO + 1) / 2 : WO;
    const int NPAIR = XPAIR ? 1 : KL / 2;
    const int NSING = XPAIR ? 0 : KL % 2;
    const int NWR = (TY - 1) * T + R;
    const int NCASES = NWR * W;
    std::vector<std::pair<std::string, std::string>> ops;  // (constraint, expression)
    auto key3 = [](int a, int b, int c) { return ((int64_t)a << 40) | ((int64_t)b << 20) | c; };
    std::map<int64_t, int> accp, accs, wp, ws;
    for (int ty = 0; ty < TY; ++ty)
        for (int m = 0; m < NX; ++m)
            for (int pi = 0; pi < NPAIR; ++pi) {
                accp[key3(ty, m, pi)] = (int)ops.size();
                ops.push_back({"\"+l\"", "accp[" + std::to_string(ty) + "][" + std::to_string(m) + "][" +
                                             std::to_string(pi) + "]"});
            }
    for (int ty = 0; ty < TY; ++ty)
        for (int m = 0; m < NX; ++m)
            for (int si = 0; si < NSING; ++si) {
                accs[key3(ty, m, 0)] = (int)ops.size();
                ops.push_back({"\"+f\"", "accs[" + std::to_string(ty) + "][" + std::to_string(m) + "]"});
            }
    std::vector<std::pair<int, int>> wkeys;
    if (XPAIR) {
        for (int r = 0; r < R; ++r)
            for (int u = 1; u < S; ++u) wkeys.push_back({r, u});
    } else {
        for (int r = 0; r < R; ++r)
            for (int t = 0; t < S; ++t) wkeys.push_back({r, t});
    }
    for (auto& k : wkeys)
        for (int pi = 0; pi < NPAIR; ++pi) {
            const int idx = (int)wp.size();
            wp[key3(k.first, k.second, pi)] = (int)ops.size();
            ops.push_back({"\"+l\"", "wp[" + std::to_string(idx) + "]"});
        }
    for (auto& k : wkeys)
        for (int si = 0; si < NSING; ++si) {
            const int idx = (int)ws.size();
            ws[key3(k.first, k.second, 0)] = (int)ops.size();
            ops.push_back({"\"+f\"", "ws[" + std::to_string(idx) + "]"});
        }
    const int n_out = (int)ops.size();
    const int pop = n_out, wlop = n_out + 1, wsop = n_out + 2, cbop = n_out + 3;
    auto op = [](int i) { return "%" + std::to_string(i); };
    auto scalar = [&](int r, int t, std::string* half) {
        if (t >= 1) {
            *half = "lo";
            return wp[key3(r, t, 0)];
        }
        *half = "hi";
        return wp[key3(r, 1, 0)];
    };
    std::vector<std::vector<std::string>> bodies;
    int n_fma = 0;
    for (int wi = 0; wi < NWR; ++wi)
        for (int j = 0; j < W; ++j) {
            std::vector<std::string> body;
            for (int ty = 0; ty < TY; ++ty) {
                const int r = wi - ty * T;
                if (!(0 <= r && r < R)) continue;
                if (!XPAIR) {
                    for (int x = 0; x < WO; ++x) {
                        const int t = j + P - x * T;
                        if (0 <= t && t < S) {
                            for (int pi = 0; pi < NPAIR; ++pi) {
                                const int a = accp[key3(ty, x, pi)];
                                body.push_back("fma.rn.f32x2 " + op(a) + ", " + op(wp[key3(r, t, pi)]) + ", vv, " +
                                               op(a) + ";");
                            }
                            if (NSING) {
                                const int a = accs[key3(ty, x, 0)];
                                body.push_back("fma.rn.f32 " + op(a) + ", " + op(ws[key3(r, t, 0)]) + ", vf, " +
                                               op(a) + ";");
                            }
                        }
                    }
                } else {
                    for (int m = 0; m < NX; ++m) {
                        const int x0 = 2 * m, x1 = 2 * m + 1;
                        const int t0 = j + P - x0, t1 = j + P - x1;
                        const bool in0 = 0 <= t0 && t0 < S;
                        const bool in1 = 0 <= t1 && t1 < S && x1 < WO;
                        const int a = accp[key3(ty, m, 0)];
                        if (in0 && in1) {
                            body.push_back("fma.rn.f32x2 " + op(a) + ", " + op(wp[key3(r, t0, 0)]) + ", vv, " + op(a) +
                                           ";");
                        } else if (in0 || in1) {
                            const int t = in0 ? t0 : t1;
                            const std::string half = in0 ? "l" : "h";
                            std::string wh;
                            const int o = scalar(r, t, &wh);
                            body.push_back("mov.b64 {al, ah}, " + op(a) + "; mov.b64 {wl, wh}, " + op(o) +
                                           "; fma.rn.f32 a" + half + ", w" + wh.substr(0, 1) + ", vf, a" + half +
                                           "; mov.b64 " + op(a) + ", {al, ah};");
                        }
                    }
                }
            }
            n_fma += (int)body.size();
            bodies.push_back(body);
        }
    const int NMASK = 1 << R;
    const int LW = NCASES, EXIT = NCASES + NMASK;
    const int chb = R * S * 32 * KL * 4;
    std::vector<std::string> asm_;
    for (const char* l : {"{", ".reg .b64 vv;", ".reg .b32 xc, cc, xn, cn, ep, ea, es, mk, mr;", ".reg .pred pm, pr;",
                          ".reg .f32 al, ah, wl, wh, vf;"})
        asm_.push_back(l);
    asm_.push_back("mov.b32 ep, " + op(pop) + ";");
    for (const char* l : {"ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;", "LOOP_%=:", "mov.b32 xc, xn;",
                          "mov.b32 cc, cn;", "ld.shared.v2.b32 {xn, cn}, [ep];", "add.u32 ep, ep, 8;",
                          "mov.b64 vv, {xc, xc};", "mov.b32 vf, xc;"})
        asm_.push_back(l);
    std::string ts = "TS_%=: .branchtargets ";
    for (size_t i = 0; i < bodies.size(); ++i) {
        ts += bodies[i].empty() ? std::string("LOOP_%=") : "C" + std::to_string(i) + "_%=";
        ts += ", ";
    }
    for (int m = 0; m < NMASK; ++m) ts += (m ? "LW" + std::to_string(m) + "_%=" : std::string("LOOP_%=")) + ", ";
    ts += "END_%=;";
    asm_.push_back(ts);
    asm_.push_back("brx.idx.uni cc, TS_%=;");
    for (size_t i = 0; i < bodies.size(); ++i) {
        if (bodies[i].empty()) continue;
        asm_.push_back("C" + std::to_string(i) + "_%=:");
        for (auto& b : bodies[i]) asm_.push_back(b);
        asm_.push_back("bra.uni LOOP_%=;");
    }
    const int tap_bytes = 32 * KL * 4;
    for (int m = 1; m < NMASK; ++m) {
        asm_.push_back("LW" + std::to_string(m) + "_%=:");
        asm_.push_back("sub.u32 ea, xc, " + op(cbop) + ";");
        if (NSING) asm_.push_back("mad.lo.u32 es, ea, " + std::to_string(chb) + ", " + op(wsop) + ";");
        asm_.push_back("mad.lo.u32 ea, ea, " + std::to_string(chb) + ", " + op(wlop) + ";");
        if (XPAIR) {
            for (int r = 0; r < R; ++r) {
                if (!((m >> r) & 1)) continue;
                for (int u = 1; u < S; ++u)
                    asm_.push_back("ld.shared.f32 wl, [ea+" + std::to_string((r * S + u) * 128) +
                                   "]; ld.shared.f32 wh, [ea+" + std::to_string((r * S + u - 1) * 128) +
                                   "]; mov.b64 " + op(wp[key3(r, u, 0)]) + ", {wl, wh};");
            }
        } else {
            for (size_t i = 0; i < wkeys.size(); ++i) {
                const int r = wkeys[i].first, t = wkeys[i].second;
                if (!((m >> r) & 1)) continue;
                // pairs (k0,k1),(k2,k3) per 16-byte load when the lane stride (8*NPAIR bytes) keeps
                // them 16-byte aligned (NPAIR even), else one 8-byte load per pair (KL = 6)
                const int step = NPAIR % 2 == 0 ? 2 : 1;
                for (int pi = 0; pi < NPAIR; pi += step) {
                    const std::string off = std::to_string(i * tap_bytes + 8 * pi);
                    if (step == 2)
                        asm_.push_back("ld.shared.v2.b64 {" + op(wp[key3(r, t, pi)]) + ", " +
                                       op(wp[key3(r, t, pi + 1)]) + "}, [ea+" + off + "];");
                    else
                        asm_.push_back("ld.shared.b64 " + op(wp[key3(r, t, pi)]) + ", [ea+" + off + "];");
                }
                if (NSING)
                    asm_.push_back("ld.shared.f32 " + op(ws[key3(r, t, 0)]) + ", [es+" +
                                   std::to_string(i * tap_bytes + 256) + "];");
            }
        }
        asm_.push_back("bra.uni LOOP_%=;");
    }
    asm_.push_back("END_%=:");
    asm_.push_back("}");

    std::string out;
    auto line = [&](const std::string& l) { out += l + "\n"; };
    line("// ---- variant " + std::to_string(p.id) + ": " + name + "  (R=" + std::to_string(R) +
         " S=" + std::to_string(S) + " P=" + std::to_string(P) + " W=" + std::to_string(W) + " WO=" +
         std::to_string(WO) + " TY=" + std::to_string(TY) + " KL=" + std::to_string(KL) + " NX=" +
         std::to_string(NX) + " NW=" + std::to_string(p.NW) + "); " + std::to_string(n_fma) +
         " FMA instructions over " + std::to_string(NCASES) + " window positions");
    line("struct " + sname + " {");
    const std::pair<const char*, int> consts[] = {
        {"R", R}, {"S", S}, {"P", P}, {"T", T}, {"W", W}, {"WO", WO}, {"NX", NX}, {"TY", TY}, {"KL", KL},
        {"NW", p.NW}, {"MINB", p.MINB}, {"NWR", NWR}, {"NCASES", NCASES}, {"CH", p.CH}, {"STAGES", p.STAGES},
        {"ID", p.id}, {"NPAIR", NPAIR}, {"NSING", NSING}, {"NWP", (int)wp.size()},
        {"NWS", ws.empty() ? 1 : (int)ws.size()}, {"SLOTS", p.SLOTS}, {"PIECE", p.PIECE}, {"KMIN", 0}};
    for (auto& c : consts) line(std::string("    static constexpr int ") + c.first + " = " + std::to_string(c.second) + ";");
    line(std::string("    static constexpr bool XPAIR = ") + (XPAIR ? "true" : "false") + ";");
    line("    static constexpr const char* NAME = \"" + name + "\";");
    line("    static constexpr int LOADW = " + std::to_string(LW) + ", EXIT = " + std::to_string(EXIT) +
         ";  // marker codes LOADW + mask, mask < 2^R");
    line("    // Run the entry stream at shared address `stream` (see tools/gen_gather.py).");
    line("    // accp/wp: f32x2 bit patterns (low word = first element); wlane / wlane_s:");
    line("    // shared address of this lane's paired / single weights of channel `cbase`.");
    line("    __device__ __forceinline__ static void run(unsigned long long (&accp)[TY][NX][NPAIR], "
         "float (&accs)[TY][NX], unsigned long long (&wp)[NWP], float (&ws)[NWS], const unsigned stream, "
         "const unsigned wlane, const unsigned wlane_s, const unsigned cbase) {");
    line("        asm volatile(");
    for (auto& a : asm_) line("            \"" + a + "\\n\\t\"");
    std::string outs = "            : ";
    for (size_t i = 0; i < ops.size(); ++i) outs += (i ? ", " : "") + ops[i].first + "(" + ops[i].second + ")";
    line(outs);
    line("            : \"r\"(stream), \"r\"(wlane), \"r\"(wlane_s), \"r\"(cbase)");
    line("            : \"memory\");");
    if (!NSING) line("        (void)accs; (void)ws;");
    line("    }");
    line("};");
    return out;
}

// ---------------------------------------------------------------------------
// Parameter choice for a plan's shape
// ---------------------------------------------------------------------------
static size_t smem_bytes(const Params& p) {
    // mirrors Smem<V> in gather_fast_kernel.cuh
    const int WO = (p.W + 2 * p.P - p.S) / p.T + 1;
    const size_t kbw = 32 * p.KL;
    const size_t stage = (size_t)p.CH * p.R * p.S * kbw;
    const size_t ring = sizeof(float) * p.STAGES * stage;
    const size_t bars = 8 * (2 * p.STAGES + p.NW * p.SLOTS);
    const size_t bars_pad = (bars + 127) / 128 * 128;
    const size_t pieces = 8 * ((size_t)p.NW * p.SLOTS * (p.PIECE + 2) + 4);
    (void)WO;
    return ring + bars_pad + pieces;
}

static bool epilogue_fits(const Params& p) {
    const int WO = (p.W + 2 * p.P - p.S) / p.T + 1;
    const int piece_floats = p.SLOTS * (p.PIECE + 2) * 2;
    int er = ((piece_floats / 32) - 1) / WO;
    if (er < 1) er = 1;
    if (er > p.TY) er = p.TY;
    return 32 * ((er * WO) | 1) <= piece_floats;
}

const char* invalid(const Geometry& g, const Params& p) {
    if (p.R != g.R || p.S != g.S || p.P != g.P || p.T != g.T || p.W != g.W) return "parameters of another shape";
    if (g.R > 7 || g.S > 7 || g.W > 64 || g.T > 3) return "shape outside the generator (R, S <= 7, W <= 64, stride <= 3)";
    if (p.KL != 1 && p.KL != 2 && p.KL != 3 && p.KL != 4 && p.KL != 6 && p.KL != 8)
        return "KL must be 1, 2, 3, 4, 6 or 8 (the weight packings of pack.cu)";
    if (p.KL == 1 && (p.T != 1 || p.S < 2)) return "x-pair tiles (KL = 1) need stride 1 and S >= 2";
    if (p.TY < 1 || p.TY > g.Ho) return "TY outside [1, Ho]";
    const int nwr = (p.TY - 1) * p.T + p.R;
    if (nwr > 31 || nwr * p.W > 2048) return "tile window beyond the jump-table / marker-mask limits";
    if (p.CH < 1 || (g.Cg + p.CH - 1) / p.CH > 63) return "more than 63 weight chunks (raise CH)";
    if (p.NW < 1 || p.STAGES < 1 || p.SLOTS < 1 || p.PIECE < 2) return "NW, STAGES, SLOTS >= 1 and PIECE >= 2";
    if (smem_bytes(p) > 220 * 1024) return "shared memory above 220 KB";
    if (!epilogue_fits(p)) return "epilogue does not fit the piece slots (raise SLOTS or PIECE)";
    return nullptr;
}

bool choose(const Geometry& g, Params* p) {
    *p = Params{};
    if (g.R > 7 || g.S > 7 || g.W > 64 || g.T > 3) return false;
    p->R = (int)g.R; p->S = (int)g.S; p->P = (int)g.P; p->T = (int)g.T; p->W = (int)g.W;
    const int WO = (int)g.Wo;
    // k-slots per lane: four when there are enough filters, x-pairs (KL=1) for few filters at stride 1
    int kl = g.Kg > 96 ? 4 : (g.Kg > 32 ? 2 : 1);
    if (kl == 1 && (g.T != 1 || g.S < 2)) kl = 2;
    // 1x1 at stride 1 with many filters: one-row tiles of the fewest k-blocks (sc_internal.h)
    const bool wide = wide_1x1_kl(g) != 0;
    if (wide) kl = wide_1x1_kl(g);
    p->KL = kl;
    const int nx = kl == 1 ? (WO + 1) / 2 : WO;
    const int acc_row = kl == 1 ? 2 * nx : nx * kl;           // registers per tile row
    const int wregs = kl == 1 ? 2 * p->R * (p->S - 1) : p->R * p->S * kl;
    const int budget = 140;                                    // V21: 104 accumulators + 36 weights
    int ty = (budget - wregs) / acc_row;
    if (ty < 1) return false;
    if (ty > (int)g.Ho) ty = (int)g.Ho;
    if (wide && kl > 4) ty = 1;
    // rebalance: the same number of tiles with the smallest tile height
    const int tiles = ((int)g.Ho + ty - 1) / ty;
    ty = ((int)g.Ho + tiles - 1) / tiles;
    p->TY = ty;
    const int nwr = (ty - 1) * p->T + p->R;
    if (nwr > 31 || nwr * p->W > 2048) return false;          // jump-table / marker-mask limits
    p->NW = 11; p->MINB = 1; p->STAGES = 2; p->SLOTS = 3; p->PIECE = 254;
    // the epilogue reuses the warp's piece slots: wide rows need more of them
    while (!epilogue_fits(*p) && p->SLOTS < 8) ++p->SLOTS;
    p->CH = 16;
    if (wide && kl > 4) { p->CH = 32; p->STAGES = 3; p->SLOTS = 2; }  // V54/V55 ring
    while (!epilogue_fits(*p) && p->SLOTS < 8) ++p->SLOTS;
    while (p->CH > 1 && smem_bytes(*p) > 200 * 1024) p->CH /= 2;
    if ((g.Cg + p->CH - 1) / p->CH > 63) p->CH = (int)((g.Cg + 62) / 63);
    p->id = 1000;
    return invalid(g, *p) == nullptr;
}

// ---------------------------------------------------------------------------
// NVRTC compile + driver-API launch
// ---------------------------------------------------------------------------
namespace {
struct Nvrtc {
    bool ok = false;
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcAddNameExpression) add_name = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) log = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) cubin = nullptr;
    decltype(&nvrtcGetLoweredName) lowered = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
};

Nvrtc& nvrtc() {
    static Nvrtc n = [] {
        Nvrtc r;
        void* h = nullptr;
        for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"})
            if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
        if (!h) return r;
#define SC_SYM(field, sym) r.field = reinterpret_cast<decltype(r.field)>(dlsym(h, #sym));
        SC_SYM(create, nvrtcCreateProgram)
        SC_SYM(add_name, nvrtcAddNameExpression)
        SC_SYM(compile, nvrtcCompileProgram)
        SC_SYM(log_size, nvrtcGetProgramLogSize)
        SC_SYM(log, nvrtcGetProgramLog)
        SC_SYM(cubin_size, nvrtcGetCUBINSize)
        SC_SYM(cubin, nvrtcGetCUBIN)
        SC_SYM(lowered, nvrtcGetLoweredName)
        SC_SYM(destroy, nvrtcDestroyProgram)
#undef SC_SYM
        r.ok = r.create && r.add_name && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.lowered &&
               r.destroy;
        return r;
    }();
    return n;
}

struct Driver {
    bool ok = false;
    PFN_cuModuleLoadData_v2000 load = nullptr;
    PFN_cuModuleGetFunction_v2000 get = nullptr;
    PFN_cuFuncSetAttribute_v9000 set_attr = nullptr;
    PFN_cuLaunchKernel_v4000 launch = nullptr;
};

Driver& driver() {
    static Driver d = [] {
        Driver r;
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuModuleLoadData", &f, cudaEnableDefault, &q) == cudaSuccess && f)
            r.load = reinterpret_cast<PFN_cuModuleLoadData_v2000>(f);
        f = nullptr;
        if (cudaGetDriverEntryPoint("cuModuleGetFunction", &f, cudaEnableDefault, &q) == cudaSuccess && f)
            r.get = reinterpret_cast<PFN_cuModuleGetFunction_v2000>(f);
        f = nullptr;
        if (cudaGetDriverEntryPoint("cuFuncSetAttribute", &f, cudaEnableDefault, &q) == cudaSuccess && f)
            r.set_attr = reinterpret_cast<PFN_cuFuncSetAttribute_v9000>(f);
        f = nullptr;
        if (cudaGetDriverEntryPoint("cuLaunchKernel", &f, cudaEnableDefault, &q) == cudaSuccess && f)
            r.launch = reinterpret_cast<PFN_cuLaunchKernel_v4000>(f);
        r.ok = r.load && r.get && r.set_attr && r.launch;
        return r;
    }();
    return d;
}

std::string key_of(const Params& p) {
    char b[160];
    snprintf(b, sizeof(b), "%d_%d_%d_%d_%d_%d_%d_%d_%d_%d_%d_%d_%d", p.R, p.S, p.P, p.T, p.W, p.TY, p.KL, p.NW,
             p.MINB, p.CH, p.STAGES, p.SLOTS, p.PIECE);
    return b;
}

std::mutex g_mu;
std::map<std::pair<int, std::string>, std::pair<CUfunction, CUfunction>>& cache() {
    static std::map<std::pair<int, std::string>, std::pair<CUfunction, CUfunction>> c;
    return c;
}
thread_local std::string g_log;
}  // namespace

bool available() { return nvrtc().ok && driver().ok; }

const char* last_log() { return g_log.c_str(); }

cudaError_t compile(const Params& p, int device, void** fn, void** fn_gated, size_t* smem) {
    *fn = *fn_gated = nullptr;
    *smem = smem_bytes(p);
    if (!available()) return cudaErrorNotSupported;
    const std::string key = key_of(p);
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = cache().find({device, key});
    if (it != cache().end()) {
        *fn = reinterpret_cast<void*>(it->second.first);
        *fn_gated = reinterpret_cast<void*>(it->second.second);
        return cudaSuccess;
    }
    Nvrtc& nv = nvrtc();
    const std::string src = std::string("#include \"sc_device.h\"\nnamespace sc {\nnamespace fast {\n") +
                            gen_variant(p, "VJ", "jit_" + key) +
                            "}  // namespace fast\n}  // namespace sc\n#include \"gather_fast_kernel.cuh\"\n";
    const char* headers[] = {kDeviceHeader, kKernelHeader};
    const char* names[] = {"sc_device.h", "gather_fast_kernel.cuh"};
    nvrtcProgram prog;
    if (nv.create(&prog, src.c_str(), "sc_jit_gather.cu", 2, headers, names) != NVRTC_SUCCESS)
        return cudaErrorNotSupported;
    const char* expr[2] = {"sc::fast::gather_fast_kernel<sc::fast::VJ, false, sc::fast::Args>",
                           "sc::fast::gather_fast_kernel<sc::fast::VJ, false, sc::fast::ArgsGated>"};
    nv.add_name(prog, expr[0]);
    nv.add_name(prog, expr[1]);
    const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-ftz=false", "-prec-div=true",
                          "-prec-sqrt=true", "-fmad=true", "-lineinfo"};
    const nvrtcResult rc = nv.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
    size_t ls = 0;
    nv.log_size(prog, &ls);
    g_log.assign(ls, '\0');
    if (ls) nv.log(prog, &g_log[0]);
    if (rc != NVRTC_SUCCESS) {
        nv.destroy(&prog);
        return cudaErrorNotSupported;
    }
    size_t cs = 0;
    nv.cubin_size(prog, &cs);
    std::vector<char> cubin(cs);
    nv.cubin(prog, cubin.data());
    std::string lname[2];
    for (int i = 0; i < 2; ++i) {
        const char* lowered = nullptr;
        nv.lowered(prog, expr[i], &lowered);
        lname[i] = lowered ? lowered : "";
    }
    nv.destroy(&prog);
    Driver& dr = driver();
    CUmodule mod;
    CUfunction f[2];
    if (dr.load(&mod, cubin.data()) != CUDA_SUCCESS) return cudaErrorNotSupported;  // stays loaded (cached)
    for (int i = 0; i < 2; ++i)
        if (dr.get(&f[i], mod, lname[i].c_str()) != CUDA_SUCCESS ||
            dr.set_attr(f[i], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)*smem) != CUDA_SUCCESS)
            return cudaErrorNotSupported;
    cache()[{device, key}] = {f[0], f[1]};
    *fn = reinterpret_cast<void*>(f[0]);
    *fn_gated = reinterpret_cast<void*>(f[1]);
    return cudaSuccess;
}

size_t variant_source(const Params& p, char* buf, size_t cap) {
    const std::string s = gen_variant(p, "V" + std::to_string(p.id), "jit");
    if (buf && cap) {
        const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
        memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
    return s.size();
}

// Same argument block and grid as fast::launch_v (gather_fast_impl.cuh); a non-null gate
// selects the gated instantiation (fn must then be the gated kernel).
cudaError_t launch(void* fn, size_t smem, const Params& p, const Geometry& g, int64_t n, const uint2* entries,
                   const uint32_t* offs, const float* wpack, const float* bias, float* out, cudaStream_t st,
                   Gate gate) {
    if (!fn || g.ty != p.TY || invalid(g, p)) return cudaErrorInvalidValue;
    fast::ArgsGated ag;
    fast::Args& a = ag;
    a.entries = entries; a.offs = offs; a.wpack = wpack; a.bias = bias; a.out = out;
    a.rowlist = nullptr; a.rowcnt = nullptr;
    a.n = (int)n; a.C = (int)g.C; a.H = (int)g.H; a.K = (int)g.K; a.Cg = (int)g.Cg; a.Kg = (int)g.Kg;
    a.kblocks = (int)g.kblocks; a.Ho = (int)g.Ho; a.relu = g.relu ? 1 : 0;
    a.cap = g.cap;
    a.ytiles = (int)g.tiles;
    a.units = (int)n * a.ytiles;
    a.ctas_per_kb = (a.units + p.NW - 1) / p.NW;
    {
        int d = 0, sms = 148;
        if (cudaGetDevice(&d) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d) != cudaSuccess)
            sms = 148;
        a.edge_last = edge_last_order((int64_t)a.ctas_per_kb * g.G * g.kblocks >= 2LL * sms * p.MINB);
    }
    ag.gate = gate;
    const int64_t grid = (int64_t)a.ctas_per_kb * g.G * g.kblocks;
    void* pa = gate.flag ? static_cast<void*>(&ag) : static_cast<void*>(&a);
    void* params[] = {pa};
    const CUresult r = driver().launch(reinterpret_cast<CUfunction>(fn), (unsigned)grid, 1, 1,
                                       (unsigned)(p.NW + 1) * 32, 1, 1, (unsigned)smem,
                                       reinterpret_cast<CUstream>(st), params, nullptr);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

}  // namespace jit
}  // namespace sc
