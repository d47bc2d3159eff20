// C ABI of libsparseconv.so (include/sparse_conv.h): validation, plan
// lifetime, launch sequencing.  No computation happens on the host.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "sc_internal.h"

using sc::BwdGeom;
using sc::DenseGeom;
using sc::Geometry;

struct sc_plan_s {
    sc_conv_params params;
    int device;
    Geometry g;
    DenseGeom dg;
    BwdGeom bg;
    float* bws = nullptr;      // backward: wgrad partials [splits_w][K][Cg][R][S]
    float* bdt = nullptr;      // backward: k-contiguous copy of dout [N][G][kchunks][Ho*Wo][kc]
    float* wpack = nullptr;    // [G][Kg_pad/kbw][Cg][R][S][kbw] (pack.cu)
    float* wdense = nullptr;   // dense path A operand [G][mtiles][kblocks][128x32], TF32, swizzled
    float* nhwc = nullptr;     // dense path: channels-last TF32 copy of the input [N][H][W][Cp]
    alignas(64) unsigned char bmap[128];  // dense path: TMA map of nhwc
    float* bias = nullptr;     // [K]
    uint2* entries = nullptr;  // stage-1 tile streams [N][tiles][cap] (+2 entries of slack)
    uint32_t* offs = nullptr;  // [N][tiles][C+1]
    uint32_t* cnt = nullptr;   // stage-1 counts [N][tiles][C] (plane-major compaction)
    uint2* plist = nullptr;    // stage-1 per-plane compacted lists [N*C][H*W]
    uint32_t* prow = nullptr;  // stage-1 per-plane row prefixes [N*C][H+1]
    // what plist/prow hold after the last enqueued stage 1 (sparse_conv_plane_lists):
    // 0 nothing valid, 1 plane lists + row prefixes, 2 a producer's per-row slots + row counts
    int lists_layout = 0;
    int variant = 0;           // > 0 generated variant, 0 generic kernel, -1 run-time generated (jit.cu)
    const char* variant_name = "generic";
    sc::jit::Params jp;        // variant -1: its parameters, kernels (ungated, gated) and shared memory
    void* jit_fn = nullptr;
    void* jit_fn_gated = nullptr;
    size_t jit_smem = 0;
    char jit_name[96] = {0};
    // staging for sparse_conv_forward_host and calibration (allocated on first use)
    float* stage_in = nullptr;
    float* stage_out = nullptr;
    // f3 crossover: device words (nnz, ticket, path flag, last nnz) and s* (< 0: unset)
    unsigned long long* sel = nullptr;
    double s_star = -1.0;
    // sparse_conv_forward_host pipeline (created on first use): copy-in, compute and
    // copy-out streams, per-chunk events
    static constexpr int kHostChunks = 8;
    static constexpr int kHostComp = 4;  // compute streams (chunks use disjoint workspace slices)
    cudaStream_t hs[2 + kHostComp] = {};  // [0] copy-in, [1] copy-out, [2..] compute
    cudaEvent_t ev_in[kHostChunks] = {}, ev_comp[kHostChunks] = {}, ev_start = nullptr, ev_done = nullptr;
    // sparse_conv_forward_host_batches: a second staging set and, per set and chunk, copy-in /
    // kernels / copy-out events (created on first use)
    float* stage_in2 = nullptr;
    float* stage_out2 = nullptr;
    cudaEvent_t hb_in[2][kHostChunks] = {}, hb_comp[2][kHostChunks] = {}, hb_out[2][kHostChunks] = {};
    // sparse_conv_forward_batches (sparse_conv_reserve_batches): a second stage-1 workspace, a
    // low-priority stage-1 stream [0] and two high-priority stage-2 streams [1], [2]
    uint2* entries2 = nullptr;
    uint32_t* offs2 = nullptr;
    uint32_t* cnt2 = nullptr;
    uint2* plist2 = nullptr;
    uint32_t* prow2 = nullptr;
    cudaStream_t bs[3] = {};
    cudaEvent_t bev_fork = nullptr, bev_s1 = nullptr, bev_g[2] = {};
    // sparse_conv_backward: dgrad + dbias on a second stream beside wgrad (created on first use)
    cudaStream_t bwd_s2 = nullptr;
    cudaEvent_t bwd_fork = nullptr, bwd_join = nullptr;
};

namespace {

thread_local std::string g_last_error;

sc_status fail(sc_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
sc_status fail(sc_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

sc_status cuda_fail(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation)
        return fail(SC_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
    return fail(SC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

constexpr int64_t kMaxElems = (int64_t(1) << 31) - 1;

sc_status validate_params(const sc_conv_params* p) {
    if (!p) return fail(SC_ERR_INVALID_ARGUMENT, "params is NULL");
    if (p->n < 1 || p->c < 1 || p->h < 1 || p->w < 1 || p->k < 1 || p->r < 1 || p->s < 1 ||
        p->stride < 1 || p->groups < 1)
        return fail(SC_ERR_SHAPE, "extents, stride and groups must be >= 1");
    if (p->pad < 0) return fail(SC_ERR_SHAPE, "pad must be >= 0");
    if (p->r > p->h + 2 * p->pad || p->s > p->w + 2 * p->pad)
        return fail(SC_ERR_SHAPE, "kernel %lldx%lld larger than padded input", (long long)p->r, (long long)p->s);
    if (p->c % p->groups || p->k % p->groups) return fail(SC_ERR_SHAPE, "groups must divide C and K");
    if (p->flags & ~SC_FLAG_FUSE_RELU) return fail(SC_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", p->flags);
    return SC_OK;
}

// Reading R9: tile-stream format for row tiles of `ty` output rows.
void stream_format(Geometry* g, int64_t ty) {
    g->ty = ty;
    g->tiles = (g->Ho + ty - 1) / ty;
    g->nwr = (ty - 1) * g->T + g->R;
    g->nwin = g->nwr * g->W;
    const int64_t rows = g->nwr < g->H ? g->nwr : g->H;
    g->cap = g->C * (1 + rows * g->W);
    g->cap += g->cap & 1;  // even: every stream starts 16-byte aligned
}

// Choose the stage-2 kernel (SC_FORCE_VARIANT env: -1 auto, 0 generic, id; SC_NO_JIT
// env: never generate at run time) and fix what it implies: packed-weight k-block
// width and the stream row tiles.  No generated variant matches -> a run-time
// generated one (variant -1, parameters in *jp) if allow_jit and the shape is in range.
// Returns why an SC_JIT_FORCE parameter set cannot run this shape (nullptr: chosen fine).
const char* choose_kernel(Geometry* g, int* variant, const char** name, bool allow_jit, sc::jit::Params* jp) {
    int force = -1;
    if (const char* f = getenv("SC_FORCE_VARIANT")) force = atoi(f);
    int kl = 1, ty = (int)g->Ho;
    *variant = sc::gather_fast_select(*g, force, name, &kl, &ty);
    if (*variant == 0) *name = "generic";
    // tuning knob: SC_JIT_FORCE="TY,KL,NW,MINB,CH,STAGES,SLOTS,PIECE" generates that variant for any shape
    if (const char* jf = getenv("SC_JIT_FORCE")) {
        if (allow_jit && sc::jit::available()) {
            sc::jit::Params q;
            if (sscanf(jf, "%d,%d,%d,%d,%d,%d,%d,%d", &q.TY, &q.KL, &q.NW, &q.MINB, &q.CH, &q.STAGES, &q.SLOTS,
                       &q.PIECE) == 8) {
                q.R = (int)g->R; q.S = (int)g->S; q.P = (int)g->P; q.T = (int)g->T; q.W = (int)g->W;
                if (const char* why = sc::jit::invalid(*g, q)) return why;
                *jp = q;
                *variant = -1;
                *name = "jit";
                kl = q.KL;
                ty = q.TY;
                allow_jit = false;
            }
        }
    }
    if (*variant == 0 && allow_jit && force != 0 && !getenv("SC_NO_JIT") && sc::jit::available() &&
        sc::jit::choose(*g, jp)) {
        *variant = -1;
        *name = "jit";
        kl = jp->KL;
        ty = jp->TY;
    }
    g->kbw = 32 * kl;
    g->Kg_pad = (g->Kg + g->kbw - 1) / g->kbw * g->kbw;
    g->kblocks = g->Kg_pad / g->kbw;
    stream_format(g, ty);
    return nullptr;
}

sc_status make_geometry(const sc_conv_params* p, Geometry* g, DenseGeom* dg, int* variant, const char** name,
                        bool allow_jit = false, sc::jit::Params* jp = nullptr) {
    g->N = p->n; g->C = p->c; g->H = p->h; g->W = p->w; g->K = p->k; g->R = p->r; g->S = p->s;
    g->T = p->stride; g->P = p->pad; g->G = p->groups;
    g->Ho = (p->h + 2 * p->pad - p->r) / p->stride + 1;
    g->Wo = (p->w + 2 * p->pad - p->s) / p->stride + 1;
    g->Cg = p->c / p->groups;
    g->Kg = p->k / p->groups;
    g->relu = (p->flags & SC_FLAG_FUSE_RELU) != 0;
    sc::jit::Params unused;
    if (const char* why = choose_kernel(g, variant, name, allow_jit && jp, jp ? jp : &unused))
        return fail(SC_ERR_UNSUPPORTED, "SC_JIT_FORCE=%s: %s", getenv("SC_JIT_FORCE"), why);
    sc::dense_geometry(*g, dg);
    const int64_t in_e = g->N * g->C * g->H * g->W, out_e = g->N * g->K * g->Ho * g->Wo;
    const int64_t w_e = g->G * g->Cg * g->R * g->S * g->Kg_pad;
    const int64_t s_e = g->N * g->tiles * g->cap;  // 8-byte entries; indices are u32 inside a stream
    const int64_t d_e = (int64_t)sc::dense_workspace_floats(*g, *dg);
    const int64_t h_e = g->N * g->H * g->W * dg->cp;
    if (in_e > kMaxElems || out_e > kMaxElems || w_e > kMaxElems || s_e > kMaxElems || d_e > kMaxElems ||
        h_e > kMaxElems)
        return fail(SC_ERR_UNSUPPORTED, "a tensor has >= 2^31 elements");
    return SC_OK;
}

sc_status check_dev_ptr(const sc_plan_s* plan, const void* ptr, const char* name) {
    if (!ptr) return fail(SC_ERR_INVALID_ARGUMENT, "%s is NULL", name);
    if (reinterpret_cast<uintptr_t>(ptr) % 16)
        return fail(SC_ERR_INVALID_ARGUMENT, "%s is not 16-byte aligned", name);
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(SC_ERR_INVALID_ARGUMENT, "%s: not a CUDA pointer (%s)", name, cudaGetErrorString(e));
    }
    if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged)
        return fail(SC_ERR_INVALID_ARGUMENT, "%s is not device memory", name);
    if (attr.device != plan->device)
        return fail(SC_ERR_INVALID_ARGUMENT, "%s is on device %d, plan is on device %d", name, attr.device,
                    plan->device);
    return SC_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

void free_plan(sc_plan_s* p) {
    cudaFree(p->wpack);
    cudaFree(p->wdense);
    cudaFree(p->nhwc);
    cudaFree(p->bias);
    cudaFree(p->entries);
    cudaFree(p->offs);
    cudaFree(p->cnt);
    cudaFree(p->plist);
    cudaFree(p->prow);
    cudaFree(p->stage_in);
    cudaFree(p->stage_out);
    cudaFree(p->stage_in2);
    cudaFree(p->stage_out2);
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < sc_plan_s::kHostChunks; ++i)
            for (cudaEvent_t ev : {p->hb_in[k][i], p->hb_comp[k][i], p->hb_out[k][i]})
                if (ev) cudaEventDestroy(ev);
    cudaFree(p->sel);
    for (auto& h : p->hs)
        if (h) cudaStreamDestroy(h);
    for (int i = 0; i < sc_plan_s::kHostChunks; ++i) {
        if (p->ev_in[i]) cudaEventDestroy(p->ev_in[i]);
        if (p->ev_comp[i]) cudaEventDestroy(p->ev_comp[i]);
    }
    if (p->ev_start) cudaEventDestroy(p->ev_start);
    if (p->ev_done) cudaEventDestroy(p->ev_done);
    cudaFree(p->bws);
    cudaFree(p->bdt);
    cudaFree(p->entries2);
    cudaFree(p->offs2);
    cudaFree(p->cnt2);
    cudaFree(p->plist2);
    cudaFree(p->prow2);
    for (auto& h : p->bs)
        if (h) cudaStreamDestroy(h);
    for (cudaEvent_t ev : {p->bev_fork, p->bev_s1, p->bev_g[0], p->bev_g[1], p->bwd_fork, p->bwd_join})
        if (ev) cudaEventDestroy(ev);
    if (p->bwd_s2) cudaStreamDestroy(p->bwd_s2);
    delete p;
}

// Stage 2 with the plan's kernel (generated, run-time generated or generic).
cudaError_t launch_stage2(sc_plan_s* p, int64_t n, const uint2* entries, const uint32_t* offs, float* out,
                          uint2* rowlist, uint32_t* rowcnt, cudaStream_t s, sc::Gate gate = {}) {
    if (p->variant > 0)
        return sc::launch_gather_fast(p->variant, p->g, n, entries, offs, p->wpack, p->bias, out, rowlist, rowcnt, s,
                                      gate);
    if (rowlist) return cudaErrorNotSupported;
    if (p->variant < 0)
        return sc::jit::launch(gate.flag ? p->jit_fn_gated : p->jit_fn, p->jit_smem, p->jp, p->g, n, entries, offs,
                               p->wpack, p->bias, out, s, gate);
    return sc::launch_gather_generic(p->g, n, entries, offs, p->wpack, p->bias, out, s, gate);
}

// stage 1 + stage 2 of the sparse path (gated: f3)
// img0: the images' slice of the plan workspace (every stage-1/stage-2 buffer is image-major), so
// launches for disjoint image ranges may run concurrently (sparse_conv_forward_host)
cudaError_t enqueue_sparse(sc_plan_s* p, int64_t n, const float* d_in, float* d_out, cudaStream_t s,
                           sc::Gate gate = {}, int64_t img0 = 0) {
    const Geometry& g = p->g;
    uint32_t* cnt = p->cnt ? p->cnt + img0 * g.tiles * g.C : nullptr;
    uint2* plist = p->plist ? p->plist + img0 * g.C * g.H * g.W : nullptr;
    uint32_t* prow = p->prow ? p->prow + img0 * g.C * (g.H + 1) : nullptr;
    uint2* entries = p->entries + img0 * g.tiles * g.cap;
    uint32_t* offs = p->offs + img0 * g.tiles * (g.C + 1);
    cudaError_t e = sc::launch_compact(g, n, d_in, cnt, plist, prow, entries, offs, s, gate);
    if (e != cudaSuccess) return e;
    p->lists_layout = (gate.flag == nullptr && sc::compact_uses_counts(g) && cnt && plist && prow) ? 1 : 0;
    return launch_stage2(p, n, entries, offs, d_out, nullptr, nullptr, s, gate);
}

cudaError_t enqueue_dense(sc_plan_s* p, int64_t n, const float* d_in, float* d_out, cudaStream_t s,
                          sc::Gate gate = {}) {
    return sc::launch_dense_tc(p->g, p->dg, n, d_in, p->nhwc, p->bmap, p->wdense, p->bias, d_out, s, gate);
}

cudaError_t ensure_staging(sc_plan_s* p) {
    const Geometry& g = p->g;
    cudaError_t e;
    if (!p->stage_in && (e = cudaMalloc(&p->stage_in, sizeof(float) * g.N * g.C * g.H * g.W)) != cudaSuccess) return e;
    if (!p->stage_out && (e = cudaMalloc(&p->stage_out, sizeof(float) * g.N * g.K * g.Ho * g.Wo)) != cudaSuccess)
        return e;
    return cudaSuccess;
}

cudaError_t ensure_host_pipeline(sc_plan_s* p) {
    cudaError_t e = cudaSuccess;
    for (auto& h : p->hs)
        if (!h && (e = cudaStreamCreateWithFlags(&h, cudaStreamNonBlocking)) != cudaSuccess) return e;
    auto mk = [](cudaEvent_t* ev) {
        return *ev ? cudaSuccess : cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    };
    for (int i = 0; i < sc_plan_s::kHostChunks; ++i)
        if ((e = mk(&p->ev_in[i])) != cudaSuccess || (e = mk(&p->ev_comp[i])) != cudaSuccess) return e;
    if ((e = mk(&p->ev_start)) != cudaSuccess) return e;
    return mk(&p->ev_done);
}

bool batches_ready(const sc_plan_s* p) {
    return p->bs[0] && p->bs[1] && p->bs[2] && p->bev_fork && p->bev_s1 && p->bev_g[0] && p->bev_g[1] &&
           p->entries2 && p->offs2 && (!sc::compact_uses_counts(p->g) || (p->cnt2 && p->plist2 && p->prow2));
}

cudaError_t ensure_batches(sc_plan_s* p) {
    const Geometry& g = p->g;
    cudaError_t e = cudaSuccess;
    const size_t ebytes = sizeof(uint2) * (g.N * g.tiles * g.cap + 2);
    if (!p->entries2) {
        if ((e = cudaMalloc(&p->entries2, ebytes)) != cudaSuccess) return e;
        // as for the plan's own streams: slack is never interpreted, but keep it initialised
        if ((e = cudaMemset(p->entries2, 0, ebytes)) != cudaSuccess) return e;
    }
    if (!p->offs2 && (e = cudaMalloc(&p->offs2, sizeof(uint32_t) * g.N * g.tiles * (g.C + 1))) != cudaSuccess)
        return e;
    if (sc::compact_uses_counts(g)) {
        if (!p->cnt2 && (e = cudaMalloc(&p->cnt2, sizeof(uint32_t) * g.N * g.tiles * g.C)) != cudaSuccess) return e;
        if (!p->plist2 && (e = cudaMalloc(&p->plist2, sizeof(uint2) * g.N * g.C * g.H * g.W)) != cudaSuccess) return e;
        if (!p->prow2 && (e = cudaMalloc(&p->prow2, sizeof(uint32_t) * g.N * g.C * (g.H + 1))) != cudaSuccess)
            return e;
    }
    int least = 0, greatest = 0;
    if ((e = cudaDeviceGetStreamPriorityRange(&least, &greatest)) != cudaSuccess) return e;
    for (int i = 0; i < 3; ++i)
        if (!p->bs[i] &&
            (e = cudaStreamCreateWithPriority(&p->bs[i], cudaStreamNonBlocking, i == 0 ? least : greatest)) != cudaSuccess)
            return e;
    for (cudaEvent_t* ev : {&p->bev_fork, &p->bev_s1, &p->bev_g[0], &p->bev_g[1]})
        if (!*ev && (e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return e;
    return cudaDeviceSynchronize();  // the workspace memset
}

// sparse_conv_forward_host(_batches): compute streams (SC_HOST_STREAMS, 1..kHostComp, default 2)
int host_comp_streams() {
    static const int ncomp = [] {
        const char* v = getenv("SC_HOST_STREAMS");  // measurement knob
        const int c = v ? atoi(v) : 2;
        return c < 1 ? 1 : (c > sc_plan_s::kHostComp ? sc_plan_s::kHostComp : c);
    }();
    return ncomp;
}

// Chunks of whole images for the host paths, boundaries at multiples of 4 images (16-byte
// aligned device pointers for any shape): a small first chunk starts the copy-out early (the
// copy-out of the dense fp32 output is the longest leg), the rest split evenly.  Returns the
// chunk count; bounds[0..chunks].  SC_HOST_CHUNKS / SC_HOST_FIRST: measurement knobs.
int host_chunk_bounds(int64_t n, int64_t* bounds) {
    static const int max_chunks = [] {
        const char* v = getenv("SC_HOST_CHUNKS");
        const int c = v ? atoi(v) : 8;
        return c < 1 ? 1 : (c > sc_plan_s::kHostChunks ? sc_plan_s::kHostChunks : c);
    }();
    static const int64_t first_env = [] {
        const char* v = getenv("SC_HOST_FIRST");  // images in the first chunk (0: even split)
        return (int64_t)(v ? atoi(v) : -1);
    }();
    int chunks = (int)(n / 4 < max_chunks ? n / 4 : max_chunks);
    if (chunks < 1) chunks = 1;
    bounds[0] = 0;
    int64_t first = first_env >= 0 ? first_env : n / 8;
    first = (first + 3) & ~(int64_t)3;
    if (chunks == 1 || first <= 0 || first >= n) {
        for (int i = 1; i <= chunks; ++i) bounds[i] = i == chunks ? n : ((n * i / chunks) & ~(int64_t)3);
    } else {
        bounds[1] = first;
        for (int i = 2; i <= chunks; ++i)
            bounds[i] = i == chunks ? n : ((first + (n - first) * (i - 1) / (chunks - 1)) & ~(int64_t)3);
    }
    return chunks;
}

// Best-of-3 device time (us) of one path on the staged input (one untimed run first).
cudaError_t time_path(sc_plan_s* p, int64_t n, bool dense, cudaStream_t s, double* us) {
    cudaEvent_t a, b;
    cudaError_t e = cudaEventCreate(&a);
    if (e != cudaSuccess) return e;
    if ((e = cudaEventCreate(&b)) != cudaSuccess) {
        cudaEventDestroy(a);
        return e;
    }
    double best = 1e30;
    for (int it = 0; it < 4 && e == cudaSuccess; ++it) {
        if ((e = cudaEventRecord(a, s)) != cudaSuccess) break;
        e = dense ? enqueue_dense(p, n, p->stage_in, p->stage_out, s) : enqueue_sparse(p, n, p->stage_in, p->stage_out, s);
        if (e != cudaSuccess) break;
        if ((e = cudaEventRecord(b, s)) != cudaSuccess || (e = cudaEventSynchronize(b)) != cudaSuccess) break;
        float ms = 0;
        if ((e = cudaEventElapsedTime(&ms, a, b)) != cudaSuccess) break;
        if (it > 0 && ms * 1e3 < best) best = ms * 1e3;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *us = best;
    return e;
}

// Sparse-path time minus dense-path time at input density rho (f3 calibration).
cudaError_t sparse_minus_dense(sc_plan_s* p, int64_t n, double rho, double dense_us, cudaStream_t s, double* f) {
    const int64_t elems = n * p->g.C * p->g.H * p->g.W;
    cudaError_t e = sc::launch_synth_relu(p->stage_in, elems, rho, 0x5eed1234u, s);
    if (e != cudaSuccess) return e;
    double us = 0;
    if ((e = time_path(p, n, false, s, &us)) != cudaSuccess) return e;
    *f = us - dense_us;
    return cudaSuccess;
}

// Largest nonzero count the sparse path is taken for: s >= s* <=> nnz <= (1 - s*) * elems.
unsigned long long auto_threshold(const sc_plan_s* p, int64_t elems) {
    if (!p->dg.supported) return ~0ull;
    const double lim = (1.0 - p->s_star) * (double)elems;
    return lim <= 0 ? 0ull : (unsigned long long)lim;
}

sc_status check_forward(sc_plan plan, int64_t n) {
    if (!plan) return fail(SC_ERR_INVALID_ARGUMENT, "plan is NULL");
    if (n < 1 || n > plan->params.n)
        return fail(SC_ERR_INVALID_ARGUMENT, "n=%lld outside [1, %lld]", (long long)n, (long long)plan->params.n);
    return SC_OK;
}

// Layers of a chain for images [img0, img0 + n) on stream s: each plan's workspace slice of
// those images (image-major), layer l+1's lists emitted by layer l's gather when it can.
sc_status enqueue_chain(const sc_plan* plans, int32_t nplans, int64_t n, int64_t img0, const float* d_in,
                        float* const* d_outs, cudaStream_t s) {
    bool lists_ready = false;  // plans[l]'s row lists were written by layer l-1's gather
    for (int l = 0; l < nplans; ++l) {
        sc_plan_s* p = plans[l];
        const Geometry& g = p->g;
        cudaError_t e;
        uint32_t* cnt = p->cnt ? p->cnt + img0 * g.tiles * g.C : nullptr;
        uint2* entries = p->entries + img0 * g.tiles * g.cap;
        uint32_t* offs = p->offs + img0 * g.tiles * (g.C + 1);
        uint2* plist = p->plist ? p->plist + img0 * g.C * g.H * g.W : nullptr;
        const float* in_prev = l > 0 && d_outs[l - 1] ? d_outs[l - 1] + img0 * g.C * g.H * g.W : nullptr;
        if (l == 0) {
            uint32_t* prow = p->prow ? p->prow + img0 * g.C * (g.H + 1) : nullptr;
            e = sc::launch_compact(g, n, d_in + img0 * g.C * g.H * g.W, cnt, plist, prow, entries, offs, s);
        } else if (lists_ready) {
            // the producer's per-(plane, row) slots and row counts (rcnt: C*H per image)
            uint32_t* rcnt = p->prow + img0 * g.C * g.H;
            e = sc::launch_compact_from_rows(g, n, cnt, plist, rcnt, entries, offs, s);
        } else {
            if (!in_prev)
                return fail(SC_ERR_UNSUPPORTED, "layer %d cannot emit chained lists: d_outs[%d] is required", l - 1,
                            l - 1);
            uint32_t* prow = p->prow ? p->prow + img0 * g.C * (g.H + 1) : nullptr;
            e = sc::launch_compact(g, n, in_prev, cnt, plist, prow, entries, offs, s);
        }
        if (e != cudaSuccess) return cuda_fail(e, "chain stage 1");
        if (!lists_ready) p->lists_layout = (sc::compact_uses_counts(g) && p->plist && p->prow) ? 1 : 0;
        sc_plan_s* next = l + 1 < nplans ? plans[l + 1] : nullptr;
        const bool emit = next && p->variant > 0 && sc::gather_fast_can_emit(p->variant) &&
                          sc::compact_uses_counts(next->g) && next->plist && next->prow;
        float* out = d_outs[l] ? d_outs[l] + img0 * g.K * g.Ho * g.Wo : nullptr;
        if (!emit && !out) return fail(SC_ERR_UNSUPPORTED, "layer %d needs an output buffer (no list emission)", l);
        uint2* rows_next = emit ? next->plist + img0 * next->g.C * next->g.H * next->g.W : nullptr;
        uint32_t* rcnt_next = emit ? next->prow + img0 * next->g.C * next->g.H : nullptr;
        e = launch_stage2(p, n, entries, offs, out, rows_next, rcnt_next, s);
        if (e != cudaSuccess) return cuda_fail(e, "chain gather");
        if (emit) next->lists_layout = 2;
        lists_ready = emit;
    }
    return SC_OK;
}

}  // namespace

extern "C" {

const char* sc_status_string(sc_status s) {
    switch (s) {
        case SC_OK: return "ok";
        case SC_ERR_INVALID_ARGUMENT: return "invalid argument";
        case SC_ERR_SHAPE: return "invalid shape";
        case SC_ERR_UNSUPPORTED: return "unsupported";
        case SC_ERR_CUDA: return "CUDA error";
        case SC_ERR_OUT_OF_MEMORY: return "out of memory";
    }
    return "unknown status";
}

const char* sc_last_error(void) { return g_last_error.c_str(); }

sc_status sparse_conv_output_shape(const sc_conv_params* params, int64_t out_nchw[4]) {
    sc_status st = validate_params(params);
    if (st != SC_OK) return st;
    if (!out_nchw) return fail(SC_ERR_INVALID_ARGUMENT, "out_nchw is NULL");
    out_nchw[0] = params->n;
    out_nchw[1] = params->k;
    out_nchw[2] = (params->h + 2 * params->pad - params->r) / params->stride + 1;
    out_nchw[3] = (params->w + 2 * params->pad - params->s) / params->stride + 1;
    return SC_OK;
}

sc_status sparse_conv_create(const sc_conv_params* params, const float* d_weight, const float* d_bias, int device,
                             sc_plan* out_plan) {
    if (!out_plan) return fail(SC_ERR_INVALID_ARGUMENT, "out_plan is NULL");
    *out_plan = nullptr;
    sc_status st = validate_params(params);
    if (st != SC_OK) return st;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return fail(SC_ERR_INVALID_ARGUMENT, "device %d not available (%d devices)", device, ndev);
    }
    sc_plan_s* plan = new (std::nothrow) sc_plan_s();
    if (!plan) return fail(SC_ERR_OUT_OF_MEMORY, "host allocation failed");
    plan->params = *params;
    plan->device = device;
    DeviceGuard guard(device);
    if ((st = make_geometry(params, &plan->g, &plan->dg, &plan->variant, &plan->variant_name, true, &plan->jp)) !=
        SC_OK) {
        delete plan;
        return st;
    }
    if (plan->variant < 0) {  // compile the run-time variant now; on failure keep the generic kernel
        if (sc::jit::compile(plan->jp, device, &plan->jit_fn, &plan->jit_fn_gated, &plan->jit_smem) == cudaSuccess) {
            const sc::jit::Params& q = plan->jp;
            snprintf(plan->jit_name, sizeof(plan->jit_name), "jit_r%ds%dp%dt%d_w%d_ty%d_kl%d_nw%d_ch%d", q.R, q.S,
                     q.P, q.T, q.W, q.TY, q.KL, q.NW, q.CH);
            plan->variant_name = plan->jit_name;
        } else if ((st = make_geometry(params, &plan->g, &plan->dg, &plan->variant, &plan->variant_name)) != SC_OK) {
            delete plan;
            return st;
        }
    }
    if ((st = check_dev_ptr(plan, d_weight, "d_weight")) != SC_OK ||
        (d_bias && (st = check_dev_ptr(plan, d_bias, "d_bias")) != SC_OK)) {
        delete plan;
        return st;
    }
    const Geometry& g = plan->g;
    const DenseGeom& dg = plan->dg;
    sc::backward_geometry(g, &plan->bg);
    cudaError_t e;
    const size_t wbytes = sizeof(float) * g.G * g.Cg * g.R * g.S * g.Kg_pad;
    const size_t dbytes = sizeof(float) * sc::dense_workspace_floats(g, dg);
    const size_t hbytes = sizeof(float) * g.N * g.H * g.W * dg.cp;
    if ((e = cudaMalloc(&plan->wpack, wbytes)) != cudaSuccess ||
        (e = cudaMalloc(&plan->wdense, dbytes)) != cudaSuccess ||
        (dg.supported && (e = cudaMalloc(&plan->nhwc, hbytes)) != cudaSuccess) ||
        (e = cudaMalloc(&plan->bias, sizeof(float) * g.K)) != cudaSuccess ||
        (e = cudaMalloc(&plan->entries, sizeof(uint2) * (g.N * g.tiles * g.cap + 2))) != cudaSuccess ||
        (e = cudaMalloc(&plan->offs, sizeof(uint32_t) * g.N * g.tiles * (g.C + 1))) != cudaSuccess ||
        (e = cudaMalloc(&plan->sel, 4 * sizeof(unsigned long long))) != cudaSuccess ||
        (plan->bg.supported &&
         ((e = cudaMalloc(&plan->bws, sizeof(float) * plan->bg.splits_w * g.K * g.Cg * g.R * g.S)) != cudaSuccess ||
          (e = cudaMalloc(&plan->bdt, sizeof(float) * plan->bg.doutT_floats)) != cudaSuccess)) ||
        (sc::compact_uses_counts(g) &&
         ((e = cudaMalloc(&plan->cnt, sizeof(uint32_t) * g.N * g.tiles * g.C)) != cudaSuccess ||
          (e = cudaMalloc(&plan->plist, sizeof(uint2) * g.N * g.C * g.H * g.W)) != cudaSuccess ||
          (e = cudaMalloc(&plan->prow, sizeof(uint32_t) * g.N * g.C * (g.H + 1))) != cudaSuccess))) {
        free_plan(plan);
        return cuda_fail(e, "sparse_conv_create: cudaMalloc");
    }
    cudaStream_t st0 = 0;
    if (d_bias)
        e = cudaMemcpyAsync(plan->bias, d_bias, sizeof(float) * g.K, cudaMemcpyDeviceToDevice, st0);
    else
        e = cudaMemsetAsync(plan->bias, 0, sizeof(float) * g.K, st0);
    // stream slack is never interpreted, but the stage-2 bulk copies round
    // piece boundaries to 16 bytes: keep the workspace initialised
    if (e == cudaSuccess) e = cudaMemsetAsync(plan->entries, 0, sizeof(uint2) * (g.N * g.tiles * g.cap + 2), st0);
    if (e == cudaSuccess) e = cudaMemsetAsync(plan->sel, 0, 4 * sizeof(unsigned long long), st0);
    if (e == cudaSuccess) e = sc::launch_pack_weights(g, d_weight, plan->wpack, st0);
    if (e == cudaSuccess) e = sc::launch_pack_dense(g, dg, d_weight, plan->wdense, st0);
    if (e == cudaSuccess && dg.supported) e = sc::encode_dense_input_map(g, dg, plan->nhwc, plan->bmap);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st0);
    if (e != cudaSuccess) {
        free_plan(plan);
        return cuda_fail(e, "sparse_conv_create: pack");
    }
    *out_plan = plan;
    return SC_OK;
}

sc_status sparse_conv_destroy(sc_plan plan) {
    if (!plan) return SC_OK;
    DeviceGuard guard(plan->device);
    free_plan(plan);
    return SC_OK;
}

sc_status sparse_conv_compact(sc_plan plan, int64_t n, const float* d_in, sc_stream_t stream) {
    sc_status st = check_forward(plan, n);
    if (st != SC_OK) return st;
    if ((st = check_dev_ptr(plan, d_in, "d_in")) != SC_OK) return st;
    DeviceGuard guard(plan->device);
    cudaError_t e = sc::launch_compact(plan->g, n, d_in, plan->cnt, plan->plist, plan->prow, plan->entries,
                                       plan->offs, (cudaStream_t)stream);
    plan->lists_layout = (e == cudaSuccess && sc::compact_uses_counts(plan->g) && plan->plist && plan->prow) ? 1 : 0;
    return e == cudaSuccess ? SC_OK : cuda_fail(e, "compact launch");
}

sc_status sparse_conv_gather(sc_plan plan, int64_t n, float* d_out, sc_stream_t stream) {
    sc_status st = check_forward(plan, n);
    if (st != SC_OK) return st;
    if ((st = check_dev_ptr(plan, d_out, "d_out")) != SC_OK) return st;
    DeviceGuard guard(plan->device);
    cudaError_t e;
    e = launch_stage2(plan, n, plan->entries, plan->offs, d_out, nullptr, nullptr, (cudaStream_t)stream);
    return e == cudaSuccess ? SC_OK : cuda_fail(e, "gather launch");
}

sc_status sparse_conv_forward(sc_plan plan, int64_t n, const float* d_in, float* d_out, sc_stream_t stream) {
    sc_status st = sparse_conv_compact(plan, n, d_in, stream);
    if (st != SC_OK) return st;
    return sparse_conv_gather(plan, n, d_out, stream);
}

sc_status sparse_conv_reserve_batches(sc_plan plan) {
    if (!plan) return fail(SC_ERR_INVALID_ARGUMENT, "plan is NULL");
    DeviceGuard guard(plan->device);
    const cudaError_t e = ensure_batches(plan);
    return e == cudaSuccess ? SC_OK : cuda_fail(e, "sparse_conv_reserve_batches");
}

sc_status sparse_conv_forward_batches(sc_plan plan, int32_t nbatch, int64_t n, const float* const* d_in,
                                      float* const* d_out, sc_stream_t stream) {
    sc_status st = check_forward(plan, n);
    if (st != SC_OK) return st;
    if (nbatch < 1 || !d_in || !d_out)
        return fail(SC_ERR_INVALID_ARGUMENT, "nbatch=%d: need nbatch >= 1 and the d_in / d_out arrays", (int)nbatch);
    for (int32_t b = 0; b < nbatch; ++b)
        if ((st = check_dev_ptr(plan, d_in[b], "d_in[b]")) != SC_OK || (st = check_dev_ptr(plan, d_out[b], "d_out[b]")) != SC_OK)
            return st;
    if (nbatch == 1) return sparse_conv_forward(plan, n, d_in[0], d_out[0], stream);
    DeviceGuard guard(plan->device);
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    if (!batches_ready(plan)) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if ((e = cudaStreamIsCapturing(s, &cs)) != cudaSuccess) return cuda_fail(e, "cudaStreamIsCapturing");
        if (cs != cudaStreamCaptureStatusNone)
            return fail(SC_ERR_INVALID_ARGUMENT,
                        "first sparse_conv_forward_batches under stream capture: call sparse_conv_reserve_batches first");
        if ((e = ensure_batches(plan)) != cudaSuccess) return cuda_fail(e, "sparse_conv_forward_batches setup");
    }
    const Geometry& g = plan->g;
    // fork: every plan stream starts after the work already queued on `stream`
    if ((e = cudaEventRecord(plan->bev_fork, s)) != cudaSuccess) return cuda_fail(e, "event record");
    for (cudaStream_t b : plan->bs)
        if ((e = cudaStreamWaitEvent(b, plan->bev_fork, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
    cudaStream_t s1 = plan->bs[0];
    for (int32_t b = 0; b < nbatch; ++b) {
        const int slot = b & 1;
        uint2* entries = slot ? plan->entries2 : plan->entries;
        uint32_t* offs = slot ? plan->offs2 : plan->offs;
        uint32_t* cnt = slot ? plan->cnt2 : plan->cnt;
        uint2* plist = slot ? plan->plist2 : plan->plist;
        uint32_t* prow = slot ? plan->prow2 : plan->prow;
        cudaStream_t s2 = plan->bs[1 + slot];
        // stage 1 of batch b overwrites the workspace batch b-2's stage 2 read
        if (b >= 2 && (e = cudaStreamWaitEvent(s1, plan->bev_g[slot], 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
        if ((e = sc::launch_compact(g, n, d_in[b], cnt, plist, prow, entries, offs, s1)) != cudaSuccess)
            return cuda_fail(e, "compact launch");
        if ((e = cudaEventRecord(plan->bev_s1, s1)) != cudaSuccess || (e = cudaStreamWaitEvent(s2, plan->bev_s1, 0)) != cudaSuccess)
            return cuda_fail(e, "stage-1 event");
        if ((e = launch_stage2(plan, n, entries, offs, d_out[b], nullptr, nullptr, s2)) != cudaSuccess)
            return cuda_fail(e, "gather launch");
        if ((e = cudaEventRecord(plan->bev_g[slot], s2)) != cudaSuccess) return cuda_fail(e, "event record");
    }
    // join: the last stage 2 of each stream (every stage 1 precedes a stage 2 of its batch)
    for (int slot = 0; slot < 2; ++slot)
        if ((e = cudaStreamWaitEvent(s, plan->bev_g[slot], 0)) != cudaSuccess) return cuda_fail(e, "stream join");
    plan->lists_layout = 0;  // the list views describe sparse_conv_forward / sparse_conv_compact only
    return SC_OK;
}

sc_status dense_conv_forward(sc_plan plan, int64_t n, const float* d_in, float* d_out, sc_stream_t stream) {
    sc_status st = check_forward(plan, n);
    if (st != SC_OK) return st;
    if ((st = check_dev_ptr(plan, d_in, "d_in")) != SC_OK) return st;
    if ((st = check_dev_ptr(plan, d_out, "d_out")) != SC_OK) return st;
    DeviceGuard guard(plan->device);
    cudaError_t e = enqueue_dense(plan, n, d_in, d_out, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) return fail(SC_ERR_UNSUPPORTED, "dense path: shape not supported");
    return e == cudaSuccess ? SC_OK : cuda_fail(e, "dense launch");
}

sc_status sparse_conv_forward_host(sc_plan plan, int64_t n, const float* h_in, float* h_out, sc_stream_t stream) {
    sc_status st = check_forward(plan, n);
    if (st != SC_OK) return st;
    if (!h_in || !h_out) return fail(SC_ERR_INVALID_ARGUMENT, "host buffer is NULL");
    DeviceGuard guard(plan->device);
    const Geometry& g = plan->g;
    cudaError_t e;
    if ((e = ensure_staging(plan)) != cudaSuccess || (e = ensure_host_pipeline(plan)) != cudaSuccess)
        return cuda_fail(e, "host pipeline setup");
    cudaStream_t s = (cudaStream_t)stream;
    cudaStream_t h2d = plan->hs[0], d2h = plan->hs[1];
    const int ncomp = host_comp_streams();
    const int64_t in_img = g.C * g.H * g.W, out_img = g.K * g.Ho * g.Wo;
    int64_t bounds[sc_plan_s::kHostChunks + 1];
    const int chunks = host_chunk_bounds(n, bounds);
    if ((e = cudaEventRecord(plan->ev_start, s)) != cudaSuccess) return cuda_fail(e, "event record");
    for (int k = 0; k < 2 + ncomp; ++k)
        if ((e = cudaStreamWaitEvent(plan->hs[k], plan->ev_start, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
    for (int i = 0; i < chunks; ++i) {
        const int64_t c0 = bounds[i], c1 = bounds[i + 1];
        if (c1 <= c0) continue;
        const size_t bi = sizeof(float) * (c1 - c0) * in_img, bo = sizeof(float) * (c1 - c0) * out_img;
        float* din = plan->stage_in + c0 * in_img;
        float* dout = plan->stage_out + c0 * out_img;
        // chunk i computes on stream 2 + i % ncomp in its own workspace slice, so the kernels of
        // consecutive chunks overlap (a small chunk fills only part of the GPU)
        cudaStream_t comp = plan->hs[2 + i % ncomp];
        if ((e = cudaMemcpyAsync(din, h_in + c0 * in_img, bi, cudaMemcpyHostToDevice, h2d)) != cudaSuccess ||
            (e = cudaEventRecord(plan->ev_in[i], h2d)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(comp, plan->ev_in[i], 0)) != cudaSuccess)
            return cuda_fail(e, "H2D copy");
        if ((e = enqueue_sparse(plan, c1 - c0, din, dout, comp, {}, c0)) != cudaSuccess) return cuda_fail(e, "forward");
        if ((e = cudaEventRecord(plan->ev_comp[i], comp)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(d2h, plan->ev_comp[i], 0)) != cudaSuccess ||
            (e = cudaMemcpyAsync(h_out + c0 * out_img, dout, bo, cudaMemcpyDeviceToHost, d2h)) != cudaSuccess)
            return cuda_fail(e, "D2H copy");
    }
    // the caller's stream resumes after everything (kernels and copies) of this call
    // (every chunk's kernels precede its copy-out, so the copy-out stream joins them all)
    if ((e = cudaEventRecord(plan->ev_done, d2h)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(s, plan->ev_done, 0)) != cudaSuccess)
        return cuda_fail(e, "stream join");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "stream sync");
    return SC_OK;
}

sc_status sparse_conv_forward_host_batches(sc_plan plan, int32_t nbatch, int64_t n, const float* const* h_in,
                                           float* const* h_out, sc_stream_t stream) {
    sc_status st = check_forward(plan, n);
    if (st != SC_OK) return st;
    if (nbatch < 1 || !h_in || !h_out)
        return fail(SC_ERR_INVALID_ARGUMENT, "nbatch=%d: need nbatch >= 1 and the h_in / h_out arrays", (int)nbatch);
    for (int32_t b = 0; b < nbatch; ++b)
        if (!h_in[b] || !h_out[b]) return fail(SC_ERR_INVALID_ARGUMENT, "host buffer of batch %d is NULL", (int)b);
    if (nbatch == 1) return sparse_conv_forward_host(plan, n, h_in[0], h_out[0], stream);
    DeviceGuard guard(plan->device);
    const Geometry& g = plan->g;
    cudaError_t e;
    if ((e = ensure_staging(plan)) != cudaSuccess || (e = ensure_host_pipeline(plan)) != cudaSuccess)
        return cuda_fail(e, "host pipeline setup");
    if ((!plan->stage_in2 && (e = cudaMalloc(&plan->stage_in2, sizeof(float) * g.N * g.C * g.H * g.W)) != cudaSuccess) ||
        (!plan->stage_out2 &&
         (e = cudaMalloc(&plan->stage_out2, sizeof(float) * g.N * g.K * g.Ho * g.Wo)) != cudaSuccess))
        return cuda_fail(e, "host staging");
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < sc_plan_s::kHostChunks; ++i)
            for (cudaEvent_t* ev : {&plan->hb_in[k][i], &plan->hb_comp[k][i], &plan->hb_out[k][i]})
                if (!*ev && (e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess)
                    return cuda_fail(e, "host events");
    cudaStream_t s = (cudaStream_t)stream;
    cudaStream_t h2d = plan->hs[0], d2h = plan->hs[1];
    const int ncomp = host_comp_streams();
    const int64_t in_img = g.C * g.H * g.W, out_img = g.K * g.Ho * g.Wo;
    int64_t bounds[sc_plan_s::kHostChunks + 1];
    const int chunks = host_chunk_bounds(n, bounds);
    if ((e = cudaEventRecord(plan->ev_start, s)) != cudaSuccess) return cuda_fail(e, "event record");
    for (int k = 0; k < 2 + ncomp; ++k)
        if ((e = cudaStreamWaitEvent(plan->hs[k], plan->ev_start, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
    for (int32_t b = 0; b < nbatch; ++b) {
        // batch b uses staging set b & 1; chunk i of every batch uses workspace slice i on compute
        // stream 2 + i % ncomp (so batch b's chunk i follows batch b-1's in stream order)
        const int set = b & 1;
        float* sin = set ? plan->stage_in2 : plan->stage_in;
        float* sout = set ? plan->stage_out2 : plan->stage_out;
        for (int i = 0; i < chunks; ++i) {
            const int64_t c0 = bounds[i], c1 = bounds[i + 1];
            if (c1 <= c0) continue;
            const size_t bi = sizeof(float) * (c1 - c0) * in_img, bo = sizeof(float) * (c1 - c0) * out_img;
            float* din = sin + c0 * in_img;
            float* dout = sout + c0 * out_img;
            cudaStream_t comp = plan->hs[2 + i % ncomp];
            // the copy-in overwrites what batch b-2's kernels read; the kernels overwrite what batch
            // b-2's copy-out read
            if (b >= 2 && (e = cudaStreamWaitEvent(h2d, plan->hb_comp[set][i], 0)) != cudaSuccess)
                return cuda_fail(e, "stream wait");
            if ((e = cudaMemcpyAsync(din, h_in[b] + c0 * in_img, bi, cudaMemcpyHostToDevice, h2d)) != cudaSuccess ||
                (e = cudaEventRecord(plan->hb_in[set][i], h2d)) != cudaSuccess ||
                (e = cudaStreamWaitEvent(comp, plan->hb_in[set][i], 0)) != cudaSuccess)
                return cuda_fail(e, "H2D copy");
            if (b >= 2 && (e = cudaStreamWaitEvent(comp, plan->hb_out[set][i], 0)) != cudaSuccess)
                return cuda_fail(e, "stream wait");
            if ((e = enqueue_sparse(plan, c1 - c0, din, dout, comp, {}, c0)) != cudaSuccess)
                return cuda_fail(e, "forward");
            if ((e = cudaEventRecord(plan->hb_comp[set][i], comp)) != cudaSuccess ||
                (e = cudaStreamWaitEvent(d2h, plan->hb_comp[set][i], 0)) != cudaSuccess ||
                (e = cudaMemcpyAsync(h_out[b] + c0 * out_img, dout, bo, cudaMemcpyDeviceToHost, d2h)) != cudaSuccess ||
                (e = cudaEventRecord(plan->hb_out[set][i], d2h)) != cudaSuccess)
                return cuda_fail(e, "D2H copy");
        }
    }
    if ((e = cudaEventRecord(plan->ev_done, d2h)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(s, plan->ev_done, 0)) != cudaSuccess)
        return cuda_fail(e, "stream join");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "stream sync");
    return SC_OK;
}

sc_status sparse_conv_forward_chain(const sc_plan* plans, int32_t nplans, int64_t n, const float* d_in,
                                   float* const* d_outs, sc_stream_t stream) {
    if (!plans || nplans < 1 || !d_outs) return fail(SC_ERR_INVALID_ARGUMENT, "bad chain arguments");
    for (int l = 0; l < nplans; ++l) {
        sc_status st = check_forward(plans[l], n);
        if (st != SC_OK) return st;
        if (l > 0 && plans[l]->device != plans[0]->device)
            return fail(SC_ERR_INVALID_ARGUMENT, "chain plans live on different devices");
        if (l + 1 < nplans) {
            const Geometry &a = plans[l]->g, &b = plans[l + 1]->g;
            if (a.K != b.C || a.Ho != b.H || a.Wo != b.W)
                return fail(SC_ERR_SHAPE, "layer %d output %lldx%lldx%lld does not match layer %d input", l,
                            (long long)a.K, (long long)a.Ho, (long long)a.Wo, l + 1);
        }
    }
    sc_status st = check_dev_ptr(plans[0], d_in, "d_in");
    if (st != SC_OK) return st;
    if ((st = check_dev_ptr(plans[0], d_outs[nplans - 1], "d_outs[last]")) != SC_OK) return st;
    for (int l = 0; l + 1 < nplans; ++l)
        if (d_outs[l] && (st = check_dev_ptr(plans[0], d_outs[l], "d_outs[l]")) != SC_OK) return st;
    DeviceGuard guard(plans[0]->device);
    cudaStream_t s = (cudaStream_t)stream;
    // Large batches run as chunks of whole images on two plan-owned streams (every workspace is
    // image-major): one chunk's layer tails (the last, partly filled wave of each gather) overlap
    // another chunk's layers.  SC_CHAIN_CHUNKS (measurement knob): chunks, 1 = none.
    static const int max_chunks = [] {
        const char* v = getenv("SC_CHAIN_CHUNKS");
        const int c = v ? atoi(v) : 2;  // C5 (N=1024): 1 / 2 / 4 / 8 chunks 4.03 / 3.96 / 3.99 / 4.31 ms
        return c < 1 ? 1 : (c > sc_plan_s::kHostChunks ? sc_plan_s::kHostChunks : c);
    }();
    int chunks = (int)(n / 128 < max_chunks ? n / 128 : max_chunks);  // chunks of >= 128 images
    if (chunks < 2) return enqueue_chain(plans, nplans, n, 0, d_in, d_outs, s);
    sc_plan_s* p0 = plans[0];
    cudaError_t e;
    if (!p0->hs[2] || !p0->hs[3] || !p0->ev_start || !p0->ev_comp[chunks - 1]) {
        // the streams are created outside stream capture only; a first call under capture runs the
        // chain unchunked on `stream` (same results)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if ((e = cudaStreamIsCapturing(s, &cs)) != cudaSuccess) return cuda_fail(e, "cudaStreamIsCapturing");
        if (cs != cudaStreamCaptureStatusNone) return enqueue_chain(plans, nplans, n, 0, d_in, d_outs, s);
        if ((e = ensure_host_pipeline(p0)) != cudaSuccess) return cuda_fail(e, "chain streams");
    }
    if ((e = cudaEventRecord(p0->ev_start, s)) != cudaSuccess) return cuda_fail(e, "event record");
    for (int k = 2; k < 4; ++k)
        if ((e = cudaStreamWaitEvent(p0->hs[k], p0->ev_start, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
    for (int c = 0; c < chunks; ++c) {
        const int64_t c0 = (n * c / chunks) & ~(int64_t)3, c1 = c + 1 == chunks ? n : ((n * (c + 1) / chunks) & ~(int64_t)3);
        cudaStream_t cs = p0->hs[2 + (c & 1)];
        sc_status st2 = enqueue_chain(plans, nplans, c1 - c0, c0, d_in, d_outs, cs);
        if (st2 != SC_OK) return st2;
        if ((e = cudaEventRecord(p0->ev_comp[c], cs)) != cudaSuccess) return cuda_fail(e, "event record");
    }
    // join: the last chunk of each stream (stream order covers the earlier ones)
    for (int c = chunks - 2; c < chunks; ++c)
        if ((e = cudaStreamWaitEvent(s, p0->ev_comp[c], 0)) != cudaSuccess) return cuda_fail(e, "stream join");
    return SC_OK;
}

sc_status sparse_conv_calibrate_crossover(sc_plan plan, int64_t n, sc_stream_t stream, double* s_star) {
    sc_status st = check_forward(plan, n);
    if (st != SC_OK) return st;
    DeviceGuard guard(plan->device);
    cudaStream_t s = (cudaStream_t)stream;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(s, &cap);
    if (e != cudaSuccess) return cuda_fail(e, "calibrate: capture query");
    if (cap != cudaStreamCaptureStatusNone)
        return fail(SC_ERR_INVALID_ARGUMENT, "calibrate: stream is capturing (calibrate before capture)");
    if (!plan->dg.supported) {
        plan->s_star = 0.0;  // no dense path: always sparse
            if (s_star) *s_star = plan->s_star;
        return SC_OK;
    }
    if ((e = ensure_staging(plan)) != cudaSuccess) return cuda_fail(e, "staging alloc");
    const int64_t elems = n * plan->g.C * plan->g.H * plan->g.W;
    double dense_us = 0;
    if ((e = sc::launch_synth_relu(plan->stage_in, elems, 0.5, 1u, s)) != cudaSuccess ||
        (e = time_path(plan, n, true, s, &dense_us)) != cudaSuccess)
        return cuda_fail(e, "calibrate: dense timing");
    // f(rho) = t_sparse(rho) - t_dense, increasing in the density rho = 1 - s
    double lo = 0.0, flo = 0, hi = 0.1, fhi = 0;
    if ((e = sparse_minus_dense(plan, n, lo, dense_us, s, &flo)) != cudaSuccess) return cuda_fail(e, "calibrate");
    double rho_star;
    if (flo >= 0) {
        rho_star = 0.0;  // sparse loses even on an all-zero input: always dense
    } else {
        if ((e = sparse_minus_dense(plan, n, hi, dense_us, s, &fhi)) != cudaSuccess) return cuda_fail(e, "calibrate");
        while (fhi < 0 && hi < 1.0) {
            lo = hi;
            flo = fhi;
            hi = hi * 2 < 1.0 ? hi * 2 : 1.0;
            if ((e = sparse_minus_dense(plan, n, hi, dense_us, s, &fhi)) != cudaSuccess) return cuda_fail(e, "calibrate");
        }
        if (fhi < 0) {
            rho_star = 1.0;  // sparse wins even on a dense input: always sparse
        } else {
            // regula falsi (Illinois) on the bracket [lo, hi]
            int side = 0;
            for (int it = 0; it < 5; ++it) {
                const double m = lo + (hi - lo) * (-flo) / (fhi - flo);
                double fm = 0;
                if ((e = sparse_minus_dense(plan, n, m, dense_us, s, &fm)) != cudaSuccess)
                    return cuda_fail(e, "calibrate");
                if (fm < 0) {
                    lo = m;
                    flo = fm;
                    if (side == -1) fhi *= 0.5;
                    side = -1;
                } else {
                    hi = m;
                    fhi = fm;
                    if (side == 1) flo *= 0.5;
                    side = 1;
                }
                if (hi - lo < 1e-3) break;
            }
            rho_star = lo + (hi - lo) * (-flo) / (fhi - flo);
        }
    }
    plan->s_star = 1.0 - rho_star;
    if (s_star) *s_star = plan->s_star;
    return SC_OK;
}

sc_status sparse_conv_set_crossover(sc_plan plan, double s_star) {
    if (!plan) return fail(SC_ERR_INVALID_ARGUMENT, "plan is NULL");
    if (!(s_star >= 0.0 && s_star <= 1.0)) return fail(SC_ERR_INVALID_ARGUMENT, "s_star outside [0, 1]");
    plan->s_star = s_star;
    return SC_OK;
}

sc_status sparse_conv_get_crossover(sc_plan plan, double* s_star) {
    if (!plan || !s_star) return fail(SC_ERR_INVALID_ARGUMENT, "NULL argument");
    *s_star = plan->s_star;
    return SC_OK;
}

sc_status sparse_conv_forward_auto(sc_plan plan, int64_t n, const float* d_in, float* d_out, sc_stream_t stream) {
    sc_status st = check_forward(plan, n);
    if (st != SC_OK) return st;
    if ((st = check_dev_ptr(plan, d_in, "d_in")) != SC_OK) return st;
    if ((st = check_dev_ptr(plan, d_out, "d_out")) != SC_OK) return st;
    if (plan->s_star < 0 && (st = sparse_conv_calibrate_crossover(plan, n, stream, nullptr)) != SC_OK) return st;
    DeviceGuard guard(plan->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t elems = n * plan->g.C * plan->g.H * plan->g.W;
    const int* flag = reinterpret_cast<const int*>(plan->sel + 2);
    cudaError_t e = sc::launch_select_path(d_in, elems, auto_threshold(plan, elems), plan->sel, s);
    if (e == cudaSuccess) e = enqueue_sparse(plan, n, d_in, d_out, s, sc::Gate{flag, sc::kPathSparse});
    if (e == cudaSuccess && plan->dg.supported)
        e = enqueue_dense(plan, n, d_in, d_out, s, sc::Gate{flag, sc::kPathDense});
    return e == cudaSuccess ? SC_OK : cuda_fail(e, "auto forward launch");
}

sc_status sparse_conv_last_path(sc_plan plan, int32_t* path, int64_t* nnz) {
    if (!plan) return fail(SC_ERR_INVALID_ARGUMENT, "plan is NULL");
    DeviceGuard guard(plan->device);
    unsigned long long h[4];
    cudaError_t e = cudaMemcpy(h, plan->sel, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "last_path copy");
    if (path) *path = (int32_t)(h[2] & 0xffffffffu);
    if (nnz) *nnz = (int64_t)h[3];
    return SC_OK;
}

sc_status sparse_conv_backward(sc_plan plan, int64_t n, const float* d_in, const float* d_dout, float* d_dw,
                               float* d_dbias, float* d_dz, sc_stream_t stream) {
    sc_status st = check_forward(plan, n);
    if (st != SC_OK) return st;
    if (!plan->bg.supported)
        return fail(SC_ERR_UNSUPPORTED, "backward: needs a plane-major plan (H*W <= 1024, H <= 31, tiles <= 32) "
                                        "and a 1x1, 3x3 or 5x5 kernel");
    if ((st = check_dev_ptr(plan, d_in, "d_in")) != SC_OK || (st = check_dev_ptr(plan, d_dout, "d_dout")) != SC_OK)
        return st;
    if ((d_dw && (st = check_dev_ptr(plan, d_dw, "d_dw")) != SC_OK) ||
        (d_dbias && (st = check_dev_ptr(plan, d_dbias, "d_dbias")) != SC_OK) ||
        (d_dz && (st = check_dev_ptr(plan, d_dz, "d_dz")) != SC_OK))
        return st;
    DeviceGuard guard(plan->device);
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (d_dw || d_dz) {
        e = sc::launch_plane_lists(plan->g, n, d_in, plan->cnt, plan->plist, plan->prow, s);
        plan->lists_layout = e == cudaSuccess ? 1 : 0;
    }
    if (e == cudaSuccess && !plan->bwd_s2) {
        // the second stream and its events are created outside stream capture (under capture the
        // kernels run on `stream` alone: same results, no overlap)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if ((e = cudaStreamIsCapturing(s, &cs)) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
            if ((e = cudaStreamCreateWithFlags(&plan->bwd_s2, cudaStreamNonBlocking)) == cudaSuccess &&
                (e = cudaEventCreateWithFlags(&plan->bwd_fork, cudaEventDisableTiming)) == cudaSuccess)
                e = cudaEventCreateWithFlags(&plan->bwd_join, cudaEventDisableTiming);
            if (e != cudaSuccess) return cuda_fail(e, "backward stream setup");
        }
    }
    if (e == cudaSuccess)
        e = sc::launch_backward(plan->g, plan->bg, n, plan->plist, plan->prow, d_dout, plan->wpack, plan->bws,
                                plan->bdt, d_dw, d_dbias, d_dz, s, plan->bwd_join ? plan->bwd_s2 : nullptr,
                                plan->bwd_fork, plan->bwd_join);
    return e == cudaSuccess ? SC_OK : cuda_fail(e, "backward launch");
}

sc_status sparse_conv_lists(sc_plan plan, sc_lists_view* out) {
    if (!plan || !out) return fail(SC_ERR_INVALID_ARGUMENT, "NULL argument");
    out->entries = reinterpret_cast<const uint32_t*>(plan->entries);
    out->offsets = plan->offs;
    out->tiles_per_image = plan->g.tiles;
    out->stream_capacity = plan->g.cap;
    out->channels = plan->g.C;
    out->tile_rows = (int32_t)plan->g.ty;
    out->window_rows = (int32_t)plan->g.nwr;
    out->window_width = (int32_t)plan->g.W;
    out->marker_code = (int32_t)plan->g.nwin;
    return SC_OK;
}

sc_status sparse_conv_plane_lists(sc_plan plan, sc_plane_lists_view* out) {
    if (!plan || !out) return fail(SC_ERR_INVALID_ARGUMENT, "NULL argument");
    if (plan->lists_layout == 0 || !plan->plist || !plan->prow)
        return fail(SC_ERR_UNSUPPORTED, "no plane lists: the plan's last stage 1 kept none (streamwise path, "
                                        "device-side path selection, or no compaction yet)");
    out->entries = reinterpret_cast<const uint32_t*>(plan->plist);
    out->row_counts = plan->prow;
    out->planes = plan->g.N * plan->g.C;
    out->height = (int32_t)plan->g.H;
    out->width = (int32_t)plan->g.W;
    out->layout = plan->lists_layout;
    return SC_OK;
}

sc_status sparse_conv_kernel_variant(sc_plan plan, int32_t* variant, const char** name) {
    if (!plan || !variant) return fail(SC_ERR_INVALID_ARGUMENT, "NULL argument");
    *variant = plan->variant;
    if (name) *name = plan->variant_name;
    return SC_OK;
}

sc_status sparse_conv_launch_count(sc_plan plan, int32_t* sparse_launches, int32_t* dense_launches) {
    if (!plan) return fail(SC_ERR_INVALID_ARGUMENT, "plan is NULL");
    if (sparse_launches) *sparse_launches = sc::compact_uses_counts(plan->g) ? 3 : 2;
    if (dense_launches) *dense_launches = 2;
    return SC_OK;
}

size_t sc_jit_variant_source(const int32_t params[14], char* buf, size_t cap) {
    if (!params) return 0;
    sc::jit::Params q;
    q.R = params[0]; q.S = params[1]; q.P = params[2]; q.T = params[3]; q.W = params[4]; q.TY = params[5];
    q.KL = params[6]; q.NW = params[7]; q.MINB = params[8]; q.CH = params[9]; q.STAGES = params[10];
    q.SLOTS = params[11]; q.PIECE = params[12]; q.id = params[13];
    return sc::jit::variant_source(q, buf, cap);
}

int32_t sc_jit_available(void) { return sc::jit::available() ? 1 : 0; }

sc_status sc_probe_fma(int32_t kind, double* fma_per_clk_per_sm) {
    if (!fma_per_clk_per_sm || kind < 0 || kind > 2) return fail(SC_ERR_INVALID_ARGUMENT, "bad probe arguments");
    cudaError_t e = sc::probe_fma(kind, fma_per_clk_per_sm);
    return e == cudaSuccess ? SC_OK : cuda_fail(e, "fma probe");
}

sc_status sc_flush_l2(void* d_scratch, size_t bytes, sc_stream_t stream) {
    if (!d_scratch || bytes < 16) return fail(SC_ERR_INVALID_ARGUMENT, "bad scratch");
    cudaError_t e = sc::launch_flush(d_scratch, bytes, (cudaStream_t)stream);
    return e == cudaSuccess ? SC_OK : cuda_fail(e, "flush");
}

}  // extern "C"
