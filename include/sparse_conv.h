/*
 * sparse_conv.h -- C ABI of libsparseconv.so, a B200 (sm_100a) implementation
 * of the ReLU-sparse forward convolution of Shi & Chu, arXiv 1704.07724
 * ("Speeding up Convolutional Neural Networks By Exploiting the Sparsity of
 * Rectifier Units", /root/reference/PAPER.md, cited as P:<line>).
 *
 * What is computed (Sec. 3 Eq. 1, with Table 1's padding P and
 * stride T, and the batch/bias/groups readings R2-R4 of DESIGN.md):
 *
 *   out[n,k,y,x] = bias[k] + sum_{c in group(k)} sum_{r<R} sum_{t<S}
 *                  in[n, c, y*T + r - P, x*T + t - P] * W[k, c - g*C/G, r, t]
 *
 * with out-of-range input reads equal to zero (virtual padding) and
 * H_out = floor((H + 2P - R)/T) + 1 (reading R1; P:37 is garbled).
 *
 * sparse_conv_forward skips every multiply-add whose input is zero (the
 * "inverse sparse convolution" of P:119-123) in two stages: (1) a compaction
 * kernel emits per-(image, channel, row-tile) nonzero lists (ISC step 1,
 * P:123); (2) an output-stationary gather kernel accumulates
 * sum_{nonzeros} v * W (ISC steps 2-3).  dense_conv_forward is the
 * GEMM-mapped dense convolution of P:109-117 (Fig. 2) on tcgen05 tensor cores
 * (TF32 inputs, fp32 accumulation) -- the in-library comparison.
 *
 * Conventions (all functions):
 *  - Tensors are fp32, contiguous NCHW (input/output) and [K][C/G][R][S]
 *    (weights).  Device pointers must be 16-byte aligned and belong to the
 *    plan's device; otherwise SC_ERR_INVALID_ARGUMENT.
 *  - Errors never abort; sc_last_error() returns a thread-local detail string.
 *  - Every element count must be < 2^31, else SC_ERR_UNSUPPORTED.
 *  - Inputs are expected to be finite (ReLU outputs).  Non-finite inputs are
 *    outside the sparse path's contract (reading R7).
 */
#ifndef SPARSE_CONV_H_
#define SPARSE_CONV_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t without including cuda_runtime.h */
typedef struct CUstream_st *sc_stream_t;

typedef enum {
    SC_OK = 0,
    SC_ERR_INVALID_ARGUMENT = 1, /* null/misaligned/wrong-device pointer, bad n */
    SC_ERR_SHAPE = 2,            /* parameters violate the shape rules below    */
    SC_ERR_UNSUPPORTED = 3,      /* valid but not implemented (e.g. >= 2^31)    */
    SC_ERR_CUDA = 4,             /* a CUDA call failed; see sc_last_error()     */
    SC_ERR_OUT_OF_MEMORY = 5
} sc_status;

/* Paper Table 1 plus batch and groups.
 * Shape rules (SC_ERR_SHAPE otherwise): n,c,h,w,k,r,s,stride,groups >= 1;
 * pad >= 0; r <= h + 2*pad; s <= w + 2*pad; groups divides c and k. */
typedef struct {
    int64_t n, c, h, w;   /* input NCHW; n = the largest batch this plan serves */
    int64_t k, r, s;      /* K filters of R x S; weight [K][C/groups][R][S]     */
    int64_t stride;       /* T, same in both dimensions                  */
    int64_t pad;          /* P, symmetric zero padding                   */
    int64_t groups;       /* grouped convolution (reading R4)                   */
    uint32_t flags;       /* 0 or SC_FLAG_FUSE_RELU                             */
} sc_conv_params;

/* Apply Z = max(0, O) (Eq. 2) in the epilogue of both forward paths. */
#define SC_FLAG_FUSE_RELU 1u

typedef struct sc_plan_s *sc_plan;

/* Read-only view of the stage-1 workspace (device pointers owned by the plan).
 * Tile-stream format (reading R9): output rows are cut into tiles
 * of TY = tile_rows rows; tile t of image n has the input window of
 * NWR = window_rows rows starting at input row t*TY*stride - pad, all W =
 * window_width columns, NWIN = marker_code = NWR*W positions.  Its stream
 * (stream id s = n*tiles_per_image + t) is entries[s*stream_capacity*2 ...],
 * a sequence of u32 pairs (a, b):
 *   for every input channel c ascending with at least one nonzero in the
 *   window: the marker (a = c, b = NWIN + mask), then every input
 *   x = in[n,c,i,j] != 0.0f inside the window (ascending
 *   i, j) as (a = bit copy of x, b = (i - (t*TY*stride - pad))*W + j).
 *   Bit r of mask is set iff one of the channel's entries sits at a window
 *   row wi with wi - r = ty*stride for a tile row 0 <= ty < TY (the filter
 *   rows the channel reaches).  Channels without a nonzero in the window have
 *   no marker and offsets[s*(C+1) + c] == offsets[s*(C+1) + c + 1].
 * offsets[s*(C+1) + c] = index of channel c's marker, offsets[s*(C+1) + C] =
 * stream length.  Entries beyond the length are undefined. */
typedef struct {
    const uint32_t *entries;   /* [N][tiles][stream_capacity][2] */
    const uint32_t *offsets;   /* [N][tiles][channels + 1]       */
    int64_t tiles_per_image;
    int64_t stream_capacity;
    int64_t channels;
    int32_t tile_rows;
    int32_t window_rows;
    int32_t window_width;
    int32_t marker_code;       /* NWIN: markers carry NWIN + mask */
} sc_lists_view;

/* Output shape (N = params.n): out_nchw = {n, k, H_out, W_out}.  Pure host
 * function; SC_ERR_SHAPE on invalid params. */
sc_status sparse_conv_output_shape(const sc_conv_params *params, int64_t out_nchw[4]);

/* Create a plan on `device`: validates params, allocates plan-owned device
 * memory (packed weights in the K-contiguous layout of ISC step 2; the
 * dense path's TF32 operand; bias; the stage-1 list workspace for params.n
 * images), packs the weights and synchronizes.  d_weight [K][C/G][R][S] and
 * d_bias [K] (NULL = zero bias) are device pointers that the caller may free
 * when this returns.  *out_plan is NULL on failure. */
sc_status sparse_conv_create(const sc_conv_params *params, const float *d_weight,
                             const float *d_bias, int device, sc_plan *out_plan);

/* The hot path: out = conv(in) skipping zero inputs (stages 1 and 2) for the
 * first n (1 <= n <= params.n) images.  d_in [n][C][H][W], d_out
 * [n][K][H_out][W_out] are caller-owned device buffers; d_out is fully
 * overwritten.  Stream-ordered and asynchronous: no allocation and no host
 * synchronization, so it can be captured in a CUDA graph.  A plan must not run
 * two forwards concurrently (the list workspace is shared).  Device faults
 * surface at the caller's next synchronization. */
sc_status sparse_conv_forward(sc_plan plan, int64_t n, const float *d_in, float *d_out,
                              sc_stream_t stream);

/* A sequence of nbatch independent batches of n images each: d_in[b] / d_out[b]
 * (host arrays of nbatch device pointers, each buffer as in sparse_conv_forward)
 * hold batch b.  Each batch's outputs are bit-identical to sparse_conv_forward on
 * that batch, since the same kernels run.  The calls are pipelined across batches:
 * - Batch b+1's stage 1 runs on a low-priority plan-owned stream while batch b's
 *   stage 2 is still running, so it fills the SMs that stage 2's last wave leaves idle.
 * - The plan keeps two stage-1 workspaces and alternates between them.
 * - Stage-2 launches alternate between two high-priority plan-owned streams, so
 *   batch b+1's stage 2 can start in batch b's last wave.
 * The work starts after everything already queued on `stream`, and `stream`
 * resumes after the last batch.  No host synchronization, so it can be captured in
 * a CUDA graph.  The first call creates the second workspace and the streams, so it
 * must not be made while `stream` is capturing (SC_ERR_INVALID_ARGUMENT);
 * sparse_conv_reserve_batches does that ahead of time.  nbatch == 1 is exactly
 * sparse_conv_forward.  The same plan must not run another forward concurrently.
 * Afterwards the list views (sparse_conv_lists / sparse_conv_plane_lists) describe no
 * batch; they describe the last sparse_conv_forward / sparse_conv_compact only.
 * Why: a stage-2 CTA holds a whole SM
 * (registers and shared memory), and C2 needs 1.66 waves of them. */
sc_status sparse_conv_forward_batches(sc_plan plan, int32_t nbatch, int64_t n, const float *const *d_in,
                                      float *const *d_out, sc_stream_t stream);

/* Allocate what sparse_conv_forward_batches needs (second stage-1 workspace,
 * streams, events); idempotent. */
sc_status sparse_conv_reserve_batches(sc_plan plan);

/* Dense comparison path: implicit GEMM on tcgen05 tensor cores,
 * operands rounded to TF32 (cvt.rna), fp32 accumulation.  Two launches: the
 * input is transposed to a plan-owned channels-last TF32 copy, then every
 * (tap, 32-channel block) of a tile of whole output rows is one 4-D TMA box
 * (zero-filled padding).  Same buffer and stream contract as
 * sparse_conv_forward.  SC_ERR_UNSUPPORTED when a tile of one output row does
 * not fit a UMMA N <= 256 (W_out > 256) or a TMA box. */
sc_status dense_conv_forward(sc_plan plan, int64_t n, const float *d_in, float *d_out,
                             sc_stream_t stream);

/* End-to-end variant of sparse_conv_forward with HOST buffers: copies h_in
 * (n images) to plan-owned device staging, runs the sparse forward, copies the
 * result back into h_out, then synchronizes `stream`.  The batch is pipelined
 * in up to 8 chunks of whole images on plan-owned streams: copy-ins, kernels
 * and copy-outs of different chunks overlap, and the kernels of consecutive
 * chunks run concurrently on two streams, each chunk in its own image slice of
 * the plan workspace; the work starts after everything already queued on
 * `stream`.  For full copy bandwidth
 * (and overlap) h_in/h_out should be pinned (cudaHostAlloc/register). */
sc_status sparse_conv_forward_host(sc_plan plan, int64_t n, const float *h_in, float *h_out,
                                   sc_stream_t stream);

/* End to end for a sequence of nbatch independent batches of n images: h_in[b] / h_out[b]
 * (host arrays of nbatch host pointers, each buffer as in sparse_conv_forward_host) hold batch
 * b.  Same chunked pipeline as sparse_conv_forward_host, continued across batches: batch b+1's
 * copy-in and kernels run while batch b's copy-out is still in flight.  The two copy directions
 * use separate copy engines, so the sequence runs at the PCIe rate rather than the sum of the
 * legs.  The plan keeps two device staging sets and alternates between them.  Every batch's
 * output is identical to sparse_conv_forward_host on that batch.  Starts after the work
 * queued on `stream`, synchronizes `stream` before returning; nbatch == 1 is exactly
 * sparse_conv_forward_host.  h_in / h_out should be pinned. */
sc_status sparse_conv_forward_host_batches(sc_plan plan, int32_t nbatch, int64_t n, const float *const *h_in,
                                           float *const *h_out, sc_stream_t stream);

/* A chain of layers (e.g. C5: conv3 -> ReLU -> conv4 -> ReLU -> conv5, the
 * ReLUs fused via SC_FLAG_FUSE_RELU) on the first n images: plans[l+1]'s input
 * is plans[l]'s output (K, H_out, W_out must match C, H, W).  d_in is layer
 * 0's NCHW input; d_outs[l] is layer l's NCHW output buffer (caller-owned).
 * d_outs[nplans-1] is required; an intermediate d_outs[l] may be NULL, in
 * which case layer l writes no dense output and instead emits layer l+1's
 * stage-1 input directly from its epilogue (ISC step 1 fused into the
 * producer: "eliminates the unused zero operands on-the-fly", P:29, P:33;
 * SURVEY 8f row f1): per-(plane, row) nonzero lists that layer l+1's stage 1
 * turns into the same R9 streams without re-reading a dense tensor.  Returns
 * SC_ERR_UNSUPPORTED if such an intermediate layer cannot emit lists (its
 * stage-2 kernel is the generic one or a KL=1 variant) and d_outs[l] is NULL.
 * Stream-ordered, asynchronous, graph-capturable like sparse_conv_forward.
 * For n >= 256 the chain runs as 2 chunks of whole images (multiples of 4),
 * each through all layers in its own image slice of every plan's workspace. The
 * chunks use two streams owned by plans[0], so one chunk's last, partly filled
 * stage-2 wave of a layer overlaps the other chunk's work. The
 * SC_CHAIN_CHUNKS env var (measurement knob, 1-8) changes the count. The first
 * chunked call made outside stream capture creates those streams; until then the
 * chain runs unchunked on `stream`, with the same results. */
sc_status sparse_conv_forward_chain(const sc_plan *plans, int32_t nplans, int64_t n, const float *d_in,
                                    float *const *d_outs, sc_stream_t stream);

/* ---- automatic sparse <-> dense crossover --------------
 * The paper claims its speedup "when the sparsity is not less than 0.9"
 * (P:23): the sparse method pays off only above a crossover sparsity
 * s*, which on B200 depends on the shape and the batch (the dense path runs on
 * tensor cores).  sparse_conv_forward_auto decides per call ON THE DEVICE:
 * one kernel counts the batch's nonzero inputs (sparsity s = 1 - nnz/(n*C*H*W))
 * and writes a path flag; the sparse path (s >= s*) and the dense path
 * (s < s*) are both enqueued and the kernels of the path not chosen return at
 * once.  No host synchronization: capturable like sparse_conv_forward (after
 * calibration).  Plans whose dense path is unsupported always run sparse. */
#define SC_PATH_SPARSE 0
#define SC_PATH_DENSE 1

/* Same buffer and stream contract as sparse_conv_forward.  If the plan has no
 * crossover yet (neither set nor calibrated), calibrates it first with
 * sparse_conv_calibrate_crossover(plan, n, stream) (synchronizes; returns
 * SC_ERR_INVALID_ARGUMENT if `stream` is capturing). */
sc_status sparse_conv_forward_auto(sc_plan plan, int64_t n, const float *d_in, float *d_out,
                                   sc_stream_t stream);

/* Measure s* for batches of n images on this device: times the dense path
 * and the sparse path on plan-owned synthetic inputs (i.i.d. nonzeros,
 * counter-based hash) at several sparsities, locates the sparsity where the
 * two times are equal (bracketing secant on the measured sparse time), stores
 * it in the plan and returns it in *s_star (may be NULL).  s* = 1 means "always
 * dense", 0 "always sparse".  Allocates the plan's staging buffers (as
 * sparse_conv_forward_host) on first use; synchronizes `stream`. */
sc_status sparse_conv_calibrate_crossover(sc_plan plan, int64_t n, sc_stream_t stream, double *s_star);

/* Set s* in [0, 1] explicitly (no calibration), or query it (*s_star < 0: not
 * set yet). */
sc_status sparse_conv_set_crossover(sc_plan plan, double s_star);
sc_status sparse_conv_get_crossover(sc_plan plan, double *s_star);

/* Which path the last sparse_conv_forward_auto on this plan took
 * (SC_PATH_SPARSE / SC_PATH_DENSE) and the nonzero count it measured.
 * Synchronizes the device. */
sc_status sparse_conv_last_path(sc_plan plan, int32_t *path, int64_t *nnz);

/* ---- backward with sparse activations ------------------
 * The paper measures the ReLU sparsity during training but gives
 * no backward algorithm; this is the chain rule of Eq. 1 (R19-R20)
 * for the first n images, skipping zero inputs:
 *   d_dw    [K][C/G][R][S]  dW[k,c,r,t] = sum_{n,y,x} in[n,c,yT+r-P,xT+t-P] * dout[n,k,y,x]
 *   d_dbias [K]             sum_{n,y,x} dout[n,k,y,x]
 *   d_dz    [n][C][H][W]    dz[n,c,i,j] = [in[n,c,i,j] != 0] *
 *                               sum_{k,r,t} W[k,c,r,t] * dout[n,k,(i+P-r)/T,(j+P-t)/T]
 *                           (terms with a non-integral or out-of-range output index dropped):
 *                           the gradient through the ReLU that produced `in` (Eq. 2), zero
 *                           wherever in == 0.
 * d_in is the forward input [n][C][H][W], d_dout the gradient of this layer's
 * convolution output [n][K][H_out][W_out] (if the plan fuses a ReLU on its
 * output, pass the gradient w.r.t. the pre-ReLU output).  d_dw, d_dbias, d_dz
 * are caller-owned outputs, each nullable (not computed), fully overwritten.
 * fp32 accumulation in a fixed order (deterministic).  Stream-ordered, no
 * allocation, graph-capturable; shares the plan's list workspace with the
 * forward (do not overlap the two).  dz and dbias run on a second plan-owned
 * stream beside dW, forked from and joined into `stream`.  That stream is
 * created by the first call made outside stream capture; until then the
 * kernels run on `stream` alone, with the same results.  SC_ERR_UNSUPPORTED unless the plan uses
 * the plane-major stage 1 (H*W <= 1024, H <= 31, <= 32 row tiles) and R x S is
 * 1x1, 3x3 or 5x5. */
sc_status sparse_conv_backward(sc_plan plan, int64_t n, const float *d_in, const float *d_dout, float *d_dw,
                               float *d_dbias, float *d_dz, sc_stream_t stream);

/* Free everything the plan owns.  NULL is a no-op. */
sc_status sparse_conv_destroy(sc_plan plan);

/* Static description of a status code; never NULL. */
const char *sc_status_string(sc_status status);
/* Detail of the last error raised on this thread ("" if none). */
const char *sc_last_error(void);

/* ---- test and bench hooks ------------------------------------------------ */

/* Stage 1 only (ISC step 1): fill the plan's list workspace from d_in. */
sc_status sparse_conv_compact(sc_plan plan, int64_t n, const float *d_in, sc_stream_t stream);

/* Stage 2 only: the gather convolution from the lists already in the plan's
 * workspace (produced by sparse_conv_compact for the same n). */
sc_status sparse_conv_gather(sc_plan plan, int64_t n, float *d_out, sc_stream_t stream);

/* Describe the plan's list workspace (device pointers, layout). */
sc_status sparse_conv_lists(sc_plan plan, sc_lists_view *out);

/* The paper-level stage-1 lists (ISC step 1, Sec. 4: "store the
 * non-zero values in a vector with their column and row information") as the
 * plan's plane-major compaction builds them, before it regroups them into the
 * stage-2 streams above.  Plane p = n*C + c; entries are u32 pairs
 * (bit copy of x, flat position i*W + j) of every x = in[n,c,i,j] != 0.0f
 * (R7), in row-major order.
 *   layout 1 (stage 1 read an input tensor): entries[p*H*W + k] for
 *     k < row_counts[p*(H+1) + H]; row_counts[p*(H+1) + i] = nonzeros of the
 *     plane before row i (exclusive row prefix), so row i's entries are
 *     k in [row_counts[p*(H+1)+i], row_counts[p*(H+1)+i+1]).
 *   layout 2 (chained layer, sparse_conv_forward_chain: written by the
 *     producing layer's epilogue): one slot per row,
 *     entries[(p*H + i)*W + k] for k < row_counts[p*H + i].
 * Device pointers owned by the plan, valid until its next call; read them after
 * synchronizing the stream of the call that produced them.  SC_ERR_UNSUPPORTED
 * when the last stage 1 of the plan kept no plane lists (planes of more than
 * 1024 elements or 31 rows use the streamwise compaction; sparse_conv_forward_auto
 * may skip stage 1; no compaction has run yet). */
typedef struct {
    const uint32_t *entries;
    const uint32_t *row_counts;
    int64_t planes;            /* N*C of the plan (params.n images) */
    int32_t height, width;     /* H, W of the input planes */
    int32_t layout;            /* 1 or 2, see above */
} sc_plane_lists_view;
sc_status sparse_conv_plane_lists(sc_plan plan, sc_plane_lists_view *out);

/* Which stage-2 kernel this plan launches: 0 = generic gather kernel (any
 * stride/shape), >0 = a shape-specialised register-tile kernel variant id. */
sc_status sparse_conv_kernel_variant(sc_plan plan, int32_t *variant, const char **name);

/* Number of kernels one sparse_conv_forward / dense_conv_forward launches
 * (sparse_conv_forward_auto launches 1 + both when the dense path is
 * supported, else 1 + sparse). */
sc_status sparse_conv_launch_count(sc_plan plan, int32_t *sparse_launches, int32_t *dense_launches);

/* Source of a stage-2 interpreter variant as generated at run time for shapes
 * without a shipped variant (csrc/jit.cu, compiled through NVRTC when a plan is
 * created); tests compare it with tools/gen_gather.py.  params = {R, S, P, T, W,
 * TY, KL, NW, MINB, CH, STAGES, SLOTS, PIECE, id}.  Writes at most cap-1 bytes
 * plus a NUL into buf (may be NULL) and returns the full length.  Host only. */
size_t sc_jit_variant_source(const int32_t params[14], char *buf, size_t cap);
/* 1 if run-time variant generation is available (NVRTC and the driver entry
 * points load), else 0; plans then use the generic stage-2 kernel instead. */
int32_t sc_jit_available(void);

/* Micro-probes for the roofline denominators (bench only).  Each runs on the
 * current device and stream 0 and synchronizes.
 *   kind 0: FFMA  (3-register form) lanes-FMA per SM-clock
 *   kind 1: FFMA2 (f32x2 with a broadcast scalar) lane-FMAs per SM-clock
 * Returns the measured rate in *fma_per_clk_per_sm (clock64 based). */
sc_status sc_probe_fma(int32_t kind, double *fma_per_clk_per_sm);

/* Overwrite `bytes` of device scratch (>= 2x L2) to evict the L2 cache. */
sc_status sc_flush_l2(void *d_scratch, size_t bytes, sc_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSE_CONV_H_ */
