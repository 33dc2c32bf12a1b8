/*
 * fsc.h — C ABI of libfsc: the expert-parallel MoE block forward of
 * FarSkip-Collective (arxiv 2511.11505) for NVIDIA B200 (sm_100a).
 *
 * Citations: PAPER.md = the paper text (/root/reference/PAPER.md, "P:<line>"),
 * readings C-amb-n = DESIGN.md "Readings of the paper".
 *
 * The operation:
 *   xn   = RMSNorm(x_in; gamma)                        ("layer-norm", C-amb-5)
 *   S,g  = top-k of softmax(xn W_R^T), renormalised    (G(A) = s(A W_R^T), C-amb-2/3)
 *   Dispatch: copies of xn rows to the ranks owning their experts
 *   y    = SwiGLU_e(row) = (row W1_e^T * SiLU(row W2_e^T)) W3_e^T  (C-amb-4)
 *   Combine: y rows back to their source rank, routed[t] = sum_j g_tj y_tj
 *   shared = SwiGLU_shared(xn) over all tokens
 *   Regular / blocking (Eq. 6):  out = (x_in + shared) + routed
 *   FarSkip:  attn-in_{k+1} = partial += shared  (compute starts at once),
 *                         mlp-in_{k+1}  = partial + routed   (far-skipped, fsc_moe_wait)
 *
 * Conventions for every entry point:
 *  - All tensor pointers are DEVICE pointers owned by the caller, 16-byte
 *    aligned, row-major, contiguous; fp32 = float, bf16 = uint16 bit patterns.
 *  - `stream` is a cudaStream_t passed as void*; all work is enqueued on it in
 *    stream order and the call returns without synchronising, except the
 *    *_host entry points, which synchronise before returning.
 *  - Return value: FSC_OK (0) or a negative fsc_status; fsc_last_error() gives
 *    the message. Validation happens before anything is enqueued. CUDA or
 *    transport failures are sticky for the context.
 *  - A context is bound to one process, one GPU and one EP rank; it is not
 *    thread-safe. The library owns only its workspace (sized once, at
 *    fsc_init, for max_cfg), its internal streams and events.
 */
#ifndef FSC_H_
#define FSC_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FSC_API __attribute__((visibility("default")))
#else
#define FSC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fsc_ctx fsc_ctx;
typedef struct fsc_handle_s* fsc_handle; /* a pending FarSkip combine (cf. P:208 handle dict) */

typedef enum {
  FSC_OK = 0,
  FSC_ERR_CONFIG = -1,    /* E % P != 0, k not in [1,E], d % 64, c % 64, T > max_tokens, ... */
  FSC_ERR_SHAPE = -2,     /* null / misaligned pointer, bad L or modes */
  FSC_ERR_CUDA = -3,      /* CUDA runtime error (sticky) */
  FSC_ERR_COMM = -4,      /* EP transport error (sticky) */
  FSC_ERR_NONFINITE = -5, /* debug finiteness check failed */
  FSC_ERR_STATE = -6      /* handle misuse: waited twice, FarSkip depth > 1, ... */
} fsc_status;

/* Per-layer residual wiring. */
enum { FSC_REGULAR = 0, FSC_HYBRID = 1 };
/* Stream schedule of the stack (P:103 vs P:198). */
enum { FSC_BLOCKING = 0, FSC_OVERLAPPED = 1 };
/* EP data movement: FSC_EP_ALLTOALL = Dispatch / Combine (training
 * path, each rank owns its T tokens); FSC_EP_ALLREDUCE = the inference variant of
 * P:215-217 (vLLM): every rank holds the SAME T tokens (replicated activations),
 * computes only its local experts' contributions and the partial outputs are
 * all-reduced (reduce-scatter + all-gather over peer memory, rank-order sums). */
enum { FSC_EP_ALLTOALL = 0, FSC_EP_ALLREDUCE = 1 };
/* Combine data path at EP > 1 (PAPER.md:100, P:198 step 7): FSC_COMBINE_STREAM (default)
 * = the down GEMM stores its rows locally and a push kernel on the communication stream
 * sends them back to their source ranks, overlapping the shared expert (step 8) and, in
 * the FarSkip stack, the next layer's attention part (a); FSC_COMBINE_FUSED = the down
 * GEMM's epilogue stores every row straight into its source rank's buffer (no local
 * round trip, but the transfer is serialised with the GEMM). Bitwise the same results. */
enum { FSC_COMBINE_STREAM = 0, FSC_COMBINE_FUSED = 1 };
/* fsc_moe_forward_blocking at EP > 1: FSC_BLOCKING_REGULAR_PLUS (default) = the
 * shared expert runs while the combine is in flight ("(c) may be partially overlapped if a
 * shared expert is present"); FSC_BLOCKING_SERIAL = the combine is waited first (the plain
 * Eq. 6 serialised run, DESIGN C-amb-16). Bitwise the same results. */
enum { FSC_BLOCKING_REGULAR_PLUS = 0, FSC_BLOCKING_SERIAL = 1 };
/* Phases of fsc_set_spin_schedule (the SPEC S:437 duration names). */
enum { FSC_SPIN_GATE = 0, FSC_SPIN_DISPATCH, FSC_SPIN_QKV, FSC_SPIN_CORE, FSC_SPIN_ROUTED, FSC_SPIN_COMBINE,
       FSC_SPIN_SHARED, FSC_SPIN_N };

/* MoE layer shape. d % 64 == 0, ffn % 64 == 0, shared_ffn % 64 == 0 (0 = no shared
 * expert; n shared experts = one SwiGLU of concatenated width, C-amb-7),
 * 1 <= top_k <= n_experts <= 128, n_experts % ep_size == 0 (C-amb-9). */
typedef struct {
  int d;
  int n_experts;
  int top_k;
  int ffn;
  int shared_ffn;
  int max_tokens; /* T per rank per call (workspace bound) */
  float rms_eps;  /* 1e-6 (C-amb-5) */
} fsc_moe_config;

/* One MoE layer's weights on this rank. Routed experts are this rank's local
 * experts [rank*E/P, (rank+1)*E/P) (contiguous placement, C-amb-9).
 *   gamma    fp32 [d]               RMSNorm weight
 *   w_router fp32 [E, d]            router W_R (replicated on every rank)
 *   w1       bf16 [E_loc, c, d]     up   (W1 of P:73-76)
 *   w2       bf16 [E_loc, c, d]     gate (W2; SiLU branch)
 *   w3       bf16 [E_loc, d, c]     down (W3)
 *   ws1/ws2  bf16 [c_s, d], ws3 bf16 [d, c_s]   shared expert, or NULL when c_s == 0 */
typedef struct {
  const float* gamma;
  const float* w_router;
  const void* w1;
  const void* w2;
  const void* w3;
  const void* ws1;
  const void* ws2;
  const void* ws3;
} fsc_moe_weights;

/* Optional outputs for tests (any may be NULL). Shapes per rank:
 *   topk_idx int32 [T,k] (ascending expert id per token), topk_w fp32 [T,k],
 *   counts int32 [E] (copies per global expert sent by this rank),
 *   pos int32 [T,k] (row of copy (t,j) in this rank's expert-sorted send buffer),
 *   logits fp32 [T,E] (fp32 router logits before near-tie refinement),
 *   shared_out fp32 [T,d], routed_out fp32 [T,d] (computed separately),
 *   n_refined int32 [1] device counter of tokens re-selected in fp64 (accumulates).
 * EP > 1 all-to-all only (the exchange of P:97-100 as this rank saw it):
 *   ep_counts int32 [P,E]: row s = copies per global expert sent by rank s (all-gathered),
 *   recv_counts int32 [E_loc]: rows received per local expert,
 *   recv_src int32 [P * max_tokens * min(k, E_loc)]: for received row r (expert-major, then
 *     source rank, then token, C-amb-11) (source rank << 24) | row in the source's
 *     expert-sorted send order; rows past sum(recv_counts) are unspecified. */
typedef struct {
  int* topk_idx;
  float* topk_w;
  int* counts;
  int* pos;
  float* logits;
  float* shared_out;
  float* routed_out;
  int* n_refined;
  int* ep_counts;
  int* recv_counts;
  int* recv_src;
} fsc_moe_debug;

/* Caller hook invoked by fsc_moe_forward_farskip while a collective is in flight:
 * phase 0 = dispatch in flight (enqueue e.g. attention part (b), P:198 step 5),
 * phase 1 = combine in flight (before the shared expert, P:198 step 8).
 * `stream` is the compute stream (cudaStream_t as void*). */
typedef void (*fsc_overlap_cb)(void* user, int phase, void* stream);

/* ---------------------------------------------------------------- lifecycle */

/* Size in bytes of the transport bootstrap blob each rank exports (0 when ep_size == 1). */
FSC_API size_t fsc_bootstrap_size(void);

/* Create a context for EP rank `rank` of `ep_size` on CUDA device `device`;
 * allocates the workspace for max_cfg (worst-case received rows
 * ep_size * max_tokens * min(top_k, E/ep_size)). For ep_size > 1 the caller then
 * exchanges blobs: fsc_bootstrap_export on every rank, an all-gather of the
 * blobs (e.g. torch.distributed), and fsc_bootstrap_import with the P blobs in
 * rank order. Errors: FSC_ERR_CONFIG for an invalid max_cfg/rank, FSC_ERR_CUDA. */
FSC_API int fsc_init(fsc_ctx** out, int rank, int ep_size, int device, const fsc_moe_config* max_cfg);
FSC_API int fsc_bootstrap_export(fsc_ctx* ctx, void* blob /* fsc_bootstrap_size() bytes */);
FSC_API int fsc_bootstrap_import(fsc_ctx* ctx, const void* blobs /* ep_size * fsc_bootstrap_size() bytes */);
FSC_API int fsc_finalize(fsc_ctx* ctx);
FSC_API const char* fsc_last_error(const fsc_ctx* ctx);
/* Persistent-grid size used by the GEMMs (<= 148); lower values leave SMs to
 * co-running comm kernels ("communication operations only utilizing a
 * fraction of the total available units"). */
FSC_API int fsc_set_gemm_ctas(fsc_ctx* ctx, int n);
/* Grouped-GEMM tile mode: 2 = CTA pairs with tcgen05 cta_group::2, 256-row
 * tiles; 1 = single-CTA 128-row tiles; 0 (default) = auto: the routed-expert
 * GEMMs use pairs when the experts receive >= 256 rows on average (prefill) and
 * single CTAs below (decode), every other GEMM uses pairs. Results are identical. */
FSC_API int fsc_set_gemm_cta_group(fsc_ctx* ctx, int cg);
/* EP = 1: on != 0 fuses the permute into GEMM1 (its TMA producer gathers the rows of
 * xn through src_row with tile::gather4) instead of the explicit permute kernel.
 * Same results bit for bit; default off (slower on the measured shapes). */
FSC_API int fsc_set_gemm_gather(fsc_ctx* ctx, int on);
/* Blocking schedule, EP = 1: on > 0 fuses the gate-weighted unpermute into the down
 * GEMM's epilogue (the k-th arriving copy of a token finishes it; k <= 8), on == 0
 * runs the separate unpermute kernel, on < 0 (default) fuses for top-1 routing only.
 * Bitwise the same result either way. */
FSC_API int fsc_set_fused_unpermute(fsc_ctx* ctx, int on);
/* Grouped-GEMM tile schedule: on > 0 dynamic (each CTA pair after its first tile claims
 * the next one from an atomic counter and hands it to its roles through a shared-memory
 * queue, so pairs that start late beside co-running kernels take fewer tiles), 0 the
 * static stride, < 0 (default) dynamic at EP > 1 only (where the dispatch / combine CTAs
 * share the SMs). The results are bitwise the same either way. */
FSC_API int fsc_set_gemm_dynamic(fsc_ctx* ctx, int on);
/* Router (K1) on the tensor cores, one fused kernel (router_tc_kernel; E <= 128,
 * d % 128 == 0, k <= 8): RMS statistics, xn, base-2^7 digit planes of x_t / s_t and
 * of gamma (.) W_R / s_e (s powers of two), their products summed exactly in int32
 * (tcgen05 kind::i8) and combined exactly in fp64, then the same selection, fp64 band
 * refinement and results contract as the fp32 SIMT router (both equal the fp64
 * oracle's selection; the fp32 gates differ by rounding). on != 0 (default -1 = auto):
 * wherever the shape allows it; 0: the fp32 SIMT router. The digit workspace
 * (3 x 128 x d int8) is allocated at fsc_init. */
FSC_API int fsc_set_router_int8(fsc_ctx* ctx, int on);
/* Router (K1) for small batches in fp64 (router_f64_kernel; d % 64 == 0, d <= 8192,
 * E <= 128): the same definition (RMSNorm C-amb-5; top-k, exact ties to the
 * lower id, slots ascending by id, renormalised gates) with every product and sum in
 * fp64 in a fixed order, so the selection is the fp64 oracle's with no error bound or
 * refinement (n_refined is not written). on = 1: every call; 0: never; -1 (default,
 * auto): calls with T x EP x d <= 2.7e8 (EP = E padded to 32 / 64 / 128: decode batches) unless fsc_set_router_int8(ctx, 0) selected the
 * fp32 SIMT router. Workspace (d x 136 doubles, gamma (.) W_R) allocated at fsc_init. Returns FSC_ERR_CONFIG for on = 1 on an unsupported
 * shape. */
FSC_API int fsc_set_router_f64(fsc_ctx* ctx, int on);
/* Select the EP data movement (FSC_EP_ALLTOALL default, FSC_EP_ALLREDUCE). Must be
 * called before fsc_bootstrap_export (it re-creates the peer region). In
 * FSC_EP_ALLREDUCE the shared expert is computed replicated on every rank (no
 * extra collective), the routed partials are all-reduced; the FarSkip entry
 * returns with the all-reduce in flight and fsc_moe_wait completes it (the
 * "synchronize only before the next MoE computation" of P:217). In this mode
 * fsc_layer_stack_forward runs the attention tensor-parallel: each rank passes its
 * head slice (n_heads / P query and n_kv_heads / P kv heads, the matching w_qkv rows
 * and w_o columns); the o-projection partials are all-reduced on a second channel
 * and, in Hybrid layers, waited only before the next attention. */
FSC_API int fsc_set_ep_mode(fsc_ctx* ctx, int mode);
/* EP > 1 all-to-all: on != 0 sends the Dispatch payload as FP8 e4m3 with one fp32
 * scale per 128 columns (s = amax / 448, q = e4m3_rn_satfinite(x / s); the receiver
 * rebuilds bf16(q * s)), halving the dispatch bytes (the paper's
 * inference runs FP8). Lossy (e4m3): its own tolerance, parity against the
 * oracle's moe_block_ep_fp8. d % 128 == 0. Call before fsc_bootstrap_export. */
FSC_API int fsc_set_dispatch_fp8(fsc_ctx* ctx, int on);

/* Combine data path (FSC_COMBINE_STREAM default / FSC_COMBINE_FUSED, see above). */
FSC_API int fsc_set_combine_mode(fsc_ctx* ctx, int mode);
/* Schedule of fsc_moe_forward_blocking at EP > 1 (FSC_BLOCKING_REGULAR_PLUS default / SERIAL). */
FSC_API int fsc_set_blocking_mode(fsc_ctx* ctx, int mode);
/* CTAs of the dispatch and combine kernels (default 64: a fraction of the 148 SMs, so that
 * the overlapped compute keeps most of them). 1 <= n <= 592. */
FSC_API int fsc_set_comm_ctas(fsc_ctx* ctx, int n);
/* Measurement instrument ("zero-byte all-to-all"): on != 0 keeps the counts
 * exchange, the flags and every kernel launch of the all-to-all but moves no payload rows
 * (the expert GEMMs run on whatever the receive buffer holds; results are garbage). The
 * exposed all-to-all time of a schedule is t_layer(real) - t_layer(zero-byte). */
FSC_API int fsc_set_a2a_zero_bytes(fsc_ctx* ctx, int on);
/* Test instrument for the stream wiring (the SPEC S:437 golden replay):
 * with unit_ns != NULL ([FSC_SPIN_N] nanoseconds), every phase of the MoE calls and of
 * fsc_layer_stack_forward launches ONE single-thread spin kernel of that duration instead
 * of its real kernels, on the same stream and behind the same events (gate = router +
 * maps, dispatch, qkv = attention part (a), core = part (b), routed = both expert GEMMs,
 * combine, shared). Nothing is computed. NULL restores the real kernels. */
FSC_API int fsc_set_spin_schedule(fsc_ctx* ctx, const long long* unit_ns);
/* Test instrument: a spin kernel of a pseudo-random duration in [0, max_ns] (xorshift32 from
 * seed) before every compute and communication stage; the results must not change. 0 = off. */
FSC_API int fsc_set_delay_fuzz(fsc_ctx* ctx, unsigned seed, long long max_ns);

/* Debug finiteness check (the error class of SPEC S:29): when on, every
 * fsc_moe_forward_blocking, fsc_moe_wait (and so every layer of
 * fsc_layer_stack_forward) counts the non-finite values of its fp32 output on the
 * device, SYNCHRONISES the stream and returns FSC_ERR_NONFINITE (not sticky) if
 * there is any. Not allowed under stream capture (FSC_ERR_STATE). Default off. */
FSC_API int fsc_set_debug_checks(fsc_ctx* ctx, int on);

/* Per-phase CUDA-event timing of the MoE calls (bench / profiling). When enabled,
 * events are recorded on the call's stream around every phase; fsc_get_timings
 * waits for the last call's events and writes n <= 9 durations in ms (-1 = phase
 * not run) in the order: router, perm_maps, dispatch (permute), gemm1 (SwiGLU),
 * gemm2 (down), combine, shared1, shared2, unpermute, dispatch_stall, combine_wait.
 * Returns the phase count. */
FSC_API int fsc_set_timing(fsc_ctx* ctx, int enable);
/* As fsc_set_timing, timing only the phases whose bit (1u << phase id) is set in
 * `mask` (0 disables timing). Used by the bench to time one kernel inside the
 * timed region without instrumenting the rest of the step. */
FSC_API int fsc_set_timing_mask(fsc_ctx* ctx, unsigned mask);
FSC_API int fsc_get_timings(fsc_ctx* ctx, float* ms, int n);
/* Every timed phase instance since fsc_set_timing (phase ids as above, then
 * 9 = dispatch stall of the compute stream, 10 = combine wait); waits for the
 * events, writes up to cap (phase, ms) pairs, returns the count and clears the log. */
FSC_API int fsc_timing_log(fsc_ctx* ctx, int* phase, float* ms, int cap);
/* Timeline of every logged phase instance (same ids, plus 11 = attention part (a): norm +
 * QKV + RoPE, 12 = attention part (b): core + o-projection, both from
 * fsc_layer_stack_forward): phase, stream (0 = the caller's compute stream, 1 = the
 * communication stream, 2 = the auxiliary compute stream), start offset from the first
 * logged instance and duration, in ms (CUDA events on the phase's stream). Waits for the
 * events, returns the count and clears the log; FSC_ERR_STATE if instances were dropped
 * (more than 4096 between two reads, or more than cap). Any output may be NULL. */
FSC_API int fsc_timeline(fsc_ctx* ctx, int* phase, int* stream, float* t0_ms, float* dur_ms, int cap);
/* Cumulative number of CUDA kernels launched by libfsc in this process. */
FSC_API long fsc_launch_count(void);

/* ---------------------------------------------------------------- MoE sub-block */

/* Regular (blocking) MoE sub-block, Eq. 6, P:103 steps 3-6:
 *   out[T,d] = (x_in + shared(xn)) + routed(xn),  fp32, out may alias x_in.
 * All collectives are waited on inside, in stream order. */
FSC_API int fsc_moe_forward_blocking(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in, float* out,
                             const fsc_moe_debug* dbg, void* stream);

/* Same as fsc_moe_forward_blocking but x_in/out are HOST buffers (pinned for
 * speed): H2D copy, forward, D2H copy, then the stream is synchronised. */
FSC_API int fsc_moe_forward_blocking_host(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in_host,
                                  float* out_host, void* stream);

/* Pipelined host-buffer variant for serving loops: enqueues the H2D copy of
 * x_in_host (pinned) on an internal copy stream, the forward on `stream` and the
 * D2H copy into out_host (pinned) on a second copy stream, ordered by events on
 * three internal staging slots, and returns at once. Step i's compute therefore
 * overlaps step i+1's upload and step i-1's download. The host buffers of call i
 * may be reused once call i+3 has returned (call i+3 waits on the host for call i's
 * download before it enqueues anything) or after fsc_host_flush. The first call
 * allocates the three device staging slots and the copy streams (kept until
 * fsc_finalize). */
FSC_API int fsc_moe_forward_host_async(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in_host,
                                       float* out_host, void* stream);
/* Wait until every fsc_moe_forward_host_async output has reached host memory. */
FSC_API int fsc_host_flush(fsc_ctx* ctx);

/* FarSkip MoE sub-block (schedule P:198 steps 3-8):
 *   x_in          = mlp-in_k = o_{k-1}        fp32 [T,d]
 *   partial_inout = attn-in_{k+1} in progress: on entry (mlp-in_k + attn-out_k),
 *                   on return (in stream order) += shared-exp-out_k  (C-amb-12)
 * The routed output stays pending in *h until fsc_moe_wait. At most one
 * handle may be outstanding per context (FSC_ERR_STATE otherwise). */
FSC_API int fsc_moe_forward_farskip(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in, float* partial_inout,
                            fsc_overlap_cb cb, void* user, fsc_handle* h, const fsc_moe_debug* dbg, void* stream);

/* Complete a FarSkip handle: waits (in stream order) for its combine and writes
 *   full_out = partial_in + routed-exp-out_k   (= mlp-in_{k+1} = o_k)
 * full_out may alias partial_in. FSC_ERR_STATE if h was already waited.
 * Stream requirement: call fsc_moe_wait on the SAME stream as the
 * fsc_moe_forward_farskip that made h, and issue the next fsc_moe_forward_farskip
 * on that stream too (or order the streams with events yourself): the next call
 * reuses the receive / combine buffers that this wait reads (write-after-read). */
FSC_API int fsc_moe_wait(fsc_ctx* ctx, fsc_handle h, const float* partial_in, float* full_out, void* stream);

/* ---------------------------------------------------------------- backward */

/* Gradients of one MoE sub-block, all fp32, caller-owned device buffers (any NULL except dx
 * = not wanted; written, not accumulated):
 *   dx        [T, d]        dL/dx_in (this rank's tokens)
 *   dgamma    [d]           RMSNorm weight (this rank's tokens)
 *   dw_router [E, d]        router W_R (this rank's tokens)
 *   dw1, dw2  [E_loc, c, d], dw3 [E_loc, d, c]   this rank's experts, from every rank's tokens
 *   dws1, dws2 [c_s, d], dws3 [d, c_s]           shared expert (this rank's tokens)
 * The data-parallel reduction of the replicated weights' gradients (gamma, W_R, shared) over
 * the EP ranks is the caller's. */
typedef struct {
  float* dx;
  float* dgamma;
  float* dw_router;
  float* dw1;
  float* dw2;
  float* dw3;
  float* dws1;
  float* dws2;
  float* dws3;
} fsc_moe_grads;

/* Backward of out = x_in + shared(xn) + routed(xn) (the sub-block of Eq. 6 / A5; the
 * far-skip connections are identities, so the FarSkip wiring routes the same gradients,
 * P:207-211) given grad_out = dL/dout fp32 [T, d]. Recomputes the forward's routing and
 * expert inputs from x_in (activation recomputation), then, in this stream order:
 * gradient Dispatch (G rows + gates to the experts' owners) on the communication stream
 * while the shared expert's backward runs; routed dgrad (dh = G W3, SwiGLU backward on the
 * recomputed u, v, dX = [dU | dV] [W1 ; W2]); gradient Combine of dX and the gate gradients
 * on the communication stream while the routed weight gradients run (the explicit order that
 * replaces the paper's autograd re-prioritisation); then the router and RMSNorm backward per
 * token. All-to-all EP mode (or EP = 1) only. Allocates its workspace on the first call.
 * Errors as the forward (FSC_ERR_CONFIG in the all-reduce EP mode). */
FSC_API int fsc_moe_backward(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in,
                             const float* grad_out, const fsc_moe_grads* grads, void* stream);

/* ---------------------------------------------------------------- stack */

/* Attention filler weights (causal GQA + RoPE, C-amb-18):
 *   gamma fp32 [d]; w_qkv bf16 [(Hq + 2 Hkv) * hd, d] (q heads, k heads, v heads);
 *   w_o bf16 [d, Hq * hd]; hd in {64, 128}... see DESIGN.md. */
typedef struct {
  const float* gamma;
  const void* w_qkv;
  const void* w_o;
  int n_heads;
  int n_kv_heads;
  int head_dim;
  float rope_theta;
} fsc_attn_weights;

/* Optional per-layer fp32 [T,d] activations; any pointer may be NULL. */
typedef struct {
  float* attn_in;
  float* mlp_in;
  float* attn_out;
  float* shared_out;
  float* routed_out;
  float* o;
} fsc_act_cache;

/* L-layer stack o_0 -> o_L (fp32 [T,d]), T tokens packed as sequences of
 * seq_len (T % seq_len == 0). modes[k] in {FSC_REGULAR, FSC_HYBRID} per layer
 * (partial conversion allowed); schedule FSC_BLOCKING serialises every
 * collective, FSC_OVERLAPPED runs the P:198 order with collectives on the comm
 * stream. attn/moe are arrays of L layers; cache is NULL or an array of L. Every
 * layer's arguments are validated before anything is enqueued. The first call allocates
 * the attention workspace (normed input, qkv, core output, 3 rotating fp32 residual
 * buffers), grown when a later call needs wider projections. */
FSC_API int fsc_layer_stack_forward(fsc_ctx* ctx, const fsc_attn_weights* attn, const fsc_moe_weights* moe, int L, int T,
                            int seq_len, const int* modes, int schedule, const float* o0, float* oL,
                            const fsc_act_cache* cache, void* stream);

/* ---------------------------------------------------------------- op-level entry points (tests, bench) */

/* K1: xn bf16 [T,d], topk_idx int32 [T,k], topk_w fp32 [T,k], logits fp32 [T,E] or NULL. */
FSC_API int fsc_op_router(fsc_ctx* ctx, const float* x, const float* gamma, const float* w_router, int T, int d, int E,
                  int k, void* xn, int* topk_idx, float* topk_w, float* logits, int* n_refined, void* stream);
/* K2: counts int32 [E], offsets int32 [E+1], pos int32 [T,k], src_row int32 [T*k]. */
FSC_API int fsc_op_perm_maps(fsc_ctx* ctx, const int* topk_idx, int T, int k, int E, int* counts, int* offsets, int* pos,
                     int* src_row, void* stream);
/* K3: xs[p] = xn[src_row[p]], bf16 rows of d, p < R. */
FSC_API int fsc_op_permute(fsc_ctx* ctx, const void* xn, const int* src_row, void* xs, int R, int d, void* stream);
/* K4: grouped GEMM over G groups with device counts [G] (NULL -> one group of m_total rows).
 *   epi 0: out bf16 [M, N] = A B0_g^T             (B0 [G*N, K])
 *   epi 1: out bf16 [M, N] = (A B0_g^T) * SiLU(A B1_g^T)   (B0 = W1, B1 = W2, each [G*N, K])
 *   epi 2: out fp32 [M, N] = resid + A B0_g^T (resid may be NULL -> 0, may alias out) */
FSC_API int fsc_op_grouped_gemm(fsc_ctx* ctx, int epi, const void* A, long a_rows, const void* B0, const void* B1, int G,
                        const int* counts, int m_total, int N, int K, void* out, const float* resid, void* stream);
/* K4 with the A operand gathered (EP = 1 fused permute, "requiring
 * permutation of A"): row r of the grouped problem is row a_idx[r] of A [a_rows, K]
 * (int32 a_idx [sum of counts], device), loaded by TMA gather4 inside the GEMM;
 * otherwise as fsc_op_grouped_gemm. a_idx == NULL is fsc_op_grouped_gemm. */
FSC_API int fsc_op_grouped_gemm_gather(fsc_ctx* ctx, int epi, const void* A, long a_rows, const int* a_idx,
                                       const void* B0, const void* B1, int G, const int* counts, int m_total, int N,
                                       int K, void* out, const float* resid, void* stream);
/* K5: out fp32 [T,d] = resid + sum_j w[t,j] y[pos[t,j]] (resid may be NULL -> 0). */
/* Core attention of the stack's filler (P:198 part (b) without the o-projection): qkv bf16
 * [T, (Hq + 2 Hkv) hd] (q heads | k heads | v heads, RoPE applied), out bf16 [T, Hq hd] =
 * softmax(q k^T / sqrt(hd), causal within packed sequences of seq_len) v per head (GQA:
 * head h reads kv head h / (Hq / Hkv)). hd = 128 with seq_len % 128 == 0 runs the tcgen05
 * kernel, otherwise the mma.sync one (hd in {16, 32, 64, 128}). Test entry point. */
FSC_API int fsc_op_attention(fsc_ctx* ctx, const void* qkv, void* out, int T, int Hq, int Hkv, int hd, int seq_len,
                             void* stream);
FSC_API int fsc_op_unpermute(fsc_ctx* ctx, const void* y, const int* pos, const float* w, const float* resid, float* out,
                     int T, int k, int d, void* stream);

/* K4 backward, dgrad (MN-major B): per group g, out[rows of g] = A[rows of g] B_g with
 * B_g = rows [g * b_group_rows, +K) of B0 read as [K, N] (row-major, N contiguous); with
 * kb_split > 0 the K rows are [B0 rows (kb_split * 64) ; B1 rows (K - kb_split * 64)].
 * epi 0: bf16 out [M, N]; epi 2: fp32 out = resid + A B (resid may be NULL). */
FSC_API int fsc_op_gemm_dgrad(fsc_ctx* ctx, int epi, const void* A, long a_rows, const void* B0, const void* B1,
                              long b_group_rows, int G, const int* counts, int m_total, int N, int K, int kb_split,
                              void* out, const float* resid, void* stream);
/* K4 backward, SwiGLU backward with recomputation: u = A W1_g^T, v = A W2_g^T (B0 = W1,
 * B1 = W2 as [G*N, K]); dh bf16 [M, N]; row_gate fp32 [M] or NULL (1): h = u SiLU(v),
 * du = g dh SiLU(v), dv = g dh u SiLU'(v) -> duv bf16 [M, 2N] = [du | dv], hg bf16 [M, N] = g h,
 * dg_part fp32 [M, dg_ld] (NULL: skipped) = per-tile partial sums of h * dh (2 per N tile). */
FSC_API int fsc_op_gemm_swiglu_bwd(fsc_ctx* ctx, const void* A, long a_rows, const void* B0, const void* B1, int G,
                                   const int* counts, int m_total, int N, int K, const void* dh,
                                   const float* row_gate, void* duv, void* hg, float* dg_part, int dg_ld,
                                   void* stream);
/* K4 backward, wgrad: out[g][i][j] (+)= sum over group g's rows m of A[m, a_col0 + i] B[m, b_col0 + j]
 * (A [a_rows, lda], B [a_rows, ldb] bf16; out fp32 [G, N1, N2]; N2 % 64 == 0). */
FSC_API int fsc_op_gemm_wgrad(fsc_ctx* ctx, const int* counts, int G, int m_total, int N1, int N2, const void* A,
                              long a_rows, long lda, int a_col0, const void* B, long ldb, int b_col0, float* out,
                              int accumulate, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FSC_H_ */
