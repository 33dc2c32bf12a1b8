// Internal definition of the opaque fsc_ctx (include/fsc.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fsc.h"

struct fsc_handle_s {
  fsc_ctx* ctx;
  int T;
  int live;
  float* dbg_routed;
};

struct fsc_peer_state;  // transport.cu

// phases timed with CUDA events when timing is enabled (fsc_get_timings order)
enum { PH_ROUTER = 0, PH_PERM, PH_DISPATCH, PH_GEMM1, PH_GEMM2, PH_COMBINE, PH_SHARED1, PH_SHARED2, PH_UNPERMUTE,
       PH_DISPATCH_STALL, PH_COMBINE_WAIT, PH_ATTN_A, PH_ATTN_B, PH_N };
constexpr int kLogEvents = 8192;   // 4096 phase instances between two fsc_timeline reads
// spin-schedule phases (fsc_set_spin_schedule; SPEC S:437 duration names)
enum { SP_GATE = 0, SP_DISPATCH, SP_QKV, SP_CORE, SP_ROUTED, SP_COMBINE, SP_SHARED, SP_N };

struct fsc_ctx {
  int rank = 0, ep = 1, device = 0;
  fsc_moe_config cfg{};
  int e_loc = 0;
  long max_recv = 0;
  int gemm_ctas = 148;
  int gemm_cg = 0;             // 0 = auto (routed GEMMs: pairs at prefill, single CTAs at decode), 1, 2
  int fuse_unpermute = -1;     // blocking EP = 1: unpermute fused into GEMM2 (-1 auto: top-1)
  int dispatch_fp8 = 0;        // FP8 (e4m3, per-128-column scales) dispatch payload, EP > 1 all-to-all
  int ep_mode = 0;             // FSC_EP_ALLTOALL (dispatch / combine) or FSC_EP_ALLREDUCE (replicated tokens)
  int gemm_dyn = -1;           // dynamic GEMM tile schedule: 1 on, 0 off, -1 auto (EP > 1)
  int router_i8 = -1;          // exact int8 tensor-core router: 1 on, 0 off, -1 auto (fsc_set_router_int8)
  int router_f64 = -1;         // fp64 small-batch router: 1 on, 0 off, -1 auto (fsc_set_router_f64)
  int gather_a = 0;            // EP = 1: GEMM1 gathers A through src_row (fused permute)
  int combine_mode = 0;        // FSC_COMBINE_STREAM (comm-stream push after GEMM2) or FSC_COMBINE_FUSED
  int blocking_mode = 0;       // fsc_moe_forward_blocking: FSC_BLOCKING_REGULAR_PLUS or FSC_BLOCKING_SERIAL
  int a2a_zero_bytes = 0;      // test instrument: all-to-all flags / counts only, no payload rows
  int comm_ctas = 64;          // CTAs of the dispatch / combine kernels (a fraction of the SMs)
  long long spin_ns[SP_N] = {};   // fsc_set_spin_schedule: one spin kernel per phase instead of the real work
  int spin = 0;
  unsigned fuzz_seed = 0;      // fsc_set_delay_fuzz: random spin delays before every stage
  long long fuzz_max_ns = 0;
  int comb_async = 0;          // the last MoE call's combine runs on the comm stream (ev_comb)
  int sticky = 0;
  int debug_checks = 0;        // fsc_set_debug_checks: finiteness check of every output (syncs)
  int* nf_count = nullptr;     // [1] device counter of non-finite output values
  char err[512] = {0};

  // per-call workspace (device), sized for cfg at fsc_init
  uint16_t* xn = nullptr;      // bf16 [T, d]        normalised tokens
  int* topk_idx = nullptr;     // [T, k]
  float* topk_w = nullptr;     // [T, k]
  int* pos = nullptr;          // [T, k]             row of copy (t,j) in the send layout
  int* src_row = nullptr;      // [T*k]              token of send row p
  int* hist = nullptr;         // [chunks, E]
  int* base = nullptr;         // [chunks, E]
  int* counts = nullptr;       // [E]                copies per global expert (this rank)
  int* offsets = nullptr;      // [E+1]
  int* comb_cnt = nullptr;     // [T, d/32]         fused-unpermute arrival counters
  int* gemm_sched = nullptr;   // [kSchedSlots, 2]  dynamic GEMM tile schedules, one per launch site (zero between launches)
  int8_t* i8_w = nullptr;      // exact tensor-core router workspace: digit planes of gamma W_R, [3, 128, d]
  float* i8_exp = nullptr;     // per-expert scale and error-bound coefficients, [3, 128]
  float* r_part = nullptr;     // [kRouterSplitRows, 128] split-d partial logits (small T)
  double* r_part_sq = nullptr; // [kRouterSplitRows]      split-d partial sums of x^2
  float* w_scaled = nullptr;   // [E, d]             gamma * W_R
  double* f64_w = nullptr;     // [d, 136]           fp64 router: gamma (.) W_R, k-major (E <= 128)
  float* w_sq = nullptr;       // [E]                ||gamma * W_R[e]||^2
  uint16_t* xs = nullptr;      // bf16 [T*k, d]      expert-sorted send buffer
  uint16_t* h = nullptr;       // bf16 [max_recv, c] SwiGLU activations
  uint16_t* y = nullptr;       // bf16 [T*k, d]      expert outputs in the send layout (EP=1)
  uint16_t* hs = nullptr;      // bf16 [T, c_s]      shared-expert activations
  float* tmp = nullptr;        // fp32 [T, d]
  float* io_in = nullptr;      // fp32 [T, d]        staging for the *_host entry point
  float* io_out = nullptr;

  // EP > 1: receive side (transport.cu); symmetric across ranks
  uint16_t* xr = nullptr;      // bf16 [max_recv, d] received rows, expert-major then source
  uint16_t* yr = nullptr;      // bf16 [max_recv, d] expert outputs in the receive layout
  uint16_t* ys = nullptr;      // bf16 [T*k, d]      combined rows back in the send layout
  int* recv_counts = nullptr;  // [E_loc]            rows received per local expert
  long recv_rows_cap = 0;
  fsc_peer_state* peer = nullptr;

  cudaStream_t comm = nullptr;  // high-priority communication stream
  cudaStream_t aux = nullptr;   // second compute stream (overlaps independent kernels)
  // pipelined host entry point (fsc_moe_forward_host_async)
  cudaStream_t h2d = nullptr, d2h = nullptr;
  static constexpr int kIoSlots = 3;   // call i reuses the slot of call i - 3
  float* io_slot_in[kIoSlots] = {};
  float* io_slot_out[kIoSlots] = {};
  cudaEvent_t ev_in[kIoSlots] = {}, ev_cdone[kIoSlots] = {}, ev_out[kIoSlots] = {};
  int io_slot = 0;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_c = nullptr, ev_d = nullptr;
  cudaEvent_t ev_t1 = nullptr, ev_t2 = nullptr;   // TP attention all-reduce (stack)
  cudaEvent_t ev_g2 = nullptr, ev_comb = nullptr; // GEMM2 done (compute) -> combine done (comm)
  int attn_pending = 0;        // 1: attention all-reduce in line, 2: on the comm stream
  float* attn_cache = nullptr;
  int attn_T = 0;

  int pending = 0;
  int no_overlap = 0;          // FarSkip call made under the BLOCKING stack schedule

  // layer-stack workspace (stack.cu), allocated on first use
  uint16_t* hn = nullptr;      // bf16 [T, d]           normalised attention input
  uint16_t* qkv = nullptr;     // bf16 [T, (Hq+2Hkv)hd]
  uint16_t* ao = nullptr;      // bf16 [T, Hq hd]       attention core output
  float* rbuf[3] = {nullptr, nullptr, nullptr};  // fp32 [T, d] rotating residual buffers
  long stack_cap_qkv = 0, stack_cap_ao = 0;
  int timing = 0;
  unsigned timing_mask = ~0u;   // bit i: time phase i
  cudaEvent_t ph_ev[PH_N][2] = {};
  int ph_used[PH_N] = {};
  // timing log: every phase instance since the last reset (bench: per-layer exposure)
  cudaEvent_t log_ev[kLogEvents] = {};
  int log_phase[kLogEvents / 2] = {};
  int log_stream[kLogEvents / 2] = {};   // 0 = caller's (compute) stream, 1 = comm, 2 = aux
  int log_n = 0;
  long log_dropped = 0;                  // phase instances not logged (log full): reported as an error
  fsc_handle_s handle{};
  // backward workspace (moe_bwd.cu), allocated on the first fsc_moe_backward call
  uint16_t* b_gb = nullptr;     // bf16 [T, d]              G
  uint16_t* b_duv = nullptr;    // bf16 [rows, 2 max(c, c_s)] [dU | dV]
  uint16_t* b_hg = nullptr;     // bf16 [rows, max(c, c_s)] g * h
  float* b_dgpart = nullptr;    // fp32 [rows, b_dg_ld]     gate-gradient partials
  int b_dg_ld = 0;
  float* b_dlrow = nullptr;     // fp32 [T * k]             logit gradients per send row
  float* b_rtok = nullptr;      // fp32 [T]                 RMS factors
  float* b_colpart = nullptr;   // fp32 [T / 64, d]         dgamma partial column sums
  uint16_t* b_gr = nullptr;     // EP = 1: bf16 [T * k, d]  gradient rows (expert-sorted)
  float* b_gate = nullptr;      // EP = 1: fp32 [T * k]     their gates
};

void fsc_set_error(fsc_ctx* c, const char* fmt, ...);
// phase timing (CUDA events on the phase's stream, logged for fsc_timeline)
cudaError_t fsc_phase_begin(fsc_ctx* ctx, int i, cudaStream_t st);
cudaError_t fsc_phase_end(fsc_ctx* ctx, int i, cudaStream_t st);
// test instruments: spin kernel for spin-schedule phase sp; random delay (delay fuzz)
cudaError_t fsc_spin(fsc_ctx* ctx, int sp, cudaStream_t st);
cudaError_t fsc_fuzz(fsc_ctx* ctx, cudaStream_t st);
// argument checks of one MoE call (weights, T, activation pointers, alignment); no enqueue
int fsc_validate_moe(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in, const void* out);
// debug finiteness check of an fp32 [n] output (fsc_set_debug_checks): synchronises s
// dynamic tile-schedule counter pairs of the grouped GEMM, one per launch site (launches
// that may run concurrently must not share one)
enum { SCHED_SHARED1 = 0, SCHED_SHARED2, SCHED_ROUTED1, SCHED_ROUTED2, SCHED_OP, kSchedSlots = 32 };
// The dynamic schedule is on where kernels co-run with the GEMMs on the same SMs (EP > 1:
// dispatch / combine CTAs); at EP = 1 the static stride is as balanced and avoids the per-tile
// hand-off (A/B). fsc_set_gemm_dynamic overrides.
inline int* gemm_sched_slot(const fsc_ctx* ctx, int slot) {
  const bool on = ctx->gemm_dyn >= 0 ? ctx->gemm_dyn != 0 : ctx->ep > 1;
  return on && ctx->gemm_sched ? ctx->gemm_sched + 2 * slot : nullptr;
}
// the exact tensor-core router (router_tc_kernel) is used for this context's forward and backward
bool router_tc_on(const fsc_ctx* ctx);
// fp64 small-batch router for this call (fsc_set_router_f64: forced, off, or auto = T small)
bool router_f64_on(const fsc_ctx* ctx, int T, int d, int E, int k);
int fsc_check_finite(fsc_ctx* ctx, const float* out, long n, cudaStream_t s, const char* what);

// transport (EP > 1). All return fsc_status.
size_t fsc_transport_blob_size();
int fsc_transport_init(fsc_ctx* ctx);
int fsc_transport_export(fsc_ctx* ctx, void* blob);
int fsc_transport_import(fsc_ctx* ctx, const void* blobs);
void fsc_transport_finalize(fsc_ctx* ctx);
int fsc_transport_dispatch(fsc_ctx* ctx, int T, cudaStream_t s);
int fsc_transport_dispatch_wait(fsc_ctx* ctx, cudaStream_t s);
int fsc_transport_combine(fsc_ctx* ctx, int T, cudaStream_t s);
int fsc_transport_combine_wait(fsc_ctx* ctx, cudaStream_t s);
int fsc_transport_combine_push(fsc_ctx* ctx, const uint16_t* y, cudaStream_t s);
void fsc_transport_debug(fsc_ctx* ctx, const int** cnt, const int** ret);
void fsc_transport_bwd_ptrs(fsc_ctx* ctx, uint16_t** gr, float** gate, float** dgs);
int fsc_transport_dispatch_grad(fsc_ctx* ctx, int T, const float* G, cudaStream_t s);
int fsc_transport_combine_grad(fsc_ctx* ctx, const uint16_t* y, const float* dg_part, int dg_n, int dg_ld,
                               cudaStream_t s);
int fsc_transport_combine_grad_wait(fsc_ctx* ctx, cudaStream_t s);
void fsc_transport_scatter_target(fsc_ctx* ctx, const int** ret, void** peer_out);
// EP all-reduce channels: 0 = MoE routed sum, 1 = TP attention o-projection (stack)
float* fsc_transport_ar_partial(fsc_ctx* ctx, int ch = 0);
int fsc_transport_ar_start(fsc_ctx* ctx, int T, cudaStream_t s, int ch = 0);
int fsc_transport_ar_finish(fsc_ctx* ctx, int T, const float* resid, float* out, cudaStream_t s, int ch = 0);
int fsc_transport_reinit(fsc_ctx* ctx);
