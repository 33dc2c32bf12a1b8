// libfsc C ABI (include/fsc.h): context, workspace, argument validation and the
// two MoE schedules of the paper (blocking; FarSkip).
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>

#include "../../include/fsc.h"
#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

using namespace fsc;

// ---------------------------------------------------------------------------- helpers

void fsc_set_error(fsc_ctx* c, const char* fmt, ...) {
  if (!c) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(c->err, sizeof(c->err), fmt, ap);
  va_end(ap);
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e__ = (call);                                                                 \
    if (e__ != cudaSuccess) {                                                                 \
      fsc_set_error(ctx, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e__)); \
      ctx->sticky = FSC_ERR_CUDA;                                                             \
      return FSC_ERR_CUDA;                                                                    \
    }                                                                                         \
  } while (0)

#define REQUIRE(cond, code, ...)            \
  do {                                      \
    if (!(cond)) {                          \
      fsc_set_error(ctx, __VA_ARGS__);      \
      return code;                          \
    }                                       \
  } while (0)

namespace fsc {
long g_launches = 0;
}

// Phase events are recorded with cudaEventRecordExternal so that, under stream
// capture, they become event-record nodes of the graph: a replayed graph then
// times its own phases (bench: per-kernel times inside the timed region).
static cudaError_t ph_record(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(st, &cs);
  if (e != cudaSuccess) return e;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal)
                                             : cudaEventRecord(ev, st);
}

static bool ph_on(const fsc_ctx* ctx, int i) { return ctx->timing && ((ctx->timing_mask >> i) & 1u); }

cudaError_t fsc_phase_begin(fsc_ctx* ctx, int i, cudaStream_t st) {
  if (!ph_on(ctx, i)) return cudaSuccess;
  cudaError_t e = ph_record(ctx->ph_ev[i][0], st);
  if (e == cudaSuccess && ctx->log_n < kLogEvents / 2) e = ph_record(ctx->log_ev[2 * ctx->log_n], st);
  return e;
}

cudaError_t fsc_phase_end(fsc_ctx* ctx, int i, cudaStream_t st) {
  if (!ph_on(ctx, i)) return cudaSuccess;
  cudaError_t e = ph_record(ctx->ph_ev[i][1], st);
  ctx->ph_used[i] = 1;
  if (ctx->log_n < kLogEvents / 2) {
    if (e == cudaSuccess) e = ph_record(ctx->log_ev[2 * ctx->log_n + 1], st);
    ctx->log_phase[ctx->log_n] = i;
    ctx->log_stream[ctx->log_n] = st == ctx->comm ? 1 : (st == ctx->aux ? 2 : 0);
    ++ctx->log_n;
  } else {
    ++ctx->log_dropped;
  }
  return e;
}
#define PH_BEGIN_ON(i, st) CK(fsc_phase_begin(ctx, i, st))
#define PH_END_ON(i, st) CK(fsc_phase_end(ctx, i, st))
#define PH_BEGIN(i) PH_BEGIN_ON(i, s)
#define PH_END(i) PH_END_ON(i, s)

// Test instruments (fsc_set_spin_schedule / fsc_set_delay_fuzz): one spin kernel of the
// phase's duration instead of its real kernels; a random delay in front of a stage.
cudaError_t fsc_spin(fsc_ctx* ctx, int sp, cudaStream_t st) { return launch_spin(ctx->spin_ns[sp], st); }

cudaError_t fsc_fuzz(fsc_ctx* ctx, cudaStream_t st) {
  if (ctx->fuzz_max_ns <= 0) return cudaSuccess;
  unsigned x = ctx->fuzz_seed ? ctx->fuzz_seed : 0x9E3779B9u;   // xorshift32
  x ^= x << 13;
  x ^= x >> 17;
  x ^= x << 5;
  ctx->fuzz_seed = x;
  return launch_spin((long long)(x % 1000u) * ctx->fuzz_max_ns / 1000, st);
}
#define FUZZ(st) CK(fsc_fuzz(ctx, st))

constexpr int TB_DEFAULT = 32;   // RouterLaunch::rpb (set by launch_router)

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static int check_cfg(const fsc_moe_config* c, int ep, char* err, size_t n) {
  if (!c) { snprintf(err, n, "null config"); return FSC_ERR_CONFIG; }
  if (c->d <= 0 || c->d % 64 || c->d > 8192) { snprintf(err, n, "d=%d must be a positive multiple of 64", c->d); return FSC_ERR_CONFIG; }
  if (c->n_experts < 1 || c->n_experts > 128) { snprintf(err, n, "n_experts=%d outside [1,128]", c->n_experts); return FSC_ERR_CONFIG; }
  if (c->top_k < 1 || c->top_k > c->n_experts) { snprintf(err, n, "top_k=%d outside [1,E]", c->top_k); return FSC_ERR_CONFIG; }
  if (c->ffn <= 0 || c->ffn % 64) { snprintf(err, n, "ffn=%d must be a positive multiple of 64", c->ffn); return FSC_ERR_CONFIG; }
  if (c->shared_ffn < 0 || c->shared_ffn % 64) { snprintf(err, n, "shared_ffn=%d must be a multiple of 64", c->shared_ffn); return FSC_ERR_CONFIG; }
  if (c->max_tokens < 0) { snprintf(err, n, "max_tokens < 0"); return FSC_ERR_CONFIG; }
  if (ep < 1 || c->n_experts % ep) { snprintf(err, n, "n_experts=%d not divisible by ep_size=%d (C-amb-9)", c->n_experts, ep); return FSC_ERR_CONFIG; }
  return FSC_OK;
}

template <typename T>
static cudaError_t dalloc(T** p, size_t n) {
  if (n == 0) n = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
}

// ---------------------------------------------------------------------------- lifecycle

extern "C" size_t fsc_bootstrap_size(void) { return fsc_transport_blob_size(); }

extern "C" int fsc_init(fsc_ctx** out, int rank, int ep_size, int device, const fsc_moe_config* max_cfg) {
  if (!out) return FSC_ERR_SHAPE;
  *out = nullptr;
  char err[256];
  int rc = check_cfg(max_cfg, ep_size, err, sizeof(err));
  if (rc) { fprintf(stderr, "fsc_init: %s\n", err); return rc; }
  if (rank < 0 || rank >= ep_size) { fprintf(stderr, "fsc_init: rank %d outside [0,%d)\n", rank, ep_size); return FSC_ERR_CONFIG; }
  fsc_ctx* ctx = new (std::nothrow) fsc_ctx();
  if (!ctx) return FSC_ERR_CUDA;
  ctx->rank = rank;
  ctx->ep = ep_size;
  ctx->device = device;
  ctx->cfg = *max_cfg;
  ctx->e_loc = max_cfg->n_experts / ep_size;
  ctx->gemm_ctas = kNumSMs;
  *out = ctx;
  CK(cudaSetDevice(device));
  const fsc_moe_config& c = ctx->cfg;
  const long T = c.max_tokens, d = c.d, k = c.top_k, E = c.n_experts;
  const long per_src = T * (k < ctx->e_loc ? k : ctx->e_loc);
  ctx->max_recv = per_src * ep_size;  // worst-case rows received (dropless, C-amb-9)
  const long nch = perm_chunks((int)T);
  CK(dalloc(&ctx->xn, T * d));
  CK(dalloc(&ctx->topk_idx, T * k));
  CK(dalloc(&ctx->topk_w, T * k));
  CK(dalloc(&ctx->pos, T * k));
  CK(dalloc(&ctx->src_row, T * k));
  CK(dalloc(&ctx->hist, nch * E));
  CK(dalloc(&ctx->base, nch * E));
  CK(dalloc(&ctx->counts, E));
  CK(dalloc(&ctx->offsets, E + 1));
  CK(dalloc(&ctx->comb_cnt, T * (d / 32)));   // [T, d / (BN/2)] fused-unpermute counters, BN/2 >= 32
  CK(cudaMemset(ctx->comb_cnt, 0, sizeof(int) * T * (d / 32)));
  CK(dalloc(&ctx->gemm_sched, 2 * kSchedSlots));
  CK(cudaMemset(ctx->gemm_sched, 0, sizeof(int) * 2 * kSchedSlots));
  CK(dalloc(&ctx->r_part, (long)kRouterSplitRows * 128));
  CK(dalloc(&ctx->r_part_sq, (long)kRouterSplitRows));
  CK(dalloc(&ctx->w_scaled, (E > 128 ? E : 128) * d));  // e-major [E][d] or k-major [d][EP<=128]
  CK(dalloc(&ctx->w_sq, E));
  if (E <= 128) CK(dalloc(&ctx->f64_w, (long)d * 136));
  CK(dalloc(&ctx->xs, (T * k > ctx->max_recv ? T * k : ctx->max_recv) * d));
  CK(dalloc(&ctx->h, ctx->max_recv * (long)c.ffn));
  CK(dalloc(&ctx->y, (T * k > ctx->max_recv ? T * k : ctx->max_recv) * d));
  if (c.shared_ffn) CK(dalloc(&ctx->hs, T * (long)c.shared_ffn));
  CK(dalloc(&ctx->tmp, T * d));
  CK(dalloc(&ctx->io_in, T * d));
  CK(dalloc(&ctx->io_out, T * d));
  CK(dalloc(&ctx->nf_count, 1));
  CK(cudaStreamCreateWithPriority(&ctx->comm, cudaStreamNonBlocking, -5));
  CK(cudaEventCreateWithFlags(&ctx->ev_a, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_b, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_c, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_d, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_t1, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_t2, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_g2, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_comb, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
  rc = fsc_transport_init(ctx);
  if (rc) return rc;
  return fsc_set_router_int8(ctx, -1);   // auto router choice (see use_router_i8)
}

extern "C" int fsc_bootstrap_export(fsc_ctx* ctx, void* blob) {
  if (!ctx) return FSC_ERR_SHAPE;
  return fsc_transport_export(ctx, blob);
}

extern "C" int fsc_bootstrap_import(fsc_ctx* ctx, const void* blobs) {
  if (!ctx) return FSC_ERR_SHAPE;
  return fsc_transport_import(ctx, blobs);
}

extern "C" int fsc_finalize(fsc_ctx* ctx) {
  if (!ctx) return FSC_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  fsc_transport_finalize(ctx);
  void* bufs[] = {ctx->xn, ctx->topk_idx, ctx->topk_w, ctx->pos, ctx->src_row, ctx->hist, ctx->base, ctx->counts,
                  ctx->offsets, ctx->xs, ctx->h, ctx->y, ctx->hs, ctx->tmp, ctx->io_in, ctx->io_out, ctx->r_part, ctx->r_part_sq, ctx->comb_cnt, ctx->gemm_sched, ctx->i8_w, ctx->i8_exp, ctx->w_scaled, ctx->w_sq, ctx->f64_w, ctx->hn, ctx->qkv, ctx->ao, ctx->rbuf[0], ctx->rbuf[1], ctx->rbuf[2], ctx->nf_count, ctx->b_gb, ctx->b_duv, ctx->b_hg, ctx->b_dgpart, ctx->b_dlrow, ctx->b_rtok, ctx->b_gr, ctx->b_gate, ctx->b_colpart};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (ctx->comm) cudaStreamDestroy(ctx->comm);
  if (ctx->ev_a) cudaEventDestroy(ctx->ev_a);
  if (ctx->ev_b) cudaEventDestroy(ctx->ev_b);
  if (ctx->ev_c) cudaEventDestroy(ctx->ev_c);
  if (ctx->ev_d) cudaEventDestroy(ctx->ev_d);
  if (ctx->ev_t1) cudaEventDestroy(ctx->ev_t1);
  if (ctx->ev_t2) cudaEventDestroy(ctx->ev_t2);
  if (ctx->ev_g2) cudaEventDestroy(ctx->ev_g2);
  if (ctx->ev_comb) cudaEventDestroy(ctx->ev_comb);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
  if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
  for (int i = 0; i < fsc_ctx::kIoSlots; ++i) {
    if (ctx->io_slot_in[i]) cudaFree(ctx->io_slot_in[i]);
    if (ctx->io_slot_out[i]) cudaFree(ctx->io_slot_out[i]);
    if (ctx->ev_in[i]) cudaEventDestroy(ctx->ev_in[i]);
    if (ctx->ev_cdone[i]) cudaEventDestroy(ctx->ev_cdone[i]);
    if (ctx->ev_out[i]) cudaEventDestroy(ctx->ev_out[i]);
  }
  for (int i = 0; i < PH_N; ++i)
    for (int j = 0; j < 2; ++j)
      if (ctx->ph_ev[i][j]) cudaEventDestroy(ctx->ph_ev[i][j]);
  for (int i = 0; i < kLogEvents; ++i)
    if (ctx->log_ev[i]) cudaEventDestroy(ctx->log_ev[i]);
  delete ctx;
  return FSC_OK;
}

extern "C" const char* fsc_last_error(const fsc_ctx* ctx) { return ctx ? ctx->err : "null context"; }

extern "C" int fsc_set_timing(fsc_ctx* ctx, int enable) {
  if (!ctx) return FSC_ERR_SHAPE;
  CK(cudaSetDevice(ctx->device));
  if (enable && !ctx->ph_ev[0][0]) {
    for (int i = 0; i < PH_N; ++i)
      for (int j = 0; j < 2; ++j) CK(cudaEventCreate(&ctx->ph_ev[i][j]));
    for (int i = 0; i < kLogEvents; ++i) CK(cudaEventCreate(&ctx->log_ev[i]));
  }
  ctx->timing = enable ? 1 : 0;
  ctx->timing_mask = ~0u;
  ctx->log_n = 0;
  return FSC_OK;
}

extern "C" int fsc_set_timing_mask(fsc_ctx* ctx, unsigned mask) {
  if (!ctx) return FSC_ERR_SHAPE;
  int rc = fsc_set_timing(ctx, mask != 0);
  ctx->timing_mask = mask;
  return rc;
}

extern "C" int fsc_get_timings(fsc_ctx* ctx, float* ms, int n) {
  if (!ctx || !ms) return FSC_ERR_SHAPE;
  for (int i = 0; i < n && i < PH_N; ++i) {
    ms[i] = -1.f;
    if (ctx->timing && ctx->ph_used[i]) {
      CK(cudaEventSynchronize(ctx->ph_ev[i][1]));
      CK(cudaEventElapsedTime(&ms[i], ctx->ph_ev[i][0], ctx->ph_ev[i][1]));
    }
  }
  return PH_N;
}

extern "C" long fsc_launch_count(void) { return fsc::g_launches; }

extern "C" int fsc_timing_log(fsc_ctx* ctx, int* phase, float* ms, int cap) {
  return fsc_timeline(ctx, phase, nullptr, nullptr, ms, cap);
}

extern "C" int fsc_timeline(fsc_ctx* ctx, int* phase, int* stream, float* t0_ms, float* dur_ms, int cap) {
  if (!ctx) return FSC_ERR_SHAPE;
  const long dropped = ctx->log_dropped;
  const int n = ctx->log_n < cap ? ctx->log_n : cap;
  const long lost = dropped + (ctx->log_n - n);
  ctx->log_dropped = 0;
  if (n > 0) CK(cudaEventSynchronize(ctx->log_ev[2 * (n - 1) + 1]));
  for (int i = 0; i < n; ++i) {
    CK(cudaEventSynchronize(ctx->log_ev[2 * i + 1]));
    if (phase) phase[i] = ctx->log_phase[i];
    if (stream) stream[i] = ctx->log_stream[i];
    if (t0_ms) CK(cudaEventElapsedTime(&t0_ms[i], ctx->log_ev[0], ctx->log_ev[2 * i]));
    if (dur_ms) CK(cudaEventElapsedTime(&dur_ms[i], ctx->log_ev[2 * i], ctx->log_ev[2 * i + 1]));
  }
  ctx->log_n = 0;
  REQUIRE(lost == 0, FSC_ERR_STATE, "timing log overflow: %ld phase instances were not logged", lost);
  return n;
}

extern "C" int fsc_set_combine_mode(fsc_ctx* ctx, int mode) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(mode == FSC_COMBINE_STREAM || mode == FSC_COMBINE_FUSED, FSC_ERR_CONFIG, "unknown combine mode %d", mode);
  REQUIRE(!ctx->pending, FSC_ERR_STATE, "a FarSkip handle is outstanding");
  ctx->combine_mode = mode;
  return FSC_OK;
}

extern "C" int fsc_set_blocking_mode(fsc_ctx* ctx, int mode) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(mode == FSC_BLOCKING_REGULAR_PLUS || mode == FSC_BLOCKING_SERIAL, FSC_ERR_CONFIG,
          "unknown blocking mode %d", mode);
  ctx->blocking_mode = mode;
  return FSC_OK;
}

extern "C" int fsc_set_a2a_zero_bytes(fsc_ctx* ctx, int on) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(!ctx->pending, FSC_ERR_STATE, "a FarSkip handle is outstanding");
  ctx->a2a_zero_bytes = on ? 1 : 0;
  return FSC_OK;
}

extern "C" int fsc_set_comm_ctas(fsc_ctx* ctx, int n) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(n >= 1 && n <= 4 * kNumSMs, FSC_ERR_CONFIG, "comm ctas %d outside [1,592]", n);
  ctx->comm_ctas = n;
  return FSC_OK;
}

extern "C" int fsc_set_spin_schedule(fsc_ctx* ctx, const long long* unit_ns) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(!ctx->pending, FSC_ERR_STATE, "a FarSkip handle is outstanding");
  if (!unit_ns) {
    ctx->spin = 0;
    return FSC_OK;
  }
  for (int i = 0; i < SP_N; ++i) {
    REQUIRE(unit_ns[i] >= 0 && unit_ns[i] <= 10000000000ll, FSC_ERR_CONFIG, "spin duration %d out of range", i);
    ctx->spin_ns[i] = unit_ns[i];
  }
  ctx->spin = 1;
  return FSC_OK;
}

extern "C" int fsc_set_delay_fuzz(fsc_ctx* ctx, unsigned seed, long long max_ns) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(max_ns >= 0 && max_ns <= 1000000000ll, FSC_ERR_CONFIG, "fuzz delay out of range");
  ctx->fuzz_seed = seed;
  ctx->fuzz_max_ns = max_ns;
  return FSC_OK;
}

extern "C" int fsc_set_debug_checks(fsc_ctx* ctx, int on) {
  if (!ctx) return FSC_ERR_SHAPE;
  ctx->debug_checks = on ? 1 : 0;
  return FSC_OK;
}

int fsc_check_finite(fsc_ctx* ctx, const float* out, long n, cudaStream_t s, const char* what) {
  if (!ctx->debug_checks || n == 0) return FSC_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(s, &cs));
  REQUIRE(cs == cudaStreamCaptureStatusNone, FSC_ERR_STATE, "debug checks synchronise: not under stream capture");
  CK(cudaMemsetAsync(ctx->nf_count, 0, sizeof(int), s));
  CK(launch_count_nonfinite(out, n, ctx->nf_count, s));
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, ctx->nf_count, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  REQUIRE(bad == 0, FSC_ERR_NONFINITE, "%s: %d non-finite values (debug check)", what, bad);
  return FSC_OK;
}

extern "C" int fsc_set_gemm_cta_group(fsc_ctx* ctx, int cg) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(cg == 0 || cg == 1 || cg == 2, FSC_ERR_CONFIG, "cta_group must be 0 (auto), 1 or 2");
  ctx->gemm_cg = cg;
  return FSC_OK;
}

extern "C" int fsc_set_ep_mode(fsc_ctx* ctx, int mode) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(mode == FSC_EP_ALLTOALL || mode == FSC_EP_ALLREDUCE, FSC_ERR_CONFIG, "unknown EP mode %d", mode);
  REQUIRE(!ctx->pending, FSC_ERR_STATE, "a FarSkip handle is outstanding");
  if (mode == ctx->ep_mode) return FSC_OK;
  ctx->ep_mode = mode;
  if (ctx->ep == 1) return FSC_OK;
  CK(cudaSetDevice(ctx->device));
  return fsc_transport_reinit(ctx);   // new symmetric layout: bootstrap (export / import) after this
}

extern "C" int fsc_set_dispatch_fp8(fsc_ctx* ctx, int on) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(!ctx->pending, FSC_ERR_STATE, "a FarSkip handle is outstanding");
  REQUIRE(!on || ctx->cfg.d % 128 == 0, FSC_ERR_CONFIG, "FP8 dispatch needs d %% 128 == 0");
  if ((on ? 1 : 0) == ctx->dispatch_fp8) return FSC_OK;
  ctx->dispatch_fp8 = on ? 1 : 0;
  if (ctx->ep == 1) return FSC_OK;
  CK(cudaSetDevice(ctx->device));
  return fsc_transport_reinit(ctx);   // new symmetric layout: bootstrap (export / import) after this
}

static bool router_i8_ok(const fsc_ctx* ctx) {
  const fsc_moe_config& c = ctx->cfg;
  return c.n_experts <= 128 && c.d % 128 == 0 && c.top_k <= 8;
}

static int router_i8_alloc(fsc_ctx* ctx) {
  if (ctx->i8_w) return FSC_OK;   // allocated once (fsc_init / fsc_set_router_int8)
  CK(cudaSetDevice(ctx->device));
  CK(dalloc(&ctx->i8_w, 3L * 128 * ctx->cfg.d));
  CK(dalloc(&ctx->i8_exp, 3 * 128));
  return FSC_OK;
}

// The exact tensor-core router (router_tc_kernel) wherever the shape allows it (auto or on);
// the fp32 SIMT router otherwise or when switched off. Both select exactly the fp64 oracle's
// experts; their fp32 gates differ by rounding.
bool router_tc_on(const fsc_ctx* ctx) {
  return ctx->i8_w && router_i8_ok(ctx) && ctx->router_i8 != 0;
}

// The fp64 router (router_f64_kernel) for small batches, where the tensor-core router's
// phases are latency-bound: auto = T x EP x d <= 2.7e8 fp64 FMAs (EP = E padded to 32 / 64 /
// 128; measured: Qwen3 up to ~1024 tokens, DS-V2-Lite ~2048, Scout ~1600) unless the fp32
// SIMT router was selected (fsc_set_router_int8(ctx, 0), the A/B reference); on = any T.
bool router_f64_on(const fsc_ctx* ctx, int T, int d, int E, int k) {
  if (ctx->router_f64 == 0 || !ctx->f64_w || !router_f64_supported(d, E, k)) return false;
  if (ctx->router_f64 > 0) return true;
  const long ep = E <= 32 ? 32 : E <= 64 ? 64 : 128;
  return ctx->router_i8 != 0 && (double)T * ep * d <= 2.7e8;
}

extern "C" int fsc_set_router_f64(fsc_ctx* ctx, int on) {
  if (!ctx) return FSC_ERR_SHAPE;
  const fsc_moe_config& c = ctx->cfg;
  REQUIRE(on <= 0 || router_f64_supported(c.d, c.n_experts, c.top_k), FSC_ERR_CONFIG,
          "fp64 router needs d %% 64 == 0, d <= 8192, E <= 128");
  ctx->router_f64 = on < 0 ? -1 : (on ? 1 : 0);
  return FSC_OK;
}

extern "C" int fsc_set_router_int8(fsc_ctx* ctx, int on) {
  if (!ctx) return FSC_ERR_SHAPE;
  if (!on) {
    ctx->router_i8 = 0;
    return FSC_OK;
  }
  if (on < 0) {
    ctx->router_i8 = -1;
    if (router_i8_ok(ctx)) return router_i8_alloc(ctx);
    return FSC_OK;
  }
  REQUIRE(router_i8_ok(ctx), FSC_ERR_CONFIG, "int8 router needs E <= 128, d %% 128 == 0, k <= 8");
  int rc = router_i8_alloc(ctx);
  if (rc) return rc;
  ctx->router_i8 = 1;
  return FSC_OK;
}

extern "C" int fsc_set_gemm_dynamic(fsc_ctx* ctx, int on) {
  if (!ctx) return FSC_ERR_SHAPE;
  ctx->gemm_dyn = on < 0 ? -1 : (on ? 1 : 0);
  return FSC_OK;
}

extern "C" int fsc_set_fused_unpermute(fsc_ctx* ctx, int on) {
  if (!ctx) return FSC_ERR_SHAPE;
  ctx->fuse_unpermute = on < 0 ? -1 : (on ? 1 : 0);
  return FSC_OK;
}

extern "C" int fsc_set_gemm_gather(fsc_ctx* ctx, int on) {
  if (!ctx) return FSC_ERR_SHAPE;
  ctx->gather_a = on ? 1 : 0;
  return FSC_OK;
}

extern "C" int fsc_set_gemm_ctas(fsc_ctx* ctx, int n) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(n >= 1 && n <= kNumSMs, FSC_ERR_CONFIG, "gemm ctas %d outside [1,148]", n);
  ctx->gemm_ctas = n;
  return FSC_OK;
}

// ---------------------------------------------------------------------------- MoE pieces

int fsc_validate_moe(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in, const void* out) {
  if (!ctx) return FSC_ERR_SHAPE;
  if (ctx->sticky) return ctx->sticky;
  REQUIRE(w && w->gamma && w->w_router && w->w1 && w->w2 && w->w3, FSC_ERR_SHAPE, "null weight pointer");
  REQUIRE(ctx->cfg.shared_ffn == 0 || (w->ws1 && w->ws2 && w->ws3), FSC_ERR_SHAPE, "null shared-expert weight");
  REQUIRE(T >= 0 && T <= ctx->cfg.max_tokens, FSC_ERR_CONFIG, "T=%d outside [0,max_tokens=%d]", T,
          ctx->cfg.max_tokens);
  REQUIRE(T == 0 || (x_in && out), FSC_ERR_SHAPE, "null activation pointer");
  REQUIRE(aligned16(x_in) && aligned16(out) && aligned16(w->w1) && aligned16(w->w2) && aligned16(w->w3) &&
              aligned16(w->gamma) && aligned16(w->w_router),
          FSC_ERR_SHAPE, "pointers must be 16-byte aligned");
  return FSC_OK;
}
static int validate_call(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in, const void* out) {
  return fsc_validate_moe(ctx, w, T, x_in, out);
}

// Forward declarations (shared expert used by the blocking overlap below)
static int moe_shared(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* resid, float* out,
                      const fsc_moe_debug* dbg, cudaStream_t s);

// Steps 3-4 of P:198 (gate + dispatch start), 6 (routed experts) and 7 (combine start).
// async_dispatch: the counts exchange and dispatch run on the comm stream while the
// caller's phase-0 callback (attention part (b)) runs on the compute stream (FarSkip).
// serial: the combine is waited before returning (plain blocking, P:103 bubble (c));
// otherwise it stays in flight on the comm stream (ctx->comb_async) and fsc_moe_wait /
// moe_finish waits for it.
// shared_resid != nullptr (blocking schedule): the shared expert out = shared_resid +
// shared runs here too - at EP = 1 right after the router, beside the permutation maps
// and the permute on the aux stream; at EP > 1 after the combine started (Regular+) or,
// serial, after it landed.
// fused_out != nullptr (blocking, EP = 1): GEMM2's epilogue also performs the
// gate-weighted unpermute, fused_out = fused_resid + routed (bitwise the unpermute kernel).
static int moe_route_and_experts(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in,
                                 const fsc_moe_debug* dbg, cudaStream_t s, fsc_overlap_cb cb, void* user,
                                 bool async_dispatch, bool serial, const float* shared_resid = nullptr,
                                 float* shared_out = nullptr, float* fused_out = nullptr,
                                 const float* fused_resid = nullptr) {
  const fsc_moe_config& c = ctx->cfg;
  const int d = c.d, E = c.n_experts, k = c.top_k;
  const bool spin = ctx->spin != 0;
  ctx->comb_async = 0;
  // ---- gate (P:198 step 3): RMSNorm + router + top-k (+ permutation maps below)
  FUZZ(s);
  PH_BEGIN(PH_ROUTER);
  if (spin) {
    CK(fsc_spin(ctx, SP_GATE, s));
  } else {
    RouterLaunch rl{x_in, w->gamma, w->w_router, T, d, E, k, c.rms_eps, ctx->xn, ctx->topk_idx, ctx->topk_w,
                    dbg ? dbg->logits : nullptr, dbg ? dbg->n_refined : nullptr,
                    ctx->r_part, ctx->r_part_sq, ctx->w_scaled, ctx->w_sq, TB_DEFAULT,
                    ctx->i8_w, ctx->i8_exp, router_tc_on(ctx) ? 1 : 0};
    rl.f64 = router_f64_on(ctx, T, d, E, k) ? 1 : 0;
    rl.f64_w = ctx->f64_w;
    CK(launch_router(rl, s));
  }
  PH_END(PH_ROUTER);
  const bool allreduce = ctx->ep > 1 && ctx->ep_mode == FSC_EP_ALLREDUCE;
  const bool early_shared = shared_out && (ctx->ep == 1 || allreduce) && !spin;
  // EP = 1 FarSkip: the local permutation (maps + permute) stands in for the dispatch and
  // runs on the comm stream, overlapping the caller's attention part (b) (P:198 steps 4-5)
  const bool ep1_async = ctx->ep == 1 && async_dispatch && !early_shared && !ctx->gather_a;
  cudaStream_t ps = early_shared ? ctx->aux : (ep1_async ? ctx->comm : s);   // stream of the permutation work
  if (early_shared || ep1_async) {
    CK(cudaEventRecord(ctx->ev_c, s));
    CK(cudaStreamWaitEvent(ps, ctx->ev_c, 0));
  }
  if (!spin) {
    PermLaunch pl{ctx->topk_idx, T, k, E, ctx->hist, ctx->base, ctx->counts, ctx->offsets, ctx->pos, ctx->src_row};
    PH_BEGIN_ON(PH_PERM, ps);
    CK(launch_perm_maps(pl, ps));
    PH_END_ON(PH_PERM, ps);
  }
  // ---- dispatch (P:97-100, P:198 step 4): permute into the expert-sorted order and,
  // for EP > 1, straight into the owning ranks' receive buffers
  const int R = T * k;
  const uint16_t* recv = ctx->xs;
  long recv_rows = R;
  const int* recv_counts = ctx->counts;
  cudaStream_t cs = async_dispatch ? ctx->comm : s;
  const int* a_idx = nullptr;
  const int* row_base = nullptr;
  bool dispatch_on_comm = false;
  if (spin) {
    if (cs != s) {
      CK(cudaEventRecord(ctx->ev_a, s));
      CK(cudaStreamWaitEvent(cs, ctx->ev_a, 0));
    }
    PH_BEGIN_ON(PH_DISPATCH, cs);
    CK(fsc_spin(ctx, SP_DISPATCH, cs));
    PH_END_ON(PH_DISPATCH, cs);
    if (cs != s) CK(cudaEventRecord(ctx->ev_b, cs));
    dispatch_on_comm = cs != s;
  } else if (allreduce) {
    // replicated tokens, local experts only. Their rows are the contiguous
    // range [offsets[e0], offsets[e0 + E_loc]) of the global expert-sorted order.
    const int e0 = ctx->rank * ctx->e_loc;
    PH_BEGIN_ON(PH_DISPATCH, ps);
    CK(launch_permute_rows(ctx->xn, ctx->src_row, ctx->xs, R, d, ps, ctx->offsets + e0, ctx->e_loc));
    PH_END_ON(PH_DISPATCH, ps);
    recv_counts = ctx->counts + e0;
    row_base = ctx->offsets + e0;
    if (early_shared) {
      CK(cudaEventRecord(ctx->ev_d, ps));
      int rc = moe_shared(ctx, w, T, shared_resid, shared_out, dbg, s);   // replicated shared expert
      if (rc) return rc;
      CK(cudaStreamWaitEvent(s, ctx->ev_d, 0));
    }
  } else if (ctx->ep == 1 && ctx->gather_a) {
    // EP = 1 with fsc_set_gemm_gather(ctx, 1): no dispatch copy; the permutation is
    // fused into GEMM1's operand load, whose producer gathers the expert-sorted rows of
    // xn through src_row (TMA gather4, only the valid rows of each tile). Off by
    // default: measured slower than the explicit permute at prefill AND decode sizes
    // (4 rows per TMA instruction cannot keep the 256-row MMA tile fed).
    recv = ctx->xn;
    recv_rows = T;
    a_idx = ctx->src_row;
    if (early_shared) {
      CK(cudaEventRecord(ctx->ev_d, ps));
      int rc = moe_shared(ctx, w, T, shared_resid, shared_out, dbg, s);   // beside the permutation maps
      if (rc) return rc;
      CK(cudaStreamWaitEvent(s, ctx->ev_d, 0));
    }
  } else if (ctx->ep == 1) {
    // EP = 1: explicit permute into the expert-sorted send buffer (full-bandwidth SM copy)
    if (ep1_async) FUZZ(ps);
    PH_BEGIN_ON(PH_DISPATCH, ps);
    CK(launch_permute_ep1(ctx->xn, ctx->src_row, ctx->pos, ctx->xs, T, k, d, ps));
    PH_END_ON(PH_DISPATCH, ps);
    if (ep1_async) {
      CK(cudaEventRecord(ctx->ev_b, ps));
      dispatch_on_comm = true;
    }
    if (early_shared) {
      CK(cudaEventRecord(ctx->ev_d, ps));
      int rc = moe_shared(ctx, w, T, shared_resid, shared_out, dbg, s);   // beside the permutation
      if (rc) return rc;
      CK(cudaStreamWaitEvent(s, ctx->ev_d, 0));
    }
  } else {
    if (cs != s) {
      CK(cudaEventRecord(ctx->ev_a, s));
      CK(cudaStreamWaitEvent(cs, ctx->ev_a, 0));
      FUZZ(cs);
    }
    PH_BEGIN_ON(PH_DISPATCH, cs);
    int rc = fsc_transport_dispatch(ctx, T, cs);
    if (rc) return rc;
    rc = fsc_transport_dispatch_wait(ctx, cs);
    if (rc) return rc;
    PH_END_ON(PH_DISPATCH, cs);
    if (cs != s) {
      CK(cudaEventRecord(ctx->ev_b, cs));
      dispatch_on_comm = true;
    }
    recv = ctx->xr;
    recv_rows = ctx->recv_rows_cap;
    recv_counts = ctx->recv_counts;
  }
  if (cb) cb(user, 0, s);  // P:198 step 5: attention part (b) while dispatch is in flight
  if (dispatch_on_comm) {  // step 6: sync Dispatch (the compute stream stalls only if late)
    PH_BEGIN(PH_DISPATCH_STALL);
    CK(cudaStreamWaitEvent(s, ctx->ev_b, 0));
    PH_END(PH_DISPATCH_STALL);
  }
  if (dbg && !spin) {
    if (dbg->topk_idx) CK(cudaMemcpyAsync(dbg->topk_idx, ctx->topk_idx, sizeof(int) * T * k, cudaMemcpyDeviceToDevice, s));
    if (dbg->topk_w) CK(cudaMemcpyAsync(dbg->topk_w, ctx->topk_w, sizeof(float) * T * k, cudaMemcpyDeviceToDevice, s));
    if (dbg->counts) CK(cudaMemcpyAsync(dbg->counts, ctx->counts, sizeof(int) * E, cudaMemcpyDeviceToDevice, s));
    if (dbg->pos) CK(cudaMemcpyAsync(dbg->pos, ctx->pos, sizeof(int) * T * k, cudaMemcpyDeviceToDevice, s));
    if (ctx->ep > 1 && !allreduce) {   // the exchanged counts matrix and the receive map (after the dispatch)
      const int *cnt = nullptr, *ret = nullptr;
      fsc_transport_debug(ctx, &cnt, &ret);
      if (dbg->ep_counts)
        CK(cudaMemcpyAsync(dbg->ep_counts, cnt, sizeof(int) * ctx->ep * E, cudaMemcpyDeviceToDevice, s));
      if (dbg->recv_counts)
        CK(cudaMemcpyAsync(dbg->recv_counts, ctx->recv_counts, sizeof(int) * ctx->e_loc, cudaMemcpyDeviceToDevice, s));
      if (dbg->recv_src)
        CK(cudaMemcpyAsync(dbg->recv_src, ret, sizeof(int) * ctx->max_recv, cudaMemcpyDeviceToDevice, s));
    }
  }

  // ---- routed experts (P:198 step 6): GEMM1 + SwiGLU, GEMM2.
  // cta_group auto: M = 256 CTA-pair tiles when the experts get >= 256 rows on average
  // (prefill), single-CTA M = 128 tiles below that (decode: weight streaming, fewer
  // wasted MMA rows; measured 0.88 -> 0.99 of HBM for Scout decode GEMM1).
  const bool fused_combine = ctx->ep > 1 && !allreduce && ctx->combine_mode == FSC_COMBINE_FUSED &&
                             !ctx->a2a_zero_bytes;
  FUZZ(s);
  if (spin) {
    PH_BEGIN(PH_GEMM1);
    CK(fsc_spin(ctx, SP_ROUTED, s));
    PH_END(PH_GEMM1);
  } else {
    const long avg_rows = (long)T * k * (allreduce ? 1 : ctx->ep) / E;
    const int routed_cg = ctx->gemm_cg ? ctx->gemm_cg : (avg_rows < 256 ? 1 : 2);
    // decode (single-CTA tiles, weight streaming): pick the tile width with the smaller
    // last-wave waste from the expected tile count (MMA width is not the bound there)
    auto pick_bn = [&](int N, bool swiglu) {
      if (routed_cg != 1 || ctx->gemm_cg) return 0;
      const long mt = ctx->e_loc * ((avg_rows + 127) / 128), slots = ctx->gemm_ctas;
      auto cost = [&](int b) { const long nt = swiglu ? N / (b / 2) : N / b; return ((mt * nt + slots - 1) / slots) * b; };
      return cost(128) * 100 < cost(256) * 95 ? 128 : 0;
    };
    GemmLaunch g1{};
    g1.A = recv; g1.a_rows = recv_rows; g1.B0 = w->w1; g1.B1 = w->w2; g1.b_rows = (long)ctx->e_loc * c.ffn;
    g1.b_group_rows = c.ffn; g1.K = d; g1.N = c.ffn; g1.G = ctx->e_loc; g1.counts = recv_counts; g1.m_total = 0;
    g1.out = ctx->h; g1.ldo = c.ffn; g1.epi = EPI_SWIGLU; g1.num_ctas = ctx->gemm_ctas; g1.cta_group = routed_cg;
    g1.a_idx = a_idx;
    g1.row_base = row_base;
    g1.bn = pick_bn(c.ffn, true);
    g1.sched = gemm_sched_slot(ctx, SCHED_ROUTED1);
    PH_BEGIN(PH_GEMM1);
    CK(launch_grouped_gemm(g1, s));
    PH_END(PH_GEMM1);
    GemmLaunch g2{};
    g2.A = ctx->h; g2.a_rows = a_idx ? (long)R : recv_rows; g2.B0 = w->w3; g2.B1 = nullptr; g2.b_rows = (long)ctx->e_loc * d;
    g2.b_group_rows = d; g2.K = c.ffn; g2.N = d; g2.G = ctx->e_loc; g2.counts = recv_counts; g2.m_total = 0;
    g2.out = ctx->y; g2.ldo = d; g2.epi = EPI_BF16; g2.num_ctas = ctx->gemm_ctas; g2.cta_group = routed_cg;
    g2.row_base = row_base;
    g2.bn = pick_bn(d, false);
    g2.sched = gemm_sched_slot(ctx, SCHED_ROUTED2);
    if (fused_combine) fsc_transport_scatter_target(ctx, &g2.ret, g2.peer_out);  // P:100 Combine, fused
    if (fused_out && ctx->ep == 1) {   // P:100 "sum the routed experts", fused into the down GEMM
      g2.comb_out = fused_out; g2.comb_resid = fused_resid; g2.src_row = ctx->src_row; g2.pos = ctx->pos;
      g2.topk_w = ctx->topk_w; g2.comb_cnt = ctx->comb_cnt; g2.top_k = k;
    }
    PH_BEGIN(PH_GEMM2);
    CK(launch_grouped_gemm(g2, s));
    PH_END(PH_GEMM2);
  }
  // ---- combine (P:100, P:198 step 7)
  if (allreduce && !spin) {
    // local partial of the routed sum (fp32, slot order) into the peer-visible buffer,
    // then the all-reduce on the comm stream (FarSkip) or in line (blocking)
    const int e0 = ctx->rank * ctx->e_loc;
    PH_BEGIN(PH_UNPERMUTE);
    CK(launch_unpermute_local(ctx->y, ctx->pos, ctx->topk_w, ctx->topk_idx, e0, e0 + ctx->e_loc,
                              fsc_transport_ar_partial(ctx), T, k, d, s));
    PH_END(PH_UNPERMUTE);
    if (async_dispatch) {
      CK(cudaEventRecord(ctx->ev_a, s));
      CK(cudaStreamWaitEvent(cs, ctx->ev_a, 0));
    }
    PH_BEGIN_ON(PH_COMBINE, cs);
    int rc = fsc_transport_ar_start(ctx, T, cs);
    if (rc) return rc;
    PH_END_ON(PH_COMBINE, cs);
    if (async_dispatch) CK(cudaEventRecord(ctx->ev_b, cs));
  } else if (fused_combine && !spin) {
    PH_BEGIN(PH_COMBINE);
    int rc = fsc_transport_combine(ctx, T, s);  // rows already stored by GEMM2: raise the flags
    if (rc) return rc;
    PH_END(PH_COMBINE);
    if (serial) {
      PH_BEGIN(PH_COMBINE_WAIT);
      rc = fsc_transport_combine_wait(ctx, s);
      if (rc) return rc;
      PH_END(PH_COMBINE_WAIT);
    }
  } else if (ctx->ep > 1 || spin) {
    // decoupled combine on the comm stream: overlaps the shared expert (step 8) and,
    // in the FarSkip stack, the next layer's attention part (a)
    CK(cudaEventRecord(ctx->ev_g2, s));
    CK(cudaStreamWaitEvent(ctx->comm, ctx->ev_g2, 0));
    FUZZ(ctx->comm);
    PH_BEGIN_ON(PH_COMBINE, ctx->comm);
    if (spin) {
      CK(fsc_spin(ctx, SP_COMBINE, ctx->comm));
    } else {
      int rc = fsc_transport_combine_push(ctx, ctx->y, ctx->comm);
      if (rc) return rc;
    }
    PH_END_ON(PH_COMBINE, ctx->comm);
    CK(cudaEventRecord(ctx->ev_comb, ctx->comm));
    ctx->comb_async = 1;
    if (serial) {   // plain blocking: the compute stream waits for the combine (P:103 bubble (c))
      PH_BEGIN(PH_COMBINE_WAIT);
      CK(cudaStreamWaitEvent(s, ctx->ev_comb, 0));
      if (ctx->ep > 1 && !spin) {
        int rc = fsc_transport_combine_wait(ctx, s);
        if (rc) return rc;
      }
      PH_END(PH_COMBINE_WAIT);
    }
  }
  if (shared_out && !early_shared) {
    int rc = moe_shared(ctx, w, T, shared_resid, shared_out, dbg, s);
    if (rc) return rc;
  }
  return FSC_OK;
}

// Shared expert (P:100-101, P:198 step 8): out = resid + SwiGLU_shared(xn).
static int moe_shared(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* resid, float* out,
                      const fsc_moe_debug* dbg, cudaStream_t s) {
  const fsc_moe_config& c = ctx->cfg;
  const int d = c.d;
  FUZZ(s);
  if (ctx->spin) {
    PH_BEGIN(PH_SHARED1);
    CK(fsc_spin(ctx, SP_SHARED, s));
    PH_END(PH_SHARED1);
    return FSC_OK;
  }
  if (c.shared_ffn == 0) {
    if (dbg && dbg->shared_out) CK(cudaMemsetAsync(dbg->shared_out, 0, sizeof(float) * T * (long)d, s));
    if (resid != out) {   // (never on the blocking / FarSkip paths: they pass resid == out or skip the call)
      PH_BEGIN(PH_SHARED2);
      CK(launch_copy_f32(resid, out, (long)T * d, s));
      PH_END(PH_SHARED2);
    }
    return FSC_OK;
  }
  GemmLaunch g1{};
  g1.A = ctx->xn; g1.a_rows = T; g1.B0 = w->ws1; g1.B1 = w->ws2; g1.b_rows = c.shared_ffn; g1.b_group_rows = c.shared_ffn;
  g1.K = d; g1.N = c.shared_ffn; g1.G = 1; g1.counts = nullptr; g1.m_total = T; g1.out = ctx->hs; g1.ldo = c.shared_ffn;
  g1.epi = EPI_SWIGLU; g1.num_ctas = ctx->gemm_ctas; g1.cta_group = ctx->gemm_cg ? ctx->gemm_cg : 2;
  g1.sched = gemm_sched_slot(ctx, SCHED_SHARED1);
  PH_BEGIN(PH_SHARED1);
  CK(launch_grouped_gemm(g1, s));
  PH_END(PH_SHARED1);
  GemmLaunch g2{};
  g2.A = ctx->hs; g2.a_rows = T; g2.B0 = w->ws3; g2.B1 = nullptr; g2.b_rows = d; g2.b_group_rows = d;
  g2.K = c.shared_ffn; g2.N = d; g2.G = 1; g2.counts = nullptr; g2.m_total = T; g2.out = out; g2.ldo = d;
  g2.resid = resid; g2.ldr = d; g2.epi = EPI_RESID_F32; g2.num_ctas = ctx->gemm_ctas; g2.cta_group = ctx->gemm_cg ? ctx->gemm_cg : 2;
  g2.sched = gemm_sched_slot(ctx, SCHED_SHARED2);
  PH_BEGIN(PH_SHARED2);
  CK(launch_grouped_gemm(g2, s));
  PH_END(PH_SHARED2);
  if (dbg && dbg->shared_out) {
    g2.out = dbg->shared_out; g2.resid = nullptr;
    CK(launch_grouped_gemm(g2, s));
  }
  return FSC_OK;
}

// Gate-weighted unpermute (+ far-skip residual add), after the combine landed.
static int moe_finish(fsc_ctx* ctx, int T, const float* resid, float* out, const fsc_moe_debug* dbg, cudaStream_t s,
                      bool fused = false) {
  const fsc_moe_config& c = ctx->cfg;
  const uint16_t* ysrc = ctx->y;
  if (ctx->ep > 1 && ctx->ep_mode == FSC_EP_ALLREDUCE) {   // out = resid + all-reduced routed sum
    PH_BEGIN(PH_COMBINE_WAIT);
    CK(cudaStreamWaitEvent(s, ctx->ev_b, 0));
    int rc = fsc_transport_ar_finish(ctx, T, resid, out, s);
    if (rc) return rc;
    PH_END(PH_COMBINE_WAIT);
    if (dbg && dbg->routed_out) {
      rc = fsc_transport_ar_finish(ctx, T, nullptr, dbg->routed_out, s);
      if (rc) return rc;
    }
    return FSC_OK;
  }
  if (ctx->ep > 1 || ctx->comb_async) {
    PH_BEGIN(PH_COMBINE_WAIT);
    if (ctx->comb_async) CK(cudaStreamWaitEvent(s, ctx->ev_comb, 0));   // my own push is done (buffer reuse)
    if (ctx->ep > 1 && !ctx->spin) {
      int rc = fsc_transport_combine_wait(ctx, s);                        // every source's rows landed
      if (rc) return rc;
    }
    PH_END(PH_COMBINE_WAIT);
    ctx->comb_async = 0;
    ysrc = ctx->ys;
  }
  if (ctx->spin) return FSC_OK;
  if (!fused) {   // (fused: done by GEMM2's epilogue)
    PH_BEGIN(PH_UNPERMUTE);
    CK(launch_unpermute(ysrc, ctx->pos, ctx->topk_w, resid, out, T, c.top_k, c.d, s));
    PH_END(PH_UNPERMUTE);
  }
  if (dbg && dbg->routed_out)
    CK(launch_unpermute(ysrc, ctx->pos, ctx->topk_w, nullptr, dbg->routed_out, T, c.top_k, c.d, s));
  return FSC_OK;
}

// ---------------------------------------------------------------------------- MoE entry points

static int moe_blocking_impl(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in, float* out,
                             const fsc_moe_debug* dbg, void* stream);

extern "C" int fsc_moe_forward_blocking(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in, float* out,
                                        const fsc_moe_debug* dbg, void* stream) {
  int rc = moe_blocking_impl(ctx, w, T, x_in, out, dbg, stream);
  if (rc) return rc;
  return fsc_check_finite(ctx, out, (long)T * ctx->cfg.d, static_cast<cudaStream_t>(stream), "fsc_moe_forward_blocking");
}

static int moe_blocking_impl(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in, float* out,
                             const fsc_moe_debug* dbg, void* stream) {
  int rc = validate_call(ctx, w, T, x_in, out);
  if (rc) return rc;
  REQUIRE(!ctx->pending, FSC_ERR_STATE, "a FarSkip handle is outstanding");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (T == 0 && ctx->ep == 1) return FSC_OK;
  memset(ctx->ph_used, 0, sizeof(ctx->ph_used));
  // Regular order (C-amb-12): tmp = x_in + shared; out = tmp + routed. The shared
  // expert overlaps the permutation (EP = 1) or follows the routed experts (EP > 1).
  // fused unpermute: auto (-1) = top-1 routing only (measured: at k = 6 / 8 the per-tile
  // counter + cooperative finish costs the down GEMM more than the separate kernel)
  const int fu = ctx->fuse_unpermute < 0 ? (ctx->cfg.top_k == 1) : ctx->fuse_unpermute;
  const bool fuse = ctx->ep == 1 && fu && ctx->cfg.top_k <= 8 && !ctx->spin;   // (the epilogue holds <= 8 slots)
  // FSC_BLOCKING_SERIAL: the combine is waited before the shared expert (P:103 bubbles
  // (b) and (c)); FSC_BLOCKING_REGULAR_PLUS: the shared expert runs while it is in flight
  const bool serial = ctx->blocking_mode == FSC_BLOCKING_SERIAL;
  if (ctx->cfg.shared_ffn == 0) {   // no shared expert: out = x_in + routed, straight from x_in
    rc = moe_route_and_experts(ctx, w, T, x_in, dbg, s, nullptr, nullptr, false, serial, nullptr, nullptr,
                               fuse ? out : nullptr, x_in);
    if (rc) return rc;
    rc = moe_shared(ctx, w, T, x_in, const_cast<float*>(x_in), dbg, s);   // debug shared_out = 0 only
    if (rc) return rc;
    return moe_finish(ctx, T, x_in, out, dbg, s, fuse);
  }
  rc = moe_route_and_experts(ctx, w, T, x_in, dbg, s, nullptr, nullptr, false, serial, x_in, ctx->tmp,
                             fuse ? out : nullptr, ctx->tmp);
  if (rc) return rc;
  return moe_finish(ctx, T, ctx->tmp, out, dbg, s, fuse);
}

extern "C" int fsc_moe_forward_blocking_host(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in_host,
                                             float* out_host, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(T == 0 || (x_in_host && out_host), FSC_ERR_SHAPE, "null host buffer");
  REQUIRE(T >= 0 && T <= ctx->cfg.max_tokens, FSC_ERR_CONFIG, "T=%d outside [0,max_tokens]", T);
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t bytes = sizeof(float) * (size_t)T * ctx->cfg.d;
  CK(cudaMemcpyAsync(ctx->io_in, x_in_host, bytes, cudaMemcpyHostToDevice, s));
  int rc = fsc_moe_forward_blocking(ctx, w, T, ctx->io_in, ctx->io_out, nullptr, stream);
  if (rc) return rc;
  CK(cudaMemcpyAsync(out_host, ctx->io_out, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return FSC_OK;
}

// Pipelined host entry: step i's H2D copy (copy stream), MoE forward (caller's
// stream) and D2H copy (second copy stream) are ordered by events on two device
// staging slots, so consecutive calls overlap step i+1's upload and step i-1's
// download with step i's compute. Returns without waiting; fsc_host_flush waits.
extern "C" int fsc_moe_forward_host_async(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in_host,
                                          float* out_host, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(T == 0 || (x_in_host && out_host), FSC_ERR_SHAPE, "null host buffer");
  REQUIRE(T >= 0 && T <= ctx->cfg.max_tokens, FSC_ERR_CONFIG, "T=%d outside [0,max_tokens]", T);
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long n = (long)ctx->cfg.max_tokens * ctx->cfg.d;
  if (!ctx->h2d) {
    CK(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
    for (int i = 0; i < fsc_ctx::kIoSlots; ++i) {
      CK(cudaMalloc(&ctx->io_slot_in[i], sizeof(float) * n));
      CK(cudaMalloc(&ctx->io_slot_out[i], sizeof(float) * n));
      CK(cudaEventCreateWithFlags(&ctx->ev_in[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_cdone[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_out[i], cudaEventDisableTiming));
      CK(cudaEventRecord(ctx->ev_cdone[i], s));
      CK(cudaEventRecord(ctx->ev_out[i], s));
    }
  }
  const int slot = ctx->io_slot;
  ctx->io_slot = (ctx->io_slot + 1) % fsc_ctx::kIoSlots;
  // the slot's previous call (three calls ago) must have finished its D2H into the caller's
  // out_host before this call returns, so that "three calls later" the host buffers are free
  CK(cudaEventSynchronize(ctx->ev_out[slot]));
  const size_t bytes = sizeof(float) * (size_t)T * ctx->cfg.d;
  CK(cudaStreamWaitEvent(ctx->h2d, ctx->ev_cdone[slot], 0));      // slot's previous compute read its input
  CK(cudaMemcpyAsync(ctx->io_slot_in[slot], x_in_host, bytes, cudaMemcpyHostToDevice, ctx->h2d));
  CK(cudaEventRecord(ctx->ev_in[slot], ctx->h2d));
  CK(cudaStreamWaitEvent(s, ctx->ev_in[slot], 0));
  CK(cudaStreamWaitEvent(s, ctx->ev_out[slot], 0));               // slot's previous download finished
  int rc = fsc_moe_forward_blocking(ctx, w, T, ctx->io_slot_in[slot], ctx->io_slot_out[slot], nullptr, stream);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev_cdone[slot], s));
  CK(cudaStreamWaitEvent(ctx->d2h, ctx->ev_cdone[slot], 0));
  CK(cudaMemcpyAsync(out_host, ctx->io_slot_out[slot], bytes, cudaMemcpyDeviceToHost, ctx->d2h));
  CK(cudaEventRecord(ctx->ev_out[slot], ctx->d2h));
  return FSC_OK;
}

extern "C" int fsc_host_flush(fsc_ctx* ctx) {
  if (!ctx) return FSC_ERR_SHAPE;
  CK(cudaSetDevice(ctx->device));
  if (ctx->d2h) CK(cudaStreamSynchronize(ctx->d2h));
  return FSC_OK;
}

extern "C" int fsc_moe_forward_farskip(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in,
                                       float* partial_inout, fsc_overlap_cb cb, void* user, fsc_handle* h,
                                       const fsc_moe_debug* dbg, void* stream) {
  int rc = validate_call(ctx, w, T, x_in, partial_inout);
  if (rc) return rc;
  REQUIRE(h, FSC_ERR_SHAPE, "null handle pointer");
  REQUIRE(!ctx->pending, FSC_ERR_STATE, "FarSkip pipeline depth is 1: wait the outstanding handle first");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  memset(ctx->ph_used, 0, sizeof(ctx->ph_used));
  // no_overlap (set by the stack): 1 = BLOCKING schedule (dispatch in line, combine waited
  // before the shared expert); 2 = Regular layer of an OVERLAPPED stack (dispatch in line,
  // shared expert beside the in-flight combine: Regular+); 0 = FarSkip
  rc = moe_route_and_experts(ctx, w, T, x_in, dbg, s, cb, user, ctx->no_overlap == 0, ctx->no_overlap == 1);
  if (rc) return rc;
  if (cb) cb(user, 1, s);  // combine in flight
  // P:198 step 8 and C-amb-12: attn-in_{k+1} = (mlp-in_k + attn-out_k) + shared-out_k
  rc = moe_shared(ctx, w, T, partial_inout, partial_inout, dbg, s);
  if (rc) return rc;
  ctx->handle.ctx = ctx;
  ctx->handle.T = T;
  ctx->handle.live = 1;
  ctx->handle.dbg_routed = dbg ? dbg->routed_out : nullptr;
  ctx->pending = 1;
  *h = &ctx->handle;
  return FSC_OK;
}

extern "C" int fsc_moe_wait(fsc_ctx* ctx, fsc_handle h, const float* partial_in, float* full_out, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(h && h == &ctx->handle, FSC_ERR_STATE, "unknown handle");
  REQUIRE(h->live && ctx->pending, FSC_ERR_STATE, "handle already waited");
  REQUIRE(h->T == 0 || (partial_in && full_out), FSC_ERR_SHAPE, "null activation pointer");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  h->live = 0;
  ctx->pending = 0;
  fsc_moe_debug dbg{};
  dbg.routed_out = h->dbg_routed;
  int rc = moe_finish(ctx, h->T, partial_in, full_out, dbg.routed_out ? &dbg : nullptr, s);
  if (rc) return rc;
  return fsc_check_finite(ctx, full_out, (long)h->T * ctx->cfg.d, s, "fsc_moe_wait");
}

// ---------------------------------------------------------------------------- op-level entry points

extern "C" int fsc_op_router(fsc_ctx* ctx, const float* x, const float* gamma, const float* w_router, int T, int d,
                             int E, int k, void* xn, int* topk_idx, float* topk_w, float* logits, int* n_refined,
                             void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(d % 64 == 0 && d <= 8192 && E >= 1 && E <= 128 && k >= 1 && k <= E, FSC_ERR_CONFIG, "bad router shape");
  REQUIRE(T >= 0 && T <= ctx->cfg.max_tokens && E <= ctx->cfg.n_experts && d <= ctx->cfg.d, FSC_ERR_CONFIG,
          "router shape beyond the context workspace");
  RouterLaunch rl{x, gamma, w_router, T, d, E, k, ctx->cfg.rms_eps, static_cast<uint16_t*>(xn), topk_idx, topk_w,
                  logits, n_refined, ctx->r_part, ctx->r_part_sq, ctx->w_scaled, ctx->w_sq, TB_DEFAULT,
                  ctx->i8_w, ctx->i8_exp, (router_tc_on(ctx) && d == ctx->cfg.d && E <= 128) ? 1 : 0};
  rl.f64 = router_f64_on(ctx, T, d, E, k) ? 1 : 0;
  rl.f64_w = ctx->f64_w;
  CK(launch_router(rl, static_cast<cudaStream_t>(stream)));
  return FSC_OK;
}

extern "C" int fsc_op_perm_maps(fsc_ctx* ctx, const int* topk_idx, int T, int k, int E, int* counts, int* offsets,
                                int* pos, int* src_row, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(T <= ctx->cfg.max_tokens && E <= ctx->cfg.n_experts, FSC_ERR_CONFIG, "perm maps beyond workspace");
  PermLaunch pl{topk_idx, T, k, E, ctx->hist, ctx->base, counts, offsets, pos, src_row};
  CK(launch_perm_maps(pl, static_cast<cudaStream_t>(stream)));
  return FSC_OK;
}

extern "C" int fsc_op_permute(fsc_ctx* ctx, const void* xn, const int* src_row, void* xs, int R, int d, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(d % 8 == 0, FSC_ERR_CONFIG, "d %% 8");
  CK(launch_permute_rows(static_cast<const uint16_t*>(xn), src_row, static_cast<uint16_t*>(xs), R, d,
                         static_cast<cudaStream_t>(stream)));
  return FSC_OK;
}

extern "C" int fsc_op_grouped_gemm_gather(fsc_ctx* ctx, int epi, const void* A, long a_rows, const int* a_idx,
                                          const void* B0, const void* B1, int G, const int* counts, int m_total, int N,
                                          int K, void* out, const float* resid, void* stream);

extern "C" int fsc_op_grouped_gemm(fsc_ctx* ctx, int epi, const void* A, long a_rows, const void* B0, const void* B1,
                                   int G, const int* counts, int m_total, int N, int K, void* out, const float* resid,
                                   void* stream) {
  return fsc_op_grouped_gemm_gather(ctx, epi, A, a_rows, nullptr, B0, B1, G, counts, m_total, N, K, out, resid,
                                    stream);
}

extern "C" int fsc_op_grouped_gemm_gather(fsc_ctx* ctx, int epi, const void* A, long a_rows, const int* a_idx,
                                          const void* B0, const void* B1, int G, const int* counts, int m_total, int N,
                                          int K, void* out, const float* resid, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(epi >= 0 && epi <= 2, FSC_ERR_CONFIG, "epi");
  REQUIRE(K % 64 == 0 && K > 0 && gemm_pick_bn(epi, N) > 0, FSC_ERR_CONFIG, "GEMM needs K%%64==0 and N%%64==0");
  REQUIRE(G >= 1 && G <= 256, FSC_ERR_CONFIG, "G outside [1,256]");
  REQUIRE(epi != 1 || B1, FSC_ERR_SHAPE, "SwiGLU needs B1");
  GemmLaunch L{};
  L.A = A; L.a_rows = a_rows; L.B0 = B0; L.B1 = B1; L.b_rows = (long)G * N; L.b_group_rows = N; L.K = K; L.N = N;
  L.G = G; L.counts = counts; L.m_total = m_total; L.out = out; L.ldo = N; L.resid = resid; L.ldr = N; L.epi = epi;
  L.num_ctas = ctx->gemm_ctas;
  L.cta_group = ctx->gemm_cg ? ctx->gemm_cg : 2;
  L.a_idx = a_idx;
  L.sched = gemm_sched_slot(ctx, SCHED_OP);
  CK(launch_grouped_gemm(L, static_cast<cudaStream_t>(stream)));
  return FSC_OK;
}

extern "C" int fsc_op_attention(fsc_ctx* ctx, const void* qkv, void* out, int T, int Hq, int Hkv, int hd, int seq_len,
                                void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(T >= 0 && Hkv >= 1 && Hq % Hkv == 0 && seq_len >= 1, FSC_ERR_CONFIG, "bad attention shape");
  REQUIRE(hd == 16 || hd == 32 || hd == 64 || hd == 128, FSC_ERR_CONFIG, "head_dim must be 16/32/64/128");
  REQUIRE(T == 0 || (qkv && out), FSC_ERR_SHAPE, "null attention buffer");
  CK(cudaSetDevice(ctx->device));
  CK(launch_flash_attn(static_cast<const uint16_t*>(qkv), static_cast<uint16_t*>(out), T, Hq, Hkv, hd, seq_len,
                       static_cast<cudaStream_t>(stream)));
  return FSC_OK;
}

extern "C" int fsc_op_unpermute(fsc_ctx* ctx, const void* y, const int* pos, const float* w, const float* resid,
                                float* out, int T, int k, int d, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  REQUIRE(d % 8 == 0, FSC_ERR_CONFIG, "d %% 8");
  CK(launch_unpermute(static_cast<const uint16_t*>(y), pos, w, resid, out, T, k, d, static_cast<cudaStream_t>(stream)));
  return FSC_OK;
}
