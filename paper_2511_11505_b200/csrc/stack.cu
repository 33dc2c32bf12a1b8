// fsc_layer_stack_forward: an L-layer (attention + MoE) stack with per-layer
// Regular (Eq. 6) or Hybrid FarSkip wiring,
// run in the BLOCKING or the OVERLAPPED schedule.
//
// Wiring (fp32 residual stream, summation order C-amb-12):
//   Regular k : A_k = o_{k-1};  M_k = A_k + attn_out_k;  o_k = (M_k + shared_k) + routed_k
//   Hybrid  k : A_k = (M_{k-1} + attn_out_{k-1}) + shared_{k-1}   (A_0 = o_0)
//               M_k = o_{k-1} = A_k + routed_{k-1}                 (M_0 = o_0)
//               o_k = ((M_k + attn_out_k) + shared_k) + routed_k
// Every layer's MoE runs through the FarSkip entry point: its partial sum
// (everything but routed_k) is available at once and routed_k stays pending in a
// handle until a consumer needs o_k. A Hybrid layer's attention only needs the
// partial, so layer k+1's attention overlaps layer k's combine, and the
// dispatch overlaps the attention core (OVERLAPPED schedule, P:198 steps 1-8).
// BLOCKING runs the same kernels with every collective waited on at once.
// In the all-reduce inference variant (FSC_EP_ALLREDUCE) the attention is
// tensor-parallel: each rank passes its head slice, the o-projection partials are
// all-reduced on channel 1 and, in Hybrid layers, waited only before the next
// attention (A_{k+1} = (M_k + shared_k) + attn_out_k in that variant).
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <utility>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

using namespace fsc;

#define SCK(call)                                                                                  \
  do {                                                                                             \
    cudaError_t e__ = (call);                                                                      \
    if (e__ != cudaSuccess) {                                                                      \
      fsc_set_error(ctx, "stack %s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e__)); \
      ctx->sticky = FSC_ERR_CUDA;                                                                  \
      return FSC_ERR_CUDA;                                                                         \
    }                                                                                              \
  } while (0)
#define SREQ(cond, code, ...)          \
  do {                                 \
    if (!(cond)) {                     \
      fsc_set_error(ctx, __VA_ARGS__); \
      return code;                     \
    }                                  \
  } while (0)
#define SRC(expr)          \
  do {                     \
    int r__ = (expr);      \
    if (r__) return r__;   \
  } while (0)

namespace {

struct AttnCall {
  fsc_ctx* ctx;
  const fsc_attn_weights* aw;
  int T, seq_len;
  const float* resid;   // residual the o-proj adds to
  float* out;           // fp32 [T,d] = resid + attn_out
  float* cache_attn_out;
  int rc;
};

int ensure_workspace(fsc_ctx* ctx, const fsc_attn_weights* aw, int L) {
  const long T = ctx->cfg.max_tokens, d = ctx->cfg.d;
  long need_qkv = 0, need_ao = 0;
  for (int k = 0; k < L; ++k) {
    need_qkv = std::max(need_qkv, (long)(aw[k].n_heads + 2 * aw[k].n_kv_heads) * aw[k].head_dim);
    need_ao = std::max(need_ao, (long)aw[k].n_heads * aw[k].head_dim);
  }
  if (!ctx->hn) {
    SCK(cudaMalloc(&ctx->hn, sizeof(uint16_t) * T * d));
    for (int i = 0; i < 3; ++i) SCK(cudaMalloc(&ctx->rbuf[i], sizeof(float) * T * d));
  }
  if (need_qkv > ctx->stack_cap_qkv) {
    if (ctx->qkv) cudaFree(ctx->qkv);
    SCK(cudaMalloc(&ctx->qkv, sizeof(uint16_t) * T * need_qkv));
    ctx->stack_cap_qkv = need_qkv;
  }
  if (need_ao > ctx->stack_cap_ao) {
    if (ctx->ao) cudaFree(ctx->ao);
    SCK(cudaMalloc(&ctx->ao, sizeof(uint16_t) * T * need_ao));
    ctx->stack_cap_ao = need_ao;
  }
  return FSC_OK;
}

// Attention part (a) of P:198: RMSNorm + QKV projection + RoPE.
int attention_a(fsc_ctx* ctx, const fsc_attn_weights* aw, int T, int seq_len, const float* attn_in, cudaStream_t s) {
  const int d = ctx->cfg.d, Hq = aw->n_heads, Hkv = aw->n_kv_heads, hd = aw->head_dim;
  const int nqkv = (Hq + 2 * Hkv) * hd;
  SCK(fsc_fuzz(ctx, s));
  SCK(fsc_phase_begin(ctx, PH_ATTN_A, s));
  if (ctx->spin) {
    SCK(fsc_spin(ctx, SP_QKV, s));
    SCK(fsc_phase_end(ctx, PH_ATTN_A, s));
    return FSC_OK;
  }
  SCK(launch_rmsnorm_bf16(attn_in, aw->gamma, ctx->hn, T, d, ctx->cfg.rms_eps, s));
  GemmLaunch g{};
  g.A = ctx->hn; g.a_rows = T; g.B0 = aw->w_qkv; g.b_rows = nqkv; g.b_group_rows = nqkv; g.K = d; g.N = nqkv;
  g.G = 1; g.m_total = T; g.out = ctx->qkv; g.ldo = nqkv; g.epi = EPI_BF16; g.num_ctas = ctx->gemm_ctas;
  g.cta_group = ctx->gemm_cg ? ctx->gemm_cg : 2;
  SCK(launch_grouped_gemm(g, s));
  SCK(launch_rope(ctx->qkv, T, Hq, Hkv, hd, seq_len, aw->rope_theta, s));
  SCK(fsc_phase_end(ctx, PH_ATTN_A, s));
  return FSC_OK;
}

bool tp_mode(const fsc_ctx* ctx) { return ctx->ep > 1 && ctx->ep_mode == FSC_EP_ALLREDUCE; }

// Attention part (b): core attention + output projection into the residual.
// TP (all-reduce inference variant): this rank holds a slice of the heads; its
// o-projection partial goes to all-reduce channel 1, launched at once (comm stream
// when overlapped); out = resid now and attn_finish adds the reduced attn_out later.
int attention_b(fsc_ctx* ctx, const fsc_attn_weights* aw, int T, int seq_len, const float* resid, float* out,
                float* cache_attn_out, cudaStream_t s) {
  const int d = ctx->cfg.d, Hq = aw->n_heads, Hkv = aw->n_kv_heads, hd = aw->head_dim;
  SCK(fsc_fuzz(ctx, s));
  SCK(fsc_phase_begin(ctx, PH_ATTN_B, s));
  if (ctx->spin) {   // wiring test: out = resid only
    SCK(fsc_spin(ctx, SP_CORE, s));
    SCK(fsc_phase_end(ctx, PH_ATTN_B, s));
    return FSC_OK;
  }
  SCK(launch_flash_attn(ctx->qkv, ctx->ao, T, Hq, Hkv, hd, seq_len, s));
  if (tp_mode(ctx)) {
    GemmLaunch g{};
    g.A = ctx->ao; g.a_rows = T; g.B0 = aw->w_o; g.b_rows = d; g.b_group_rows = d; g.K = Hq * hd; g.N = d;
    g.G = 1; g.m_total = T; g.out = fsc_transport_ar_partial(ctx, 1); g.ldo = d; g.resid = nullptr; g.ldr = d;
    g.epi = EPI_RESID_F32; g.num_ctas = ctx->gemm_ctas; g.cta_group = ctx->gemm_cg ? ctx->gemm_cg : 2;
    SCK(launch_grouped_gemm(g, s));
    if (out != resid) SCK(cudaMemcpyAsync(out, resid, sizeof(float) * (long)T * d, cudaMemcpyDeviceToDevice, s));
    cudaStream_t cs = ctx->no_overlap ? s : ctx->comm;
    if (cs != s) {
      SCK(cudaEventRecord(ctx->ev_t1, s));
      SCK(cudaStreamWaitEvent(cs, ctx->ev_t1, 0));
    }
    SRC(fsc_transport_ar_start(ctx, T, cs, 1));
    if (cs != s) SCK(cudaEventRecord(ctx->ev_t2, cs));
    ctx->attn_pending = cs != s ? 2 : 1;
    ctx->attn_cache = cache_attn_out;
    ctx->attn_T = T;
    SCK(fsc_phase_end(ctx, PH_ATTN_B, s));
    return FSC_OK;
  }
  GemmLaunch g{};
  g.A = ctx->ao; g.a_rows = T; g.B0 = aw->w_o; g.b_rows = d; g.b_group_rows = d; g.K = Hq * hd; g.N = d;
  g.G = 1; g.m_total = T; g.out = out; g.ldo = d; g.resid = resid; g.ldr = d; g.epi = EPI_RESID_F32;
  g.num_ctas = ctx->gemm_ctas; g.cta_group = ctx->gemm_cg ? ctx->gemm_cg : 2;
  SCK(launch_grouped_gemm(g, s));
  SCK(fsc_phase_end(ctx, PH_ATTN_B, s));
  if (cache_attn_out) {
    g.out = cache_attn_out;
    g.resid = nullptr;
    SCK(launch_grouped_gemm(g, s));
  }
  return FSC_OK;
}

// TP: buf += reduced attn_out (waits the all-reduce of the last attention_b).
int attn_finish(fsc_ctx* ctx, float* buf, cudaStream_t s) {
  if (!ctx->attn_pending) return FSC_OK;
  if (ctx->attn_pending == 2) SCK(cudaStreamWaitEvent(s, ctx->ev_t2, 0));
  SRC(fsc_transport_ar_finish(ctx, ctx->attn_T, buf, buf, s, 1));
  if (ctx->attn_cache) SRC(fsc_transport_ar_finish(ctx, ctx->attn_T, nullptr, ctx->attn_cache, s, 1));
  ctx->attn_pending = 0;
  ctx->attn_cache = nullptr;
  return FSC_OK;
}

void attn_b_callback(void* user, int phase, void* stream) {
  AttnCall* a = static_cast<AttnCall*>(user);
  if (phase != 0 || a->rc) return;
  a->rc = attention_b(a->ctx, a->aw, a->T, a->seq_len, a->resid, a->out, a->cache_attn_out,
                      static_cast<cudaStream_t>(stream));
}

int copy_f32(fsc_ctx* ctx, float* dst, const float* src, long n, cudaStream_t s) {
  if (dst && src && dst != src) SCK(cudaMemcpyAsync(dst, src, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
  return FSC_OK;
}

}  // namespace

static int stack_body(fsc_ctx* ctx, const fsc_attn_weights* attn, const fsc_moe_weights* moe, int L, int T,
                      int seq_len, const int* modes, int schedule, const float* o0, float* oL,
                      const fsc_act_cache* cache, cudaStream_t s, fsc_handle* h_out);

// Everything is validated before the first enqueue (fsc.h contract). If an enqueue
// fails half way (a CUDA error, sticky), the pending FarSkip handle is completed into
// scratch so that the context (and, at EP > 1, the peers) is not left waiting.
extern "C" int fsc_layer_stack_forward(fsc_ctx* ctx, const fsc_attn_weights* attn, const fsc_moe_weights* moe, int L,
                                       int T, int seq_len, const int* modes, int schedule, const float* o0, float* oL,
                                       const fsc_act_cache* cache, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  if (ctx->sticky) return ctx->sticky;
  SREQ(attn && moe && modes && L >= 1, FSC_ERR_SHAPE, "stack: null arrays or L < 1");
  SREQ(T >= 0 && T <= ctx->cfg.max_tokens, FSC_ERR_CONFIG, "stack: T=%d outside [0,max_tokens]", T);
  SREQ(seq_len >= 1, FSC_ERR_CONFIG, "stack: seq_len < 1");
  SREQ(schedule == FSC_BLOCKING || schedule == FSC_OVERLAPPED, FSC_ERR_CONFIG, "stack: bad schedule");
  SREQ(T == 0 || (o0 && oL), FSC_ERR_SHAPE, "stack: null o0/oL");
  SREQ(!ctx->pending, FSC_ERR_STATE, "stack: a FarSkip handle is outstanding");
  for (int k = 0; k < L; ++k) {
    const fsc_attn_weights& a = attn[k];
    SREQ(modes[k] == FSC_REGULAR || modes[k] == FSC_HYBRID, FSC_ERR_CONFIG, "stack: mode[%d]", k);
    SREQ(a.gamma && a.w_qkv && a.w_o, FSC_ERR_SHAPE, "stack: null attention weight (layer %d)", k);
    SREQ(a.n_kv_heads >= 1 && a.n_heads % a.n_kv_heads == 0, FSC_ERR_CONFIG, "stack: heads %d/%d", a.n_heads,
         a.n_kv_heads);
    SREQ(a.head_dim == 16 || a.head_dim == 32 || a.head_dim == 64 || a.head_dim == 128, FSC_ERR_CONFIG,
         "stack: head_dim %d not in {16,32,64,128}", a.head_dim);
    SREQ(((a.n_heads + 2 * a.n_kv_heads) * a.head_dim) % 64 == 0 && (a.n_heads * a.head_dim) % 64 == 0,
         FSC_ERR_CONFIG, "stack: projection widths must be multiples of 64");
  }
  for (int k = 0; k < L; ++k) {
    SRC(fsc_validate_moe(ctx, &moe[k], T, o0, oL));
    SREQ(((reinterpret_cast<uintptr_t>(attn[k].w_qkv) | reinterpret_cast<uintptr_t>(attn[k].w_o) |
           reinterpret_cast<uintptr_t>(attn[k].gamma)) & 15) == 0,
         FSC_ERR_SHAPE, "stack: attention weights of layer %d must be 16-byte aligned", k);
  }
  SCK(cudaSetDevice(ctx->device));
  SRC(ensure_workspace(ctx, attn, L));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  fsc_handle h = nullptr;
  const int rc = stack_body(ctx, attn, moe, L, T, seq_len, modes, schedule, o0, oL, cache, s, &h);
  if (rc && ctx->pending && h) fsc_moe_wait(ctx, h, ctx->rbuf[0], ctx->rbuf[1], s);   // best effort
  ctx->no_overlap = 0;
  ctx->attn_pending = 0;
  return rc;
}

static int stack_body(fsc_ctx* ctx, const fsc_attn_weights* attn, const fsc_moe_weights* moe, int L, int T,
                      int seq_len, const int* modes, int schedule, const float* o0, float* oL,
                      const fsc_act_cache* cache, cudaStream_t s, fsc_handle* h_out) {
  const int d = ctx->cfg.d;
  const long n = (long)T * d;
  const bool ov = schedule == FSC_OVERLAPPED;
  float* bufA = ctx->rbuf[0];   // attn-in of the current layer (A_k) / o_{k-1} when nothing is pending
  float* bufM = ctx->rbuf[1];   // mlp-in of the current layer (M_k)
  float* bufP = ctx->rbuf[2];   // partial of the current layer (A_{k+1} in progress)
  SRC(copy_f32(ctx, bufA, o0, n, s));
  fsc_handle& h = *h_out;       // pending routed output: o_{k-1} = bufA + routed_{k-1}
  ctx->no_overlap = ov ? 0 : 1;
  int prev_k = -1;
  for (int k = 0; k < L; ++k) {
    const fsc_act_cache* ck = cache ? &cache[k] : nullptr;
    const fsc_moe_weights* mw = &moe[k];
    fsc_moe_debug dbg{};
    dbg.shared_out = ck ? ck->shared_out : nullptr;
    dbg.routed_out = ck ? ck->routed_out : nullptr;
    const fsc_moe_debug* dbgp = (dbg.shared_out || dbg.routed_out) ? &dbg : nullptr;
    SRC(attn_finish(ctx, bufA, s));   // TP: A_k += attn_out_{k-1} (synchronised before the next attention)
    if (modes[k] == FSC_REGULAR) {
      // o_{k-1} must be complete: wait the previous routed output into bufA
      if (h) {
        SRC(fsc_moe_wait(ctx, h, bufA, bufA, s));
        h = nullptr;
        if (cache && prev_k >= 0) SRC(copy_f32(ctx, cache[prev_k].o, bufA, n, s));
      }
      if (ck) SRC(copy_f32(ctx, ck->attn_in, bufA, n, s));
      SRC(attention_a(ctx, &attn[k], T, seq_len, bufA, s));
      SRC(attention_b(ctx, &attn[k], T, seq_len, bufA, bufM, ck ? ck->attn_out : nullptr, s));  // M = A + attn_out
      SRC(attn_finish(ctx, bufM, s));   // Regular: the MoE input needs attn_out now
      if (ck) SRC(copy_f32(ctx, ck->mlp_in, bufM, n, s));
      // partial := M (+= shared inside); routed pending. Nothing can overlap the
      // dispatch here (Regular wiring), so it runs on the compute stream.
      const int save = ctx->no_overlap;
      ctx->no_overlap = ov ? 2 : 1;   // OVERLAPPED: Regular+ (shared expert beside the combine)
      int rc = fsc_moe_forward_farskip(ctx, mw, T, bufM, bufM, nullptr, nullptr, &h, dbgp, s);
      ctx->no_overlap = save;
      SRC(rc);
      std::swap(bufA, bufM);   // bufA = M_k + shared_k = next layer's hybrid A_{k+1}
    } else {
      // Hybrid: A_k is in bufA; M_k = o_{k-1} = A_k + routed_{k-1} (pending) or o_0
      if (ck) SRC(copy_f32(ctx, ck->attn_in, bufA, n, s));
      const float* Mk = bufA;   // layer 0 / after a completed o_{k-1}: M_k = A_k = o_{k-1}
      if (!ov && h) {           // BLOCKING: the combine is waited before anything else
        SRC(fsc_moe_wait(ctx, h, bufA, bufM, s));
        h = nullptr;
        Mk = bufM;
        if (cache && prev_k >= 0) SRC(copy_f32(ctx, cache[prev_k].o, bufM, n, s));
      }
      SRC(attention_a(ctx, &attn[k], T, seq_len, bufA, s));                 // P:198 step 1
      if (h) {                                                              // step 2: sync Combine_{k-1}
        SRC(fsc_moe_wait(ctx, h, bufA, bufM, s));
        h = nullptr;
        Mk = bufM;
        if (cache && prev_k >= 0) SRC(copy_f32(ctx, cache[prev_k].o, bufM, n, s));
      }
      if (ck) SRC(copy_f32(ctx, ck->mlp_in, Mk, n, s));
      AttnCall ac{ctx, &attn[k], T, seq_len, Mk, bufP, ck ? ck->attn_out : nullptr, 0};
      // steps 3-8: gate, dispatch (comm stream) || attention (b) = o-proj into
      // bufP = M_k + attn_out_k, routed experts, combine (fused), shared: bufP += shared_k
      SRC(fsc_moe_forward_farskip(ctx, mw, T, Mk, bufP, attn_b_callback, &ac, &h, dbgp, s));
      SRC(ac.rc);
      std::swap(bufA, bufP);   // bufA = A_{k+1}
    }
    prev_k = k;
  }
  // final o_L = A_{L+1} + routed_L: the last combine has nothing to overlap
  SRC(attn_finish(ctx, bufA, s));
  SRC(fsc_moe_wait(ctx, h, bufA, oL, s));
  h = nullptr;
  if (cache) SRC(copy_f32(ctx, cache[L - 1].o, oL, n, s));
  return FSC_OK;
}
