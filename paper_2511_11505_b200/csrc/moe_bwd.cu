// fsc_moe_backward: gradients of one MoE sub-block (the backward of
// PAPER.md:73-76 and P:92-103, overlapped as P:207-211 describes) on sm_100a.
//
// Forward being differentiated (oracle/moe_backward.py; readings C-amb-2,4,5,7):
//   r_t = (mean x_t^2 + eps)^-1/2, xn = gamma x r; l = xn W_R^T; S_t = top-k, g = softmax_S(l);
//   y_e(a) = (a W1_e^T * SiLU(a W2_e^T)) W3_e^T; out = x + shared(xn) + sum_j g_tj y_{e_j}(xn_t)
//
// Schedule on this rank (compute stream s, high-priority comm stream):
//   s    : router + permutation maps (recomputed: the selection is piecewise constant), G -> bf16
//   comm : Dispatch of the xn rows (recompute) and of the gradient rows G[t] + gates g_tj to the
//          experts' owners (the gradient of the Combine)
//   s    : shared-expert backward (dgrad + wgrad) while those fly
//   s    : routed dgrad: dh_u = G_r W3 (MN-major B), SwiGLU backward on the recomputed
//          u, v (fused epilogue: du, dv, g h, dg partials), dX = [dU | dV] [W1 ; W2]
//   comm : dX rows + gate gradients back to their sources (the gradient of the Dispatch)
//   s    : routed wgrads dW3 = G_r^T (g h), dW1 = dU^T X, dW2 = dV^T X while that flies -
//          the explicit stream order that replaces the paper's autograd sequence-number hijack
//   s    : per token: router backward (softmax over the selected logits), sum of the dX
//          copies, RMSNorm backward; dgamma column sums; dW_R per expert.
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

using namespace fsc;

#define BCK(call)                                                                                 \
  do {                                                                                            \
    cudaError_t e__ = (call);                                                                     \
    if (e__ != cudaSuccess) {                                                                     \
      fsc_set_error(ctx, "backward %s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e__)); \
      ctx->sticky = FSC_ERR_CUDA;                                                                 \
      return FSC_ERR_CUDA;                                                                        \
    }                                                                                             \
  } while (0)
#define BREQ(cond, code, ...)          \
  do {                                 \
    if (!(cond)) {                     \
      fsc_set_error(ctx, __VA_ARGS__); \
      return code;                     \
    }                                  \
  } while (0)
#define BRC(expr)          \
  do {                     \
    int r__ = (expr);      \
    if (r__) return r__;   \
  } while (0)

namespace {

// G fp32 [T, d] -> bf16 (the GEMM operand of the shared expert's dgrad / wgrad)
__global__ void __launch_bounds__(256) f32_to_bf16_kernel(const float4* __restrict__ x, uint2* __restrict__ y, long n4) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    const float4 v = __ldg(x + i);
    y[i] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
  }
}

// EP = 1 gradient "dispatch": row pos[t,j] of the expert-sorted layout gets bf16(G[t]) and
// its gate g_tj (the receive layout is the send layout). One warp per copy.
__global__ void __launch_bounds__(256) permute_grad_kernel(const float* __restrict__ G, const int* __restrict__ pos,
                                                           const float* __restrict__ topk_w, long n_copies, int k,
                                                           int d, uint4* __restrict__ gr, float* __restrict__ gate) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dv = d / 8;
  for (long c = (long)blockIdx.x * 8 + w; c < n_copies; c += (long)gridDim.x * 8) {
    const long t = c / k;
    const int q = __ldg(pos + c);
    const float4* a = reinterpret_cast<const float4*>(G + t * d);
    for (int i = lane; i < dv; i += 32) {
      const float4 lo = __ldg(a + 2 * i), hi = __ldg(a + 2 * i + 1);
      gr[(long)q * dv + i] = make_uint4(pack_bf16x2(lo.x, lo.y), pack_bf16x2(lo.z, lo.w), pack_bf16x2(hi.x, hi.y),
                                        pack_bf16x2(hi.z, hi.w));
    }
    if (lane == 0) gate[q] = __ldg(topk_w + c);
  }
}

// Per token t (one WARP per token, 8 per CTA; lane l owns columns 8l + 256 m):
//   dg_j   = gate gradient of copy j (dgs[pos] at EP > 1, sum of dg_part[pos] at EP = 1)
//   dl_j   = g_j (dg_j - sum_i g_i dg_i)                (softmax over the selected logits)
//   dxn    = dxn_shared[t] + sum_j (dX[pos[t,j]] + dl_j W_R[e_j])   (slot order, fp32)
//   r      = (mean x^2 + eps)^-1/2;  q = dxn gamma;  dx = G + r q - x r^3 (q . x) / d
//   zg[t]  = dxn x r  (dgamma summands, summed over tokens by the colsum kernels)
// dxn is staged in place in dxn_zg (each lane re-reads only what it wrote) between the
// pass that forms it (and reduces sum x^2, q . x over the warp) and the pass that needs r.
// Also dl_row[pos[t,j]] = dl_j and r_tok[t] = r (for dW_R).
__global__ void __launch_bounds__(256) token_bwd_kernel(const float* __restrict__ x, const float* __restrict__ G,
                                                        const float* __restrict__ gamma, const float* __restrict__ w_router,
                                                        const int* __restrict__ idx, const int* __restrict__ pos,
                                                        const float* __restrict__ topk_w, const uint16_t* __restrict__ dxr,
                                                        const float* __restrict__ dgs, const float* __restrict__ dg_part,
                                                        int dg_n, int dg_ld, float* dxn_zg, float* __restrict__ dx,
                                                        float* __restrict__ dl_row, float* __restrict__ r_tok, int T,
                                                        int d, int k, float eps) {
  const int lane = threadIdx.x & 31;
  const long t = (long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  // slot j lives in lane j (k <= 8)
  int qj = 0, ej = 0;
  float gj = 0.f, dgj = 0.f;
  if (lane < k) {
    qj = __ldg(pos + t * k + lane);
    ej = __ldg(idx + t * k + lane);
    gj = __ldg(topk_w + t * k + lane);
    if (dgs) {
      dgj = __ldcg(dgs + qj);
    } else {
      for (int i = 0; i < dg_n; ++i) dgj += __ldg(dg_part + (long)qj * dg_ld + i);
    }
  }
  float gd = gj * dgj;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) gd += __shfl_xor_sync(0xffffffffu, gd, o);
  const float dlj = gj * (dgj - gd);
  int qs[8], es[8];
  float dl[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {                // (full-warp shuffles: before the column loop)
    qs[j] = __shfl_sync(0xffffffffu, qj, j);
    es[j] = __shfl_sync(0xffffffffu, ej, j);
    dl[j] = __shfl_sync(0xffffffffu, dlj, j);
  }
  const float* xt = x + t * d;
  float* zt = dxn_zg + t * d;
  float ss = 0.f, qx = 0.f;
  for (int c = 8 * lane; c < d; c += 256) {
    const float4 x0 = __ldg(reinterpret_cast<const float4*>(xt + c)), x1 = __ldg(reinterpret_cast<const float4*>(xt + c + 4));
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + c)), g1 = __ldg(reinterpret_cast<const float4*>(gamma + c + 4));
    float4 a0 = *reinterpret_cast<const float4*>(zt + c), a1 = *reinterpret_cast<const float4*>(zt + c + 4);
    float v[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    uint4 yv[8];
    float4 w0[8], w1[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {              // every slot's loads in flight together
      const int q = qs[j], e = es[j];
      if (j < k) {
        yv[j] = __ldcg(reinterpret_cast<const uint4*>(dxr + (long)q * d + c));
        w0[j] = __ldg(reinterpret_cast<const float4*>(w_router + (long)e * d + c));
        w1[j] = __ldg(reinterpret_cast<const float4*>(w_router + (long)e * d + c + 4));
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < k) {
        const float wv[8] = {w0[j].x, w0[j].y, w0[j].z, w0[j].w, w1[j].x, w1[j].y, w1[j].z, w1[j].w};
        const uint32_t yw[4] = {yv[j].x, yv[j].y, yv[j].z, yv[j].w};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v[u] += (u & 1) ? bf16hi(yw[u >> 1]) : bf16lo(yw[u >> 1]);
          v[u] = fmaf(dl[j], wv[u], v[u]);
        }
      }
    }
    const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      ss = fmaf(xv[u], xv[u], ss);
      qx = fmaf(v[u] * gv[u], xv[u], qx);
    }
    *reinterpret_cast<float4*>(zt + c) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(zt + c + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    qx += __shfl_xor_sync(0xffffffffu, qx, o);
  }
  const float r = rsqrtf(ss / (float)d + eps);
  const float c3 = r * r * r * qx / (float)d;
  const float* gt = G + t * d;
  float* dxt = dx + t * d;
  for (int c = 8 * lane; c < d; c += 256) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float4 a = *reinterpret_cast<const float4*>(zt + c + 4 * h);
      const float4 xx = __ldg(reinterpret_cast<const float4*>(xt + c + 4 * h));
      const float4 gg = __ldg(reinterpret_cast<const float4*>(gamma + c + 4 * h));
      const float4 G4 = __ldg(reinterpret_cast<const float4*>(gt + c + 4 * h));
      *reinterpret_cast<float4*>(dxt + c + 4 * h) =
          make_float4(G4.x + r * a.x * gg.x - xx.x * c3, G4.y + r * a.y * gg.y - xx.y * c3,
                      G4.z + r * a.z * gg.z - xx.z * c3, G4.w + r * a.w * gg.w - xx.w * c3);
      *reinterpret_cast<float4*>(zt + c + 4 * h) =
          make_float4(a.x * xx.x * r, a.y * xx.y * r, a.z * xx.z * r, a.w * xx.w * r);
    }
  }
  if (lane < k) dl_row[qj] = dlj;
  if (lane == 0) r_tok[t] = r;
}

// dgamma[i] = sum_t zg[t, i]: partial sums over 64-token chunks (token order), then the
// chunks in order - deterministic and spread over the GPU
constexpr int kColChunk = 64;
__global__ void __launch_bounds__(256) colsum_part_kernel(const float* __restrict__ zg, float* __restrict__ part, int T,
                                                          int d) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int t0 = blockIdx.y * kColChunk, t1 = min(T, t0 + kColChunk);
  if (i >= d) return;
  float a = 0.f;
#pragma unroll 8
  for (int t = t0; t < t1; ++t) a += __ldcg(zg + (long)t * d + i);
  part[(long)blockIdx.y * d + i] = a;
}
__global__ void __launch_bounds__(256) colsum_final_kernel(const float* __restrict__ part, float* __restrict__ out,
                                                           int nchunk, int d) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= d) return;
  float a = 0.f;
  for (int c = 0; c < nchunk; ++c) a += part[(long)c * d + i];
  out[i] = a;
}

// dW_R[e, i] = sum over the copies q of expert e (send order) of dl_row[q] * xn32[src_row[q], i],
// xn32 = x r gamma in fp32 (gamma applied once at the end). Copies are staged 256 at a time
// in shared memory (token, dl r), so every thread's x loads are independent (8 in flight).
__global__ void __launch_bounds__(256) dwr_kernel(const float* __restrict__ x, const float* __restrict__ gamma,
                                                  const float* __restrict__ r_tok, const int* __restrict__ offsets,
                                                  const int* __restrict__ src_row, const float* __restrict__ dl_row,
                                                  float* __restrict__ dwr, int d) {
  __shared__ int s_t[256];
  __shared__ float s_c[256];
  const int e = blockIdx.y;
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int q0 = offsets[e], q1 = offsets[e + 1];
  float a = 0.f;
  for (int b = q0; b < q1; b += 256) {
    const int n = min(256, q1 - b);
    __syncthreads();
    if ((int)threadIdx.x < n) {
      const int t = __ldg(src_row + b + threadIdx.x);
      s_t[threadIdx.x] = t;
      s_c[threadIdx.x] = __ldg(dl_row + b + threadIdx.x) * __ldg(r_tok + t);
    }
    __syncthreads();
    if (i < d) {
#pragma unroll 8
      for (int u = 0; u < n; ++u) a = fmaf(s_c[u], __ldg(x + (long)s_t[u] * d + i), a);
    }
  }
  if (i < d) dwr[(long)e * d + i] = a * __ldg(gamma + i);
}

}  // namespace

// ---------------------------------------------------------------------------- host

namespace {

template <typename T>
cudaError_t balloc(T** p, size_t n) {
  return cudaMalloc(reinterpret_cast<void**>(p), (n ? n : 1) * sizeof(T));
}

// backward workspace, allocated on the first fsc_moe_backward call
int ensure_bwd_workspace(fsc_ctx* ctx) {
  if (ctx->b_duv) return FSC_OK;
  const fsc_moe_config& c = ctx->cfg;
  const long T = c.max_tokens, d = c.d, k = c.top_k;
  const long rows = std::max(ctx->max_recv, std::max(T * k, T));
  const long cmax = std::max(c.ffn, c.shared_ffn);
  BCK(balloc(&ctx->b_gb, T * d));
  BCK(balloc(&ctx->b_duv, rows * 2 * cmax));
  BCK(balloc(&ctx->b_hg, rows * cmax));
  ctx->b_dg_ld = 2 * (c.ffn / 64) + 2;
  BCK(balloc(&ctx->b_dgpart, rows * ctx->b_dg_ld));
  BCK(balloc(&ctx->b_dlrow, T * k));
  BCK(balloc(&ctx->b_rtok, T));
  BCK(balloc(&ctx->b_colpart, ((T + 63) / 64) * d));
  if (ctx->ep == 1) {
    BCK(balloc(&ctx->b_gr, T * k * d));
    BCK(balloc(&ctx->b_gate, T * k));
  }
  return FSC_OK;
}

int launch_wgrad(fsc_ctx* ctx, const int* counts, int G, int m_total, int N1, int N2, const uint16_t* A, long lda,
                 int a_col0, const uint16_t* B, long ldb, float* out, long rows, cudaStream_t s) {
  if (!out) return FSC_OK;
  WgradParams p{};
  p.counts = counts; p.G = G; p.m_total = m_total; p.row_base = nullptr; p.N1 = N1; p.N2 = N2;
  p.A = A; p.lda = lda; p.a_col0 = a_col0; p.B = B; p.ldb = ldb; p.b_col0 = 0; p.out = out; p.accumulate = 0;
  BCK(launch_wgrad_gemm(p, rows, rows, ctx->gemm_ctas, s));
  return FSC_OK;
}

}  // namespace

extern "C" int fsc_moe_backward(fsc_ctx* ctx, const fsc_moe_weights* w, int T, const float* x_in,
                                const float* grad_out, const fsc_moe_grads* gr, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  BRC(fsc_validate_moe(ctx, w, T, x_in, grad_out));
  BREQ(gr && gr->dx, FSC_ERR_SHAPE, "backward: dx is required");
  BREQ(!ctx->pending, FSC_ERR_STATE, "backward: a FarSkip handle is outstanding");
  BREQ(ctx->ep == 1 || ctx->ep_mode == FSC_EP_ALLTOALL, FSC_ERR_CONFIG,
       "backward: the all-reduce inference variant has no backward");
  BREQ(!ctx->spin, FSC_ERR_STATE, "backward: spin schedule active");
  BREQ(!ctx->a2a_zero_bytes, FSC_ERR_STATE, "backward: zero-byte instrument active");
  const fsc_moe_config& c = ctx->cfg;
  const int d = c.d, E = c.n_experts, k = c.top_k, cf = c.ffn, cs = c.shared_ffn;
  BREQ(cf % 64 == 0 && cs % 64 == 0, FSC_ERR_CONFIG, "backward: ffn widths must be multiples of 64");
  BREQ(k <= 8, FSC_ERR_CONFIG, "backward: top_k <= 8");
  BCK(cudaSetDevice(ctx->device));
  if (T == 0) return FSC_OK;
  BRC(ensure_bwd_workspace(ctx));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long R = (long)T * k;
  memset(ctx->ph_used, 0, sizeof(ctx->ph_used));

  // ---- recompute the selection (router + maps) and G in bf16
  BCK(fsc_phase_begin(ctx, PH_ROUTER, s));
  RouterLaunch rl{x_in, w->gamma, w->w_router, T, d, E, k, c.rms_eps, ctx->xn, ctx->topk_idx, ctx->topk_w,
                  nullptr, nullptr, ctx->r_part, ctx->r_part_sq, ctx->w_scaled, ctx->w_sq, 32,
                  ctx->i8_w, ctx->i8_exp, router_tc_on(ctx) ? 1 : 0};   // the forward's router
  rl.f64 = router_f64_on(ctx, T, d, E, k) ? 1 : 0;
  rl.f64_w = ctx->f64_w;
  BCK(launch_router(rl, s));
  PermLaunch pl{ctx->topk_idx, T, k, E, ctx->hist, ctx->base, ctx->counts, ctx->offsets, ctx->pos, ctx->src_row};
  BCK(launch_perm_maps(pl, s));
  BCK(fsc_phase_end(ctx, PH_ROUTER, s));
  {
    const long n4 = (long)T * d / 4;
    ++g_launches;
    f32_to_bf16_kernel<<<(int)std::min<long>((n4 + 255) / 256, 4 * kNumSMs), 256, 0, s>>>(
        reinterpret_cast<const float4*>(grad_out), reinterpret_cast<uint2*>(ctx->b_gb), n4);
    BCK(cudaGetLastError());
  }
  // ---- comm stream: Dispatch of the xn rows (recompute) and of the gradient rows
  BCK(cudaEventRecord(ctx->ev_a, s));
  BCK(cudaStreamWaitEvent(ctx->comm, ctx->ev_a, 0));
  const uint16_t* xrows;      // expert input rows (receive layout)
  const int* rcounts;         // rows per local expert
  long rows_cap;
  uint16_t* g_rows;
  float* g_gate;
  float* dgs = nullptr;
  BCK(fsc_phase_begin(ctx, PH_DISPATCH, ctx->comm));
  if (ctx->ep == 1) {
    BCK(launch_permute_ep1(ctx->xn, ctx->src_row, ctx->pos, ctx->xs, T, k, d, ctx->comm));
    g_rows = ctx->b_gr;
    g_gate = ctx->b_gate;
    ++g_launches;
    permute_grad_kernel<<<(int)std::min<long>((R + 7) / 8, 4 * kNumSMs), 256, 0, ctx->comm>>>(
        grad_out, ctx->pos, ctx->topk_w, R, k, d, reinterpret_cast<uint4*>(g_rows), g_gate);
    BCK(cudaGetLastError());
    xrows = ctx->xs;
    rcounts = ctx->counts;
    rows_cap = R;
  } else {
    BRC(fsc_transport_dispatch(ctx, T, ctx->comm));
    BRC(fsc_transport_dispatch_wait(ctx, ctx->comm));
    BRC(fsc_transport_dispatch_grad(ctx, T, grad_out, ctx->comm));
    fsc_transport_bwd_ptrs(ctx, &g_rows, &g_gate, &dgs);
    xrows = ctx->xr;
    rcounts = ctx->recv_counts;
    rows_cap = ctx->recv_rows_cap;
  }
  BCK(fsc_phase_end(ctx, PH_DISPATCH, ctx->comm));
  BCK(cudaEventRecord(ctx->ev_b, ctx->comm));

  // ---- shared expert backward (beside the dispatches): dxn = shared part, dWs
  const int cg = ctx->gemm_cg ? ctx->gemm_cg : 2;
  BCK(fsc_phase_begin(ctx, PH_SHARED1, s));
  if (cs) {
    GemmLaunch a{};   // dh_s = G Ws3                      [T, c_s]
    a.A = ctx->b_gb; a.a_rows = T; a.B0 = w->ws3; a.b_rows = d; a.b_group_rows = d; a.K = d; a.N = cs; a.G = 1;
    a.m_total = T; a.out = ctx->hs; a.ldo = cs; a.epi = EPI_BF16; a.b_mn = true; a.num_ctas = ctx->gemm_ctas;
    a.cta_group = cg;
    BCK(launch_grouped_gemm(a, s));
    GemmLaunch b{};   // recompute u, v on xn; du, dv, h
    b.A = ctx->xn; b.a_rows = T; b.B0 = w->ws1; b.B1 = w->ws2; b.b_rows = cs; b.b_group_rows = cs; b.K = d; b.N = cs;
    b.G = 1; b.m_total = T; b.out = ctx->b_duv; b.ldo = 2 * cs; b.out2 = ctx->b_hg; b.dh = ctx->hs;
    b.epi = EPI_SWIGLU_BWD; b.num_ctas = ctx->gemm_ctas; b.cta_group = cg;
    BCK(launch_grouped_gemm(b, s));
    GemmLaunch cc{};  // dxn_s = [du | dv] [Ws1 ; Ws2]     fp32 [T, d]
    cc.A = ctx->b_duv; cc.a_rows = T; cc.B0 = w->ws1; cc.B1 = w->ws2; cc.b_rows = cs; cc.b_group_rows = cs;
    cc.K = 2 * cs; cc.N = d; cc.kb_split = cs / 64; cc.b_mn = true; cc.G = 1; cc.m_total = T; cc.out = ctx->tmp;
    cc.ldo = d; cc.resid = nullptr; cc.ldr = d; cc.epi = EPI_RESID_F32; cc.num_ctas = ctx->gemm_ctas; cc.cta_group = cg;
    BCK(launch_grouped_gemm(cc, s));
    BRC(launch_wgrad(ctx, nullptr, 1, T, d, cs, ctx->b_gb, d, 0, ctx->b_hg, cs, gr->dws3, T, s));
    BRC(launch_wgrad(ctx, nullptr, 1, T, cs, d, ctx->b_duv, 2 * cs, 0, ctx->xn, d, gr->dws1, T, s));
    BRC(launch_wgrad(ctx, nullptr, 1, T, cs, d, ctx->b_duv, 2 * cs, cs, ctx->xn, d, gr->dws2, T, s));
  } else {
    BCK(cudaMemsetAsync(ctx->tmp, 0, sizeof(float) * (size_t)T * d, s));
  }
  BCK(fsc_phase_end(ctx, PH_SHARED1, s));

  // ---- routed dgrad (after the dispatches)
  BCK(fsc_phase_begin(ctx, PH_DISPATCH_STALL, s));
  BCK(cudaStreamWaitEvent(s, ctx->ev_b, 0));
  BCK(fsc_phase_end(ctx, PH_DISPATCH_STALL, s));
  const long avg_rows = R * ctx->ep / E;
  const int rcg = ctx->gemm_cg ? ctx->gemm_cg : (avg_rows < 256 ? 1 : 2);
  BCK(fsc_phase_begin(ctx, PH_GEMM1, s));
  {
    GemmLaunch a{};   // dh_u = G_r W3_e                     [rows, c]
    a.A = g_rows; a.a_rows = rows_cap; a.B0 = w->w3; a.b_rows = (long)ctx->e_loc * d; a.b_group_rows = d; a.K = d;
    a.N = cf; a.G = ctx->e_loc; a.counts = rcounts; a.out = ctx->h; a.ldo = cf; a.epi = EPI_BF16; a.b_mn = true;
    a.num_ctas = ctx->gemm_ctas; a.cta_group = rcg;
    BCK(launch_grouped_gemm(a, s));
    GemmLaunch b{};   // recompute u, v; du, dv (gate-scaled), g h, dg partials
    b.A = xrows; b.a_rows = rows_cap; b.B0 = w->w1; b.B1 = w->w2; b.b_rows = (long)ctx->e_loc * cf;
    b.b_group_rows = cf; b.K = d; b.N = cf; b.G = ctx->e_loc; b.counts = rcounts; b.out = ctx->b_duv; b.ldo = 2 * cf;
    b.out2 = ctx->b_hg; b.dh = ctx->h; b.row_gate = g_gate; b.dg_part = ctx->b_dgpart; b.dg_ld = ctx->b_dg_ld;
    b.epi = EPI_SWIGLU_BWD; b.num_ctas = ctx->gemm_ctas; b.cta_group = rcg;
    BCK(launch_grouped_gemm(b, s));
  }
  BCK(fsc_phase_end(ctx, PH_GEMM1, s));
  // dg partials per row: 2 per N tile of the SwiGLU-backward GEMM (tile width HALF = BN / 2)
  const int dg_n = 2 * (cf / (gemm_pick_bn(EPI_SWIGLU_BWD, cf) / 2));
  BCK(fsc_phase_begin(ctx, PH_GEMM2, s));
  {
    GemmLaunch cc{};  // dX = [dU | dV] [W1_e ; W2_e]         [rows, d]
    cc.A = ctx->b_duv; cc.a_rows = rows_cap; cc.B0 = w->w1; cc.B1 = w->w2; cc.b_rows = (long)ctx->e_loc * cf;
    cc.b_group_rows = cf; cc.K = 2 * cf; cc.N = d; cc.kb_split = cf / 64; cc.b_mn = true; cc.G = ctx->e_loc;
    cc.counts = rcounts; cc.out = ctx->y; cc.ldo = d; cc.epi = EPI_BF16; cc.num_ctas = ctx->gemm_ctas;
    cc.cta_group = rcg;
    BCK(launch_grouped_gemm(cc, s));
  }
  BCK(fsc_phase_end(ctx, PH_GEMM2, s));
  // ---- gradient combine on the comm stream, routed wgrads beside it
  if (ctx->ep > 1) {
    BCK(cudaEventRecord(ctx->ev_g2, s));
    BCK(cudaStreamWaitEvent(ctx->comm, ctx->ev_g2, 0));
    BCK(fsc_phase_begin(ctx, PH_COMBINE, ctx->comm));
    BRC(fsc_transport_combine_grad(ctx, ctx->y, ctx->b_dgpart, dg_n, ctx->b_dg_ld, ctx->comm));
    BCK(fsc_phase_end(ctx, PH_COMBINE, ctx->comm));
    BCK(cudaEventRecord(ctx->ev_comb, ctx->comm));
  }
  BCK(fsc_phase_begin(ctx, PH_SHARED2, s));
  BRC(launch_wgrad(ctx, rcounts, ctx->e_loc, 0, d, cf, g_rows, d, 0, ctx->b_hg, cf, gr->dw3, rows_cap, s));
  BRC(launch_wgrad(ctx, rcounts, ctx->e_loc, 0, cf, d, ctx->b_duv, 2 * cf, 0, xrows, d, gr->dw1, rows_cap, s));
  BRC(launch_wgrad(ctx, rcounts, ctx->e_loc, 0, cf, d, ctx->b_duv, 2 * cf, cf, xrows, d, gr->dw2, rows_cap, s));
  BCK(fsc_phase_end(ctx, PH_SHARED2, s));
  const uint16_t* dxr = ctx->y;
  if (ctx->ep > 1) {
    BCK(fsc_phase_begin(ctx, PH_COMBINE_WAIT, s));
    BCK(cudaStreamWaitEvent(s, ctx->ev_comb, 0));
    BRC(fsc_transport_combine_grad_wait(ctx, s));
    BCK(fsc_phase_end(ctx, PH_COMBINE_WAIT, s));
    dxr = ctx->ys;
  }
  // ---- per token: router backward, sum of the copies, RMSNorm backward; dgamma; dW_R
  BCK(fsc_phase_begin(ctx, PH_UNPERMUTE, s));
  ++g_launches;
  token_bwd_kernel<<<(T + 7) / 8, 256, 0, s>>>(x_in, grad_out, w->gamma, w->w_router, ctx->topk_idx, ctx->pos,
                                               ctx->topk_w, dxr, dgs, ctx->b_dgpart, dg_n, ctx->b_dg_ld, ctx->tmp,
                                               gr->dx, ctx->b_dlrow, ctx->b_rtok, T, d, k, c.rms_eps);
  BCK(cudaGetLastError());
  if (gr->dgamma) {
    const int nchunk = (T + kColChunk - 1) / kColChunk;
    g_launches += 2;
    colsum_part_kernel<<<dim3((d + 255) / 256, nchunk), 256, 0, s>>>(ctx->tmp, ctx->b_colpart, T, d);
    colsum_final_kernel<<<(d + 255) / 256, 256, 0, s>>>(ctx->b_colpart, gr->dgamma, nchunk, d);
    BCK(cudaGetLastError());
  }
  if (gr->dw_router) {
    ++g_launches;
    dwr_kernel<<<dim3((d + 255) / 256, E), 256, 0, s>>>(x_in, w->gamma, ctx->b_rtok, ctx->offsets, ctx->src_row,
                                                       ctx->b_dlrow, gr->dw_router, d);
    BCK(cudaGetLastError());
  }
  BCK(fsc_phase_end(ctx, PH_UNPERMUTE, s));
  return fsc_check_finite(ctx, gr->dx, (long)T * d, s, "fsc_moe_backward");
}

// ---------------------------------------------------------------------------- op-level entry points (tests)

extern "C" int fsc_op_gemm_dgrad(fsc_ctx* ctx, int epi, const void* A, long a_rows, const void* B0, const void* B1,
                                 long b_group_rows, int G, const int* counts, int m_total, int N, int K,
                                 int kb_split, void* out, const float* resid, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  BREQ(epi == EPI_BF16 || epi == EPI_RESID_F32, FSC_ERR_CONFIG, "dgrad epilogue must be bf16 or fp32-residual");
  BREQ(K % 64 == 0 && N % 64 == 0 && G >= 1 && G <= 256 && kb_split >= 0 && kb_split * 64 <= K, FSC_ERR_CONFIG,
       "bad dgrad GEMM shape");
  GemmLaunch L{};
  L.A = A; L.a_rows = a_rows; L.B0 = B0; L.B1 = B1 ? B1 : B0; L.b_rows = (long)G * b_group_rows;
  L.b_group_rows = (int)b_group_rows; L.K = K; L.N = N; L.G = G; L.counts = counts; L.m_total = m_total; L.out = out;
  L.ldo = N; L.resid = resid; L.ldr = N; L.epi = epi; L.b_mn = true; L.kb_split = kb_split;
  L.num_ctas = ctx->gemm_ctas; L.cta_group = ctx->gemm_cg ? ctx->gemm_cg : 2;
  BCK(launch_grouped_gemm(L, static_cast<cudaStream_t>(stream)));
  return FSC_OK;
}

extern "C" int fsc_op_gemm_swiglu_bwd(fsc_ctx* ctx, const void* A, long a_rows, const void* B0, const void* B1, int G,
                                      const int* counts, int m_total, int N, int K, const void* dh,
                                      const float* row_gate, void* duv, void* hg, float* dg_part, int dg_ld,
                                      void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  BREQ(K % 64 == 0 && N % 64 == 0 && G >= 1 && G <= 256 && dh && duv && hg, FSC_ERR_CONFIG,
       "bad SwiGLU-backward GEMM arguments");
  GemmLaunch L{};
  L.A = A; L.a_rows = a_rows; L.B0 = B0; L.B1 = B1; L.b_rows = (long)G * N; L.b_group_rows = N; L.K = K; L.N = N;
  L.G = G; L.counts = counts; L.m_total = m_total; L.out = duv; L.ldo = 2 * N; L.out2 = hg;
  L.dh = static_cast<const uint16_t*>(dh); L.row_gate = row_gate; L.dg_part = dg_part; L.dg_ld = dg_ld;
  L.epi = EPI_SWIGLU_BWD; L.num_ctas = ctx->gemm_ctas; L.cta_group = ctx->gemm_cg ? ctx->gemm_cg : 2;
  BCK(launch_grouped_gemm(L, static_cast<cudaStream_t>(stream)));
  return FSC_OK;
}

extern "C" int fsc_op_gemm_wgrad(fsc_ctx* ctx, const int* counts, int G, int m_total, int N1, int N2, const void* A,
                                 long a_rows, long lda, int a_col0, const void* B, long ldb, int b_col0, float* out,
                                 int accumulate, void* stream) {
  if (!ctx) return FSC_ERR_SHAPE;
  WgradParams p{};
  p.counts = counts; p.G = G; p.m_total = m_total; p.N1 = N1; p.N2 = N2;
  p.A = static_cast<const uint16_t*>(A); p.lda = lda; p.a_col0 = a_col0;
  p.B = static_cast<const uint16_t*>(B); p.ldb = ldb; p.b_col0 = b_col0; p.out = out; p.accumulate = accumulate;
  BCK(launch_wgrad_gemm(p, a_rows, a_rows, ctx->gemm_ctas, static_cast<cudaStream_t>(stream)));
  return FSC_OK;
}
