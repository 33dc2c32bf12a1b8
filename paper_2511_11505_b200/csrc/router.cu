// K1: fused RMSNorm + fp32 router logits + top-k + renormalised gates.
//
//   r_t   = (mean_i x_ti^2 + eps)^-1/2                  (RMSNorm, C-amb-5; sum of squares in fp64)
//   xn_t  = x_t * gamma * r_t  -> bf16 (expert GEMM operand)
//   l_te  = r_t * sum_i x_ti W'_ei,  W' = gamma * W_R     (G(A) = s(A W_R^T))
//   S_t   = top-k of l_t, exact ties -> lower expert id; slots ascending by id (C-amb-3)
//   g_tj  = exp(l_tj - max) / sum_{S_t} exp(l - max)     (softmax over E then renormalise
//                                                         == softmax over the selected logits)
// Exact selection. Every fp32 logit carries an error
// |v_e - l_e| <= B_t = r_t (chain + 6) u ||x_t||_2 max_e ||W'_e||_2 (worst-case
// rounding of the accumulation chain, Cauchy-Schwarz). With t_hi / t_lo the k-th /
// (k+1)-th largest fp32 logits, an expert with v > t_hi + 2B is certainly selected
// and one with v < t_lo - 2B certainly not; only the experts in between ("the
// band", usually 2-3) of tokens with t_hi - t_lo <= 2B are recomputed in fp64 by
// the same CTA (refine_block) and the missing slots filled by their fp64 order. The
// selection therefore equals the fp64 selection of the oracle for every token.
//
// Main kernel: block = 32 tokens x 32/64/128 (padded) experts, 8 warps; each warp
// owns one k-slice of every 64-wide chunk (k-split, summed in a fixed order at the
// end) and an 8 tokens x 8 (or 4) experts register tile per lane; operands are
// staged by a 2-4 deep cp.async pipeline, read with conflict-free LDS.64 (128 FMA
// per shared-memory wavefront, the binding resource of an fp32 SIMT contraction on
// sm_100). sum x^2 is accumulated from the staged chunks (no extra pass over x).
// Small T (decode): the grid also splits d (gridDim.y), raw partials go to a
// workspace and router_finish_kernel sums them in a fixed order and selects.
#include <cudaTypedefs.h>
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace fsc {

namespace {
constexpr int TB = 32;      // tokens per block
constexpr int DC = 64;      // k per staged chunk
constexpr int LDS = DC + 4; // padded smem row (floats): rows r, r+1 start 4 banks apart
constexpr float kU = 5.9604645e-08f;  // 2^-24
constexpr int kMaxD = 8192;
constexpr int kThreadSelK1 = 9;
constexpr int kMaxSplit = 8;
constexpr int kFinishRows = 8;  // thread-per-token selection for k <= 8

FSC_DEVINL uint32_t ordered_f32(float v) {
  uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
FSC_DEVINL unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffff, v, o);
    v = w > v ? w : v;
  }
  return v;
}
FSC_DEVINL double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}
FSC_DEVINL float warp_sum_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}
FSC_DEVINL float warp_max_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, o));
  return v;
}
FSC_DEVINL void cp_async16(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
FSC_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
FSC_DEVINL void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// Per-CTA state of the in-block band refinement (see refine_block), for blocks of ROWS tokens.
template <int ROWS>
struct RefineSmemT {
  int flag[ROWS];        // token of the block has an ambiguous top-k boundary
  float thr[ROWS][3];    // {2B + 4u(|l_(k)| + |l_(k+1)|), l_(k), l_(k+1)} of flagged tokens
  int band[128];
  int nb;
  double l64[128];
};
using RefineSmem = RefineSmemT<TB>;
}  // namespace

// W'[e][i] = gamma_i * W_R[e][i] and ||W'_e||^2 (error bound). One CTA per expert.
// ldt > 0: W' is written k-major (W'T[i][e], row stride ldt, rows padded with
// zeros for E <= e < ldt by the CTAs with e >= E) for the FFMA2 main kernel.
__global__ void __launch_bounds__(256) router_prescale_kernel(const float* __restrict__ W,
                                                              const float* __restrict__ gamma, float* __restrict__ Wg,
                                                              float* __restrict__ wq, int E, int d, int ldt) {
  __shared__ float red[8];
  const int e = blockIdx.x, tid = threadIdx.x;
  if (e >= E) {                                  // zero padding columns of W'T
    for (int c = tid; c < d; c += 256) Wg[(long)c * ldt + e] = 0.f;
    return;
  }
  const float4* w = reinterpret_cast<const float4*>(W + (long)e * d);
  const float4* g = reinterpret_cast<const float4*>(gamma);
  float s = 0.f;
  for (int c = tid; c < d / 4; c += 256) {
    const float4 a = w[c], b = g[c];
    const float4 v = make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
    if (ldt > 0) {
      float* o = Wg + (long)(4 * c) * ldt + e;
      o[0] = v.x;
      o[ldt] = v.y;
      o[2 * ldt] = v.z;
      o[3 * ldt] = v.w;
    } else {
      reinterpret_cast<float4*>(Wg + (long)e * d)[c] = v;
    }
    s += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  s = warp_sum_f32(s);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i];
    wq[e] = t;
  }
}

// packed fp32x2 FMA (sm_100 FFMA2) with a scalar operand broadcast to both lanes:
// acc.{x,y} += a * b.{x,y}
FSC_DEVINL void ffma2_bcast(float2& acc, float a, float2 b) {
  unsigned long long B = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long C = *reinterpret_cast<unsigned long long*>(&acc);
  unsigned long long A;
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
  acc = *reinterpret_cast<float2*>(&C);
}

// Phase C for one token (one warp): top-k over the fp32 logits of row `lg`, gates,
// or hand-off of the token to the band refinement when its boundary is ambiguous.
template <int QN, class RS>
FSC_DEVINL void select_token(const float* lg, long t, int tt, float B, const RouterLaunch& L, RS& rs, int lane) {
  const int E = L.E, k = L.k;
  float v[QN];
#pragma unroll
  for (int q = 0; q < QN; ++q) {
    const int e = lane + 32 * q;
    v[q] = (e < E) ? lg[e] : -FLT_MAX;
  }
#ifndef FSC_ROUTER_PROF
  if (L.logits)
    for (int e = lane; e < E; e += 32) L.logits[t * E + e] = lg[e];
#endif
  // k (+1 for the boundary) rounds of warp argmax, ties -> lower id
  uint32_t selbits = 0;
  float vtop = 0.f, vk = 0.f, vk1 = -FLT_MAX;
  const int rounds = k < E ? k + 1 : k;
  for (int rd = 0; rd < rounds; ++rd) {
    unsigned long long best = 0;
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const int e = lane + 32 * q;
      if (e < E && !((selbits >> q) & 1u)) {
        unsigned long long key = ((unsigned long long)ordered_f32(v[q]) << 32) | (0xFFFFFFFFu - (uint32_t)e);
        best = key > best ? key : best;
      }
    }
    best = warp_max_u64(best);
    const int ew = (int)(0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFu));
    float val = 0.f;
#pragma unroll
    for (int q = 0; q < QN; ++q)
      if (lane + 32 * q == ew) val = v[q];
    val = __shfl_sync(0xffffffff, val, ew & 31);
    if (rd < k) {
      if ((ew & 31) == lane) selbits |= 1u << (ew >> 5);
      if (rd == 0) vtop = val;
      if (rd == k - 1) vk = val;
    } else {
      vk1 = val;
    }
  }
  const float thr2 = 2.f * B + 4.f * kU * (fabsf(vk) + fabsf(vk1)) + 1e-7f;
  if (k < E && vk - vk1 <= thr2) {   // ambiguous boundary: refined by the block (refine_block)
    if (lane == 0) {
      if (L.n_refined) atomicAdd(L.n_refined, 1);
      rs.flag[tt] = 1;
      rs.thr[tt][0] = thr2;
      rs.thr[tt][1] = vk;
      rs.thr[tt][2] = vk1;
    }
    return;
  }
  float ex[QN], sum = 0.f;
#pragma unroll
  for (int q = 0; q < QN; ++q) {
    ex[q] = ((selbits >> q) & 1u) ? expf(v[q] - vtop) : 0.f;
    sum += ex[q];
  }
  sum = warp_sum_f32(sum);
  int slot = 0;
#pragma unroll
  for (int q = 0; q < QN; ++q) {
    const uint32_t m = __ballot_sync(0xffffffff, (selbits >> q) & 1u);
    if ((selbits >> q) & 1u) {
      const int s = slot + __popc(m & ((1u << lane) - 1u));
      L.topk_idx[t * k + s] = lane + 32 * q;
      L.topk_w[t * k + s] = ex[q] / sum;
    }
    slot += __popc(m);
  }
}

// Phase C, one THREAD per token (k < K1): the top-(k+1) of the row by insertion
// over the E logits in ascending expert order (strict '>' keeps the lower id on
// exact ties), then the boundary test, gates and ascending-id slots exactly as in
// select_token. A warp selects 32 tokens at once with no shuffles (the warp
// version above is latency-bound on k+1 rounds of 64-bit shuffle argmax).
template <int K1, class RS>   // K1 = k + 1 (compile time: every register array index is static)
FSC_DEVINL void select_token_thread(const float* lg, long t, int tt, float B, const RouterLaunch& L, RS& rs) {
  constexpr int k = K1 - 1;
  const int E = L.E;
  float val[K1];
  int idx[K1];
#pragma unroll
  for (int j = 0; j < K1; ++j) {
    val[j] = -INFINITY;
    idx[j] = 0x7fffffff;
  }
  bool finite = true;   // a non-finite input row (NaN logits) still selects valid ids, never refined
  // the row (16-byte aligned, E <= padded width, a multiple of 16) is read 16
  // logits at a time with independent LDS.128: one shared-memory latency per 16
  // insertions instead of one per logit (the MIO queue is busy with the xn warps)
  for (int e0 = 0; e0 < E; e0 += 16) {
    float vv[16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 q = *reinterpret_cast<const float4*>(lg + e0 + 4 * u);
      vv[4 * u] = q.x;
      vv[4 * u + 1] = q.y;
      vv[4 * u + 2] = q.z;
      vv[4 * u + 3] = q.w;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = e0 + u;
      float v = e < E ? vv[u] : -INFINITY;
      if (e < E && !(fabsf(v) <= FLT_MAX)) {
        finite = false;
        v = -FLT_MAX;
      }
      if (v > val[K1 - 1]) {
        bool gt[K1];
#pragma unroll
        for (int j = 0; j < K1; ++j) gt[j] = v > val[j];
#pragma unroll
        for (int j = K1 - 1; j >= 1; --j) {
          if (gt[j]) {
            val[j] = gt[j - 1] ? val[j - 1] : v;
            idx[j] = gt[j - 1] ? idx[j - 1] : e;
          }
        }
        if (gt[0]) {
          val[0] = v;
          idx[0] = e;
        }
      }
    }
  }
#ifndef FSC_ROUTER_PROF
  if (L.logits)
    for (int e = 0; e < E; ++e) L.logits[t * E + e] = lg[e];
#endif
  const float vk = val[k - 1], vk1 = k < E ? val[k] : -FLT_MAX;
  const float thr2 = 2.f * B + 4.f * kU * (fabsf(vk) + fabsf(vk1)) + 1e-7f;
  if (finite && k < E && vk - vk1 <= thr2) {   // ambiguous boundary: refined by the block (refine_block)
    if (L.n_refined) atomicAdd(L.n_refined, 1);
    rs.flag[tt] = 1;
    rs.thr[tt][0] = thr2;
    rs.thr[tt][1] = vk;
    rs.thr[tt][2] = vk1;
    return;
  }
  const float vtop = val[0];
  float ex[K1], sum = 0.f;
#pragma unroll
  for (int j = 0; j < K1; ++j) {
    ex[j] = j < k ? expf(val[j] - vtop) : 0.f;
    sum += ex[j];
  }
#pragma unroll
  for (int j = 0; j < K1; ++j) {
    if (j < k) {
      int rank = 0;
#pragma unroll
      for (int i = 0; i < K1; ++i) rank += (i < k && idx[i] < idx[j]) ? 1 : 0;
      L.topk_idx[t * k + rank] = idx[j];
      L.topk_w[t * k + rank] = ex[j] / sum;
    }
  }
}

// xn = bf16(x gamma r) for the block's rows (rows were just streamed: L2 hits);
// loads are issued in batches of 8 per thread to keep enough bytes in flight.
FSC_DEVINL void write_xn(const RouterLaunch& L, long t0, int rows, const float* s_r, int tid, int nt) {
  const int d = L.d;
  const int dv = d / 4;
  const int n = rows * dv;
  const float4* g4 = reinterpret_cast<const float4*>(L.gamma);
  const float4* x4 = reinterpret_cast<const float4*>(L.x + t0 * d);
  uint2* o2 = reinterpret_cast<uint2*>(L.xn + t0 * d);
  for (int base = tid; base < n; base += 8 * nt) {
    float4 v[8], g[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * nt;
      if (i < n) {
        v[u] = x4[i];
        g[u] = g4[i % dv];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * nt;
      if (i < n) {
        const float r = s_r[i / dv];
        o2[i] = make_uint2(pack_bf16x2(v[u].x * g[u].x * r, v[u].y * g[u].y * r),
                           pack_bf16x2(v[u].z * g[u].z * r, v[u].w * g[u].w * r));
      }
    }
  }
}

#ifdef FSC_ROUTER_PROF
#define RSTAMP(kk)                                                                   \
  if (tid == 0) {                                                                    \
    unsigned long long g__;                                                          \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g__));                          \
    reinterpret_cast<unsigned long long*>(L.logits)[blockIdx.x * 8 + (kk)] = g__;    \
  }
#define I8STAMP(kk)                                                                                  \
  if (threadIdx.x == 64) {                                                                           \
    unsigned long long g__;                                                                          \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g__));                                          \
    reinterpret_cast<unsigned long long*>(L.logits)[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + (kk)] = g__; \
  }
#else
#define RSTAMP(kk)
#define I8STAMP(kk)
#endif

// Band refinement of the block's flagged tokens, by the whole CTA (after the
// selection, so the fp32 logits rows are in shared memory). For each flagged token:
// warp 0 classifies the experts against the token's fp32 band (certainly in / band /
// certainly out); the 8 warps compute the fp64 raw dots sum_i x_i gamma_i W_ei of
// the band experts, one warp per expert (the positive factor r_t does not change
// their order; x_i gamma_i is exact in fp64); warp 0 fills the k - |certain| open
// slots with the best band experts (fp64 value, ties -> lower id) and writes the
// indices and gates (from the fp32 logits, as for every other token).
template <int QN, class RS>
FSC_DEVINL void refine_block(const RouterLaunch& L, const float* lg, int lgs, RS& rs, long t0, int rows) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int d = L.d, E = L.E, k = L.k;
  for (int tt = 0; tt < rows; ++tt) {
    if (!rs.flag[tt]) continue;                  // block-uniform
    const long t = t0 + tt;
    const float* row = lg + tt * lgs;
    const float thr2 = rs.thr[tt][0], hi = rs.thr[tt][1], lo = rs.thr[tt][2];
    float v[QN];
    uint32_t sel = 0, band = 0;
    if (warp == 0) {
      int nb = 0;
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        const int e = lane + 32 * q;
        v[q] = e < E ? row[e] : -FLT_MAX;
        const bool in = e < E && v[q] > hi + thr2;
        const bool bnd = e < E && !in && !(v[q] < lo - thr2);
        if (in) sel |= 1u << q;
        if (bnd) band |= 1u << q;
        const uint32_t m = __ballot_sync(0xffffffff, bnd);
        if (bnd) rs.band[nb + __popc(m & ((1u << lane) - 1u))] = e;
        nb += __popc(m);
      }
      if (lane == 0) rs.nb = nb;
    }
    __syncthreads();
    const int nb = rs.nb;
    const float4* x4 = reinterpret_cast<const float4*>(L.x + t * d);
    const float4* g4 = reinterpret_cast<const float4*>(L.gamma);
    for (int b = warp; b < nb; b += nwarps) {
      const int e = rs.band[b];
      const float4* w4 = reinterpret_cast<const float4*>(L.w_router + (long)e * d);
      double a0 = 0.0, a1 = 0.0;
      for (int c0 = lane; c0 < d / 4; c0 += 128) {   // 4 float4 of each operand in flight
        float4 xv[4], gv[4], wv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + 32 * u;
          const bool ok = c < d / 4;
          xv[u] = ok ? x4[c] : make_float4(0.f, 0.f, 0.f, 0.f);
          gv[u] = ok ? g4[c] : make_float4(0.f, 0.f, 0.f, 0.f);
          wv[u] = ok ? w4[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a0 = fma((double)xv[u].x * (double)gv[u].x, (double)wv[u].x, a0);
          a1 = fma((double)xv[u].y * (double)gv[u].y, (double)wv[u].y, a1);
          a0 = fma((double)xv[u].z * (double)gv[u].z, (double)wv[u].z, a0);
          a1 = fma((double)xv[u].w * (double)gv[u].w, (double)wv[u].w, a1);
        }
      }
      const double sum = warp_sum_f64(a0 + a1);
      if (lane == 0) rs.l64[e] = sum;
    }
    __syncthreads();
    if (warp == 0) {
      double l64[QN];
#pragma unroll
      for (int q = 0; q < QN; ++q) l64[q] = ((band >> q) & 1u) ? rs.l64[lane + 32 * q] : -DBL_MAX;
      int nsel = 0;
#pragma unroll
      for (int q = 0; q < QN; ++q) nsel += __popc(__ballot_sync(0xffffffff, (sel >> q) & 1u));
      for (int rd = nsel; rd < k; ++rd) {
        double bv = -DBL_MAX;
        int bi = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < QN; ++q) {
          const int e = lane + 32 * q;
          if (((band >> q) & 1u) && !((sel >> q) & 1u) && (l64[q] > bv || (l64[q] == bv && e < bi))) {
            bv = l64[q];
            bi = e;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffff, bv, o);
          const int oi = __shfl_xor_sync(0xffffffff, bi, o);
          if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        if (bi != 0x7fffffff && (bi & 31) == lane) sel |= 1u << (bi >> 5);
      }
      float vtop = -FLT_MAX;
#pragma unroll
      for (int q = 0; q < QN; ++q)
        if ((sel >> q) & 1u) vtop = fmaxf(vtop, v[q]);
      vtop = warp_max_f32(vtop);
      float ex[QN], sum = 0.f;
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        ex[q] = ((sel >> q) & 1u) ? expf(v[q] - vtop) : 0.f;
        sum += ex[q];
      }
      sum = warp_sum_f32(sum);
      int slot = 0;
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        const uint32_t m = __ballot_sync(0xffffffff, (sel >> q) & 1u);
        if ((sel >> q) & 1u) {
          const int s = slot + __popc(m & ((1u << lane) - 1u));
          L.topk_idx[t * k + s] = lane + 32 * q;
          L.topk_w[t * k + s] = ex[q] / sum;
        }
        slot += __popc(m);
      }
    }
  }
}

// Epilogue of one block of <= 32 tokens whose fp32 logits lg[tt][e] (row stride
// 32*EW + 4) and RMS factors are in shared memory: warp 0 selects (one thread per
// token) while warps 1-7 write xn; for k > 8 warps 0-3 select (one warp per token)
// and warps 4-7 write xn. Then the CTA refines the flagged tokens in fp64.
// `chain` bounds the rounding chain of every logit. rs.flag must be zero on entry.
template <int EW>
FSC_DEVINL void router_select_and_xn(const RouterLaunch& L, const float* lg, const float* s_r, const float* s_xn,
                                     const float* s_wsq, RefineSmem& rs, long t0, int rows, float chain) {
  constexpr int LGS = 32 * EW + 4, NT = 256;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float wm = 0.f;
  for (int e = lane; e < L.E; e += 32) wm = fmaxf(wm, s_wsq[e]);
  const float wmax = sqrtf(warp_max_f32(wm)) * 1.01f;
  if (L.k < kThreadSelK1) {
    if (warp == 0) {
      if (lane < rows) {
        const float* row = lg + lane * LGS;
        const float B = s_r[lane] * chain * kU * s_xn[lane] * wmax;
        const long t = t0 + lane;
        switch (L.k) {
          case 1: select_token_thread<2>(row, t, lane, B, L, rs); break;
          case 2: select_token_thread<3>(row, t, lane, B, L, rs); break;
          case 3: select_token_thread<4>(row, t, lane, B, L, rs); break;
          case 4: select_token_thread<5>(row, t, lane, B, L, rs); break;
          case 5: select_token_thread<6>(row, t, lane, B, L, rs); break;
          case 6: select_token_thread<7>(row, t, lane, B, L, rs); break;
          case 7: select_token_thread<8>(row, t, lane, B, L, rs); break;
          default: select_token_thread<9>(row, t, lane, B, L, rs); break;
        }
      }
    } else {
      write_xn(L, t0, rows, s_r, tid - 32, NT - 32);
    }
  } else if (warp < 4) {
    for (int tt = warp; tt < rows; tt += 4)
      select_token<EW>(lg + tt * LGS, t0 + tt, tt, s_r[tt] * chain * kU * s_xn[tt] * wmax, L, rs, lane);
  } else {
    write_xn(L, t0, rows, s_r, tid - 128, 128);
  }
  __syncthreads();
  refine_block<EW>(L, lg, LGS, rs, t0, rows);
}

// Main kernel: 8 warps = KS k-groups x NEH expert halves of 64 (E <= 64 is padded
// to 64 with zero W' columns, masked in the selection). Each lane owns 8 tokens
// (lt + 4i) x 4 expert pairs (2 le + 16 j + {0,1}); x is staged token-major, W'
// k-major, so one LDS.64 yields an expert pair at one k and every product is an
// FFMA2 with the token value broadcast (full fp32 issue rate on sm_100).
// gridDim.y = nsplit > 1 (small T, decode): block (x, y) covers the y-th 1/nsplit of
// d and writes raw partial dots + partial sum x^2 to L.part / L.part_sq;
// router_finish_kernel sums the splits in a fixed order and selects.
template <int EW>
__global__ void __launch_bounds__(256, 2) router_kernel(RouterLaunch L) {
  constexpr int EP = 32 * EW;          // padded experts: 32, 64 or 128
  constexpr int NEH = EP >= 64 ? EP / 64 : 1;   // 64-expert halves
  constexpr int NJ = EP >= 64 ? 4 : EP / 16;    // expert pairs per lane (2 le + 16 j)
  constexpr int KS = 8 / NEH;          // k-groups (warps sharing a chunk)
  constexpr int KW = DC / KS;          // k per warp per chunk (8 or 16)
  constexpr int NT = 256;
  constexpr int XV = TB * DC / 4 / NT; // float4 of the x chunk per thread (2)
  constexpr int WV = EP * DC / 4 / NT; // float4 of the W' chunk per thread (2 / 4 / 8)
  constexpr int XBUF = TB * LDS;       // x chunk, token-major [TB][LDS]
  constexpr int BUF = XBUF + DC * EP;  // + W' chunk, k-major [DC][EP]
  constexpr int NS = EW >= 4 ? 2 : 4;  // cp.async pipeline depth (E=128: 2 stages -> 2 CTAs/SM)
  constexpr int LGS = EP + 4;          // logits row stride: float4 rows, conflict-free LDS.128 across rows
  static_assert(KS * TB * EP + TB * LGS <= NS * BUF, "partials + logits must fit in the stages");
  extern __shared__ __align__(16) float sm[];
  float* stage0 = sm;                  // [NS][BUF]
  float* red = sm;                     // [KS][TB][EP] k-group partials (after the loop)
  float* lg = sm + KS * TB * EP;       // [TB][LGS] fp32 logits (16-byte rows)
  float* s_r = sm + NS * BUF;          // [TB]
  float* s_xn = s_r + TB;              // [TB] ||x_t||
  float* s_wsq = s_xn + TB;            // [EP]
  __shared__ RefineSmem rs;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = L.d;
  if (tid < TB) rs.flag[tid] = 0;
  const long t0 = (long)blockIdx.x * L.rpb;    // rpb <= TB rows per block (balanced grid)
  const int rows = (int)min((long)L.rpb, (long)L.T - t0);
  const long T = t0 + rows;                    // rows >= T are padding
  const int nsplit = gridDim.y, split = blockIdx.y;
  const int nch_all = d / DC;
  const int ch0 = split * nch_all / nsplit, nch = (split + 1) * nch_all / nsplit - ch0;
  const float* __restrict__ x = L.x;
  const float* __restrict__ WT = L.w_scaled;   // [d][EP]
  RSTAMP(0);
  auto issue_chunk = [&](int c0, float* buf) {
#pragma unroll
    for (int v = 0; v < XV; ++v) {
      const int i = tid + v * NT;
      const int tt = i / (DC / 4), cc = (i % (DC / 4)) * 4;
      const long t = t0 + tt;
      cp_async16(buf + tt * LDS + cc, x + (t < T ? t : 0) * d + c0 + cc, t < T);
    }
#pragma unroll
    for (int v = 0; v < WV; ++v) {
      const int i = tid + v * NT;       // float4 index inside the [DC][EP] chunk
      cp_async16(buf + XBUF + 4 * i, WT + (long)c0 * EP + 4 * i, true);
    }
    cp_async_commit();
  };
  auto chunk = [&](int i) { return ch0 + i; };
#pragma unroll
  for (int i = 0; i < NS - 1; ++i) {
    if (i < nch) issue_chunk(chunk(i) * DC, stage0 + i * BUF);
    else cp_async_commit();
  }
  if (nsplit == 1)
    for (int e = tid; e < EP; e += NT) s_wsq[e] = e < L.E ? L.w_sq[e] : 0.f;

  const int eh = warp % NEH, ks = warp / NEH, lt = lane >> 3, le = lane & 7;
  float2 acc[8][NJ];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j] = make_float2(0.f, 0.f);
  double ssp = 0.0;                     // partial sum x^2 of row tid/8 (8 values per chunk)
  const int srow = tid >> 3, scol = (tid & 7) * 8;

  for (int it = 0; it < nch; ++it) {
    const float* buf = stage0 + (it % NS) * BUF;
    cp_async_wait<NS - 2>();
    __syncthreads();
    if (it + NS - 1 < nch) issue_chunk(chunk(it + NS - 1) * DC, stage0 + ((it + NS - 1) % NS) * BUF);
    else cp_async_commit();
    {
      const float4 p = *reinterpret_cast<const float4*>(buf + srow * LDS + scol);
      const float4 q = *reinterpret_cast<const float4*>(buf + srow * LDS + scol + 4);
      ssp += ((double)p.x * p.x + (double)p.y * p.y) + ((double)p.z * p.z + (double)p.w * p.w) +
             ((double)q.x * q.x + (double)q.y * q.y) + ((double)q.z * q.z + (double)q.w * q.w);
    }
    const float* xa = buf + lt * LDS + ks * KW;
    const float* wb = buf + XBUF + (ks * KW) * EP + eh * 64 + 2 * le;
#pragma unroll
    for (int kk = 0; kk < KW; kk += 2) {
      float2 a[8], b0[NJ], b1[NJ];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float2*>(xa + 4 * i * LDS + kk);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        b0[j] = *reinterpret_cast<const float2*>(wb + kk * EP + 16 * j);
        b1[j] = *reinterpret_cast<const float2*>(wb + (kk + 1) * EP + 16 * j);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          ffma2_bcast(acc[i][j], a[i].x, b0[j]);
          ffma2_bcast(acc[i][j], a[i].y, b1[j]);
        }
    }
  }
  __syncthreads();                       // stages free: reuse for the k-group partials
  RSTAMP(1);
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
      *reinterpret_cast<float2*>(&red[(ks * TB + lt + 4 * i) * EP + eh * 64 + 2 * le + 16 * j]) = acc[i][j];
  // per-row sum x^2: the 8 threads of a row are consecutive lanes
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) ssp += __shfl_xor_sync(0xffffffff, ssp, o);
  if (nsplit > 1) {                      // raw partials of this d-split (the finish kernel selects)
    if ((tid & 7) == 0 && srow < rows) L.part_sq[(long)split * L.T + t0 + srow] = ssp;
    __syncthreads();
    for (int i = tid; i < rows * EP; i += NT) {
      const int tt = i / EP, e = i % EP;
      float s = red[tt * EP + e];
#pragma unroll
      for (int g = 1; g < KS; ++g) s += red[(g * TB + tt) * EP + e];
      L.part[((long)split * L.T + t0 + tt) * EP + e] = s;
    }
    return;
  }
  if ((tid & 7) == 0) {
    s_r[srow] = (float)(1.0 / sqrt(ssp / (double)d + (double)L.eps));
    s_xn[srow] = (float)sqrt(ssp) * 1.0001f;
  }
  __syncthreads();
  for (int i = tid; i < TB * EP; i += NT) {   // k-groups summed in a fixed order
    const int tt = i / EP, e = i % EP;
    float s = red[tt * EP + e];
#pragma unroll
    for (int g = 1; g < KS; ++g) s += red[(g * TB + tt) * EP + e];
    lg[tt * LGS + e] = s * s_r[tt];
  }
  __syncthreads();
  RSTAMP(2);
  router_select_and_xn<EW>(L, lg, s_r, s_xn, s_wsq, rs, t0, rows, (float)(d / KS + KS + 6));
  RSTAMP(3);
  __syncthreads();
  RSTAMP(4);
}

// Split-d finish: logit = r * (sum over splits, in split order, of the raw partials),
// r from the split partial sums of x^2 (fp64, split order); then the same selection
// and xn write as the single-pass kernel. Rounding chain: d/(nsplit KS) + KS + nsplit.
template <int EW>
__global__ void __launch_bounds__(256) router_finish_kernel(RouterLaunch L, int nsplit, float chain) {
  constexpr int EP = 32 * EW, LGS = EP + 4, NT = 256;
  __shared__ __align__(16) float lg[TB * LGS];
  __shared__ float s_r[TB], s_xn[TB], s_wsq[EP];
  __shared__ RefineSmem rs;
  const int tid = threadIdx.x;
  if (tid < TB) rs.flag[tid] = 0;
  const long t0 = (long)blockIdx.x * L.rpb;
  const int rows = (int)min((long)L.rpb, (long)L.T - t0);
  for (int e = tid; e < EP; e += NT) s_wsq[e] = e < L.E ? L.w_sq[e] : 0.f;
  if (tid < rows) {                       // all split partials in flight, summed in split order
    double q[kMaxSplit];
#pragma unroll
    for (int sp = 0; sp < kMaxSplit; ++sp) q[sp] = sp < nsplit ? L.part_sq[(long)sp * L.T + t0 + tid] : 0.0;
    double ssp = q[0];
#pragma unroll
    for (int sp = 1; sp < kMaxSplit; ++sp)
      if (sp < nsplit) ssp += q[sp];
    s_r[tid] = (float)(1.0 / sqrt(ssp / (double)L.d + (double)L.eps));
    s_xn[tid] = (float)sqrt(ssp) * 1.0001f;
  }
  __syncthreads();
  for (int i0 = tid; i0 < rows * EP; i0 += 4 * NT) {   // 4 items x nsplit partials in flight per thread
    float v[4][kMaxSplit];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * NT;
      const float* pp = L.part + (t0 + i / EP) * EP + i % EP;
#pragma unroll
      for (int sp = 0; sp < kMaxSplit; ++sp)
        v[u][sp] = (i < rows * EP && sp < nsplit) ? pp[(long)sp * L.T * EP] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * NT;
      if (i >= rows * EP) break;
      float sacc = v[u][0];
#pragma unroll
      for (int sp = 1; sp < kMaxSplit; ++sp)
        if (sp < nsplit) sacc += v[u][sp];
      lg[(i / EP) * LGS + i % EP] = sacc * s_r[i / EP];
    }
  }
  __syncthreads();
  router_select_and_xn<EW>(L, lg, s_r, s_xn, s_wsq, rs, t0, rows, chain);
}

// ============================================================================
// Exact int8 tensor-core router (E <= 128, d % 128 == 0, k <= 8).
//
// Fixed point, exactly: with s_t, s_e powers of two (|x_t| / s_t < 1, |w_e| / s_e < 1,
// w_e = gamma (.) W_R[e] formed exactly in fp64), truncating base-2^7 digits give
//   x_t / s_t = sum_{i<3} a_i 2^{-7(i+1)} + dx,   w_e / s_e = sum_{j<3} b_j 2^{-7(j+1)} + dw,
// a_i, b_j in [-127, 127] (int8), |dx|, |dw| < 2^-21 per element. Then
//   l_te = r_t s_t s_e ( sum_{i+j<=3} 2^{-7(i+j+2)} <a_i, b_j>  + err ),
//   |err| <= 2^-21 (||x_t/s_t||_1 + ||w_e/s_e||_1 + 2d 2^-21) + d 2^-42 + 2^-42 127^2 d
// where every <a_i, b_j> is an exact int32 tensor-core sum (|.| <= 127^2 d), pairs with
// equal i + j share one TMEM accumulator (4 x EP columns) and the one dropped pair
// (2, 2) is bounded by the last term. That bound (~2e-4 of the logit scale, vs ~7e-4
// for the fp32 SIMT chain) decides the band exactly as in the SIMT path; flagged
// tokens go through the same fp64 refine_block. One CTA = 128 tokens (TMEM lanes) x
// EP (64 or 128) padded experts x a 1/nsplit slice of d: warp 0 TMA (ring of 3 + 3
// planes), warp 1 MMA (8 plane pairs x 4 K-steps of 32 per 128-wide k-block), warps
// 2-5 epilogue (one thread per token). nsplit > 1 (to fill the SMs): each CTA writes
// its int32 partial sums, column-major [split][column][token] so that a warp's stores
// and loads are 128-byte rows; the last CTA of a token block (ticket) adds them -
// integer sums, so exact and order-free - then combines in fp64, selects and refines.
namespace {
constexpr int I8_BM = 128, I8_BK = 128, I8_NP = 3, I8_NACC = 2 * I8_NP - 2;   // 4 accumulators
constexpr int I8_A_TILE = I8_BM * I8_BK;                    // 16 KB
constexpr int I8_THREADS = 192;
constexpr int I8_MAX_SPLIT = 8;
template <int EP>
struct I8Cfg {
  static constexpr int B_TILE = EP * I8_BK;                 // 8 / 16 KB
  static constexpr int STAGE = I8_NP * (I8_A_TILE + B_TILE); // 72 / 96 KB
  static constexpr int STAGES = EP == 64 ? 3 : 2;
  static constexpr int LGS = EP + 4;
  static constexpr int ACC_COLS = I8_NACC * EP;             // 256 / 512 int32 per token
  static constexpr int SMEM = 1024 + STAGES * STAGE + 256;
  static_assert(I8_BM * LGS * 4 <= STAGES * STAGE, "logits must fit in the stages");
};

template <typename F>
FSC_DEVINL void split3(F v, int8_t (&q)[I8_NP]) {   // |v| < 1: truncating base-128 digits, exact
#pragma unroll
  for (int i = 0; i < I8_NP; ++i) {
    v *= (F)128;
    const F t = trunc(v);
    q[i] = (int8_t)(int)t;
    v -= t;
  }
}

// xn + planes of 4 consecutive columns of one token (c = float4 index)
FSC_DEVINL float quant_store4(const RouterLaunch& L, long t, int c, float4 v, float4 g, float rf, float inv) {
  uint2* xo = reinterpret_cast<uint2*>(L.xn + t * L.d);
  xo[c] = make_uint2(pack_bf16x2(v.x * g.x * rf, v.y * g.y * rf), pack_bf16x2(v.z * g.z * rf, v.w * g.w * rf));
  int8_t q0[I8_NP], q1[I8_NP], q2[I8_NP], q3[I8_NP];
  split3(v.x * inv, q0);
  split3(v.y * inv, q1);
  split3(v.z * inv, q2);
  split3(v.w * inv, q3);
#pragma unroll
  for (int i = 0; i < I8_NP; ++i) {
    const uint32_t pk = (uint32_t)(uint8_t)q0[i] | ((uint32_t)(uint8_t)q1[i] << 8) |
                        ((uint32_t)(uint8_t)q2[i] << 16) | ((uint32_t)(uint8_t)q3[i] << 24);
    reinterpret_cast<uint32_t*>(L.i8_x + ((long)i * L.T + t) * L.d)[c] = pk;
  }
  return (fabsf(v.x) + fabsf(v.y) + fabsf(v.z) + fabsf(v.w)) * inv;
}
}  // namespace

// Per token (one warp): r_t, s_t, ||x_t/s_t||_1, xn = bf16(x gamma r) and the planes of x_t/s_t.
// NV > 0: the row stays in registers (d = 128 NV, one read of x); NV = 0: two passes over x.
template <int NV>
__global__ void __launch_bounds__(256) router_i8_quant_x_kernel(RouterLaunch L) {
  const int lane = threadIdx.x & 31;
  const long t = (long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= L.T) return;
  const int d = L.d, dv = d / 4;
  const float4* x4 = reinterpret_cast<const float4*>(L.x + t * d);
  const float4* g4 = reinterpret_cast<const float4*>(L.gamma);
  double ss = 0.0;
  float mx = 0.f;
  float4 row[NV > 0 ? NV : 1];
  if (NV > 0) {
#pragma unroll
    for (int u = 0; u < NV; ++u) row[u] = __ldcs(x4 + lane + 32 * u);
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const float4 v = row[u];
      ss += ((double)v.x * v.x + (double)v.y * v.y) + ((double)v.z * v.z + (double)v.w * v.w);
      mx = fmaxf(fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y))), fmaxf(fabsf(v.z), fabsf(v.w)));
    }
  } else {
    for (int c0 = lane; c0 < dv; c0 += 128) {           // 4 float4 per lane in flight
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = c0 + 32 * u < dv ? x4[c0 + 32 * u] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ss += ((double)v[u].x * v[u].x + (double)v[u].y * v[u].y) + ((double)v[u].z * v[u].z + (double)v[u].w * v[u].w);
        mx = fmaxf(fmaxf(mx, fmaxf(fabsf(v[u].x), fabsf(v[u].y))), fmaxf(fabsf(v[u].z), fabsf(v[u].w)));
      }
    }
  }
  ss = warp_sum_f64(ss);
  mx = warp_max_f32(mx);
  const double r = 1.0 / sqrt(ss / (double)d + (double)L.eps);
  const float rf = (float)r;
  int ex = 0;
  frexpf(mx, &ex);                                   // mx = m 2^ex, m in [0.5, 1)
  const float st = mx > 0.f ? ldexpf(1.f, ex) : 1.f;  // |x| / st < 1
  const float inv = 1.f / st;                        // exact (power of two)
  float l1 = 0.f;
  if (NV > 0) {
#pragma unroll
    for (int u = 0; u < NV; ++u) l1 += quant_store4(L, t, lane + 32 * u, row[u], __ldg(g4 + lane + 32 * u), rf, inv);
  } else {
    for (int c0 = lane; c0 < dv; c0 += 128) {
      float4 v[4], g[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool ok = c0 + 32 * u < dv;
        v[u] = ok ? x4[c0 + 32 * u] : make_float4(0.f, 0.f, 0.f, 0.f);
        g[u] = ok ? g4[c0 + 32 * u] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 32 * u;
        if (c >= dv) break;
        l1 += quant_store4(L, t, c, v[u], g[u], rf, inv);
      }
    }
  }
  l1 = warp_sum_f32(l1);
  if (lane == 0) {
    L.i8_tok[t] = st;
    L.i8_tok[L.T + t] = l1 * 1.0001f + 1e-6f;          // rounding of the fp32 sum, upward
    L.i8_tok[2 * L.T + t] = rf;
    L.i8_r[t] = r;
  }
}

// Per padded expert (one CTA): w = gamma (.) W_R[e] exactly in fp64, s_e, the planes of
// w / s_e and the per-expert error-bound coefficients; zero planes for e >= E.
__global__ void __launch_bounds__(256) router_i8_quant_w_kernel(RouterLaunch L, int EP) {
  __shared__ double red_l1[8];
  __shared__ float red_mx[8];
  const int e = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = L.d;
  float mx = 0.f;
  if (e < L.E)
    for (int c = tid; c < d; c += 256)
      mx = fmaxf(mx, (float)fabs((double)L.gamma[c] * (double)L.w_router[(long)e * d + c]));
  mx = warp_max_f32(mx);
  if (lane == 0) red_mx[warp] = mx;
  __syncthreads();
  mx = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) mx = fmaxf(mx, red_mx[w]);
  // (float)|w| may round up to the next power of two: frexp of the rounded max is then
  // one binade higher, which still satisfies |w| / s_e < 1
  int ex = 0;
  frexpf(mx, &ex);
  const double se = mx > 0.f ? ldexp(1.0, ex) : 1.0;
  const double inv = 1.0 / se;
  double l1 = 0.0;
  for (int c = tid; c < d; c += 256) {
    int8_t q[I8_NP] = {};
    if (e < L.E) {
      const double v = (double)L.gamma[c] * (double)L.w_router[(long)e * d + c] * inv;
      split3(v, q);
      l1 += fabs(v);
    }
#pragma unroll
    for (int j = 0; j < I8_NP; ++j) L.i8_w[((long)j * EP + e) * d + c] = q[j];
  }
  l1 = warp_sum_f64(l1);
  if (lane == 0) red_l1[warp] = l1;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int w = 0; w < 8; ++w) tot += red_l1[w];
    const double u21 = ldexp(1.0, -21), u42 = ldexp(1.0, -42);
    L.i8_exp[e] = (float)se;
    L.i8_exp[EP + e] = e < L.E ? (float)(se * u21 * 1.0001) : 0.f;
    L.i8_exp[2 * EP + e] =
        e < L.E ? (float)(se * (u21 * (tot * 1.0001 + 2.0 * d * u21) + d * u42 + u42 * 127.0 * 127.0 * d) * 1.0001)
                : 0.f;
  }
}

template <int EP>
__global__ void __launch_bounds__(I8_THREADS, 1)
    router_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, RouterLaunch L) {
  using C = I8Cfg<EP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                        // [stage][plane][128][128]
  uint8_t* sB = smem + C::STAGES * I8_NP * I8_A_TILE;        // [stage][plane][EP][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tfull + 1);
  int* s_last = reinterpret_cast<int*>(s_tmem + 1);
  float* lg = reinterpret_cast<float*>(smem);                // [128][LGS] after the MMAs (stages free)
  __shared__ RefineSmemT<I8_BM> rs;
  const int tid = threadIdx.x, lane = tid & 31, warp = warp_id();
  const int blk = blockIdx.x, nsplit = gridDim.y, split = blockIdx.y;
  const long t0 = (long)blk * I8_BM;
  const int rows = (int)min((long)I8_BM, (long)L.T - t0);
  const int nkb = L.d / I8_BK;
  const int kb0 = split * nkb / nsplit, kb1 = (split + 1) * nkb / nsplit;
  if (tid < I8_BM) rs.flag[tid] = 0;
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int st = 0; st < C::STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  } else if (warp == 1) {
    tmem_alloc<C::ACC_COLS>(s_tmem);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  I8STAMP(0);
  if (warp == 0) {
    if (elect_one()) {                                     // TMA producer
      int st = 0;
      uint32_t ph = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], C::STAGE);
#pragma unroll
        for (int i = 0; i < I8_NP; ++i)
          tma_load_2d(sA + (st * I8_NP + i) * I8_A_TILE, &tmA, &full[st], kb * I8_BK, (int)(i * L.T + t0),
                      kEvictNormal);
#pragma unroll
        for (int j = 0; j < I8_NP; ++j)
          tma_load_2d(sB + (st * I8_NP + j) * C::B_TILE, &tmB, &full[st], kb * I8_BK, j * EP, kEvictLast);
        if (++st == C::STAGES) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {                                     // MMA issuer
      const uint32_t idesc = idesc_s8_s32(I8_BM, EP);
      int st = 0;
      uint32_t ph = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[st], ph);
        tc_fence_after();
        uint32_t touched = kb > kb0 ? 0xFu : 0u;
#pragma unroll
        for (int i = 0; i < I8_NP; ++i)
#pragma unroll
          for (int j = 0; j < I8_NP; ++j) {
            if (i + j >= I8_NACC) continue;               // the dropped pair (2, 2)
            const uint32_t a = smem_u32(sA + (st * I8_NP + i) * I8_A_TILE);
            const uint32_t b = smem_u32(sB + (st * I8_NP + j) * C::B_TILE);
#pragma unroll
            for (int kk = 0; kk < I8_BK / 32; ++kk)
              umma_s8_ss(tmem + (i + j) * EP, umma_desc_sw128(a + kk * 32), umma_desc_sw128(b + kk * 32), idesc,
                         (kk > 0 || ((touched >> (i + j)) & 1u)) ? 1u : 0u);
            touched |= 1u << (i + j);
          }
        umma_commit(&empty[st]);
        if (++st == C::STAGES) { st = 0; ph ^= 1; }
      }
      umma_commit(tfull);
    }
  } else if (nsplit > 1) {                                 // warps 2-5: write this split's int32 partials
    mbar_wait(tfull, 0);
    tc_fence_after();
    I8STAMP(1);
    const int q = warp & 3, row = q * 32 + lane;
    const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16);
    int* dst = L.i8_part + (long)split * C::ACC_COLS * L.T + t0 + row;   // column-major: token fastest
#pragma unroll 1
    for (int c = 0; c < C::ACC_COLS; c += 16) {
      uint32_t S[16];
      tmem_ld16(tb + c, S);
      tmem_ld_wait();
      if (row < rows)
#pragma unroll
        for (int u = 0; u < 16; ++u) __stcg(dst + (long)(c + u) * L.T, (int)S[u]);
    }
  }
  tc_fence_before();
  if (nsplit > 1) {                                        // last CTA of the token block finishes it
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const int prev = atomicAdd(L.i8_cnt + blk, 1);
      *s_last = prev == nsplit - 1;
      if (prev == nsplit - 1) L.i8_cnt[blk] = 0;
    }
    __syncthreads();
    I8STAMP(2);
    if (!*s_last) {
      if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::ACC_COLS>(tmem);
      }
      return;
    }
    __threadfence();
  }
  if (warp >= 2) {                                         // combine in fp64 (thread = token)
    if (nsplit == 1) {
      mbar_wait(tfull, 0);
      tc_fence_after();
    }
    const int q = warp & 3, row = q * 32 + lane;
    const long t = t0 + row;
    const bool valid = row < rows;
    const double sc = valid ? L.i8_r[t] * (double)L.i8_tok[t] : 0.0;
    const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
    for (int e0 = 0; e0 < EP; e0 += 16) {
      int S[I8_NACC][16];
      if (nsplit == 1) {
#pragma unroll
        for (int a = 0; a < I8_NACC; ++a) tmem_ld16(tb + a * EP + e0, reinterpret_cast<uint32_t(&)[16]>(S[a]));
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int a = 0; a < I8_NACC; ++a)
#pragma unroll
          for (int u = 0; u < 16; ++u) S[a][u] = 0;
        if (valid)
          for (int sp = 0; sp < nsplit; ++sp) {
            const int* src = L.i8_part + (long)sp * C::ACC_COLS * L.T + t;
#pragma unroll
            for (int a = 0; a < I8_NACC; ++a)
#pragma unroll
              for (int u = 0; u < 16; ++u) S[a][u] += __ldcg(src + (long)(a * EP + e0 + u) * L.T);
          }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const double v = (double)S[0][u] * 0x1p-14 + (double)S[1][u] * 0x1p-21 + (double)S[2][u] * 0x1p-28 +
                         (double)S[3][u] * 0x1p-35;
        lg[row * C::LGS + e0 + u] = (float)(sc * (double)L.i8_exp[e0 + u] * v);
      }
    }
  }
  tc_fence_before();
  __syncthreads();                                         // all logits in shared memory
  I8STAMP(3);
  if (warp >= 2) {
    const int q = warp & 3, row = q * 32 + lane;
    if (row < rows) {
      const long t = t0 + row;
      const float l1x = L.i8_tok[L.T + t];
      float bmax = 0.f;
      for (int e = 0; e < L.E; ++e) bmax = fmaxf(bmax, fmaf(L.i8_exp[EP + e], l1x, L.i8_exp[2 * EP + e]));
      const float B = (float)(L.i8_r[t] * (double)L.i8_tok[t] * (double)bmax * 1.0001) + 1e-12f;
      const float* rowp = lg + row * C::LGS;
      switch (L.k) {
        case 1: select_token_thread<2>(rowp, t, row, B, L, rs); break;
        case 2: select_token_thread<3>(rowp, t, row, B, L, rs); break;
        case 3: select_token_thread<4>(rowp, t, row, B, L, rs); break;
        case 4: select_token_thread<5>(rowp, t, row, B, L, rs); break;
        case 5: select_token_thread<6>(rowp, t, row, B, L, rs); break;
        case 6: select_token_thread<7>(rowp, t, row, B, L, rs); break;
        case 7: select_token_thread<8>(rowp, t, row, B, L, rs); break;
        default: select_token_thread<9>(rowp, t, row, B, L, rs); break;
      }
    }
  }
  __syncthreads();
  I8STAMP(4);
  refine_block<EP / 32>(L, lg, C::LGS, rs, t0, rows);
  __syncthreads();
  I8STAMP(5);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::ACC_COLS>(tmem);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 i8_get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// int8 [rows, cols] row-major map, {128 cols x box_rows} box, 128B swizzle
static bool i8_make_map(CUtensorMap* m, const void* base, long rows, long cols, int box_rows) {
  auto enc = i8_get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols};
  cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int EP>
static cudaError_t launch_router_i8_t(const RouterLaunch& L, cudaStream_t s) {
  using C = I8Cfg<EP>;
  CUtensorMap ma, mb;
  if (!i8_make_map(&ma, L.i8_x, (long)I8_NP * L.T, L.d, I8_BM)) return cudaErrorInvalidValue;
  if (!i8_make_map(&mb, L.i8_w, (long)I8_NP * EP, L.d, EP)) return cudaErrorInvalidValue;
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = ensure_smem_attr(router_i8_kernel<EP>, C::SMEM, attr)) return e;
  const int nblk = (L.T + I8_BM - 1) / I8_BM;
  int nsplit = kNumSMs / nblk;                                 // fill the SMs: split d across CTAs
  if (nsplit > I8_MAX_SPLIT) nsplit = I8_MAX_SPLIT;
  if (nsplit > L.d / I8_BK) nsplit = L.d / I8_BK;
  if (nsplit < 1 || (long)nsplit * L.T > kI8SplitRows) nsplit = 1;
  router_i8_quant_w_kernel<<<EP, 256, 0, s>>>(L, EP);
  if (L.d == 2048)
    router_i8_quant_x_kernel<16><<<(L.T + 7) / 8, 256, 0, s>>>(L);
  else if (L.d == 1024)
    router_i8_quant_x_kernel<8><<<(L.T + 7) / 8, 256, 0, s>>>(L);
  else
    router_i8_quant_x_kernel<0><<<(L.T + 7) / 8, 256, 0, s>>>(L);
  router_i8_kernel<EP><<<dim3(nblk, nsplit), I8_THREADS, C::SMEM, s>>>(ma, mb, L);
  g_launches += 3;
  return cudaGetLastError();
}

static cudaError_t launch_router_i8(const RouterLaunch& L, cudaStream_t s) {
  return L.E <= 64 ? launch_router_i8_t<64>(L, s) : launch_router_i8_t<128>(L, s);
}

template <int EW>
static cudaError_t launch_router_t(const RouterLaunch& L, cudaStream_t s) {
  constexpr int EP = 32 * EW, NS = EW >= 4 ? 2 : 4, NEH = EP >= 64 ? EP / 64 : 1, KS = 8 / NEH;
  RouterLaunch LL = L;
  const int slots = 2 * kNumSMs;                     // two CTAs per SM
  int nsplit = 1;
  const int nblk32 = (L.T + TB - 1) / TB;
  if (nblk32 < kNumSMs) {                            // small T (decode): split d across CTAs
    nsplit = slots / nblk32;
    if (nsplit > kMaxSplit) nsplit = kMaxSplit;       // finish-kernel traffic: nsplit x T x E partials
    if (nsplit > L.d / DC) nsplit = L.d / DC;
    if (nsplit < 1) nsplit = 1;
  }
  if (nsplit > 1) {
    LL.rpb = TB;
  } else {                                           // balance the grid: whole waves of 2 CTAs per SM
    const int waves = (L.T + slots * TB - 1) / (slots * TB);
    LL.rpb = (L.T + slots * waves - 1) / (slots * waves);
    if (LL.rpb > TB) LL.rpb = TB;
    if (LL.rpb < 1) LL.rpb = 1;
  }
  const int grid = (L.T + LL.rpb - 1) / LL.rpb;
  if (nsplit > 1 && (long)nsplit * L.T > kRouterSplitRows) return cudaErrorInvalidValue;
  router_prescale_kernel<<<EP, 256, 0, s>>>(L.w_router, L.gamma, L.w_scaled, L.w_sq, L.E, L.d, EP);
  const size_t smem = (size_t)(NS * (TB * LDS + DC * EP) + 2 * TB + EP) * 4 + 16;
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = ensure_smem_attr(router_kernel<EW>, (int)smem, attr)) return e;
  router_kernel<EW><<<dim3(grid, nsplit), 256, smem, s>>>(LL);
  g_launches += 2;
  if (nsplit > 1) {   // 8 tokens per finish CTA: more CTAs in flight for the latency-bound epilogue
    const float chain = (float)(L.d / (nsplit * KS) + KS + nsplit + 6);
    RouterLaunch LF = LL;
    LF.rpb = kFinishRows;
    router_finish_kernel<EW><<<(L.T + kFinishRows - 1) / kFinishRows, 256, 0, s>>>(LF, nsplit, chain);
    ++g_launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_router(const RouterLaunch& L, cudaStream_t s) {
  if (L.T == 0) return cudaSuccess;
  if (L.d % DC || L.d > kMaxD || L.E < 1 || L.E > 128 || L.k < 1 || L.k > L.E) return cudaErrorInvalidValue;
  if (!L.part || !L.part_sq || !L.w_scaled || !L.w_sq)
    return cudaErrorInvalidValue;
  if (L.i8_x && L.E <= 128 && L.d % 128 == 0 && L.k <= 8) return launch_router_i8(L, s);
  if (L.E <= 32) return launch_router_t<1>(L, s);   // padded to 32 / 64 / 128 (zero W' columns)
  if (L.E <= 64) return launch_router_t<2>(L, s);
  return launch_router_t<4>(L, s);
}

}  // namespace fsc
