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
#define TC_KNOB (L.rpb)
#define TCSTAMP(kk)                                                                          \
  if (threadIdx.x == 64) {                                                                   \
    unsigned long long g__;                                                                  \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g__));                                  \
    reinterpret_cast<unsigned long long*>(L.logits)[blockIdx.x * 8 + (kk)] = g__;            \
  }
#else
#define RSTAMP(kk)
#define I8STAMP(kk)
#define TCSTAMP(kk)
#define TC_KNOB 0
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
// Exact tensor-core router: ONE fused kernel per call (E <= 128, d % 128 == 0, k <= 8),
// after a small per-call pass that puts W' = gamma (.) W_R into digit planes.
//
// Fixed point, exactly. s_t, s_e powers of two with |x_ti| < s_t and |w_ei| < s_e
// (w_e = gamma (.) W_R[e], formed exactly in fp64). q_ti = floor(x_ti 2^21 / s_t) and
// p_ei = floor(w_ei 2^21 / s_e) lie in [-2^21, 2^21) and are written in base 2^7,
//   q = a0 2^14 + a1 2^7 + a2,   a0 in [-128, 127], a1, a2 in [0, 127]   (all int8),
// the same for p with digits b0, b1, b2. With x/s_t = q 2^-21 + dx, w/s_e = p 2^-21 + dw,
// 0 <= dx, dw < 2^-21, and x w - q p 2^-42 = dx (w/s_e) + (q 2^-21) dw:
//   sum_i x_ti w_ei / (s_t s_e) = 2^-42 sum_{a+b<=3} 2^{7(4-a-b)} <a_a, b_b> + err,
//   |err| <= 2^-21 (||x_t/s_t||_1 + ||w_e/s_e||_1) + 3 d 2^-42 + 127^2 d 2^-42,
// the last term the one dropped digit pair (2, 2). Every <a_a, b_b> is an exact int32
// tcgen05 kind::i8 sum (|.| <= 2^14 d); the pairs with equal a + b share one TMEM
// accumulator (4 x EP columns) and the four accumulators combine exactly in fp64 (at
// most ~50 significant bits). So l_te = r_t s_t s_e (... + err) with a rigorous bound
// B_t = r_t s_t max_e s_e |err|, which decides the selection exactly as in the SIMT
// path (select_token_thread: experts certainly in / out of the top-k; the band experts
// of an ambiguous token are recomputed in fp64 and ranked, ties -> lower id).
//
// The digits of x are made inside the kernel: for |y| < 2^21 (y = x 2^21 / s_t, exact),
// fma_rz(x, 2^21 / s_t, 1.5 2^23) = 1.5 2^23 + floor(y) exactly, so a2, a1 and a0 are the
// bit fields [0,7), [7,14) and [14,22) of that float (two's complement for a0).
//
// Grid: one cluster of CS CTAs per tile of 128 tokens; CTA c of the cluster owns the
// d-slice [c d/CS, (c+1) d/CS) (CS fills the SMs when T is small and keeps each CTA's
// slice of x small enough to be re-read from L2). Per CTA, 10 warps. Warp 0 streams the
// slice of x twice through a ring of TMA boxes (128 rows x 64 fp32 columns, 3 x 32 KB in
// flight) and the digit planes of W' per 64-column k-block; warps 2-9 (workers):
//   phase 1: sum x^2, sum |x| (fp64) and max |x| of the tile's rows over the slice; cluster
//     barrier; each CTA combines the CS partials in rank order (so r_t and s_t agree);
//   phase 2, per k-block: xn = bf16(x gamma r) to global and the three digit planes of x
//     into shared memory in the 64B-swizzled K-major layout TMA would produce;
// warp 1 issues 8 digit pairs x 2 MMAs (M = 128, N = EP, K = 32) per k-block into the 4
// accumulators. Epilogue: CS = 1: TMEM -> fp64 combine -> fp32 logits in shared memory.
// CS > 1: CTA o of the cluster finishes the rows [o 128/CS, (o+1) 128/CS): every CTA sends
// the int32 accumulators of those rows to o (st.shared::cluster, <= 64 experts per pass)
// and o adds them (integers: exact, any order) before the combine. Then one thread per
// token selects; the band dots of each ambiguous token are split over the 8 workers' d-slices.
namespace {
constexpr int TC_BM = 128, TC_BK = 64, TC_NP = 3, TC_NACC = 4;
constexpr int TC_WORKERS = 8;                          // warps 2..9
constexpr int TC_THREADS = 64 + 32 * TC_WORKERS;       // 320
constexpr int TC_A_PLANE = TC_BM * TC_BK;              // 8 KB (64-byte rows)
constexpr int TC_XBOX = TC_BM * TC_BK * 4;             // 32 KB: 128 rows x 64 fp32
constexpr int TC_NXS = 3;                              // x boxes in flight
constexpr int TC_MAX_CS = 16;                         // 16: non-portable cluster size (small T)
constexpr float kTcMagic = 12582912.0f;                // 1.5 * 2^23

template <int EP>
struct TcCfg {
  static constexpr int B_PLANE = EP * TC_BK;                       // 2 / 4 / 8 KB
  static constexpr int AB = TC_NP * (TC_A_PLANE + B_PLANE);        // 30 / 36 / 48 KB
  static constexpr int NAB = EP == 128 ? 2 : 3;
  static constexpr int XRING = TC_NXS * TC_XBOX;                   // 96 KB
  static constexpr int BYTES = XRING + NAB * AB;
  static constexpr int NX1 = NAB * AB / TC_XBOX;                  // phase-1 x boxes also in the AB region
  static constexpr int NP1 = TC_NXS + NX1;                         // (idle until phase 2): 5 / 6 in flight
  static constexpr int ACC_COLS = TC_NACC * EP;                    // 128 / 256 / 512
  static constexpr int LGS = EP + 4;
  static constexpr int RSTRD = EP + 2;                             // receive row stride (doubles, padded)
  static constexpr int RECV = TC_BM * RSTRD * 8;                   // bytes
  static constexpr int SMEM = 1024 + BYTES;
  static_assert(RECV + (TC_BM / 2) * LGS * 4 <= BYTES, "CS > 1 epilogue must fit");
  static_assert(NP1 <= TC_NXS + 3, "x barrier arrays");
  static_assert(TC_BM * LGS * 4 <= BYTES, "CS = 1 epilogue must fit");
};

struct TcShared {
  double p_ss[TC_BM], p_pos[TC_BM], p_neg[TC_BM];   // this CTA's partials over its d-slice (read by the cluster)
  float p_mx[TC_BM];
  double f_r[TC_BM];                 // r_t
  float f_qs[TC_BM], f_rf[TC_BM], f_st[TC_BM], f_l1[TC_BM];   // 2^21/s_t, (float) r_t, s_t, X_t
  float se[128];                     // per expert s_e
  float c1max, c2max;                // max_e of the two bound coefficients
  uint64_t x_full[TC_NXS + 3], x_empty[TC_NXS + 3], full_a[3], full_b[3], ab_empty[3], tfull, p1done;
  uint32_t tmem;
  int nflag;
  int flist[TC_BM];
  int flag[TC_BM];                   // select_token_thread's refinement hand-off
  float thr[TC_BM][3];
  int np;                            // refinement: (token, band expert) pairs
};

FSC_DEVINL double ld_cluster_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
FSC_DEVINL float ld_cluster_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
FSC_DEVINL void st_cluster_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared::cluster.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w)
               : "memory");
}
FSC_DEVINL double2 ld_cluster_f64x2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
FSC_DEVINL void st_cluster_v2_f64(uint32_t a, double x, double y) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1,%2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
FSC_DEVINL void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
FSC_DEVINL void cluster_arrive_release() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
FSC_DEVINL void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
FSC_DEVINL void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
FSC_DEVINL void worker_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * TC_WORKERS) : "memory"); }
FSC_DEVINL void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
FSC_DEVINL void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// K-major operand with 64-byte rows and the 64B swizzle (16-byte chunk c of row r at
// chunk c ^ ((r >> 1) & 3)): 8-row groups SBO = 512 B apart, layout type 4 = SWIZZLE_64B
FSC_DEVINL uint64_t umma_desc_sw64(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

// x box n (n < NKB: phase 1, else phase 2 of box n - NKB) -> ring slot s and its use index u
// (the u-th fill of slot s). Phase 1 cycles through NP1 slots (the ring plus the AB region,
// idle until phase 2), phase 2 through the TC_NXS ring slots only.
FSC_DEVINL int tc_uses1(int s, int nkb, int NP1) { return s < nkb ? (nkb - 1 - s) / NP1 + 1 : 0; }
FSC_DEVINL void tc_xslot(int n, int nkb, int NP1, int& s, int& u) {
  if (n < nkb) {
    s = n % NP1;
    u = n / NP1;
  } else {
    const int m = n - nkb;
    s = m % TC_NXS;
    u = tc_uses1(s, nkb, NP1) + m / TC_NXS;
  }
}
FSC_DEVINL uint8_t* tc_xbox(uint8_t* smem, uint8_t* abase, int s) {
  return s < TC_NXS ? smem + s * TC_XBOX : abase + (s - TC_NXS) * TC_XBOX;
}

// digit planes of 4 consecutive x values (one float4), as 3 packed int8x4 words
FSC_DEVINL void tc_digits(float4 v, float qs, uint32_t& w0, uint32_t& w1, uint32_t& w2) {
  const uint32_t b0 = __float_as_uint(__fmaf_rz(v.x, qs, kTcMagic));
  const uint32_t b1 = __float_as_uint(__fmaf_rz(v.y, qs, kTcMagic));
  const uint32_t b2 = __float_as_uint(__fmaf_rz(v.z, qs, kTcMagic));
  const uint32_t b3 = __float_as_uint(__fmaf_rz(v.w, qs, kTcMagic));
  w2 = __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410) & 0x7F7F7F7Fu;
  const uint32_t c0 = b0 << 1, c1 = b1 << 1, c2 = b2 << 1, c3 = b3 << 1;      // bits [7,14) -> byte 1
  w1 = __byte_perm(__byte_perm(c0, c1, 0x0051), __byte_perm(c2, c3, 0x0051), 0x5410) & 0x7F7F7F7Fu;
  const uint32_t e0 = c0 << 1, e1 = c1 << 1, e2 = c2 << 1, e3 = c3 << 1;      // bits [14,22) -> byte 2
  w0 = __byte_perm(__byte_perm(e0, e1, 0x0062), __byte_perm(e2, e3, 0x0062), 0x5410);
}

// Selection by a group of G consecutive threads per token (G in {1, 2, 4}; every thread of
// the warp calls it, threads of groups without a token with tt < 0). Thread j of a group
// takes the top-(k+1) of its contiguous E/G experts by insertion (64-bit keys: the ordered
// fp32 value, then the complemented id, so equal values rank the lower id first), the
// groups' lists are merged by shuffles (the i-th largest of two sorted lists is
// max_j min(a_{j-1}, b_{i-j})), and thread 0 of the group applies the rule of
// select_token_thread: boundary test against the bound B (ambiguous -> rs.flag for the
// fp64 refinement), else gates over the selected set and slots in ascending expert id.
template <int K1, class RS>
FSC_DEVINL void select_token_group(const float* lg, long t, int tt, int G, int j, float B, const RouterLaunch& L,
                                   RS& rs) {
  constexpr int k = K1 - 1;
  const int E = L.E, ne = (E + G - 1) / G, e0 = j * ne, e1 = min(E, e0 + ne);
  float val[K1];
  int id[K1];
#pragma unroll
  for (int i = 0; i < K1; ++i) {
    val[i] = -INFINITY;
    id[i] = 0x7fffffff;
  }
  bool finite = true;
  auto insert = [&](float v, int e) {                   // ascending e, strict '>': lower id first on ties
    if (!(fabsf(v) <= FLT_MAX)) {
      finite = false;
      v = -FLT_MAX;
    }
    if (v > val[K1 - 1]) {
      bool gt[K1];
#pragma unroll
      for (int i = 0; i < K1; ++i) gt[i] = v > val[i];
#pragma unroll
      for (int i = K1 - 1; i >= 1; --i)
        if (gt[i]) {
          val[i] = gt[i - 1] ? val[i - 1] : v;
          id[i] = gt[i - 1] ? id[i - 1] : e;
        }
      if (gt[0]) {
        val[0] = v;
        id[0] = e;
      }
    }
  };
  if (tt >= 0) {
    if ((ne & 3) == 0) {
      for (int e = e0; e < e1; e += 4) {                 // 16-byte rows: LDS.128
        const float4 q = *reinterpret_cast<const float4*>(lg + e);
        insert(q.x, e);
        if (e + 1 < e1) insert(q.y, e + 1);
        if (e + 2 < e1) insert(q.z, e + 2);
        if (e + 3 < e1) insert(q.w, e + 3);
      }
    } else {
      for (int e = e0; e < e1; ++e) insert(lg[e], e);
    }
  }
  unsigned long long key[K1];
#pragma unroll
  for (int i = 0; i < K1; ++i)
    key[i] = id[i] == 0x7fffffff ? 0ull
                                 : ((unsigned long long)ordered_f32(val[i]) << 32) | (0xFFFFFFFFu - (uint32_t)id[i]);
  for (int off = 1; off < G; off <<= 1) {               // merge with the partner thread's list
    unsigned long long b[K1];
#pragma unroll
    for (int i = 0; i < K1; ++i) b[i] = __shfl_xor_sync(0xffffffff, key[i], off);
    unsigned long long c[K1];
#pragma unroll
    for (int i = 0; i < K1; ++i) {
      unsigned long long m = 0ull;
#pragma unroll
      for (int a = 0; a <= i + 1; ++a) {                // a - 1 from the own list, i - a from b
        const unsigned long long x = a == 0 ? ~0ull : key[a - 1];
        const unsigned long long y = i - a < 0 ? ~0ull : b[i - a];
        const unsigned long long mn = x < y ? x : y;
        m = mn > m ? mn : m;
      }
      c[i] = m;
    }
#pragma unroll
    for (int i = 0; i < K1; ++i) key[i] = c[i];
  }
  bool fin = finite;                                      // a non-finite row selects valid ids, never refined
  for (int off = 1; off < G; off <<= 1) fin = __shfl_xor_sync(0xffffffff, (int)fin, off) && fin;
  if (tt < 0) return;
#ifndef FSC_ROUTER_PROF
  if (L.logits)
    for (int e = e0; e < e1; ++e) L.logits[t * E + e] = lg[e];
#endif
  if (j != 0) return;
  int idx[K1];
#pragma unroll
  for (int i = 0; i < K1; ++i) {
    const uint32_t u = (uint32_t)(key[i] >> 32);
    val[i] = __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
    idx[i] = (int)(0xFFFFFFFFu - (uint32_t)key[i]);
  }
  const float vk = val[k - 1], vk1 = k < E ? val[k] : -FLT_MAX;
  const float thr2 = 2.f * B + 4.f * kU * (fabsf(vk) + fabsf(vk1)) + 1e-7f;
  if (fin && k < E && vk - vk1 <= thr2) {
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
  for (int i = 0; i < K1; ++i) {
    ex[i] = i < k ? expf(val[i] - vtop) : 0.f;
    sum += ex[i];
  }
#pragma unroll
  for (int i = 0; i < K1; ++i) {
    if (i < k) {
      int rank = 0;
#pragma unroll
      for (int m = 0; m < K1; ++m) rank += (m < k && idx[m] < idx[i]) ? 1 : 0;
      L.topk_idx[t * k + rank] = idx[i];
      L.topk_w[t * k + rank] = ex[i] / sum;
    }
  }
}

// fp64 raw dot sum_i x_ti gamma_i W_R[e, i] by one warp (x_ti gamma_i exact in fp64);
// the slow path of refine_tc when a tile's band experts overflow the pair list
FSC_DEVINL double warp_dot_f64(const RouterLaunch& L, long t, int e, int lane) {
  const int dv = L.d / 4;
  const float4* x4 = reinterpret_cast<const float4*>(L.x + t * L.d);
  const float4* g4 = reinterpret_cast<const float4*>(L.gamma);
  const float4* w4 = reinterpret_cast<const float4*>(L.w_router + (long)e * L.d);
  double a0 = 0.0, a1 = 0.0;
  for (int c = lane; c < dv; c += 32) {
    const float4 xv = x4[c], gv = __ldg(g4 + c), wv = __ldg(w4 + c);
    a0 = fma((double)xv.x * gv.x, (double)wv.x, a0);
    a1 = fma((double)xv.y * gv.y, (double)wv.y, a1);
    a0 = fma((double)xv.z * gv.z, (double)wv.z, a0);
    a1 = fma((double)xv.w * gv.w, (double)wv.w, a1);
  }
  return warp_sum_f64(a0 + a1);
}

// fp64 refinement of every ambiguous token of the tile, by the 8 workers (lg: fp32 logits
// of the tile's rows; flist: the nf flagged rows with their band thresholds in sh.thr).
//  1. warp per flagged token: experts certainly in (fp32 logit above the band), the band
//     experts appended to a (token, expert) pair list;
//  2. every worker computes, over its 1/8 of d, the fp64 raw dots sum_i x_ti gamma_i W_R[e,i]
//     of all pairs (x_ti gamma_i exact in fp64), 4 pairs in flight;
//  3. warp per flagged token: the pair's dot = the 8 partials added in worker order, the
//     open slots filled with the best band experts (fp64 value, ties -> lower id), indices
//     in ascending id and gates from the fp32 logits of the selected set.
// The positive factor r_t does not change the order of a token's raw dots.
constexpr int TC_PCAP = 512;
struct TcRefine {
  double part[TC_WORKERS][TC_PCAP];
  int pr[TC_PCAP];                   // (flag index << 8) | expert
  int fbase[TC_BM], fcnt[TC_BM];
  uint32_t fsel[TC_BM][4], fbnd[TC_BM][4];
};

template <int QN>
FSC_DEVINL void refine_tc(const RouterLaunch& L, const float* lg, int lgs, const int* flist, const float (*thr)[3],
                          int nf, long t0, int wk, int lane, TcRefine& R, int* np_sh) {
  const int E = L.E, k = L.k, d = L.d;
  for (int f = wk; f < nf; f += TC_WORKERS) {
    const int tt = flist[f];
    const float* row = lg + tt * lgs;
    const float thr2 = thr[tt][0], hi = thr[tt][1], lo = thr[tt][2];
    int nb = 0;
    uint32_t band = 0;
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const int e = lane + 32 * q;
      const float v = e < E ? row[e] : -FLT_MAX;
      const bool in = e < E && v > hi + thr2;
      const bool bnd = e < E && !in && !(v < lo - thr2);
      const uint32_t mi = __ballot_sync(0xffffffff, in), mb = __ballot_sync(0xffffffff, bnd);
      if (lane == 0) {
        R.fsel[f][q] = mi;
        R.fbnd[f][q] = mb;
      }
      if (bnd) band |= 1u << q;
      nb += __popc(mb);
    }
    int base = 0;
    if (lane == 0) base = atomicAdd(np_sh, nb);
    base = __shfl_sync(0xffffffff, base, 0);
    if (lane == 0) {
      R.fbase[f] = base;
      R.fcnt[f] = nb;
    }
    int o = base;
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const uint32_t m = __ballot_sync(0xffffffff, (band >> q) & 1u);
      const int pos = o + __popc(m & ((1u << lane) - 1u));
      if (((band >> q) & 1u) && pos < TC_PCAP) R.pr[pos] = (f << 8) | (lane + 32 * q);
      o += __popc(m);
    }
  }
  worker_bar();
  const int np = min(*np_sh, TC_PCAP);
  const int dw = d / TC_WORKERS, c0 = wk * dw;            // this worker's d-slice
  const float4* g4 = reinterpret_cast<const float4*>(L.gamma + c0);
  for (int p0 = 0; p0 < np; p0 += 4) {
    const float4* x4[4];
    const float4* w4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int pr = R.pr[min(p0 + u, np - 1)];
      x4[u] = reinterpret_cast<const float4*>(L.x + (t0 + flist[pr >> 8]) * d + c0);
      w4[u] = reinterpret_cast<const float4*>(L.w_router + (long)(pr & 255) * d + c0);
    }
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c = lane; c < dw / 4; c += 32) {
      const float4 gv = __ldg(g4 + c);
      float4 xv[4], wv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xv[u] = x4[u][c];
        wv[u] = __ldg(w4[u] + c);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc[u] = fma((double)xv[u].x * gv.x, (double)wv[u].x, acc[u]);
        acc[u] = fma((double)xv[u].y * gv.y, (double)wv[u].y, acc[u]);
        acc[u] = fma((double)xv[u].z * gv.z, (double)wv[u].z, acc[u]);
        acc[u] = fma((double)xv[u].w * gv.w, (double)wv[u].w, acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double sum = warp_sum_f64(acc[u]);
      if (lane == 0 && p0 + u < np) R.part[wk][p0 + u] = sum;
    }
  }
  worker_bar();
  for (int f = wk; f < nf; f += TC_WORKERS) {
    const int tt = flist[f];
    const long t = t0 + tt;
    const float* row = lg + tt * lgs;
    const int base = R.fbase[f], cnt = R.fcnt[f];
    uint32_t sel = 0, band = 0;
    float v[QN];
    double l64[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const int e = lane + 32 * q;
      v[q] = e < E ? row[e] : -FLT_MAX;
      sel |= ((R.fsel[f][q] >> lane) & 1u) << q;
      band |= ((R.fbnd[f][q] >> lane) & 1u) << q;
      l64[q] = -DBL_MAX;
    }
    for (int i = 0; i < cnt; ++i) {                      // the token's pairs, in list order
      const int p = base + i;
      int e;
      double val;
      if (p < TC_PCAP) {
        e = R.pr[p] & 255;
        val = 0.0;
        for (int w = 0; w < TC_WORKERS; ++w) val += R.part[w][p];
      } else {                                           // pair list overflow: the slow path
        int cntq = i;
        e = -1;
#pragma unroll
        for (int q = 0; q < QN; ++q) {
          const uint32_t m = R.fbnd[f][q];
          if (e < 0 && cntq < __popc(m)) {
            uint32_t mm = m;
            for (int j = 0; j < cntq; ++j) mm &= mm - 1;
            e = 32 * q + __ffs(mm) - 1;
          }
          if (e < 0) cntq -= __popc(m);
        }
        val = warp_dot_f64(L, t, e, lane);
      }
#pragma unroll
      for (int q = 0; q < QN; ++q)
        if (e == lane + 32 * q) l64[q] = val;
    }
    int nsel = 0;
#pragma unroll
    for (int q = 0; q < QN; ++q) nsel += __popc(R.fsel[f][q]);
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
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
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
}  // namespace

// Per padded expert (one CTA of 256 threads; small, so that it co-resides with the fused
// kernel that starts beside it): w = gamma (.) W_R[e] exactly in fp64, s_e, the digit planes
// of floor(w 2^21 / s_e) and the error-bound coefficients (each rounded up), zero for e >= E:
//   c1_e = s_e 2^-21,   c2_e = s_e (2^-21 max(P_e, N_e) + 127^2 d 2^-42),
// P_e / N_e = the sums of the positive / negative parts of w_e / s_e. The truncation errors
// are one-signed (0 <= dx, dw < 2^-21), so |sum_i dx_i w_i/s_e| <= 2^-21 max(P_e, N_e),
// |sum_i q_i 2^-21 dw_i| <= 2^-21 max(Xp_t, Xn_t + d 2^-21) (the token's sums, phase 1),
// and the dropped pair 2^-42 sum a2 b2 lies in [0, 127^2 d 2^-42]: |err| <= c1 X_t + c2.
constexpr int TC_QW_THREADS = 256;
FSC_DEVINL double pow2d(int n) { return __longlong_as_double((long long)(1023 + n) << 52); }   // |n| < 1000
__global__ void __launch_bounds__(TC_QW_THREADS) router_tc_quant_w_kernel(RouterLaunch L, int EP) {
  griddep_launch();   // the fused kernel may start its pass over x right away (PDL)
#ifdef FSC_ROUTER_PROF
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long g__;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g__));
    reinterpret_cast<unsigned long long*>(L.logits)[148 * 8 * 8 - 2] = g__;
  }
#endif
  __shared__ float red_mx[TC_QW_THREADS / 32];
  __shared__ double red[2][TC_QW_THREADS / 32];
  const int e = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = L.d;
  const bool ok = e < L.E;
  const float* wrow = L.w_router + (long)e * d;
  float mx = 0.f;
  if (ok)
#pragma unroll 8
    for (int c = tid; c < d; c += TC_QW_THREADS)   // (float)|g w| may round up to a power of two:
      mx = fmaxf(mx, fabsf(__ldg(L.gamma + c) * __ldg(wrow + c)));   // frexp then gives one binade more
  mx = warp_max_f32(mx);
  if (lane == 0) red_mx[warp] = mx;
  __syncthreads();
  mx = 0.f;
#pragma unroll
  for (int i = 0; i < TC_QW_THREADS / 32; ++i) mx = fmaxf(mx, red_mx[i]);
  int ex = 0;
  frexpf(mx, &ex);                                    // |w| < 2^ex
  if (!(mx > 0.f)) ex = 0;
  const double scale = pow2d(21 - ex), inv = pow2d(-ex);   // 2^21 / s_e, 1 / s_e
  double pos = 0.0, neg = 0.0;
#pragma unroll 8
  for (int c = tid; c < d; c += TC_QW_THREADS) {
    const double w = ok ? (double)__ldg(L.gamma + c) * (double)__ldg(wrow + c) : 0.0;   // exact
    const int p = (int)floor(w * scale);              // exact: |w 2^21 / s_e| < 2^21
    L.i8_w[(long)e * d + c] = (int8_t)(p >> 14);                          // b0 in [-128, 127]
    L.i8_w[((long)EP + e) * d + c] = (int8_t)((p >> 7) & 127);             // b1
    L.i8_w[(2L * EP + e) * d + c] = (int8_t)(p & 127);                     // b2
    if (w > 0.0) pos += w * inv;
    else neg -= w * inv;
  }
  pos = warp_sum_f64(pos);
  neg = warp_sum_f64(neg);
  if (lane == 0) {
    red[0][warp] = pos;
    red[1][warp] = neg;
  }
  __syncthreads();
  if (tid == 0) {
    double P = 0.0, N = 0.0;
#pragma unroll
    for (int i = 0; i < TC_QW_THREADS / 32; ++i) {
      P += red[0][i];
      N += red[1][i];
    }
    const double se = pow2d(ex), u21 = pow2d(-21), u42 = pow2d(-42);
    L.i8_exp[e] = ok ? (float)se : 0.f;
    L.i8_exp[EP + e] = ok ? (float)(se * u21 * 1.0001) : 0.f;
    L.i8_exp[2 * EP + e] = ok ? (float)(se * (u21 * fmax(P, N) * 1.0001 + 127.0 * 127.0 * d * u42) * 1.0001) : 0.f;
#ifdef FSC_ROUTER_PROF
    unsigned long long g__;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g__));
    atomicMax(reinterpret_cast<unsigned long long*>(L.logits) + 148 * 8 * 8 - 1, g__);
#endif
  }
}

template <int EP>
__global__ void __launch_bounds__(TC_THREADS, 1)
    router_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmXw,
                     const __grid_constant__ CUtensorMap tmB, RouterLaunch L, int CS) {
  using C = TcCfg<EP>;
  constexpr int QN = EP / 32, NAB = C::NAB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* abase = smem + C::XRING;
  __shared__ TcShared sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = warp_id();
  const int rank = CS > 1 ? (int)cluster_ctarank() : 0;
  const long t0 = (long)(blockIdx.x / CS) * TC_BM;
  const int T = L.T, d = L.d;
  const int rows = (int)min((long)TC_BM, (long)T - t0);
  const int DK = d / CS, NKB = DK / TC_BK;
  const int col0 = rank * DK;                            // first column of this CTA's slice
  const bool wide = DK % 256 == 0;                       // phase-1 boxes of 32 rows x 256 columns
  constexpr int NP1 = C::NP1;
  if (tid < TC_BM) sh.flag[tid] = 0;
  if (tid == 0) {
    sh.nflag = 0;
    sh.np = 0;
  }
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmXw);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::NP1; ++s) {
      mbar_init(&sh.x_full[s], 1);
      mbar_init(&sh.x_empty[s], TC_WORKERS);
    }
    for (int s = 0; s < NAB; ++s) {
      mbar_init(&sh.full_a[s], TC_WORKERS);
      mbar_init(&sh.full_b[s], 1);
      mbar_init(&sh.ab_empty[s], 1);
    }
    mbar_init(&sh.tfull, 1);
    mbar_init(&sh.p1done, TC_WORKERS);
    fence_barrier_init();
  } else if (warp == 1) {
    tmem_alloc<C::ACC_COLS>(&sh.tmem);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh.tmem;
  const int wk = warp - 2, rb = wk * 16;                 // worker: rows [rb, rb + 16) of the tile
  TCSTAMP(0);

  if (warp == 0) {
    // ---------------- producer: x boxes (phase 1, then phase 2) and W' digit planes
    cluster_arrive_relaxed();                            // the stats barrier: nothing to publish
    if (lane == 0) {                                     // x: the slice twice (phase 1: NP1 boxes in flight)
      for (int n = 0; n < 2 * NKB; ++n) {
        int s, u;
        tc_xslot(n, NKB, NP1, s, u);
        if (u > 0) mbar_wait(&sh.x_empty[s], (u - 1) & 1);
        mbar_arrive_expect_tx(&sh.x_full[s], TC_XBOX);
        if (n < NKB && wide)                             // phase 1: 32 rows x 256 columns
          tma_load_2d(tc_xbox(smem, abase, s), &tmXw, &sh.x_full[s], col0 + (n >> 2) * 256, (int)t0 + (n & 3) * 32,
                      kEvictLast);
        else
          tma_load_2d(tc_xbox(smem, abase, s), &tmX, &sh.x_full[s], col0 + (n % NKB) * TC_BK, (int)t0,
                      n < NKB ? kEvictLast : kEvictFirst);
      }
    } else if (lane == 1) {                              // W' digit planes, NAB k-blocks ahead
      griddep_wait();                                    // (written by router_tc_quant_w_kernel)
      mbar_wait(&sh.p1done, 0);                          // the phase-1 boxes in the AB region are consumed
      for (int kb = 0; kb < NKB; ++kb) {
        const int a = kb % NAB;
        if (kb >= NAB) mbar_wait(&sh.ab_empty[a], ((kb / NAB) - 1) & 1);
        uint8_t* sb = abase + a * C::AB + TC_NP * TC_A_PLANE;
        mbar_arrive_expect_tx(&sh.full_b[a], TC_NP * C::B_PLANE);
#pragma unroll
        for (int j = 0; j < TC_NP; ++j)
          tma_load_2d(sb + j * C::B_PLANE, &tmB, &sh.full_b[a], col0 + kb * TC_BK, j * EP, kEvictLast);
      }
    }
    __syncwarp();
    cluster_wait();
  } else if (warp == 1) {
    // ---------------- MMA issuer
    cluster_arrive_relaxed();
    if (elect_one()) {
      // the B digit planes are one tall K-major tile [b0; b1; b2]: an MMA of x's plane i against
      // planes [jb, jb + nj) written at column (i + jb) EP adds <a_i, b_j> into accumulator i + j
      // for every j at once (fewer, wider MMAs: x's planes are read from shared memory 3 times
      // instead of 8). The first K-step initialises each accumulator exactly once.
      for (int kb = 0; kb < NKB; ++kb) {
        const int a = kb % NAB;
        const uint32_t ph = (kb / NAB) & 1;
        mbar_wait(&sh.full_b[a], ph);
        mbar_wait(&sh.full_a[a], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(abase + a * C::AB), sb = sa + TC_NP * TC_A_PLANE;
#pragma unroll
        for (int kk = 0; kk < TC_BK / 32; ++kk) {
          const bool first = kb == 0 && kk == 0;
          auto mma = [&](int i, int jb, int nj, bool init) {
            if (!(TC_KNOB & 1))
              umma_s8_ss(tmem + (i + jb) * EP, umma_desc_sw64(sa + i * TC_A_PLANE + kk * 32),
                         umma_desc_sw64(sb + jb * C::B_PLANE + kk * 32), idesc_s8_s32(TC_BM, nj * EP),
                         init ? 0u : 1u);
          };
          if (EP <= 64) {                                // N = 3 EP <= 192
            mma(0, 0, 3, first);                         // acc 0, 1, 2
            if (first) {
              mma(1, 0, 2, false);                       // acc 1, 2
              mma(1, 2, 1, true);                        // acc 3 (first write)
            } else {
              mma(1, 0, 3, false);                       // acc 1, 2, 3
            }
            mma(2, 0, 2, false);                         // acc 2, 3 (pair (2, 2) dropped)
          } else {                                       // N <= 256: [b0; b1] and b2 separately
            mma(0, 0, 2, first);                         // acc 0, 1
            mma(0, 2, 1, first);                         // acc 2
            mma(1, 0, 2, false);                         // acc 1, 2
            mma(1, 2, 1, first);                         // acc 3
            mma(2, 0, 2, false);                         // acc 2, 3
          }
        }
        umma_commit(&sh.ab_empty[a]);
      }
      umma_commit(&sh.tfull);
    }
    __syncwarp();
    cluster_wait();
  } else {
    // ---------------- phase 1: row statistics over this CTA's d-slice (lane: 2 columns)
    double ss[16];
    float sp[16], sn[16], mx[16];   // per-lane sums of the positive / negative parts (fp32: <= 64 terms)
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
      ss[rr] = 0.0;
      sp[rr] = sn[rr] = mx[rr] = 0.f;
    }
    auto accum = [&](int rr, float a, float b) {
      ss[rr] = fma((double)b, (double)b, fma((double)a, (double)a, ss[rr]));
      sp[rr] += fmaxf(a, 0.f) + fmaxf(b, 0.f);
      sn[rr] += fmaxf(-a, 0.f) + fmaxf(-b, 0.f);
      mx[rr] = fmaxf(mx[rr], fmaxf(fabsf(a), fabsf(b)));
    };
    if (wide) {                                          // boxes of 32 rows x 256 columns (4 per column block)
      for (int cb = 0; cb < NKB / 4; ++cb) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          int s, u;
          tc_xslot(cb * 4 + g, NKB, NP1, s, u);
          mbar_wait(&sh.x_full[s], u & 1);
          const float* xs = reinterpret_cast<const float*>(tc_xbox(smem, abase, s)) + wk * 4 * 256 + 8 * lane;
#pragma unroll
          for (int r = 0; r < 4; ++r) {                  // rows g 32 + wk 4 + r: partial index g 4 + r
            const float4 v0 = *reinterpret_cast<const float4*>(xs + r * 256);
            const float4 v1 = *reinterpret_cast<const float4*>(xs + r * 256 + 4);
            accum(g * 4 + r, v0.x, v0.y);
            accum(g * 4 + r, v0.z, v0.w);
            accum(g * 4 + r, v1.x, v1.y);
            accum(g * 4 + r, v1.z, v1.w);
          }
          fence_proxy_async_smem();                      // these reads before the next TMA fill of the slot
          __syncwarp();
          if (lane == 0) mbar_arrive(&sh.x_empty[s]);
        }
      }
    } else {                                             // boxes of 128 rows x 64 columns
      for (int n = 0; n < NKB; ++n) {
        int s, u;
        tc_xslot(n, NKB, NP1, s, u);
        mbar_wait(&sh.x_full[s], u & 1);
        const float* xs = reinterpret_cast<const float*>(tc_xbox(smem, abase, s)) + rb * TC_BK + 2 * lane;
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
          const float2 v = *reinterpret_cast<const float2*>(xs + rr * TC_BK);
          accum(rr, v.x, v.y);
        }
        fence_proxy_async_smem();                        // these reads before the next TMA fill of the slot
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.x_empty[s]);
      }
    }
    if (lane == 0) mbar_arrive(&sh.p1done);
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
      const double a = warp_sum_f64(ss[rr]), bp = warp_sum_f64((double)sp[rr]), bn = warp_sum_f64((double)sn[rr]);
      const float m = warp_max_f32(mx[rr]);
      const int row = wide ? (rr >> 2) * 32 + wk * 4 + (rr & 3) : rb + rr;
      if (lane == rr) {
        sh.p_ss[row] = a;
        sh.p_pos[row] = bp;
        sh.p_neg[row] = bn;
        sh.p_mx[row] = m;
      }
    }
    TCSTAMP(1);
    cluster_sync();   // every CTA's partials are in its shared memory
    TCSTAMP(2);
    if (lane < 16) {                                     // combine the cluster's partials, rank order
      const int row = rb + lane;
      double a = 0.0, bp = 0.0, bn = 0.0;
      float m = 0.f;
      for (int c = 0; c < CS; ++c) {
        a += ld_cluster_f64(mapa_shared(smem_u32(&sh.p_ss[row]), c));
        bp += ld_cluster_f64(mapa_shared(smem_u32(&sh.p_pos[row]), c));
        bn += ld_cluster_f64(mapa_shared(smem_u32(&sh.p_neg[row]), c));
        m = fmaxf(m, ld_cluster_f32(mapa_shared(smem_u32(&sh.p_mx[row]), c)));
      }
      const double r = 1.0 / sqrt(a / (double)d + (double)L.eps);
      int ex = 0;
      frexpf(m, &ex);                                    // m = f 2^ex, f in [0.5, 1)
      if (!(m > 0.f)) ex = 0;                            // zero row (or a NaN row: garbage, never refined)
      const float st = ldexpf(1.f, ex);
      sh.f_r[row] = r;
      sh.f_rf[row] = (float)r;
      sh.f_st[row] = st;
      sh.f_qs[row] = ldexpf(1.f, 21 - ex);
      // X_t = max(Xp_t, Xn_t + d 2^-21) of x_t / s_t, rounded up (fp32 lane sums: <= 64 terms)
      sh.f_l1[row] = (float)(fmax(bp, bn + ldexp((double)d, -21) * st) / (double)st * 1.0001) + 1e-30f;
    }
    __syncwarp();
    // ---------------- phase 2: xn and the digit planes of x, per 64-column k-block
    const int cq = lane & 15, rh = lane >> 4;            // lane: 4 columns of row rb + 2 i + rh
    for (int kb = 0; kb < NKB; ++kb) {
      const int a = kb % NAB;
      int s, u;
      tc_xslot(NKB + kb, NKB, NP1, s, u);
      mbar_wait(&sh.x_full[s], u & 1);
      if (kb >= NAB) mbar_wait(&sh.ab_empty[a], ((kb / NAB) - 1) & 1);
      const float* xs = reinterpret_cast<const float*>(tc_xbox(smem, abase, s));
      const int c = col0 + kb * TC_BK + 4 * cq;          // global column of this lane's float4
      const float4 g = __ldg(reinterpret_cast<const float4*>(L.gamma + c));
      uint8_t* sa = abase + a * C::AB;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = rb + 2 * i + rh;
        const float4 v = *reinterpret_cast<const float4*>(xs + row * TC_BK + 4 * cq);
        uint32_t w0, w1, w2;
        tc_digits(v, sh.f_qs[row], w0, w1, w2);
        const uint32_t off = row * 64 + (((cq >> 2) ^ ((row >> 1) & 3)) << 4) + ((cq & 3) << 2);
        if (!(TC_KNOB & 2)) {
          *reinterpret_cast<uint32_t*>(sa + off) = w0;
          *reinterpret_cast<uint32_t*>(sa + TC_A_PLANE + off) = w1;
          *reinterpret_cast<uint32_t*>(sa + 2 * TC_A_PLANE + off) = w2;
        }
        const long t = t0 + row;
        if (t < T && !(TC_KNOB & 4)) {
          const float rf = sh.f_rf[row];
          *reinterpret_cast<uint2*>(L.xn + t * d + c) =
              make_uint2(pack_bf16x2(v.x * g.x * rf, v.y * g.y * rf), pack_bf16x2(v.z * g.z * rf, v.w * g.w * rf));
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sh.full_a[a]);
        mbar_arrive(&sh.x_empty[s]);
      }
    }
    TCSTAMP(3);
    griddep_wait();                                      // the expert coefficients (quant_w kernel)
    if (wk == 0) {
      float m1 = 0.f, m2 = 0.f;
      for (int e = lane; e < EP; e += 32) {
        sh.se[e] = L.i8_exp[e];
        m1 = fmaxf(m1, L.i8_exp[EP + e]);
        m2 = fmaxf(m2, L.i8_exp[2 * EP + e]);
      }
      m1 = warp_max_f32(m1);
      m2 = warp_max_f32(m2);
      if (lane == 0) {
        sh.c1max = m1;
        sh.c2max = m2;
      }
    }
  }

  // ---------------- epilogue: exact logits of the rows this CTA finishes
  const int RPO = TC_BM / CS;                            // rows finished per CTA
  const int own0 = rank * RPO;
  const int nown = max(0, min(RPO, rows - own0));
  float* lg = reinterpret_cast<float*>(smem + (CS > 1 ? C::RECV : 0));   // [RPO][LGS]
  const int q = warp & 3, half = (warp - 2) >> 2;        // TMEM lane quarter; expert half / accumulator pair
  const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16);
  const int trow = q * 32 + lane;                        // tile row of this thread's TMEM lane
  if (warp >= 2) {
    mbar_wait(&sh.tfull, 0);
    tc_fence_after();
    worker_bar();                                        // sh.se / c1max / c2max loaded
    TCSTAMP(4);
  }
  if (CS == 1) {
    if (warp >= 2) {
      const double sc = trow < rows ? sh.f_r[trow] * (double)sh.f_st[trow] : 0.0;
#pragma unroll 1
      for (int e0 = half * (EP / 2); e0 < (half + 1) * (EP / 2); e0 += 16) {
        uint32_t S[TC_NACC][16];
#pragma unroll
        for (int a = 0; a < TC_NACC; ++a) tmem_ld16(tb + a * EP + e0, S[a]);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double v = (double)(int)S[0][u] * 0x1p-14 + (double)(int)S[1][u] * 0x1p-21 +
                           (double)(int)S[2][u] * 0x1p-28 + (double)(int)S[3][u] * 0x1p-35;
          lg[trow * C::LGS + e0 + u] = (float)(sc * (double)sh.se[e0 + u] * v);
        }
      }
    }
  } else {
    // every CTA's partial sum over its d-slice, v = sum_a acc_a 2^-(14 + 7a), is exact in fp64
    // (a multiple of 2^-35 below 2^13), and so is any sum of them: the owner adds the CS
    // partials in rank order and the result is the full-d value, bit for bit
    // (no barrier before the local stores: only this CTA's own TMA and MMAs used this shared
    // memory, and they are complete once tfull fired)
    double* part = reinterpret_cast<double*>(smem);      // this CTA's partials [tile row][RSTRD]
    if (warp >= 2) {                                     // my partials, expert half `half`, local stores
      double* dst = part + trow * C::RSTRD;
#pragma unroll 1
      for (int e0 = half * (EP / 2); e0 < (half + 1) * (EP / 2); e0 += 16) {
        uint32_t S[TC_NACC][16];
#pragma unroll
        for (int a = 0; a < TC_NACC; ++a) tmem_ld16(tb + a * EP + e0, S[a]);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
          const double v0 = (double)(int)S[0][u] * 0x1p-14 + (double)(int)S[1][u] * 0x1p-21 +
                            (double)(int)S[2][u] * 0x1p-28 + (double)(int)S[3][u] * 0x1p-35;
          const double v1 = (double)(int)S[0][u + 1] * 0x1p-14 + (double)(int)S[1][u + 1] * 0x1p-21 +
                            (double)(int)S[2][u + 1] * 0x1p-28 + (double)(int)S[3][u + 1] * 0x1p-35;
          *reinterpret_cast<double2*>(dst + e0 + u) = make_double2(v0, v1);
        }
      }
    }
    cluster_sync();                                      // every CTA's partials are written
    if (warp >= 2) {                                     // the owned rows: read the CS partials (rank order)
      const uint32_t base = smem_u32(part);
      for (int i = tid - 64; i < RPO * (EP / 2); i += 32 * TC_WORKERS) {
        const int lr = i / (EP / 2), e = 2 * (i - lr * (EP / 2));
        const uint32_t off = ((own0 + lr) * C::RSTRD + e) * 8;
        double v0 = 0.0, v1 = 0.0;
        for (int c = 0; c < CS; ++c) {
          const double2 p = ld_cluster_f64x2(mapa_shared(base + off, c));
          v0 += p.x;
          v1 += p.y;
        }
        const int row = own0 + lr;
        const double sc = row < rows ? sh.f_r[row] * (double)sh.f_st[row] : 0.0;
        lg[lr * C::LGS + e] = (float)(sc * (double)sh.se[e] * v0);
        lg[lr * C::LGS + e + 1] = (float)(sc * (double)sh.se[e + 1] * v1);
      }
      cluster_arrive_release();                          // done reading the peers' partials; the wait
    } else {                                             // comes before this CTA overwrites / leaves
      cluster_sync();
    }
  }
  tc_fence_before();
  __syncthreads();                                       // logits of the owned rows in shared memory
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::ACC_COLS>(tmem);
  }
  if (warp < 2) return;
  TCSTAMP(5);

  // ---------------- selection (G threads per token) and fp64 refinement
  {
    const int wt = tid - 64;
    const int G = nown <= 64 ? 4 : (nown <= 128 ? 2 : 1);
    const int tt = wt / G < nown ? wt / G : -1, j = wt % G;
    const int row = own0 + max(tt, 0);
    const long t = t0 + row;
    const float B = (float)(sh.f_r[row] * (double)sh.f_st[row] *
                            (double)fmaf(sh.c1max, sh.f_l1[row], sh.c2max) * 1.0001) + 1e-12f;
    const float* rowp = lg + max(tt, 0) * C::LGS;
    switch (L.k) {
      case 1: select_token_group<2>(rowp, t, tt, G, j, B, L, sh); break;
      case 2: select_token_group<3>(rowp, t, tt, G, j, B, L, sh); break;
      case 3: select_token_group<4>(rowp, t, tt, G, j, B, L, sh); break;
      case 4: select_token_group<5>(rowp, t, tt, G, j, B, L, sh); break;
      case 5: select_token_group<6>(rowp, t, tt, G, j, B, L, sh); break;
      case 6: select_token_group<7>(rowp, t, tt, G, j, B, L, sh); break;
      case 7: select_token_group<8>(rowp, t, tt, G, j, B, L, sh); break;
      default: select_token_group<9>(rowp, t, tt, G, j, B, L, sh); break;
    }
    if (tt >= 0 && j == 0 && sh.flag[tt]) sh.flist[atomicAdd(&sh.nflag, 1)] = tt;
  }
  worker_bar();
  TCSTAMP(6);
  const int nf = sh.nflag;
  constexpr bool kInRecv = sizeof(TcRefine) <= (size_t)C::RECV;
  bool waited = CS == 1;
  if (nf > 0) {                                          // block-uniform
    // refinement scratch: the partials buffer (once every peer has read it) when it is large
    // enough, else after the logits
    if (!waited && kInRecv) {
      cluster_wait();
      waited = true;
    }
    uint8_t* rbase = (CS > 1 && kInRecv) ? smem : smem + (CS > 1 ? C::RECV : 0) + RPO * C::LGS * 4;
    static_assert((kInRecv || C::RECV + (TC_BM / 2) * C::LGS * 4 + sizeof(TcRefine) <= (size_t)C::BYTES) &&
                      TC_BM * C::LGS * 4 + sizeof(TcRefine) <= (size_t)C::BYTES,
                  "refinement scratch must fit");
    TcRefine& R = *reinterpret_cast<TcRefine*>(rbase);
    refine_tc<QN>(L, lg, C::LGS, sh.flist, sh.thr, nf, t0 + own0, wk, lane, R, &sh.np);
  }
  if (!waited) cluster_wait();                           // no CTA leaves while its partials are read
#ifdef FSC_ROUTER_PROF
  worker_bar();
  TCSTAMP(7);
#endif
}


static PFN_cuTensorMapEncodeTiled_v12000 tc_get_encode() {
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

// row-major [rows, cols] map with a {box_cols x box_rows} box
static bool tc_make_map(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base, long rows, long cols,
                        int box_cols, int box_rows, CUtensorMapSwizzle sw) {
  auto enc = tc_get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * esize};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Cluster size: the largest power of two (<= 16, dividing the 64-column k-blocks, leaving each
// CTA >= 4 of them) that keeps the grid within one wave of the SMs (one CTA per SM); 16 is a
// non-portable cluster size (Scout decode: d = 5120). FSC_ROUTER_CS overrides (A/B runs).
static int router_tc_cluster(int T, int d) {
  const int tiles = (T + TC_BM - 1) / TC_BM, nkb = d / TC_BK;
  int cs = 0;
  if (const char* env = getenv("FSC_ROUTER_CS")) cs = atoi(env);
  if (cs >= 1 && cs <= TC_MAX_CS && !(cs & (cs - 1)) && nkb % cs == 0) return cs;
  cs = 1;
  while (2 * cs <= TC_MAX_CS && nkb % (2 * cs) == 0 && nkb / (2 * cs) >= 4 && (long)tiles * 2 * cs <= kNumSMs)
    cs *= 2;   // (>= 4 k-blocks per CTA: below that the cluster exchange costs more than it saves)
  return cs;
}

template <int EP>
static cudaError_t launch_router_tc_t(const RouterLaunch& L, cudaStream_t s) {
  using C = TcCfg<EP>;
  CUtensorMap mx, mxw, mb;
  if (!tc_make_map(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, L.x, L.T, L.d, TC_BK, TC_BM,
                   CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !tc_make_map(&mxw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, L.x, L.T, L.d, 256, 32, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !tc_make_map(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, L.i8_w, (long)TC_NP * EP, L.d, TC_BK, EP,
                   CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = ensure_smem_attr(router_tc_kernel<EP>, C::SMEM, attr)) return e;
  int cs = router_tc_cluster(L.T, L.d);
  if (cs > 8) {
    static std::atomic<unsigned long long> np{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(np.load() & bit)) {
      if (cudaFuncSetAttribute(router_tc_kernel<EP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)
        np.fetch_or(bit);
      else
        cs = 8;
    }
    if (cs > 8 && !(np.load() & bit)) cs = 8;
  }
  const int tiles = (L.T + TC_BM - 1) / TC_BM;
  router_tc_quant_w_kernel<<<EP, TC_QW_THREADS, 0, s>>>(L, EP);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles * cs);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  g_launches += 2;
  if (cudaError_t e = cudaGetLastError()) return e;
#ifdef FSC_ROUTER_PROF
  RouterLaunch LP = L;
  LP.rpb = getenv("FSC_TC_KNOB") ? atoi(getenv("FSC_TC_KNOB")) : 0;
  return cudaLaunchKernelEx(&cfg, router_tc_kernel<EP>, mx, mxw, mb, LP, cs);
#else
  return cudaLaunchKernelEx(&cfg, router_tc_kernel<EP>, mx, mxw, mb, L, cs);
#endif
}

static cudaError_t launch_router_tc(const RouterLaunch& L, cudaStream_t s) {
  if (L.E <= 32) return launch_router_tc_t<32>(L, s);
  if (L.E <= 64) return launch_router_tc_t<64>(L, s);
  return launch_router_tc_t<128>(L, s);
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
  if (L.f64) return launch_router_f64(L, s);
  if (L.d % DC || L.d > kMaxD || L.E < 1 || L.E > 128 || L.k < 1 || L.k > L.E) return cudaErrorInvalidValue;
  if (!L.part || !L.part_sq || !L.w_scaled || !L.w_sq)
    return cudaErrorInvalidValue;
  if (L.tc && L.i8_w && L.i8_exp && L.E <= 128 && L.d % 128 == 0 && L.k <= 8) return launch_router_tc(L, s);
  if (L.E <= 32) return launch_router_t<1>(L, s);   // padded to 32 / 64 / 128 (zero W' columns)
  if (L.E <= 64) return launch_router_t<2>(L, s);
  return launch_router_t<4>(L, s);
}

}  // namespace fsc
