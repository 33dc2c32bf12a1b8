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
// band", usually 2-3) of tokens with t_hi - t_lo <= 2B are recomputed in fp64
// (router_refine_kernel) and the missing slots filled by their fp64 order. The
// selection therefore equals the fp64 selection of the oracle for every token.
//
// Main kernel (E > 32): block = 32 tokens x 64/128 experts, 8 warps; each warp
// owns one k-slice of every 64-wide chunk (k-split, summed in a fixed order at the
// end) and an 8 tokens x 8 experts register tile per lane; operands are staged by a
// 3-4 deep cp.async pipeline, read with conflict-free LDS.64 (128 FMA per shared
// memory wavefront, the binding resource of an fp32 SIMT contraction on sm_100).
// sum x^2 is accumulated from the staged chunks (no extra pass over x).
#include <float.h>

#include "common.cuh"
#include "kernels.h"

namespace fsc {

namespace {
constexpr int TB = 32;      // tokens per block
constexpr int DC = 64;      // k per staged chunk
constexpr int LDS = DC + 4; // padded smem row (floats): rows r, r+1 start 4 banks apart
constexpr float kU = 5.9604645e-08f;  // 2^-24
constexpr int kMaxD = 8192;

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
template <int QN>
FSC_DEVINL void select_token(const float* lg, long t, float B, const RouterLaunch& L, int lane) {
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
  if (k < E && vk - vk1 <= thr2) {
    // ambiguous boundary: record the token, its fp32 row and thresholds for router_refine_kernel
    int slot = 0;
    if (lane == 0) {
      if (L.n_refined) atomicAdd(L.n_refined, 1);
      slot = atomicAdd(&L.rf_ctrl[0], 1);
      L.rf_list[slot] = (int)t;
      L.rf_thr[3 * slot] = thr2;
      L.rf_thr[3 * slot + 1] = vk;
      L.rf_thr[3 * slot + 2] = vk1;
    }
    slot = __shfl_sync(0xffffffff, slot, 0);
    for (int e = lane; e < E; e += 32) L.rf_lg[(long)slot * E + e] = lg[e];
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
#else
#define RSTAMP(kk)
#endif

// E in (32, 128]: 8 warps = KS k-groups x NEH expert halves of 64. Each lane owns
// 8 tokens (lt + 4i) x 4 expert pairs (2 le + 16 j + {0,1}); x is staged token-major,
// W' k-major, so one LDS.64 yields an expert pair at one k and every product is an
// FFMA2 with the token value broadcast (full fp32 issue rate on sm_100).
template <int EW>
__global__ void __launch_bounds__(256, 2) router_kernel(RouterLaunch L) {
  constexpr int EP = 32 * EW;          // padded experts: 64 or 128
  constexpr int NEH = EP / 64;         // 64-expert halves
  constexpr int KS = 8 / NEH;          // k-groups (warps sharing a chunk)
  constexpr int KW = DC / KS;          // k per warp per chunk (8 or 16)
  constexpr int NT = 256;
  constexpr int XV = TB * DC / 4 / NT; // float4 of the x chunk per thread (2)
  constexpr int WV = EP * DC / 4 / NT; // float4 of the W' chunk per thread (4 / 8)
  constexpr int XBUF = TB * LDS;       // x chunk, token-major [TB][LDS]
  constexpr int BUF = XBUF + DC * EP;  // + W' chunk, k-major [DC][EP]
  constexpr int NS = EW >= 4 ? 3 : 4;  // cp.async pipeline depth
  extern __shared__ __align__(16) float sm[];
  float* stage0 = sm;                  // [NS][BUF]
  float* red = sm;                     // [KS][TB][EP] k-group partials (after the loop)
  float* lg = sm + KS * TB * EP;       // [TB][EP+1] fp32 logits
  float* s_r = sm + NS * BUF;          // [TB]
  float* s_xn = s_r + TB;              // [TB] ||x_t||
  float* s_wsq = s_xn + TB;            // [EP]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = L.d, E = L.E;
  const long t0 = (long)blockIdx.x * L.rpb;    // rpb <= TB rows per block (balanced grid)
  const int rows = (int)min((long)L.rpb, (long)L.T - t0);
  const long T = t0 + rows;                    // rows >= T are padding
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
  const int nch = d / DC;
#pragma unroll
  for (int i = 0; i < NS - 1; ++i) {
    if (i < nch) issue_chunk(i * DC, stage0 + i * BUF);
    else cp_async_commit();
  }
  for (int e = tid; e < EP; e += NT) s_wsq[e] = e < E ? L.w_sq[e] : 0.f;

  const int eh = warp % NEH, ks = warp / NEH, lt = lane >> 3, le = lane & 7;
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  double ssp = 0.0;                     // partial sum x^2 of row tid/8 (8 values per chunk)
  const int srow = tid >> 3, scol = (tid & 7) * 8;

  for (int it = 0; it < nch; ++it) {
    const float* buf = stage0 + (it % NS) * BUF;
    cp_async_wait<NS - 2>();
    __syncthreads();
    if (it + NS - 1 < nch) issue_chunk((it + NS - 1) * DC, stage0 + ((it + NS - 1) % NS) * BUF);
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
      float2 a[8], b0[4], b1[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float2*>(xa + 4 * i * LDS + kk);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        b0[j] = *reinterpret_cast<const float2*>(wb + kk * EP + 16 * j);
        b1[j] = *reinterpret_cast<const float2*>(wb + (kk + 1) * EP + 16 * j);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
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
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<float2*>(&red[(ks * TB + lt + 4 * i) * EP + eh * 64 + 2 * le + 16 * j]) = acc[i][j];
  // per-row sum x^2: the 8 threads of a row are consecutive lanes
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) ssp += __shfl_xor_sync(0xffffffff, ssp, o);
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
    lg[tt * (EP + 1) + e] = s * s_r[tt];
  }
  __syncthreads();
  RSTAMP(2);
  float wm = 0.f;
  for (int e = lane; e < E; e += 32) wm = fmaxf(wm, s_wsq[e]);
  const float wmax = sqrtf(warp_max_f32(wm)) * 1.01f;
  const float chain = (float)(d / KS + KS + 6);
  if (warp < 4) {            // warps 0-3 select while warps 4-7 write xn
    for (int tt = warp; tt < rows; tt += 4)
      select_token<EW>(lg + tt * (EP + 1), t0 + tt, s_r[tt] * chain * kU * s_xn[tt] * wmax, L, lane);
  } else {
    write_xn(L, t0, rows, s_r, tid - 128, 128);
  }
  RSTAMP(3);
  __syncthreads();
  RSTAMP(4);
}

// E <= 32: 4 warps, 4x4 tile per lane (tokens lt + 4i + 16 wt, experts le + 8j), k split in halves.
__global__ void __launch_bounds__(128) router_kernel_small(RouterLaunch L) {
  constexpr int EP = 32, NT = 128, XV = TB * DC / 4 / NT, WV = EP * DC / 4 / NT;
  constexpr int BUF = (TB + EP) * LDS, NS = 4;
  extern __shared__ __align__(16) float sm[];
  float* stage0 = sm;
  float* lg = sm;                      // [TB][EP+1]
  float* red = sm + TB * (EP + 1);     // [TB][EP]
  float* s_r = sm + NS * BUF;
  float* s_xn = s_r + TB;
  float* s_wsq = s_xn + TB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = L.T, d = L.d, E = L.E;
  const long t0 = (long)blockIdx.x * TB;
  const float* __restrict__ x = L.x;
  const float* __restrict__ W = L.w_scaled;
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
      const int i = tid + v * NT;
      const int e = i / (DC / 4), cc = (i % (DC / 4)) * 4;
      cp_async16(buf + (TB + e) * LDS + cc, W + (long)(e < E ? e : 0) * d + c0 + cc, e < E);
    }
    cp_async_commit();
  };
  const int nch = d / DC;
#pragma unroll
  for (int i = 0; i < NS - 1; ++i) {
    if (i < nch) issue_chunk(i * DC, stage0 + i * BUF);
    else cp_async_commit();
  }
  for (int e = tid; e < EP; e += NT) s_wsq[e] = e < E ? L.w_sq[e] : 0.f;
  const int kg = warp >> 1, wt = warp & 1, lt = lane >> 3, le = lane & 7;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  double ssp = 0.0;
  const int srow = tid >> 2, scol = (tid & 3) * 16;
  for (int it = 0; it < nch; ++it) {
    const float* buf = stage0 + (it % NS) * BUF;
    cp_async_wait<NS - 2>();
    __syncthreads();
    if (it + NS - 1 < nch) issue_chunk((it + NS - 1) * DC, stage0 + ((it + NS - 1) % NS) * BUF);
    else cp_async_commit();
#pragma unroll
    for (int c = 0; c < 16; c += 4) {
      const float4 p = *reinterpret_cast<const float4*>(buf + srow * LDS + scol + c);
      ssp += ((double)p.x * p.x + (double)p.y * p.y) + ((double)p.z * p.z + (double)p.w * p.w);
    }
    const float* xa = buf + (16 * wt + lt) * LDS + kg * (DC / 2);
    const float* wb = buf + (TB + le) * LDS + kg * (DC / 2);
#pragma unroll
    for (int kk = 0; kk < DC / 2; kk += 2) {
      float2 a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = *reinterpret_cast<const float2*>(xa + 4 * i * LDS + kk);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = *reinterpret_cast<const float2*>(wb + 8 * j * LDS + kk);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j] = fmaf(a[i].x, b[j].x, acc[i][j]);
          acc[i][j] = fmaf(a[i].y, b[j].y, acc[i][j]);
        }
    }
  }
  __syncthreads();
#pragma unroll
  for (int o = 2; o > 0; o >>= 1) ssp += __shfl_xor_sync(0xffffffff, ssp, o);
  if ((tid & 3) == 0) {
    s_r[srow] = (float)(1.0 / sqrt(ssp / (double)d + (double)L.eps));
    s_xn[srow] = (float)sqrt(ssp) * 1.0001f;
  }
  if (kg == 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) red[(16 * wt + lt + 4 * i) * EP + le + 8 * j] = acc[i][j];
  }
  __syncthreads();
  if (kg == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int tt = 16 * wt + lt + 4 * i;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        lg[tt * (EP + 1) + le + 8 * j] = (acc[i][j] + red[tt * EP + le + 8 * j]) * s_r[tt];
    }
  }
  __syncthreads();
  float wm = 0.f;
  for (int e = lane; e < E; e += 32) wm = fmaxf(wm, s_wsq[e]);
  const float wmax = sqrtf(warp_max_f32(wm)) * 1.01f;
  const float chain = (float)(d / 2 + 8);
  for (int tt = warp; tt < TB; tt += 4) {
    const long t = t0 + tt;
    if (t >= T) break;
    select_token<1>(lg + tt * (EP + 1), t, s_r[tt] * chain * kU * s_xn[tt] * wmax, L, lane);
  }
  write_xn(L, t0, (int)min((long)TB, (long)T - t0), s_r, tid, NT);
}

// Band refinement (one CTA per flagged token, grid-stride): warp 0 classifies the
// experts against the token's fp32 band (certainly in / band / certainly out);
// the 8 warps compute the fp64 raw dots sum_i x_i gamma_i W_ei of the band experts
// (the positive factor r_t does not change their order); warp 0 then fills the
// k - |certain| open slots with the best band experts (fp64 value, ties -> lower
// id) and writes indices and gates (fp32 logits, as for every other token). The
// last CTA resets the flag list for the next call.
template <int QN>
__global__ void __launch_bounds__(256) router_refine_kernel(RouterLaunch L) {
  __shared__ int s_band[128];
  __shared__ int s_nb;
  __shared__ double s_l64[128];
  __shared__ double s_red[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = L.d, E = L.E, k = L.k;
  const int n = *reinterpret_cast<volatile int*>(&L.rf_ctrl[0]);
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const long t = L.rf_list[i];
    const float thr2 = L.rf_thr[3 * i], hi = L.rf_thr[3 * i + 1], lo = L.rf_thr[3 * i + 2];
    float v[QN];
    uint32_t sel = 0, band = 0;
    if (warp == 0) {
      int nb = 0;
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        const int e = lane + 32 * q;
        v[q] = e < E ? L.rf_lg[(long)i * E + e] : -FLT_MAX;
        const bool in = e < E && v[q] > hi + thr2;
        const bool bnd = e < E && !in && !(v[q] < lo - thr2);
        if (in) sel |= 1u << q;
        if (bnd) band |= 1u << q;
        const uint32_t m = __ballot_sync(0xffffffff, bnd);
        if (bnd) s_band[nb + __popc(m & ((1u << lane) - 1u))] = e;
        nb += __popc(m);
      }
      if (lane == 0) s_nb = nb;
    }
    __syncthreads();
    const int nb = s_nb;
    const float* xr = L.x + t * d;
    for (int b = 0; b < nb; ++b) {            // all 256 threads on one band expert at a time
      const int e = s_band[b];
      const float* wr = L.w_router + (long)e * d;
      double acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = 0.0;
      for (int c0 = 0; c0 < d; c0 += 2048) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + tid + 256 * u;
          if (c < d) acc[u] = fma((double)xr[c] * (double)L.gamma[c], (double)wr[c], acc[u]);
        }
      }
      double sum = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      sum = warp_sum_f64(sum);
      if (lane == 0) s_red[warp] = sum;
      __syncthreads();
      if (tid == 0) {
        double tot = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) tot += s_red[w];
        s_l64[e] = tot;
      }
      __syncthreads();
    }
    if (warp == 0) {
      double l64[QN];
#pragma unroll
      for (int q = 0; q < QN; ++q) l64[q] = ((band >> q) & 1u) ? s_l64[lane + 32 * q] : -DBL_MAX;
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
    __syncthreads();
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&L.rf_ctrl[1], 1) == (int)gridDim.x - 1) {
      L.rf_ctrl[0] = 0;
      L.rf_ctrl[1] = 0;
      __threadfence();
    }
  }
}

template <int EW>
static cudaError_t launch_router_t(const RouterLaunch& L, cudaStream_t s) {
  RouterLaunch LL = L;
  LL.rpb = TB;
  if constexpr (EW > 1) {   // balance the grid: exactly 2 CTAs per SM when T is large
    const int want = 2 * kNumSMs;
    LL.rpb = (L.T + want - 1) / want;
    if (LL.rpb > TB) LL.rpb = TB;
    if (LL.rpb < 1) LL.rpb = 1;
  }
  const int grid = (L.T + LL.rpb - 1) / LL.rpb;
  g_launches += 3;
  constexpr int EPAD = 32 * EW;
  router_prescale_kernel<<<EW == 1 ? L.E : EPAD, 256, 0, s>>>(L.w_router, L.gamma, L.w_scaled, L.w_sq, L.E, L.d,
                                                              EW == 1 ? 0 : EPAD);
  if constexpr (EW == 1) {
    constexpr int NS = 4, EP = 32;
    const size_t smem = (size_t)(NS * (TB + EP) * LDS + 2 * TB + EP) * 4 + 16;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(router_kernel_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    router_kernel_small<<<grid, 128, smem, s>>>(LL);
  } else {
    constexpr int EP = 32 * EW, NS = EW >= 4 ? 3 : 4;
    const size_t smem = (size_t)(NS * (TB * LDS + DC * EP) + 2 * TB + EP) * 4 + 16;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(router_kernel<EW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    router_kernel<EW><<<grid, 256, smem, s>>>(LL);
  }
  router_refine_kernel<EW><<<kNumSMs, 256, 0, s>>>(L);
  return cudaGetLastError();
}

cudaError_t launch_router(const RouterLaunch& L, cudaStream_t s) {
  if (L.T == 0) return cudaSuccess;
  if (L.d % DC || L.d > kMaxD || L.E < 1 || L.E > 128 || L.k < 1 || L.k > L.E) return cudaErrorInvalidValue;
  if (!L.rf_list || !L.rf_ctrl || !L.rf_l64 || !L.rf_lg || !L.rf_thr || !L.w_scaled || !L.w_sq)
    return cudaErrorInvalidValue;
  if (L.E <= 32) return launch_router_t<1>(L, s);
  if (L.E <= 64) return launch_router_t<2>(L, s);
  return launch_router_t<4>(L, s);
}

}  // namespace fsc
