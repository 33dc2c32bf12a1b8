// K1: fused RMSNorm + fp32 router logits + top-k + renormalised gates.
//
//   r_t   = (mean_i x_ti^2 + eps)^-1/2                  (RMSNorm, C-amb-5; sum of squares in fp64)
//   xn_t  = x_t * gamma * r_t  -> bf16 (expert GEMM operand)
//   l_te  = r_t * sum_i (x_ti gamma_i) W_R[e,i]          (G(A) = s(A W_R^T))
//   S_t   = top-k of l_t, exact ties -> lower expert id; slots ascending by id (C-amb-3)
//   g_tj  = exp(l_tj - max) / sum_{S_t} exp(l - max)     (softmax over E then renormalise
//                                                         == softmax over the selected logits)
// Near-tie refinement: the fp32 logits carry an error
// bounded by B_t = r_t * (24 + d/64) u * ||x_t*gamma||_2 * max_e ||W_R[e]||_2
// (per chunk of 64: two k-halves x even/odd FFMA2 lanes = 4 chains of 16 products,
// then d/64 chunk adds: chains of <= 16 + 3 + d/64 roundings, +5 for x*gamma, r, the pair sum;
// Cauchy-Schwarz). A token whose fp32 boundary gap l_(k) - l_(k+1) is within
// 2 B_t (+ slack) is recomputed in fp64 (router_refine_*) and re-selected, so the
// selection equals the fp64 selection for every token whose true gap exceeds the
// fp64 rounding.
//
// Layout: block = 256 threads = 32 tokens; the [32 x E] logit tile is a
// register-tiled fp32 SIMT GEMM over d in chunks of 64 staged in shared memory.
#include <float.h>

#include "common.cuh"
#include "kernels.h"

namespace fsc {

namespace {
constexpr int TB = 32;
constexpr int DC = 64;
constexpr int LDS = DC + 4;
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
// packed fp32x2 FMA (sm_100 FFMA2): two lanes of independent fp32 FMAs per instruction
FSC_DEVINL void fma2(float2& acc, float2 a, float2 b) {
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long B = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long C = *reinterpret_cast<unsigned long long*>(&acc);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
  acc = *reinterpret_cast<float2*>(&C);
}
FSC_DEVINL float warp_max_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, o));
  return v;
}
}  // namespace

FSC_DEVINL void cp_async16(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
FSC_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
FSC_DEVINL void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
FSC_DEVINL void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// W'[e][i] = gamma_i * W_R[e][i] (so the logit is sum_i x_i W'[e][i]) and the
// per-expert ||W'_e||^2 used by the near-tie error bound. One warp per expert.
__global__ void __launch_bounds__(256) router_prescale_kernel(const float* __restrict__ W,
                                                              const float* __restrict__ gamma, float* __restrict__ Wg,
                                                              float* __restrict__ wq, int E, int d) {
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (e >= E) return;
  const float4* w = reinterpret_cast<const float4*>(W + (long)e * d);
  const float4* g = reinterpret_cast<const float4*>(gamma);
  float4* o = reinterpret_cast<float4*>(Wg + (long)e * d);
  float s = 0.f;
  for (int c = lane; c < d / 4; c += 32) {
    const float4 a = w[c], b = g[c];
    const float4 v = make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
    o[c] = v;
    s += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  s = warp_sum_f32(s);
  if (lane == 0) wq[e] = s;
}

template <int EW>
__global__ void __launch_bounds__(128 * EW) router_kernel(RouterLaunch L) {
  constexpr int EP = 32 * EW;          // experts padded to a multiple of 32
  constexpr int QN = EW;               // logits per lane in the selection phase
  constexpr int NW = 4 * EW;           // warps: 2 k-halves x 2 token halves x EW expert groups of 32
  constexpr int NT = 32 * NW;
  constexpr int XV = TB * DC / 4 / NT; // float4 of the x chunk per thread
  constexpr int WV = EP * DC / 4 / NT; // float4 of the W chunk per thread
  constexpr int BUF = (TB + EP) * LDS; // one stage: x chunk rows then W' chunk rows
  constexpr int NS = EW >= 4 ? 3 : 4;  // cp.async pipeline depth (chunks in flight)
  extern __shared__ __align__(16) float sm[];
  float* stage0 = sm;                  // [NS][TB+EP][LDS] multi-buffered chunks
  float* lg = sm;                      // [TB][EP+1] fp32 logits (reuses the stages after the loop)
  float* s_r = sm + NS * BUF;          // [TB]
  float* s_xgn = s_r + TB;             // [TB]  ||x_t||_2 (error bound)
  float* s_wsq = s_xgn + TB;           // [EP]  ||W'_e||^2

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = L.T, d = L.d, E = L.E, k = L.k;
  const long t0 = (long)blockIdx.x * TB;
  const float* __restrict__ x = L.x;
  const float* __restrict__ gamma = L.gamma;
  const float* __restrict__ W = L.w_scaled;   // gamma-scaled router weights

#ifdef FSC_ROUTER_PROF
  auto stamp = [&](int kk) {
    if (tid == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      reinterpret_cast<unsigned long long*>(L.logits)[blockIdx.x * 8 + kk] = g;
    }
  };
#else
  auto stamp = [&](int) {};
#endif
  stamp(0);
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
  for (int i = 0; i < NS - 1; ++i) {      // prologue: chunks 0 .. NS-2 in flight
    if (i < nch) issue_chunk(i * DC, stage0 + i * BUF);
    else cp_async_commit();
  }
  for (int e = tid; e < EP; e += NT) s_wsq[e] = e < E ? L.w_sq[e] : 0.f;

  // ---- phase A: r_t (sum x^2 in fp64), ||x_t||, and xn = bf16(x gamma r) written
  // in a second pass over the row (L1/L2 hit); 8 independent 16-byte loads per lane
  for (int tt = warp; tt < TB; tt += NW) {
    const long t = t0 + tt;
    if (t >= T) break;
    const float4* xr = reinterpret_cast<const float4*>(x + t * d);
    const int dv = d / 4;
    double ss = 0.0;
    for (int c = lane; c < dv; c += 256) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (c + 32 * u < dv) ? xr[c + 32 * u] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        ss += ((double)v[u].x * v[u].x + (double)v[u].y * v[u].y) + ((double)v[u].z * v[u].z + (double)v[u].w * v[u].w);
    }
    ss = warp_sum_f64(ss);
    const float r = (float)(1.0 / sqrt(ss / (double)d + (double)L.eps));
    if (lane == 0) {
      s_r[tt] = r;
      s_xgn[tt] = (float)sqrt(ss) * 1.0001f;
    }
    uint2* xo = reinterpret_cast<uint2*>(L.xn + t * d);
    for (int c = lane; c < dv; c += 256) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (c + 32 * u < dv) {
          const float4 v = xr[c + 32 * u];
          const float4 g = reinterpret_cast<const float4*>(gamma)[c + 32 * u];
          xo[c + 32 * u] = make_uint2(pack_bf16x2(v.x * g.x * r, v.y * g.y * r), pack_bf16x2(v.z * g.z * r, v.w * g.w * r));
        }
      }
    }
  }
  stamp(1);

  // ---- phase B: 4x4 register tile per thread, fp32, two-level accumulation.
  // warp: kg = k-half of each chunk, wt = token half, we = expert group of 32;
  // lane: lt = 0..3 tokens, le = 0..7 experts. Thread tokens 16 wt + lt + 4 i,
  // experts 32 we + le + 8 j: every LDS.128 of a warp touches 4 (x) or 8 (W')
  // distinct rows -> one conflict-free wavefront. One barrier per chunk.
  const int kg = warp / (2 * EW), rem = warp % (2 * EW);
  const int wt = rem & 1, we = rem >> 1, lt = lane >> 3, le = lane & 7;
  float tot[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) tot[i][j] = 0.f;

  for (int it = 0; it < nch; ++it) {
    const float* buf = stage0 + (it % NS) * BUF;
    cp_async_wait<NS - 2>();             // chunk `it` has landed (this thread's copies)
    __syncthreads();                     // ... and everyone's; slot it-1 is free again
    if (it + NS - 1 < nch) issue_chunk((it + NS - 1) * DC, stage0 + ((it + NS - 1) % NS) * BUF);
    else cp_async_commit();              // keep the group count uniform
    // even / odd k products accumulate in the two halves of an FFMA2 register pair
    float2 part[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) part[i][j] = make_float2(0.f, 0.f);
    const float* xa = buf + (16 * wt + lt) * LDS + kg * (DC / 2);
    const float* wb = buf + (TB + 32 * we + le) * LDS + kg * (DC / 2);
#pragma unroll
    for (int kk = 0; kk < DC / 2; kk += 4) {
      float4 a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = *reinterpret_cast<const float4*>(xa + 4 * i * LDS + kk);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = *reinterpret_cast<const float4*>(wb + 8 * j * LDS + kk);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          fma2(part[i][j], make_float2(a[i].x, a[i].y), make_float2(b[j].x, b[j].y));
          fma2(part[i][j], make_float2(a[i].z, a[i].w), make_float2(b[j].z, b[j].w));
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) tot[i][j] += part[i][j].x + part[i][j].y;
  }
  __syncthreads();   // all compute done before lg overwrites the stages
  stamp(2);
  // combine the two k-halves in a fixed order: lg = (tot_0 + tot_1) * r
  if (kg == 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) lg[(16 * wt + lt + 4 * i) * (EP + 1) + 32 * we + le + 8 * j] = tot[i][j];
  }
  __syncthreads();
  if (kg == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int tt = 16 * wt + lt + 4 * i;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float* p = &lg[tt * (EP + 1) + 32 * we + le + 8 * j];
        *p = (tot[i][j] + *p) * s_r[tt];
      }
    }
  }
  __syncthreads();
  stamp(3);

  // ---- phase C: per-token top-k (one warp per token)
  float wm = 0.f;
  for (int e = lane; e < E; e += 32) wm = fmaxf(wm, s_wsq[e]);
  const float wmax = sqrtf(warp_max_f32(wm)) * 1.01f;

  for (int tt = warp; tt < TB; tt += NW) {
    const long t = t0 + tt;
    if (t >= T) break;
    float v[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const int e = lane + 32 * q;
      v[q] = (e < E) ? lg[tt * (EP + 1) + e] : -FLT_MAX;
    }
#ifndef FSC_ROUTER_PROF
    if (L.logits) {
      for (int e = lane; e < E; e += 32) L.logits[t * E + e] = lg[tt * (EP + 1) + e];
    }
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
    bool refine = false;
    if (k < E) {
      const float gap = vk - vk1;
      const float B = s_r[tt] * (float)(24 + d / 64) * kU * s_xgn[tt] * wmax;  // chain length + 5, C-S
      const float thr = 2.f * B + 4.f * kU * (fabsf(vk) + fabsf(vk1)) + 1e-7f;
      refine = gap <= thr;
    }
    if (!refine) {
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
    } else if (lane == 0) {
      // near tie: hand the token to router_refine_kernel (fp64 recomputation)
      if (L.n_refined) atomicAdd(L.n_refined, 1);
      L.rf_list[atomicAdd(&L.rf_ctrl[0], 1)] = (int)t;
    }
  }
  __syncthreads();
  stamp(4);
}

// fp64 recomputation of the logits of flagged tokens: one warp per (token, expert),
// eight independent accumulators per lane so 8 W loads are in flight per step.
// Stores the raw dot sum_i (x_i gamma_i) W_ei (exact fp64 products of fp32 inputs).
__global__ void __launch_bounds__(256) router_refine_logits_kernel(RouterLaunch L) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int d = L.d, E = L.E;
  const int n = *reinterpret_cast<volatile int*>(&L.rf_ctrl[0]);
  for (int item = gw; item < n * E; item += nw) {
    const long t = L.rf_list[item / E];
    const int e = item % E;
    const float* xr = L.x + t * d;
    const float* wr = L.w_router + (long)e * d;
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    for (int c0 = 0; c0 < d; c0 += 256) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + lane + 32 * u;
        if (c < d) acc[u] = fma((double)xr[c] * (double)L.gamma[c], (double)wr[c], acc[u]);
      }
    }
    double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    s = warp_sum_f64(s);
    if (lane == 0) L.rf_l64[item] = s;
  }
}

// Re-selection of the flagged tokens from their fp64 logits (one warp per token);
// the last CTA to finish resets the flag list for the next call.
template <int EW>
__global__ void __launch_bounds__(256) router_refine_select_kernel(RouterLaunch L) {
  constexpr int QN = EW;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int d = L.d, E = L.E, k = L.k;
  const int n = *reinterpret_cast<volatile int*>(&L.rf_ctrl[0]);
  for (int i = gw; i < n; i += nw) {
    const long t = L.rf_list[i];
    const float* xr = L.x + t * d;
    double ss = 0.0;
    for (int c = lane; c < d; c += 32) ss += (double)xr[c] * (double)xr[c];
    ss = warp_sum_f64(ss);
    const double rinv = 1.0 / sqrt(ss / (double)d + (double)L.eps);
    double l64[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const int e = lane + 32 * q;
      l64[q] = e < E ? L.rf_l64[(long)i * E + e] * rinv : -DBL_MAX;
    }
    uint32_t sb = 0;
    double dtop = 0.0;
    for (int rd = 0; rd < k; ++rd) {
      double bv = -DBL_MAX;
      int bi = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        const int e = lane + 32 * q;
        if (e < E && !((sb >> q) & 1u) && (l64[q] > bv || (l64[q] == bv && e < bi))) { bv = l64[q]; bi = e; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffff, bv, o);
        const int oi = __shfl_xor_sync(0xffffffff, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if ((bi & 31) == lane) sb |= 1u << (bi >> 5);
      if (rd == 0) dtop = bv;
    }
    double ex[QN], sum = 0.0;
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      ex[q] = ((sb >> q) & 1u) ? exp(l64[q] - dtop) : 0.0;
      sum += ex[q];
    }
    sum = warp_sum_f64(sum);
    int slot = 0;
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const uint32_t m = __ballot_sync(0xffffffff, (sb >> q) & 1u);
      if ((sb >> q) & 1u) {
        const int s = slot + __popc(m & ((1u << lane) - 1u));
        L.topk_idx[t * k + s] = lane + 32 * q;
        L.topk_w[t * k + s] = (float)(ex[q] / sum);
      }
      slot += __popc(m);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
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
  constexpr int EP = 32 * EW;
  constexpr int NS = EW >= 4 ? 3 : 4;
  const size_t smem = (size_t)(NS * (TB + EP) * LDS + 2 * TB + EP) * 4 + 16;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(router_kernel<EW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = (L.T + TB - 1) / TB;
  g_launches += 4;
  router_prescale_kernel<<<(L.E * 32 + 255) / 256, 256, 0, s>>>(L.w_router, L.gamma, L.w_scaled, L.w_sq, L.E, L.d);
  router_kernel<EW><<<grid, 128 * EW, smem, s>>>(L);
  router_refine_logits_kernel<<<4 * kNumSMs, 256, 0, s>>>(L);
  router_refine_select_kernel<EW><<<16, 256, 0, s>>>(L);
  return cudaGetLastError();
}

cudaError_t launch_router(const RouterLaunch& L, cudaStream_t s) {
  if (L.T == 0) return cudaSuccess;
  if (L.d % DC || L.d > kMaxD || L.E < 1 || L.E > 128 || L.k < 1 || L.k > L.E) return cudaErrorInvalidValue;
  if (!L.rf_list || !L.rf_ctrl || !L.rf_l64 || !L.w_scaled || !L.w_sq) return cudaErrorInvalidValue;
  if (L.E <= 32) return launch_router_t<1>(L, s);
  if (L.E <= 64) return launch_router_t<2>(L, s);
  return launch_router_t<4>(L, s);
}

}  // namespace fsc
