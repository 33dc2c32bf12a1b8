// K1: fused RMSNorm + fp32 router logits + top-k + renormalised gates.
//
//   r_t   = (mean_i x_ti^2 + eps)^-1/2                  (RMSNorm, C-amb-5; sum of squares in fp64)
//   xn_t  = x_t * gamma * r_t  -> bf16 (expert GEMM operand)
//   l_te  = r_t * sum_i (x_ti gamma_i) W_R[e,i]          (G(A) = s(A W_R^T))
//   S_t   = top-k of l_t, exact ties -> lower expert id; slots ascending by id (C-amb-3)
//   g_tj  = exp(l_tj - max) / sum_{S_t} exp(l - max)     (softmax over E then renormalise
//                                                         == softmax over the selected logits)
// Near-tie refinement: the fp32 logits carry an error
// bounded by B_t = r_t * 100u * ||x_t*gamma||_2 * max_e ||W_R[e]||_2
// (two-level fp32 sum: 64-term chunks + d/64 chunk adds, Cauchy-Schwarz). A token
// whose fp32 boundary gap l_(k) - l_(k+1) is within 2 B_t (+ slack) is recomputed
// by its warp in fp64 and re-selected, so the selection equals the fp64
// selection for every token whose true gap exceeds the fp64 rounding.
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
}  // namespace

template <int JE>
__global__ void __launch_bounds__(256) router_kernel(RouterLaunch L) {
  constexpr int EP = 16 * JE;          // experts padded to a multiple of 16
  constexpr int QN = (EP + 31) / 32;   // logits per lane in the selection phase
  extern __shared__ __align__(16) float sm[];
  float* xs = sm;                      // [TB][LDS]   x*gamma chunk
  float* ws = xs + TB * LDS;           // [EP][LDS]   W_R chunk
  float* lg = ws + EP * LDS;           // [TB][EP+1]  fp32 logits
  float* s_r = lg + TB * (EP + 1);     // [TB]
  float* s_xgn = s_r + TB;             // [TB]
  float* s_wsq = s_xgn + TB;           // [EP]
  double* s_ss = reinterpret_cast<double*>(s_wsq + EP);  // [TB] sum x^2 (fp64)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = L.T, d = L.d, E = L.E, k = L.k;
  const long t0 = (long)blockIdx.x * TB;
  const float* __restrict__ x = L.x;
  const float* __restrict__ gamma = L.gamma;
  const float* __restrict__ W = L.w_router;

  // ---- phase A: per-token sum of squares (fp64) and ||x*gamma|| (bound only)
  for (int i = 0; i < TB / 8; ++i) {
    const int tt = warp * (TB / 8) + i;
    const long t = t0 + tt;
    double ss = 0.0;
    float xg2 = 0.f;
    if (t < T) {
      const float* xr = x + t * d;
      for (int c = lane * 4; c < d; c += 128) {
        float4 v = *reinterpret_cast<const float4*>(xr + c);
        float4 g = *reinterpret_cast<const float4*>(gamma + c);
        ss += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
        float a = v.x * g.x, b = v.y * g.y, cc = v.z * g.z, dd = v.w * g.w;
        xg2 += a * a + b * b + cc * cc + dd * dd;
      }
    }
    ss = warp_sum_f64(ss);
    xg2 = warp_sum_f32(xg2);
    if (lane == 0) {
      s_ss[tt] = ss;
      s_r[tt] = (float)(1.0 / sqrt(ss / (double)d + (double)L.eps));
      s_xgn[tt] = sqrtf(xg2);
    }
  }
  __syncthreads();

  // ---- phase B: register-tiled fp32 logits, two-level accumulation
  const int ty = tid >> 4, tx = tid & 15;
  float tot[2][JE], wsq[JE];
#pragma unroll
  for (int j = 0; j < JE; ++j) { tot[0][j] = tot[1][j] = 0.f; wsq[j] = 0.f; }

  for (int c0 = 0; c0 < d; c0 += DC) {
    for (int i = tid; i < TB * DC / 4; i += 256) {
      const int tt = i / (DC / 4), cc = (i % (DC / 4)) * 4;
      const long t = t0 + tt;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < T) v = *reinterpret_cast<const float4*>(x + t * d + c0 + cc);
      const float4 g = *reinterpret_cast<const float4*>(gamma + c0 + cc);
      float4 xg = make_float4(v.x * g.x, v.y * g.y, v.z * g.z, v.w * g.w);
      *reinterpret_cast<float4*>(xs + tt * LDS + cc) = xg;
      if (t < T) {
        const float r = s_r[tt];
        uint2 o = make_uint2(pack_bf16x2(xg.x * r, xg.y * r), pack_bf16x2(xg.z * r, xg.w * r));
        *reinterpret_cast<uint2*>(L.xn + t * d + c0 + cc) = o;
      }
    }
    for (int i = tid; i < EP * DC / 4; i += 256) {
      const int e = i / (DC / 4), cc = (i % (DC / 4)) * 4;
      float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < E) w = *reinterpret_cast<const float4*>(W + (long)e * d + c0 + cc);
      *reinterpret_cast<float4*>(ws + e * LDS + cc) = w;
    }
    __syncthreads();
    float part[2][JE];
#pragma unroll
    for (int j = 0; j < JE; ++j) part[0][j] = part[1][j] = 0.f;
#pragma unroll 4
    for (int kk = 0; kk < DC; kk += 4) {
      const float4 a0 = *reinterpret_cast<const float4*>(xs + ty * LDS + kk);
      const float4 a1 = *reinterpret_cast<const float4*>(xs + (ty + 16) * LDS + kk);
#pragma unroll
      for (int j = 0; j < JE; ++j) {
        const float4 b = *reinterpret_cast<const float4*>(ws + (tx + 16 * j) * LDS + kk);
        part[0][j] = fmaf(a0.x, b.x, part[0][j]);
        part[0][j] = fmaf(a0.y, b.y, part[0][j]);
        part[0][j] = fmaf(a0.z, b.z, part[0][j]);
        part[0][j] = fmaf(a0.w, b.w, part[0][j]);
        part[1][j] = fmaf(a1.x, b.x, part[1][j]);
        part[1][j] = fmaf(a1.y, b.y, part[1][j]);
        part[1][j] = fmaf(a1.z, b.z, part[1][j]);
        part[1][j] = fmaf(a1.w, b.w, part[1][j]);
        if (ty == 0) wsq[j] += b.x * b.x + b.y * b.y + b.z * b.z + b.w * b.w;
      }
    }
#pragma unroll
    for (int j = 0; j < JE; ++j) { tot[0][j] += part[0][j]; tot[1][j] += part[1][j]; }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < JE; ++j) {
    lg[ty * (EP + 1) + tx + 16 * j] = tot[0][j] * s_r[ty];
    lg[(ty + 16) * (EP + 1) + tx + 16 * j] = tot[1][j] * s_r[ty + 16];
    if (ty == 0) s_wsq[tx + 16 * j] = wsq[j];
  }
  __syncthreads();

  // ---- phase C: per-token top-k (one warp per token)
  float wm = 0.f;
  for (int e = lane; e < E; e += 32) wm = fmaxf(wm, s_wsq[e]);
  const float wmax = sqrtf(warp_max_f32(wm)) * 1.01f;

  for (int i = 0; i < TB / 8; ++i) {
    const int tt = warp * (TB / 8) + i;
    const long t = t0 + tt;
    if (t >= T) break;
    float v[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const int e = lane + 32 * q;
      v[q] = (e < E) ? lg[tt * (EP + 1) + e] : -FLT_MAX;
    }
    if (L.logits) {
      for (int e = lane; e < E; e += 32) L.logits[t * E + e] = lg[tt * (EP + 1) + e];
    }
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
      const float B = s_r[tt] * 100.f * kU * s_xgn[tt] * wmax;
      const float thr = 2.f * B + 4.f * kU * (fabsf(vk) + fabsf(vk1)) + 1e-7f;
      refine = gap <= thr;
    }
    const float* xr = x + t * d;
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
    } else {
      // fp64 recomputation of every logit of this token, then re-selection
      if (lane == 0 && L.n_refined) atomicAdd(L.n_refined, 1);
      const double rinv = 1.0 / sqrt(s_ss[tt] / (double)d + (double)L.eps);
      double l64[QN];
#pragma unroll
      for (int q = 0; q < QN; ++q) l64[q] = -DBL_MAX;
      for (int e = 0; e < E; ++e) {
        const float* wr = W + (long)e * d;
        double s = 0.0;
        for (int c = lane; c < d; c += 32) s += (double)xr[c] * (double)gamma[c] * (double)wr[c];
        s = warp_sum_f64(s) * rinv;
        if ((e & 31) == lane) {
#pragma unroll
          for (int q = 0; q < QN; ++q)
            if ((e >> 5) == q) l64[q] = s;
        }
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
  }
}

template <int JE>
static cudaError_t launch_router_t(const RouterLaunch& L, cudaStream_t s) {
  constexpr int EP = 16 * JE;
  const size_t smem = (size_t)(TB * LDS + EP * LDS + TB * (EP + 1) + 2 * TB + EP) * 4 + TB * 8 + 16;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(router_kernel<JE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = (L.T + TB - 1) / TB;
  router_kernel<JE><<<grid, 256, smem, s>>>(L);
  return cudaGetLastError();
}

cudaError_t launch_router(const RouterLaunch& L, cudaStream_t s) {
  if (L.T == 0) return cudaSuccess;
  if (L.d % DC || L.E < 1 || L.E > 128 || L.k < 1 || L.k > L.E) return cudaErrorInvalidValue;
  if (L.E <= 16) return launch_router_t<1>(L, s);
  if (L.E <= 32) return launch_router_t<2>(L, s);
  if (L.E <= 64) return launch_router_t<4>(L, s);
  return launch_router_t<8>(L, s);
}

}  // namespace fsc
