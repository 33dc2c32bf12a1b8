// K1 for small batches (decode): RMSNorm + router logits + top-k + gates in fp64.
//
//   l_te = r_t * sum_i x_ti (gamma_i W_R[e][i])          (G(A) = s(A W_R^T))
//   r_t  = (mean_i x_ti^2 + eps)^-1/2,  xn_t = bf16(x_t gamma r_t)   (C-amb-5)
//   S_t  = top-k of l_t (exact ties -> lower id; slots ascending by id, C-amb-3)
//   g_tj = exp(l_tj - max_S l) / sum_S exp(l - max_S l)  (softmax then renormalise)
//
// Why a separate kernel: at decode sizes (T <= ~1k tokens) the exact tensor-core router
// (router.cu) is a chain of latency-bound phases on a handful of 128-token tiles (TMA
// ring, digit planes, TMEM, fp32 selection with an error bound, fp64 band refinement).
// Here the whole contraction is done in fp64 (DFMA, 64 / clk / SM on B200): gamma_i
// W_R[e][i] is an exact fp64 product of two fp32 values, every sum is an fp64 sum in a
// fixed order, so the selection equals the fp64 oracle's (the oracle sums in another
// order: the two differ by ~1e-16 relative, far inside the R-1 gap of 1e-6) with no
// error bound, band or refinement.
//
// Structure: one cluster of CS CTAs per tile of TT = 8 WT tokens; CTA c owns the
// d-slice [c d/CS, (c+1) d/CS) and streams it in 32-column chunks. Per chunk, every
// thread converts its part of the next chunk (x -> fp64, gamma W_R -> fp64 in k-major
// [32][EP] layout) from registers loaded one chunk ahead, while the 4 warps run the
// DFMA loop of the current one: warp (g, kp) owns tokens 8g..8g+7 and every KW-th
// quarter of the chunk's columns; lane l accumulates experts l + 32 j (j < EP / 32) of
// its 8 tokens (x read as shared-memory broadcasts, W' as conflict-free rows). The
// exact-order reductions: warps' column parts (kp ascending), then the CTAs' d-slices
// (cluster rank ascending, over DSMEM); r_t likewise from the CTAs' sums of x^2. Token
// t of the tile is finished (logits, selection, gates) by cluster rank t % CS; every
// CTA writes xn for its own d-slice.
#include <float.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>

#include "common.cuh"
#include "kernels.h"

namespace fsc {

namespace {
constexpr int F_THREADS = 256;
constexpr int F_DK = 64;          // columns per chunk
constexpr int F_XS = F_DK + 2;    // fp64 row stride of the x chunk (16-byte aligned rows)
constexpr int F_MAX_CS = 16;

FSC_DEVINL double ldc_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
FSC_DEVINL double2 ldc_f64x2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
FSC_DEVINL void cl_arrive_release() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
FSC_DEVINL void cl_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
FSC_DEVINL double sanitize(double v) { return fabs(v) <= DBL_MAX ? v : -DBL_MAX; }
FSC_DEVINL void gdc_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
FSC_DEVINL void gdc_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
FSC_DEVINL void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// fp64 tensor-core step (DMMA): D[8x8] += A[8x4] B[4x8]; per lane a = A[g][q], b = B[q][g],
// c = D[g][2q .. 2q+1] with g = lane / 4, q = lane % 4
FSC_DEVINL void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

#ifdef FSC_ROUTER_PROF   // per-CTA phase stamps (%globaltimer) into L.logits (tools/router_f64_prof.py)
#define F64STAMP(kk)                                                                          \
  if (threadIdx.x == 0) {                                                                     \
    unsigned long long g__;                                                                   \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g__));                                   \
    reinterpret_cast<unsigned long long*>(L.logits)[blockIdx.x * 8 + (kk)] = g__;             \
  }
#else
#define F64STAMP(kk)
#endif

template <int EP, int WT>
struct F64Cfg {
  static constexpr int TE = EP / 32;                // experts per lane (SIMT variant)
  static constexpr int NT = EP / 8;                 // 8-expert MMA tiles (DMMA variant)
  static constexpr int WS = EP + 8;                 // W' row stride (doubles): DMMA B loads conflict-free
  static constexpr int KW = 8 / WT;                 // warps splitting a chunk's columns
  static constexpr int TT = 8 * WT;                 // tokens per tile
  static constexpr int KWC = F_DK / KW;             // columns per warp per chunk
  static constexpr int NXV = TT / 4;                // x values per thread per chunk
  static constexpr int XTPR = F_DK / NXV;           // threads per x row
  static constexpr int KPT = F_DK * EP / F_THREADS; // W' k-values per thread per chunk
  static constexpr int WBUF = F_DK * WS;            // doubles per W' chunk buffer
  static constexpr int XBUF = TT * F_XS;            // doubles per x chunk buffer
  // dynamic smem: 2 W' buffers | 2 x buffers | gamma slice (floats)
  // after the loop the W' buffers hold the partials [KW][TT][EP] and the owned logits
  static constexpr int PART = KW * TT * EP;         // == 64 EP
  static_assert(PART + TT * EP <= 2 * WBUF, "partials + logits must fit the W' buffers");
  static size_t smem(int dsl) { return (size_t)(2 * WBUF + 2 * XBUF) * 8 + (size_t)dsl * 4; }
};
}  // namespace

template <int EP, int WT, bool MMA>
__global__ void __launch_bounds__(F_THREADS, 1) router_f64_kernel(RouterLaunch L, int cs) {
  using C = F64Cfg<EP, WT>;
  extern __shared__ __align__(16) uint8_t f64_smem[];
  double* wbuf = reinterpret_cast<double*>(f64_smem);                    // [2][F_DK][EP]
  double* xbuf = wbuf + 2 * C::WBUF;                                     // [2][TT][F_XS]
  float* gsl = reinterpret_cast<float*>(xbuf + 2 * C::XBUF);             // [dsl]
  __shared__ double s_ssq[C::TT];     // this CTA's sum of x^2 over its d-slice
  __shared__ double s_r[C::TT];       // r_t (identical in every CTA of the cluster)
  __shared__ __align__(8) uint64_t s_full[2];   // W' chunk buffers filled (bulk copy tx)

  F64STAMP(0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = cs > 1 ? (int)cluster_ctarank() : 0;
  const int tile = blockIdx.x / cs;
  const int d = L.d, E = L.E, T = L.T;
  const int dsl = d / cs, col0 = rank * dsl, nch = dsl / F_DK;
  const long t0 = (long)tile * C::TT;

  for (int i = tid; i < dsl / 4; i += F_THREADS)
    reinterpret_cast<float4*>(gsl)[i] = __ldg(reinterpret_cast<const float4*>(L.gamma + col0) + i);

  // ---- per-thread prefetch roles
  // x: row xr, columns [xc, xc + NXV) of each chunk
  const int xr = tid / C::XTPR, xc = (tid % C::XTPR) * C::NXV;
  const bool xvalid = t0 + xr < T;
  const float* xrow = L.x + (t0 + (xvalid ? xr : 0)) * d + col0 + xc;
  float px[C::NXV];
  auto fetch = [&](int ch) {
#pragma unroll
    for (int u = 0; u < C::NXV; u += 2) {
      const float2 v = xvalid ? __ldg(reinterpret_cast<const float2*>(xrow + ch * F_DK + u)) : make_float2(0.f, 0.f);
      px[u] = v.x;
      px[u + 1] = v.y;
    }
  };
  double ssq = 0.0;
  auto stage = [&](int b) {   // registers -> fp64 x chunk buffer (+ sum of x^2)
    double* xb = xbuf + b * C::XBUF + xr * F_XS + xc;
#pragma unroll
    for (int u = 0; u < C::NXV; u += 2) {
      const double a = (double)px[u], c = (double)px[u + 1];
      ssq = fma(a, a, ssq);
      ssq = fma(c, c, ssq);
      *reinterpret_cast<double2*>(xb + u) = make_double2(a, c);
    }
  };
  // W' = gamma (.) W_R in fp64, k-major [d][WS] (router_f64_prep_kernel): one bulk copy per chunk
  const double* wsrc = L.f64_w + (long)col0 * C::WS;
  constexpr uint32_t kWBytes = F_DK * C::WS * 8;
  auto load_w = [&](int ch, int b) {
    mbar_arrive_expect_tx(&s_full[b], kWBytes);
    bulk_g2s(wbuf + b * C::WBUF, wsrc + (long)ch * F_DK * C::WS, kWBytes, &s_full[b]);
  };

  const int g = warp % WT, kp = warp / WT;
  // PAIR (fp64 tensor cores, tiles of >= 16 tokens): warp (g2, eh) of column part kp owns
  // tokens 16 g2 .. 16 g2 + 15 and experts [eh EP/2, (eh + 1) EP/2)
  constexpr bool PAIR = MMA && WT >= 2;
  const int g2 = (warp % WT) % (WT / 2 > 0 ? WT / 2 : 1), eh = (warp % WT) / (WT / 2 > 0 ? WT / 2 : 1);
  constexpr int NACC = MMA ? 2 * C::NT : 8 * C::TE;
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;

  if (tid == 0) {
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    fence_barrier_init();
  }
  fetch(0);
  __syncthreads();   // gamma slice, barriers
  if (tid == 0) {
    gdc_wait();      // W' is written by router_f64_prep_kernel (programmatic dependent launch)
    load_w(0, 0);
  }
  stage(0);
  __syncthreads();
  F64STAMP(1);
  for (int ch = 0; ch < nch; ++ch) {
    const int b = ch & 1;
    if (ch + 1 < nch) {
      if (tid == 0) load_w(ch + 1, b ^ 1);   // buffer b^1 was released by the last __syncthreads
      fetch(ch + 1);
    }
    mbar_wait(&s_full[b], (ch >> 1) & 1);
    const double* xb = xbuf + b * C::XBUF + (g * 8) * F_XS + kp * C::KWC;
    const double* wb = wbuf + b * C::WBUF + kp * C::KWC * C::WS;
    if constexpr (PAIR) {
      // warp = 16 tokens (two 8-row MMA tiles) x one half of the experts: each B fragment
      // feeds two MMAs (2 + NT/2 shared-memory loads per NT MMAs instead of 1 + NT)
      const int gq = lane >> 2, q = lane & 3;
      const double* xa0 = xbuf + b * C::XBUF + (g2 * 16 + gq) * F_XS + kp * C::KWC + q;
      const double* xa1 = xa0 + 8 * F_XS;
      const double* wq = wb + q * C::WS + eh * (EP / 2) + gq;
#pragma unroll 2
      for (int kk = 0; kk < C::KWC; kk += 4) {
        const double a0 = xa0[kk], a1 = xa1[kk];
        double bv[C::NT / 2];
#pragma unroll
        for (int n = 0; n < C::NT / 2; ++n) bv[n] = wq[kk * C::WS + 8 * n];
#pragma unroll
        for (int n = 0; n < C::NT / 2; ++n) {
          dmma_8x8x4(*reinterpret_cast<double(*)[2]>(&acc[2 * n]), a0, bv[n]);
          dmma_8x8x4(*reinterpret_cast<double(*)[2]>(&acc[C::NT + 2 * n]), a1, bv[n]);
        }
      }
    } else if constexpr (MMA) {
      const int gq = lane >> 2, q = lane & 3;
      const double* xa = xb + gq * F_XS + q;
      const double* wq = wb + q * C::WS + gq;
#pragma unroll 2
      for (int kk = 0; kk < C::KWC; kk += 4) {
        const double a = xa[kk];
        double bv[C::NT];
#pragma unroll
        for (int n = 0; n < C::NT; ++n) bv[n] = wq[kk * C::WS + 8 * n];
#pragma unroll
        for (int n = 0; n < C::NT; ++n) dmma_8x8x4(*reinterpret_cast<double(*)[2]>(&acc[2 * n]), a, bv[n]);
      }
    } else {
      const double* wl = wb + lane;
#pragma unroll 4
      for (int kk = 0; kk < C::KWC; kk += 2) {
        double2 xv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[i] = *reinterpret_cast<const double2*>(xb + i * F_XS + kk);
        double w0[C::TE], w1[C::TE];
#pragma unroll
        for (int j = 0; j < C::TE; ++j) {
          w0[j] = wl[kk * C::WS + 32 * j];
          w1[j] = wl[(kk + 1) * C::WS + 32 * j];
        }
        // all first-column FMAs, then all second-column ones: a dependent pair is 8 TE apart
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < C::TE; ++j) acc[i * C::TE + j] = fma(xv[i].x, w0[j], acc[i * C::TE + j]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < C::TE; ++j) acc[i * C::TE + j] = fma(xv[i].y, w1[j], acc[i * C::TE + j]);
      }
    }
    if (ch + 1 < nch) stage(b ^ 1);
    __syncthreads();
  }

  F64STAMP(2);
  // ---- this CTA's partials: [kp][token][EP] over the W' buffers (free after the last sync),
  // then summed over kp (ascending) into slot 0 so the cluster reduction reads one value
  double* part = wbuf;
  if constexpr (PAIR) {
    const int gq = lane >> 2, q = lane & 3;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      double* pr = part + (kp * C::TT + g2 * 16 + mt * 8 + gq) * EP + eh * (EP / 2) + 2 * q;
#pragma unroll
      for (int n = 0; n < C::NT / 2; ++n)
        *reinterpret_cast<double2*>(pr + 8 * n) = make_double2(acc[mt * C::NT + 2 * n], acc[mt * C::NT + 2 * n + 1]);
    }
  } else if constexpr (MMA) {
    const int gq = lane >> 2, q = lane & 3;
    double* pr = part + (kp * C::TT + g * 8 + gq) * EP + 2 * q;
#pragma unroll
    for (int n = 0; n < C::NT; ++n) *reinterpret_cast<double2*>(pr + 8 * n) = make_double2(acc[2 * n], acc[2 * n + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < C::TE; ++j) part[(kp * C::TT + g * 8 + i) * EP + lane + 32 * j] = acc[i * C::TE + j];
  }
  // sum of x^2 of row xr over this slice: the XTPR threads of the row, fixed butterfly order
#pragma unroll
  for (int o = C::XTPR / 2; o > 0; o >>= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
  if (tid % C::XTPR == 0) s_ssq[xr] = ssq;
  if (C::KW > 1) {
    __syncthreads();
    for (int it = tid; it < C::TT * EP; it += F_THREADS) {
      double v = part[it];
#pragma unroll
      for (int q = 1; q < C::KW; ++q) v += part[q * C::TT * EP + it];
      part[it] = v;
    }
  }
  __syncthreads();
  if (cs > 1) cluster_sync();   // every CTA's partials and sums are in its shared memory
  F64STAMP(3);

  // ---- r_t of every token of the tile (rank order: the same value in every CTA); the
  // remote loads are all issued before the adds (one DSMEM latency, not cs of them)
  if (tid < C::TT) {
    double a = s_ssq[tid];
    if (cs > 1) {
      double p[F_MAX_CS];
      const uint32_t adr = smem_u32(&s_ssq[tid]);
#pragma unroll
      for (int c = 0; c < F_MAX_CS; ++c)
        if (c < cs) p[c] = ldc_f64(mapa_shared(adr, c));
      a = 0.0;
#pragma unroll
      for (int c = 0; c < F_MAX_CS; ++c)
        if (c < cs) a += p[c];
    }
    s_r[tid] = 1.0 / sqrt(a / (double)d + (double)L.eps);
  }
  __syncthreads();
  // ---- logits of the owned tokens (t % cs == rank): the CTAs' partials in rank order
  const int nown = rank < C::TT ? (C::TT - rank + cs - 1) / cs : 0;
  double* lg = wbuf + C::PART;   // [nown][EP]
  {
    const uint32_t pbase = smem_u32(part);
    for (int it = tid; it < nown * (EP / 2); it += F_THREADS) {
      const int i = it / (EP / 2), e = 2 * (it - i * (EP / 2));
      const int t = rank + i * cs;
      double v0, v1;
      if (cs > 1) {
        const uint32_t a = pbase + (uint32_t)((t * EP + e) * 8);
        double2 p[F_MAX_CS];
#pragma unroll
        for (int c = 0; c < F_MAX_CS; ++c)
          if (c < cs) p[c] = ldc_f64x2(mapa_shared(a, c));
        v0 = 0.0;
        v1 = 0.0;
#pragma unroll
        for (int c = 0; c < F_MAX_CS; ++c)
          if (c < cs) {
            v0 += p[c].x;
            v1 += p[c].y;
          }
      } else {
        v0 = part[t * EP + e];
        v1 = part[t * EP + e + 1];
      }
      const double r = s_r[t];
      v0 *= r;
      v1 *= r;
      const long tg = t0 + t;
#ifndef FSC_ROUTER_PROF
      if (L.logits && tg < T) {
        if (e < E) L.logits[tg * E + e] = (float)v0;
        if (e + 1 < E) L.logits[tg * E + e + 1] = (float)v1;
      }
#endif
      lg[i * EP + e] = sanitize(v0);
      lg[i * EP + e + 1] = sanitize(v1);
    }
  }
  __syncthreads();
  F64STAMP(4);
  if (cs > 1) cl_arrive_release();   // done reading the peers (their exit waits for it)

  // ---- selection: one warp per owned token; rank_e = #{e' : l_e' > l_e or (= and e' < e)}
  const int k = L.k;
  for (int i = warp; i < nown; i += F_THREADS / 32) {
    const int t = rank + i * cs;
    const long tg = t0 + t;
    if (tg >= T) break;
    const double* row = lg + i * EP;
    double v[C::TE];
    bool sel[C::TE];
#pragma unroll
    for (int j = 0; j < C::TE; ++j) {
      v[j] = lane + 32 * j < E ? row[lane + 32 * j] : -INFINITY;   // (non-finite logits: -DBL_MAX)
      sel[j] = false;
    }
    // k rounds of a warp argmax over (value desc, id asc) of the unselected experts: the
    // order-preserving 64-bit key of the fp64 value (0 = unavailable), reduced exactly in
    // three warp reductions (high word, low word, lowest id among the equal keys)
    unsigned long long key[C::TE];
#pragma unroll
    for (int j = 0; j < C::TE; ++j) {
      const unsigned long long u = (unsigned long long)__double_as_longlong(v[j]);
      key[j] = lane + 32 * j < E ? ((u >> 63) ? ~u : (u | 0x8000000000000000ull)) : 0ull;
    }
    double vmax = 0.0;
    for (int r = 0; r < k; ++r) {
      unsigned long long bk = 0ull;
      int bj = -1;
#pragma unroll
      for (int j = 0; j < C::TE; ++j)
        if (!sel[j] && key[j] > bk) {
          bk = key[j];
          bj = j;
        }
      const uint32_t hi = (uint32_t)(bk >> 32), lo = (uint32_t)bk;
      const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
      const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      const bool cand = bj >= 0 && hi == mh && lo == ml;
      const uint32_t wid = __reduce_min_sync(0xffffffffu, cand ? (uint32_t)(lane + 32 * bj) : 0xffffffffu);
      if (r == 0) {
        const unsigned long long wk = ((unsigned long long)mh << 32) | ml;
        const unsigned long long ub = (wk >> 63) ? (wk & 0x7fffffffffffffffull) : ~wk;
        vmax = __longlong_as_double((long long)ub);
      }
#pragma unroll
      for (int j = 0; j < C::TE; ++j)
        if (wid == (uint32_t)(lane + 32 * j)) sel[j] = true;
    }
    int slot0[C::TE + 1];
    slot0[0] = 0;
#pragma unroll
    for (int j = 0; j < C::TE; ++j) slot0[j + 1] = slot0[j] + __popc(__ballot_sync(0xffffffffu, sel[j]));
    double ex[C::TE], sum = 0.0;
#pragma unroll
    for (int j = 0; j < C::TE; ++j) {
      ex[j] = sel[j] ? exp(v[j] - vmax) : 0.0;
      sum += ex[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
#pragma unroll
    for (int j = 0; j < C::TE; ++j) {
      const uint32_t m = __ballot_sync(0xffffffffu, sel[j]);
      if (sel[j]) {
        const int s = slot0[j] + __popc(m & ((1u << lane) - 1u));
        L.topk_idx[tg * k + s] = lane + 32 * j;
        L.topk_w[tg * k + s] = (float)(ex[j] / sum);
      }
    }
  }

  F64STAMP(5);
  // ---- xn = bf16(x gamma r) of this CTA's d-slice (x re-read, L2 hits; 8 loads in flight)
  {
    const int dv = dsl / 4, n = C::TT * dv;
    for (int base = tid; base < n; base += 8 * F_THREADS) {
      float4 xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int it = base + u * F_THREADS, t = it / dv;
        if (it < n && t0 + t < T)
          xv[u] = __ldg(reinterpret_cast<const float4*>(L.x + (t0 + t) * d + col0) + (it - t * dv));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int it = base + u * F_THREADS, t = it / dv, c4 = it - t * dv;
        if (it < n && t0 + t < T) {
          const float4 gv = reinterpret_cast<const float4*>(gsl)[c4];
          const float rf = (float)s_r[t];
          *reinterpret_cast<uint2*>(L.xn + (t0 + t) * d + col0 + 4 * c4) =
              make_uint2(pack_bf16x2(xv[u].x * gv.x * rf, xv[u].y * gv.y * rf),
                         pack_bf16x2(xv[u].z * gv.z * rf, xv[u].w * gv.w * rf));
        }
      }
    }
  }
  F64STAMP(6);
  if (cs > 1) cl_wait();   // no CTA leaves while a peer may still read its partials
  F64STAMP(7);
}

// W'T[i][e] = gamma_i W_R[e][i] in fp64 (exact: a product of two fp32 values), zero for
// E <= e < WS; one CTA per 16 columns, W_R read coalesced along i, transposed in shared
// memory. Releases the dependent router kernel at once (PDL): it waits only before its
// first W' copy.
__global__ void __launch_bounds__(256) router_f64_prep_kernel(const float* __restrict__ W,
                                                              const float* __restrict__ gamma, int E, int d, int WS,
                                                              double* __restrict__ wt
#ifdef FSC_ROUTER_PROF
                                                              , unsigned long long* st
#endif
) {
  gdc_launch();
#ifdef FSC_ROUTER_PROF
  unsigned long long g0__;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0__));
  if (threadIdx.x == 0) atomicMin(st + 148 * 64 - 2, g0__);
#endif
  constexpr int PC = 16;   // columns per CTA (d / 16 CTAs: the copy is latency-bound)
  __shared__ float tile[128][PC + 1];
  const int k0 = blockIdx.x * PC, tid = threadIdx.x;
  float v[128 * PC / 256];   // every load in flight before the shared-memory stores
#pragma unroll
  for (int u = 0; u < 128 * PC / 256; ++u) {
    const int i = tid + 256 * u, e = i / PC, c = i - e * PC;
    v[u] = e < E ? __ldg(W + (long)e * d + k0 + c) : 0.f;
  }
#pragma unroll
  for (int u = 0; u < 128 * PC / 256; ++u) {
    const int i = tid + 256 * u, e = i / PC, c = i - e * PC;
    tile[e][c] = v[u];
  }
  __syncthreads();
  for (int i = tid; i < PC * WS; i += 256) {
    const int c = i / WS, e = i - c * WS;
    wt[(long)(k0 + c) * WS + e] = e < 128 ? (double)gamma[k0 + c] * (double)tile[e][c] : 0.0;
  }
#ifdef FSC_ROUTER_PROF
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0__));
  if (threadIdx.x == 0) atomicMax(st + 148 * 64 - 1, g0__);
#endif
}

namespace {
template <int EP, int WT>
size_t f64_smem(int d, int cs) { return F64Cfg<EP, WT>::smem(d / cs); }

// Co-resident clusters of a plan (cudaOccupancyMaxActiveClusters: SMs per GPC, CTAs per SM
// by registers and shared memory), per device and d.
template <int EP, int WT>
int f64_max_clusters(int d, int cs) {
  static int cache[8][5][2];   // [device][log2 cs] -> {d, clusters}
  int dev = 0;
  cudaGetDevice(&dev);
  const int ci = cs == 1 ? 0 : cs == 2 ? 1 : cs == 4 ? 2 : cs == 8 ? 3 : 4;
  int* c = cache[dev & 7][ci];
  if (c[0] == d && c[1] > 0) return c[1];
  static std::atomic<unsigned long long> attr{0};
  ensure_smem_attr(router_f64_kernel<EP, WT, true>, (int)F64Cfg<EP, WT>::smem(8192), attr);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * 16);
  cfg.blockDim = dim3(F_THREADS);
  cfg.dynamicSmemBytes = f64_smem<EP, WT>(d, cs);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, router_f64_kernel<EP, WT, true>, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = kNumSMs / (2 * cs) > 0 ? kNumSMs / (2 * cs) : 1;   // conservative
  }
  c[0] = d;
  c[1] = n;
  return n;
}

// Plan = (WT warps of 8 tokens per tile, cluster size CS). Cost model fitted to a sweep of
// every plan on the B200 (tools/f64_plans.sh): a fixed ~10 us plus, per wave of
// co-resident clusters, ~5 us of CTA prologue / epilogue and the chunks of one CTA at 0.1 us +
// 0.06 us per token x EP / 128 (the fp64 tensor-core work of a 64-column chunk). Cluster sizes above 8 are not used
// (16-CTA clusters measured slower: few fit at once).
struct F64Plan {
  int wt, cs;
};
template <int EP>
F64Plan f64_plan(int T, int d) {
  if (const char* env = getenv("FSC_ROUTER_F64_PLAN")) {   // "wt,cs" (A/B runs)
    int a = 0, b = 0;
    if (sscanf(env, "%d,%d", &a, &b) == 2 && (a == 1 || a == 2 || a == 4) && b >= 1 && b <= F_MAX_CS &&
        !(b & (b - 1)) && d % (b * F_DK) == 0)
      return {a, b};
  }
  F64Plan best{1, 1};
  double best_cost = 1e30;
  for (int wt = 1; wt <= 4; wt *= 2) {
    const int tt = 8 * wt, tiles = (T + tt - 1) / tt;
    for (int cs = 1; cs <= 8; cs *= 2) {
      if (d % (cs * F_DK)) break;
      const int maxc = wt == 1 ? f64_max_clusters<EP, 1>(d, cs)
                                : wt == 2 ? f64_max_clusters<EP, 2>(d, cs) : f64_max_clusters<EP, 4>(d, cs);
      const int waves = (tiles + maxc - 1) / maxc;
      const int nch = d / cs / F_DK;
      const double cost = waves * (5.0 + nch * (0.1 + 0.06 * tt * EP / 128.0));   // + per-wave prologue / epilogue
      if (cost < best_cost * 0.999) {
        best_cost = cost;
        best = {wt, cs};
      }
    }
  }
  return best;
}

template <int EP, int WT, bool MMA>
cudaError_t launch_f64_t(const RouterLaunch& L, int cs, cudaStream_t s) {
  using C = F64Cfg<EP, WT>;
  const size_t smem = C::smem(L.d / cs);
  static std::atomic<unsigned long long> attr{0};   // set once for the largest slice (d = 8192, cs = 1)
  if (cudaError_t e = ensure_smem_attr(router_f64_kernel<EP, WT, MMA>, (int)C::smem(8192), attr)) return e;
  if (cs > 8) {
    static std::atomic<unsigned long long> np{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(np.load() & bit)) {
      if (cudaFuncSetAttribute(router_f64_kernel<EP, WT, MMA>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
          cudaSuccess)
        return cudaErrorInvalidValue;
      np.fetch_or(bit);
    }
  }
  const int tiles = (L.T + C::TT - 1) / C::TT;
  {   // the prep kernel runs with the maximum shared-memory carveout: an SM holding a prep CTA
      // with a small-smem configuration could not take the router's CTA (PDL overlap lost)
    static std::atomic<unsigned long long> co{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(co.load() & bit) &&
        cudaFuncSetAttribute(router_f64_prep_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100) ==
            cudaSuccess)
      co.fetch_or(bit);
  }
  router_f64_prep_kernel<<<L.d / 16, 256, 0, s>>>(L.w_router, L.gamma, L.E, L.d, C::WS, L.f64_w
#ifdef FSC_ROUTER_PROF
                                                   , reinterpret_cast<unsigned long long*>(L.logits)
#endif
  );
  ++g_launches;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles * cs);
  cfg.blockDim = dim3(F_THREADS);
  cfg.dynamicSmemBytes = smem;
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
  ++g_launches;
  return cudaLaunchKernelEx(&cfg, router_f64_kernel<EP, WT, MMA>, L, cs);
}

template <int EP>
cudaError_t launch_f64_ep(const RouterLaunch& L, cudaStream_t s) {
  const F64Plan p = f64_plan<EP>(L.T, L.d);
  const char* se = getenv("FSC_ROUTER_F64_SIMT");   // A/B: the DFMA (SIMT) contraction
  const int simt = se ? atoi(se) : 0;
  if (simt) {
    if (p.wt == 4) return launch_f64_t<EP, 4, false>(L, p.cs, s);
    if (p.wt == 2) return launch_f64_t<EP, 2, false>(L, p.cs, s);
    return launch_f64_t<EP, 1, false>(L, p.cs, s);
  }
  if (p.wt == 4) return launch_f64_t<EP, 4, true>(L, p.cs, s);
  if (p.wt == 2) return launch_f64_t<EP, 2, true>(L, p.cs, s);
  return launch_f64_t<EP, 1, true>(L, p.cs, s);
}
}  // namespace

bool router_f64_supported(int d, int E, int k) { return d % F_DK == 0 && d <= 8192 && E >= 1 && E <= 128 && k >= 1 && k <= E; }

cudaError_t launch_router_f64(const RouterLaunch& L, cudaStream_t s) {
  if (L.T == 0) return cudaSuccess;
  if (!router_f64_supported(L.d, L.E, L.k) || !L.f64_w) return cudaErrorInvalidValue;
  if (L.E <= 32) return launch_f64_ep<32>(L, s);
  if (L.E <= 64) return launch_f64_ep<64>(L, s);
  return launch_f64_ep<128>(L, s);
}

}  // namespace fsc
