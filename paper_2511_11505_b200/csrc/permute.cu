// K2 (histogram / scan / positions), K3 (permute) and K5 (gate-weighted
// unpermute + far-skip residual add) of the MoE dispatch path.
//
// K2 computes the expert-sorted permutation of the (token, slot) copies that
// the Dispatch of PAPER.md:96-100 needs ("grouped and mapped ... requiring
// permutation of A"), deterministically: within an expert, copies keep
// ascending token order (C-amb-11). Each 32-token chunk is one warp; a warp
// builds, per expert, the 32-bit mask of its lanes that selected the expert
// (atomicOr is order independent), so a copy's rank inside its chunk is
// popc(mask & lanes_below), chunk totals are popc(mask), and a column scan over
// chunks gives every chunk's base. No result depends on atomic ordering.
//
// K5: out[t] = resid[t] + (sum_j w[t,j] * y[pos[t,j]]) with the inner sum
// started at 0 and taken in slot order (C-amb-12), fp32. In the FarSkip wiring
// resid = attn-in_{k+1} and out = mlp-in_{k+1} = o_k.
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace fsc {

namespace {
constexpr int kMaxE = 256;
}

__global__ void __launch_bounds__(256) perm_hist_kernel(const int* __restrict__ idx, int T, int k, int E,
                                                        int* __restrict__ hist, int n_chunks) {
  __shared__ uint32_t mask[8][kMaxE];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 8 + w;
  for (int e = lane; e < E; e += 32) mask[w][e] = 0;
  __syncwarp();
  if (c >= n_chunks) return;
  const int t = c * 32 + lane;
  if (t < T)
    for (int j = 0; j < k; ++j) atomicOr(&mask[w][idx[(long)t * k + j]], 1u << lane);
  __syncwarp();
  for (int e = lane; e < E; e += 32) hist[(long)c * E + e] = __popc(mask[w][e]);
}

// Column scan, one CTA per expert: base[c][e] = sum_{c' < c} hist[c'][e] (local to e),
// counts[e] = column total. Offsets across experts are added by perm_pos_kernel.
__global__ void __launch_bounds__(256) perm_scan_kernel(const int* __restrict__ hist, int* __restrict__ base,
                                                        int* __restrict__ counts, int n_chunks, int E) {
  __shared__ int s_w[8];
  const int e = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n_chunks + 255) / 256;
  const int c0 = tid * per;
  int loc = 0;
  for (int i = 0; i < per; ++i)
    if (c0 + i < n_chunks) loc += hist[(long)(c0 + i) * E + e];
  int inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffff, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  int wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += s_w[w];
  int run = wbase + inc - loc;
  for (int i = 0; i < per; ++i) {
    if (c0 + i < n_chunks) {
      const long off = (long)(c0 + i) * E + e;
      const int h = hist[off];
      base[off] = run;
      run += h;
    }
  }
  if (tid == 255) counts[e] = wbase + inc;
}

__global__ void __launch_bounds__(256) perm_pos_kernel(const int* __restrict__ idx, int T, int k, int E,
                                                       const int* __restrict__ base,
                                                       const int* __restrict__ counts, int* __restrict__ offsets,
                                                       int* __restrict__ pos, int* __restrict__ src_row,
                                                       int n_chunks) {
  __shared__ uint32_t mask[8][kMaxE];
  __shared__ int s_off[kMaxE + 1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    // exclusive scan of the expert totals (E <= 256: 8 per lane)
    int v[8], loc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = lane * 8 + i;
      v[i] = e < E ? counts[e] : 0;
      loc += v[i];
    }
    int inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffff, inc, o);
      if (lane >= o) inc += u;
    }
    int run = inc - loc;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = lane * 8 + i;
      if (e < E) s_off[e] = run;
      run += v[i];
    }
    if (lane == 31) s_off[E] = inc;
  }
  const int c = blockIdx.x * 8 + w;
  for (int e = lane; e < E; e += 32) mask[w][e] = 0;
  __syncthreads();
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e <= E; e += 256) offsets[e] = s_off[e];
  if (c >= n_chunks) return;
  const int t = c * 32 + lane;
  if (t < T)
    for (int j = 0; j < k; ++j) atomicOr(&mask[w][idx[(long)t * k + j]], 1u << lane);
  __syncwarp();
  if (t < T) {
    const uint32_t below = (1u << lane) - 1u;
    for (int j = 0; j < k; ++j) {
      const int e = idx[(long)t * k + j];
      const int p = s_off[e] + base[(long)c * E + e] + __popc(mask[w][e] & below);
      pos[(long)t * k + j] = p;
      src_row[p] = t;
    }
  }
}

// Small T (decode, <= 32 chunks of 32 tokens, E <= 128): the three steps above in ONE
// CTA of 32 warps (warp = chunk): chunk masks, per-expert column scan (one thread per
// expert), exclusive scan of the totals, positions. Same definition, same results; one
// launch instead of three with global round trips in between.
constexpr int kFusedChunks = 32, kFusedE = 128;
__global__ void __launch_bounds__(1024) perm_fused_kernel(const int* __restrict__ idx, int T, int k, int E,
                                                         int* __restrict__ counts, int* __restrict__ offsets,
                                                         int* __restrict__ pos, int* __restrict__ src_row,
                                                         int n_chunks) {
  __shared__ uint32_t mask[kFusedChunks][kFusedE];
  __shared__ int base[kFusedChunks][kFusedE];
  __shared__ int s_cnt[kFusedE];
  __shared__ int s_off[kFusedE + 1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  for (int e = lane; e < E; e += 32) mask[w][e] = 0;
  __syncwarp();
  const int t = w * 32 + lane;
  const bool valid = w < n_chunks && t < T;
  int ids[8];                             // the token's first 8 slots stay in registers
#pragma unroll
  for (int j = 0; j < 8; ++j) ids[j] = valid && j < k ? idx[(long)t * k + j] : 0;
  if (valid) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < k) atomicOr(&mask[w][ids[j]], 1u << lane);
    for (int j = 8; j < k; ++j) atomicOr(&mask[w][idx[(long)t * k + j]], 1u << lane);
  }
  __syncthreads();
  if (tid < E) {                          // column scan over the chunks, chunk order
    int run = 0;
    for (int c = 0; c < n_chunks; ++c) {
      base[c][tid] = run;
      run += __popc(mask[c][tid]);
    }
    s_cnt[tid] = run;
  }
  __syncthreads();
  if (w == 0) {                           // exclusive scan of the expert totals (4 per lane)
    int v[4], loc = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = lane * 4 + i;
      v[i] = e < E ? s_cnt[e] : 0;
      loc += v[i];
    }
    int inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    int run = inc - loc;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = lane * 4 + i;
      if (e < E) {
        s_off[e] = run;
        offsets[e] = run;
        counts[e] = v[i];
      }
      run += v[i];
    }
    if (lane == 31) {
      s_off[E] = inc;
      offsets[E] = inc;
    }
  }
  __syncthreads();
  if (valid) {
    const uint32_t below = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < k) {
        const int e = ids[j];
        const int p = s_off[e] + base[w][e] + __popc(mask[w][e] & below);
        pos[(long)t * k + j] = p;
        src_row[p] = t;
      }
    for (int j = 8; j < k; ++j) {
      const int e = idx[(long)t * k + j];
      const int p = s_off[e] + base[w][e] + __popc(mask[w][e] & below);
      pos[(long)t * k + j] = p;
      src_row[p] = t;
    }
  }
}

cudaError_t launch_perm_maps(const PermLaunch& L, cudaStream_t s) {
  if (L.E > kMaxE || L.E < 1) return cudaErrorInvalidValue;
  const int nc = perm_chunks(L.T);
  if (nc == 0) {
    cudaError_t e = cudaMemsetAsync(L.counts, 0, sizeof(int) * L.E, s);
    if (e != cudaSuccess) return e;
    return cudaMemsetAsync(L.offsets, 0, sizeof(int) * (L.E + 1), s);
  }
  if (nc <= kFusedChunks && L.E <= kFusedE) {
    ++g_launches;
    perm_fused_kernel<<<1, 1024, 0, s>>>(L.topk_idx, L.T, L.k, L.E, L.counts, L.offsets, L.pos, L.src_row, nc);
    return cudaGetLastError();
  }
  const int blocks = (nc + 7) / 8;
  g_launches += 3;
  perm_hist_kernel<<<blocks, 256, 0, s>>>(L.topk_idx, L.T, L.k, L.E, L.hist, nc);
  perm_scan_kernel<<<L.E, 256, 0, s>>>(L.hist, L.base, L.counts, nc, L.E);
  perm_pos_kernel<<<blocks, 256, 0, s>>>(L.topk_idx, L.T, L.k, L.E, L.base, L.counts, L.offsets, L.pos, L.src_row,
                                         nc);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K3 permute
__global__ void __launch_bounds__(256) permute_rows_kernel(const uint4* __restrict__ xn,
                                                           const int* __restrict__ src_row,
                                                           uint4* __restrict__ xs, int R, int dv,
                                                           const int* __restrict__ rng, int rng_n) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long r = (long)blockIdx.x * 8 + w;
  if (r >= R) return;
  if (rng && (r < rng[0] || r >= rng[rng_n])) return;
  const long src = src_row[r];
  const uint4* a = xn + src * dv;
  uint4* b = xs + r * dv;
  // 8 loads in flight per lane before the stores (one row of d = 2048 per warp round):
  // the copy is bound by the bytes in flight per SM, not by instruction issue. xn (read k
  // times, gathered) is kept in L2 (evict_last) while the permuted rows, written once and
  // read back by the GEMM much later, stream through it (evict_first): otherwise the
  // writes evict xn and every gather goes to HBM (Qwen3: 604 MB -> ~1.1 GB of traffic).
  for (int i0 = lane; i0 < dv; i0 += 256) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + 32 * u < dv) v[u] = ld_keep_u4(a + i0 + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + 32 * u < dv) st_stream_u4(b + i0 + 32 * u, v[u]);
  }
}

// Same result as permute_rows_kernel (xs[pos[t, j]] = xn[t]), by SOURCE token: a warp reads
// row t of xn once (streamed, evict-first) and writes it to its k destination rows. Every
// xn byte leaves HBM once whatever the L2 holds: the gather order re-reads xn k times and
// relies on L2 keeping it (Qwen3: 67 MB of xn, evicted by the 537 MB of permuted rows).
__global__ void __launch_bounds__(256) permute_scatter_kernel(const uint4* __restrict__ xn,
                                                              const int* __restrict__ pos,
                                                              uint4* __restrict__ xs, int T, int k, int dv) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long t = (long)blockIdx.x * 8 + w;
  if (t >= T) return;
  int p[8];
  for (int j0 = 0; j0 < k; j0 += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = j0 + j < k ? pos[t * k + j0 + j] : -1;
    const uint4* a = xn + t * dv;
    for (int i0 = lane; i0 < dv; i0 += 256) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + 32 * u < dv) v[u] = ld_stream_u4(a + i0 + 32 * u);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (p[j] < 0) continue;
        uint4* b = xs + (long)p[j] * dv;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + 32 * u < dv) st_stream_u4(b + i0 + 32 * u, v[u]);
      }
    }
  }
}

cudaError_t launch_permute_scatter(const uint16_t* xn, const int* pos, uint16_t* xs, int T, int k, int d,
                                   cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  ++g_launches;
  permute_scatter_kernel<<<(T + 7) / 8, 256, 0, s>>>(reinterpret_cast<const uint4*>(xn), pos,
                                                     reinterpret_cast<uint4*>(xs), T, k, d / 8);
  return cudaGetLastError();
}

// EP = 1 permute: by source token when xn is too large to stay in L2 between its k reads
// (A/B on the B200: Qwen3 prefill, xn 67 MB, 128 -> 103 us, step -24 us), by destination
// row otherwise (DS-V2-Lite, xn 34 MB, beside the shared expert: gather 23 us faster per
// step; decode: more CTAs in flight). FSC_PERMUTE_GATHER=0/1 forces one (A/B runs).
cudaError_t launch_permute_ep1(const uint16_t* xn, const int* src_row, const int* pos, uint16_t* xs, int T, int k,
                               int d, cudaStream_t s) {
  const char* env = getenv("FSC_PERMUTE_GATHER");
  const bool scatter = env ? atoi(env) == 0 : (long)T * d * 2 > (48l << 20);
  return scatter ? launch_permute_scatter(xn, pos, xs, T, k, d, s)
                 : launch_permute_rows(xn, src_row, xs, T * k, d, s);
}

cudaError_t launch_permute_rows(const uint16_t* xn, const int* src_row, uint16_t* xs, int R, int d,
                                cudaStream_t s, const int* rng, int rng_n) {
  if (R == 0) return cudaSuccess;
  const int dv = d / 8;
  ++g_launches;
  permute_rows_kernel<<<(R + 7) / 8, 256, 0, s>>>(reinterpret_cast<const uint4*>(xn), src_row,
                                                  reinterpret_cast<uint4*>(xs), R, dv, rng, rng_n);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K5 unpermute
// One thread per (token, 8 columns), the k slots summed in slot order. (A variant with
// every slot's row load in flight at once measured slower: 78 registers, fewer CTAs per
// SM - DS 63.5 -> 71.7 us, Qwen3 137 -> 141 us.)
__global__ void __launch_bounds__(256) unpermute_kernel(const uint4* __restrict__ y, const int* __restrict__ pos,
                                                               const float* __restrict__ w,
                                                               const float* __restrict__ resid, float* __restrict__ out,
                                                               long items, int dv, int k) {
  for (long it = (long)blockIdx.x * blockDim.x + threadIdx.x; it < items; it += (long)gridDim.x * blockDim.x) {
    const long t = it / dv;
    const int c = (int)(it - t * dv);
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    for (int j = 0; j < k; ++j) {
      const long p = pos[t * k + j];
      const float g = w[t * k + j];
      const uint4 v = y[p * dv + c];
      acc[0] = fmaf(g, bf16lo(v.x), acc[0]);
      acc[1] = fmaf(g, bf16hi(v.x), acc[1]);
      acc[2] = fmaf(g, bf16lo(v.y), acc[2]);
      acc[3] = fmaf(g, bf16hi(v.y), acc[3]);
      acc[4] = fmaf(g, bf16lo(v.z), acc[4]);
      acc[5] = fmaf(g, bf16hi(v.z), acc[5]);
      acc[6] = fmaf(g, bf16lo(v.w), acc[6]);
      acc[7] = fmaf(g, bf16hi(v.w), acc[7]);
    }
    const float4* rr = reinterpret_cast<const float4*>(resid + t * (long)dv * 8 + c * 8);
    float4* oo = reinterpret_cast<float4*>(out + t * (long)dv * 8 + c * 8);
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if (resid) { a = rr[0]; b = rr[1]; }
    a.x += acc[0]; a.y += acc[1]; a.z += acc[2]; a.w += acc[3];
    b.x += acc[4]; b.y += acc[5]; b.z += acc[6]; b.w += acc[7];
    oo[0] = a;
    oo[1] = b;
  }
}

cudaError_t launch_unpermute(const uint16_t* y, const int* pos, const float* w, const float* resid, float* out,
                             int T, int k, int d, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int dv = d / 8;
  const long items = (long)T * dv;
  long blocks = (items + 255) / 256;
  if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
  ++g_launches;
  unpermute_kernel<<<(int)blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(y), pos, w, resid, out, items, dv, k);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) unpermute_local_kernel(const uint4* __restrict__ y, const int* __restrict__ pos,
                                                              const float* __restrict__ w, const int* __restrict__ idx,
                                                              int e_lo, int e_hi, float* __restrict__ out, long items,
                                                              int dv, int k) {
  for (long it = (long)blockIdx.x * blockDim.x + threadIdx.x; it < items; it += (long)gridDim.x * blockDim.x) {
    const long t = it / dv;
    const int c = (int)(it - t * dv);
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    for (int j = 0; j < k; ++j) {
      const int e = idx[t * k + j];
      if (e < e_lo || e >= e_hi) continue;
      const long p = pos[t * k + j];
      const float g = w[t * k + j];
      const uint4 v = y[p * dv + c];
      acc[0] = fmaf(g, bf16lo(v.x), acc[0]);
      acc[1] = fmaf(g, bf16hi(v.x), acc[1]);
      acc[2] = fmaf(g, bf16lo(v.y), acc[2]);
      acc[3] = fmaf(g, bf16hi(v.y), acc[3]);
      acc[4] = fmaf(g, bf16lo(v.z), acc[4]);
      acc[5] = fmaf(g, bf16hi(v.z), acc[5]);
      acc[6] = fmaf(g, bf16lo(v.w), acc[6]);
      acc[7] = fmaf(g, bf16hi(v.w), acc[7]);
    }
    float4* oo = reinterpret_cast<float4*>(out + t * (long)dv * 8 + c * 8);
    oo[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    oo[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

cudaError_t launch_unpermute_local(const uint16_t* y, const int* pos, const float* w, const int* idx, int e_lo,
                                   int e_hi, float* out, int T, int k, int d, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int dv = d / 8;
  const long items = (long)T * dv;
  long blocks = (items + 255) / 256;
  if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
  ++g_launches;
  unpermute_local_kernel<<<(int)blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(y), pos, w, idx, e_lo, e_hi, out,
                                                     items, dv, k);
  return cudaGetLastError();
}

__global__ void copy_f32_kernel(const float4* __restrict__ a, float4* __restrict__ b, long n4) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}

cudaError_t launch_copy_f32(const float* src, float* dst, long n, cudaStream_t s) {
  if (n == 0 || src == dst) return cudaSuccess;
  long n4 = n / 4;
  long blocks = (n4 + 255) / 256;
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  ++g_launches;
  copy_f32_kernel<<<(int)blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst),
                                             n4);
  return cudaGetLastError();
}

__global__ void spin_kernel(long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(200);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((long long)(t - t0) < ns);
}

cudaError_t launch_spin(long long ns, cudaStream_t s) {
  if (ns <= 0) return cudaSuccess;
  ++g_launches;
  spin_kernel<<<1, 1, 0, s>>>(ns);
  return cudaGetLastError();
}

// Debug finiteness check (FSC_ERR_NONFINITE, fsc_set_debug_checks): count the
// non-finite fp32 values of x [n] into *bad.
__global__ void __launch_bounds__(256) nonfinite_kernel(const float4* __restrict__ x, long n4, int* bad) {
  int c = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    c += !isfinite(v.x) + !isfinite(v.y) + !isfinite(v.z) + !isfinite(v.w);
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(bad, c);
}

cudaError_t launch_count_nonfinite(const float* x, long n, int* bad, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  long blocks = (n / 4 + 255) / 256;
  if (blocks > kNumSMs * 4) blocks = kNumSMs * 4;
  if (blocks < 1) blocks = 1;
  ++g_launches;
  nonfinite_kernel<<<(int)blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(x), n / 4, bad);
  return cudaGetLastError();
}

}  // namespace fsc
