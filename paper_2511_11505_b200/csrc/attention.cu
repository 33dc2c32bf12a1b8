// Attention sub-block used as the overlap filler of the layer stack (
// PAPER.md:198 splits it into (a) q,k,v preparation and (b) core attention +
// output projection). MLA is out of scope; this is causal grouped-query
// attention with rotary embedding over packed sequences (C-amb-18):
//   (a) hn = RMSNorm(attn_in) -> bf16; qkv = hn W_qkv^T (grouped_gemm, 1 group);
//       RoPE on q and k in place (rotate-half pairs (i, i + hd/2), pos = t mod seq_len)
//   (b) o = softmax(q k^T / sqrt(hd), causal within the sequence) v  (this file)
//       out = resid + o W_o^T  (grouped_gemm, fp32 residual epilogue)
// The core kernel is a FlashAttention-2 style forward with mma.sync bf16 tiles
// (64 queries x 64 keys per step, online softmax in fp32). It is the filler, not
// the hot path, and is not roofline-graded.
#include <cudaTypedefs.h>
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace fsc {

// ---------------------------------------------------------------------------- RMSNorm -> bf16
__global__ void __launch_bounds__(256) rmsnorm_bf16_kernel(const float* __restrict__ x, const float* __restrict__ gamma,
                                                           uint16_t* __restrict__ y, int T, int d, float eps) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= T) return;
  const float4* xr = reinterpret_cast<const float4*>(x + (long)warp * d);
  const int dv = d / 4;
  double ss = 0.0;
  for (int c = lane; c < dv; c += 32) {
    const float4 v = xr[c];
    ss += ((double)v.x * v.x + (double)v.y * v.y) + ((double)v.z * v.z + (double)v.w * v.w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
  const float r = (float)(1.0 / sqrt(ss / (double)d + (double)eps));
  for (int c = lane; c < dv; c += 32) {
    const float4 v = xr[c];
    const float4 g = reinterpret_cast<const float4*>(gamma)[c];
    uint2 o = make_uint2(pack_bf16x2(v.x * g.x * r, v.y * g.y * r), pack_bf16x2(v.z * g.z * r, v.w * g.w * r));
    *reinterpret_cast<uint2*>(y + (long)warp * d + c * 4) = o;
  }
}

cudaError_t launch_rmsnorm_bf16(const float* x, const float* gamma, uint16_t* y, int T, int d, float eps,
                                cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  ++g_launches;
  rmsnorm_bf16_kernel<<<(T + 7) / 8, 256, 0, s>>>(x, gamma, y, T, d, eps);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- RoPE (in place)
// qkv row t: [q heads | k heads | v heads], each head hd wide. Rotates the q and k heads.
__global__ void rope_kernel(uint16_t* __restrict__ qkv, int T, int n_rot_heads, int ld, int hd, int seq_len,
                            float theta) {
  const int half = hd / 2;
  const long total = (long)T * n_rot_heads * half;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i % half);
    const long th = i / half;
    const int h = (int)(th % n_rot_heads);
    const long t = th / n_rot_heads;
    const float pos = (float)(t % seq_len);
    const float inv = powf(theta, -2.0f * (float)c / (float)hd);
    float sn, cs;
    sincosf(pos * inv, &sn, &cs);
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(qkv) + t * ld + (long)h * hd;
    const float x1 = __bfloat162float(p[c]), x2 = __bfloat162float(p[c + half]);
    p[c] = __float2bfloat16_rn(x1 * cs - x2 * sn);
    p[c + half] = __float2bfloat16_rn(x2 * cs + x1 * sn);
  }
}

cudaError_t launch_rope(uint16_t* qkv, int T, int n_heads, int n_kv_heads, int hd, int seq_len, float theta,
                        cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int ld = (n_heads + 2 * n_kv_heads) * hd;
  const long total = (long)T * (n_heads + n_kv_heads) * (hd / 2);
  long blocks = (total + 255) / 256;
  if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
  ++g_launches;
  rope_kernel<<<(int)blocks, 256, 0, s>>>(qkv, T, n_heads + n_kv_heads, ld, hd, seq_len, theta);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------- flash attention fwd
namespace {
constexpr int FA_BM = 64;  // queries per CTA (4 warps x 16 rows)
constexpr int FA_BN = 64;  // keys per step

FSC_DEVINL void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
FSC_DEVINL void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
FSC_DEVINL void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
FSC_DEVINL void cp16(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
}  // namespace

template <int HD>
__global__ void __launch_bounds__(128) flash_attn_fwd_kernel(const uint16_t* __restrict__ qkv, uint16_t* __restrict__ out,
                                                             int T, int Hq, int Hkv, int seq_len, float scale_log2) {
  constexpr int LD = HD + 8;                  // padded smem row (bf16) -> conflict-free ldmatrix
  constexpr int NK = HD / 16;                 // k-steps over the head dim
  constexpr int ND = HD / 8;                  // n-tiles of the output
  extern __shared__ __align__(16) uint16_t fsm[];
  uint16_t* sQ = fsm;                         // [BM][LD]
  uint16_t* sK = sQ + FA_BM * LD;             // [2][BN][LD]
  uint16_t* sV = sK + 2 * FA_BN * LD;         // [2][BN][LD]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.y, kvh = h / (Hq / Hkv);
  const int ld = (Hq + 2 * Hkv) * HD;
  const long q0 = (long)blockIdx.x * FA_BM;
  const long seq0 = (q0 / seq_len) * seq_len;            // first key any query of this block may see
  const long q_last = min((long)T, q0 + FA_BM) - 1;
  const long kb_begin = (seq0 / FA_BN) * FA_BN;

  auto load_tile = [&](uint16_t* dst, long row0, int col) {
    for (int i = tid; i < FA_BN * (HD / 8); i += 128) {
      const int r = i / (HD / 8), c = (i % (HD / 8)) * 8;
      const long t = row0 + r;
      cp16(dst + r * LD + c, qkv + (t < T ? t : 0) * ld + col + c, t < T);
    }
  };
  load_tile(sQ, q0, h * HD);
  load_tile(sK, kb_begin, (Hq + kvh) * HD);
  load_tile(sV, kb_begin, (Hq + Hkv + kvh) * HD);
  asm volatile("cp.async.commit_group;" ::: "memory");

  const int g = lane >> 2, t4 = lane & 3;
  const long qa = q0 + warp * 16 + g, qb = qa + 8;       // the two query rows of this thread
  const long sa = (qa / seq_len) * seq_len, sb = (qb / seq_len) * seq_len;
  float o[ND][4];
#pragma unroll
  for (int n = 0; n < ND; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_a = -FLT_MAX, m_b = -FLT_MAX, l_a = 0.f, l_b = 0.f;
  uint32_t qf[NK][4];

  int buf = 0;
  for (long kb = kb_begin; kb <= q_last; kb += FA_BN, buf ^= 1) {
    if (kb + FA_BN <= q_last) {   // prefetch the next key block
      load_tile(sK + (buf ^ 1) * FA_BN * LD, kb + FA_BN, (Hq + kvh) * HD);
      load_tile(sV + (buf ^ 1) * FA_BN * LD, kb + FA_BN, (Hq + Hkv + kvh) * HD);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (kb == kb_begin) {
#pragma unroll
      for (int kk = 0; kk < NK; ++kk) {
        const int row = warp * 16 + (lane & 15), col = kk * 16 + (lane >> 4) * 8;
        ldsm_x4(smem_u32(sQ + row * LD + col), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const uint16_t* K = sK + buf * FA_BN * LD;
    const uint16_t* V = sV + buf * FA_BN * LD;
    // S = Q K^T (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
#pragma unroll
      for (int n = 0; n < 8; n += 2) {
        // two key n-tiles x (k 0-7, k 8-15): matrices (n,k0) (n,k8) (n+1,k0) (n+1,k8)
        const int krow = n * 8 + (lane & 7) + ((lane >> 4) << 3), kcol = kk * 16 + ((lane >> 3) & 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(smem_u32(K + krow * LD + kcol), b0, b1, b2, b3);
        mma_bf16_16816(s[n], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
        mma_bf16_16816(s[n + 1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
      }
    }
    // causal + same-sequence mask, online softmax (base 2)
    float mx_a = -FLT_MAX, mx_b = -FLT_MAX;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const long key = kb + n * 8 + 2 * t4 + e;
        const bool oka = key <= qa && key >= sa && key < T;
        const bool okb = key <= qb && key >= sb && key < T;
        s[n][e] = oka ? s[n][e] * scale_log2 : -FLT_MAX;
        s[n][2 + e] = okb ? s[n][2 + e] * scale_log2 : -FLT_MAX;
        mx_a = fmaxf(mx_a, s[n][e]);
        mx_b = fmaxf(mx_b, s[n][2 + e]);
      }
    }
#pragma unroll
    for (int o2 = 1; o2 <= 2; o2 <<= 1) {
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffff, mx_a, o2));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffff, mx_b, o2));
    }
    const float nm_a = fmaxf(m_a, mx_a), nm_b = fmaxf(m_b, mx_b);
    const float ca = (m_a == -FLT_MAX) ? 0.f : exp2f(m_a - nm_a);
    const float cb = (m_b == -FLT_MAX) ? 0.f : exp2f(m_b - nm_b);
    m_a = nm_a;
    m_b = nm_b;
    float ps_a = 0.f, ps_b = 0.f;
    uint32_t pf[8][2];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const float p0 = s[n][0] == -FLT_MAX ? 0.f : exp2f(s[n][0] - m_a);
      const float p1 = s[n][1] == -FLT_MAX ? 0.f : exp2f(s[n][1] - m_a);
      const float p2 = s[n][2] == -FLT_MAX ? 0.f : exp2f(s[n][2] - m_b);
      const float p3 = s[n][3] == -FLT_MAX ? 0.f : exp2f(s[n][3] - m_b);
      ps_a += p0 + p1;
      ps_b += p2 + p3;
      pf[n][0] = pack_bf16x2(p0, p1);
      pf[n][1] = pack_bf16x2(p2, p3);
    }
    l_a = l_a * ca + ps_a;
    l_b = l_b * cb + ps_b;
#pragma unroll
    for (int n = 0; n < ND; ++n) {
      o[n][0] *= ca;
      o[n][1] *= ca;
      o[n][2] *= cb;
      o[n][3] *= cb;
    }
    // O += P V : P (16 x 64) as A fragments (two S n-tiles per k16 step), V^T via ldmatrix.trans
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t a0 = pf[2 * kk][0], a1 = pf[2 * kk][1], a2 = pf[2 * kk + 1][0], a3 = pf[2 * kk + 1][1];
#pragma unroll
      for (int n = 0; n < ND; n += 2) {
        // matrices (keys k0-7, dims n), (keys k8-15, dims n), (k0-7, n+1), (k8-15, n+1)
        const int vrow = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, vcol = n * 8 + (lane >> 4) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(smem_u32(V + vrow * LD + vcol), b0, b1, b2, b3);
        mma_bf16_16816(o[n], a0, a1, a2, a3, b0, b1);
        mma_bf16_16816(o[n + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();
  }
  // normalise and store (row sums reduced over the quad)
#pragma unroll
  for (int o2 = 1; o2 <= 2; o2 <<= 1) {
    l_a += __shfl_xor_sync(0xffffffff, l_a, o2);
    l_b += __shfl_xor_sync(0xffffffff, l_b, o2);
  }
  const float ia = l_a > 0.f ? 1.f / l_a : 0.f, ib = l_b > 0.f ? 1.f / l_b : 0.f;
  const int ldo = Hq * HD;
#pragma unroll
  for (int n = 0; n < ND; ++n) {
    const int col = h * HD + n * 8 + 2 * t4;
    if (qa < T) *reinterpret_cast<uint32_t*>(out + qa * ldo + col) = pack_bf16x2(o[n][0] * ia, o[n][1] * ia);
    if (qb < T) *reinterpret_cast<uint32_t*>(out + qb * ldo + col) = pack_bf16x2(o[n][2] * ib, o[n][3] * ib);
  }
}

template <int HD>
static cudaError_t launch_fa_t(const uint16_t* qkv, uint16_t* out, int T, int Hq, int Hkv, int seq_len,
                               cudaStream_t s) {
  constexpr int LD = HD + 8;
  const size_t smem = (size_t)(FA_BM + 4 * FA_BN) * LD * 2;
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = ensure_smem_attr(flash_attn_fwd_kernel<HD>, (int)smem, attr)) return e;
  dim3 grid((T + FA_BM - 1) / FA_BM, Hq);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  ++g_launches;
  flash_attn_fwd_kernel<HD><<<grid, 128, smem, s>>>(qkv, out, T, Hq, Hkv, seq_len, scale_log2);
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------- tcgen05 flash attention fwd
// Causal attention of one head over a 128-query tile on the 5th-generation tensor cores
// (HD = 128, seq_len % 128 == 0): S = Q K^T and O += P V are tcgen05 MMAs (M = 128,
// N = 128, accumulators in TMEM: S double-buffered, O resident); Q, K and V arrive by TMA
// (K-major Q / K boxes, V as MN-major B boxes), P goes through shared memory in the
// 128B-swizzled K-major layout. Warp 0: TMA; warp 1: MMA issue (S_{j+1} is issued before
// PV_j, so the next scores overlap this block's softmax); warps 2-5: one query row per
// thread (the TMEM lane): mask, online softmax in base 2 with a lazy rescale (the running
// max is only raised when a block's max exceeds it by 2^8, FA4-style: p <= 2^8 stays exact
// enough in fp32 / bf16 and O is rescaled in TMEM only then), then O / l -> bf16.
namespace {
constexpr int TA_BM = 128, TA_BN = 128, TA_HD = 128;
constexpr int TA_THREADS = 320;            // warp 0 TMA, warp 1 MMA, warps 2-9 softmax (2 per lane quarter)
constexpr int TA_TILE = TA_BM * TA_HD * 2;     // 32 KB: Q / K / V / P tiles
constexpr int TA_SMEM = 1024 + 6 * TA_TILE + 256;
constexpr float kLazy = 8.f;                   // log2 units: rescale O when the max grows by more

FSC_DEVINL void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
FSC_DEVINL void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
FSC_DEVINL void fence_proxy_async_smem_ta() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
}  // namespace

__global__ void __launch_bounds__(TA_THREADS, 1)
    flash_attn_tc_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmV, uint16_t* out,
                         int T, int Hq, int Hkv, int seq_len, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                   // [2 atoms][128 rows][128 B]
  uint8_t* sK = smem + TA_TILE;                         // [2 stages] x 32 KB
  uint8_t* sV = smem + 3 * TA_TILE;                     // [2 stages] x [2 key halves][2 dim blocks][64 keys][128 B]
  uint8_t* sP = smem + 5 * TA_TILE;                     // [2 atoms][128 rows][128 B]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 6 * TA_TILE);
  uint64_t* q_full = bar;
  uint64_t* k_full = bar + 1;                           // [2]
  uint64_t* k_empty = bar + 3;                          // [2]
  uint64_t* v_full = bar + 5;                           // [2]
  uint64_t* v_empty = bar + 7;                          // [2]
  uint64_t* s_full = bar + 9;                           // [2]
  uint64_t* s_empty = bar + 11;                         // [2]
  uint64_t* p_full = bar + 13;
  uint64_t* pv_done = bar + 14;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bar + 15);
  __shared__ float s_red[2][TA_BM];                    // the two column halves' row maxima / sums

  const int warp = warp_id(), lane = lane_id();
  const int h = blockIdx.y, kvh = h / (Hq / Hkv);
  // query tiles in decreasing order of their key-block count (heavy tiles first)
  const int tps = seq_len / TA_BM, nseq = (T + seq_len - 1) / seq_len;
  const int i = blockIdx.x, pos = tps - 1 - i / nseq, sq = i % nseq;
  const long q0 = (long)sq * seq_len + (long)pos * TA_BM;
  if (q0 >= T) return;
  const long seq0 = (long)sq * seq_len;
  const int nb = pos + 1;                               // key blocks seq0 .. q0 (the diagonal one last)
  const int qcol = h * TA_HD, kcol = (Hq + kvh) * TA_HD, vcol = (Hq + Hkv + kvh) * TA_HD;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 8);
    }
    mbar_init(p_full, 8);
    mbar_init(pv_done, 1);
    fence_barrier_init();
  } else if (warp == 1) {
    tmem_alloc<512>(s_tmem);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;                        // S0 [0,128), S1 [128,256), O [256,384)

  if (warp == 0) {
    if (elect_one()) {                                   // TMA producer
      mbar_arrive_expect_tx(q_full, TA_TILE);
      tma_load_2d(sQ, &tmQK, q_full, qcol, (int)q0, kEvictFirst);
      tma_load_2d(sQ + TA_TILE / 2, &tmQK, q_full, qcol + 64, (int)q0, kEvictFirst);
      for (int j = 0; j < nb; ++j) {
        const int st = j & 1;
        const int k0 = (int)(seq0 + (long)j * TA_BN);
        if (j >= 2) mbar_wait(&k_empty[st], ((j >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&k_full[st], TA_TILE);
        tma_load_2d(sK + st * TA_TILE, &tmQK, &k_full[st], kcol, k0, kEvictLast);
        tma_load_2d(sK + st * TA_TILE + TA_TILE / 2, &tmQK, &k_full[st], kcol + 64, k0, kEvictLast);
        if (j >= 2) mbar_wait(&v_empty[st], ((j >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&v_full[st], TA_TILE);
#pragma unroll
        for (int kh = 0; kh < 2; ++kh)
#pragma unroll
          for (int db = 0; db < 2; ++db)
            tma_load_2d(sV + st * TA_TILE + kh * (TA_TILE / 2) + db * (TA_TILE / 4), &tmV, &v_full[st],
                        vcol + db * 64, k0 + kh * 64, kEvictLast);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {                                   // MMA issuer
      const uint32_t idesc_s = idesc_bf16_f32(TA_BM, TA_BN);
      const uint32_t idesc_o = idesc_bf16_f32(TA_BM, TA_HD) | kIdescBMN;
      const uint32_t aq = smem_u32(sQ), ap = smem_u32(sP);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        if (j >= 2) mbar_wait(&s_empty[st], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t bk = smem_u32(sK + st * TA_TILE);
#pragma unroll
        for (int kk = 0; kk < TA_HD / 16; ++kk) {      // over the head dim: 2 atoms of 64
          const uint32_t off = (kk >> 2) * (TA_TILE / 2) + (kk & 3) * 32;
          umma_bf16_ss(tmem + st * TA_BN, umma_desc_sw128(aq + off), umma_desc_sw128(bk + off), idesc_s, kk > 0);
        }
        umma_commit(&s_full[st]);
        umma_commit(&k_empty[st]);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < nb; ++j) {
        if (j + 1 < nb) issue_s(j + 1);
        const int st = j & 1;
        mbar_wait(p_full, j & 1);                        // P_j written (and O rescaled if needed)
        mbar_wait(&v_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t bv = smem_u32(sV + st * TA_TILE);
#pragma unroll
        for (int kk = 0; kk < TA_BN / 16; ++kk) {      // over the keys: P atoms of 64, V key halves of 64
          const uint32_t pa = ap + (kk >> 2) * (TA_TILE / 2) + (kk & 3) * 32;
          const uint32_t vb = bv + (kk >> 2) * (TA_TILE / 2) + (kk & 3) * 2048;
          umma_bf16_ss(tmem + 2 * TA_BN, umma_desc_sw128(pa), umma_desc_sw128_mn(vb, TA_TILE / 4), idesc_o,
                       (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(pv_done);
        umma_commit(&v_empty[st]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax / epilogue: thread = query row (its TMEM lane) x one half of the
    // 128 key columns (8 warps, two per lane quarter); the halves exchange their row maxima
    // through shared memory, keep separate partial row sums, and each writes its half of P
    // (one 64-key atom) and rescales / stores its half of O's 128 dims
    const int q = warp & 3, hh = (warp - 2) >> 2, r = q * 32 + lane;
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    const long qrow = q0 + r;
    constexpr int HC = TA_BN / 2;
    float m = -1e30f, l = 0.f;
    for (int j = 0; j < nb; ++j) {
      const int st = j & 1;
      const long k0 = seq0 + (long)j * TA_BN + hh * HC;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float sv[HC];
#pragma unroll
      for (int c = 0; c < HC; c += 32) {
        uint32_t u[32];
        tmem_ld32(tq + st * TA_BN + hh * HC + c, u);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) sv[c + e] = __uint_as_float(u[e]);   // raw scores (scale > 0 folded below)
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[st]);
      const bool diag = j == nb - 1, tail = k0 + HC > T;
      if (diag || tail) {
#pragma unroll
        for (int c = 0; c < HC; ++c) {
          const long key = k0 + c;
          if (key > qrow || key >= T) sv[c] = -INFINITY;
        }
      }
      float bm = -INFINITY;
#pragma unroll
      for (int c = 0; c < HC; ++c) bm = fmaxf(bm, sv[c]);
      bm *= scale_log2;                                  // max of the scaled scores
      s_red[hh][r] = bm;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      bm = fmaxf(bm, s_red[hh ^ 1][r]);
      asm volatile("bar.sync 1, 256;" ::: "memory");   // s_red is rewritten next block
      float alpha = 1.f;
      if (bm > m + kLazy) {                              // raise the reference max (rescale O and l)
        alpha = exp2f(m - bm);
        m = bm;
      }
      float ps = 0.f;
      uint32_t pk[HC / 2];
#pragma unroll
      for (int c = 0; c < HC; c += 2) {
        const float p0 = exp2f(fmaf(sv[c], scale_log2, -m)), p1 = exp2f(fmaf(sv[c + 1], scale_log2, -m));
        ps += p0 + p1;
        pk[c / 2] = pack_bf16x2(p0, p1);
      }
      l = l * alpha + ps;                                // this half's partial row sum
      if (j > 0) mbar_wait(pv_done, (j - 1) & 1);        // PV_{j-1} done: P buffer and O are free
      if (j > 0 && __any_sync(0xffffffff, alpha != 1.f)) {
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < TA_HD / 2; c += 32) {
          uint32_t u[32];
          tmem_ld32(tq + 2 * TA_BN + hh * (TA_HD / 2) + c, u);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) u[e] = __float_as_uint(__uint_as_float(u[e]) * alpha);
          tmem_st32(tq + 2 * TA_BN + hh * (TA_HD / 2) + c, u);
        }
        tmem_st_wait();
      }
      // this half of P row r: atom hh (keys hh*64 ..), 8 chunks of 8 bf16, 128B-swizzled
#pragma unroll
      for (int cc = 0; cc < 8; ++cc)
        *reinterpret_cast<uint4*>(sP + hh * (TA_TILE / 2) + r * 128 + ((cc ^ (r & 7)) << 4)) =
            make_uint4(pk[4 * cc], pk[4 * cc + 1], pk[4 * cc + 2], pk[4 * cc + 3]);
      fence_proxy_async_smem_ta();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    s_red[hh][r] = l;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const float lt = s_red[0][r] + s_red[1][r];
    mbar_wait(pv_done, (nb - 1) & 1);
    tc_fence_after();
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    uint16_t* orow = out + qrow * (long)(Hq * TA_HD) + h * TA_HD + hh * (TA_HD / 2);
#pragma unroll
    for (int c = 0; c < TA_HD / 2; c += 32) {
      uint32_t u[32];
      tmem_ld32(tq + 2 * TA_BN + hh * (TA_HD / 2) + c, u);
      tmem_ld_wait();
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) pk[e] = pack_bf16x2(__uint_as_float(u[2 * e]) * inv, __uint_as_float(u[2 * e + 1]) * inv);
      if (qrow < T)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          st_global_v4(orow + c + 8 * e, make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 ta_get_encode() {
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

static bool ta_make_map(CUtensorMap* m, const void* base, long rows, long cols, int box_rows) {
  auto enc = ta_get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static cudaError_t launch_fa_tc(const uint16_t* qkv, uint16_t* out, int T, int Hq, int Hkv, int seq_len,
                                cudaStream_t s) {
  const long ld = (long)(Hq + 2 * Hkv) * TA_HD;
  CUtensorMap mqk, mv;
  if (!ta_make_map(&mqk, qkv, T, ld, 128) || !ta_make_map(&mv, qkv, T, ld, 64)) return cudaErrorInvalidValue;
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = ensure_smem_attr(flash_attn_tc_kernel, TA_SMEM, attr)) return e;
  const int nseq = (T + seq_len - 1) / seq_len;
  dim3 grid(nseq * (seq_len / TA_BM), Hq);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)TA_HD);
  ++g_launches;
  flash_attn_tc_kernel<<<grid, TA_THREADS, TA_SMEM, s>>>(mqk, mv, out, T, Hq, Hkv, seq_len, scale_log2);
  return cudaGetLastError();
}

cudaError_t launch_flash_attn(const uint16_t* qkv, uint16_t* out, int T, int Hq, int Hkv, int hd, int seq_len,
                              cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  if (Hkv < 1 || Hq % Hkv) return cudaErrorInvalidValue;
  // tensor-core path (HD = 128, 128-aligned sequences); FSC_ATTN_MMA_SYNC=1 forces the mma.sync one (A/B)
  static const bool force_sync = getenv("FSC_ATTN_MMA_SYNC") && atoi(getenv("FSC_ATTN_MMA_SYNC"));
  if (hd == TA_HD && seq_len % TA_BM == 0 && !force_sync) return launch_fa_tc(qkv, out, T, Hq, Hkv, seq_len, s);
  switch (hd) {
    case 16: return launch_fa_t<16>(qkv, out, T, Hq, Hkv, seq_len, s);
    case 32: return launch_fa_t<32>(qkv, out, T, Hq, Hkv, seq_len, s);
    case 64: return launch_fa_t<64>(qkv, out, T, Hq, Hkv, seq_len, s);
    case 128: return launch_fa_t<128>(qkv, out, T, Hq, Hkv, seq_len, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fsc
