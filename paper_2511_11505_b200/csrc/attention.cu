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
#include <float.h>

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

cudaError_t launch_flash_attn(const uint16_t* qkv, uint16_t* out, int T, int Hq, int Hkv, int hd, int seq_len,
                              cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  if (Hkv < 1 || Hq % Hkv) return cudaErrorInvalidValue;
  switch (hd) {
    case 16: return launch_fa_t<16>(qkv, out, T, Hq, Hkv, seq_len, s);
    case 32: return launch_fa_t<32>(qkv, out, T, Hq, Hkv, seq_len, s);
    case 64: return launch_fa_t<64>(qkv, out, T, Hq, Hkv, seq_len, s);
    case 128: return launch_fa_t<128>(qkv, out, T, Hq, Hkv, seq_len, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fsc
