// K4-backward: persistent tcgen05 weight-gradient GEMM for the
// routed experts, the contraction over each expert's (ragged) token rows:
//
//   out_g[i, j] = sum_{m in group g} A[m, a_col0 + i] * B[m, b_col0 + j]     (i < N1, j < N2)
//
// i.e. dW3_e = dY_e^T (g h)_e, dW1_e = dU_e^T X_e, dW2_e = dV_e^T X_e (backward of
// PAPER.md:73-76 per expert, the oracle's swiglu_backward). Both operands are read
// MN-major straight from their row-major token layouts (no transposes): a stage holds
// 64 token rows of 128 (A) and BN (B) columns as TMA boxes {64 columns x 64 rows}.
// The last, partial k-block of a group is loaded by TMA like the others, but its A tile
// lands on a side barrier: the producer warp zeroes A's rows past the group end (the next
// group's rows) before it releases the stage to the MMA, so they never enter the sum.
// fp32 accumulation in TMEM, fp32 output.
//
// Roles (320 threads): warp 0 = producer (TMA; all lanes zero partial blocks), warp 1 =
// TMEM allocator + MMA issuer, warps 2..9 = epilogue (TMEM lane quarter = warp % 4,
// column half = (warp - 2) / 4), as in the forward grouped GEMM (gemm.cu).
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace fsc {

namespace {
constexpr int WBM = 128;             // output rows (i) per tile = TMEM lanes
constexpr int WBK = 64;              // token rows per stage
constexpr int kWMaxGroups = 256;
constexpr int kWEpiWarps = 8;
constexpr int kWThreads = 64 + 32 * kWEpiWarps;

template <int BN>
struct WCfg {
  static constexpr int A_BYTES = WBM * WBK * 2;               // 2 boxes of {64 cols, 64 rows}
  static constexpr int B_BYTES = BN * WBK * 2;                // BN / 64 boxes
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SCRATCH = kWEpiWarps * 32 * 36 * 4;    // fp32 32 x 32 transposes
  static constexpr int STAGES_RAW = (227 * 1024 - 4096 - SCRATCH) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256 + 2 * (kWMaxGroups + 1) * 4 + 16 + SCRATCH;
  static_assert((2 * 6 + 5) * 8 + 8 <= 256, "barriers + tmem slot fit the 256-byte control block");
};

FSC_DEVINL void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
FSC_DEVINL void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
}  // namespace

template <int BN>
__global__ void __launch_bounds__(kWThreads, 1)
    wgrad_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      WgradParams p) {
  using C = WCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* pbar = tempty + 2;                // partial k-block: A landed, rows past the group end to zero
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(pbar + 1);
  int* s_row_off = reinterpret_cast<int*>(smem + C::STAGES * C::STAGE_BYTES + 256);
  int* s_cnt = s_row_off + (kWMaxGroups + 1);
  float* s_scr = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(s_cnt + (kWMaxGroups + 1)) + 15) &
                                          ~uintptr_t(15));
  const int warp = warp_id();
  const int lane = lane_id();
  const int G = p.G;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], kWEpiWarps);
      }
      mbar_init(pbar, 1);
      fence_barrier_init();
    }
  } else if (warp == 1) {
    tmem_alloc<C::TMEM_COLS>(s_tmem);
  } else if (warp == 2) {
    int run = 0;
    if (lane == 0) s_row_off[0] = 0;
    for (int base = 0; base < G; base += 32) {
      const int g = base + lane;
      const int m = g < G ? (p.counts ? p.counts[g] : p.m_total) : 0;
      int im = m;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, im, o);
        if (lane >= o) im += a;
      }
      if (g < G) {
        s_row_off[g + 1] = run + im;
        s_cnt[g] = m;
      }
      run += __shfl_sync(0xffffffffu, im, 31);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const uint32_t tmem_base = *s_tmem;
  const int rbase = p.row_base ? __ldg(p.row_base) : 0;
  const int n_mb = (p.N1 + WBM - 1) / WBM, n_nb = p.N2 / BN;
  const int tpg = n_mb * n_nb;
  const int total = G * tpg;

  if (warp == 0) {
    // ------------------------------------------------ producer (whole warp)
    int stage = 0;
    uint32_t phase = 0, pphase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const int g = t / tpg, r = t - g * tpg, mb = r / n_nb, nb = r - mb * n_nb;
      const int M = s_cnt[g];
      const int row0 = rbase + s_row_off[g];
      const int acol = p.a_col0 + mb * WBM, bcol = p.b_col0 + nb * BN;
      for (int kb = 0; kb * WBK < M; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* a = sA + stage * C::A_BYTES;
        uint8_t* b = sB + stage * C::B_BYTES;
        const int m0 = row0 + kb * WBK;
        const int valid = min(WBK, M - kb * WBK);
        if (valid == WBK) {
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
            tma_load_2d(a, &tmA, &full[stage], acol, m0, kEvictNormal);
            tma_load_2d(a + 64 * WBK * 2, &tmA, &full[stage], acol + 64, m0, kEvictNormal);
#pragma unroll
            for (int i = 0; i < BN / 64; ++i) tma_load_2d(b + i * 64 * WBK * 2, &tmB, &full[stage], bcol + 64 * i, m0, kEvictNormal);
          }
        } else {
          // partial block: B by TMA onto full[stage] (its extra rows meet zero A rows); A by
          // TMA onto pbar, then the warp zeroes A's rows past the group end (whole 128-byte
          // k-rows: the swizzle only permutes 16-byte chunks inside a row) and arrives
          if (lane == 0) {
            mbar_expect_tx(&full[stage], C::B_BYTES);
#pragma unroll
            for (int i = 0; i < BN / 64; ++i) tma_load_2d(b + i * 64 * WBK * 2, &tmB, &full[stage], bcol + 64 * i, m0, kEvictNormal);
            mbar_arrive_expect_tx(pbar, C::A_BYTES);
            tma_load_2d(a, &tmA, pbar, acol, m0, kEvictNormal);
            tma_load_2d(a + 64 * WBK * 2, &tmA, pbar, acol + 64, m0, kEvictNormal);
          }
          mbar_wait(pbar, pphase);
          pphase ^= 1;
          for (int idx = valid * 8 + lane; idx < 64 * 8; idx += 32) {
            const int rr = idx >> 3, j = idx & 7;
#pragma unroll
            for (int box = 0; box < 2; ++box)
              *reinterpret_cast<uint4*>(a + box * 64 * WBK * 2 + rr * 128 + j * 16) = make_uint4(0u, 0u, 0u, 0u);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[stage]);
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16_f32(WBM, BN) | kIdescAMN | kIdescBMN;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        const int g = t / tpg;
        const int M = s_cnt[g];
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb * WBK < M; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < WBK / 16; ++k)
            umma_bf16_ss(d_tmem, umma_desc_sw128_mn(a_addr + k * 2048, 64 * WBK * 2),
                         umma_desc_sw128_mn(b_addr + k * 2048, 64 * WBK * 2), idesc, (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);   // (no MMA for an empty group: arrives at once)
      }
    }
  } else {
    // ------------------------------------------------ epilogue warps 2..9
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    float* scr = s_scr + (warp - 2) * 32 * 36;
    const int sub = lane >> 3, c4 = (lane & 7) * 4;
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
      const int g = t / tpg, r = t - g * tpg, mb = r / n_nb, nb = r - mb * n_nb;
      const bool empty_group = s_cnt[g] == 0;
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      float* out = p.out + (long)g * p.N1 * p.N2;
      const int i0 = mb * WBM + q * 32;                   // first output row of this warp
#pragma unroll 1
      for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
        uint32_t v[32];
        if (!empty_group) {
          tmem_ld32(tb + c, v);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0u;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4*>(scr + lane * 36 + 4 * i) =
              make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]), __uint_as_float(v[4 * i + 2]),
                          __uint_as_float(v[4 * i + 3]));
        __syncwarp();
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) {
          const int rr = k8 * 4 + sub;
          if (i0 + rr < p.N1) {
            float4 d4 = *reinterpret_cast<const float4*>(scr + rr * 36 + c4);
            float4* o = reinterpret_cast<float4*>(out + (long)(i0 + rr) * p.N2 + nb * BN + c + c4);
            if (p.accumulate) {
              const float4 a4 = *o;
              d4.x += a4.x;
              d4.y += a4.y;
              d4.z += a4.z;
              d4.w += a4.w;
            }
            *o = d4;
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_relaxed(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------------- host

static bool wmap(CUtensorMap* m, const void* base, long rows, long cols) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
static cudaError_t wlaunch(const WgradParams& p, long a_rows, long b_rows, int ctas, cudaStream_t s) {
  using C = WCfg<BN>;
  CUtensorMap ma, mb;
  if (!wmap(&ma, p.A, a_rows, p.lda) || !wmap(&mb, p.B, b_rows, p.ldb)) return cudaErrorInvalidValue;
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = ensure_smem_attr(wgrad_gemm_kernel<BN>, C::SMEM, attr)) return e;
  ++g_launches;
  wgrad_gemm_kernel<BN><<<ctas, kWThreads, C::SMEM, s>>>(ma, mb, p);
  return cudaGetLastError();
}

cudaError_t launch_wgrad_gemm(const WgradParams& p, long a_rows, long b_rows, int ctas, cudaStream_t s) {
  if (p.G < 1 || p.G > kWMaxGroups || p.N1 <= 0 || p.N2 % 64 || p.lda % 8 || p.ldb % 8 || p.a_col0 % 64 ||
      p.b_col0 % 64 || p.a_col0 + p.N1 > p.lda || p.b_col0 + p.N2 > p.ldb)
    return cudaErrorInvalidValue;
  if (ctas < 1 || ctas > kNumSMs) ctas = kNumSMs;
  a_rows = a_rows > 0 ? a_rows : 1;
  b_rows = b_rows > 0 ? b_rows : 1;
  if (p.N2 % 256 == 0) return wlaunch<256>(p, a_rows, b_rows, ctas, s);
  if (p.N2 % 128 == 0) return wlaunch<128>(p, a_rows, b_rows, ctas, s);
  return wlaunch<64>(p, a_rows, b_rows, ctas, s);
}

}  // namespace fsc
