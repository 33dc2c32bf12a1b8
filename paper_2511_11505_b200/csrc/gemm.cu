// K4: persistent, warp-specialised tcgen05 grouped GEMM for sm_100a.
//
// Computes, for every group g (a local expert, "expert"),
//   D_g = A_g . B_g^T        A_g = rows [row_off[g], row_off[g]+M_g) of A (bf16, K-major)
//                            B_g = rows [g*N', (g+1)*N') of B       (bf16, K-major)
// with fp32 accumulation in TMEM and one of three fused epilogues:
//   EPI_SWIGLU   : h = U * SiLU(G), U from B0 = W1 (up), G from B1 = W2 (gate)
//                  (sigma = id, g = SiLU on the W2 branch) -> bf16
//   EPI_BF16     : plain bf16 store (expert down projection W3, the combine payload)
//   EPI_RESID_F32: out = resid + D in fp32 (shared-expert down projection / o-proj
//                  into the fp32 residual stream, PAPER.md:166-175 wiring)
// M_g comes from device-resident counts (no host sync): every CTA rebuilds the
// per-group row / tile prefix in shared memory and walks a static tile stride.
//
// Roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA
// issuer (one elected lane), warps 2..9 = epilogue (TMEM lane quarter = warp%4,
// column half = (warp-2)/4).
// Tiles: BM=128 rows x BN cols, BK=64 (one 128-byte swizzle atom of bf16).
#include <cudaTypedefs.h>
#include <limits.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace fsc {

namespace {
constexpr int BM = 128;              // rows per CTA (TMEM lanes)
constexpr int BK = 64;
constexpr int kMaxGroups = 256;
constexpr int kEpiWarps = 8;         // two warps per TMEM lane quarter, each half the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;

template <int BN, int CG, int EPI = 0>
struct Cfg {
  static constexpr int HALF = BN / 2;
  static constexpr int TILE_M = BM * CG;                       // rows per (pair) tile
  static constexpr int A_BYTES = BM * BK * 2;                  // per CTA
  static constexpr int B_ROWS = CG == 2 ? BN / 2 : BN;         // B rows held per CTA
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // fp32 epilogue: per-warp 32 x 32 transpose scratch (rows padded to 36 floats) so the
  // residual loads and output stores are row-contiguous 128-byte accesses
  // bf16 epilogues: per-warp 32 rows x 32 columns (64 B + 16 B pad per row) staging
  static constexpr int SCRATCH = EPI == EPI_RESID_F32 ? kEpiWarps * 32 * 36 * 4 : kEpiWarps * 32 * 80;
  static constexpr int STAGES_RAW = (227 * 1024 - 4096 - SCRATCH) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN;                     // double-buffered accumulator
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256 + 2 * (kMaxGroups + 1) * 4 + 16 + SCRATCH;
  // dynamic schedule: tile queue depth, as deep as the rest of the 256-byte barrier area allows
  static constexpr int TQ_RAW = (256 - (2 * STAGES + 4) * 8 - 8) / 20;   // (8-byte aligned barriers)
  static constexpr int TQ = TQ_RAW > 8 ? 8 : TQ_RAW;
  static_assert(TQ >= 4, "barriers + tile queue in the 256-byte area");
};

// SiLU with the fast divide (2 ulp; 0 for denominators beyond 2^126, where SiLU ~ 0)
FSC_DEVINL float silu_f(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

struct TileInfo {
  int g, mb, nb, row0, rows;
};

template <int TILE_M>
FSC_DEVINL TileInfo decode_tile(int t, int n_tiles, int G, const int* s_row_off, const int* s_tile_off) {
  TileInfo ti;
  int mt = t / n_tiles;
  ti.nb = t - mt * n_tiles;
  int lo = 0, hi = G;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (s_tile_off[mid] <= mt) lo = mid; else hi = mid;
  }
  ti.g = lo;
  ti.mb = mt - s_tile_off[lo];
  ti.row0 = s_row_off[lo] + ti.mb * TILE_M;
  int m = s_row_off[lo + 1] - s_row_off[lo];
  ti.rows = min(TILE_M, m - ti.mb * TILE_M);
  return ti;
}
// Store one 32-row x 32-column bf16 chunk of the warp's rows row-contiguously: lane i
// holds pk[] = 32 bf16 of its own row (row i of the warp), dst_i = that row's output
// address (nullptr: row not stored). Staged through the warp's shared scratch so that
// 4 lanes write one row's 64 bytes (8 rows per instruction) instead of 32 rows x 16 B.
FSC_DEVINL void store_rows_bf16(uint8_t* scr, const uint32_t (&pk)[16], __nv_bfloat16* dst, int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<uint4*>(scr + lane * 80 + 16 * i) = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2],
                                                                     pk[4 * i + 3]);
  __syncwarp();
  const uint64_t mine = reinterpret_cast<uint64_t>(dst);
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int r = it * 8 + (lane >> 2), seg = lane & 3;
    const uint64_t d = __shfl_sync(0xffffffffu, mine, r);
    if (d) {
      const uint4 v = *reinterpret_cast<const uint4*>(scr + r * 80 + seg * 16);
      st_global_v4(reinterpret_cast<__nv_bfloat16*>(d) + seg * 8, v);
    }
  }
  __syncwarp();
}

// Fused gate-weighted unpermute (see GemmParams::comb_out). Called by an epilogue
// warp after each lane stored the y columns [c0, c0 + BN/2) of its row (token
// `tok`, -1 = no row): each lane bumps its (token, column block) counter with a
// release RMW (orders its y stores); the lane that brings it to k acquires (the RMW
// chain makes every copy's stores visible) and __syncwarp passes that on to the
// warp, which then finishes those tokens cooperatively, up to 4 at a time with all
// their k row loads in flight (lane i owns columns c0 + CPL*i ...), in slot order
// exactly as unpermute_kernel: acc = 0; acc = fma(w_j, y_j, acc), j = 0..k-1;
// out = resid + acc. Requires k <= 8.
FSC_DEVINL int atom_add_release_gpu(int* p, int v) {
  int old;
  asm volatile("atom.release.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
FSC_DEVINL void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

template <int BN>
FSC_DEVINL void fused_unpermute(const GemmParams& p, long tok, int c0, int lane) {
  constexpr int CPL = BN / 2 / 32;      // columns per lane: 4 (BN 256), 2 (128), 1 (64)
  constexpr int TQ = 4;                 // tokens finished together
  const int k = p.top_k;
  __syncwarp();                          // the rows were stored by other lanes (store_rows_bf16)
  bool last = false;
  if (tok >= 0) {
    int* cp = p.comb_cnt + tok * p.n_cb + c0 / (BN / 2);
    last = atom_add_release_gpu(cp, 1) == k - 1;
    if (last) {
      fence_acquire_gpu();
      *cp = 0;                          // every copy arrived: reset for the next call
    }
  }
  uint32_t m = __ballot_sync(0xffffffffu, last);
  if (!m) return;
  __syncwarp();
  const int ld = p.n_cb * (BN / 2);     // = d
  const uint16_t* y = reinterpret_cast<const uint16_t*>(p.out);
  const int col = c0 + CPL * lane;
  while (m) {
    long tq[TQ];
    int nq = 0;
#pragma unroll
    for (int q = 0; q < TQ; ++q) {
      tq[q] = -1;
      if (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        tq[q] = __shfl_sync(0xffffffffu, tok, src);
        ++nq;
      }
    }
    // lane q*k + j holds pos / w of (token q, slot j)
    int pj = 0;
    float wj = 0.f;
    {
      const int q = lane / k, j = lane - (lane / k) * k;
      if (q < nq) {
        long tt = tq[0];
#pragma unroll
        for (int u = 1; u < TQ; ++u)
          if (q == u) tt = tq[u];
        pj = __ldcg(p.pos + tt * k + j);
        wj = __ldcg(p.topk_w + tt * k + j);
      }
    }
    uint32_t yv[TQ][8][(CPL + 1) / 2];
    float rv[TQ][CPL];
#pragma unroll
    for (int q = 0; q < TQ; ++q) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int pr = __shfl_sync(0xffffffffu, pj, (q * k + j) & 31);
        if (q < nq && j < k) {
          const uint16_t* yr = y + (long)pr * ld + col;
          if (CPL == 4) {
            const uint2 u = __ldcg(reinterpret_cast<const uint2*>(yr));
            yv[q][j][0] = u.x;
            yv[q][j][(CPL + 1) / 2 - 1] = u.y;
          } else if (CPL == 2) {
            yv[q][j][0] = __ldcg(reinterpret_cast<const unsigned int*>(yr));
          } else {
            yv[q][j][0] = (uint32_t)__ldcg(reinterpret_cast<const unsigned short*>(yr));
          }
        }
      }
#pragma unroll
      for (int i = 0; i < CPL; ++i)
        rv[q][i] = (q < nq && p.comb_resid) ? __ldcg(p.comb_resid + tq[q] * ld + col + i) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < TQ; ++q) {
      if (q >= nq) break;
      float acc[CPL];
#pragma unroll
      for (int i = 0; i < CPL; ++i) acc[i] = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float g = __shfl_sync(0xffffffffu, wj, (q * k + j) & 31);
        if (j < k) {
          if (CPL == 4) {
            acc[0] = fmaf(g, bf16lo(yv[q][j][0]), acc[0]);
            acc[1 % CPL] = fmaf(g, bf16hi(yv[q][j][0]), acc[1 % CPL]);
            acc[2 % CPL] = fmaf(g, bf16lo(yv[q][j][(CPL + 1) / 2 - 1]), acc[2 % CPL]);
            acc[3 % CPL] = fmaf(g, bf16hi(yv[q][j][(CPL + 1) / 2 - 1]), acc[3 % CPL]);
          } else if (CPL == 2) {
            acc[0] = fmaf(g, bf16lo(yv[q][j][0]), acc[0]);
            acc[1 % CPL] = fmaf(g, bf16hi(yv[q][j][0]), acc[1 % CPL]);
          } else {
            acc[0] = fmaf(g, bf16lo(yv[q][j][0]), acc[0]);
          }
        }
      }
      float* oo = p.comb_out + tq[q] * ld + col;
      if (CPL == 4) {
        *reinterpret_cast<float4*>(oo) =
            make_float4(rv[q][0] + acc[0], rv[q][1 % CPL] + acc[1 % CPL], rv[q][2 % CPL] + acc[2 % CPL],
                        rv[q][3 % CPL] + acc[3 % CPL]);
      } else {
#pragma unroll
        for (int i = 0; i < CPL; ++i) oo[i] = rv[q][i] + acc[i];
      }
    }
  }
}
}  // namespace

// CG = 1: one CTA per 128-row tile (tcgen05 cta_group::1).
// CG = 2: a CTA pair (cluster of 2) per 256-row tile: MMA M=256 issued by the
// leader (cta_group::2); each CTA stages its 128 rows of A and half of the B
// columns, so per-SM smem traffic per MAC drops by a third and the pipeline is
// 1.5x deeper at the same shared-memory footprint.
template <int BN, int EPI, int CG, bool BMN>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                        const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmA32,
                        const __grid_constant__ CUtensorMap tmA64, GemmParams p) {
  using C = Cfg<BN, CG, EPI>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + 2);
  // tile queue of the dynamic schedule: the last 80 bytes of the 256-byte barrier area
  constexpr int kTQ = C::TQ;
  uint64_t* tq_full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + ((256 - 20 * kTQ) & ~7));
  uint64_t* tq_empty = tq_full + kTQ;
  int* s_tq = reinterpret_cast<int*>(tq_empty + kTQ);
  int* s_row_off = reinterpret_cast<int*>(smem + C::STAGES * C::STAGE_BYTES + 256);
  int* s_tile_off = s_row_off + (kMaxGroups + 1);
  float* s_scr = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(s_tile_off + (kMaxGroups + 1)) + 15) &
                                          ~uintptr_t(15));   // epilogue transpose scratch (16-byte rows)

  const int warp = warp_id();
  const int lane = lane_id();
  const int G = p.G;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  const bool leader = rank == 0;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmA32);
      tma_prefetch_desc(&tmA64);
      tma_prefetch_desc(&tmB0);
      tma_prefetch_desc(&tmB1);
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], kEpiWarps * CG);
      }
      for (int i = 0; i < kTQ; ++i) {     // consumers of a queue entry: MMA + epilogue warps (+ the peer producer)
        mbar_init(&tq_full[i], 1);
        mbar_init(&tq_empty[i], 1 + kEpiWarps * CG + (CG == 2 ? 1 : 0));
      }
      fence_barrier_init();
    }
  } else if (warp == 1) {
    if (CG == 2) tmem_alloc_2sm<C::TMEM_COLS>(s_tmem);
    else tmem_alloc<C::TMEM_COLS>(s_tmem);
  } else if (warp == 2) {
    // per-group row and tile prefix sums from the device-resident counts
    int run_rows = 0, run_tiles = 0;
    if (lane == 0) { s_row_off[0] = 0; s_tile_off[0] = 0; }
    for (int base = 0; base < G; base += 32) {
      int g = base + lane;
      int m = 0;
      if (g < G) m = p.counts ? p.counts[g] : p.m_total;
      int tl = (m + C::TILE_M - 1) / C::TILE_M;
      int im = m, it = tl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int a = __shfl_up_sync(0xffffffff, im, o);
        int b = __shfl_up_sync(0xffffffff, it, o);
        if (lane >= o) { im += a; it += b; }
      }
      if (g < G) { s_row_off[g + 1] = run_rows + im; s_tile_off[g + 1] = run_tiles + it; }
      run_rows += __shfl_sync(0xffffffff, im, 31);
      run_tiles += __shfl_sync(0xffffffff, it, 31);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();   // peer barriers initialised before any remote arrive / 2-SM TMA
  tc_fence_after();

  const uint32_t tmem_base = *s_tmem;
  const int rbase = p.row_base ? __ldg(p.row_base) : 0;
  // bf16 epilogue store mode: staged through shared memory into row-contiguous 64-byte
  // segments (4 lanes per row) instead of 32 rows x 16 B per store instruction. A/B in
  // one run: down GEMM 200.7 -> 194.6 us (DS, K = 1408), 357 -> 307 us (Qwen3, K = 768)
  const bool stage_rows = p.stage_rows != 0;
  constexpr bool SWI = EPI == EPI_SWIGLU || EPI == EPI_SWIGLU_BWD;   // [U | G] accumulator halves
  const int n_tiles = SWI ? p.N / C::HALF : p.N / BN;
  const int total = s_tile_off[G] * n_tiles;
  const int kblocks = p.K / BK;
  const int t_first = blockIdx.x / CG, t_step = gridDim.x / CG;
  // Tile schedule. Static: the u-th tile of this CTA (pair) is t_first + u t_step. Dynamic
  // (p.sched): the first tile is static, later ones are claimed from an atomic counter by
  // the (leader's) producer and handed to every role through a kTQ-deep shared-memory queue
  // (the peer CTA's copy written over DSMEM): a CTA (pair) that gets its SMs late, beside
  // co-running kernels, takes fewer tiles instead of leaving a tail of pre-assigned ones.
  const bool dyn = p.sched != nullptr && !p.a_idx;
  const uint32_t tq_empty_leader = CG == 2 ? mapa_shared(smem_u32(tq_empty), 0) : smem_u32(tq_empty);
  // claimer (producer thread of the leader CTA): the u-th tile, published to the queue
  // The claimer publishes entry u + 1 when it starts tile u (so the peer CTA's producer
  // learns its next tile a tile ahead, as with the static stride), and the atomic behind
  // entry u + 2 is issued right after, so its round trip overlaps the tile's loads.
  int pend = 0, last = 0;
  auto publish = [&](int u, int t) {
    const int sl = u % kTQ;
    if (u >= kTQ) mbar_wait(&tq_empty[sl], ((u / kTQ) - 1) & 1);
    s_tq[sl] = t;
    if (CG == 2) {
      st_cluster_s32(mapa_shared(smem_u32(&s_tq[sl]), 1), t);
      mbar_arrive_cluster(mapa_shared(smem_u32(&tq_full[sl]), 1));   // release.cluster: after the store
    }
    mbar_arrive(&tq_full[sl]);
  };
  auto claim_tile = [&](int u) -> int {
    if (!dyn) return t_first + u * t_step < total ? t_first + u * t_step : -1;
    if (u == 0) {
      last = t_first < total ? t_first : -1;
      publish(0, last);
      if (last >= 0) pend = atomicAdd(p.sched, 1);
    }
    const int t = last;                                  // entry u (published one tile ago)
    if (t >= 0) {
      int nx = pend + t_step;
      if (nx >= total) nx = -1;
      publish(u + 1, nx);
      if (nx >= 0) pend = atomicAdd(p.sched, 1);
      last = nx;
    }
    return t;
  };
  // consumer: the u-th tile from the queue (arrive = this consumer is done reading the entry;
  // an epilogue warp passes arrive only on lane 0, after __syncwarp)
  auto next_tile = [&](int u, bool arrive) -> int {
    if (!dyn) return t_first + u * t_step < total ? t_first + u * t_step : -1;
    const int sl = u % kTQ;
    if (CG == 2 && !leader) mbar_wait_acq_cluster(&tq_full[sl], (u / kTQ) & 1);   // published over DSMEM
    else mbar_wait(&tq_full[sl], (u / kTQ) & 1);
    const int t = s_tq[sl];
    __syncwarp(__activemask());
    // relaxed arrive: a release here would make an epilogue warp wait for its global stores
    // to drain; the branch on the loaded value orders the shared-memory read before it
    if (arrive && t != INT_MIN) {
      if (CG == 2) mbar_arrive_cluster_relaxed(tq_empty_leader + sl * 8);
      else mbar_arrive_relaxed(&tq_empty[sl]);
    }
    return t;
  };

  if (warp == 0 && p.a_idx) {
    // ------------------------------------------------ TMA producer, gathered A (whole warp 0):
    // lane j gathers rows 4j..4j+3 of this CTA's 128-row slice (fused permute, EP = 1)
    int stage = 0;
    uint32_t phase = 0;
    for (int t = t_first; t < total; t += t_step) {
      TileInfo ti = decode_tile<C::TILE_M>(t, n_tiles, G, s_row_off, s_tile_off);
      ti.row0 += rbase;
      const int arow = ti.row0 + (int)rank * BM;
      const int rend = ti.row0 + ti.rows;
      // only the groups of 4 rows that hold valid rows are gathered (rows past the
      // group end are never stored, so stale shared memory there is harmless)
      const int v0 = min(BM, max(0, ti.rows)), v1 = min(BM, max(0, ti.rows - BM));
      const int my_valid = rank ? v1 : v0;
      const uint32_t a_bytes = (uint32_t)((v0 + 3) / 4 + (CG == 2 ? (v1 + 3) / 4 : 0)) * 4 * BK * 2;
      int ri[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = arow + 4 * lane + u;
        ri[u] = r < rend ? __ldg(p.a_idx + r) : 0;   // rows past the group: any valid row (not stored)
      }
      int brow0, brow1 = 0;
      const CUtensorMap* mb0 = &tmB0;
      const CUtensorMap* mb1 = &tmB0;
      if (CG == 2) {
        if (EPI == EPI_SWIGLU) {
          brow0 = ti.g * p.b_group_rows + ti.nb * C::HALF;
          mb0 = rank ? &tmB1 : &tmB0;
        } else {
          brow0 = ti.g * p.b_group_rows + ti.nb * BN + (int)rank * C::HALF;
        }
      } else {
        if (EPI == EPI_SWIGLU) {
          brow0 = ti.g * p.b_group_rows + ti.nb * C::HALF;
          brow1 = brow0;
          mb1 = &tmB1;
        } else {
          brow0 = ti.g * p.b_group_rows + ti.nb * BN;
          brow1 = brow0 + C::HALF;
        }
      }
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* b = sB + stage * C::B_BYTES;
        if (lane == 0) {
          if (CG == 2) {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::B_BYTES + a_bytes);
            tma_load_2d_2sm(b, mb0, &full[stage], kb * BK, brow0, kEvictLast);
          } else {
            mbar_arrive_expect_tx(&full[stage], C::B_BYTES + a_bytes);
            tma_load_2d(b, mb0, &full[stage], kb * BK, brow0, kEvictLast);
            tma_load_2d(b + C::HALF * BK * 2, mb1, &full[stage], kb * BK, brow1, kEvictLast);
          }
        }
        __syncwarp();
        if (4 * lane < my_valid)
          tma_gather4<CG>(sA + stage * C::A_BYTES + lane * 4 * BK * 2, &tmA, &full[stage], kb * BK, ri[0], ri[1],
                          ri[2], ri[3], kEvictNormal);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------ TMA producer (both CTAs of a pair)
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = 0;; ++u) {
        const int t = leader ? claim_tile(u) : next_tile(u, true);
        if (t < 0) break;
        TileInfo ti = decode_tile<C::TILE_M>(t, n_tiles, G, s_row_off, s_tile_off);
        ti.row0 += rbase;
        const int arow = ti.row0 + (int)rank * BM;
        int brow0, brow1 = 0;
        const CUtensorMap* mb0 = &tmB0;
        const CUtensorMap* mb1 = &tmB0;
        if (CG == 2) {
          if (SWI) {                         // CTA0: U columns from W1, CTA1: G columns from W2
            brow0 = ti.g * p.b_group_rows + ti.nb * C::HALF;
            mb0 = rank ? &tmB1 : &tmB0;
          } else {
            brow0 = ti.g * p.b_group_rows + ti.nb * BN + (int)rank * C::HALF;
          }
        } else {
          if (SWI) {
            brow0 = ti.g * p.b_group_rows + ti.nb * C::HALF;
            brow1 = brow0;
            mb1 = &tmB1;
          } else {
            brow0 = ti.g * p.b_group_rows + ti.nb * BN;
            brow1 = brow0 + C::HALF;
          }
        }
        // A rows actually needed by each CTA of the tile: a ragged group end (decode:
        // a few rows per expert) loads a 32 / 64-row box or nothing instead of 128 rows
        // (rows past the group end are never stored; stale shared memory is harmless)
        const int v0 = min(BM, ti.rows), v1 = min(BM, max(0, ti.rows - BM));
        auto box_rows = [](int v) { return v == 0 ? 0 : (v <= 32 ? 32 : (v <= 64 ? 64 : BM)); };
        const int mybox = box_rows(rank ? v1 : v0);
        const CUtensorMap* ma = mybox == 32 ? &tmA32 : (mybox == 64 ? &tmA64 : &tmA);
        const uint32_t a_bytes = (uint32_t)(box_rows(v0) + (CG == 2 ? box_rows(v1) : 0)) * BK * 2;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* b = sB + stage * C::B_BYTES;
          if (BMN) {
            // MN-major B: this CTA's B_ROWS output columns x BK k-rows as boxes of
            // {64 columns, 64 k-rows} (128-byte k-rows, 8 KB per box)
            const bool hi = p.kb_split > 0 && kb >= p.kb_split;
            const CUtensorMap* mk = hi ? &tmB1 : &tmB0;
            const int krow = ti.g * p.b_group_rows + (hi ? kb - p.kb_split : kb) * BK;
            const int ncol = ti.nb * BN + (CG == 2 ? (int)rank * C::HALF : 0);
            if (CG == 2) {
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::B_BYTES + a_bytes);
              if (mybox) tma_load_2d_2sm(sA + stage * C::A_BYTES, ma, &full[stage], kb * BK, arow, kEvictNormal);
#pragma unroll
              for (int i = 0; i < C::B_ROWS / 64; ++i)
                tma_load_2d_2sm(b + i * 64 * BK * 2, mk, &full[stage], ncol + 64 * i, krow, kEvictLast);
            } else {
              mbar_arrive_expect_tx(&full[stage], C::B_BYTES + a_bytes);
              if (mybox) tma_load_2d(sA + stage * C::A_BYTES, ma, &full[stage], kb * BK, arow, kEvictNormal);
#pragma unroll
              for (int i = 0; i < C::B_ROWS / 64; ++i)
                tma_load_2d(b + i * 64 * BK * 2, mk, &full[stage], ncol + 64 * i, krow, kEvictLast);
            }
          } else if (CG == 2) {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::B_BYTES + a_bytes);
            if (mybox) tma_load_2d_2sm(sA + stage * C::A_BYTES, ma, &full[stage], kb * BK, arow, kEvictNormal);
            tma_load_2d_2sm(b, mb0, &full[stage], kb * BK, brow0, kEvictLast);
          } else {
            mbar_arrive_expect_tx(&full[stage], C::B_BYTES + a_bytes);
            if (mybox) tma_load_2d(sA + stage * C::A_BYTES, ma, &full[stage], kb * BK, arow, kEvictNormal);
            tma_load_2d(b, mb0, &full[stage], kb * BK, brow0, kEvictLast);
            tma_load_2d(b + C::HALF * BK * 2, mb1, &full[stage], kb * BK, brow1, kEvictLast);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader CTA only)
    if (leader && elect_one()) {
      const uint32_t idesc = idesc_bf16_f32(C::TILE_M, BN) | (BMN ? kIdescBMN : 0u);
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        if (next_tile(it, true) < 0) break;
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t bdesc = BMN ? umma_desc_sw128_mn(b_addr + k * 2048, 64 * BK * 2)
                                       : umma_desc_sw128(b_addr + k * 32);
            if (CG == 2)
              umma_bf16_ss_2sm(d_tmem, umma_desc_sw128(a_addr + k * 32), bdesc, idesc, (kb | k) != 0);
            else
              umma_bf16_ss(d_tmem, umma_desc_sw128(a_addr + k * 32), bdesc, idesc, (kb | k) != 0);
          }
          if (CG == 2) umma_commit_2sm(&empty[stage]);
          else umma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (CG == 2) umma_commit_2sm(&tfull[acc]);
        else umma_commit(&tfull[acc]);
      }
    }
  } else {
    // ------------------------------------------------ epilogue warps 2..9 (own 128 rows)
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;   // column half handled by this warp
    const int r = q * 32 + lane;
    const uint32_t tempty_leader = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0;
    for (int it = 0;; ++it) {
      const int t = next_tile(it, lane == 0);
      if (t < 0) break;
      TileInfo ti = decode_tile<C::TILE_M>(t, n_tiles, G, s_row_off, s_tile_off);
      ti.row0 += rbase;
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const int rr = r + (int)rank * BM;          // row inside the pair tile
      const bool valid = rr < ti.rows;
      const long grow = (long)ti.row0 + rr;
      if (EPI != EPI_RESID_F32) {
        mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
      }
      const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (EPI == EPI_SWIGLU) {
        __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out) + grow * p.ldo + ti.nb * C::HALF;
#pragma unroll 1
        for (int c = half * (C::HALF / 2); c < (half + 1) * (C::HALF / 2); c += 32) {
          uint32_t u[32], gv[32];
          tmem_ld32(tb + c, u);
          tmem_ld32(tb + C::HALF + c, gv);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float h0 = __uint_as_float(u[2 * i]) * silu_f(__uint_as_float(gv[2 * i]));
            float h1 = __uint_as_float(u[2 * i + 1]) * silu_f(__uint_as_float(gv[2 * i + 1]));
            pk[i] = pack_bf16x2(h0, h1);
          }
          if (stage_rows) {
            store_rows_bf16(reinterpret_cast<uint8_t*>(s_scr) + (warp - 2) * 32 * 80, pk, valid ? out + c : nullptr,
                            lane);
          } else if (valid) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              st_global_v4(out + c + 8 * i, make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]));
          }
        }
      } else if (EPI == EPI_SWIGLU_BWD) {
        // backward of h = u SiLU(v) with the recomputed u, v (see GemmParams)
        const long col0 = (long)ti.nb * C::HALF;
        __nv_bfloat16* o_du = reinterpret_cast<__nv_bfloat16*>(p.out) + grow * p.ldo + col0;
        __nv_bfloat16* o_dv = o_du + p.N;
        __nv_bfloat16* o_h = reinterpret_cast<__nv_bfloat16*>(p.out2) + grow * (long)p.N + col0;
        const uint16_t* i_dh = p.dh + grow * (long)p.N + col0;
        const float gr = (valid && p.row_gate) ? __ldg(p.row_gate + grow) : 1.f;
        float dgp = 0.f;
#pragma unroll 1
        for (int c = half * (C::HALF / 2); c < (half + 1) * (C::HALF / 2); c += 32) {
          uint32_t u[32], gv[32];
          tmem_ld32(tb + c, u);
          tmem_ld32(tb + C::HALF + c, gv);
          uint4 dq[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dq[i] = valid ? __ldg(reinterpret_cast<const uint4*>(i_dh + c) + i) : make_uint4(0u, 0u, 0u, 0u);
          tmem_ld_wait();
          const uint32_t* dw = reinterpret_cast<const uint32_t*>(dq);
          uint32_t pu[16], pv[16], ph[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float hh[2], du[2], dv[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float uu = __uint_as_float(u[2 * i + e]), vv = __uint_as_float(gv[2 * i + e]);
              const float dhu = e ? bf16hi(dw[i]) : bf16lo(dw[i]);
              const float sg = __fdividef(1.0f, 1.0f + __expf(-vv));     // logistic(v)
              const float sv = vv * sg;                                   // SiLU(v)
              const float dsv = sg * (1.0f + vv * (1.0f - sg));           // SiLU'(v)
              hh[e] = uu * sv;
              const float dh = gr * dhu;
              du[e] = dh * sv;
              dv[e] = dh * uu * dsv;
              dgp = fmaf(hh[e], dhu, dgp);
            }
            pu[i] = pack_bf16x2(du[0], du[1]);
            pv[i] = pack_bf16x2(dv[0], dv[1]);
            ph[i] = pack_bf16x2(gr * hh[0], gr * hh[1]);
          }
          if (valid) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              st_global_v4(o_du + c + 8 * i, make_uint4(pu[4 * i], pu[4 * i + 1], pu[4 * i + 2], pu[4 * i + 3]));
              st_global_v4(o_dv + c + 8 * i, make_uint4(pv[4 * i], pv[4 * i + 1], pv[4 * i + 2], pv[4 * i + 3]));
              st_global_v4(o_h + c + 8 * i, make_uint4(ph[4 * i], ph[4 * i + 1], ph[4 * i + 2], ph[4 * i + 3]));
            }
          }
        }
        if (p.dg_part && valid) p.dg_part[grow * p.dg_ld + ti.nb * 2 + half] = dgp;
      } else if (EPI == EPI_BF16) {
        __nv_bfloat16* out;
        if (p.ret) {     // fused combine: write the row straight into its source rank's buffer
          const int v = valid ? p.ret[grow] : 0;
          out = reinterpret_cast<__nv_bfloat16*>(p.peer_out[(uint32_t)v >> 24]) + (long)(v & 0xFFFFFF) * p.ldo +
                ti.nb * BN;
        } else {
          out = reinterpret_cast<__nv_bfloat16*>(p.out) + grow * p.ldo + ti.nb * BN;
        }
        const long tok = (p.comb_out && valid) ? (long)__ldg(p.src_row + grow) : -1;
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
          uint32_t v[32];
          tmem_ld32(tb + c, v);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
          if (stage_rows) {   // short K: the epilogue is on the critical path, store rows contiguously
            store_rows_bf16(reinterpret_cast<uint8_t*>(s_scr) + (warp - 2) * 32 * 80, pk, valid ? out + c : nullptr,
                            lane);
          } else if (valid) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              st_global_v4(out + c + 8 * i, make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]));
          }
        }
        if (p.comb_out) fused_unpermute<BN>(p, tok, ti.nb * BN + half * (BN / 2), lane);
      } else {
        // thread = row after tcgen05.ld; transpose each 32 x 32 chunk through shared
        // memory so that 8 lanes cover one row's 32 floats (128-byte residual loads and
        // output stores, 4 rows per instruction)
        float* scr = s_scr + (warp - 2) * 32 * 36;
        const int rbase = (int)rank * BM + q * 32;              // first row of this warp inside the tile
        const int sub = lane >> 3, c4 = (lane & 7) * 4;
        const int c_beg = half * (BN / 2), c_end = (half + 1) * (BN / 2);
        mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
#pragma unroll 1
        for (int c = c_beg; c < c_end; c += 32) {
          uint32_t v[32];
          tmem_ld32(tb + c, v);
          float4 rv[8];
#pragma unroll
          for (int it = 0; it < 8; ++it) {                       // residual of rows it*4 + sub (in flight)
            const int rr2 = rbase + it * 4 + sub;
            rv[it] = (p.resid && rr2 < ti.rows)
                         ? *reinterpret_cast<const float4*>(p.resid + ((long)ti.row0 + rr2) * p.ldr + ti.nb * BN + c + c4)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 8; ++i)
            *reinterpret_cast<float4*>(scr + lane * 36 + 4 * i) =
                make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]), __uint_as_float(v[4 * i + 2]),
                            __uint_as_float(v[4 * i + 3]));
          __syncwarp();
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int r = it * 4 + sub;
            if (rbase + r < ti.rows) {
              const float4 d4 = *reinterpret_cast<const float4*>(scr + r * 36 + c4);
              float4 a = rv[it];
              a.x += d4.x;
              a.y += d4.y;
              a.z += d4.z;
              a.w += d4.w;
              *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + ((long)ti.row0 + rbase + r) * p.ldo +
                                         ti.nb * BN + c + c4) = a;
            }
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster_relaxed(tempty_leader + acc * 8);
        else mbar_arrive_relaxed(&tempty[acc]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();   // the peer may still arrive on / commit to our barriers until here
  if (dyn && threadIdx.x == 0) {  // the last CTA out resets the schedule for the next launch
    __threadfence();
    if (atomicAdd(p.sched + 1, 1) == (int)gridDim.x - 1) {
      p.sched[0] = 0;
      p.sched[1] = 0;
      __threadfence();
    }
  }
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_2sm<C::TMEM_COLS>(tmem_base);
    else tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------------- host

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

// 2-D bf16 row-major [rows, cols] map (row stride ld elements, default cols) with a
// {64 cols x box_rows} box, 128B swizzle.
static bool make_map(CUtensorMap* m, const void* base, long rows, long cols, int box_rows, long ld = 0) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld ? ld : cols) * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int EPI, int CG, bool BMN = false>
static cudaError_t launch_t(const GemmLaunch& L, cudaStream_t s) {
  using C = Cfg<BN, CG, EPI>;
  CUtensorMap ma, mb0, mb1, ma32, ma64;
  long a_rows = L.a_rows > 0 ? L.a_rows : 1;
  const long lda = L.lda ? L.lda : L.K;
  if (!make_map(&ma, L.A, a_rows, L.K, L.a_idx ? 1 : BM, lda)) return cudaErrorInvalidValue;   // gather4: {64, 1} box
  if (!make_map(&ma32, L.A, a_rows, L.K, 32, lda)) return cudaErrorInvalidValue;               // ragged group ends
  if (!make_map(&ma64, L.A, a_rows, L.K, 64, lda)) return cudaErrorInvalidValue;
  if (BMN) {   // B = [K rows, N cols] per group: boxes of {64 columns, 64 k-rows}
    if (!make_map(&mb0, L.B0, L.b_rows, L.N, 64)) return cudaErrorInvalidValue;
    if (!make_map(&mb1, L.B1 ? L.B1 : L.B0, L.b_rows, L.N, 64)) return cudaErrorInvalidValue;
  } else {
    if (!make_map(&mb0, L.B0, L.b_rows, L.K, C::HALF)) return cudaErrorInvalidValue;
    if (!make_map(&mb1, L.B1 ? L.B1 : L.B0, L.b_rows, L.K, C::HALF)) return cudaErrorInvalidValue;
  }
  auto kern = grouped_gemm_kernel<BN, EPI, CG, BMN>;
  static std::atomic<unsigned long long> attr_set{0};
  if (cudaError_t e = ensure_smem_attr(kern, C::SMEM, attr_set)) return e;
  GemmParams p;
  p.counts = L.counts;
  p.G = L.G;
  p.m_total = L.m_total;
  p.N = L.N;
  p.K = L.K;
  p.b_group_rows = L.b_group_rows;
  p.out = L.out;
  p.ldo = L.ldo;
  p.resid = L.resid;
  p.ldr = L.ldr;
  p.ret = L.ret;
  for (int i = 0; i < 8; ++i) p.peer_out[i] = L.peer_out[i];
  p.a_idx = L.a_idx;
  p.row_base = L.row_base;
  p.comb_out = L.comb_out;
  p.comb_resid = L.comb_resid;
  p.src_row = L.src_row;
  p.pos = L.pos;
  p.topk_w = L.topk_w;
  p.comb_cnt = L.comb_cnt;
  p.top_k = L.top_k;
  p.n_cb = L.N / (BN / 2);
  p.kb_split = L.kb_split;
  p.dh = L.dh;
  p.row_gate = L.row_gate;
  p.out2 = L.out2;
  p.dg_part = L.dg_part;
  p.dg_ld = L.dg_ld;
  // FSC_GEMM_STAGE_ROWS = 0 / 1 overrides the K-based choice (A/B measurements)
  static const int stage_env = getenv("FSC_GEMM_STAGE_ROWS") ? atoi(getenv("FSC_GEMM_STAGE_ROWS")) : -1;
  p.stage_rows = stage_env >= 0 ? stage_env : (L.epi == EPI_BF16 ? 1 : 0);
  p.sched = L.sched;
  int grid = L.num_ctas > 0 ? L.num_ctas : kNumSMs;
  if (CG == 2) grid &= ~1;
  if (grid < CG) grid = CG;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launches;
  return cudaLaunchKernelEx(&cfg, kern, ma, mb0, mb1, ma32, ma64, p);
}

int gemm_pick_bn(int epi, int N) {
  if (epi == EPI_SWIGLU || epi == EPI_SWIGLU_BWD) return (N % 128 == 0) ? 256 : (N % 64 == 0 ? 128 : 0);
  return (N % 256 == 0) ? 256 : (N % 128 == 0 ? 128 : (N % 64 == 0 ? 64 : 0));
}

cudaError_t launch_grouped_gemm(const GemmLaunch& L, cudaStream_t s) {
  if (L.G < 1 || L.G > kMaxGroups || L.K % BK || L.K <= 0) return cudaErrorInvalidValue;
  int bn = gemm_pick_bn(L.epi, L.N);
  if (!bn) return cudaErrorInvalidValue;
  if (L.bn == 128 && bn == 256 && (L.epi == EPI_SWIGLU ? L.N % 64 == 0 : L.N % 128 == 0)) bn = 128;
  if (L.a_rows == 0) return cudaSuccess;
  if (L.b_mn && L.epi != EPI_BF16 && L.epi != EPI_RESID_F32) return cudaErrorInvalidValue;
  // MN-major B is loaded as 64-column boxes: a CTA of a pair holds BN / 2 columns, so BN = 64
  // runs single-CTA tiles
  const int cgsel = (L.b_mn && bn == 64) ? 1 : L.cta_group;
#define FSC_GEMM_CASE(BNV, EV)                                          \
  if (bn == BNV && L.epi == EV) {                                       \
    if (L.b_mn) {                                                       \
      if (cgsel == 1) return launch_t<BNV, EV, 1, true>(L, s);          \
      return launch_t<BNV, EV, 2, true>(L, s);                          \
    }                                                                   \
    if (cgsel == 1) return launch_t<BNV, EV, 1>(L, s);                  \
    return launch_t<BNV, EV, 2>(L, s);                                  \
  }
#define FSC_GEMM_CASE_K(BNV, EV)                                        \
  if (bn == BNV && L.epi == EV) {                                       \
    if (L.cta_group == 1) return launch_t<BNV, EV, 1>(L, s);            \
    return launch_t<BNV, EV, 2>(L, s);                                  \
  }
  FSC_GEMM_CASE_K(256, EPI_SWIGLU)
  FSC_GEMM_CASE_K(128, EPI_SWIGLU)
  FSC_GEMM_CASE_K(256, EPI_SWIGLU_BWD)
  FSC_GEMM_CASE_K(128, EPI_SWIGLU_BWD)
  FSC_GEMM_CASE(256, EPI_BF16)
  FSC_GEMM_CASE(128, EPI_BF16)
  FSC_GEMM_CASE(64, EPI_BF16)
  FSC_GEMM_CASE(256, EPI_RESID_F32)
  FSC_GEMM_CASE(128, EPI_RESID_F32)
  FSC_GEMM_CASE(64, EPI_RESID_F32)
#undef FSC_GEMM_CASE
#undef FSC_GEMM_CASE_K
  return cudaErrorInvalidValue;
}

}  // namespace fsc
