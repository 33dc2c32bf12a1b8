// Internal launch interface of the libfsc kernels (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fsc {

// number of kernels this process has launched through libfsc (evidence for bench's gpu_launches)
extern long g_launches;

enum { EPI_BF16 = 0, EPI_SWIGLU = 1, EPI_RESID_F32 = 2, EPI_SWIGLU_BWD = 3 };

struct GemmParams {
  const int* counts;  // [G] rows per group (device) or nullptr -> one group of m_total rows
  int G;
  int m_total;
  int N;              // output columns (h columns for SwiGLU)
  int K;
  int b_group_rows;   // rows of B0/B1 per group
  void* out;
  long ldo;
  const float* resid;
  long ldr;
  // EPI_BF16 scatter (fused combine): row r of the tile goes to rank
  // (ret[r] >> 24), row (ret[r] & 0xFFFFFF) of peer_out[rank]; nullptr = local store
  const int* ret;
  void* peer_out[8];
  // A gather (EP = 1, fused permute): row r of the grouped problem is row a_idx[r]
  // of A (TMA gather4); nullptr = A rows are contiguous in group order
  const int* a_idx;
  // EPI_BF16 fused gate-weighted unpermute (EP = 1 blocking): after a
  // row's y columns are stored, its (token, column block) counter is bumped; the
  // k-th arrival computes comb_out[t] = comb_resid[t] + sum_j w[t,j] y[pos[t,j]]
  // (slot order, fp32, bitwise the unpermute kernel) for that column block.
  // all-reduce EP mode: the local experts' rows sit at [*row_base, ...) of the
  // globally expert-sorted A / out buffers (device int, nullptr = 0)
  const int* row_base;
  float* comb_out;             // nullptr: no fusion
  const float* comb_resid;
  const int* src_row;          // [R] token of send row
  const int* pos;              // [T, k]
  const float* topk_w;         // [T, k]
  int* comb_cnt;               // [T, n_cb] zero between calls (the last arrival resets)
  int top_k, n_cb;
  int stage_rows;              // bf16 epilogue: 1 = staged row-contiguous stores, 0 = direct
  int* sched;                  // dynamic tile schedule {claim counter, done counter} or nullptr
  // MN-major B (dgrad GEMMs, template BMN): B is [K rows, N cols] per group, group g's K rows
  // start at g * b_group_rows; kb_split > 0: k-blocks >= kb_split read tmB1 (rows restart at
  // 0), i.e. the K dimension is [B0 rows ; B1 rows] (dX = [dU | dV] [W1 ; W2])
  int kb_split;
  // EPI_SWIGLU_BWD (recomputed u = A W1^T, v = A W2^T; N = c): with dh_u = dh [M, N] bf16 and
  // the row gate g (row_gate, nullptr = 1): h = u SiLU(v), dh = g dh_u, du = dh SiLU(v),
  // dv = dh u SiLU'(v); out (ldo = 2N) = [du | dv] bf16, out2 [M, N] = g h bf16,
  // dg_part[row * dg_ld + tile * 2 + half] = partial sum_cols h dh_u (fp32, per warp half)
  const uint16_t* dh;
  const float* row_gate;
  void* out2;
  float* dg_part;
  int dg_ld;
};

struct GemmLaunch {
  const void* A;      // bf16 [a_rows, K] (row stride lda, 0 = K)
  long a_rows;
  long lda = 0;
  const void* B0;     // bf16 [b_rows, K]  (W1 for SwiGLU, else the only B)
  const void* B1;     // bf16 [b_rows, K]  (W2 for SwiGLU) or nullptr
  long b_rows;
  int b_group_rows;
  int K, N, G;
  const int* counts;
  int m_total;
  void* out;
  long ldo;
  const float* resid;
  long ldr;
  int epi;
  int num_ctas;       // persistent grid (<= 148); 0 = all SMs
  int* sched = nullptr;  // dynamic tile schedule: 2 ints, zero between launches (nullptr: static stride)
  int cta_group = 2;  // 2: CTA pairs, MMA M=256 (default); 1: single-CTA M=128 tiles
  const int* ret = nullptr;           // scatter map (see GemmParams)
  void* peer_out[8] = {};
  const int* a_idx = nullptr;         // A gather map (see GemmParams); A then has a_rows source rows
  const int* row_base = nullptr;      // device row offset of group 0 (see GemmParams)
  int bn = 0;                         // tile width override (0 = auto); must suit N and the epilogue
  float* comb_out = nullptr;          // fused unpermute (see GemmParams)
  const float* comb_resid = nullptr;
  const int* src_row = nullptr;
  const int* pos = nullptr;
  const float* topk_w = nullptr;
  int* comb_cnt = nullptr;
  int top_k = 0;
  bool b_mn = false;                  // B MN-major [K rows, N cols] per group (dgrad)
  int kb_split = 0;                   // see GemmParams
  const uint16_t* dh = nullptr;       // EPI_SWIGLU_BWD inputs / outputs (see GemmParams)
  const float* row_gate = nullptr;
  void* out2 = nullptr;
  float* dg_part = nullptr;
  int dg_ld = 0;
};

cudaError_t launch_grouped_gemm(const GemmLaunch& L, cudaStream_t s);

// K4 backward, weight gradients (gemm_wgrad.cu): per group g (rows [row_off[g], +M_g) of
// A and B, M_g from counts or m_total, offset by *row_base):
//   out[g][i][j] (+)= sum_m A[m, a_col0 + i] * B[m, b_col0 + j],  i < N1, j < N2  (fp32)
struct WgradParams {
  const int* counts;   // [G] device, or nullptr -> one group of m_total rows
  int G, m_total;
  const int* row_base; // device int or nullptr
  int N1, N2;          // N2 % 64 == 0
  const uint16_t* A;   // bf16 row-major, row stride lda
  long lda;
  int a_col0;
  const uint16_t* B;
  long ldb;
  int b_col0;
  float* out;          // fp32 [G, N1, N2]
  int accumulate;      // 1: out += (gradient accumulation)
};
cudaError_t launch_wgrad_gemm(const WgradParams& p, long a_rows, long b_rows, int ctas, cudaStream_t s);
int gemm_pick_bn(int epi, int N);

// K1: RMSNorm + fp32 router logits + top-k + renormalised gates (+ fp64 near-tie refinement)
struct RouterLaunch {
  const float* x;        // [T, d]
  const float* gamma;    // [d]
  const float* w_router; // [E, d]
  int T, d, E, k;
  float eps;
  uint16_t* xn;          // bf16 [T, d]
  int* topk_idx;         // [T, k]
  float* topk_w;         // [T, k]
  float* logits;         // optional [T, E]
  int* n_refined;        // optional device counter of tokens refined in fp64
  float* part;           // workspace [kRouterSplitRows, 128]: split-d raw partial logits (small T)
  double* part_sq;       // workspace [kRouterSplitRows]: split-d partial sums of x^2
  float* w_scaled;       // workspace [E, d]: gamma * W_R
  float* w_sq;           // workspace [E]: ||gamma * W_R[e]||^2
  int rpb = 32;          // tokens per CTA (set by launch_router)
  // exact tensor-core path (router_tc_kernel; E <= 128, d % 128 == 0, k <= 8), used when tc != 0
  int8_t* i8_w;          // workspace [3, EP, d]: base-2^7 digit planes of floor((gamma W_R)_e 2^21 / s_e)
  float* i8_exp;         // workspace [3, EP]: s_e and the two per-expert error-bound coefficients
  int tc;
  int f64 = 0;           // fp64 small-batch router (router_f64_kernel), chosen by the caller
  double* f64_w = nullptr;  // its workspace [d, 136]: gamma (.) W_R in fp64, k-major
};
// split-d partials: (token blocks) x (d splits) <= 2 x 148 CTAs of <= 32 rows
constexpr int kRouterSplitRows = 2 * 148 * 32;
cudaError_t launch_router(const RouterLaunch& L, cudaStream_t s);
// fp64 router for small batches (router_f64.cu): d % 64 == 0, d <= 8192, E <= 128
bool router_f64_supported(int d, int E, int k);
cudaError_t launch_router_f64(const RouterLaunch& L, cudaStream_t s);

// K2: deterministic histogram / scan / positions
//   hist   [n_chunks, E] per 32-token chunk; base [n_chunks, E]
//   counts [E], offsets [E+1], pos [T,k], src_row [T*k]
struct PermLaunch {
  const int* topk_idx;
  int T, k, E;
  int* hist;
  int* base;
  int* counts;
  int* offsets;
  int* pos;
  int* src_row;
};
cudaError_t launch_perm_maps(const PermLaunch& L, cudaStream_t s);
inline int perm_chunks(int T) { return (T + 31) / 32; }

// K3: xs[p] = xn[src_row[p]]  (bf16 rows of d); rng != nullptr: only rows p in
// [rng[0], rng[rng_n]) (device offsets of a range of experts)
// EP = 1 permute (picks scatter or gather by the size of xn against L2)
cudaError_t launch_permute_ep1(const uint16_t* xn, const int* src_row, const int* pos, uint16_t* xs, int T, int k,
                               int d, cudaStream_t s);
// xs[pos[t, j]] = xn[t] by source token (EP = 1 dispatch): each xn row read once
cudaError_t launch_permute_scatter(const uint16_t* xn, const int* pos, uint16_t* xs, int T, int k, int d,
                                   cudaStream_t s);
cudaError_t launch_permute_rows(const uint16_t* xn, const int* src_row, uint16_t* xs, int R, int d,
                                cudaStream_t s, const int* rng = nullptr, int rng_n = 0);

// K5: out[t] = resid[t] + sum_j w[t,j] * y[pos[t,j]]   (fp32 out, bf16 y, slot order)
cudaError_t launch_unpermute(const uint16_t* y, const int* pos, const float* w, const float* resid,
                             float* out, int T, int k, int d, cudaStream_t s);
// K5, local experts only (all-reduce EP mode): out[t] = sum over slots j with
// e_lo <= idx[t,j] < e_hi of w[t,j] * y[pos[t,j]], from 0 in slot order
cudaError_t launch_unpermute_local(const uint16_t* y, const int* pos, const float* w, const int* idx, int e_lo,
                                   int e_hi, float* out, int T, int k, int d, cudaStream_t s);

// attention filler (attention.cu)
cudaError_t launch_rmsnorm_bf16(const float* x, const float* gamma, uint16_t* y, int T, int d, float eps,
                                cudaStream_t s);
cudaError_t launch_rope(uint16_t* qkv, int T, int n_heads, int n_kv_heads, int hd, int seq_len, float theta,
                        cudaStream_t s);
cudaError_t launch_flash_attn(const uint16_t* qkv, uint16_t* out, int T, int Hq, int Hkv, int hd, int seq_len,
                              cudaStream_t s);

// elementwise helpers
cudaError_t launch_copy_f32(const float* src, float* dst, long n, cudaStream_t s);
// test instrument: one thread spinning for ns nanoseconds of %globaltimer (ns <= 0: no launch)
cudaError_t launch_spin(long long ns, cudaStream_t s);
// debug: *bad += number of non-finite values of x [n] (n % 4 == 0)
cudaError_t launch_count_nonfinite(const float* x, long n, int* bad, cudaStream_t s);

}  // namespace fsc
