// EP transport: Dispatch / Combine between the P ranks of an expert-parallel
// group (§2 "Dispatch" and "Combine"), device-initiated over
// peer memory. Every rank exports one symmetric region (CUDA IPC handle) that
// the others map; all data movement and synchronisation then happens inside
// kernels, with no host round trip:
//
//   counts  (a5): each source s writes its per-expert counts into row s of every
//                 peer's cnt matrix [P][E], raises flag_cnt[s] there, and waits
//                 until all P rows of its own matrix are in. Every rank then
//                 knows the full matrix and derives, without further exchange,
//                 where its rows land in each destination's receive buffer.
//   dispatch(a6): the permute kernel writes each copy (t, j) of xn straight into
//                 the owning rank's receive buffer xr (expert-major, then source
//                 rank, then token: C-amb-11) plus the return address of the row;
//                 the last CTA raises flag_disp[s] at every destination.
//   combine (a9): fused into the down-projection GEMM's epilogue (gemm.cu,
//                 EPI_BF16 with a scatter map): each output row is stored into its
//                 source rank's ys buffer at the row it was sent from; a signal
//                 kernel then raises flag_comb at every source.
// Flags carry a per-call epoch, so nothing is ever reset. The epoch lives in device
// memory (bumped by the counts kernel, read by the others), so a captured CUDA graph
// of a whole layer replays correctly. The same code serves
// P processes on one GPU (tests) and one process per GPU over NVLink/NVSwitch.
#include <cuda_fp16.h>
#include <string.h>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

using namespace fsc;

namespace {
constexpr int kMaxP = 8;
constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

struct Layout {  // byte offsets inside every rank's symmetric region
  size_t flags, cnt, ret, xr, ys, part[2], red[2], xq, xsc, gr, gate, dgs, total;
};

// FLAG_CNT, FLAG_DISP, FLAG_COMB, then (READY, DONE) per all-reduce channel
// (channel 0: MoE routed sum; channel 1: TP attention o-projection), then the backward's
// gradient dispatch / gradient combine
constexpr int kFlagRows = 9;
constexpr int kEpochs = 2;     // epoch counters: [0] all-to-all + AR channel 0, [1] AR channel 1

Layout layout_for(const fsc_ctx* c) {
  Layout L{};
  const size_t P = c->ep, E = c->cfg.n_experts, d = c->cfg.d, T = c->cfg.max_tokens;
  const size_t Tk = T * c->cfg.top_k;
  L.flags = 0;                                       // int [kFlagRows][kMaxP] + epochs
  L.cnt = align_up(L.flags + (kFlagRows * kMaxP + kEpochs) * sizeof(int));
  if (c->ep_mode == FSC_EP_ALLREDUCE) {              // replicated tokens: fp32 partial + reduced rows, x2
    L.ret = L.xr = L.ys = L.cnt;
    size_t o = L.cnt;
    for (int ch = 0; ch < 2; ++ch) {
      L.part[ch] = o;
      L.red[ch] = align_up(L.part[ch] + T * d * sizeof(float));
      o = align_up(L.red[ch] + T * d * sizeof(float));
    }
    L.xq = L.xsc = L.gr = L.gate = L.dgs = L.total = o;
    return L;
  }
  L.ret = align_up(L.cnt + P * E * sizeof(int));     // int [max_recv]
  L.xr = align_up(L.ret + (size_t)c->max_recv * sizeof(int));
  L.ys = align_up(L.xr + (size_t)c->max_recv * d * 2);
  // backward (fsc_moe_backward): gradient rows + gates received per expert row, gate
  // gradients combined back per send row (the dX rows come back into ys)
  L.gr = align_up(L.ys + Tk * d * 2);
  L.gate = align_up(L.gr + (size_t)c->max_recv * d * 2);
  L.dgs = align_up(L.gate + (size_t)c->max_recv * sizeof(float));
  L.part[0] = L.part[1] = L.red[0] = L.red[1] = L.xq = L.xsc = L.total = align_up(L.dgs + Tk * sizeof(float));
  if (c->dispatch_fp8) {                             // FP8 payload: e4m3 rows + fp32 per-128-column scales
    L.xq = L.total;
    L.xsc = align_up(L.xq + (size_t)c->max_recv * d);
    L.total = align_up(L.xsc + (size_t)c->max_recv * (d / 128) * sizeof(float));
  }
  return L;
}

struct Peers {
  char* base[kMaxP];
};

enum { FLAG_CNT = 0, FLAG_DISP = 1, FLAG_COMB = 2, FLAG_AR_READY = 3, FLAG_AR_DONE = 4,   // + 2 ch for AR
       FLAG_GDISP = 7, FLAG_GCOMB = 8 };
constexpr int kEpochSlot = kFlagRows * kMaxP;   // int index of the epoch counters in the flags area

FSC_DEVINL int read_epoch(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

FSC_DEVINL int* flag_ptr(char* base, int slot, int src) {
  return reinterpret_cast<int*>(base) + slot * kMaxP + src;
}
FSC_DEVINL void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
FSC_DEVINL int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FSC_DEVINL unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until every source's flag reached this call's epoch. A peer that never
// arrives (dead rank, broken bootstrap) must not hang the GPU: after 30 s the kernel
// traps, which surfaces as FSC_ERR_CUDA on the host instead of a hung stream.
constexpr unsigned long long kFlagTimeoutNs = 30ull * 1000 * 1000 * 1000;
FSC_DEVINL void wait_flags(char* mybase, int slot, int P, int epoch) {
  const unsigned long long t0 = global_ns();
  for (int s = 0; s < P; ++s) {
    const int* f = flag_ptr(mybase, slot, s);
    while (ld_acquire_sys(f) - epoch < 0) {
      __nanosleep(64);
      if (global_ns() - t0 > kFlagTimeoutNs) __trap();
    }
  }
}
// Copy one row of dv uint4 with a warp, 8 loads in flight per lane before the stores
// (remote stores are posted; the loads' latency is what limits a warp's throughput).
// STREAM: the source is read once (evict-first); else it stays in L2 (xn rows are read k times).
template <bool STREAM>
FSC_DEVINL void copy_row_warp(const uint4* __restrict__ a, uint4* b, int dv, int lane) {
  for (int i0 = lane; i0 < dv; i0 += 256) {
    uint4 buf[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + 32 * u < dv) buf[u] = STREAM ? __ldcs(a + i0 + 32 * u) : ld_keep_u4(a + i0 + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + 32 * u < dv) b[i0 + 32 * u] = buf[u];
  }
}
}  // namespace

struct fsc_peer_state {
  char* local = nullptr;          // my symmetric region
  Layout lay{};
  Peers peers{};                  // mapped regions of every rank (peers.base[rank] == local)
  cudaIpcMemHandle_t my_handle{};
  bool opened[kMaxP] = {};
  int* send_base = nullptr;       // [E]   first row of my expert-e rows in the owner's xr
  int* ticket = nullptr;          // [1]   dispatch-kernel completion ticket
};

// ----------------------------------------------------------------------------- kernels

// a5: counts all-gather through peer stores + receive-side bookkeeping.
__global__ void __launch_bounds__(256) ep_counts_kernel(Peers peers, int rank, int P, int E, int e_loc, int* epoch_ptr,
                                                        size_t off_cnt, const int* __restrict__ counts,
                                                        int* __restrict__ send_base, int* __restrict__ recv_counts) {
  __shared__ int cnt[kMaxP * 128];
  __shared__ int s_epoch;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_epoch = read_epoch(epoch_ptr) + 1;   // this call's epoch
    *epoch_ptr = s_epoch;
  }
  __syncthreads();
  const int epoch = s_epoch;
  for (int i = tid; i < P * E; i += blockDim.x) {
    const int p = i / E, e = i % E;
    reinterpret_cast<int*>(peers.base[p] + off_cnt)[rank * E + e] = counts[e];
  }
  __threadfence_system();
  __syncthreads();
  if (tid < P) st_release_sys(flag_ptr(peers.base[tid], FLAG_CNT, rank), epoch);
  if (tid == 0) wait_flags(peers.base[rank], FLAG_CNT, P, epoch);
  __syncthreads();
  const int* my = reinterpret_cast<const int*>(peers.base[rank] + off_cnt);
  for (int i = tid; i < P * E; i += blockDim.x) cnt[i] = ld_acquire_sys(my + i);
  __syncthreads();
  // send_base[e]: where my copies for expert e start inside its owner's receive
  // buffer = rows of the owner's earlier local experts (all sources) + rows of
  // expert e from lower-ranked sources (C-amb-11 layout).
  for (int e = tid; e < E; e += blockDim.x) {
    const int p = e / e_loc;
    int b = 0;
    for (int e2 = p * e_loc; e2 < e; ++e2)
      for (int s = 0; s < P; ++s) b += cnt[s * E + e2];
    for (int s = 0; s < rank; ++s) b += cnt[s * E + e];
    send_base[e] = b;
  }
  for (int el = tid; el < e_loc; el += blockDim.x) {
    int m = 0;
    for (int s = 0; s < P; ++s) m += cnt[s * E + rank * e_loc + el];
    recv_counts[el] = m;
  }
}

// a4 + a6: permute-and-dispatch. One warp per send row q (expert-sorted order).
__global__ void __launch_bounds__(256) ep_dispatch_kernel(Peers peers, int rank, int P, int R, int d, int E,
                                                          int e_loc, const int* epoch_ptr, size_t off_xr,
                                                          size_t off_ret,
                                                          const uint4* __restrict__ xn, const int* __restrict__ src_row,
                                                          const int* __restrict__ offsets,
                                                          const int* __restrict__ send_base, int* ticket,
                                                          int zero_bytes) {
  __shared__ int s_off[129];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) s_off[i] = offsets[i];
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dv = d / 8;
  for (long q = (long)blockIdx.x * 8 + w; q < (zero_bytes ? 0 : R); q += (long)gridDim.x * 8) {
    int lo = 0, hi = E;                    // expert of send row q
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_off[mid] <= q) lo = mid; else hi = mid;
    }
    const int e = lo, p = e / e_loc;
    const long dst = send_base[e] + (q - s_off[e]);
    const uint4* a = xn + (long)src_row[q] * dv;
    uint4* b = reinterpret_cast<uint4*>(peers.base[p] + off_xr) + dst * dv;
    copy_row_warp<false>(a, b, dv, lane);
    if (lane == 0) reinterpret_cast<int*>(peers.base[p] + off_ret)[dst] = (rank << 24) | (int)q;
  }
  // last CTA out raises the dispatch flag at every destination
  const int epoch = read_epoch(epoch_ptr);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(ticket, 1) == (int)gridDim.x - 1) {
      *ticket = 0;
      __threadfence_system();
      for (int p = 0; p < P; ++p) st_release_sys(flag_ptr(peers.base[p], FLAG_DISP, rank), epoch);
    }
  }
}

// a4 + a6 with the FP8 payload: every row is sent as e4m3 with
// one fp32 scale per 128 columns: s_b = amax_b / 448, q = e4m3_rn_satfinite(x / s_b)
// (oracle/moe.py fp8_dispatch_payload). One warp per send row; a lane's 8 columns
// lie in one 128-column block, so a half-warp reduction gives the block amax.
FSC_DEVINL uint32_t f32x2_to_e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}
__global__ void __launch_bounds__(256) ep_dispatch_fp8_kernel(Peers peers, int rank, int P, int R, int d, int E,
                                                              int e_loc, const int* epoch_ptr, size_t off_xq,
                                                              size_t off_xsc, size_t off_ret,
                                                              const uint4* __restrict__ xn,
                                                              const int* __restrict__ src_row,
                                                              const int* __restrict__ offsets,
                                                              const int* __restrict__ send_base, int* ticket,
                                                          int zero_bytes) {
  __shared__ int s_off[129];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) s_off[i] = offsets[i];
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dv = d / 8;
  for (long q = (long)blockIdx.x * 8 + w; q < (zero_bytes ? 0 : R); q += (long)gridDim.x * 8) {
    int lo = 0, hi = E;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_off[mid] <= q) lo = mid; else hi = mid;
    }
    const int e = lo, p = e / e_loc;
    const long dst = send_base[e] + (q - s_off[e]);
    const uint4* a = xn + (long)src_row[q] * dv;
    uint2* bq = reinterpret_cast<uint2*>(peers.base[p] + off_xq) + dst * dv;
    float* bs = reinterpret_cast<float*>(peers.base[p] + off_xsc) + dst * (d / 128);
    for (int c0 = 0; c0 < dv; c0 += 32) {          // warp-uniform trip count (half-warp shuffles below)
      const int c = c0 + lane;
      const bool ok = c < dv;
      const uint4 u = ok ? a[c] : make_uint4(0u, 0u, 0u, 0u);
      float v[8] = {bf16lo(u.x), bf16hi(u.x), bf16lo(u.y), bf16hi(u.y),
                    bf16lo(u.z), bf16hi(u.z), bf16lo(u.w), bf16hi(u.w)};
      float m = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) m = fmaxf(m, fabsf(v[i]));
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));   // 16 lanes = 128 cols
      const float sc = m > 0.f ? __fdiv_rn(m, 448.f) : 1.f;
      uint32_t w01 = f32x2_to_e4m3x2(__fdiv_rn(v[0], sc), __fdiv_rn(v[1], sc));
      uint32_t w23 = f32x2_to_e4m3x2(__fdiv_rn(v[2], sc), __fdiv_rn(v[3], sc));
      uint32_t w45 = f32x2_to_e4m3x2(__fdiv_rn(v[4], sc), __fdiv_rn(v[5], sc));
      uint32_t w67 = f32x2_to_e4m3x2(__fdiv_rn(v[6], sc), __fdiv_rn(v[7], sc));
      if (ok) {
        bq[c] = make_uint2(w01 | (w23 << 16), w45 | (w67 << 16));
        if ((c & 15) == 0) bs[c / 16] = sc;
      }
    }
    if (lane == 0) reinterpret_cast<int*>(peers.base[p] + off_ret)[dst] = (rank << 24) | (int)q;
  }
  const int epoch = read_epoch(epoch_ptr);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(ticket, 1) == (int)gridDim.x - 1) {
      *ticket = 0;
      __threadfence_system();
      for (int p = 0; p < P; ++p) st_release_sys(flag_ptr(peers.base[p], FLAG_DISP, rank), epoch);
    }
  }
}

// receiver: xr = bf16(fp32(q * s)) for every received row (after the dispatch flags)
__global__ void __launch_bounds__(256) ep_dequant_fp8_kernel(const uint2* __restrict__ xq, const float* __restrict__ xsc,
                                                             const int* __restrict__ recv_counts, int e_loc,
                                                             uint4* __restrict__ xr, int d) {
  __shared__ long s_rows;
  if (threadIdx.x == 0) {
    long n = 0;
    for (int i = 0; i < e_loc; ++i) n += recv_counts[i];
    s_rows = n;
  }
  __syncthreads();
  const int dv = d / 8;
  const long items = s_rows * dv;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < items; i += (long)gridDim.x * blockDim.x) {
    const long r = i / dv;
    const int c = (int)(i - r * dv);
    const uint2 qq = __ldcv(xq + i);
    const float sc = __ldcv(xsc + r * (d / 128) + c / 16);
    float f[8];
    const uint32_t wds[2] = {qq.x, qq.y};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const uint16_t pair = (uint16_t)(wds[h / 2] >> (16 * (h & 1)));
      uint32_t hx2;
      asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(hx2) : "h"(pair));
      const __half2 h2 = *reinterpret_cast<const __half2*>(&hx2);
      f[2 * h] = __low2float(h2) * sc;
      f[2 * h + 1] = __high2float(h2) * sc;
    }
    xr[i] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                       pack_bf16x2(f[6], f[7]));
  }
}

__global__ void ep_signal_kernel(Peers peers, int rank, int P, int slot, const int* epoch_ptr) {
  const int epoch = read_epoch(epoch_ptr);
  __threadfence_system();
  if (threadIdx.x < P) st_release_sys(flag_ptr(peers.base[threadIdx.x], slot, rank), epoch);
}

// a9, decoupled from the down GEMM (FSC_COMBINE_STREAM): runs on the comm stream after
// GEMM2 stored the expert outputs y locally in the receive layout; every received row r
// goes back to its source rank (ret[r] >> 24), row (ret[r] & 0xFFFFFF) of that rank's
// ys (the send layout, "Combine"). One warp per row, 16 B per lane; the
// last CTA raises FLAG_COMB at every source. zero_bytes: flags only (test instrument).
__global__ void __launch_bounds__(256) ep_combine_kernel(Peers peers, int rank, int P, int e_loc,
                                                         const int* __restrict__ recv_counts,
                                                         const int* __restrict__ ret, const uint4* __restrict__ y,
                                                         size_t off_ys, int d, const int* epoch_ptr, int* ticket,
                                                         int zero_bytes) {
  __shared__ long s_rows;
  if (threadIdx.x == 0) {
    long n = 0;
    for (int i = 0; i < e_loc; ++i) n += recv_counts[i];
    s_rows = zero_bytes ? 0 : n;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dv = d / 8;
  for (long r = (long)blockIdx.x * 8 + w; r < s_rows; r += (long)gridDim.x * 8) {
    const int v = __ldg(ret + r);
    const uint4* a = y + r * dv;
    uint4* b = reinterpret_cast<uint4*>(peers.base[(uint32_t)v >> 24] + off_ys) + (long)(v & 0xFFFFFF) * dv;
    copy_row_warp<true>(a, b, dv, lane);
  }
  const int epoch = read_epoch(epoch_ptr);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(ticket, 1) == (int)gridDim.x - 1) {
      *ticket = 0;
      __threadfence_system();
      for (int p = 0; p < P; ++p) st_release_sys(flag_ptr(peers.base[p], FLAG_COMB, rank), epoch);
    }
  }
}

// Backward gradient dispatch (the mirror of the Combine): every copy
// (t, j) sends G[t] (fp32 -> bf16) and its gate g_tj to the row of the owner's receive
// buffer where the forward's Dispatch put xn[t] (same send_base / offsets). One warp per
// copy; the last CTA raises FLAG_GDISP at every destination.
__global__ void __launch_bounds__(256) ep_dispatch_grad_kernel(Peers peers, int rank, int P, int T, int k, int d,
                                                               int e_loc, const int* epoch_ptr, size_t off_gr,
                                                               size_t off_gate, const float* __restrict__ G,
                                                               const int* __restrict__ idx, const int* __restrict__ pos,
                                                               const float* __restrict__ topk_w,
                                                               const int* __restrict__ offsets,
                                                               const int* __restrict__ send_base, int* ticket) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dv = d / 8;
  for (long c = (long)blockIdx.x * 8 + w; c < (long)T * k; c += (long)gridDim.x * 8) {
    const long t = c / k;
    const int e = __ldg(idx + c), q = __ldg(pos + c), p = e / e_loc;
    const long dst = __ldg(send_base + e) + (q - __ldg(offsets + e));
    const float4* a = reinterpret_cast<const float4*>(G + t * d);
    uint4* b = reinterpret_cast<uint4*>(peers.base[p] + off_gr) + dst * dv;
    for (int i = lane; i < dv; i += 32) {
      const float4 lo = __ldg(a + 2 * i), hi = __ldg(a + 2 * i + 1);
      b[i] = make_uint4(pack_bf16x2(lo.x, lo.y), pack_bf16x2(lo.z, lo.w), pack_bf16x2(hi.x, hi.y),
                        pack_bf16x2(hi.z, hi.w));
    }
    if (lane == 0) reinterpret_cast<float*>(peers.base[p] + off_gate)[dst] = __ldg(topk_w + c);
  }
  const int epoch = read_epoch(epoch_ptr);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(ticket, 1) == (int)gridDim.x - 1) {
      *ticket = 0;
      __threadfence_system();
      for (int p = 0; p < P; ++p) st_release_sys(flag_ptr(peers.base[p], FLAG_GDISP, rank), epoch);
    }
  }
}

// Backward gradient combine (the mirror of the Dispatch): received row r's dX row (y, the
// dgrad GEMM output, receive layout) goes back to its source's ys at the send row it came
// from, with its gate gradient dg = sum of the row's dg_part entries (fixed order).
__global__ void __launch_bounds__(256) ep_combine_grad_kernel(Peers peers, int rank, int P, int e_loc,
                                                              const int* __restrict__ recv_counts,
                                                              const int* __restrict__ ret,
                                                              const uint4* __restrict__ y, size_t off_ys,
                                                              size_t off_dgs, const float* __restrict__ dg_part,
                                                              int dg_n, int dg_ld, int d, const int* epoch_ptr,
                                                              int* ticket) {
  __shared__ long s_rows;
  if (threadIdx.x == 0) {
    long n = 0;
    for (int i = 0; i < e_loc; ++i) n += recv_counts[i];
    s_rows = n;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dv = d / 8;
  for (long r = (long)blockIdx.x * 8 + w; r < s_rows; r += (long)gridDim.x * 8) {
    const int v = __ldg(ret + r);
    char* base = peers.base[(uint32_t)v >> 24];
    const long q = v & 0xFFFFFF;
    copy_row_warp<true>(y + r * dv, reinterpret_cast<uint4*>(base + off_ys) + q * dv, dv, lane);
    if (lane == 0) {
      float g = 0.f;
      for (int i = 0; i < dg_n; ++i) g += __ldg(dg_part + r * dg_ld + i);
      reinterpret_cast<float*>(base + off_dgs)[q] = g;
    }
  }
  const int epoch = read_epoch(epoch_ptr);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(ticket, 1) == (int)gridDim.x - 1) {
      *ticket = 0;
      __threadfence_system();
      for (int p = 0; p < P; ++p) st_release_sys(flag_ptr(peers.base[p], FLAG_GCOMB, rank), epoch);
    }
  }
}

__global__ void ep_wait_kernel(char* mybase, int slot, int P, const int* epoch_ptr) {
  if (threadIdx.x == 0) wait_flags(mybase, slot, P, read_epoch(epoch_ptr));
  __syncthreads();
}

// ----------------------------------------------------------------------------- EP all-reduce (inference variant)
// PAPER.md:215-217 (vLLM): activations replicated on every rank, experts EP-sharded;
// each rank's local-expert partial sum is all-reduced. Reduce-scatter + all-gather
// over peer memory in one kernel: rank p sums rows [p T/P, (p+1) T/P) of the P
// partials IN RANK ORDER (deterministic, identical on every rank) and stores the
// result into every rank's `red` buffer; the last CTA raises FLAG_AR_DONE there.

// bump the epoch and announce "my partial is complete" (stream order after the unpermute)
__global__ void ar_begin_kernel(Peers peers, int rank, int P, int* epoch_ptr, int ready_slot) {
  __shared__ int s_epoch;
  if (threadIdx.x == 0) {
    s_epoch = read_epoch(epoch_ptr) + 1;
    *epoch_ptr = s_epoch;
  }
  __syncthreads();
  __threadfence_system();
  if (threadIdx.x < P) st_release_sys(flag_ptr(peers.base[threadIdx.x], ready_slot, rank), s_epoch);
}

__global__ void __launch_bounds__(256) ar_reduce_kernel(Peers peers, int rank, int P, long rows0, long rows1, int d,
                                                        size_t off_part, size_t off_red, const int* epoch_ptr,
                                                        int* ticket, int ready_slot, int done_slot) {
  const int epoch = read_epoch(epoch_ptr);
  if (threadIdx.x == 0) wait_flags(peers.base[rank], ready_slot, P, epoch);
  __syncthreads();
  const long dv = d / 4;
  const long n = (rows1 - rows0) * dv;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long off = rows0 * dv + i;
    float4 acc = __ldcv(reinterpret_cast<const float4*>(peers.base[0] + off_part) + off);
    for (int p = 1; p < P; ++p) {
      const float4 v = __ldcv(reinterpret_cast<const float4*>(peers.base[p] + off_part) + off);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    for (int p = 0; p < P; ++p) reinterpret_cast<float4*>(peers.base[p] + off_red)[off] = acc;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(ticket, 1) == (int)gridDim.x - 1) {
      *ticket = 0;
      __threadfence_system();
      for (int p = 0; p < P; ++p) st_release_sys(flag_ptr(peers.base[p], done_slot, rank), epoch);
    }
  }
}

// wait every rank's slice, then out = resid + reduced (fp32; resid may alias out)
__global__ void __launch_bounds__(256) ar_finish_kernel(char* mybase, int P, const int* epoch_ptr, size_t off_red,
                                                        const float* resid, float* out, long n4, int done_slot) {
  if (threadIdx.x == 0) wait_flags(mybase, done_slot, P, read_epoch(epoch_ptr));
  __syncthreads();
  const float4* red = reinterpret_cast<const float4*>(mybase + off_red);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    const float4 r = __ldcv(red + i);
    float4 a = resid ? reinterpret_cast<const float4*>(resid)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    a.x += r.x;
    a.y += r.y;
    a.z += r.z;
    a.w += r.w;
    reinterpret_cast<float4*>(out)[i] = a;
  }
}

// ----------------------------------------------------------------------------- host side

size_t fsc_transport_blob_size() { return sizeof(cudaIpcMemHandle_t); }

#define TCK(call)                                                                                 \
  do {                                                                                            \
    cudaError_t e__ = (call);                                                                     \
    if (e__ != cudaSuccess) {                                                                     \
      fsc_set_error(ctx, "transport %s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e__)); \
      ctx->sticky = FSC_ERR_COMM;                                                                 \
      return FSC_ERR_COMM;                                                                        \
    }                                                                                             \
  } while (0)

int fsc_transport_init(fsc_ctx* ctx) {
  if (ctx->ep == 1) return FSC_OK;
  if (ctx->ep > kMaxP) {
    fsc_set_error(ctx, "ep_size %d > %d", ctx->ep, kMaxP);
    return FSC_ERR_CONFIG;
  }
  fsc_peer_state* st = new fsc_peer_state();
  ctx->peer = st;
  st->lay = layout_for(ctx);
  TCK(cudaMalloc(&st->local, st->lay.total));
  TCK(cudaMemset(st->local, 0, st->lay.flags + (kFlagRows * kMaxP + kEpochs) * sizeof(int)));
  TCK(cudaIpcGetMemHandle(&st->my_handle, st->local));
  TCK(cudaMalloc(&st->send_base, sizeof(int) * ctx->cfg.n_experts));
  TCK(cudaMalloc(&st->ticket, 3 * sizeof(int)));            // [0] dispatch / AR channel 0, [1] AR channel 1
  TCK(cudaMemset(st->ticket, 0, 3 * sizeof(int)));
  TCK(cudaMalloc(&ctx->recv_counts, sizeof(int) * ctx->e_loc));
  ctx->xr = reinterpret_cast<uint16_t*>(st->local + st->lay.xr);
  ctx->ys = reinterpret_cast<uint16_t*>(st->local + st->lay.ys);
  ctx->recv_rows_cap = ctx->max_recv;
  st->peers.base[ctx->rank] = st->local;
  TCK(cudaDeviceSynchronize());
  return FSC_OK;
}

int fsc_transport_export(fsc_ctx* ctx, void* blob) {
  if (ctx->ep == 1) return FSC_OK;
  memcpy(blob, &ctx->peer->my_handle, sizeof(cudaIpcMemHandle_t));
  return FSC_OK;
}

int fsc_transport_import(fsc_ctx* ctx, const void* blobs) {
  if (ctx->ep == 1) return FSC_OK;
  fsc_peer_state* st = ctx->peer;
  TCK(cudaSetDevice(ctx->device));
  for (int p = 0; p < ctx->ep; ++p) {
    if (p == ctx->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char*>(blobs) + p * sizeof(cudaIpcMemHandle_t), sizeof(h));
    void* ptr = nullptr;
    TCK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    st->peers.base[p] = static_cast<char*>(ptr);
    st->opened[p] = true;
  }
  return FSC_OK;
}

void fsc_transport_finalize(fsc_ctx* ctx) {
  fsc_peer_state* st = ctx->peer;
  if (!st) return;
  for (int p = 0; p < kMaxP; ++p)
    if (st->opened[p]) cudaIpcCloseMemHandle(st->peers.base[p]);
  if (st->local) cudaFree(st->local);
  if (st->send_base) cudaFree(st->send_base);
  if (st->ticket) cudaFree(st->ticket);
  if (ctx->recv_counts) cudaFree(ctx->recv_counts);
  delete st;
  ctx->peer = nullptr;
}

static int* epoch_ptr(fsc_ctx* ctx) {
  return reinterpret_cast<int*>(ctx->peer->local + ctx->peer->lay.flags) + kEpochSlot;
}

static bool connected(fsc_ctx* ctx) {
  for (int p = 0; p < ctx->ep; ++p)
    if (!ctx->peer->peers.base[p]) return false;
  return true;
}

// counts exchange + permute-and-dispatch on stream s (the caller picks compute or comm stream)
int fsc_transport_dispatch(fsc_ctx* ctx, int T, cudaStream_t s) {
  fsc_peer_state* st = ctx->peer;
  if (!connected(ctx)) {
    fsc_set_error(ctx, "EP transport not bootstrapped (fsc_bootstrap_export/import)");
    return FSC_ERR_STATE;
  }
  const fsc_moe_config& c = ctx->cfg;
  const int E = c.n_experts, P = ctx->ep;
  ++g_launches;
  ep_counts_kernel<<<1, 256, 0, s>>>(st->peers, ctx->rank, P, E, ctx->e_loc, epoch_ptr(ctx), st->lay.cnt, ctx->counts,
                                     st->send_base, ctx->recv_counts);
  TCK(cudaGetLastError());
  const int R = T * c.top_k;
  int blocks = (R + 7) / 8;
  if (blocks > ctx->comm_ctas) blocks = ctx->comm_ctas;   // a fraction of the SMs
  if (blocks < 1) blocks = 1;
  ++g_launches;
  if (ctx->dispatch_fp8)
    ep_dispatch_fp8_kernel<<<blocks, 256, 0, s>>>(st->peers, ctx->rank, P, R, c.d, E, ctx->e_loc, epoch_ptr(ctx),
                                                  st->lay.xq, st->lay.xsc, st->lay.ret,
                                                  reinterpret_cast<const uint4*>(ctx->xn), ctx->src_row, ctx->offsets,
                                                  st->send_base, st->ticket, ctx->a2a_zero_bytes);
  else
    ep_dispatch_kernel<<<blocks, 256, 0, s>>>(st->peers, ctx->rank, P, R, c.d, E, ctx->e_loc, epoch_ptr(ctx),
                                              st->lay.xr, st->lay.ret, reinterpret_cast<const uint4*>(ctx->xn),
                                              ctx->src_row, ctx->offsets, st->send_base, st->ticket,
                                              ctx->a2a_zero_bytes);
  TCK(cudaGetLastError());
  return FSC_OK;
}

int fsc_transport_dispatch_wait(fsc_ctx* ctx, cudaStream_t s) {
  ++g_launches;
  ep_wait_kernel<<<1, 32, 0, s>>>(ctx->peer->local, FLAG_DISP, ctx->ep, epoch_ptr(ctx));
  TCK(cudaGetLastError());
  if (ctx->dispatch_fp8) {
    fsc_peer_state* st = ctx->peer;
    const int d = ctx->cfg.d;
    ++g_launches;
    ep_dequant_fp8_kernel<<<4 * kNumSMs, 256, 0, s>>>(reinterpret_cast<const uint2*>(st->local + st->lay.xq),
                                                      reinterpret_cast<const float*>(st->local + st->lay.xsc),
                                                      ctx->recv_counts, ctx->e_loc,
                                                      reinterpret_cast<uint4*>(st->local + st->lay.xr), d);
    TCK(cudaGetLastError());
  }
  return FSC_OK;
}

// the combine payload itself is written by the GEMM2 epilogue (fsc_transport_scatter_target);
// this raises the per-source completion flags once that GEMM is done.
int fsc_transport_combine(fsc_ctx* ctx, int, cudaStream_t s) {
  ++g_launches;
  ep_signal_kernel<<<1, 32, 0, s>>>(ctx->peer->peers, ctx->rank, ctx->ep, FLAG_COMB, epoch_ptr(ctx));
  TCK(cudaGetLastError());
  return FSC_OK;
}

// decoupled combine (FSC_COMBINE_STREAM): y = this rank's expert outputs, receive layout
int fsc_transport_combine_push(fsc_ctx* ctx, const uint16_t* y, cudaStream_t s) {
  fsc_peer_state* st = ctx->peer;
  const int d = ctx->cfg.d;
  int blocks = (int)((ctx->max_recv + 7) / 8);
  if (blocks > ctx->comm_ctas) blocks = ctx->comm_ctas;
  if (blocks < 1) blocks = 1;
  ++g_launches;
  ep_combine_kernel<<<blocks, 256, 0, s>>>(st->peers, ctx->rank, ctx->ep, ctx->e_loc, ctx->recv_counts,
                                           reinterpret_cast<const int*>(st->local + st->lay.ret),
                                           reinterpret_cast<const uint4*>(y), st->lay.ys, d, epoch_ptr(ctx),
                                           st->ticket + 2, ctx->a2a_zero_bytes);
  TCK(cudaGetLastError());
  return FSC_OK;
}

// ---- backward (fsc_moe_backward)
void fsc_transport_bwd_ptrs(fsc_ctx* ctx, uint16_t** gr, float** gate, float** dgs) {
  fsc_peer_state* st = ctx->peer;
  *gr = reinterpret_cast<uint16_t*>(st->local + st->lay.gr);
  *gate = reinterpret_cast<float*>(st->local + st->lay.gate);
  *dgs = reinterpret_cast<float*>(st->local + st->lay.dgs);
}

// G rows + gates to the experts' owners (after fsc_transport_dispatch of the same call:
// send_base and the epoch are that call's), then wait for every source's rows
int fsc_transport_dispatch_grad(fsc_ctx* ctx, int T, const float* G, cudaStream_t s) {
  fsc_peer_state* st = ctx->peer;
  const fsc_moe_config& c = ctx->cfg;
  const long R = (long)T * c.top_k;
  int blocks = (int)((R + 7) / 8);
  if (blocks > ctx->comm_ctas) blocks = ctx->comm_ctas;
  if (blocks < 1) blocks = 1;
  g_launches += 2;
  ep_dispatch_grad_kernel<<<blocks, 256, 0, s>>>(st->peers, ctx->rank, ctx->ep, T, c.top_k, c.d, ctx->e_loc,
                                                 epoch_ptr(ctx), st->lay.gr, st->lay.gate, G, ctx->topk_idx, ctx->pos,
                                                 ctx->topk_w, ctx->offsets, st->send_base, st->ticket);
  TCK(cudaGetLastError());
  ep_wait_kernel<<<1, 32, 0, s>>>(st->local, FLAG_GDISP, ctx->ep, epoch_ptr(ctx));
  TCK(cudaGetLastError());
  return FSC_OK;
}

// dX rows (y, receive layout) + gate gradients back to their sources
int fsc_transport_combine_grad(fsc_ctx* ctx, const uint16_t* y, const float* dg_part, int dg_n, int dg_ld,
                               cudaStream_t s) {
  fsc_peer_state* st = ctx->peer;
  int blocks = (int)((ctx->max_recv + 7) / 8);
  if (blocks > ctx->comm_ctas) blocks = ctx->comm_ctas;
  if (blocks < 1) blocks = 1;
  ++g_launches;
  ep_combine_grad_kernel<<<blocks, 256, 0, s>>>(st->peers, ctx->rank, ctx->ep, ctx->e_loc, ctx->recv_counts,
                                                reinterpret_cast<const int*>(st->local + st->lay.ret),
                                                reinterpret_cast<const uint4*>(y), st->lay.ys, st->lay.dgs, dg_part,
                                                dg_n, dg_ld, ctx->cfg.d, epoch_ptr(ctx), st->ticket + 2);
  TCK(cudaGetLastError());
  return FSC_OK;
}

int fsc_transport_combine_grad_wait(fsc_ctx* ctx, cudaStream_t s) {
  ++g_launches;
  ep_wait_kernel<<<1, 32, 0, s>>>(ctx->peer->local, FLAG_GCOMB, ctx->ep, epoch_ptr(ctx));
  TCK(cudaGetLastError());
  return FSC_OK;
}

// device pointers of the exchanged counts matrix [P][E] and the receive map [max_recv]
void fsc_transport_debug(fsc_ctx* ctx, const int** cnt, const int** ret) {
  fsc_peer_state* st = ctx->peer;
  *cnt = reinterpret_cast<const int*>(st->local + st->lay.cnt);
  *ret = reinterpret_cast<const int*>(st->local + st->lay.ret);
}

int fsc_transport_combine_wait(fsc_ctx* ctx, cudaStream_t s) {
  ++g_launches;
  ep_wait_kernel<<<1, 32, 0, s>>>(ctx->peer->local, FLAG_COMB, ctx->ep, epoch_ptr(ctx));
  TCK(cudaGetLastError());
  return FSC_OK;
}

// scatter map + per-rank destination pointers for the fused GEMM2 -> combine epilogue
void fsc_transport_scatter_target(fsc_ctx* ctx, const int** ret, void** peer_out) {
  fsc_peer_state* st = ctx->peer;
  *ret = reinterpret_cast<const int*>(st->local + st->lay.ret);
  for (int p = 0; p < kMaxP; ++p)
    peer_out[p] = (p < ctx->ep && st->peers.base[p]) ? st->peers.base[p] + st->lay.ys : nullptr;
}

// ----------------------------------------------------------------------------- EP all-reduce (host)
static int* epoch_ptr_ch(fsc_ctx* ctx, int ch) {
  return reinterpret_cast<int*>(ctx->peer->local + ctx->peer->lay.flags) + kEpochSlot + ch;
}

float* fsc_transport_ar_partial(fsc_ctx* ctx, int ch) {
  return reinterpret_cast<float*>(ctx->peer->local + ctx->peer->lay.part[ch]);
}

int fsc_transport_ar_start(fsc_ctx* ctx, int T, cudaStream_t s, int ch) {
  fsc_peer_state* st = ctx->peer;
  if (!connected(ctx)) {
    fsc_set_error(ctx, "EP transport not bootstrapped (fsc_bootstrap_export/import)");
    return FSC_ERR_STATE;
  }
  const int P = ctx->ep, d = ctx->cfg.d;
  const long r0 = (long)T * ctx->rank / P, r1 = (long)T * (ctx->rank + 1) / P;
  const int ready = FLAG_AR_READY + 2 * ch, done = FLAG_AR_DONE + 2 * ch;
  g_launches += 2;
  ar_begin_kernel<<<1, 32, 0, s>>>(st->peers, ctx->rank, P, epoch_ptr_ch(ctx, ch), ready);
  TCK(cudaGetLastError());
  long blocks = ((r1 - r0) * (d / 4) + 255) / 256;
  if (blocks > 2 * kNumSMs) blocks = 2 * kNumSMs;
  if (blocks < 1) blocks = 1;
  ar_reduce_kernel<<<(int)blocks, 256, 0, s>>>(st->peers, ctx->rank, P, r0, r1, d, st->lay.part[ch], st->lay.red[ch],
                                                epoch_ptr_ch(ctx, ch), st->ticket + ch, ready, done);
  TCK(cudaGetLastError());
  return FSC_OK;
}

int fsc_transport_ar_finish(fsc_ctx* ctx, int T, const float* resid, float* out, cudaStream_t s, int ch) {
  fsc_peer_state* st = ctx->peer;
  const long n4 = (long)T * ctx->cfg.d / 4;
  long blocks = (n4 + 255) / 256;
  if (blocks > 8 * kNumSMs) blocks = 8 * kNumSMs;
  if (blocks < 1) blocks = 1;
  ++g_launches;
  ar_finish_kernel<<<(int)blocks, 256, 0, s>>>(st->local, ctx->ep, epoch_ptr_ch(ctx, ch), st->lay.red[ch], resid, out,
                                               n4, FLAG_AR_DONE + 2 * ch);
  TCK(cudaGetLastError());
  return FSC_OK;
}

// re-create the symmetric region for a new EP mode (before fsc_bootstrap_export)
int fsc_transport_reinit(fsc_ctx* ctx) {
  fsc_transport_finalize(ctx);
  return fsc_transport_init(ctx);
}
