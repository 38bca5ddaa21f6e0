// HBM-bound / exchange kernels of the split-FC path.
//
//   bridge_gather_kernel   A2  all-gather of X_r, y_r into every rank's gathered buffer
//                              (one-sided NVLink stores + release flags); N > 1 only -- at
//                              N = 1 the GEMMs read the caller's X directly
//   stats_rows_kernel      A4+A5  one CTA per row: (m_r, s_r, z_y,r) over the class tiles;
//                              N > 1: push the float4 to every peer; the last CTA combines
//                              in rank order (lse, per-row loss) and sums the mean loss in a
//                              fixed order -> identical bits on every rank
//   softmax_grad_kernel    A6  G = (P~ e^{m_tile - lse} - onehot) / B_tot, in place
//   dx_reduce_kernel       A8  owner side of the dX reduce-scatter: wait for the peers'
//                              pushes (done by the dX GEMM's fused fixup), sum in rank order
//   transpose_f32_kernel       fp32 (kind::tf32) backward only: K-major operand copies
//
// Every kernel begins with griddepcontrol.wait (programmatic dependent launch).
#pragma once
#include <cuda_bf16.h>

#include "ptx_sm100.cuh"

namespace whale {

enum ErrBits : int { ERR_LABEL = 1, ERR_COMM = 8 };

// Last-block-done ticket: true in exactly one (the last) block, after all blocks' prior
// global writes are visible at `sys` (cross-GPU) or gpu scope.
template <bool kSys>
__device__ __forceinline__ bool last_block_ticket(unsigned* counter) {
  __shared__ bool is_last;
  if (kSys) __threadfence_system(); else __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) {
    if (kSys) __threadfence_system(); else __threadfence();
  }
  return is_last;
}

// ---------------------------------------------------------------- A2 bridge gather
// Rank r writes its B rows at row offset r*B of every rank's gathered X buffer, and its
// labels likewise; the last block then raises flag[GATHER][r] = epoch on every peer.
__global__ void bridge_gather_kernel(const uint4* __restrict__ x_local, const int32_t* __restrict__ y_local,
                                     int64_t x_vecs /*B*row_bytes/16*/, int B, int rank, int world,
                                     PeerPtrs dst_x /*slab base on each rank*/, PeerPtrs dst_y,
                                     PeerFlags flags /*&flag[GATHER][rank] on each rank*/, uint32_t epoch,
                                     unsigned* counter) {
  pdl_wait();
  pdl_trigger();
  const int64_t off_vec = static_cast<int64_t>(rank) * x_vecs;
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < x_vecs;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 val = __ldg(x_local + v);
#pragma unroll
    for (int p = 0; p < kMaxRanks; ++p)
      if (p < world) reinterpret_cast<uint4*>(dst_x.p[p])[off_vec + v] = val;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B; i += gridDim.x * blockDim.x) {
    const int32_t y = y_local[i];
#pragma unroll
    for (int p = 0; p < kMaxRanks; ++p)
      if (p < world) reinterpret_cast<int32_t*>(dst_y.p[p])[rank * B + i] = y;
  }
  if (last_block_ticket<true>(counter)) {
    if (threadIdx.x < world) st_release_sys(flags.p[threadIdx.x], epoch);
    __syncthreads();
    if (threadIdx.x == 0) *counter = 0;
  }
}

// ---------------------------------------------------------------- A4 + A5 statistics
struct StatsArgs {
  const float* m_tile;   // [Bt x T]
  const float* s_tile;   // [Bt x T]
  const float* zy_r;     // [Bt]
  const int32_t* y;      // [Bt] labels (global ids) of the gathered batch
  int T, Bt, B, rank, world;
  long long o_r, C_r, C;
  PeerPtrs peer_stats;   // float4 [world x Bt] slab on each rank (this parity)
  PeerFlags peer_flags;  // &flag[STATS][rank] on each rank
  const uint32_t* my_flags;  // flag[STATS][0..world) on this rank
  uint32_t epoch;
  float4* my_stats;      // this rank's slab (N > 1)
  float* lse;            // [Bt]
  float* row_loss_all;   // [Bt]
  float* loss;           // scalar (device)
  float* row_loss_local; // [B] or NULL
  unsigned* counter;
  int* err;
};

constexpr int kStatsThreads = 128;

__device__ __forceinline__ float block_max128(float v, float* red) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  const float r = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  return r;
}
__device__ __forceinline__ float block_sum128(float v, float* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  const float r = (red[0] + red[1]) + (red[2] + red[3]);
  __syncthreads();
  return r;
}

// One CTA (128 threads) per row: all of the row's tile partials are loaded at once
// (latency-bound otherwise), then s = sum_t s_t e^{m_t - m} (online-softmax combine).
template <bool kMulti>
__global__ void __launch_bounds__(kStatsThreads) stats_rows_kernel(const StatsArgs a) {
  __shared__ float red[4];
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x;
  const float* mt = a.m_tile + static_cast<size_t>(i) * a.T;
  const float* st = a.s_tile + static_cast<size_t>(i) * a.T;
  float mloc[8], sloc[8];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int t = threadIdx.x + k * kStatsThreads;
    mloc[k] = t < a.T ? mt[t] : -INFINITY;
    sloc[k] = t < a.T ? st[t] : 0.f;
    m = fmaxf(m, mloc[k]);
  }
  for (int t = threadIdx.x + 8 * kStatsThreads; t < a.T; t += kStatsThreads) m = fmaxf(m, mt[t]);
  m = block_max128(m, red);
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += sloc[k] * __expf(mloc[k] - m);
  for (int t = threadIdx.x + 8 * kStatsThreads; t < a.T; t += kStatsThreads) s += st[t] * __expf(mt[t] - m);
  s = block_sum128(s, red);
  if (threadIdx.x == 0) {
    const long long y = a.y[i];
    if (y < 0 || y >= a.C) atomicOr(a.err, ERR_LABEL);
    const bool own = (y >= a.o_r) && (y < a.o_r + a.C_r);
    const float zy = own ? a.zy_r[i] : 0.f;
    if constexpr (!kMulti) {
      const float l = m + logf(s);
      a.lse[i] = l;
      a.row_loss_all[i] = l - zy;
      if (a.row_loss_local) a.row_loss_local[i] = l - zy;
    } else {
      const float4 rec = make_float4(m, s, zy, 0.f);
      for (int p = 0; p < a.world; ++p)
        reinterpret_cast<float4*>(a.peer_stats.p[p])[static_cast<size_t>(a.rank) * a.Bt + i] = rec;
    }
  }
  if (!last_block_ticket<kMulti>(a.counter)) return;
  // ---- last CTA: (N > 1) exchange + rank-ordered combine; fixed-order mean loss ----
  if constexpr (kMulti) {
    if (threadIdx.x < a.world) st_release_sys(a.peer_flags.p[threadIdx.x], a.epoch);
    if (threadIdx.x < a.world) wait_flag_geq(a.my_flags + threadIdx.x, a.epoch, a.err, ERR_COMM);
    __syncthreads();
    __threadfence_system();
    for (int r = threadIdx.x; r < a.Bt; r += kStatsThreads) {
      float mm = -INFINITY;
      for (int p = 0; p < a.world; ++p) mm = fmaxf(mm, a.my_stats[static_cast<size_t>(p) * a.Bt + r].x);
      float ss = 0.f, zz = 0.f;
      for (int p = 0; p < a.world; ++p) {
        const float4 rec = a.my_stats[static_cast<size_t>(p) * a.Bt + r];
        ss += rec.y * __expf(rec.x - mm);
        zz += rec.z;  // exactly one rank owns the label; the others contribute 0
      }
      const float l = mm + logf(ss);
      a.lse[r] = l;
      a.row_loss_all[r] = l - zz;
      if (a.row_loss_local && r >= a.rank * a.B && r < (a.rank + 1) * a.B) a.row_loss_local[r - a.rank * a.B] = l - zz;
    }
    __syncthreads();
  }
  double acc = 0.0;
  for (int r = threadIdx.x; r < a.Bt; r += kStatsThreads) acc += static_cast<double>(__ldcg(a.row_loss_all + r));
  __shared__ double part[4];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.loss = static_cast<float>(((part[0] + part[1]) + (part[2] + part[3])) / a.Bt);
    *a.counter = 0;
  }
}

// ---------------------------------------------------------------- A6 gradient
// G[i, j] = (P~[i, j] * exp(m_tile[i, j / BN] - lse_i) - [j == y_i - o_r]) / B_tot, in place.
// One thread per 8 (bf16) / 4 (fp32) consecutive classes of one row (16-byte vectors).
template <int ES>
__global__ void __launch_bounds__(256) softmax_grad_kernel(void* P, long long ldp, int Bt, long long C_r, int BN,
                                                           int T, const float* __restrict__ m_tile,
                                                           const float* __restrict__ lse,
                                                           const int32_t* __restrict__ y, long long o_r,
                                                           float inv_bt) {
  constexpr int V = 16 / ES;
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.y;
  const long long j0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * V;
  if (j0 >= C_r) return;
  const float l = lse[i];
  const long long yl = static_cast<long long>(y[i]) - o_r;
  const float* mt = m_tile + static_cast<size_t>(i) * T;
  // BN is a multiple of V, so the V classes share one tile scale
  const float scale = __expf(mt[j0 / BN] - l) * inv_bt;
  if constexpr (ES == 2) {
    uint4* p = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(P) + i * ldp + j0);
    uint4 raw = *p;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = __bfloat1622float2(h[k]);
      const long long j = j0 + 2 * k;
      f.x = f.x * scale - ((j == yl) ? inv_bt : 0.f);
      f.y = f.y * scale - ((j + 1 == yl) ? inv_bt : 0.f);
      h[k] = __floats2bfloat162_rn(f.x, f.y);
    }
    *p = raw;
  } else {
    float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(P) + i * ldp + j0);
    float4 f = *p;
    f.x = f.x * scale - ((j0 == yl) ? inv_bt : 0.f);
    f.y = f.y * scale - ((j0 + 1 == yl) ? inv_bt : 0.f);
    f.z = f.z * scale - ((j0 + 2 == yl) ? inv_bt : 0.f);
    f.w = f.w * scale - ((j0 + 3 == yl) ? inv_bt : 0.f);
    *p = f;
  }
}

// ---------------------------------------------------------------- A4-A6 fused (N = 1)
// With a single shard the statistics need no exchange, so the forward finishes with one
// kernel: grid (chunks, B_tot); every CTA recomputes its row's lse from the class-tile
// partials (T <= a few thousand floats, L2-resident), turns its chunk of P~ into
// G = (P~ e^{m_tile - lse} - onehot) / B_tot in place, chunk 0 writes lse / row loss, and
// the last CTA sums the mean loss in a fixed order.
constexpr int kGradVecs = 4;  // 16-byte vectors per thread
template <int ES>
__global__ void __launch_bounds__(kStatsThreads) stats_grad_kernel(const StatsArgs a, void* P, long long ldp,
                                                                   int BN, float inv_bt) {
  constexpr int V = 16 / ES;
  __shared__ float red[4];
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.y;
  const float* mt = a.m_tile + static_cast<size_t>(i) * a.T;
  const float* st = a.s_tile + static_cast<size_t>(i) * a.T;
  float mloc[8], sloc[8];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int t = threadIdx.x + k * kStatsThreads;
    mloc[k] = t < a.T ? __ldg(mt + t) : -INFINITY;
    sloc[k] = t < a.T ? __ldg(st + t) : 0.f;
    m = fmaxf(m, mloc[k]);
  }
  for (int t = threadIdx.x + 8 * kStatsThreads; t < a.T; t += kStatsThreads) m = fmaxf(m, __ldg(mt + t));
  m = block_max128(m, red);
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += sloc[k] * __expf(mloc[k] - m);
  for (int t = threadIdx.x + 8 * kStatsThreads; t < a.T; t += kStatsThreads) s += __ldg(st + t) * __expf(__ldg(mt + t) - m);
  s = block_sum128(s, red);
  const float l = m + logf(s);
  const long long y = a.y[i];
  const long long yl = y - a.o_r;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (y < 0 || y >= a.C) atomicOr(a.err, ERR_LABEL);
    const bool own = (y >= a.o_r) && (y < a.o_r + a.C_r);
    const float zy = own ? a.zy_r[i] : 0.f;
    a.lse[i] = l;
    a.row_loss_all[i] = l - zy;
    if (a.row_loss_local) a.row_loss_local[i] = l - zy;
  }
  // ---- G for this CTA's chunk of the row
  const long long chunk = static_cast<long long>(kStatsThreads) * kGradVecs * V;
#pragma unroll
  for (int k = 0; k < kGradVecs; ++k) {
    const long long j0 = blockIdx.x * chunk + (static_cast<long long>(k) * kStatsThreads + threadIdx.x) * V;
    if (j0 >= a.C_r) break;
    const float scale = __expf(__ldg(mt + j0 / BN) - l) * inv_bt;
    if constexpr (ES == 2) {
      uint4* p = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(P) + i * ldp + j0);
      uint4 raw = *p;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 f = __bfloat1622float2(h[q]);
        const long long j = j0 + 2 * q;
        f.x = f.x * scale - ((j == yl) ? inv_bt : 0.f);
        f.y = f.y * scale - ((j + 1 == yl) ? inv_bt : 0.f);
        h[q] = __floats2bfloat162_rn(f.x, f.y);
      }
      *p = raw;
    } else {
      float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(P) + i * ldp + j0);
      float4 f = *p;
      f.x = f.x * scale - ((j0 == yl) ? inv_bt : 0.f);
      f.y = f.y * scale - ((j0 + 1 == yl) ? inv_bt : 0.f);
      f.z = f.z * scale - ((j0 + 2 == yl) ? inv_bt : 0.f);
      f.w = f.w * scale - ((j0 + 3 == yl) ? inv_bt : 0.f);
      *p = f;
    }
  }
  // ---- mean loss: last CTA, fixed order
  if (!last_block_ticket<false>(a.counter)) return;
  double acc = 0.0;
  for (int r = threadIdx.x; r < a.Bt; r += kStatsThreads) acc += static_cast<double>(__ldcg(a.row_loss_all + r));
  __shared__ double part[4];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.loss = static_cast<float>(((part[0] + part[1]) + (part[2] + part[3])) / a.Bt);
    *a.counter = 0;
  }
}

// ---------------------------------------------------------------- A8 dX reduce-scatter (owner)
// The dX GEMM's fixup pushed every peer's reduced rows into recv[p][B x D] and raised
// flag[RS][p]; wait for all, then dX_r = sum_p recv[p] in rank order.
template <int ES>
__global__ void __launch_bounds__(256) dx_reduce_kernel(const float4* __restrict__ recv, int B, int D, int world,
                                                        const uint32_t* my_flags, uint32_t epoch, void* dx_local,
                                                        int* err) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x < world) wait_flag_geq(my_flags + threadIdx.x, epoch, err, ERR_COMM);
  __syncthreads();
  __threadfence_system();
  const int64_t total = static_cast<int64_t>(B) * (D / 4);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 acc = __ldcg(recv + e);
    for (int p = 1; p < world; ++p) {
      const float4 v = __ldcg(recv + p * total + e);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if constexpr (ES == 2) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&lo);
      o.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(dx_local)[e] = o;
    } else {
      reinterpret_cast<float4*>(dx_local)[e] = acc;
    }
  }
}

// ---------------------------------------------------------------- fp32 operand transposes
// kind::tf32 takes only K-major smem operands in the plain 128B swizzle, so the fp32
// (tiny) backward feeds dW / dX from transposed copies: dst[c, r] = src[r, c].
__global__ void __launch_bounds__(1024) transpose_f32_kernel(const float* __restrict__ src, long long src_ld,
                                                             float* __restrict__ dst, long long dst_ld, int R,
                                                             int Cc) {
  __shared__ float t[32][33];
  pdl_wait();
  pdl_trigger();
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (r0 + ty < R && c0 + tx < Cc) t[ty][tx] = src[(r0 + ty) * src_ld + c0 + tx];
  __syncthreads();
  if (c0 + ty < Cc && r0 + tx < R) dst[(c0 + ty) * dst_ld + r0 + tx] = t[tx][ty];
}

}  // namespace whale
