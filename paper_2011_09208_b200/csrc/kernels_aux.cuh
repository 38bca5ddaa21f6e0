// HBM-bound / exchange kernels of the split-FC path.
//
//   bridge_gather_kernel   A2  all-gather of X_r, y_r into every rank's gathered buffer
//                              (one-sided NVLink stores + release flags; N=1: local copy)
//   stats_combine_kernel   A4+A5  per-row (m_r, s_r, z_y,r) over class tiles, exchange of
//                              B_tot float4 with every peer, rank-ordered combine, lse and
//                              the mean loss (deterministic: identical bits on every rank)
//   softmax_grad_kernel    A6  G = (P~ e^{m_tile - lse} - onehot) / B_tot, in place
//   dx_push_kernel         A8  sum split-K partials of dX and push each owner's rows to it
//   dx_reduce_kernel       A8  owner: wait, sum the N pushed slabs in rank order -> dX_r
#pragma once
#include <cuda_bf16.h>

#include "ptx_sm100.cuh"

namespace whale {

constexpr int kMaxRanks = 8;

enum ErrBits : int { ERR_LABEL = 1, ERR_COMM = 8 };

struct PeerPtrs {
  void* p[kMaxRanks];
};
struct PeerFlags {
  uint32_t* p[kMaxRanks];
};

// Last-block-done ticket: returns true in exactly one (the last) block, after all blocks'
// prior global writes are visible at system scope.
__device__ __forceinline__ bool last_block_ticket(unsigned* counter) {
  __shared__ bool is_last;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) __threadfence_system();
  return is_last;
}

// ---------------------------------------------------------------- A2 bridge gather
// Rank r writes its B rows (row bytes = row_bytes) at row offset r*B of every rank's
// gathered X buffer, and its labels likewise; the last block then raises
// flag[GATHER][r] = epoch on every peer (st.release.sys).
__global__ void bridge_gather_kernel(const uint4* __restrict__ x_local, const int32_t* __restrict__ y_local,
                                     int64_t x_vecs /*B*row_bytes/16*/, int B, int rank, int world,
                                     PeerPtrs dst_x /*slab base on each rank*/, PeerPtrs dst_y,
                                     PeerFlags flags /*&flag[GATHER][rank] on each rank*/, uint32_t epoch,
                                     unsigned* counter) {
  const int64_t off_vec = static_cast<int64_t>(rank) * x_vecs;
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < x_vecs;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 val = __ldg(x_local + v);
    for (int p = 0; p < world; ++p) reinterpret_cast<uint4*>(dst_x.p[p])[off_vec + v] = val;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B; i += gridDim.x * blockDim.x) {
    const int32_t y = y_local[i];
    for (int p = 0; p < world; ++p) reinterpret_cast<int32_t*>(dst_y.p[p])[rank * B + i] = y;
  }
  if (world == 1) return;
  if (last_block_ticket(counter)) {
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
  const int32_t* y;      // [Bt] gathered labels (global ids)
  int T, Bt, B, rank, world;
  long long o_r, C_r, C;
  PeerPtrs peer_stats;   // float4 [world x Bt] slab on each rank (this parity)
  PeerFlags peer_flags;  // &flag[STATS][rank] on each rank
  const uint32_t* my_flags;  // flag[STATS][0..world) on this rank
  uint32_t epoch;
  float4* my_stats;      // this rank's slab (== peer_stats.p[rank])
  float* lse;            // [Bt]
  float* row_loss_all;   // [Bt]
  float* loss;           // scalar (device)
  float* row_loss_local; // [B] or NULL
  unsigned* counter;
  int* err;
};

// One warp per row: reduce the row's class-tile partials (online-softmax rule
// s = sum_t s_t e^{m_t - m}), then the last block combines across ranks.
__global__ void __launch_bounds__(256) stats_combine_kernel(const StatsArgs a) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < a.Bt; i += gridDim.x * wpb) {
    const float* mt = a.m_tile + static_cast<size_t>(i) * a.T;
    const float* st = a.s_tile + static_cast<size_t>(i) * a.T;
    float m = -INFINITY;
    for (int t = lane; t < a.T; t += 32) m = fmaxf(m, mt[t]);
    m = warp_max(m);
    float s = 0.f;
    for (int t = lane; t < a.T; t += 32) s += st[t] * __expf(mt[t] - m);
    s = warp_sum(s);
    if (lane == 0) {
      const long long y = a.y[i];
      if (y < 0 || y >= a.C) atomicOr(a.err, ERR_LABEL);
      const bool own = (y >= a.o_r) && (y < a.o_r + a.C_r);
      const float zy = own ? a.zy_r[i] : 0.f;
      const float4 rec = make_float4(m, s, zy, 0.f);
      if (a.world == 1) {
        a.my_stats[i] = rec;
      } else {
        for (int p = 0; p < a.world; ++p)
          reinterpret_cast<float4*>(a.peer_stats.p[p])[static_cast<size_t>(a.rank) * a.Bt + i] = rec;
      }
    }
  }
  if (!last_block_ticket(a.counter)) return;
  // ---- last block: exchange, combine in rank order, loss ----
  if (a.world > 1) {
    if (threadIdx.x < a.world) st_release_sys(a.peer_flags.p[threadIdx.x], a.epoch);
    if (threadIdx.x < a.world) wait_flag_geq(a.my_flags + threadIdx.x, a.epoch, a.err, ERR_COMM);
    __syncthreads();
    __threadfence_system();
  }
  double acc = 0.0;
  for (int i = threadIdx.x; i < a.Bt; i += blockDim.x) {
    float m = -INFINITY;
    for (int p = 0; p < a.world; ++p) m = fmaxf(m, a.my_stats[static_cast<size_t>(p) * a.Bt + i].x);
    float s = 0.f, zy = 0.f;
    for (int p = 0; p < a.world; ++p) {
      const float4 r = a.my_stats[static_cast<size_t>(p) * a.Bt + i];
      s += r.y * __expf(r.x - m);
      zy += r.z;
    }
    const float l = m + logf(s);
    a.lse[i] = l;
    const float rl = l - zy;
    a.row_loss_all[i] = rl;
    if (a.row_loss_local && i >= a.rank * a.B && i < (a.rank + 1) * a.B) a.row_loss_local[i - a.rank * a.B] = rl;
    acc += static_cast<double>(rl);
  }
  // fixed-order block reduction (warp xor tree, then warp 0 over warp partials)
  __shared__ double part[32];
  acc = warp_sum(acc);
  if (lane == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = (threadIdx.x < wpb) ? part[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      *a.loss = static_cast<float>(v / a.Bt);
      *a.counter = 0;
    }
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

// ---------------------------------------------------------------- A8 dX reduce-scatter
// Push: v = sum_s part[s][row, :] (split-K partials, fixed order) -> owner's slab
//       recv[owner][rank][row - owner*B, :] (NVLink store); last block raises flag[RS][rank].
// N=1: writes the final dX (converted to the operand dtype) directly.
template <int ES>
__global__ void __launch_bounds__(256) dx_push_kernel(const float4* __restrict__ part, int S, int Bt, int B,
                                                      int D, int rank, int world, PeerPtrs recv /*slab base*/,
                                                      PeerFlags flags, uint32_t epoch, void* dx_local,
                                                      unsigned* counter) {
  const int dv = D / 4;
  const int64_t total = static_cast<int64_t>(Bt) * dv;
  const int64_t split_stride = total;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 acc = part[e];
    for (int s = 1; s < S; ++s) {
      const float4 v = part[s * split_stride + e];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (world == 1) {
      if constexpr (ES == 2) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
        uint2 o;
        o.x = *reinterpret_cast<uint32_t*>(&lo);
        o.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(dx_local)[e] = o;
      } else {
        reinterpret_cast<float4*>(dx_local)[e] = acc;
      }
    } else {
      const int row = static_cast<int>(e / dv);
      const int owner = row / B;
      const int64_t local = e - static_cast<int64_t>(owner) * B * dv;  // index inside owner's B rows
      reinterpret_cast<float4*>(recv.p[owner])[static_cast<int64_t>(rank) * B * dv + local] = acc;
    }
  }
  if (world == 1) return;
  if (last_block_ticket(counter)) {
    if (threadIdx.x < world) st_release_sys(flags.p[threadIdx.x], epoch);
    __syncthreads();
    if (threadIdx.x == 0) *counter = 0;
  }
}

// Owner side: wait for every peer's slab, then dX_r = sum_p recv[p] in rank order.
template <int ES>
__global__ void __launch_bounds__(256) dx_reduce_kernel(const float4* __restrict__ recv, int B, int D, int world,
                                                        const uint32_t* my_flags, uint32_t epoch, void* dx_local,
                                                        int* err) {
  if (threadIdx.x < world) wait_flag_geq(my_flags + threadIdx.x, epoch, err, ERR_COMM);
  __syncthreads();
  __threadfence_system();
  const int64_t total = static_cast<int64_t>(B) * (D / 4);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 acc = recv[e];
    for (int p = 1; p < world; ++p) {
      const float4 v = recv[p * total + e];
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
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (r0 + ty < R && c0 + tx < Cc) t[ty][tx] = src[(r0 + ty) * src_ld + c0 + tx];
  __syncthreads();
  if (c0 + ty < Cc && r0 + tx < R) dst[(c0 + ty) * dst_ld + r0 + tx] = t[tx][ty];
}

}  // namespace whale
