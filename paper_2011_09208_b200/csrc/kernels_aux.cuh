// HBM-bound / exchange kernels of the split-FC path.
//
//   bridge_gather_kernel   A2  all-gather of X_r, y_r into every rank's gathered buffer
//                              (one-sided NVLink stores + release flags); N > 1 only -- at
//                              N = 1 the GEMMs read the caller's X directly
//   stats_grad_kernel      A4-A6 (N = 1): lse from the class-tile partials, loss, and
//                              G = (P~ e^{m_tile - lse} - onehot) / B_tot in place
//   stats_grad_multi_kernel A4-A6 (N > 1): the same with the per-row (m_r, s_r, z_y,r, top-1)
//                              exchange as LL words over NVLink; rank-order combine ->
//                              identical loss bits on every rank
//   bias_grad_*_kernel     NEXT-4 db_r = column sums of G_r (two fixed-order passes)
//   dx_reduce_kernel       A8  owner side of the dX reduce-scatter: wait for the peers'
//                              pushes (done by the dX GEMM's fused fixup), sum in rank order
//   transpose_f32_kernel       fp32 (kind::tf32) backward only: K-major operand copies
//
// Every kernel begins with griddepcontrol.wait (programmatic dependent launch).
#pragma once
#include <cuda_bf16.h>

#include "ptx_sm100.cuh"

namespace whale {


// debug timestamps (globaltimer ns) for latency experiments; read via whale_debug_timestamps
__device__ unsigned long long g_dbg_ts[32];
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Last-block-done ticket: true in exactly one (the last) block, after all blocks' prior
// global writes are visible at `sys` (cross-GPU) or gpu scope.
template <bool kSys>
__device__ __forceinline__ bool last_block_ticket(unsigned* counter) {
  __shared__ bool is_last;
  if (kSys) __threadfence_system(); else __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x * gridDim.y * gridDim.z - 1);
  }
  __syncthreads();
  if (is_last) {
    if (kSys) __threadfence_system(); else __threadfence();
  }
  return is_last;
}

// Same, over a subset of n participating CTAs (e.g. the chunk-0 CTA of every row).
__device__ __forceinline__ bool last_of_n(unsigned* counter, unsigned n) {
  __shared__ bool is_last_n;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last_n = (atomicAdd(counter, 1u) == n - 1);
  __syncthreads();
  if (is_last_n) __threadfence();
  return is_last_n;
}

// ---------------------------------------------------------------- A2 bridge gather
// Stand-alone form of the bridge all-gather (used when it is not fused into the logits / F1
// prologue, WHALE_FUSED_GATHER=0): block j runs piece j (gather_copy / gather_signal).
// dbg & 16: globaltimer stamps of the first and last block (scripts/gather_ts.py).
__global__ void bridge_gather_kernel(const GatherArgs g, int dbg) {
  const bool ts = (dbg & 16) && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1);
  const int tso = blockIdx.x == 0 ? 0 : 8;
  if (ts) g_dbg_ts[tso + 0] = globaltimer();
  pdl_wait();
  pdl_trigger();
  TraceScope _trace(0);
  if (ts) g_dbg_ts[tso + 1] = globaltimer();
  gather_copy(g, blockIdx.x, threadIdx.x, blockDim.x);
  if (ts) g_dbg_ts[tso + 2] = globaltimer();
  __syncthreads();
  if (ts) g_dbg_ts[tso + 3] = globaltimer();
  if (threadIdx.x == 0) {
    gather_signal(g, 1);
    if (ts) g_dbg_ts[tso + 5] = globaltimer();
  }
}

// ---------------------------------------------------------------- A4 + A5 statistics
struct StatsArgs {
  const float* m_tile;   // [Bt x T]
  const float* s_tile;   // [Bt x T]
  const float* zy_r;     // [Bt]
  const int32_t* y;      // [Bt] labels (global ids) of the gathered batch
  int T, Bt, B, rank, world;
  int row0;              // this rank's first row in the gathered batch (R_r); its rows: [row0, row0 + B)
  long long o_r, C_r, C;
  PeerPtrs peer_stats;   // LL-word slab [world x Bt x 4] on each rank (N > 1)
  const uint32_t* dev_epoch; // step epoch e = *dev_epoch + 1 (device-resident, graph-capturable)
  float4* my_stats;      // this rank's slab (N > 1)
  float* lse;            // [Bt]
  float* row_loss_all;   // [Bt]
  float* loss;           // scalar (device)
  float* row_loss_local; // [B] or NULL
  unsigned* counter;
  int* err;
  int grad_vecs;         // 16-byte vectors of P~ per thread in the fused gradient (chunk size)
  int chunks;            // G-rewrite chunks per row (0 with gscale: the backward forms G itself)
  // G-fused backward (NEXT-4b): instead of rewriting P~ into G, write the per-(row, tile)
  // factor gscale[i, t] = e^{m_tile(i, t) - lse_i} / B_tot; the backward applies it (and the
  // one-hot) to each P~ operand stage in shared memory.  NULL: rewrite P~ -> G in place.
  float* gscale;         // [T x Bt] (tile-major) or NULL
  // NEXT-4 predictions (optional): top-1 class of each local row and its probability
  const int32_t* a_tile; // [Bt x T] argmax class per (row, tile) from the logits epilogue
  const float* mx_tile;  // [Bt x T] true tile maxima when m_tile holds references (F1), else NULL
  int32_t* pred_local;   // [B] or NULL
  float* prob_local;     // [B] or NULL
};

__device__ __forceinline__ int block_min_int128(int v, int* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  const int r = min(min(red[0], red[1]), min(red[2], red[3]));
  __syncthreads();
  return r;
}

// Lowest tile index whose max equals the row max m (the row's top-1 lives there).
__device__ __forceinline__ int argmax_tile(const float* mt, int T, float m, int* red) {
  int tmin = 0x7fffffff;
  for (int t = threadIdx.x; t < T; t += 128)
    if (__ldg(mt + t) == m) tmin = min(tmin, t);
  return block_min_int128(tmin, red);
}

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

// This rank's row statistics over its class tiles: m = row max (true tile maxima), s = sum
// of the tile sums rescaled to m (identical on every CTA of the row: fixed order).
__device__ __forceinline__ void row_stats(const StatsArgs& a, int i, float& m_out, float& s_out, float* red) {
  const float* mt = a.m_tile + static_cast<size_t>(i) * a.T;
  const float* st = a.s_tile + static_cast<size_t>(i) * a.T;
  const float* mx = a.mx_tile ? a.mx_tile + static_cast<size_t>(i) * a.T : mt;  // true maxima
  float mloc[8], sloc[8];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int t = threadIdx.x + k * kStatsThreads;
    mloc[k] = t < a.T ? __ldg(mt + t) : -INFINITY;
    sloc[k] = t < a.T ? __ldg(st + t) : 0.f;
    m = fmaxf(m, t < a.T ? __ldg(mx + t) : -INFINITY);
  }
  for (int t = threadIdx.x + 8 * kStatsThreads; t < a.T; t += kStatsThreads) m = fmaxf(m, __ldg(mx + t));
  m = block_max128(m, red);
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += sloc[k] * __expf(mloc[k] - m);
  for (int t = threadIdx.x + 8 * kStatsThreads; t < a.T; t += kStatsThreads) s += __ldg(st + t) * __expf(__ldg(mt + t) - m);
  m_out = m;
  s_out = block_sum128(s, red);
}

// G-fused mode: gscale[t, i] = e^{m_tile(i, t) - lse_i} / B_tot (the factor the in-place
// rewrite would apply to P~; same expression, so G is bit-identical either way).  Stored
// tile-major [T x B_tot]: the backward's transformer threads (consecutive batch rows) then
// read consecutive words.
__device__ __forceinline__ void write_gscale(const StatsArgs& a, int i, float l, float inv_bt) {
  const float* mt = a.m_tile + static_cast<size_t>(i) * a.T;
  for (int t = threadIdx.x; t < a.T; t += kStatsThreads)
    a.gscale[static_cast<size_t>(t) * a.Bt + i] = __expf(__ldg(mt + t) - l) * inv_bt;
}

// ---------------------------------------------------------------- A4-A6 fused (N = 1)
// With a single shard the statistics need no exchange, so the forward finishes with one
// kernel: grid (1 + rewrite CTAs, B_tot); CTA 0 of a row computes its lse from the class-tile
// partials (T <= a few thousand floats, L2-resident), writes lse / row loss (and gscale in
// the G-fused mode) and takes the mean-loss ticket; the other CTAs recompute the same lse and
// turn chunks of P~ into G = (P~ e^{m_tile - lse} - onehot) / B_tot in place.
constexpr int kGradVecs = 4;  // 16-byte vectors per thread
// Loads are issued kU vectors at a time before any store (the stores may alias later loads as
// far as the compiler knows, so a plain loop serialises load -> store round trips).
constexpr int kRowWriter = 32;  // thread that writes a row's lse / loss (warp 1: no peer stores)

// Mean loss over the global batch: every row's chunk-0 CTA takes a ticket after writing its
// row loss; the last one sums the B_tot row losses in a fixed order (identical bits on every
// rank) and re-arms the counter.
__device__ __forceinline__ void mean_loss_ticket(const StatsArgs& a) {
  // only the row-result writer fences (a GPU-scope fence by a thread that just stored to a
  // peer over NVLink would wait for those remote stores)
  __shared__ bool is_last;
  if (threadIdx.x == kRowWriter) {
    __threadfence();
    is_last = atomicAdd(a.counter, 1u) == static_cast<unsigned>(a.Bt) - 1u;
    if (is_last) __threadfence();
  }
  __syncthreads();
  if (!is_last) return;
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

template <int ES>
__device__ __forceinline__ void grad_rewrite(const StatsArgs& a, void* P, long long ldp, int BN, float inv_bt, int i,
                                             int chunk_id, const float* mt, float l, long long yl) {
  constexpr int V = 16 / ES;
  constexpr int kU = 4;
  const long long chunk = static_cast<long long>(kStatsThreads) * a.grad_vecs * V;
  for (int k0 = 0; k0 < a.grad_vecs; k0 += kU) {
    uint4 raw[kU];
    long long j0s[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      j0s[u] = chunk_id * chunk + (static_cast<long long>(k0 + u) * kStatsThreads + threadIdx.x) * V;
      if (k0 + u < a.grad_vecs && j0s[u] < a.C_r)
        raw[u] = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(P) + (i * ldp + j0s[u]) * ES);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long j0 = j0s[u];
      if (k0 + u >= a.grad_vecs || j0 >= a.C_r) continue;
      const float scale = __expf(__ldg(mt + j0 / BN) - l) * inv_bt;
      if constexpr (ES == 2) {
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw[u]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 f = __bfloat1622float2(h[q]);
          const long long j = j0 + 2 * q;
          f.x = f.x * scale - ((j == yl) ? inv_bt : 0.f);
          f.y = f.y * scale - ((j + 1 == yl) ? inv_bt : 0.f);
          h[q] = __floats2bfloat162_rn(f.x, f.y);
        }
      } else {
        float* f = reinterpret_cast<float*>(&raw[u]);
#pragma unroll
        for (int q = 0; q < 4; ++q) f[q] = f[q] * scale - ((j0 + q == yl) ? inv_bt : 0.f);
      }
      *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(P) + (i * ldp + j0) * ES) = raw[u];
    }
  }
}

template <int ES>
__global__ void __launch_bounds__(kStatsThreads) stats_grad_kernel(const StatsArgs a, void* P, long long ldp,
                                                                   int BN, float inv_bt) {
  __shared__ float red[4];
  pdl_wait();
  pdl_trigger();
  TraceScope _trace(2);
  const int i = blockIdx.y;
  float m, s;
  row_stats(a, i, m, s, red);
  const float l = m + logf(s);
  const long long y = a.y[i];
  const long long yl = y - a.o_r;
  if (blockIdx.x == 0 && threadIdx.x == kRowWriter) {
    if (y < 0 || y >= a.C) atomicOr(a.err, ERR_LABEL);
    const bool own = (y >= a.o_r) && (y < a.o_r + a.C_r);
    const float zy = own ? a.zy_r[i] : 0.f;
    a.lse[i] = l;
    a.row_loss_all[i] = l - zy;
    if (a.row_loss_local) a.row_loss_local[i] = l - zy;
  }
  if (a.pred_local != nullptr && blockIdx.x == 0) {  // top-1: first tile holding the row max
    __shared__ int redi[4];
    const float* mx = a.mx_tile ? a.mx_tile + static_cast<size_t>(i) * a.T : a.m_tile + static_cast<size_t>(i) * a.T;
    const int ts = argmax_tile(mx, a.T, m, redi);
    if (threadIdx.x == 0) {
      a.pred_local[i] = a.a_tile[static_cast<size_t>(i) * a.T + ts];
      if (a.prob_local) a.prob_local[i] = 1.f / s;  // e^{m - lse}
    }
  }
  // ---- CTA 0 of a row: the row's results (+ gscale) and the mean-loss ticket only; CTAs
  //      >= 1 rewrite G chunks blockIdx.x - 1, + (gridDim.x - 1), ... (keeps the ticket's
  //      fence off the rewrite path)
  if (blockIdx.x == 0) {
    if (a.gscale) write_gscale(a, i, l, inv_bt);
    mean_loss_ticket(a);
    return;
  }
  const float* mt = a.m_tile + static_cast<size_t>(i) * a.T;
  for (int c = blockIdx.x - 1; c < a.chunks; c += gridDim.x - 1) grad_rewrite<ES>(a, P, ldp, BN, inv_bt, i, c, mt, l, yl);
}

// ---------------------------------------------------------------- A4-A6 fused (N > 1)
// grid (row CTAs, 1 + rewrite CTAs); a row CTA x serves rows x, x + gridDim.x, ... (one row
// each when gridDim.x = B_tot; fewer CTAs when ranks share a device, so only a few CTAs spin).
// Phase 1 (y = 0): for each of its rows, reduce this rank's class tiles to (m_r, s_r), take
// z_y,r and the top-1 class and push the record {m_r, s_r, z_y,r, top-1} as LL words into
// every peer's slab [rank][row] -- no waiting in this phase, so every record of every rank
// is eventually pushed whatever order CTAs run in.  Phase 2 (all CTAs): for each row, wait
// for the world records, combine them in rank order (identical bits on every rank and
// every CTA); y = 0 writes lse / row loss (and gscale in the G-fused mode) and takes the
// mean-loss ticket (the last row sums the mean in a fixed order); y >= 1 (rewrite mode)
// turns chunks y - 1, y - 1 + (gridDim.y - 1), ... of P~ into G.
template <int ES>
__global__ void __launch_bounds__(kStatsThreads) stats_grad_multi_kernel(const StatsArgs a, void* P, long long ldp,
                                                                         int BN, float inv_bt) {
  __shared__ float red[4];
  __shared__ float4 recs[kMaxRanks];
  __shared__ int redi[4];
  pdl_wait();
  pdl_trigger();
  TraceScope _trace(2);
  const int cta = blockIdx.y;
  const uint32_t e = ld_acquire_gpu(a.dev_epoch) + 1u;
  if (cta == 0) {
    for (int i = blockIdx.x; i < a.Bt; i += gridDim.x) {
      const int tslot = (g_trace_on && threadIdx.x == 0) ? (i == 0 ? 16 : (i == a.Bt - 1 ? 24 : -1)) : -1;
      if (tslot >= 0) g_dbg_ts[tslot] = gtime_ns();
      const long long y = a.y[i];
      float m, s;
      row_stats(a, i, m, s, red);
      if (tslot >= 0) g_dbg_ts[tslot + 1] = gtime_ns();
      int top_class = 0;
      if (a.a_tile != nullptr) {  // predictions requested: this rank's top-1 tile for the row
        const float* mx = a.mx_tile ? a.mx_tile + static_cast<size_t>(i) * a.T : a.m_tile + static_cast<size_t>(i) * a.T;
        const int top = argmax_tile(mx, a.T, m, redi);
        top_class = a.a_tile[static_cast<size_t>(i) * a.T + top];
      }
      if (threadIdx.x < a.world) {  // thread p pushes the record to peer p
        if (threadIdx.x == 0 && (y < 0 || y >= a.C)) atomicOr(a.err, ERR_LABEL);
        const bool own = (y >= a.o_r) && (y < a.o_r + a.C_r);
        const float zy = own ? a.zy_r[i] : 0.f;
        const int p = threadIdx.x;
        // LL-style: four 8-byte {value, epoch} words; each 8-byte store is single-copy atomic,
        // so the reader validates every word by its epoch half -- no fence, no separate flag
        uint2* dst = reinterpret_cast<uint2*>(a.peer_stats.p[p]) + (static_cast<size_t>(a.rank) * a.Bt + i) * 4;
        st_relaxed_sys_v2(dst + 0, __float_as_uint(m), e);
        st_relaxed_sys_v2(dst + 1, __float_as_uint(s), e);
        st_relaxed_sys_v2(dst + 2, __float_as_uint(zy), e);
        st_relaxed_sys_v2(dst + 3, static_cast<uint32_t>(top_class), e);
      }
      if (tslot >= 0) g_dbg_ts[tslot + 2] = gtime_ns();
    }
  }
  for (int i = blockIdx.x; i < a.Bt; i += gridDim.x) {
    const int tslot = (g_trace_on && cta == 0 && threadIdx.x == 0) ? (i == 0 ? 16 : (i == a.Bt - 1 ? 24 : -1)) : -1;
    // ---- the row's records from every rank, combined in rank order
    if (threadIdx.x < a.world) {
      const uint2* src = reinterpret_cast<const uint2*>(a.my_stats) + (static_cast<size_t>(threadIdx.x) * a.Bt + i) * 4;
      const float mv = __uint_as_float(wait_ll(src + 0, e, a.err, ERR_COMM | ERR_AT_STATS));
      const float sv = __uint_as_float(wait_ll(src + 1, e, a.err, ERR_COMM | ERR_AT_STATS));
      const float zv = __uint_as_float(wait_ll(src + 2, e, a.err, ERR_COMM | ERR_AT_STATS));
      const uint32_t cv = wait_ll(src + 3, e, a.err, ERR_COMM | ERR_AT_STATS);
      recs[threadIdx.x] = make_float4(mv, sv, zv, __uint_as_float(cv));
    }
    __syncthreads();
    if (tslot >= 0) g_dbg_ts[tslot + 3] = gtime_ns();
    float mm = -INFINITY;
    int top_rank = 0;
    for (int p = 0; p < a.world; ++p)
      if (recs[p].x > mm) {  // strict: the lowest rank (= lowest class ids) wins ties
        mm = recs[p].x;
        top_rank = p;
      }
    float ss = 0.f, zz = 0.f;
    for (int p = 0; p < a.world; ++p) {
      ss += recs[p].y * __expf(recs[p].x - mm);
      zz += recs[p].z;  // exactly one rank owns the label; the others contribute 0
    }
    const int32_t top_cls = static_cast<int32_t>(__float_as_uint(recs[top_rank].w));
    __syncthreads();  // recs is reused by the next row
    const float l = mm + logf(ss);
    if (cta == 0) {
      if (threadIdx.x == 0 && a.pred_local && i >= a.row0 && i < a.row0 + a.B) {
        a.pred_local[i - a.row0] = top_cls;
        if (a.prob_local) a.prob_local[i - a.row0] = 1.f / ss;  // e^{m - lse}
      }
      if (threadIdx.x == kRowWriter) {  // not a thread that pushed to peers
        a.lse[i] = l;
        a.row_loss_all[i] = l - zz;
        if (a.row_loss_local && i >= a.row0 && i < a.row0 + a.B) a.row_loss_local[i - a.row0] = l - zz;
      }
      // gscale, then the mean-loss ticket (its fence covers only this CTA's row results)
      if (a.gscale) write_gscale(a, i, l, inv_bt);
      mean_loss_ticket(a);
      if (tslot >= 0) g_dbg_ts[tslot + 4] = gtime_ns();
    } else {
      const float* mt = a.m_tile + static_cast<size_t>(i) * a.T;
      const long long yl = static_cast<long long>(a.y[i]) - a.o_r;
      for (int c = cta - 1; c < a.chunks; c += gridDim.y - 1) grad_rewrite<ES>(a, P, ldp, BN, inv_bt, i, c, mt, l, yl);
    }
  }
}

// ---------------------------------------------------------------- A8 dX reduce-scatter (owner)
// The dX GEMM's fixup pushed every peer's reduced rows into recv[p][B_r x D] (slabs of
// B_max rows) and raised flag[RS][p]; wait for all, then dX_r = sum_p recv[p] in rank order.
// NVLS (mc_mine != NULL): every rank left its rows for this owner in slot `rank` of its OWN
// slab; one multimem.ld_reduce per 16 bytes returns their sum, formed in the NVSwitch.
template <int ES>
__global__ void __launch_bounds__(256) dx_reduce_kernel(const float4* __restrict__ recv, int B, int B_slab, int D,
                                                        int world,
                                                        const uint32_t* my_flags, const uint32_t* dev_epoch,
                                                        void* dx_local, int* err, const float4* mc_mine) {
  pdl_wait();
  pdl_trigger();
  TraceScope _trace(6);
  // the backward GEMM already published this step's epoch (end-of-step ticket)
  const uint32_t e = ld_acquire_gpu(dev_epoch);
  if (threadIdx.x < world) wait_flag_geq(my_flags + threadIdx.x, e, err, ERR_COMM | ERR_AT_RS);
  __syncthreads();
  __threadfence_system();
  const int64_t total = static_cast<int64_t>(B) * (D / 4);
  const int64_t slab = static_cast<int64_t>(B_slab) * (D / 4);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 acc;
    if (mc_mine != nullptr) {
      acc = multimem_ld_reduce_add_v4f32(mc_mine + e);
    } else {
      acc = __ldcg(recv + e);
      for (int p = 1; p < world; ++p) {
        const float4 v = __ldcg(recv + p * slab + e);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
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

// ---------------------------------------------------------------- NEXT-4 bias gradient
// db_r[j] = sum_i G_r[i, j] (the FC bias gradient; G already includes 1/B_tot).  In the
// G-fused mode the buffer still holds P~ and G[i, j] = P~[i, j] gscale[i, j / BN] - [j == y_i
// - o_r] / B_tot is formed here (the same arithmetic as the in-place rewrite).
// Pass 1: grid (column vectors, 128-row chunks) -> part[chunk][j]; pass 2 sums the chunks
// in order.  Both passes use fixed summation orders (deterministic).
constexpr int kDbRows = 128;
struct DbFused {
  const float* gscale;   // [T x Bt] or NULL (buffer holds G)
  const int32_t* y;      // [Bt]
  long long o_r;
  int T, BN;
  float inv_bt;
};
template <int ES>
__global__ void __launch_bounds__(128) bias_grad_part_kernel(const void* G, long long ldp, int Bt, long long C_r,
                                                             float* part /*[chunks x C_r]*/, const DbFused fz) {
  constexpr int V = 16 / ES;
  pdl_wait();
  pdl_trigger();
  const long long j0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * V;
  if (j0 >= C_r) return;
  const int r0 = blockIdx.y * kDbRows, r1 = min(Bt, r0 + kDbRows);
  float acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
  const int tile = static_cast<int>(j0 / (fz.BN > 0 ? fz.BN : 1));
#pragma unroll 4
  for (int r = r0; r < r1; ++r) {
    float g[V];
    if constexpr (ES == 2) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(G) + r * ldp + j0));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h[k]);
        g[2 * k] = f.x;
        g[2 * k + 1] = f.y;
      }
    } else {
      const float4 f = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(G) + r * ldp + j0));
      g[0] = f.x; g[1] = f.y; g[2] = f.z; g[3] = f.w;
    }
    if (fz.gscale != nullptr) {  // P~ -> G, rounded to the operand type like the rewrite
      const float sc = __ldg(fz.gscale + static_cast<size_t>(tile) * Bt + r);
      const long long yl = static_cast<long long>(__ldg(fz.y + r)) - fz.o_r;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float v = g[k] * sc - ((j0 + k == yl) ? fz.inv_bt : 0.f);
        g[k] = ES == 2 ? __bfloat162float(__float2bfloat16_rn(v)) : v;
      }
    }
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] += g[k];
  }
  float* o = part + static_cast<size_t>(blockIdx.y) * C_r + j0;
#pragma unroll
  for (int k = 0; k < V; ++k)
    if (j0 + k < C_r) o[k] = acc[k];
}
__global__ void __launch_bounds__(256) bias_grad_sum_kernel(const float* part, int chunks, long long C_r, float* db,
                                                            const float* grad_scale) {
  pdl_wait();
  pdl_trigger();
  const float gs = grad_scale ? __ldg(grad_scale) : 1.f;
  for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < C_r;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < chunks; ++c) s += part[c * C_r + j];
    db[j] = grad_scale ? s * gs : s;
  }
}

// Forward-only steps (a forward not followed by a backward) end here: publish the epoch.
__global__ void epoch_bump_kernel(uint32_t* dev_epoch) {
  pdl_wait();
  pdl_trigger();
  TraceScope _trace(9);
  if (threadIdx.x == 0) atomicAdd(dev_epoch, 1u);
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
  TraceScope _trace(7);
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (r0 + ty < R && c0 + tx < Cc) t[ty][tx] = src[(r0 + ty) * src_ld + c0 + tx];
  __syncthreads();
  if (c0 + ty < Cc && r0 + tx < R) dst[(c0 + ty) * dst_ld + r0 + tx] = t[tx][ty];
}

}  // namespace whale
