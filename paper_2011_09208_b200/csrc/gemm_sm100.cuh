// Persistent, warp-specialised tcgen05 GEMM for sm_100a with the split-FC epilogues.
//
//   D[M x N] = A[M x K] * B[N x K]^T    (bf16 operands -> kind::f16, or fp32 -> kind::tf32;
//                                         fp32 accumulator in TMEM)
//
// A and B are each either K-major (K contiguous) or MN-major (M/N contiguous); both are
// fed by TMA into 128B-swizzled shared memory and consumed by tcgen05.mma issued from one
// thread.  One CTA per SM, grid = min(#tiles, #SMs), static round-robin tile order with
// M fastest (CTAs running concurrently share the same B tile -> it is read from HBM once).
//
//   warp 0      TMA producer (one lane)       smem ring: full/empty mbarriers
//   warp 1      MMA issuer (one lane)         TMEM ring: 2 accumulators x 256 columns
//   warp 2      TMEM allocator
//   warps 4..7  epilogue (TMEM lane quadrant = warp % 4, one thread per output row)
//
// Epilogues:
//   EPI_FWD_STATS  split-FC forward (north star (b)): the logits tile
//                  Z = X W_r^T never leaves the SM as fp32.  Per row and class tile the
//                  epilogue writes m_tile = max_j z, s_tile = sum_j exp(z - m_tile),
//                  P~ = exp(z - m_tile) (bf16 / fp32, TMA store) and captures the label
//                  logit z_y when the label falls in this tile.
//   EPI_STORE_F32  fp32 tile store through swizzled smem stages + TMA (3-D map
//                  {N, M, split}); used for dW (A7) and the split-K dX partials (A8).
//                  With fix_mode != 0 (dX) the split-K partials are reduced in a fixed
//                  split order inside this kernel (all CTAs co-resident -> each reduces
//                  1/S of its tile after a counter barrier) and the result is either
//                  written as the final dX (N = 1) or pushed over NVLink into the owner
//                  rank's receive slab (N > 1, fused GEMM -> reduce-scatter).
//
// Every kernel is PDL-ready (griddepcontrol.wait after its prologue -- barrier init, TMEM
// alloc, descriptor prefetch); the host launches with programmatic dependent launch only on
// request (WHALE_PDL=1: measured slower in round 2).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "ptx_sm100.cuh"

namespace whale {

enum EpiKind : int { EPI_FWD_STATS = 0, EPI_STORE_F32 = 1 };
enum FixMode : int { FIX_NONE = 0, FIX_LOCAL = 1, FIX_PUSH = 2 };

constexpr int kBM = 128;               // MMA M (rows of A per tile)
constexpr int kRowBytes = 128;         // one SWIZZLE_128B row: K elements per stage = 128 / ES
constexpr int kMaxBN = 256;            // accumulator columns per TMEM buffer
constexpr int kGemmThreads = 256;      // 8 warps
constexpr int kStatsGemmThreads = 384; // EPI_FWD_STATS: 12 warps (warps 4..11 = 2 epilogue groups)
constexpr int kStageABytes = kBM * kRowBytes;   // 16 KB
constexpr int kEpiBufBytes = 4096;     // per epilogue warp per buffer: 32 rows x 128 B
constexpr int kTmemCols = 512;

struct GemmArgs {
  int M, N;                 // valid output rows / cols
  int BN;                   // N tile (multiple of 128/ES when B is MN-major or EPI_FWD_STATS)
  int m_blocks, n_blocks, splits;
  int num_kb, kb_per_split; // k-blocks of 128/ES elements
  int num_tiles;
  int stages;
  int stage_bytes;
  int epi_bufs;             // smem store buffers per epilogue warp (2, 4 or 8)
  int bk;                   // K elements per stage: 128/ES, or 32 (bf16) when both operands are
                            // MN-major and K is short (dW at small B_tot)
  int a_rows;               // K-major A: rows per TMA box = per smem A stage (kBM, or M rounded
                            // up to 8 when all of M fits one block -- the B_tot-row operands at
                            // small B_tot: no zero-filled rows take smem or TMA time, and the
                            // freed bytes buy pipeline depth).  The M = 128 MMA still reads 128
                            // rows: rows >= a_rows read whatever follows in smem, and their
                            // accumulator rows (>= M) are never stored or used.
  // EPI_FWD_STATS
  const int32_t* labels;    // [M] global class ids
  long long class_offset;   // first class of this shard
  float* m_tile;            // [M x n_blocks]
  float* s_tile;            // [M x n_blocks]
  float* zy;                // [M] label logit (written by the owner tile only)
  const void* bias;         // [N] FC bias of this shard (ES-sized elements) or NULL (NEXT-4)
  int32_t* a_tile;          // [M x n_blocks] argmax class (global id) per row and tile, or NULL
  // producer-side wait for peer data (NVLink all-gather) before the first A load
  const uint32_t* wait_flags;  // [wait_count] local flag words, NULL = no wait
  int wait_count;
  uint32_t wait_mult;       // wait until flag >= epoch * wait_mult (monotonic counters)
  // EPI_FWD_STATS at N > 1: the bridge all-gather fused into this kernel (gather_on = 1): the
  // epilogue warps run the gather pieces blockIdx.x, blockIdx.x + gridDim.x, ... before their
  // first tile, and the producer issues the B (W_r) loads of the first ring stages before it
  // waits for the gathered A rows -- the W stream overlaps the NVLink exchange
  int gather_on;
  GatherArgs gather;
  // EPI_FWD_STATS: P~ written straight from registers (each thread its row's 64-byte pieces)
  // instead of through per-warp smem staging + TMA stores -- frees the 32 KB of staging for one
  // more load stage when the whole batch is one M block (the N > 1 shard shapes)
  void* p_direct;           // P~ base [M x ldp] (ES-sized elements) or NULL
  long long p_ld;           // its row pitch in elements
  int b_keep;               // 1: B (W_r) loads marked L2 evict_last -- W_r small enough to stay in L2
                            // for the backward's dX pass, which reads it again (w_l2)
  // step epoch: every kernel reads e = *dev_epoch + 1 (device-resident, so a whole step can
  // be captured once in a CUDA graph and replayed); the last backward kernel bumps it
  uint32_t* dev_epoch;
  int bump_epoch;           // 1: this launch ends the step (end ticket -> RS signal, epoch++)
  // split-K fixup (EPI_STORE_F32, dX)
  int fix_mode;             // FixMode
  const float* part;        // [splits x M x N] fp32 partials (the tmOut tensor)
  uint32_t* tile_cnt;       // [m_blocks x n_blocks] split-K arrival counters (re-armed by the end ticket)
  uint32_t* done_cnt;       // end-of-launch ticket (CTAs; re-armed by the last CTA)
  void* out;                // FIX_LOCAL: final dX [M x N] (ES-sized elements)
  int B, rank, world;       // FIX_PUSH: B = slab rows per source rank (B_max)
  int row_off[kMaxRanks + 1];  // FIX_PUSH: rows [row_off[r], row_off[r+1]) belong to rank r
  PeerPtrs recv;            // FIX_PUSH: owner's fp32 slab [world][B x N]
  PeerFlags rs_flags;       // N > 1: &flag[RS][rank] on every rank
  int rs_signal;            // 1: this launch ends the step at N > 1 -> raise the RS flags
  int store_mode;           // EPI_STORE_F32: 0 per-warp TMA box, 1 CTA-wide TMA box, 2 st.global
  int n_fastest;            // tile order: 0 = M fastest (share B), 1 = N fastest (share A)
  int cluster;              // 1, or 2: CTA pairs run M = 256 tcgen05.mma.cta_group::2 tiles over
                            // M-adjacent blocks (each CTA holds its 128 rows of A and half of
                            // B; only CTA 0 issues); num_tiles then counts pair tiles
  int debug;                // timing experiments only: bit0 skip stores, bit1 skip TMEM loads
  float* st_out;            // store_mode 2: output base ([splits x] M x N fp32)
  int* err;
  // d loss / d (mean loss) as a device scalar (the autograd grad_output), or NULL (= 1):
  // multiplied into the stored outputs (plain store epilogue) / the split-K fixup result
  const float* grad_scale;
};

// The backward's output factor: *grad_scale, or 1 without one.
__device__ __forceinline__ float grad_factor(const float* grad_scale) { return grad_scale ? __ldg(grad_scale) : 1.f; }
__device__ __forceinline__ void scale32(uint32_t (&v)[32], float s) {
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(__uint_as_float(v[k]) * s);
}

__host__ __device__ inline int gemm_smem_bytes(int stages, int stage_bytes, int epi_bufs) {
  return 1024 /*align slack*/ + stages * stage_bytes + 4 * epi_bufs * kEpiBufBytes + 256 /*barriers*/;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void decode_tile(const GemmArgs& a, int tile, int& mb, int& nb, int& sp, int& kb0,
                                            int& kb1) {
  if (a.n_fastest) {
    nb = tile % a.n_blocks;
    const int r = tile / a.n_blocks;
    mb = r % a.m_blocks;
    sp = r / a.m_blocks;
  } else {
    mb = tile % a.m_blocks;
    const int r = tile / a.m_blocks;
    nb = r % a.n_blocks;
    sp = r / a.n_blocks;
  }
  kb0 = sp * a.kb_per_split;
  kb1 = min(kb0 + a.kb_per_split, a.num_kb);
}

// Hand an accumulator back to the MMA issuer: every epilogue thread arrives on tempty -- in a
// CTA pair on the LEADER's barrier (its MMA overwrites both CTAs' halves).
// Relaxed: the TMEM loads completed (tcgen05.wait::ld) before the fence, so the arrive orders
// nothing else; .release would emit a GPU-scope MEMBAR per thread and tile (it waits for the
// thread's outstanding global stores).
__device__ __forceinline__ void release_acc(uint64_t* tempty_acc, bool pair) {
  tc_fence_before();
  if (pair) mbar_arrive_remote(mapa_smem(smem_u32(tempty_acc), 0));
  else mbar_arrive(tempty_acc);
}

// Unit -> tile for a CTA of rank `crank` in its cluster: with pairs (cluster = 2) a unit is
// an M-adjacent tile pair (2 mp, nb), (2 mp + 1, nb) sharing the B tile.
__device__ __forceinline__ void decode_unit(const GemmArgs& a, int unit, uint32_t crank, int& mb, int& nb, int& sp,
                                            int& kb0, int& kb1) {
  if (a.cluster == 2) {
    const int mpairs = a.m_blocks / 2;
    if (a.n_fastest) {
      nb = unit % a.n_blocks;
      const int r = unit / a.n_blocks;
      mb = r % mpairs;
      sp = r / mpairs;
    } else {
      mb = unit % mpairs;
      const int r = unit / mpairs;
      nb = r % a.n_blocks;
      sp = r / a.n_blocks;
    }
    mb = 2 * mb + static_cast<int>(crank);
    kb0 = sp * a.kb_per_split;
    kb1 = min(kb0 + a.kb_per_split, a.num_kb);
  } else {
    decode_tile(a, unit, mb, nb, sp, kb0, kb1);
  }
}

// Wait until <= n bulk stores of this thread are still reading smem (n = bufs - 1).
__device__ __forceinline__ void bulk_wait_read_n(int bufs) {
  if (bufs >= 8) bulk_wait_read<7>();
  else if (bufs >= 4) bulk_wait_read<3>();
  else bulk_wait_read<1>();
}

// Split-K fixup share of one tile (called by the 128 epilogue threads of every CTA that
// contributed split `sp`, after all splits arrived): reduce partials[0..S) in split order.
template <int ES>
__device__ __forceinline__ void fixup_share(const GemmArgs& a, int mb, int nb, int sp, int tid) {
  const int r0 = mb * kBM;
  const int nrows = min(kBM, a.M - r0);
  const int c0 = nb * a.BN;
  const int nc4 = min(a.BN, a.N - c0) / 4;
  const int total = nrows * nc4;
  const int per = (total + a.splits - 1) / a.splits;
  const int e0 = sp * per, e1 = min(total, e0 + per);
  const size_t split_stride = static_cast<size_t>(a.M) * a.N;
  const float gs = grad_factor(a.grad_scale);
  for (int e = e0 + tid; e < e1; e += 128) {
    const int r = r0 + e / nc4;
    const int c = c0 + (e % nc4) * 4;
    const float* src = a.part + static_cast<size_t>(r) * a.N + c;
    float4 acc = __ldcg(reinterpret_cast<const float4*>(src));
    for (int s = 1; s < a.splits; ++s) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(src + s * split_stride));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    if (a.grad_scale) {
      acc.x *= gs;
      acc.y *= gs;
      acc.z *= gs;
      acc.w *= gs;
    }
    if (a.fix_mode == FIX_LOCAL) {
      if constexpr (ES == 2) {
        uint2 o;
        o.x = pack_bf16x2(acc.x, acc.y);
        o.y = pack_bf16x2(acc.z, acc.w);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.out) + static_cast<size_t>(r) * a.N + c) = o;
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + static_cast<size_t>(r) * a.N + c) = acc;
      }
    } else {
      int owner = 0;  // the last rank whose rows start at or before r (empty ranks are skipped)
#pragma unroll
      for (int q = 1; q < kMaxRanks; ++q)
        if (q < a.world && a.row_off[q] <= r) owner = q;
      float* dst = reinterpret_cast<float*>(a.recv.p[owner]) +
                   (static_cast<size_t>(a.rank) * a.B + (r - a.row_off[owner])) * a.N + c;
      *reinterpret_cast<float4*>(dst) = acc;  // NVLink store into the owner's slab
    }
  }
}

// End of the backward's last launch (after the CTA-wide __syncthreads): the last CTA to
// finish raises flag[RS] = e on every rank (N > 1: all of this rank's dX pushes have landed
// AND every CTA finished reading the gathered X, so peers may overwrite it next step),
// re-arms the launch-local counters (done ticket, split-K tile counters, the dynamic
// scheduler) for the next backward -- they depend on no epoch, so forward-only steps in
// between are harmless -- and publishes the step epoch for the following kernels.
// pushes_fenced: every CTA already published its NVLink pushes with a system-scope fence right
// after them (the fused backward), so only the last CTA, which raises the RS flags, needs one.
__device__ __forceinline__ void end_of_step_ticket(const GemmArgs& a, uint32_t e, int& s_last,
                                                   unsigned* sched_cnt = nullptr, bool pushes_fenced = false) {
  // the RS flags (N > 1) publish this rank's dX pushes to the peers: system scope; at N = 1
  // the ticket orders only this GPU's kernels (gpu scope)
  const bool sys = a.rs_signal != 0 || (a.debug & 32);  // (debug bit 32: the old sys fences, for A/B)
  if (threadIdx.x == 0) {
    if (sys && !pushes_fenced) __threadfence_system();
    else __threadfence();
    const uint32_t done = atomicAdd(a.done_cnt, 1u) + 1u;
    s_last = (done == gridDim.x);
  }
  __syncthreads();
  if (!s_last) return;
  if (sys) __threadfence_system();
  else __threadfence();
  if (threadIdx.x < a.world && a.rs_signal) st_relaxed_sys(a.rs_flags.p[threadIdx.x], e);  // fenced above
  if (a.tile_cnt != nullptr)
    for (int k = threadIdx.x; k < a.m_blocks * a.n_blocks; k += blockDim.x) a.tile_cnt[k] = 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.done_cnt = 0u;
    if (sched_cnt != nullptr) *sched_cnt = 0u;
    __threadfence();
    atomicExch(a.dev_epoch, e);
  }
}

// Debug timeline of the logits kernel (WHALE_EPI_DEBUG bit 16, results unaffected): per CTA
// [entry, after prologue, producer's last load issued, MMA's last commit, epilogue's first
// accumulator, epilogue done] in globaltimer ns -- whale_debug_gemm_timeline.
__device__ unsigned long long g_gemm_cta[160 * 6];
#define WHALE_GEMM_STAMP(slot)                                                              \
  do {                                                                                     \
    if ((a.debug & 16) && blockIdx.x < 160) g_gemm_cta[blockIdx.x * 6 + (slot)] = gtime_ns(); \
  } while (0)

// Split-FC forward epilogue (EPI_FWD_STATS) by warps 4..11: warp w reads TMEM lane quadrant
// w % 4 (one thread per output row) and belongs to column group g = (w - 4) / 4, which owns the
// tile's P~ chunks (128-byte rows: 128 / ES columns) g, g + 2, ...  Pass 1: row max over the
// group's chunks (8 independent chains), combined through smem with the other group; pass 2:
// P~ = exp(z - m_tile) -> bf16 / fp32 staging -> TMA store, partial sum-exp (4 chains), the
// first column holding the max and the label logit; group 0 writes the tile statistics from
// both groups' partials in a fixed order.  Two 256-thread named barriers per tile.
template <int ES>
__device__ __forceinline__ void fwd_stats_epilogue(const GemmArgs& a, const CUtensorMap& tmOut, uint32_t tmem_base,
                                                   uint8_t* epi_smem, uint64_t* tfull, uint64_t* tempty, int unit0,
                                                   int ustride, uint32_t crank, int warp, int lane, bool pair) {
  // 1.5 KB of static smem (the GEMM's stage budget leaves ~1.7 KB): s_x[g][r] holds group g's
  // row max after pass 1; after pass 2 group 1 puts its partial sum into s_x[0][r] (a slot only
  // thread (1, r) reads, and already has) and its first-max column into s_arg1[r]
  __shared__ float s_x[2][kBM];
  __shared__ int s_arg1[kBM];
  constexpr int kChunk = kRowBytes / ES;  // P~ columns per 128-byte smem row
  constexpr float kLog2e = 1.4426950408889634f;
  const int q = warp & 3;
  const int g = (warp - 4) >> 2;
  const int r = q * 32 + lane;  // row within the tile
  const int nbw = a.epi_bufs / 2 > 0 ? a.epi_bufs / 2 : 1;  // staging buffers per warp
  uint8_t* ebuf = epi_smem + (g * 4 + q) * nbw * kEpiBufBytes;
  const bool has_bias = a.bias != nullptr;
  int buf = 0;
  int it = 0;
  for (int tile = unit0; tile < a.num_tiles; tile += ustride, ++it) {
    int mb, nb, sp, kb0, kb1;
    decode_unit(a, tile, crank, mb, nb, sp, kb0, kb1);
    const int acc = it & 1;
    mbar_wait(&tfull[acc], (it >> 1) & 1);
    tc_fence_after();
    if (it == 0 && threadIdx.x == 128) WHALE_GEMM_STAMP(4);
    const uint32_t tbase = tmem_base + acc * kMaxBN + (static_cast<uint32_t>(q * 32) << 16);
    const int row0 = mb * kBM + q * 32;
    const int row = row0 + lane;
    const bool rv = row < a.M;
    const bool wv = row0 < a.M;  // warp-uniform: rows of this warp exist
    const int ncol = min(a.BN, a.N - nb * a.BN);  // valid classes in this tile
    const int nch = a.BN / kChunk;
    const long long bcol0 = static_cast<long long>(nb) * a.BN;
    auto bias_at = [&](int c) -> float {
      if (bcol0 + c >= a.N) return 0.f;
      if constexpr (ES == 2) return __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(a.bias) + bcol0 + c));
      else return __ldg(reinterpret_cast<const float*>(a.bias) + bcol0 + c);
    };
    // fast path (full tile, no bias, no top-1 wanted): ~4 instructions per logit
    const bool want_arg = a.a_tile != nullptr;
    const bool fast = ncol == a.BN && !has_bias && !want_arg;
    // ---- pass 1: this group's row max
    float mxk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) mxk[k] = -INFINITY;
    if (wv) {
      for (int ch = g; ch < nch; ch += 2) {
        for (int h = 0; h < kChunk; h += 32) {
          const int c0 = ch * kChunk + h;
          uint32_t v[32];
          tmem_ld32(tbase + c0, v);
          tmem_ld_wait();
          if (fast) {
#pragma unroll
            for (int c = 0; c < 32; ++c) mxk[c & 7] = fmaxf(mxk[c & 7], __uint_as_float(v[c]));
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const float z = __uint_as_float(v[c]) + (has_bias ? bias_at(c0 + c) : 0.f);
              mxk[c & 7] = fmaxf(mxk[c & 7], (c0 + c < ncol) ? z : -INFINITY);
            }
          }
        }
      }
    }
    const float my_mx = fmaxf(fmaxf(fmaxf(mxk[0], mxk[1]), fmaxf(mxk[2], mxk[3])),
                              fmaxf(fmaxf(mxk[4], mxk[5]), fmaxf(mxk[6], mxk[7])));
    s_x[g][r] = my_mx;
    named_bar_sync(2, 256);
    const float mx = g == 0 ? fmaxf(my_mx, s_x[1][r]) : fmaxf(s_x[0][r], my_mx);  // same order: max(g0, g1)
    const float mxl = mx * kLog2e;
    long long yl = -1;
    if (rv) yl = static_cast<long long>(a.labels[row]) - a.class_offset - bcol0;
    // ---- pass 2: P~, partial sums, first column of the max, label logit
    float sk[4] = {0.f, 0.f, 0.f, 0.f};
    int am = 0x7fffffff;
    float zy = 0.f;
    bool has_zy = false;
    const bool direct = a.p_direct != nullptr;
    if (wv) {
      for (int ch = g; ch < nch; ch += 2) {
        if (!direct) {
          if (lane == 0) {  // the store that last used this buffer has read it
            if (nbw >= 4) bulk_wait_read<3>();
            else if (nbw >= 2) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          __syncwarp();
        }
        uint8_t* b = ebuf + buf * kEpiBufBytes + lane * 128;
        for (int h = 0; h < kChunk; h += 32) {
          const int c0 = ch * kChunk + h;
          uint32_t v[32];
          tmem_ld32(tbase + c0, v);
          tmem_ld_wait();
          uint32_t pk[32];
          // the label logit: one select per logit, stored once per tile below
          const long long yrel = yl - c0;
          if (yrel >= 0 && yrel < 32 && c0 + yrel < ncol) {
            has_zy = true;
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (c == yrel) zy = __uint_as_float(v[c]) + (has_bias ? bias_at(c0 + c) : 0.f);
          }
          if (fast) {
#pragma unroll
            for (int c = 0; c < 32; c += 2) {
              const float p0 = ex2_approx(fmaf(__uint_as_float(v[c]), kLog2e, -mxl));
              const float p1 = ex2_approx(fmaf(__uint_as_float(v[c + 1]), kLog2e, -mxl));
              sk[(c >> 1) & 3] += p0 + p1;
              if constexpr (ES == 2) {
                pk[c >> 1] = pack_bf16x2(p0, p1);
              } else {
                pk[c] = __float_as_uint(p0);
                pk[c + 1] = __float_as_uint(p1);
              }
            }
          } else {
#pragma unroll
            for (int c = 0; c < 32; c += 2) {
              const float z0 = __uint_as_float(v[c]) + (has_bias ? bias_at(c0 + c) : 0.f);
              const float z1 = __uint_as_float(v[c + 1]) + (has_bias ? bias_at(c0 + c + 1) : 0.f);
              const bool ok0 = c0 + c < ncol, ok1 = c0 + c + 1 < ncol;
              const float p0 = ok0 ? ex2_approx(fmaf(z0, kLog2e, -mxl)) : 0.f;
              const float p1 = ok1 ? ex2_approx(fmaf(z1, kLog2e, -mxl)) : 0.f;
              sk[(c >> 1) & 3] += p0 + p1;
              if (want_arg) {
                if (ok0 && z0 == mx) am = min(am, c0 + c);
                if (ok1 && z1 == mx) am = min(am, c0 + c + 1);
              }
              if constexpr (ES == 2) {
                pk[c >> 1] = pack_bf16x2(p0, p1);
              } else {
                pk[c] = __float_as_uint(p0);
                pk[c + 1] = __float_as_uint(p1);
              }
            }
          }
          // this half-chunk's 16-byte pieces: bf16 -> 4 pieces at h / 8, fp32 -> 8 pieces
          constexpr int kPieces = 32 * ES / 16;
          if (direct) {  // this row's 32 values straight to global (clipped to the valid columns)
            if (rv) {
              uint8_t* gp = static_cast<uint8_t*>(a.p_direct) +
                            (static_cast<size_t>(row) * a.p_ld + static_cast<size_t>(bcol0 + c0)) * ES;
              if (c0 + 32 <= ncol) {
#pragma unroll
                for (int k = 0; k < kPieces; ++k)
                  *reinterpret_cast<uint4*>(gp + 16 * k) = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
              } else {
#pragma unroll
                for (int c = 0; c < 32; ++c) {  // unrolled: pk stays in registers (static indices)
                  if (c0 + c >= ncol) continue;
                  if constexpr (ES == 2) {
                    const uint32_t w2 = pk[c >> 1];
                    *reinterpret_cast<uint16_t*>(gp + 2 * c) = static_cast<uint16_t>((c & 1) ? (w2 >> 16) : (w2 & 0xffffu));
                  } else {
                    *reinterpret_cast<uint32_t*>(gp + 4 * c) = pk[c];
                  }
                }
              }
            }
            continue;
          }
#pragma unroll
          for (int k = 0; k < kPieces; ++k) {
            const int pc = (h * ES) / 16 + k;  // 16-byte piece within the 128-byte row
            *reinterpret_cast<uint4*>(b + ((pc ^ (lane & 7)) << 4)) =
                make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
          }
        }
        if (direct) continue;
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmOut, ebuf + buf * kEpiBufBytes, nb * a.BN + ch * kChunk, row0);
          bulk_commit();
        }
        if (++buf == nbw) buf = 0;
      }
    }
    release_acc(&tempty[acc], pair);  // this thread's TMEM reads of the tile are done (256 arrivals)
    if (has_zy) a.zy[row] = zy;
    const float my_sum = (sk[0] + sk[1]) + (sk[2] + sk[3]);
    if (g == 1) {
      s_x[0][r] = my_sum;
      s_arg1[r] = am;
    }
    named_bar_sync(2, 256);
    if (g == 0 && rv) {
      const float sum = my_sum + s_x[0][r];
      int amin = min(am, s_arg1[r]);
      if (amin == 0x7fffffff) amin = 0;  // no column equals the max (NaN inputs): any valid id
      a.m_tile[static_cast<size_t>(row) * a.n_blocks + nb] = mx;
      a.s_tile[static_cast<size_t>(row) * a.n_blocks + nb] = sum;
      if (a.a_tile != nullptr)
        a.a_tile[static_cast<size_t>(row) * a.n_blocks + nb] = static_cast<int32_t>(a.class_offset + bcol0 + amin);
    }
  }
  if (lane == 0) bulk_wait<0>();
  if (threadIdx.x == 128) WHALE_GEMM_STAMP(5);
}

// ES = operand element size: 2 -> bf16 (kind::f16), 4 -> fp32 storage run as kind::tf32.
// EPI_FWD_STATS runs 12 warps: its epilogue (two passes over the accumulator, an exp per
// logit) is the slow side of the TMEM double buffer when K is short (c4: D = 512), so two
// groups of 4 warps split each tile's column chunks (interleaved) and combine their row
// max / sum / top-1 through shared memory.
// PAIR: the cta_group::2 instantiation (launched as 2-CTA clusters; a kernel that contains
// cta_group::2 instructions cannot be launched without a cluster).
template <int EPI, bool A_MN, bool B_MN, int ES, bool PAIR = false>
__global__ void __launch_bounds__(EPI == EPI_FWD_STATS ? kStatsGemmThreads : kGemmThreads, 1)
    splitfc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmOut, const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_fix_go;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi_smem = smem + a.stages * a.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + 4 * a.epi_bufs * kEpiBufBytes);
  uint64_t* empty = full + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  if (EPI == EPI_FWD_STATS && threadIdx.x == 0) WHALE_GEMM_STAMP(0);

  constexpr int kBK = kRowBytes / ES;        // K elements per stage
  constexpr int kAtom = kRowBytes / ES;      // MN elements per swizzle atom (MN-major)
  constexpr int kKStepMN = (32 / ES) * kRowBytes;  // MN-major: UMMA_K rows per MMA
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // CTA pairs (cluster = 2): unit u = pair tile, this CTA takes M block 2*mp + crank
  constexpr int cs = PAIR ? 2 : 1;
  const uint32_t crank = cs > 1 ? cluster_ctarank() : 0u;
  const int unit0 = cs > 1 ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int ustride = cs > 1 ? static_cast<int>(ncluster_x()) : static_cast<int>(gridDim.x);

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);   // pairs: the leader's expect_tx; both CTAs' TMA bytes land here
      mbar_init(&empty[i], 1);  // pairs: the leader's multicast commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], (EPI == EPI_FWD_STATS ? 256 : 128) * cs);  // pairs: both CTAs' epilogues
    }
    fence_mbar_init();
  }
  if (threadIdx.x == 32) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmOut);
  }
  if (cs > 1) cluster_sync();  // peer barriers initialised before any pair TMA / commit lands
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_pair(tmem_holder, kTmemCols);
    else tmem_alloc(tmem_holder, kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();      // everything below reads/writes memory the previous kernel may touch
  pdl_trigger();
  TraceScope _trace(EPI == EPI_FWD_STATS ? 1 : (a.fix_mode != FIX_NONE ? 5 : 4));
  const uint32_t e = ld_acquire_gpu(a.dev_epoch) + 1u;  // this step's epoch
  if (EPI == EPI_FWD_STATS && threadIdx.x == 0) WHALE_GEMM_STAMP(1);

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      // peers' rows of A were pushed over NVLink by generic-proxy stores; acquire their
      // flags, then order the async-proxy (TMA) reads after them.  With the fused gather (K-major
      // A, no pairs) the first ring stages get their B loads at once and their A loads after
      // the wait (deferred), so W_r streams while the all-gather lands.
      // (no lambdas / arrays: captured or indexed locals would live in local memory; the
      // deferred stages are stages 0 .. ndef - 1, all in this CTA's first tile: k-blocks
      // kb0f .. kb0f + ndef - 1 of M block mbf)
      bool a_ready = a.wait_flags == nullptr;
      const bool defer = !a_ready && a.gather_on && !PAIR && !A_MN;
      if (!a_ready && !defer) {
        for (int p = 0; p < a.wait_count; ++p) wait_flag_geq(a.wait_flags + p, e * a.wait_mult, a.err, ERR_COMM | ERR_AT_GATHER);
        fence_proxy_async_global();
        a_ready = true;
      }
      int ndef = 0, kb0f = 0, mbf = 0;
      int stage = 0;
      uint32_t phase = 0;
      const int bk = (A_MN && B_MN) ? a.bk : kBK;
      const int box_bytes = bk * kRowBytes;
      const int a_bytes = A_MN ? (kBM / kAtom) * box_bytes : a.a_rows * kRowBytes;
      // pairs: this CTA's half of B; the leader expects both CTAs' bytes
      const int bn_cta = a.BN / cs;
      const uint32_t tx = static_cast<uint32_t>(cs) *
                          static_cast<uint32_t>((WHALE_SKIP(a.debug & 8) ? 0 : a_bytes) +
                                                (B_MN ? (bn_cta / kAtom) * box_bytes : bn_cta * kRowBytes));
      for (int tile = unit0; tile < a.num_tiles; tile += ustride) {
        int mb, nb, sp, kb0, kb1;
        decode_unit(a, tile, crank, mb, nb, sp, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          uint8_t* sA = smem + stage * a.stage_bytes;
          uint8_t* sB = sA + a_bytes;
          if constexpr (PAIR) {
            mbar_wait(&empty[stage], phase ^ 1u);
            // pair: both CTAs load their own A rows and their half of B into their own smem;
            // the bytes complete on the leader's full barrier, which the leader alone arms
            const uint32_t fl = mapa_smem(smem_u32(&full[stage]), 0);
            if (crank == 0) mbar_arrive_expect_tx(&full[stage], tx);
            if (!A_MN) {
              tma_load_2d_pair(sA, &tmA, fl, kb * kBK, mb * kBM);
            } else {
#pragma unroll
              for (int j = 0; j < kBM / kAtom; ++j)
                tma_load_2d_pair(sA + j * box_bytes, &tmA, fl, mb * kBM + j * kAtom, kb * bk);
            }
            if (!B_MN) {  // tmB box = {kBK, BN/2}
              tma_load_2d_pair(sB, &tmB, fl, kb * kBK, nb * a.BN + static_cast<int>(crank) * bn_cta);
            } else {
              for (int j = 0; j < bn_cta / kAtom; ++j)
                tma_load_2d_pair(sB + j * box_bytes, &tmB, fl, nb * a.BN + static_cast<int>(crank) * bn_cta + j * kAtom,
                                 kb * bk);
            }
            if (++stage == a.stages) {
              stage = 0;
              phase ^= 1u;
            }
            continue;
          }
          if (!a_ready && (ndef == a.stages || tile != unit0)) {  // resolve before a deferred stage's reuse
            for (int p = 0; p < a.wait_count; ++p) wait_flag_geq(a.wait_flags + p, e * a.wait_mult, a.err, ERR_COMM | ERR_AT_GATHER);
            fence_proxy_async_global();
            a_ready = true;
            for (int i = 0; i < ndef; ++i)
              tma_load_2d(smem + i * a.stage_bytes, &tmA, &full[i], (kb0f + i) * kBK, mbf * kBM);
          }
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_arrive_expect_tx(&full[stage], tx);
          if (WHALE_SKIP(a.debug & 8)) {
            // timing experiment: A operand not loaded
          } else if (!a_ready) {
            if (ndef == 0) {  // A after the all-gather (K-major A only)
              kb0f = kb;
              mbf = mb;
            }
            ++ndef;
          } else if (!A_MN) {
            tma_load_2d(sA, &tmA, &full[stage], kb * kBK, mb * kBM);
          } else {
#pragma unroll
            for (int j = 0; j < kBM / kAtom; ++j)
              tma_load_2d(sA + j * box_bytes, &tmA, &full[stage], mb * kBM + j * kAtom, kb * bk);
          }
          if (!B_MN) {
            if (a.b_keep) tma_load_2d_hint(sB, &tmB, &full[stage], kb * kBK, nb * a.BN, l2_policy_evict_last());
            else tma_load_2d(sB, &tmB, &full[stage], kb * kBK, nb * a.BN);
          } else {
            for (int j = 0; j < a.BN / kAtom; ++j)
              tma_load_2d(sB + j * box_bytes, &tmB, &full[stage], nb * a.BN + j * kAtom, kb * bk);
          }
          if (++stage == a.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      if (EPI == EPI_FWD_STATS) WHALE_GEMM_STAMP(2);
      if (!a_ready) {  // fewer k-blocks than ring stages (or no tile)
        for (int p = 0; p < a.wait_count; ++p) wait_flag_geq(a.wait_flags + p, e * a.wait_mult, a.err, ERR_COMM | ERR_AT_GATHER);
        fence_proxy_async_global();
        for (int i = 0; i < ndef; ++i)
          tma_load_2d(smem + i * a.stage_bytes, &tmA, &full[i], (kb0f + i) * kBK, mbf * kBM);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (pairs: the leader only, M = 256) =====================
    if (lane == 0 && crank == 0) {
      const uint32_t idesc = umma_idesc(kBM * cs, a.BN, A_MN, B_MN, ES == 2 ? 1u : 2u);
      const int bk = (A_MN && B_MN) ? a.bk : kBK;
      const uint32_t box_bytes = bk * kRowBytes;
      const uint32_t a_bytes = A_MN ? (kBM / kAtom) * box_bytes : a.a_rows * kRowBytes;
      const int kmma = bk / (32 / ES);  // MMAs (32 bytes of K each) per stage
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = unit0; tile < a.num_tiles; tile += ustride, ++it) {
        int mb, nb, sp, kb0, kb1;
        decode_unit(a, tile, crank, mb, nb, sp, kb0, kb1);
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kMaxBN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t aS = smem_u32(smem + stage * a.stage_bytes);
          const uint32_t bS = aS + a_bytes;
#pragma unroll 4
          for (int k = 0; k < (WHALE_SKIP(a.debug & 4) ? 0 : kmma); ++k) {  // MMAs of 32 bytes of K
            const uint64_t ad = A_MN ? umma_sdesc(aS + k * kKStepMN, box_bytes, 1024)
                                     : umma_sdesc(aS + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_sdesc(bS + k * kKStepMN, box_bytes, 1024)
                                     : umma_sdesc(bS + k * 32, 16, 1024);
            if constexpr (PAIR) {
              if constexpr (ES == 2)
                umma_bf16_pair(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
              else
                umma_tf32_pair(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            } else if constexpr (ES == 2) {
              umma_bf16(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            } else {
              umma_tf32(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          }
          // frees this smem stage (pairs: in both CTAs) once the MMAs have read it
          if constexpr (PAIR) umma_commit_pair_mc(&empty[stage], 0x3);
          else umma_commit(&empty[stage]);
          if (++stage == a.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if constexpr (PAIR) umma_commit_pair_mc(&tfull[acc], 0x3);  // both halves ready
        else umma_commit(&tfull[acc]);                     // accumulator ready for the epilogue
      }
      if (EPI == EPI_FWD_STATS) WHALE_GEMM_STAMP(3);
    }
  } else if (EPI == EPI_FWD_STATS && warp >= 4) {
    // ===================== logits epilogue: 8 warps, 2 column groups =====================
    if (a.gather_on) {  // the fused bridge all-gather: this CTA's pieces, then one signal
      int n = 0;
      for (int part = static_cast<int>(blockIdx.x); part < a.gather.parts; part += static_cast<int>(gridDim.x), ++n)
        gather_copy(a.gather, part, threadIdx.x - 128, 256);
      named_bar_sync(2, 256);
      if (threadIdx.x == 128 && n > 0) gather_signal(a.gather, n);
    }
    // N > 1: the gathered labels are peer-written (bridge_gather); acquire the gather flags
    // here too before any label read (the producer's acquire orders only its own lane)
    if (a.wait_flags != nullptr && threadIdx.x == 128)
      for (int p = 0; p < a.wait_count; ++p) wait_flag_geq(a.wait_flags + p, e * a.wait_mult, a.err, ERR_COMM | ERR_AT_GATHER);
    named_bar_sync(2, 256);
    fwd_stats_epilogue<ES>(a, tmOut, tmem_base, epi_smem, tfull, tempty, unit0, ustride, crank, warp, lane, cs > 1);
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int nbuf = a.epi_bufs;
    uint8_t* ebuf = epi_smem + q * nbuf * kEpiBufBytes;
    int buf = 0;
    int it = 0;
    for (int tile = unit0; tile < a.num_tiles; tile += ustride, ++it) {
      int mb, nb, sp, kb0, kb1;
      decode_unit(a, tile, crank, mb, nb, sp, kb0, kb1);
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * kMaxBN + (static_cast<uint32_t>(q * 32) << 16);
      const int row0 = mb * kBM + q * 32;  // first output row of this warp
      const int row = row0 + lane;
      if constexpr (EPI == EPI_STORE_F32) {
        // plain stores (dW) carry the grad_output factor; split-K partials get it in the fixup
        const bool do_scale = a.grad_scale != nullptr && a.fix_mode == FIX_NONE;
        const float gsc = do_scale ? grad_factor(a.grad_scale) : 1.f;
        if (a.store_mode == 1) {
          // CTA-wide 128-row box: all 4 warps fill one 16 KB stage, one thread stores it
          for (int c0 = 0; c0 < a.BN; c0 += 32) {
            uint32_t v[32];
            if (!WHALE_SKIP(a.debug & 2)) {
              tmem_ld32(tbase + c0, v);
              tmem_ld_wait();
            } else {
#pragma unroll
              for (int k = 0; k < 32; ++k) v[k] = k;
            }
            if (do_scale) scale32(v, gsc);
            if (c0 + 32 >= a.BN) {
              release_acc(&tempty[acc], cs > 1);
            }
            if (WHALE_SKIP(a.debug & 1)) continue;
            if (threadIdx.x == 128) bulk_wait_read_n(nbuf);
            named_bar_sync(1, 128);
            uint8_t* b = epi_smem + buf * 4 * kEpiBufBytes + (q * 32 + lane) * 128;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch)
              *reinterpret_cast<uint4*>(b + ((ch ^ (lane & 7)) << 4)) =
                  make_uint4(v[4 * ch], v[4 * ch + 1], v[4 * ch + 2], v[4 * ch + 3]);
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (threadIdx.x == 128) {
              tma_store_3d(&tmOut, epi_smem + buf * 4 * kEpiBufBytes, nb * a.BN + c0, mb * kBM, sp);
              bulk_commit();
            }
            if (++buf == nbuf) buf = 0;
          }
        } else if (a.store_mode == 2) {
          // direct 16-byte global stores from registers (each thread: its row, 128 B per chunk)
          const bool rv = row < a.M;
          float* orow = a.st_out + (static_cast<size_t>(sp) * a.M + (rv ? row : 0)) * a.N;
          for (int c0 = 0; c0 < a.BN; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tbase + c0, v);
            tmem_ld_wait();
            if (c0 + 32 >= a.BN) {
              release_acc(&tempty[acc], cs > 1);
            }
            if (do_scale) scale32(v, gsc);
            const int col = nb * a.BN + c0;
            if (rv) {
#pragma unroll
              for (int ch = 0; ch < 8; ++ch)
                if (col + 4 * ch < a.N)
                  __stcs(reinterpret_cast<float4*>(orow + col + 4 * ch),
                         make_float4(__uint_as_float(v[4 * ch]), __uint_as_float(v[4 * ch + 1]),
                                     __uint_as_float(v[4 * ch + 2]), __uint_as_float(v[4 * ch + 3])));
            }
          }
        } else if (row0 < a.M) {
          for (int c0 = 0; c0 < a.BN; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tbase + c0, v);
            tmem_ld_wait();
            if (c0 + 32 >= a.BN) {  // accumulator fully read: hand TMEM back to the MMA warp
              release_acc(&tempty[acc], cs > 1);
            }
            if (do_scale) scale32(v, gsc);
            if (lane == 0) bulk_wait_read_n(nbuf);  // the store that last used this buffer has read it
            __syncwarp();
            uint8_t* b = ebuf + buf * kEpiBufBytes + lane * 128;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch)
              *reinterpret_cast<uint4*>(b + ((ch ^ (lane & 7)) << 4)) =
                  make_uint4(v[4 * ch], v[4 * ch + 1], v[4 * ch + 2], v[4 * ch + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&tmOut, ebuf + buf * kEpiBufBytes, nb * a.BN + c0, row0, sp);
              bulk_commit();
            }
            if (++buf == nbuf) buf = 0;
          }
        } else {
          release_acc(&tempty[acc], cs > 1);
        }
      }
      if constexpr (EPI == EPI_STORE_F32) {
        if (a.fix_mode != FIX_NONE) {
          // ---- split-K fixup: publish this split, wait for all, reduce my 1/S share ----
          if (lane == 0 || threadIdx.x == 128) bulk_wait<0>();  // this CTA's partial stores are complete
          __syncwarp();
          fence_proxy_async_global();
          __threadfence();
          named_bar_sync(1, 128);
          uint32_t* cnt = a.tile_cnt + mb * a.n_blocks + nb;
          if (threadIdx.x == 128) {
            atomicAdd(cnt, 1u);
            const uint32_t target = static_cast<uint32_t>(a.splits);
            if (static_cast<int32_t>(ld_acquire_gpu(cnt) - target) < 0) {
              SpinGuard g;
              while (static_cast<int32_t>(ld_acquire_gpu(cnt) - target) < 0)
                if (g.expired(a.err, ERR_SPLITK)) break;
            }
          }
          named_bar_sync(1, 128);
          __threadfence();
          fixup_share<ES>(a, mb, nb, sp, threadIdx.x - 128);
        }
      }
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  // pairs: the peer may still multicast into this CTA's smem / arrive on its barriers
  if (cs > 1) cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair(tmem_base, kTmemCols);
    else tmem_dealloc(tmem_base, kTmemCols);
  }
  if (a.bump_epoch) end_of_step_ticket(a, e, s_fix_go);
}

}  // namespace whale
