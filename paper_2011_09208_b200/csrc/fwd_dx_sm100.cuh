// Fused forward + dX for small global batches (B_tot <= 32) on sm_100a: "F1".
//
// Why: with B_tot = 32 the split-FC step is HBM-bound on W_r, which the plain pipeline
// streams twice -- once for the logits Z = X W_r^T and once more for dX = G W_r in the
// backward (G needs the global log-sum-exp, known only after every class was seen).  F1
// reads W_r from HBM once.  It is flash-attention's forward with Q = X and K = V = W_r:
// for every class tile t it forms Z_t, a per-row reference max, P~_t = exp(Z_t - ref), and
// accumulates U = sum_t P~_t W_t in TMEM, rescaling U when a row's reference moves up
// (lazily: only when the new tile max exceeds the reference by > 2^8).  The backward then
// finishes dX = (1/B_tot) (sum_clusters e^{ref - lse} U - W_{y}) with a tiny combine kernel,
// and its GEMM shrinks to dW alone.
//
// Transposed formulation (B_tot is the MMA N, so TMEM holds U for a D range):
//   G1:  Z_t^T [128 classes x 32 rows]  += W_t[:, d-chunk] (K-major) * X[:, d-chunk]^T
//   G2:  U^T   [D_q rows x 32 rows]     += W_t^T (MN-major view of the same W tile) * P~_t^T
// A cluster of KC = 2 CTAs shares each class tile; CTA q owns the D half
// [q*D/2, (q+1)*D/2): it runs G1 over its half only, the two partial Z_t^T (16 KB each)
// are exchanged through distributed shared memory (st.async + mbarrier tx counts, summed
// in cluster-rank order so both CTAs hold bit-identical Z_t), both compute the same P~_t,
// and G2 accumulates the CTA's own D half of U.  G2 re-reads its W half (just read by G1)
// from L2, so DRAM sees W once.  (KC = 2, not 4: every CTA of a cluster repeats the tile's
// softmax epilogue, so fewer, larger D parts halve that work; TMEM holds U for D/2 <= 1024.)
//
// The per-(row, tile) statistics written for the rest of the pipeline generalise the
// logits GEMM's EPI_FWD_STATS epilogue: m_tile = the row's reference for the tile,
// s_tile = sum exp(z - m_tile), P~ = exp(z - m_tile) in bf16 (the backward's dW operand,
// TMA-stored straight from the G2 operand buffer), z_y, plus mx_tile = the true tile max and
// a_tile = its class (predictions).  Any reference gives the same lse; the statistics
// kernels take the row max from mx_tile.
//
//   warp 0      TMA producer (one lane): X part once (resident), then W chunks in MMA order
//   warp 1      MMA issuer (one lane):   period p = G1(p) interleaved with G2(p - 2)
//   warp 2      TMEM allocator (512 columns: Z x 2 and U blocks x D_q/128, 32 columns each)
//   warp 3      TMA producer for the G2 ring (L2 re-reads)
//   warps 4..11 epilogue: thread = class row of the tile (TMEM lane) x 16 batch columns
#pragma once
#include "gemm_sm100.cuh"

namespace whale {

constexpr int kF1NB = 32;                          // batch columns (B_tot padded with zero rows)
constexpr int kF1KC = 2;                           // CTAs per cluster = D parts
constexpr int kF1TileC = 128;                      // classes per tile (MMA M of G1)
constexpr int kF1StageBytes = kF1TileC * kRowBytes;  // 128 classes x 64 D bf16 = 16 KB
constexpr int kF1XChunkBytes = kF1NB * kRowBytes;    // 32 rows x 64 D bf16 = 4 KB
constexpr int kF1SlotBytes = kF1TileC * kF1NB * 4;   // one partial Z_t^T, fp32 = 16 KB
constexpr int kF1PBytes = 2 * kF1NB * kRowBytes;     // P~_t^T operand: 2 atoms x 32 rows x 128 B
constexpr int kF1TmemCols = 512;
constexpr int kF1G1SlotBytes = kF1StageBytes + kF1XChunkBytes;  // G1 ring slot: W chunk + X chunk
constexpr int kF1G2SlotBytes = 2 * kF1StageBytes;                 // G2 ring slot: 128 D rows of W
constexpr int kF1S2Max = 4;                                       // G2 ring slots (runtime: F1Args.s2)
constexpr int kF1EpiThreads = 256;                                // 8 epilogue warps
constexpr int kF1Threads = 128 + kF1EpiThreads;
constexpr float kF1Tau = 8.0f;  // lazy rescale threshold, log2 units

struct F1Args {
  int Bt;                  // valid rows (<= 32)
  int D, Dq;               // feature dim, D / KC (multiple of 128, <= 1024)
  int C_r;                 // classes of this shard
  int num_tiles;           // ceil(C_r / 128) = T
  int stages;              // G1 ring slots
  int s2;                  // G2 ring slots (<= kF1S2Max)
  int split_issue;         // 1: G1 and G2 issued by two threads (warps 1 and 2)
  long long class_offset;  // o_r
  const int32_t* labels;   // [Bt] global class ids
  const void* bias;        // [C_r] bf16 or NULL
  float* m_tile;           // [Bt x T] reference the tile's P~ and s_tile are relative to
  float* s_tile;           // [Bt x T]
  float* mx_tile;          // [Bt x T] true tile max
  float* zy;               // [Bt]
  int32_t* a_tile;         // [Bt x T] global class id of the tile's max, or NULL
  float* upart;            // [ncl x Bt x D] per-cluster U (relative to uref)
  float* uref;             // [ncl x Bt]
  const uint32_t* wait_flags;  // N > 1: gather flags (as GemmArgs)
  int wait_count;
  uint32_t wait_mult;
  int gather_on;           // N > 1: the bridge all-gather fused into the prologue (as GemmArgs)
  GatherArgs gather;
  uint32_t* dev_epoch;
  int* err;
  int debug;               // timing experiments: bit 0 = record a per-period timeline of CTA 0,
                           // bit 1 = skip G2 (dX wrong)
};

// Debug timeline (CTA 0): [period][16] globaltimer stamps, see splitfc_fwd_dx_kernel.
__device__ unsigned long long g_f1_ts[64 * 16];
__device__ unsigned long long g_f1_cta[160 * 5];  // per-CTA [entry, after prologue, end, after cluster sync, thread 0 at exit sync] (debug bit 0)

__host__ __device__ constexpr int f1_smem_bytes(int stages, int s2) {
  return 1024 + stages * kF1G1SlotBytes + s2 * kF1G2SlotBytes + (kF1KC - 1) * kF1SlotBytes + 2 * kF1PBytes + 512;
}

// Warp-wide fp32 max (sm_100a redux.sync .f32), result in every lane.
__device__ __forceinline__ float redux_max_f32(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

// Column-wise sum of a 32 x 32 register block across the warp: afterwards v[0] of lane l
// holds column l's sum (31 shuffles instead of 32 x 5).
__device__ __forceinline__ void f1_colsum32(float (&v)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool hi = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float sv = hi ? v[i] : v[i + w];
      const float kv = hi ? v[i + w] : v[i];
      v[i] = kv + __shfl_xor_sync(0xffffffffu, sv, w);
    }
  }
}

__global__ void __launch_bounds__(kF1Threads, 1)
    splitfc_fwd_dx_kernel(const __grid_constant__ CUtensorMap tmW /*box {64, 128}*/,
                          const __grid_constant__ CUtensorMap tmX /*box {64, 32}*/,
                          const __grid_constant__ CUtensorMap tmP /*P~ [B_tot x C_r], box {64, 32}*/, const F1Args a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ float red_v[4][32];
  __shared__ int red_i[4][32];
  __shared__ __align__(16) float s_ref[32];
  __shared__ float s_fac[32], s_max[32];
  __shared__ int s_arg[32], s_lab[32];
  __shared__ int s_rescale;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int KQ = a.Dq / 64;  // 64-wide D chunks of this CTA's part
  const int S1 = a.stages;   // G1 ring: W chunk (16 KB) + X chunk (4 KB) per slot
  uint8_t* ring1 = smem;
  uint8_t* ring2 = ring1 + S1 * kF1G1SlotBytes;  // G2 ring: one 128-D block (2 W chunks) per slot
  uint8_t* recv = ring2 + a.s2 * kF1G2SlotBytes;
  uint8_t* pbuf = recv + (kF1KC - 1) * kF1SlotBytes;  // 2 buffers
  uint64_t* full1 = reinterpret_cast<uint64_t*>(pbuf + 2 * kF1PBytes);
  uint64_t* empty1 = full1 + S1;
  uint64_t* full2 = empty1 + S1;
  uint64_t* empty2 = full2 + a.s2;
  uint64_t* zfull = empty2 + a.s2;  // 3 Z buffers
  uint64_t* zempty = zfull + 3;
  uint64_t* pfull = zempty + 3;      // 2 P~ buffers
  uint64_t* pempty = pfull + 2;      // completes when G2 of that buffer's tile finished
  uint64_t* xfull = pempty + 2;
  uint64_t* xempty = xfull + 1;
  uint64_t* ublk = xempty + 1;        // [KQ / 2 <= 8]: U block i final (the last tile's G2 block i done)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(ublk + 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t q = cluster_ctarank();
  const int cl = static_cast<int>(cluster_id_x());
  const int ncl = static_cast<int>(ncluster_x());
  const int my_tiles = cl < a.num_tiles ? (a.num_tiles - 1 - cl) / ncl + 1 : 0;
  const uint32_t ucol0 = 3 * kF1NB;  // TMEM: Z buffers at 0, 32, 64; U blocks from 96
  if ((a.debug & 1) && threadIdx.x == 0 && blockIdx.x < 160) g_f1_cta[blockIdx.x * 5] = gtime_ns();

  if (threadIdx.x == 0) {
    for (int i = 0; i < S1; ++i) {
      mbar_init(&full1[i], 1);
      mbar_init(&empty1[i], 1);
    }
    for (int i = 0; i < a.s2; ++i) {
      mbar_init(&full2[i], 1);
      mbar_init(&empty2[i], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&zfull[i], 1);
      mbar_init(&zempty[i], kF1EpiThreads);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&pfull[i], kF1EpiThreads);
      mbar_init(&pempty[i], 1);
    }
    mbar_init(xfull, 1);
    mbar_init(xempty, kF1KC - 1);
    for (int i = 0; i < 8; ++i) mbar_init(&ublk[i], 1);
    fence_mbar_init();
  }
  if (threadIdx.x == 32) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmP);
  }
  if (warp == 2) tmem_alloc(tmem_holder, kF1TmemCols);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // every CTA's barriers are initialised before any remote arrive / st.async
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();
  pdl_trigger();
  TraceScope _trace(1);
  const uint32_t e = ld_acquire_gpu(a.dev_epoch) + 1u;
  const int d0 = static_cast<int>(q) * a.Dq;  // first feature column of this CTA's part
  if ((a.debug & 1) && threadIdx.x == 0 && blockIdx.x < 160) g_f1_cta[blockIdx.x * 5 + 1] = gtime_ns();

  // Schedule: G1 of tile p streams through ring 1 (from HBM); G2 of tile p - 1 re-reads its
  // W part through ring 2 (from L2, one period after G1 brought it in); the MMA issuer
  // interleaves G2 blocks between G1 chunk pairs as soon as tile p - 1's epilogue has
  // published P~.  Separate rings let the HBM stream keep all of ring 1 in flight while the
  // short-latency L2 re-reads cycle through the small ring 2.
  if (warp == 0 || warp == 3) {
    // ===================== TMA producers: warp 0 -> ring 1 (G1), warp 3 -> ring 2 (G2) =====
    if (lane == 0) {
      // only ring 1 carries X (the gathered rows); ring 2 re-reads the local W_r.  Fused gather:
      // the first S1 slots get their W chunk at once and their X chunk after the wait.
      // (no lambdas / arrays here: captured or indexed locals would live in local memory and
      // measurably slowed the issue loop; the deferred slots are simply slots 0 .. ndef - 1,
      // and slot i's X chunk is chunk i % KQ)
      bool x_ready = warp == 3 || a.wait_flags == nullptr;
      if (!x_ready && !a.gather_on) {
        for (int p = 0; p < a.wait_count; ++p) wait_flag_geq(a.wait_flags + p, e * a.wait_mult, a.err, ERR_COMM | ERR_AT_GATHER);
        fence_proxy_async_global();
        x_ready = true;
      }
      int ndef = 0;
      // L2 policy: G1 reads keep their lines (evict_last) until G2 re-reads them two periods
      // later (evict_first: last use), so DRAM sees W_r once
      const uint64_t keep = l2_policy_evict_last(), drop = l2_policy_evict_first();
      const bool dbg = (a.debug & 1) && blockIdx.x == 0 && warp == 0;
      int stage = 0;
      uint32_t phase = 0;
      if (warp == 0) {
        for (int it = 0; it < my_tiles; ++it) {
          if (dbg && it < 64) g_f1_ts[it * 16 + 7] = gtime_ns();
          const int row0 = (cl + it * ncl) * kF1TileC;
          for (int k = 0; k < KQ; ++k) {
            if (!x_ready && ndef == S1) {  // ring full of slots waiting for X: the gathered rows
              for (int p = 0; p < a.wait_count; ++p) wait_flag_geq(a.wait_flags + p, e * a.wait_mult, a.err, ERR_COMM | ERR_AT_GATHER);
              fence_proxy_async_global();
              x_ready = true;
              for (int i = 0; i < ndef; ++i)
                tma_load_2d(ring1 + i * kF1G1SlotBytes + kF1StageBytes, &tmX, &full1[i], d0 + (i % KQ) * 64, 0);
            }
            mbar_wait(&empty1[stage], phase ^ 1u);
            uint8_t* slot = ring1 + stage * kF1G1SlotBytes;
            mbar_arrive_expect_tx(&full1[stage], kF1StageBytes + kF1XChunkBytes);
            tma_load_2d_hint(slot, &tmW, &full1[stage], d0 + k * 64, row0, keep);
            if (x_ready) tma_load_2d(slot + kF1StageBytes, &tmX, &full1[stage], d0 + k * 64, 0);
            else ++ndef;  // slot ndef (= stage), chunk k: X after the gather flags
            if (++stage == S1) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
        if (!x_ready) {  // fewer chunks than slots
          for (int p = 0; p < a.wait_count; ++p) wait_flag_geq(a.wait_flags + p, e * a.wait_mult, a.err, ERR_COMM | ERR_AT_GATHER);
          fence_proxy_async_global();
          for (int i = 0; i < ndef; ++i)
            tma_load_2d(ring1 + i * kF1G1SlotBytes + kF1StageBytes, &tmX, &full1[i], d0 + (i % KQ) * 64, 0);
        }
      } else if (!WHALE_SKIP(a.debug & 2)) {  // debug bit 2: timing experiment without G2
        for (int it = 0; it < my_tiles; ++it) {
          const int row0 = (cl + it * ncl) * kF1TileC;
          for (int m = 0; m < KQ / 2; ++m) {
            mbar_wait(&empty2[stage], phase ^ 1u);
            uint8_t* slot = ring2 + stage * kF1G2SlotBytes;
            mbar_arrive_expect_tx(&full2[stage], 2 * kF1StageBytes);
            tma_load_2d_hint(slot, &tmW, &full2[stage], d0 + (2 * m) * 64, row0, drop);
            tma_load_2d_hint(slot + kF1StageBytes, &tmW, &full2[stage], d0 + (2 * m + 1) * 64, row0, drop);
            if (++stage == a.s2) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1 || (warp == 2 && a.split_issue)) {
    // ===================== MMA issuer(s) =====================
    // split_issue: warp 1 issues G1 only and warp 2 (the TMEM allocator, idle otherwise) G2
    // only, so a G2 block waiting on its L2 re-read never holds back the G1 stream from HBM
    // (tcgen05.commit tracks the issuing thread's MMAs; G1 and G2 touch disjoint TMEM / smem).
    if (lane == 0) {
      const uint32_t idesc1 = umma_idesc(kF1TileC, kF1NB, false, false, 1u);
      const uint32_t idesc2 = umma_idesc(128, kF1NB, true, false, 1u);
      int s1 = 0, s2 = 0;
      uint32_t ph1 = 0, ph2 = 0;
      const uint32_t r1 = smem_u32(ring1), r2 = smem_u32(ring2), p_s = smem_u32(pbuf);
      const bool dbg = (a.debug & 1) && blockIdx.x == 0;
      auto g2_block = [&](int j, int i) {  // one G2 block: U^T[128 D rows of block i] += W^T P~_j^T
        mbar_wait(&full2[s2], ph2);
        tc_fence_after();
        const uint32_t aS = r2 + s2 * kF1G2SlotBytes;
        const uint32_t bS = p_s + (j & 1) * kF1PBytes;
#pragma unroll
        for (int kk = 0; kk < kF1TileC / 16; ++kk) {
          const uint64_t ad = umma_sdesc(aS + kk * 2048, kF1StageBytes, 1024);  // MN-major: 16 class rows / step
          const uint64_t bd = umma_sdesc(bS + (kk >> 2) * (kF1NB * kRowBytes) + (kk & 3) * 32, 16, 1024);
          umma_bf16(tmem_base + ucol0 + i * kF1NB, ad, bd, idesc2, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&empty2[s2]);
        if (j == my_tiles - 1) umma_commit(&ublk[i]);  // U block i is final: the epilogue writes it out
        if (++s2 == a.s2) {
          s2 = 0;
          ph2 ^= 1u;
        }
      };
      if (a.split_issue) {
        if (warp == 1) {
          for (int p = 0; p < my_tiles; ++p) {
            if (dbg && p < 64) g_f1_ts[p * 16 + 0] = gtime_ns();
            const int zb = p % 3;
            mbar_wait(&zempty[zb], ((p / 3) & 1) ^ 1u);
            tc_fence_after();
            for (int k = 0; k < KQ; ++k) {
              mbar_wait(&full1[s1], ph1);
              tc_fence_after();
              const uint32_t aS = r1 + s1 * kF1G1SlotBytes;
              const uint32_t bS = aS + kF1StageBytes;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                umma_bf16(tmem_base + zb * kF1NB, umma_sdesc(aS + kk * 32, 16, 1024), umma_sdesc(bS + kk * 32, 16, 1024),
                          idesc1, (k > 0 || kk > 0) ? 1u : 0u);
              umma_commit(&empty1[s1]);
              if (++s1 == S1) {
                s1 = 0;
                ph1 ^= 1u;
              }
            }
            umma_commit(&zfull[zb]);
            if (dbg && p < 64) g_f1_ts[p * 16 + 1] = gtime_ns();
          }
        } else {
          for (int j = 0; j < my_tiles; ++j) {
            mbar_wait(&pfull[j & 1], static_cast<uint32_t>((j >> 1) & 1));  // P~_j^T in smem, U rescaled
            tc_fence_after();
            if (WHALE_SKIP(a.debug & 2)) {  // timing experiment without G2: keep the P~ protocol alive
              mbar_arrive(&pempty[j & 1]);
              continue;
            }
            for (int i = 0; i < KQ / 2; ++i) g2_block(j, i);
            umma_commit(&pempty[j & 1]);
            if (dbg && j < 64) g_f1_ts[j * 16 + 2] = gtime_ns();
          }
        }
      } else
      // Period p: G1 of tile p, with G2 of tile p - 1 interleaved (one block per G1 chunk pair)
      // as soon as that tile's epilogue has published P~, and drained at the period end -- so
      // G2 re-reads W about one period after G1 brought it into L2 (short reuse distance).
      // G2 order, and hence U's summation order, is fixed.
      for (int p = 0; p <= my_tiles; ++p) {
        const bool has1 = p < my_tiles, has2 = p >= 1 && !WHALE_SKIP(a.debug & 2);
        if (dbg && p < 64) g_f1_ts[p * 16 + 0] = gtime_ns();
        const int zb = p % 3;
        const int j = p - 1;  // G2 tile
        if (has1) {
          mbar_wait(&zempty[zb], ((p / 3) & 1) ^ 1u);
          tc_fence_after();
        }
        int g2_next = 0;
        bool g2_ready = false;
        const uint32_t pf = smem_u32(&pfull[(j + 2) & 1]);
        const uint32_t pf_par = static_cast<uint32_t>((j >> 1) & 1);
        for (int i = 0; i < KQ / 2 && has1; ++i) {
          for (int h = 0; h < 2; ++h) {
            const int k = 2 * i + h;
            mbar_wait(&full1[s1], ph1);
            tc_fence_after();
            const uint32_t aS = r1 + s1 * kF1G1SlotBytes;
            const uint32_t bS = aS + kF1StageBytes;
            if (WHALE_SKIP(a.debug & 8)) {  // timing experiment: consume the slot without MMAs
              mbar_arrive(&empty1[s1]);
            } else {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                umma_bf16(tmem_base + zb * kF1NB, umma_sdesc(aS + kk * 32, 16, 1024),
                          umma_sdesc(bS + kk * 32, 16, 1024), idesc1, (k > 0 || kk > 0) ? 1u : 0u);
              umma_commit(&empty1[s1]);
            }
            if (++s1 == S1) {
              s1 = 0;
              ph1 ^= 1u;
            }
          }
          if (i == KQ / 2 - 1) {
            if (WHALE_SKIP(a.debug & 8)) mbar_arrive(&zfull[zb]);
            else umma_commit(&zfull[zb]);
            if (dbg && p < 64) g_f1_ts[p * 16 + 1] = gtime_ns();
          }
          if (has2 && g2_next < KQ / 2) {
            if (!g2_ready && mbar_test(pf, pf_par)) {
              g2_ready = true;
              tc_fence_after();
            }
            if (g2_ready) g2_block(j, g2_next++);
          }
        }
        if (has2) {
          if (!g2_ready) {
            mbar_wait(&pfull[j & 1], pf_par);  // P~_j^T in smem (and U rescaled if needed)
            tc_fence_after();
          }
          while (g2_next < KQ / 2) g2_block(j, g2_next++);
          if (WHALE_SKIP(a.debug & 8)) mbar_arrive(&pempty[j & 1]);
          else umma_commit(&pempty[j & 1]);
        } else if (p >= 1) {  // debug bit 2: G2 skipped, keep the P~ buffer protocol alive
          mbar_wait(&pfull[j & 1], pf_par);
          mbar_arrive(&pempty[j & 1]);
        }
        if (dbg && p < 64) g_f1_ts[p * 16 + 2] = gtime_ns();
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: 8 warps, thread = (class row, 16 batch columns) ========
    // warp 4 + e: TMEM lane quadrant e % 4 (class rows), batch columns [16 (e / 4), + 16)
    const int et = threadIdx.x - 128;  // 0 .. 255
    const int ew = warp - 4;
    const int qd = ew & 3;
    const int c0 = (ew >> 2) * 16;      // first batch column of this thread
    const int cl_row = qd * 32 + lane;  // class within the tile = TMEM lane
    const bool store_role = (qd % kF1KC) == static_cast<int>(q);  // one CTA stores each class row
    constexpr float kL2e = 1.4426950408889634f;
    constexpr int kE = kF1EpiThreads;
    if (a.gather_on) {  // the fused bridge all-gather: this CTA's pieces, then one signal
      int n = 0;
      for (int part = static_cast<int>(blockIdx.x); part < a.gather.parts; part += static_cast<int>(gridDim.x), ++n)
        gather_copy(a.gather, part, et, kE);
      named_bar_sync(2, kE);
      if (et == 0 && n > 0) gather_signal(a.gather, n);
    }
    // N > 1: the gathered labels were stored by the peers' bridge_gather (generic stores +
    // fence.sc.sys + flag increments): acquire those flags before reading them (the producer
    // lanes' acquire does not order this thread's loads); the CTA barrier then orders the
    // other epilogue threads' label reads after it.
    if (a.wait_flags != nullptr && et == 0)
      for (int p = 0; p < a.wait_count; ++p) wait_flag_geq(a.wait_flags + p, e * a.wait_mult, a.err, ERR_COMM | ERR_AT_GATHER);
    named_bar_sync(2, kE);
    if (et < 32) {
      s_lab[et] = et < a.Bt ? a.labels[et] : -1;
      s_ref[et] = -INFINITY;
    }
    named_bar_sync(2, kE);
    const uint32_t lane_off = static_cast<uint32_t>(qd * 32) << 16;
    const uint32_t xfull_s = smem_u32(xfull), xempty_s = smem_u32(xempty);
    const uint32_t my_slot_row = smem_u32(recv) + cl_row * 128;
    for (int it = 0; it < my_tiles; ++it) {
      const int t = cl + it * ncl;
      const int zb = it % 3;
      const long long cls = static_cast<long long>(t) * kF1TileC + cl_row;  // shard-local class
      const bool valid = cls < a.C_r;
      const bool dbg = (a.debug & 1) && blockIdx.x == 0 && et == 0 && it < 64;
      if (WHALE_SKIP(a.debug & 4)) {  // timing experiment: epilogue does nothing
        mbar_wait(&zfull[zb], (it / 3) & 1);
        mbar_arrive(&zempty[zb]);
        if (it >= 2) mbar_wait(&pempty[it & 1], ((it >> 1) & 1) ^ 1u);
        mbar_arrive(&pfull[it & 1]);
        continue;
      }
      mbar_wait(&zfull[zb], (it / 3) & 1);
      if (dbg) g_f1_ts[it * 16 + 3] = gtime_ns();
      tc_fence_after();
      uint32_t v[16];
      tmem_ld16(tmem_base + zb * kF1NB + c0 + lane_off, v);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&zempty[zb]);
      // ---- all-reduce of the partial Z_t^T over the cluster (DSMEM), fixed rank order
      if (it > 0) mbar_wait(xempty, (it - 1) & 1);  // peers consumed my previous partial
#pragma unroll
      for (uint32_t p = 0; p < kF1KC; ++p) {
        if (p == q) continue;
        const uint32_t slot = q < p ? q : q - 1;  // my slot in p's receive buffer
        const uint32_t dst = mapa_smem(my_slot_row + slot * kF1SlotBytes, p);
        const uint32_t bar = mapa_smem(xfull_s, p);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int ch = (c0 >> 2) + c;
          st_async_v4(dst + ((ch ^ (cl_row & 7)) << 4), bar, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        }
      }
      if (et == 0) mbar_arrive_expect_tx(xfull, (kF1KC - 1) * kF1SlotBytes);
      mbar_wait(xfull, it & 1);  // st.async data is visible once its complete_tx lands
      if (dbg) g_f1_ts[it * 16 + 4] = gtime_ns();
      float z[16];
#pragma unroll
      for (uint32_t src = 0; src < kF1KC; ++src) {
        float pv[16];
        if (src == q) {
#pragma unroll
          for (int j = 0; j < 16; ++j) pv[j] = __uint_as_float(v[j]);
        } else {
          const uint32_t slot = src < q ? src : src - 1;
          const uint8_t* row = recv + slot * kF1SlotBytes + cl_row * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int ch = (c0 >> 2) + c;
            const float4 f = *reinterpret_cast<const float4*>(row + ((ch ^ (cl_row & 7)) << 4));
            pv[4 * c] = f.x;
            pv[4 * c + 1] = f.y;
            pv[4 * c + 2] = f.z;
            pv[4 * c + 3] = f.w;
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = src == 0 ? pv[j] : z[j] + pv[j];
      }
      named_bar_sync(2, kE);  // every thread has read the receive buffer
      if (et < kF1KC && et != static_cast<int>(q)) mbar_arrive_remote(mapa_smem(xempty_s, et));
      if (a.bias != nullptr && valid) {
        const float bv = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.bias)[cls]);
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] += bv;
      }
      // ---- per-row tile max and top-1 class (ties -> lowest class): one redux per row; lane jj
      //      keeps row c0 + jj's result (selects, no branches)
      float my_m = -INFINITY;
      int my_i = 0;
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const float zv = valid ? z[jj] : -INFINITY;
        const float m = redux_max_f32(zv);
        const unsigned hit = __ballot_sync(0xffffffffu, zv == m);
        my_m = lane == jj ? m : my_m;
        my_i = lane == jj ? static_cast<int>(__ffs(hit)) - 1 : my_i;
      }
      if (lane < 16) {
        red_v[qd][c0 + lane] = my_m;
        red_i[qd][c0 + lane] = qd * 32 + my_i;
      }
      if (et == 0 && it >= 2) bulk_wait_read<1>();  // the P~ store of tile it - 2 has read its buffer
      named_bar_sync(2, kE);
      if (dbg) g_f1_ts[it * 16 + 8] = gtime_ns();
      if (et < 32) {
        float bm = red_v[0][et];
        int bi = red_i[0][et];
#pragma unroll
        for (int w = 1; w < 4; ++w) {
          const float cv = red_v[w][et];
          const int ci = red_i[w][et];
          if (cv > bm || (cv == bm && ci < bi)) {
            bm = cv;
            bi = ci;
          }
        }
        const float old = s_ref[et];
        const bool first = it == 0;
        const bool move = first || (bm - old) * kL2e > kF1Tau;
        const float nref = move ? bm : old;
        s_fac[et] = (move && !first) ? exp2f((old - nref) * kL2e) : 1.f;
        s_ref[et] = nref;
        s_max[et] = bm;
        s_arg[et] = bi;
        const unsigned any = __ballot_sync(0xffffffffu, move && !first);
        if (et == 0) s_rescale = any != 0u;
      }
      named_bar_sync(2, kE);
      if (dbg) g_f1_ts[it * 16 + 9] = gtime_ns();
      // ---- U rescale when a reference moved: G2(it - 1) must have finished (G2(it) waits for
      //      this tile's pfull); then the P~ buffer of G2(it - 2) must be free
      if (s_rescale) {
        mbar_wait(&pempty[(it - 1) & 1], ((it - 1) >> 1) & 1);
        tc_fence_after();
        for (int m = 0; m < KQ / 2; ++m) {
          uint32_t u[16];
          const uint32_t ta = tmem_base + ucol0 + m * kF1NB + c0 + lane_off;
          tmem_ld16(ta, u);
          tmem_ld_wait();
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) u[jj] = __float_as_uint(__uint_as_float(u[jj]) * s_fac[c0 + jj]);
          tmem_st16(ta, u);
        }
        tmem_st_wait();
      }
      if (it >= 2) mbar_wait(&pempty[it & 1], ((it >> 1) & 1) ^ 1u);
      if (dbg) g_f1_ts[it * 16 + 10] = gtime_ns();
      // ---- P~ = exp(z - ref) -> G2 operand (also the global P~ tile, stored by TMA); s_tile
      float rf[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 r4 = *reinterpret_cast<const float4*>(&s_ref[c0 + 4 * c]);
        rf[4 * c] = r4.x;
        rf[4 * c + 1] = r4.y;
        rf[4 * c + 2] = r4.z;
        rf[4 * c + 3] = r4.w;
      }
      float ps[16];
      uint8_t* pb = pbuf + (it & 1) * kF1PBytes;
      uint8_t* prow = pb + (cl_row >> 6) * (kF1NB * kRowBytes);
      const int cb = (cl_row & 63) * 2;  // byte column within the 128-byte row
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int j = c0 + jj;
        const float pr = valid ? ex2_approx((z[jj] - rf[jj]) * kL2e) : 0.f;
        ps[jj] = pr;
        *reinterpret_cast<__nv_bfloat16*>(prow + j * 128 + ((((cb >> 4) ^ (jj & 7)) << 4) | (cb & 15))) =
            __float2bfloat16_rn(pr);
      }
      if (store_role && valid) {  // the label logit (rows whose label falls in this tile)
#pragma unroll
        for (int jj = 0; jj < 16; ++jj)
          if (c0 + jj < a.Bt && static_cast<long long>(s_lab[c0 + jj]) - a.class_offset == cls) a.zy[c0 + jj] = z[jj];
      }
      if (dbg) g_f1_ts[it * 16 + 11] = gtime_ns();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&pfull[it & 1]);
      if (dbg) g_f1_ts[it * 16 + 5] = gtime_ns();
      // column sums over the warp's 32 class rows: lanes l and l ^ 16 first, then a transposed
      // reduction over 16 columns -> lane l (< 16) holds column c0 + l
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) ps[jj] += __shfl_xor_sync(0xffffffffu, ps[jj], 16);
#pragma unroll
      for (int w = 8; w >= 1; w >>= 1) {
        const bool hi = (lane & w) != 0;
#pragma unroll
        for (int i = 0; i < w; ++i) {
          const float sv = hi ? ps[i] : ps[i + w];
          const float kv = hi ? ps[i + w] : ps[i];
          ps[i] = kv + __shfl_xor_sync(0xffffffffu, sv, w);
        }
      }
      if (lane < 16) red_v[qd][c0 + lane] = ps[0];
      named_bar_sync(2, kE);
      if (et == 0) {  // this CTA's 64-class half of the P~ tile -> global (rows >= B_tot clipped)
        tma_store_2d(&tmP, pb + q * (kF1NB * kRowBytes), t * kF1TileC + static_cast<int>(q) * 64, 0);
        bulk_commit();
      }
      if (q == 0 && et < a.Bt) {
        const float s = (red_v[0][et] + red_v[1][et]) + (red_v[2][et] + red_v[3][et]);
        const size_t o = static_cast<size_t>(et) * a.num_tiles + t;
        a.m_tile[o] = s_ref[et];  // P~ and s_tile are relative to the reference
        a.s_tile[o] = s;
        a.mx_tile[o] = s_max[et];  // true tile max (predictions)
        if (a.a_tile) a.a_tile[o] = static_cast<int32_t>(a.class_offset + static_cast<long long>(t) * kF1TileC + s_arg[et]);
      }
      named_bar_sync(2, kE);  // red_v is reused by the next tile
      if (dbg) g_f1_ts[it * 16 + 6] = gtime_ns();
    }
    // ---- this CTA's part of U (relative to s_ref) -> global partials (lanes: consecutive d,
    //      128-byte warp stores; staging the 128 KB in smem for 1-D bulk copies measured slower)
    //      Block m is written as soon as the last tile's G2 block m has completed (ublk[m]),
    //      so the write-out overlaps the remaining G2 blocks of the last tile.
    const size_t ubase = static_cast<size_t>(cl) * a.Bt;
    for (int m = 0; m < KQ / 2; ++m) {
      uint32_t u[16];
      if (my_tiles > 0) {
        if (!WHALE_SKIP(a.debug & 2)) mbar_wait(&ublk[m], 0u);
        tc_fence_after();
        tmem_ld16(tmem_base + ucol0 + m * kF1NB + c0 + lane_off, u);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) u[jj] = 0u;
      }
      const int d = d0 + m * 128 + cl_row;
#pragma unroll
      for (int jj = 0; jj < 16; ++jj)
        if (c0 + jj < a.Bt) __stcg(a.upart + (ubase + c0 + jj) * a.D + d, __uint_as_float(u[jj]));
    }
    if (q == 0 && et < a.Bt) a.uref[ubase + et] = s_ref[et];
    if (et == 0) bulk_wait<0>();
    if (a.debug & 32) __threadfence();  // timing experiment: drain the stores before the end stamp
    // the peers' last remote operation on this CTA's shared memory is their "consumed"
    // arrive for the last tile's partial: once it has landed nothing targets this CTA
    if (my_tiles > 0 && !WHALE_SKIP(a.debug & 4)) mbar_wait(xempty, (my_tiles - 1) & 1);
  }
  // debug timeline: the exit stamps are kept in registers and stored together at the end (a
  // store between two timer reads would time its own issue stall)
  const unsigned long long t_pre = (a.debug & 1) ? gtime_ns() : 0ull;
  tc_fence_before();
  __syncthreads();
  const unsigned long long t_end = (a.debug & 1) ? gtime_ns() : 0ull;
  // no CTA leaves while a peer may still write into its shared memory: every remote write
  // into this CTA was awaited above (Z partials via xfull, the consumed arrives via xempty),
  // so the exit barrier orders nothing else and needs no release (no MEMBAR: the .release
  // form waited ~12 us for the U write-out to drain)
  if (!(a.debug & 64)) cluster_sync_relaxed();
  const unsigned long long t_sync = (a.debug & 1) ? gtime_ns() : 0ull;
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kF1TmemCols);
  }
  if ((a.debug & 1) && threadIdx.x == 0 && blockIdx.x < 160) {
    g_f1_cta[blockIdx.x * 5 + 2] = t_end;
    g_f1_cta[blockIdx.x * 5 + 3] = t_sync;
    g_f1_cta[blockIdx.x * 5 + 4] = t_pre;  // thread 0 (TMA producer) reached the exit sync
  }
}

// dX = (1/B_tot) (sum_cl e^{uref[cl] - lse} U_cl - W_{y}) for this shard: N = 1 writes dX,
// N > 1 pushes the rows into their owners' fp32 receive slabs (reduce-scatter, as FIX_PUSH).
struct RowSplit {
  int off[kMaxRanks + 1];
};
template <int ES>
__global__ void __launch_bounds__(256) dx_combine_kernel(const float* __restrict__ upart, const float* __restrict__ uref,
                                                         int ncl, int Bt, int D, const float* __restrict__ lse,
                                                         const int32_t* __restrict__ y, long long o_r, long long C_r,
                                                         const void* __restrict__ w, float inv_bt, void* dx_out,
                                                         PeerPtrs recv, RowSplit rows, int rank, int world, int Bslab,
                                                         const float* grad_scale) {
  // block = 8 cluster groups x 32 float4 columns of one row b; group g sums clusters
  // g, g + 8, ... and the 8 group sums are added in group order (deterministic)
  constexpr int kG = 8, kCols = 32;
  __shared__ float fac[160];
  __shared__ float4 part[kG][kCols];
  pdl_wait();
  pdl_trigger();
  TraceScope _trace(5);
  const int b = blockIdx.y;
  const float l = lse[b];
  for (int i = threadIdx.x; i < ncl; i += blockDim.x) fac[i] = __expf(uref[static_cast<size_t>(i) * Bt + b] - l);
  __syncthreads();
  const int g = threadIdx.x / kCols, cx = threadIdx.x % kCols;
  const int d = (blockIdx.x * kCols + cx) * 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (d < D) {
    const float* src = upart + static_cast<size_t>(b) * D + d;
    const size_t cstride = static_cast<size_t>(Bt) * D;
    for (int i = g; i < ncl; i += kG) {
      const float4 u = __ldcg(reinterpret_cast<const float4*>(src + i * cstride));
      const float f = fac[i];
      acc.x = fmaf(f, u.x, acc.x);
      acc.y = fmaf(f, u.y, acc.y);
      acc.z = fmaf(f, u.z, acc.z);
      acc.w = fmaf(f, u.w, acc.w);
    }
  }
  part[g][cx] = acc;
  __syncthreads();
  if (g == 0 && d < D) {
#pragma unroll
    for (int k = 1; k < kG; ++k) {
      acc.x += part[k][cx].x;
      acc.y += part[k][cx].y;
      acc.z += part[k][cx].z;
      acc.w += part[k][cx].w;
    }
    const long long lab = static_cast<long long>(y[b]) - o_r;
    if (lab >= 0 && lab < C_r) {  // the one-hot term, on the shard that owns the label
      const uint2 raw = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(w) + lab * D + d);
      const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
      const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
      acc.x -= w01.x;
      acc.y -= w01.y;
      acc.z -= w23.x;
      acc.w -= w23.y;
    }
    const float f = inv_bt * (grad_scale ? __ldg(grad_scale) : 1.f);
    acc.x *= f;
    acc.y *= f;
    acc.z *= f;
    acc.w *= f;
    if (world == 1) {
      uint2 o;
      o.x = pack_bf16x2(acc.x, acc.y);
      o.y = pack_bf16x2(acc.z, acc.w);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(dx_out) + static_cast<size_t>(b) * D + d) = o;
    } else {
      int owner = 0;
#pragma unroll
      for (int r = 1; r < kMaxRanks; ++r)
        if (r < world && rows.off[r] <= b) owner = r;
      float* dst = reinterpret_cast<float*>(recv.p[owner]) +
                   (static_cast<size_t>(rank) * Bslab + (b - rows.off[owner])) * D + d;
      *reinterpret_cast<float4*>(dst) = acc;  // NVLink store into the owner's slab
    }
  }
  if (world > 1) __threadfence_system();
}

}  // namespace whale
