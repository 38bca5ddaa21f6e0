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
// The per-(row, tile) statistics written for the rest of the pipeline are the same as the
// logits GEMM's EPI_FWD_STATS epilogue: m_tile = tile max, s_tile = sum exp(z - m_tile),
// P~ = exp(z - m_tile) in bf16 (the backward's dW operand), z_y, a_tile (top-1 class).
//
//   warp 0      TMA producer (one lane): X part once (resident), then W chunks in MMA order
//   warp 1      MMA issuer (one lane):   period p = G1(p) interleaved with G2(p - 2)
//   warp 2      TMEM allocator (512 columns: Z x 2 and U blocks x D_q/128, 32 columns each)
//   warps 4..7  epilogue: thread = class row of the tile (TMEM lane)
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
constexpr float kF1Tau = 8.0f;  // lazy rescale threshold, log2 units

struct F1Args {
  int Bt;                  // valid rows (<= 32)
  int D, Dq;               // feature dim, D / KC (multiple of 128, <= 1024)
  int C_r;                 // classes of this shard
  int num_tiles;           // ceil(C_r / 128) = T
  int stages;              // W ring stages (even)
  long long class_offset;  // o_r
  const int32_t* labels;   // [Bt] global class ids
  const void* bias;        // [C_r] bf16 or NULL
  float* m_tile;           // [Bt x T]
  float* s_tile;           // [Bt x T]
  float* zy;               // [Bt]
  int32_t* a_tile;         // [Bt x T] global class id of the tile's max, or NULL
  __nv_bfloat16* P;        // P~ [Bt x ldp]
  long long ldp;
  float* upart;            // [ncl x Bt x D] per-cluster U (relative to uref)
  float* uref;             // [ncl x Bt]
  const uint32_t* wait_flags;  // N > 1: gather flags (as GemmArgs)
  int wait_count;
  uint32_t wait_mult;
  uint32_t* dev_epoch;
  int* err;
  int debug;               // timing experiments: bit 0 = record a per-period timeline of CTA 0,
                           // bit 1 = skip G2 (dX wrong)
};

// Debug timeline (CTA 0): [period][8] globaltimer stamps, see splitfc_fwd_dx_kernel.
__device__ unsigned long long g_f1_ts[64 * 8];

__host__ __device__ constexpr int f1_smem_bytes(int stages, int Dq) {
  return 1024 + stages * kF1StageBytes + (Dq / 64) * kF1XChunkBytes + (kF1KC - 1) * kF1SlotBytes + 2 * kF1PBytes + 240;
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

__global__ void __launch_bounds__(kGemmThreads, 1)
    splitfc_fwd_dx_kernel(const __grid_constant__ CUtensorMap tmW /*box {64, 128}*/,
                          const __grid_constant__ CUtensorMap tmX /*box {64, 32}*/, const F1Args a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ float red_v[4][32];
  __shared__ int red_i[4][32];
  __shared__ float s_ref[32], s_c[32], s_fac[32], s_max[32];
  __shared__ int s_arg[32], s_lab[32];
  __shared__ int s_rescale;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int KQ = a.Dq / 64;  // 64-wide D chunks of this CTA's part
  uint8_t* ring = smem;
  uint8_t* xres = ring + a.stages * kF1StageBytes;
  uint8_t* recv = xres + KQ * kF1XChunkBytes;
  uint8_t* pbuf = recv + (kF1KC - 1) * kF1SlotBytes;  // 2 buffers
  uint64_t* full = reinterpret_cast<uint64_t*>(pbuf + 2 * kF1PBytes);
  uint64_t* empty = full + a.stages;
  uint64_t* zfull = empty + a.stages;  // 3 Z buffers
  uint64_t* zempty = zfull + 3;
  uint64_t* pfull = zempty + 3;        // 2 P~ buffers
  uint64_t* pempty = pfull + 2;        // completes when G2 of that buffer's tile finished
  uint64_t* xbar = pempty + 2;
  uint64_t* xfull = xbar + 1;
  uint64_t* xempty = xfull + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(xempty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t q = cluster_ctarank();
  const int cl = static_cast<int>(cluster_id_x());
  const int ncl = static_cast<int>(ncluster_x());
  const int my_tiles = cl < a.num_tiles ? (a.num_tiles - 1 - cl) / ncl + 1 : 0;
  const uint32_t ucol0 = 3 * kF1NB;  // TMEM: Z buffers at 0, 32, 64; U blocks from 96

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&zfull[i], 1);
      mbar_init(&zempty[i], 128);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&pfull[i], 128);
      mbar_init(&pempty[i], 1);
    }
    mbar_init(xbar, 1);
    mbar_init(xfull, 1);
    mbar_init(xempty, kF1KC - 1);
    fence_mbar_init();
  }
  if (threadIdx.x == 32) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
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

  // Schedule (producer and MMA walk the same sequence): period p streams G1 of tile p from
  // HBM interleaved with G2 of tile p - 2 from L2, in units of [G1 chunk pair, G2 block]
  // (a G2 block = the two chunks of 128 D rows).  The lag of two periods gives every tile's
  // epilogue a whole period before its P~ is needed, so neither stream waits on it.
  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      if (a.wait_flags != nullptr) {
        for (int p = 0; p < a.wait_count; ++p) wait_flag_geq(a.wait_flags + p, e * a.wait_mult, a.err, 8);
        fence_proxy_async_global();
      }
      mbar_arrive_expect_tx(xbar, static_cast<uint32_t>(KQ * kF1XChunkBytes));
      for (int k = 0; k < KQ; ++k) tma_load_2d(xres + k * kF1XChunkBytes, &tmX, xbar, d0 + k * 64, 0);
      int stage = 0;
      uint32_t phase = 0;
      // L2 policy: G1 reads keep their lines (evict_last) until G2 re-reads them two periods
      // later (evict_first: last use), so DRAM sees W_r once
      const uint64_t keep = l2_policy_evict_last(), drop = l2_policy_evict_first();
      auto load_w = [&](int it, int k, uint64_t pol) {
        mbar_wait(&empty[stage], phase ^ 1u);
        mbar_arrive_expect_tx(&full[stage], kF1StageBytes);
        tma_load_2d_hint(ring + stage * kF1StageBytes, &tmW, &full[stage], d0 + k * 64, (cl + it * ncl) * kF1TileC,
                         pol);
        if (++stage == a.stages) {
          stage = 0;
          phase ^= 1u;
        }
      };
      const bool dbg = (a.debug & 1) && blockIdx.x == 0;
      for (int p = 0; p < my_tiles + 2; ++p) {
        if (dbg && p < 64) g_f1_ts[p * 8 + 7] = gtime_ns();
        for (int i = 0; i < KQ / 2; ++i) {
          if (p < my_tiles) {
            load_w(p, 2 * i, keep);
            load_w(p, 2 * i + 1, keep);
          }
          if (p >= 2 && !(a.debug & 2)) {  // debug bit 2: timing experiment without G2
            load_w(p - 2, 2 * i, drop);
            load_w(p - 2, 2 * i + 1, drop);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc1 = umma_idesc(kF1TileC, kF1NB, false, false, 1u);
      const uint32_t idesc2 = umma_idesc(128, kF1NB, true, false, 1u);
      mbar_wait(xbar, 0);
      tc_fence_after();
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t ring_s = smem_u32(ring), x_s = smem_u32(xres), p_s = smem_u32(pbuf);
      const bool dbg = (a.debug & 1) && blockIdx.x == 0;
      for (int p = 0; p < my_tiles + 2; ++p) {
        const bool has1 = p < my_tiles, has2 = p >= 2;
        if (dbg && p < 64) g_f1_ts[p * 8 + 0] = gtime_ns();
        const int zb = p % 3;
        const int j = p - 2;  // G2 tile
        if (has1) {
          mbar_wait(&zempty[zb], ((p / 3) & 1) ^ 1u);
          tc_fence_after();
        }
        if (has2) {
          mbar_wait(&pfull[j & 1], (j >> 1) & 1);  // P~_j^T in smem (and U rescaled if needed)
          tc_fence_after();
        }
        for (int i = 0; i < KQ / 2; ++i) {
          if (has1) {
            for (int h = 0; h < 2; ++h) {
              const int k = 2 * i + h;
              mbar_wait(&full[stage], phase);
              tc_fence_after();
              const uint32_t aS = ring_s + stage * kF1StageBytes;
              const uint32_t bS = x_s + k * kF1XChunkBytes;
              if (a.debug & 8) {  // timing experiment: consume the stage without MMAs
                mbar_arrive(&empty[stage]);
              } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  umma_bf16(tmem_base + zb * kF1NB, umma_sdesc(aS + kk * 32, 16, 1024),
                            umma_sdesc(bS + kk * 32, 16, 1024), idesc1, (k > 0 || kk > 0) ? 1u : 0u);
                umma_commit(&empty[stage]);
              }
              if (++stage == a.stages) {
                stage = 0;
                phase ^= 1u;
              }
            }
            if (i == KQ / 2 - 1) {
              if (a.debug & 8) mbar_arrive(&zfull[zb]);
              else umma_commit(&zfull[zb]);
              if (dbg && p < 64) g_f1_ts[p * 8 + 1] = gtime_ns();
            }
          }
          if (has2 && !(a.debug & 2)) {
            const int s0 = stage;  // even (ring size and every unit are even)
            mbar_wait(&full[s0], phase);
            mbar_wait(&full[s0 + 1], phase);
            tc_fence_after();
            const uint32_t aS = ring_s + s0 * kF1StageBytes;
            const uint32_t bS = p_s + (j & 1) * kF1PBytes;
#pragma unroll
            for (int kk = 0; kk < kF1TileC / 16; ++kk) {
              const uint64_t ad = umma_sdesc(aS + kk * 2048, kF1StageBytes, 1024);  // MN-major: 16 class rows / step
              const uint64_t bd = umma_sdesc(bS + (kk >> 2) * (kF1NB * kRowBytes) + (kk & 3) * 32, 16, 1024);
              umma_bf16(tmem_base + ucol0 + i * kF1NB, ad, bd, idesc2, (j > 0 || kk > 0) ? 1u : 0u);
            }
            umma_commit(&empty[s0]);
            umma_commit(&empty[s0 + 1]);
            stage += 2;
            if (stage == a.stages) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
        if (has2) {
          if (a.debug & 8) mbar_arrive(&pempty[j & 1]);
          else umma_commit(&pempty[j & 1]);
        }
        if (dbg && p < 64) g_f1_ts[p * 8 + 2] = gtime_ns();
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: thread = class row of the tile =====================
    const int et = threadIdx.x - 128;
    const int qd = warp & 3;
    const int cl_row = qd * 32 + lane;  // class within the tile = TMEM lane
    const bool store_role = (qd % kF1KC) == static_cast<int>(q);  // one CTA stores each class row
    constexpr float kL2e = 1.4426950408889634f;
    if (et < 32) {
      s_lab[et] = et < a.Bt ? a.labels[et] : -1;
      s_ref[et] = -INFINITY;
    }
    named_bar_sync(2, 128);
    const uint32_t lane_off = static_cast<uint32_t>(qd * 32) << 16;
    const uint32_t xfull_s = smem_u32(xfull), xempty_s = smem_u32(xempty);
    const uint32_t my_slot_row = smem_u32(recv) + cl_row * 128;
    for (int it = 0; it < my_tiles; ++it) {
      const int t = cl + it * ncl;
      const int zb = it % 3;
      const long long cls = static_cast<long long>(t) * kF1TileC + cl_row;  // shard-local class
      const bool valid = cls < a.C_r;
      const bool dbg = (a.debug & 1) && blockIdx.x == 0 && et == 0 && it < 64;
      if (a.debug & 4) {  // timing experiment: epilogue does nothing
        mbar_wait(&zfull[zb], (it / 3) & 1);
        mbar_arrive(&zempty[zb]);
        if (it >= 2) mbar_wait(&pempty[it & 1], ((it >> 1) & 1) ^ 1u);
        mbar_arrive(&pfull[it & 1]);
        continue;
      }
      mbar_wait(&zfull[zb], (it / 3) & 1);
      if (dbg) g_f1_ts[it * 8 + 3] = gtime_ns();
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(tmem_base + zb * kF1NB + lane_off, v);
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
        for (int ch = 0; ch < 8; ++ch)
          st_async_v4(dst + ((ch ^ (cl_row & 7)) << 4), bar, v[4 * ch], v[4 * ch + 1], v[4 * ch + 2], v[4 * ch + 3]);
      }
      if (et == 0) mbar_arrive_expect_tx(xfull, (kF1KC - 1) * kF1SlotBytes);
      mbar_wait(xfull, it & 1);  // st.async data is visible once its complete_tx lands
      if (dbg) g_f1_ts[it * 8 + 4] = gtime_ns();
      float z[32];
#pragma unroll
      for (uint32_t src = 0; src < kF1KC; ++src) {
        float pv[32];
        if (src == q) {
#pragma unroll
          for (int j = 0; j < 32; ++j) pv[j] = __uint_as_float(v[j]);
        } else {
          const uint32_t slot = src < q ? src : src - 1;
          const uint8_t* row = recv + slot * kF1SlotBytes + cl_row * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const float4 f = *reinterpret_cast<const float4*>(row + ((ch ^ (cl_row & 7)) << 4));
            pv[4 * ch] = f.x;
            pv[4 * ch + 1] = f.y;
            pv[4 * ch + 2] = f.z;
            pv[4 * ch + 3] = f.w;
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) z[j] = src == 0 ? pv[j] : z[j] + pv[j];
      }
      named_bar_sync(2, 128);  // every thread has read the receive buffer
      if (et < kF1KC && et != static_cast<int>(q)) mbar_arrive_remote(mapa_smem(xempty_s, et));
      if (a.bias != nullptr && valid) {
        const float bv = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.bias)[cls]);
#pragma unroll
        for (int j = 0; j < 32; ++j) z[j] += bv;
      }
      // ---- per-row tile max and top-1 class (ties -> lowest class): one redux per row
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float zv = valid ? z[j] : -INFINITY;
        const float m = redux_max_f32(zv);
        const unsigned hit = __ballot_sync(0xffffffffu, zv == m);
        if (lane == j) {
          red_v[qd][j] = m;
          red_i[qd][j] = qd * 32 + __ffs(hit) - 1;
        }
      }
      named_bar_sync(2, 128);
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
        s_c[et] = exp2f((nref - bm) * kL2e);  // exp(z - max) = exp(z - ref) * exp(ref - max)
        s_max[et] = bm;
        s_arg[et] = bi;
        const unsigned any = __ballot_sync(0xffffffffu, move && !first);
        if (et == 0) s_rescale = any != 0u;
      }
      named_bar_sync(2, 128);
      // ---- U rescale when a reference moved: G2(it - 1) must have finished (G2(it) waits for
      //      this tile's pfull); then the P~ buffer of G2(it - 2) must be free
      if (s_rescale) {
        mbar_wait(&pempty[(it - 1) & 1], ((it - 1) >> 1) & 1);
        tc_fence_after();
        for (int m = 0; m < KQ / 2; ++m) {
          uint32_t u[32];
          const uint32_t ta = tmem_base + ucol0 + m * kF1NB + lane_off;
          tmem_ld32(ta, u);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) u[j] = __float_as_uint(__uint_as_float(u[j]) * s_fac[j]);
          tmem_st32(ta, u);
        }
        tmem_st_wait();
      }
      if (it >= 2) mbar_wait(&pempty[it & 1], ((it >> 1) & 1) ^ 1u);
      // ---- P~ (reference) -> G2 operand; P~ (tile max) -> global; s_tile; z_y
      float ps[32];
      uint8_t* prow = pbuf + (it & 1) * kF1PBytes + (cl_row >> 6) * (kF1NB * kRowBytes);
      const int cb = (cl_row & 63) * 2;  // byte column within the 128-byte row
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float pr = valid ? ex2_approx((z[j] - s_ref[j]) * kL2e) : 0.f;
        *reinterpret_cast<__nv_bfloat16*>(prow + j * 128 + ((((cb >> 4) ^ (j & 7)) << 4) | (cb & 15))) =
            __float2bfloat16_rn(pr);
        const float pt = pr * s_c[j];
        ps[j] = pt;
        if (store_role && valid && j < a.Bt) {
          a.P[static_cast<long long>(j) * a.ldp + cls] = __float2bfloat16_rn(pt);
          if (static_cast<long long>(s_lab[j]) - a.class_offset == cls) a.zy[j] = z[j];
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&pfull[it & 1]);
      if (dbg) g_f1_ts[it * 8 + 5] = gtime_ns();
      f1_colsum32(ps, lane);
      red_v[qd][lane] = ps[0];
      named_bar_sync(2, 128);
      if (q == 0 && et < a.Bt) {
        const float s = (red_v[0][et] + red_v[1][et]) + (red_v[2][et] + red_v[3][et]);
        const size_t o = static_cast<size_t>(et) * a.num_tiles + t;
        a.m_tile[o] = s_max[et];
        a.s_tile[o] = s;
        if (a.a_tile) a.a_tile[o] = static_cast<int32_t>(a.class_offset + static_cast<long long>(t) * kF1TileC + s_arg[et]);
      }
      named_bar_sync(2, 128);  // red_v is reused by the next tile
      if (dbg) g_f1_ts[it * 8 + 6] = gtime_ns();
    }
    // ---- this CTA's part of U (relative to s_ref) -> global partials
    const size_t ubase = static_cast<size_t>(cl) * a.Bt;
    if (my_tiles > 0) {
      mbar_wait(&pempty[(my_tiles - 1) & 1], ((my_tiles - 1) >> 1) & 1);
      tc_fence_after();
    }
    for (int m = 0; m < KQ / 2; ++m) {
      uint32_t u[32];
      if (my_tiles > 0) {
        tmem_ld32(tmem_base + ucol0 + m * kF1NB + lane_off, u);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) u[j] = 0u;
      }
      const int d = d0 + m * 128 + cl_row;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < a.Bt) __stcg(a.upart + (ubase + j) * a.D + d, __uint_as_float(u[j]));
    }
    if (q == 0 && et < a.Bt) a.uref[ubase + et] = s_ref[et];
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while a peer may still write into its shared memory
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kF1TmemCols);
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
                                                         PeerPtrs recv, RowSplit rows, int rank, int world, int Bslab) {
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
    acc.x *= inv_bt;
    acc.y *= inv_bt;
    acc.z *= inv_bt;
    acc.w *= inv_bt;
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
