// Host side of the C-ABI (include/whale_splitfc.h): shard plan, workspace layout, tile
// configuration, TMA descriptors and the launch sequence of the split-FC forward/backward.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/whale_splitfc.h"
#include "gemm_sm100.cuh"
#include "bwd_sm100.cuh"
#include "fwd_dx_sm100.cuh"
#include "kernels_aux.cuh"

using namespace whale;

// ============================================================================ errors
static thread_local std::string g_last_error;

static whale_status_t fail(whale_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define CUDA_TRY(expr)                                                                         \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess)                                                                     \
      return fail(WHALE_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                  __LINE__);                                                                   \
  } while (0)

extern "C" const char* whale_last_error(void) { return g_last_error.c_str(); }

// ============================================================================ plan (A1)
// Hamilton / largest-remainder apportionment in exact integer arithmetic
// (SPEC.md:281).  Ties in the remainder go to the lower rank.
extern "C" whale_status_t whale_splitfc_plan(int64_t num_classes, int32_t world_size, const uint32_t* capacity,
                                             int64_t* shard_counts, int64_t* shard_offsets) {
  if (world_size < 1 || world_size > kMaxRanks)
    return fail(WHALE_ERR_INVALID_ARG, "world_size %d outside [1, %d]", world_size, kMaxRanks);
  if (num_classes < 1) return fail(WHALE_ERR_INVALID_ARG, "num_classes must be >= 1");
  if (!shard_counts || !shard_offsets) return fail(WHALE_ERR_INVALID_ARG, "NULL output array");
  const int N = world_size;
  __int128 wsum = 0;
  for (int i = 0; i < N; ++i) {
    const uint32_t w = capacity ? capacity[i] : 1u;
    if (w == 0) return fail(WHALE_ERR_INVALID_ARG, "capacity[%d] == 0 (weights must be > 0)", i);
    wsum += w;
  }
  if (num_classes < N) return fail(WHALE_ERR_UNSPLITTABLE, "C=%lld < world=%d", (long long)num_classes, N);
  int64_t q[kMaxRanks];
  __int128 rho[kMaxRanks];
  int64_t assigned = 0;
  for (int i = 0; i < N; ++i) {
    const __int128 num = static_cast<__int128>(num_classes) * (capacity ? capacity[i] : 1u);
    q[i] = static_cast<int64_t>(num / wsum);
    rho[i] = num % wsum;
    assigned += q[i];
  }
  int order[kMaxRanks];
  for (int i = 0; i < N; ++i) order[i] = i;
  std::stable_sort(order, order + N, [&](int a, int b) { return rho[a] > rho[b]; });  // ties: lower rank
  for (int64_t k = 0; k < num_classes - assigned; ++k) q[order[k]] += 1;
  for (int i = 0; i < N; ++i)
    if (q[i] == 0) return fail(WHALE_ERR_UNSPLITTABLE, "shard %d would receive 0 classes", i);
  int64_t off = 0;
  for (int i = 0; i < N; ++i) {
    shard_counts[i] = q[i];
    shard_offsets[i] = off;
    off += q[i];
  }
  return WHALE_OK;
}

// ============================================================================ plan + memory (NEXT-1)
// Algorithm 1 "Memory-Constraint Load Balancing" in whole classes,
// starting from the proportional plan; exact rational comparisons (cross-multiplied).
namespace {
struct Ratio {  // num / den, den > 0
  __int128 num, den;
};
inline bool lt(const Ratio& a, const Ratio& b) { return a.num * b.den < b.num * a.den; }
inline bool eq(const Ratio& a, const Ratio& b) { return a.num * b.den == b.num * a.den; }
}  // namespace

extern "C" whale_status_t whale_splitfc_plan_mem(int64_t num_classes, int32_t world_size, const uint32_t* capacity,
                                                 const uint64_t* mem_bytes, uint64_t bytes_per_class,
                                                 uint64_t fixed_bytes, int64_t* shard_counts,
                                                 int64_t* shard_offsets) {
  whale_status_t st = whale_splitfc_plan(num_classes, world_size, capacity, shard_counts, shard_offsets);
  if (mem_bytes == nullptr) return st;
  if (bytes_per_class == 0) return fail(WHALE_ERR_INVALID_ARG, "bytes_per_class must be > 0");
  if (st != WHALE_OK) return st;
  const int N = world_size;
  int64_t n[kMaxRanks], cap[kMaxRanks];
  __int128 room[kMaxRanks];
  bool in_oom[kMaxRanks], in_free[kMaxRanks];
  for (int i = 0; i < N; ++i) {
    n[i] = shard_counts[i];
    room[i] = static_cast<__int128>(mem_bytes[i]) - static_cast<__int128>(fixed_bytes);
    cap[i] = room[i] > 0 ? static_cast<int64_t>(room[i] / bytes_per_class) : 0;
    in_oom[i] = n[i] > cap[i];
    in_free[i] = !in_oom[i];
  }
  auto mem_util = [&](int i) -> Ratio {
    if (room[i] <= 0) return Ratio{static_cast<__int128>(1) << 100, 1};
    return Ratio{static_cast<__int128>(n[i]) * bytes_per_class, room[i]};
  };
  auto flop_util = [&](int i) -> Ratio { return Ratio{n[i], capacity ? capacity[i] : 1u}; };
  for (;;) {
    int peak = -1, valley = -1;
    for (int i = 0; i < N; ++i)
      if (in_oom[i] && (peak < 0 || lt(mem_util(peak), mem_util(i)))) peak = i;  // ties: lower index
    for (int i = 0; i < N; ++i) {
      if (!in_free[i]) continue;
      if (valley < 0) {
        valley = i;
        continue;
      }
      const Ratio fi = flop_util(i), fv = flop_util(valley);
      if (lt(fi, fv) || (eq(fi, fv) && lt(mem_util(i), mem_util(valley)))) valley = i;
    }
    if (peak < 0 || valley < 0) break;
    const int64_t head = cap[valley] - n[valley];
    if (head > 0) {
      const int64_t b = std::min(n[peak] - cap[peak], head);
      n[peak] -= b;
      n[valley] += b;
      if (n[peak] <= cap[peak]) in_oom[peak] = false;  // leaves oom only once it fits
    } else {
      in_free[valley] = false;
    }
  }
  for (int i = 0; i < N; ++i)
    if (in_oom[i]) return fail(WHALE_ERR_UNSPLITTABLE, "memory-infeasible: device %d still overloaded", i);
  for (int i = 0; i < N; ++i)
    if (n[i] == 0) return fail(WHALE_ERR_UNSPLITTABLE, "shard %d would receive 0 classes", i);
  int64_t off = 0;
  for (int i = 0; i < N; ++i) {
    shard_counts[i] = n[i];
    shard_offsets[i] = off;
    off += n[i];
  }
  return WHALE_OK;
}

// ============================================================================ configuration
struct GemmCfg {
  int BN = 0, bk = 64, m_blocks = 0, n_blocks = 0, splits = 1, num_kb = 0, kb_per_split = 0, num_tiles = 0;
  int stages = 0, stage_bytes = 0, epi_bufs = 2, smem = 0, grid = 0;
  int cluster = 1;  // 2: CTA pairs share (TMA-multicast) the B tile of M-adjacent tiles
  int a_rows = 128;  // K-major A rows per TMA box / smem stage (GemmArgs::a_rows)
  bool p_direct = false;  // logits: P~ stored from registers, no epilogue staging (GemmArgs::p_direct)
};

static int env_int(const char* name, int dflt);
static constexpr int kSmemLimit = 232448;  // 227 KB opt-in per CTA on sm_100 (static + dynamic)
static constexpr int kStaticSmemSlack = 1664;  // the GEMM's own __shared__ words (logits epilogue: 1.5 KB)

// CTA pairs (cta_group::2): M-adjacent tiles run as one M = 256 MMA; each CTA keeps its 128
// rows of A and HALF of the B tile, so a stage costs a_bytes + B/2 and more stages fit.  The
// grid is 2 x pair tiles (capped at the SM count); an odd M block count gets one all-padding
// tile (TMA zero-fills its loads, clips its stores).  WHALE_CLUSTER=2 forces pairs, 1 forbids
// them; by default (-1) the logits pair up when K is long (>= 32 k-blocks: the tensor-bound
// c5, where pairs take the logits from 0.84 to 0.91 of the burst bf16 peak) -- with a short K the
// two-pass softmax epilogue, not the operand feed, sets the pace and pairs lose (c4: -13 %).
static void maybe_pair(GemmCfg& g, int sms, bool b_mn, int atom, int es = 2, bool auto_ok = false) {
  const int want = env_int("WHALE_CLUSTER", -1);
  const bool on = want == 2 || (want < 0 && auto_ok && g.num_kb >= 32);
  const bool ok = on && g.m_blocks >= 2 && (b_mn ? (g.BN / atom) % 2 == 0 : (g.BN / 2) % 16 == 0) && g.splits == 1;
  if (!ok) return;
  g.cluster = 2;
  g.m_blocks += g.m_blocks & 1;
  g.num_tiles = g.m_blocks * g.n_blocks * g.splits;
  const int units = g.num_tiles / 2;
  g.grid = 2 * std::min(units, sms / 2);
  // per-CTA stage: own A + half of B
  const int box = g.bk * kRowBytes;
  const int a_bytes = (b_mn ? (kBM / atom) * box : kStageABytes);
  g.stage_bytes = a_bytes + (b_mn ? (g.BN / 2 / atom) * box : (g.BN / 2) * kRowBytes);
  const int avail = kSmemLimit - kStaticSmemSlack - 1024 - 256 - 4 * g.epi_bufs * kEpiBufBytes;
  g.stages = std::min(8, avail / g.stage_bytes);
  g.smem = gemm_smem_bytes(g.stages, g.stage_bytes, g.epi_bufs);
  (void)es;
}

struct Layout {
  // local workspace offsets
  size_t P = 0, m_tile = 0, s_tile = 0, zy = 0, lse = 0, row_loss = 0, dxpart = 0, counters = 0, tile_cnt = 0;
  size_t a_tile = 0, dbpart = 0;  // NEXT-4: per-(row, tile) top-1 class; bias-gradient partials
  size_t upart = 0, uref = 0;     // F1: per-cluster U = sum_t P~_t W_t partials and their row references
  size_t mx_tile = 0;             // F1: true per-(row, tile) maxima (m_tile holds the references)
  size_t gscale = 0;              // G-fused backward: e^{m_tile - lse} / B_tot per (row, tile)
  size_t local_total = 0;
  // fp32 (kind::tf32) backward only: K-major transposed operands
  size_t XT = 0, GT = 0, WT = 0;
  int64_t ld_bt = 0;
  // symmetric buffer offsets (per parity for the slabs); world > 1 only
  // single-buffered: a rank overwrites a peer's slab only after that peer's end-of-step
  // ticket (RS flag) proved it finished reading it (see end_of_step_ticket)
  size_t flags = 0, xg = 0, yg = 0, stats = 0, dxrecv = 0, symm_total = 0;
};

enum FlagKind { FLAG_GATHER = 0, FLAG_STATS = 1, FLAG_RS = 2 };
enum CounterIdx { CNT_GATHER = 0, CNT_STATS = 1, CNT_DONE = 2, CNT_SCHED = 3, CNT_EPOCH = 4, CNT_ERR = 16 };

struct Plan {
  int rank = 0, world = 1, es = 2;
  bool dw_bf16 = false;  // dW_r stored in bf16 (fused backward only)
  int64_t B = 0, Bt = 0, D = 0, C = 0, Cr = 0, o_r = 0, ldp = 0;
  int64_t Bmax = 0;                  // largest per-rank batch (dX receive slab rows)
  int64_t Boff[kMaxRanks + 1] = {};  // rank r's rows: [Boff[r], Boff[r+1]) of the gathered batch
  int sms = 148;
  GemmCfg fwd, dw, dx;
  // F1 (fwd_dx_sm100.cuh): fused logits + dX partials, W_r read once (bf16, B_tot <= 32)
  bool f1 = false;
  int f1_ncl = 0, f1_stages = 0, f1_smem = 0, f1_Dq = 0, f1_s2 = 2;
  Layout L;
};


static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
static int cdiv(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// Stages / store buffers: short K loops (dW: K = B_tot) are store-bound -> deep store
// pipelining (8 x 4 KB in flight per epilogue warp); long K loops keep 4+ load stages.
static void finish_cfg(GemmCfg& g, int sms, bool store_heavy, int es = 2, bool both_mn = false) {
  if (both_mn) {  // MN-major boxes {atom, bk}: A = 128/atom boxes, B = BN/atom boxes
    const int atom = kRowBytes / es;
    g.stage_bytes = (kBM / atom + g.BN / atom) * g.bk * kRowBytes;
  } else {
    g.stage_bytes = g.a_rows * kRowBytes + g.BN * kRowBytes;
  }
  g.epi_bufs = store_heavy ? 8 : 2;
  const int avail = kSmemLimit - kStaticSmemSlack - 1024 - 256 - 4 * g.epi_bufs * kEpiBufBytes;
  g.stages = std::min(8, avail / g.stage_bytes);
  if (g.stages < 2) {
    g.epi_bufs = 2;
    g.stages = std::min(8, (kSmemLimit - kStaticSmemSlack - 1024 - 256 - 4 * 2 * kEpiBufBytes) / g.stage_bytes);
  }
  g.smem = gemm_smem_bytes(g.stages, g.stage_bytes, g.epi_bufs);
  g.num_tiles = g.m_blocks * g.n_blocks * g.splits;
  g.grid = std::min(g.num_tiles, sms);
}

// Pick BN (multiple of `gran`, <= 256) minimising waves x per-tile cost.
static GemmCfg choose_plain(int64_t M, int64_t N, int64_t K, int gran, int kbk, int sms) {
  GemmCfg best;
  double best_cost = 1e300;
  const int64_t nmax = std::min<int64_t>(256, align_up(N, gran));
  for (int BN = static_cast<int>(nmax / gran * gran); BN >= gran; BN -= gran) {
    GemmCfg g;
    g.BN = BN;
    g.m_blocks = cdiv(M, kBM);
    g.n_blocks = cdiv(N, BN);
    g.num_kb = cdiv(K, kbk);
    g.splits = 1;
    g.kb_per_split = g.num_kb;
    const int64_t tiles = static_cast<int64_t>(g.m_blocks) * g.n_blocks;
    const double cost = static_cast<double>(cdiv(tiles, sms)) * (BN + 48);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = g;
    }
  }
  finish_cfg(best, sms, best.num_kb <= 4);
  return best;
}

// dX: M = B_tot, N = D, K = C_r.  Split K so that tiles fill the SMs; the partial sums
// ([S x B_tot x D] fp32) are reduced inside the kernel (fixup), which needs every CTA of a
// tile co-resident: S > 1 only when all tiles fit in one wave.
static GemmCfg choose_splitk(int64_t M, int64_t N, int64_t K, int gran, int kbk, int sms) {
  GemmCfg best;
  double best_cost = 1e300;
  const int64_t nmax = std::min<int64_t>(256, align_up(N, gran));
  const int num_kb = cdiv(K, kbk);
  for (int BN = static_cast<int>(nmax / gran * gran); BN >= gran; BN -= gran) {
    const int mb = cdiv(M, kBM), nb = cdiv(N, BN);
    const int64_t mn = static_cast<int64_t>(mb) * nb;
    for (int S = 1; S <= std::min(num_kb, 64); ++S) {
      const int kbps = cdiv(num_kb, S);
      if (cdiv(num_kb, kbps) != S) continue;
      const int64_t tiles = mn * S;
      if (S > 1 && tiles > sms) break;
      const double kblock_bytes = (128.0 + BN) * kRowBytes;
      const double cost = static_cast<double>(cdiv(tiles, sms)) * kbps * kblock_bytes +
                          static_cast<double>(S) * M * N * 8.0 / sms;
      if (cost < best_cost * 0.999) {
        best_cost = cost;
        GemmCfg g;
        g.BN = BN;
        g.m_blocks = mb;
        g.n_blocks = nb;
        g.splits = S;
        g.num_kb = num_kb;
        g.kb_per_split = kbps;
        best = g;
      }
    }
  }
  finish_cfg(best, sms, false);
  return best;
}

static whale_status_t build_plan(const whale_splitfc_desc* d, Plan& p, int sms) {
  if (!d) return fail(WHALE_ERR_INVALID_ARG, "NULL descriptor");
  if (d->world_size < 1 || d->world_size > kMaxRanks)
    return fail(WHALE_ERR_UNSUPPORTED, "world_size %d outside [1, %d]", d->world_size, kMaxRanks);
  if (d->rank < 0 || d->rank >= d->world_size) return fail(WHALE_ERR_INVALID_ARG, "rank out of range");
  if (d->local_batch < 0 || d->feature_dim < 1 || d->num_classes < 1)
    return fail(WHALE_ERR_INVALID_ARG, "B >= 0, D >= 1 and C >= 1 required");
  if (d->feature_dim % 8 != 0) return fail(WHALE_ERR_UNSUPPORTED, "feature_dim %% 8 != 0 (TMA 16-byte rows)");
  if (d->x_dtype != WHALE_BF16 && d->x_dtype != WHALE_F32) return fail(WHALE_ERR_UNSUPPORTED, "x_dtype");
  if (d->dw_dtype != WHALE_F32 && !(d->dw_dtype == WHALE_BF16 && d->x_dtype == WHALE_BF16))
    return fail(WHALE_ERR_UNSUPPORTED, "dw_dtype must be WHALE_F32 (or WHALE_BF16 with bf16 operands)");
  if (!d->shard_counts || !d->shard_offsets) return fail(WHALE_ERR_INVALID_ARG, "NULL shard plan");
  int64_t off = 0;
  for (int r = 0; r < d->world_size; ++r) {
    if (d->shard_counts[r] < 1 || d->shard_offsets[r] != off)
      return fail(WHALE_ERR_INVALID_ARG, "shard plan is not a partition of [0, C) at rank %d", r);
    off += d->shard_counts[r];
  }
  if (off != d->num_classes) return fail(WHALE_ERR_INVALID_ARG, "shard counts do not sum to C");
  p.rank = d->rank;
  p.world = d->world_size;
  p.es = d->x_dtype == WHALE_BF16 ? 2 : 4;
  p.dw_bf16 = d->dw_dtype == WHALE_BF16;
  p.B = d->local_batch;
  p.Boff[0] = 0;
  for (int r = 0; r < p.world; ++r) {
    const int64_t br = d->batch_counts ? d->batch_counts[r] : d->local_batch;
    if (br < 0 || br > 65535) return fail(WHALE_ERR_INVALID_ARG, "batch_counts[%d] = %lld outside [0, 65535]", r, (long long)br);
    p.Boff[r + 1] = p.Boff[r] + br;
    p.Bmax = std::max(p.Bmax, br);
  }
  if (d->batch_counts && d->batch_counts[p.rank] != d->local_batch)
    return fail(WHALE_ERR_INVALID_ARG, "local_batch != batch_counts[rank]");
  p.Bt = p.Boff[p.world];
  if (p.Bt < 1 || (p.world == 1 && p.B < 1)) return fail(WHALE_ERR_INVALID_ARG, "empty global batch");
  p.D = d->feature_dim;
  p.C = d->num_classes;
  p.Cr = d->shard_counts[p.rank];
  p.o_r = d->shard_offsets[p.rank];
  if (p.Bt > 65535) return fail(WHALE_ERR_UNSUPPORTED, "global batch > 65535");
  if (p.Cr > (1ll << 31) - 256 || p.D > (1ll << 31) - 256) return fail(WHALE_ERR_UNSUPPORTED, "dimension too large");
  const int vec = 16 / p.es;
  p.ldp = static_cast<int64_t>(align_up(p.Cr, vec));
  {
    // heterogeneity emulation (NEXT-1 experiment): WHALE_SM_LIMIT_R<rank>=n caps the SMs
    // this rank's kernels use, making it a "slower GPU" (E8)
    char name[32];
    snprintf(name, sizeof(name), "WHALE_SM_LIMIT_R%d", p.rank);
    const char* e = getenv(name);
    if (e && atoi(e) > 0) sms = std::min(sms, atoi(e));
  }
  p.sms = sms;
  const int kbk = kRowBytes / p.es;   // K elements per stage
  const int atom = kRowBytes / p.es;  // MN-major atom / fwd P~ chunk
  p.fwd = choose_plain(p.Bt, p.Cr, p.D, atom, kbk, sms);
  maybe_pair(p.fwd, sms, false, atom, p.es, p.es == 2);
  {
    // dW: both operands MN-major; a short K (= B_tot <= 32) uses 32-row K stages (no
    // zero-padded half stage), which doubles the pipeline depth for the same smem.
    const int bk = (p.es == 2 && p.Bt <= 32) ? 32 : kbk;
    p.dw = choose_plain(p.Cr, p.D, p.Bt, atom, bk, sms);
    const int force_bn = env_int("WHALE_DW_BN", 0);  // experiments: dW N tile (multiple of the atom)
    if (force_bn >= atom && force_bn <= 256 && force_bn % atom == 0) {
      p.dw.BN = force_bn;
      p.dw.n_blocks = cdiv(p.D, force_bn);
    }
    p.dw.bk = bk;
    finish_cfg(p.dw, sms, p.dw.num_kb <= 4, p.es, p.es == 2);
  }
  p.dx = choose_splitk(p.Bt, p.D, p.Cr, atom, kbk, sms);
  // the B_tot-row operands (X for the logits, G for dX): when all of B_tot fits one M block,
  // load only its rows rounded up to 8 (one SW128 atom) -- at B_tot = 64 (c2, N = 2) a stage
  // shrinks from 40 to 32 KB and the ring deepens from 4 to 6 stages
  auto shrink_a = [&](GemmCfg& g, bool store_heavy) {
    if (g.m_blocks == 1 && g.cluster == 1 && p.Bt < kBM && env_int("WHALE_SHRINK_A", 1) != 0) {
      g.a_rows = static_cast<int>(align_up(p.Bt, 8));
      finish_cfg(g, sms, store_heavy);
    }
  };
  shrink_a(p.fwd, p.fwd.num_kb <= 4);  // as choose_plain
  shrink_a(p.dx, false);               // as choose_splitk
  // logits with one M block (the N > 1 shard shapes): P~ from registers when dropping the 32 KB
  // of epilogue staging buys another load stage (each CTA streams one or two long-K tiles)
  if (p.fwd.m_blocks == 1 && p.fwd.cluster == 1 && env_int("WHALE_P_DIRECT", 1) != 0) {
    const int stages0 = std::min(8, (kSmemLimit - kStaticSmemSlack - 1024 - 256) / p.fwd.stage_bytes);
    if (stages0 > p.fwd.stages) {
      p.fwd.p_direct = true;
      p.fwd.epi_bufs = 0;
      p.fwd.stages = stages0;
      p.fwd.smem = gemm_smem_bytes(p.fwd.stages, p.fwd.stage_bytes, 0);
    }
  }
  {
    const char* e = getenv("WHALE_F1");
    p.f1 = p.es == 2 && p.Bt <= kF1NB && p.D % (kF1KC * 128) == 0 && p.D / kF1KC <= 1024 &&
           !(e && e[0] == '0');
    if (p.f1) {
      p.f1_Dq = static_cast<int>(p.D / kF1KC);
      const int T = cdiv(p.Cr, kF1TileC);
      p.f1_ncl = std::min(sms / kF1KC, T);  // upper bound; create() lowers it to the co-resident count
      // stages: provisional here (host-only planning); create() sizes them with the kernel's
      // real static shared memory
      p.f1_s2 = std::max(1, std::min(kF1S2Max, env_int("WHALE_F1_S2", 3)));
      const int fixed = f1_smem_bytes(0, p.f1_s2) + 2048;
      p.f1_stages = std::min(std::min(env_int("WHALE_F1_S1", 8), 8), (kSmemLimit - fixed) / kF1G1SlotBytes);
      p.f1_smem = f1_smem_bytes(p.f1_stages, p.f1_s2);
      if (p.f1_stages < 3) p.f1 = false;
    }
    if (p.f1) {  // the statistics / gradient pipeline sees 128-class tiles
      p.fwd.BN = kF1TileC;
      p.fwd.n_blocks = cdiv(p.Cr, kF1TileC);
    }
  }

  Layout& L = p.L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + bytes, 1024);
    return at;
  };
  const int T = p.fwd.n_blocks;
  L.P = take(static_cast<size_t>(p.Bt) * p.ldp * p.es);
  L.m_tile = take(static_cast<size_t>(p.Bt) * T * 4);
  L.s_tile = take(static_cast<size_t>(p.Bt) * T * 4);
  L.zy = take(p.Bt * 4);
  L.lse = take(p.Bt * 4);
  L.row_loss = take(p.Bt * 4);
  L.dxpart = take(static_cast<size_t>(p.dx.splits) * p.Bt * p.D * 4);
  L.counters = take(64 * 4);
  L.tile_cnt = take(static_cast<size_t>(p.dx.m_blocks + 1) * p.dx.n_blocks * 4);  // +1: a CTA-pair padding block
  L.a_tile = take(static_cast<size_t>(p.Bt) * T * 4);
  L.dbpart = take(static_cast<size_t>(cdiv(p.Bt, kDbRows)) * p.Cr * 4);
  L.gscale = take(static_cast<size_t>(p.Bt) * T * 4);
  if (p.f1) {
    L.upart = take(static_cast<size_t>(p.f1_ncl) * p.Bt * p.D * 4);
    L.uref = take(static_cast<size_t>(p.f1_ncl) * p.Bt * 4);
    L.mx_tile = take(static_cast<size_t>(p.Bt) * p.fwd.n_blocks * 4);
  }
  if (p.es == 4) {
    L.ld_bt = static_cast<int64_t>(align_up(p.Bt, 4));
    L.XT = take(static_cast<size_t>(p.D) * L.ld_bt * 4);
    L.GT = take(static_cast<size_t>(p.Cr) * L.ld_bt * 4);
    L.WT = take(static_cast<size_t>(p.D) * p.ldp * 4);
  }
  L.local_total = o;
  o = 0;
  if (p.world > 1) {
    L.flags = take(4 * kMaxRanks * 4);
    L.xg = take(static_cast<size_t>(p.Bt) * p.D * p.es);
    L.yg = take(p.Bt * 4);
    L.stats = take(static_cast<size_t>(p.world) * p.Bt * 32);  // LL words {m,s,zy,-} x {data, epoch}
    L.dxrecv = take(static_cast<size_t>(p.world) * p.Bmax * p.D * 4);
  }
  L.symm_total = o;
  return WHALE_OK;
}

extern "C" whale_status_t whale_splitfc_workspace_size(const whale_splitfc_desc* desc, size_t* symm_bytes,
                                                       size_t* local_bytes) {
  Plan p;
  // SM count only shapes the tile choice; query it if a device is present, else 148.
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) sms = v;
  } else {
    cudaGetLastError();
  }
  whale_status_t st = build_plan(desc, p, sms);
  if (st != WHALE_OK) return st;
  if (symm_bytes) *symm_bytes = p.L.symm_total;
  if (local_bytes) *local_bytes = p.L.local_total;
  return WHALE_OK;
}

// ============================================================================ TMA descriptors
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static whale_status_t get_encoder() {
  if (g_encode) return WHALE_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(WHALE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return WHALE_OK;
}

// rank-2 or rank-3 map; dims/box innermost first; strides in bytes for dims 1..rank-1.
static whale_status_t make_map(CUtensorMap* m, const void* base, int es, int rank, const uint64_t* dims,
                               const uint64_t* strides, const uint32_t* box) {
  whale_status_t st = get_encoder();
  if (st != WHALE_OK) return st;
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) return fail(WHALE_ERR_INVALID_ARG, "tensor base not 16-byte aligned");
  cuuint64_t gd[3], gs[2];
  cuuint32_t bd[3], es1[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bd[i] = box[i];
  }
  for (int i = 0; i < rank - 1; ++i) gs[i] = strides[i];
  const CUtensorMapDataType dt = es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUresult r = g_encode(m, dt, rank, const_cast<void*>(base), gd, gs, bd, es1, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(WHALE_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return WHALE_OK;
}

static whale_status_t map2d(CUtensorMap* m, const void* base, int es, uint64_t inner, uint64_t outer,
                            uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
  const uint64_t dims[2] = {inner, outer};
  const uint64_t strides[1] = {row_bytes};
  const uint32_t box[2] = {box_inner, box_outer};
  return make_map(m, base, es, 2, dims, strides, box);
}

static int g_store_mode = [] {
  const char* e = getenv("WHALE_STORE_MODE");
  return e ? atoi(e) : 1;
}();

// fp32 (or bf16) output map {N, rows, splits}; box {128 B of columns, 128 rows for the
// CTA-wide store (mode 1) else 32, 1}.
static whale_status_t map3d_out(CUtensorMap* m, const void* base, uint64_t n, uint64_t rows, uint64_t splits,
                                int es = 4) {
  const uint64_t dims[3] = {n, rows, splits};
  const uint64_t strides[2] = {n * es, n * rows * es};
  const uint32_t box[3] = {static_cast<uint32_t>(kRowBytes / es), g_store_mode == 1 ? 128u : 32u, 1};
  return make_map(m, base, es, 3, dims, strides, box);
}

// ============================================================================ context
struct ProfRec {
  int kind;
  cudaEvent_t a, b;
};
static const char* kKindNames[] = {"bridge_gather", "logits_gemm",  "stats_combine", "softmax_grad", "dw_gemm",
                                   "dx_gemm",       "dx_rs_reduce", "transpose_f32", "bwd_gemm", "bias_grad"};
enum KernelKind { K_GATHER, K_LOGITS, K_STATS, K_GRAD, K_DW, K_DX, K_RS_REDUCE, K_TRANSPOSE, K_BWD, K_DB, K_NUM };

struct whale_splitfc_ctx {
  Plan p;
  uint8_t* ws = nullptr;
  uint8_t* symm[kMaxRanks] = {};
  uint8_t* mc = nullptr;  // NVLS multicast address of the symmetric buffer (or NULL)
  // static maps (X maps: per parity at N > 1; cached on the caller's X at N = 1)
  CUtensorMap tmX_fwd, tmX_dw, tmP_store, tmG_dx, tmG_dw, tmDxPart;
  CUtensorMap tmGT, tmXT, tmWT;  // fp32 path: K-major transposed operands
  // pointer-cached maps
  const void* x_cached = nullptr;
  const void* w_cached = nullptr;
  CUtensorMap tmW_fwd, tmW_dx, tmW_f1, tmX_f1, tmP_f1;
  const void* dw_cached = nullptr;
  CUtensorMap tmDW;
  const void* x_fwd = nullptr;       // N = 1: the forward's X (read again by dW)
  const int32_t* y_fwd = nullptr;    // N = 1: the forward's labels
  uint32_t epoch = 0;                // forward count (flag epochs, parity)
  uint32_t bwd_epoch = 0;            // backward count (fixup counters)
  bool have_fwd = false;
  bool pdl = false;
  int pdl_mask = 0;                  // per-kernel PDL (WHALE_PDL_MASK): 1 stats, 2 backward, 4 owner reduce, 8 logits/F1
  int cur_kbit = 0;                  // the PDL bit of the launch being issued
  bool fused_bwd = true;             // dW + dX in one persistent launch (bf16)
  bool gfuse = true;                 // G-fused backward (NEXT-4b): G formed from P~ in the bwd operand path
  bool row_bulk = false;             // dW tiles stored as 1-D bulk row copies (bwd_sm100.cuh)
  bool fused_gather = true;          // N > 1: bridge all-gather inside the logits / F1 prologue
  bool bwd_pair = false;             // fused backward as CTA pairs (cta_group::2)
  bool nvls_rs = false;              // dX reduce-scatter through the NVSwitch (multimem.ld_reduce)
  bool fused_reduce = true;          // N > 1: the owner reduce in the fused backward's tail
  bool w_l2 = false;                 // W_r kept in L2 between the logits and the backward's dX pass
  bool shared_device = false;        // ranks emulated on one device (tests): no PDL, bounded grids
  int bwd_stages = 0, bwd_stage_bytes = 0, bwd_epi_bufs = 4, bwd_smem = 0;
  bool profile = false;
  std::vector<ProfRec> prof;
  double prof_ms[K_NUM] = {};
  int64_t prof_n[K_NUM] = {};
};

template <typename T>
static T* wsp(whale_splitfc_ctx* c, size_t off) {
  return reinterpret_cast<T*>(c->ws + off);
}

// PDL for the launch being issued (WHALE_PDL=1: every launch; WHALE_PDL_MASK: selected
// kernels); consumes the launch's PDL bit.
static bool pdl_for(whale_splitfc_ctx* c) {
  const bool on = c->pdl || (c->pdl_mask & c->cur_kbit) != 0;
  c->cur_kbit = 0;
  return on;
}

// Launch with programmatic dependent launch (PDL): kernels call griddepcontrol.wait.
template <typename... KArgs, typename... Args>
static whale_status_t launch(whale_splitfc_ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_for(c) ? 1 : 0;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
  return WHALE_OK;
}

// cudaFuncSetAttribute acts on the current device: remember per (device, kernel slot) that the
// opt-in shared-memory limit has been raised (slots 0..7: GEMMs, 8 / 9: fused backward fp32 / bf16 dW,
// 10..17: the GEMMs' CTA-pair instantiations).
static constexpr int kMaxDevices = 64;
static bool g_attr_done[kMaxDevices][20] = {};

template <typename K>
static whale_status_t ensure_smem_attr(K kern, int slot) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(WHALE_ERR_UNSUPPORTED, "device index %d", dev);
  if (g_attr_done[dev][slot]) return WHALE_OK;
  cudaFuncAttributes fa{};
  CUDA_TRY(cudaFuncGetAttributes(&fa, kern));
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemLimit - static_cast<int>(fa.sharedSizeBytes)));
  g_attr_done[dev][slot] = true;
  return WHALE_OK;
}

template <int EPI, bool AMN, bool BMN, int ES>
static whale_status_t launch_gemm(whale_splitfc_ctx* c, int slot, const GemmCfg& g, const CUtensorMap& A,
                                  const CUtensorMap& B, const CUtensorMap& O, const GemmArgs& args,
                                  cudaStream_t s) {
  auto kern = g.cluster > 1 ? splitfc_gemm_kernel<EPI, AMN, BMN, ES, true> : splitfc_gemm_kernel<EPI, AMN, BMN, ES, false>;
  {
    const whale_status_t st = ensure_smem_attr(kern, slot + (g.cluster > 1 ? 10 : 0));
    if (st != WHALE_OK) return st;
  }
  constexpr int kThreads = EPI == EPI_FWD_STATS ? kStatsGemmThreads : kGemmThreads;
  if (g.cluster <= 1) return launch(c, kern, dim3(g.grid), dim3(kThreads), g.smem, s, A, B, O, args);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = g.cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_for(c) ? 2 : 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, A, B, O, args));
  return WHALE_OK;
}

static void prof_begin(whale_splitfc_ctx* c, int kind, cudaStream_t s, ProfRec& r) {
  if (!c->profile) return;
  r.kind = kind;
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, s);
}
static void prof_end(whale_splitfc_ctx* c, cudaStream_t s, ProfRec& r) {
  if (!c->profile) return;
  cudaEventRecord(r.b, s);
  c->prof.push_back(r);
}

#define PROFILED(kind, stream, body)            \
  do {                                          \
    ProfRec _r{};                               \
    prof_begin(c, kind, stream, _r);            \
    whale_status_t _st = (body);                \
    if (_st != WHALE_OK) return _st;            \
    prof_end(c, stream, _r);                    \
  } while (0)

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
static int g_n_fastest = env_int("WHALE_N_FASTEST", 0);
static int g_epi_debug = env_int("WHALE_EPI_DEBUG", 0);
static int g_dw_m_fastest = env_int("WHALE_DW_M_FASTEST", 0);

static GemmArgs base_args(const GemmCfg& g, int M, int N) {
  GemmArgs a{};
  a.M = M;
  a.N = N;
  a.BN = g.BN;
  a.m_blocks = g.m_blocks;
  a.n_blocks = g.n_blocks;
  a.splits = g.splits;
  a.num_kb = g.num_kb;
  a.kb_per_split = g.kb_per_split;
  a.num_tiles = g.cluster > 1 ? g.num_tiles / g.cluster : g.num_tiles;  // units (pair tiles)
  a.cluster = g.cluster;
  a.stages = g.stages;
  a.stage_bytes = g.stage_bytes;
  a.epi_bufs = g.epi_bufs;
  a.bk = g.bk;
  a.a_rows = g.a_rows;
  a.store_mode = g_store_mode;
  a.n_fastest = g_n_fastest;
  a.debug = g_epi_debug;
  return a;
}

#define MAP_TRY(x)                 \
  do {                             \
    whale_status_t _s = (x);       \
    if (_s != WHALE_OK) {          \
      delete c;                    \
      return _s;                   \
    }                              \
  } while (0)

// Load every kernel of the library into the current context now (CUDA lazy loading would
// otherwise load a function at its first launch, and loading may wait for the device's
// running kernels -- a deadlock when those kernels spin on flags that a not-yet-launched
// kernel of another rank sharing the device must raise, and a latency spike mid-step).
static whale_status_t preload_kernels() {
  const void* fns[] = {
      reinterpret_cast<const void*>(bridge_gather_kernel),
      reinterpret_cast<const void*>(splitfc_gemm_kernel<EPI_FWD_STATS, false, false, 2>),
      reinterpret_cast<const void*>(splitfc_gemm_kernel<EPI_FWD_STATS, false, false, 4>),
      reinterpret_cast<const void*>(splitfc_gemm_kernel<EPI_STORE_F32, true, true, 2>),
      reinterpret_cast<const void*>(splitfc_gemm_kernel<EPI_STORE_F32, false, true, 2>),
      reinterpret_cast<const void*>(splitfc_gemm_kernel<EPI_STORE_F32, false, false, 4>),
      reinterpret_cast<const void*>(splitfc_gemm_kernel<EPI_FWD_STATS, false, false, 2, true>),
      reinterpret_cast<const void*>(splitfc_gemm_kernel<EPI_FWD_STATS, false, false, 4, true>),
      reinterpret_cast<const void*>(splitfc_gemm_kernel<EPI_STORE_F32, true, true, 2, true>),
      reinterpret_cast<const void*>(splitfc_gemm_kernel<EPI_STORE_F32, false, true, 2, true>),
      reinterpret_cast<const void*>(splitfc_gemm_kernel<EPI_STORE_F32, false, false, 4, true>),
      reinterpret_cast<const void*>(splitfc_fwd_dx_kernel),
      reinterpret_cast<const void*>(splitfc_bwd_kernel<2, false>),
      reinterpret_cast<const void*>(splitfc_bwd_kernel<2, true>),
      reinterpret_cast<const void*>(splitfc_bwd_kernel<2, false, true>),
      reinterpret_cast<const void*>(splitfc_bwd_kernel<2, true, true>),
      reinterpret_cast<const void*>(stats_grad_kernel<2>),
      reinterpret_cast<const void*>(stats_grad_kernel<4>),
      reinterpret_cast<const void*>(stats_grad_multi_kernel<2>),
      reinterpret_cast<const void*>(stats_grad_multi_kernel<4>),
      reinterpret_cast<const void*>(dx_reduce_kernel<2>),
      reinterpret_cast<const void*>(dx_reduce_kernel<4>),
      reinterpret_cast<const void*>(dx_combine_kernel<2>),
      reinterpret_cast<const void*>(bias_grad_part_kernel<2>),
      reinterpret_cast<const void*>(bias_grad_part_kernel<4>),
      reinterpret_cast<const void*>(bias_grad_sum_kernel),
      reinterpret_cast<const void*>(epoch_bump_kernel),
      reinterpret_cast<const void*>(transpose_f32_kernel),
  };
  for (const void* f : fns) {
    cudaFuncAttributes fa{};
    CUDA_TRY(cudaFuncGetAttributes(&fa, f));
  }
  return WHALE_OK;
}

extern "C" whale_status_t whale_splitfc_create(const whale_splitfc_desc* desc, whale_splitfc_ctx** out) {
  if (!out) return fail(WHALE_ERR_INVALID_ARG, "NULL out");
  *out = nullptr;
  int dev = 0, major = 0, sms = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (major != 10) return fail(WHALE_ERR_UNSUPPORTED, "needs an sm_100 (B200) device, found major %d", major);
  {
    const whale_status_t pst = preload_kernels();
    if (pst != WHALE_OK) return pst;
  }
  auto* c = new whale_splitfc_ctx();
  whale_status_t st = build_plan(desc, c->p, sms);
  if (st != WHALE_OK) {
    delete c;
    return st;
  }
  const Plan& p = c->p;
  if (!desc->local_workspace || desc->local_workspace_bytes < p.L.local_total ||
      reinterpret_cast<uintptr_t>(desc->local_workspace) % 256) {
    delete c;
    return fail(WHALE_ERR_STATE, "local workspace missing, misaligned or < %zu bytes", p.L.local_total);
  }
  c->ws = static_cast<uint8_t*>(desc->local_workspace);
  if (p.world > 1) {
    if (!desc->peer_symm_ptrs || desc->symm_bytes < p.L.symm_total) {
      delete c;
      return fail(WHALE_ERR_STATE, "symmetric buffers missing or < %zu bytes", p.L.symm_total);
    }
    for (int r = 0; r < p.world; ++r) c->symm[r] = static_cast<uint8_t*>(desc->peer_symm_ptrs[r]);
    c->mc = static_cast<uint8_t*>(desc->multicast_ptr);
    // NVLS reduce-scatter (multimem.ld_reduce): parity-green and bitwise reproducible at N = 2,
    // but measured slower than the unicast pushes (owner reduce 12.8 -> 17.0 us): opt-in
    c->nvls_rs = c->mc != nullptr && env_int("WHALE_NVLS_RS", 0) != 0;
  }
  const char* pdl_env = getenv("WHALE_PDL");
  // WHALE_SHARED_DEVICE=1: several ranks share this device (the single-GPU multi-rank test
  // harness): their kernels wait on one another, so no kernel may sit resident ahead of its
  // turn (no PDL) and the exchange kernels keep bounded grids; combine with
  // WHALE_SM_LIMIT_R<r> so every rank's persistent grid fits beside the others.
  c->shared_device = env_int("WHALE_SHARED_DEVICE", 0) != 0;
  // programmatic dependent launch: off by default -- measured slower in every configuration
  // (c2 N=1 249.0 -> 248.1 us, N=2 194 -> 189, c4 1265 -> 1176, c5 10.65 -> 10.38 ms without
  // it); WHALE_PDL=1 turns it on (the kernels' griddepcontrol.wait keeps either mode correct)
  c->pdl = (pdl_env && pdl_env[0] == '1') && !c->shared_device;
  c->pdl_mask = c->shared_device ? 0 : env_int("WHALE_PDL_MASK", 0);
  {
    // peer-wait timeout (flags, LL records, split-K counters): WHALE_TIMEOUT_MS, default 300 s
    const unsigned long long ns = static_cast<unsigned long long>(std::max(1, env_int("WHALE_TIMEOUT_MS", 300000))) * 1000000ull;
    CUDA_TRY(cudaMemcpyToSymbol(g_wait_timeout_ns, &ns, sizeof(ns)));
  }
  c->fused_bwd = p.es == 2 && env_int("WHALE_FUSED_BWD", 1) != 0 && g_store_mode == 1;
  c->fused_gather = env_int("WHALE_FUSED_GATHER", 1) != 0;
  c->fused_reduce = env_int("WHALE_FUSED_REDUCE", 1) != 0;
  c->gfuse = c->fused_bwd && env_int("WHALE_GFUSE", 0) != 0;
  if (p.dw_bf16 && !c->fused_bwd) {
    delete c;
    return fail(WHALE_ERR_UNSUPPORTED, "bf16 dW needs the fused backward (WHALE_FUSED_BWD / WHALE_STORE_MODE overrides)");
  }
  if (c->fused_bwd) {
    // CTA pairs in the fused backward (cta_group::2, M = 256 units over two M blocks): when dX
    // needs no split-K (large B_tot x D: the tensor-bound shapes, e.g. c5) and both N tiles
    // split into whole swizzle atoms per CTA.  Not with F1 (combine units) or the G-fused path.
    const int atom = kRowBytes / p.es;
    c->bwd_pair = !p.f1 && !c->gfuse && p.es == 2 && env_int("WHALE_BWD_PAIR", 1) != 0 && p.dx.splits == 1 &&
                  p.dx.m_blocks >= 2 && p.dw.m_blocks >= 2 && p.dx.a_rows == kBM && (p.dx.BN / atom) % 2 == 0 &&
                  (p.dw.BN / atom) % 2 == 0;
    if (c->bwd_pair) {
      for (GemmCfg* g : {&c->p.dx, &c->p.dw}) {
        g->cluster = 2;
        g->m_blocks += g->m_blocks & 1;  // an odd M block count gets one all-padding tile
        g->num_tiles = g->m_blocks * g->n_blocks * g->splits;
      }
      const int kbk = kRowBytes / p.es;
      c->p.dx.stage_bytes = kBM * kRowBytes + (p.dx.BN / 2 / atom) * kbk * kRowBytes;  // own A + half of B
      c->p.dw.stage_bytes = (kBM / atom) * p.dw.bk * kRowBytes + (p.dw.BN / 2 / atom) * p.dw.bk * kRowBytes;
    }
    // F1: the backward runs dW tiles only (dX came from the forward)
    c->bwd_stage_bytes = p.f1 ? p.dw.stage_bytes : std::max(p.dx.stage_bytes, p.dw.stage_bytes);
    // CTA-wide 16 KB store stages: dW-only (F1) deep; with dX units the load ring wants the
    // smem (measured: 2 store stages + 4 load stages beat 4 + 3 at c4 / c5 by 7-11 %)
    c->bwd_epi_bufs = env_int("WHALE_BWD_EPI", p.f1 ? 8 : (c->bwd_pair ? 4 : 2));
    // dW-only schedule (F1): row-bulk dW stores need 128 padded rows of BN fp32 of staging
    c->row_bulk = (p.f1 && env_int("WHALE_ROW_BULK", 1) != 0) || env_int("WHALE_ROW_BULK", 1) == 2;
    if (c->row_bulk)
      c->bwd_epi_bufs = std::max(c->bwd_epi_bufs, (kBM * (p.dw.BN + 4) * 4 + 4 * kEpiBufBytes - 1) / (4 * kEpiBufBytes));
    const int fixed = 1024 + 512 + c->bwd_epi_bufs * 4 * kEpiBufBytes;
    cudaFuncAttributes fa{};
    CUDA_TRY(cudaFuncGetAttributes(&fa, splitfc_bwd_kernel<2, false>));  // the kernel's own __shared__ bytes
    c->bwd_stages = std::min(8, (kSmemLimit - static_cast<int>(fa.sharedSizeBytes) - fixed) / c->bwd_stage_bytes);
    c->bwd_smem = fixed + c->bwd_stages * c->bwd_stage_bytes;
    if (c->bwd_stages < 2) c->fused_bwd = false;
  }
  {
    // The logits load W_r evict_last and the backward's dX pass, its second and last read,
    // evict_first, so the part of W_r that L2 holds survives the statistics kernel and the dW
    // stores in between (WHALE_W_L2: 1 on, 0 off, else auto).  Measured: c2 N = 2 (W_r 205 MB)
    // 185.0 -> 179.7-181.6 us, N = 4 / 8 shard shapes and c4 neutral, c5 (4 GB, CTA pairs) -2 %:
    // auto for W_r <= 256 MB on the unpaired plain path.
    const int wl2 = env_int("WHALE_W_L2", -1);
    const double w_bytes = static_cast<double>(p.Cr) * p.D * p.es;
    c->w_l2 = p.es == 2 && !p.f1 && !c->bwd_pair && (wl2 == 1 || (wl2 < 0 && w_bytes <= 256.0 * (1 << 20)));
  }

  if (!c->fused_bwd && p.es == 2) {
    maybe_pair(c->p.dw, sms, true, kRowBytes / p.es);  // standalone dW GEMM
    // standalone dX GEMM (only without split-K and with whole pairs of M blocks: the split-K
    // tile counters were laid out for the unpaired grid)
    if (p.dx.splits == 1 && p.dx.m_blocks % 2 == 0) maybe_pair(c->p.dx, sms, true, kRowBytes / p.es);
  }
  if (p.f1) {
    // F1 clusters must all be co-resident (one wave): not every GPC holds a multiple of KC SMs
    cudaFuncAttributes fa{};
    CUDA_TRY(cudaFuncGetAttributes(&fa, splitfc_fwd_dx_kernel));
    const int fixed = f1_smem_bytes(0, p.f1_s2) + static_cast<int>(fa.sharedSizeBytes);
    c->p.f1_stages = std::min(std::min(env_int("WHALE_F1_S1", 8), 8), (kSmemLimit - fixed) / kF1G1SlotBytes);
    c->p.f1_smem = f1_smem_bytes(c->p.f1_stages, p.f1_s2);
    if (c->p.f1_stages < 3) {
      delete c;
      return fail(WHALE_ERR_UNSUPPORTED, "F1 shared memory: %d static bytes leave < 3 stages", (int)fa.sharedSizeBytes);
    }
    CUDA_TRY(cudaFuncSetAttribute(splitfc_fwd_dx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemLimit - static_cast<int>(fa.sharedSizeBytes)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c->p.f1_ncl * kF1KC);
    cfg.blockDim = dim3(kF1Threads);
    cfg.dynamicSmemBytes = p.f1_smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kF1KC;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    CUDA_TRY(cudaOccupancyMaxActiveClusters(&ncl, splitfc_fwd_dx_kernel, &cfg));
    if (ncl < 1) {
      delete c;
      return fail(WHALE_ERR_UNSUPPORTED, "F1 cluster cannot be resident");
    }
    c->p.f1_ncl = std::min(c->p.f1_ncl, ncl);
  }
  // static TMA maps
  const int es = p.es, kbk = kRowBytes / es, atom = kRowBytes / es;
  if (p.world > 1) {
    {
      const void* xg = c->symm[p.rank] + p.L.xg;
      MAP_TRY(map2d(&c->tmX_fwd, xg, es, p.D, p.Bt, p.D * es, kbk, p.fwd.a_rows));
      MAP_TRY(map2d(&c->tmX_dw, xg, es, p.D, p.Bt, p.D * es, atom, p.dw.bk));
      if (p.f1) MAP_TRY(map2d(&c->tmX_f1, xg, es, p.D, p.Bt, p.D * es, 64, kF1NB));
    }
  }
  void* P = c->ws + p.L.P;
  MAP_TRY(map2d(&c->tmP_store, P, es, p.Cr, p.Bt, p.ldp * es, kRowBytes / es, 32));
  if (p.f1) MAP_TRY(map2d(&c->tmP_f1, P, es, p.Cr, p.Bt, p.ldp * es, 64, kF1NB));
  MAP_TRY(map2d(&c->tmG_dx, P, es, p.Cr, p.Bt, p.ldp * es, kbk, p.dx.a_rows));
  MAP_TRY(map2d(&c->tmG_dw, P, es, p.Cr, p.Bt, p.ldp * es, atom, p.dw.bk));
  MAP_TRY(map3d_out(&c->tmDxPart, c->ws + p.L.dxpart, p.D, p.Bt, p.dx.splits));
  if (es == 4) {
    const int64_t ldb = p.L.ld_bt;
    MAP_TRY(map2d(&c->tmGT, c->ws + p.L.GT, 4, p.Bt, p.Cr, ldb * 4, kbk, kBM));
    MAP_TRY(map2d(&c->tmXT, c->ws + p.L.XT, 4, p.Bt, p.D, ldb * 4, kbk, p.dw.BN));
    MAP_TRY(map2d(&c->tmWT, c->ws + p.L.WT, 4, p.Cr, p.D, p.ldp * 4, kbk, p.dx.BN));
  }
  CUDA_TRY(cudaMemset(c->ws + p.L.counters, 0, 64 * 4));
  CUDA_TRY(cudaMemset(c->ws + p.L.tile_cnt, 0, static_cast<size_t>(p.dx.m_blocks) * p.dx.n_blocks * 4));
  *out = c;
  return WHALE_OK;
}
#undef MAP_TRY

extern "C" whale_status_t whale_splitfc_destroy(whale_splitfc_ctx* ctx) {
  if (!ctx) return WHALE_OK;
  for (auto& r : ctx->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  delete ctx;
  return WHALE_OK;
}

// (re)encode the weight maps when the shard pointer changes (host-only, ~us)
static whale_status_t ensure_w_maps(whale_splitfc_ctx* c, const void* w) {
  if (w == c->w_cached) return WHALE_OK;
  const Plan& p = c->p;
  const int kbk = kRowBytes / p.es, atom = kRowBytes / p.es;
  // paired forward: each CTA of the pair loads (and multicasts) half of the W tile
  const uint32_t box_rows = p.fwd.cluster > 1 ? p.fwd.BN / 2 : p.fwd.BN;
  whale_status_t st = map2d(&c->tmW_fwd, w, p.es, p.D, p.Cr, p.D * p.es, kbk, box_rows);
  if (st != WHALE_OK) return st;
  st = map2d(&c->tmW_dx, w, p.es, p.D, p.Cr, p.D * p.es, atom, kbk);
  if (st != WHALE_OK) return st;
  if (p.f1) {
    st = map2d(&c->tmW_f1, w, p.es, p.D, p.Cr, p.D * p.es, 64, kF1TileC);
    if (st != WHALE_OK) return st;
  }
  c->w_cached = w;
  return WHALE_OK;
}

// N = 1: the bridge is the identity -- the GEMMs read the caller's X through maps cached
// on its pointer (slot 0).
static whale_status_t ensure_x_maps(whale_splitfc_ctx* c, const void* x) {
  if (x == c->x_cached) return WHALE_OK;
  const Plan& p = c->p;
  const int kbk = kRowBytes / p.es, atom = kRowBytes / p.es;
  whale_status_t st = map2d(&c->tmX_fwd, x, p.es, p.D, p.Bt, p.D * p.es, kbk, p.fwd.a_rows);
  if (st != WHALE_OK) return st;
  st = map2d(&c->tmX_dw, x, p.es, p.D, p.Bt, p.D * p.es, atom, p.dw.bk);
  if (st != WHALE_OK) return st;
  if (p.f1) {
    st = map2d(&c->tmX_f1, x, p.es, p.D, p.Bt, p.D * p.es, 64, kF1NB);
    if (st != WHALE_OK) return st;
  }
  c->x_cached = x;
  return WHALE_OK;
}

// Blocks of the bridge gather: identical on every rank (depends on B_max, D only); each
// block raises the peers' GATHER counters once, so the consumer waits for epoch * grid.
static int gather_grid(const Plan& p) {
  const int64_t x_vecs = p.Bmax * p.D * p.es / 16;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cdiv(x_vecs, 256), 64)));
}

// ============================================================================ forward
template <int ES>
static whale_status_t forward_impl(whale_splitfc_ctx* c, const void* x_local, const int32_t* y_local,
                                   const void* w, const void* bias, float* loss, float* row_loss,
                                   int32_t* pred, float* prob, cudaStream_t s) {
  const Plan& p = c->p;
  const Layout& L = p.L;
  unsigned* counters = wsp<unsigned>(c, L.counters);
  int* err = reinterpret_cast<int*>(counters + CNT_ERR);
  uint32_t* dev_epoch = counters + CNT_EPOCH;
  {
    whale_status_t st = ensure_w_maps(c, w);
    if (st != WHALE_OK) return st;
  }
  const int32_t* yg;
  GatherArgs gth{};
  bool gather_fused = false;
  if (p.world == 1) {
    whale_status_t st = ensure_x_maps(c, x_local);
    if (st != WHALE_OK) return st;
    yg = y_local;
    c->x_fwd = x_local;
    c->y_fwd = y_local;
  } else {
    // ---- A2 bridge all-gather over NVLink: fused into the logits / F1 prologue (default), or
    //      a kernel of its own (WHALE_FUSED_GATHER=0)
    gth.x_local = static_cast<const uint4*>(x_local);
    gth.y_local = y_local;
    gth.x_vecs = p.B * p.D * ES / 16;
    gth.B = static_cast<int>(p.B);
    gth.row_off = static_cast<int>(p.Boff[p.rank]);
    gth.row_vecs = p.D * ES / 16;
    gth.rank = p.rank;
    gth.world = p.world;
    gth.parts = gather_grid(p);
    for (int r = 0; r < p.world; ++r) {
      gth.dst_x.p[r] = c->symm[r] + L.xg;
      gth.dst_y.p[r] = c->symm[r] + L.yg;
      gth.flags.p[r] = reinterpret_cast<uint32_t*>(c->symm[r] + L.flags) + FLAG_GATHER * kMaxRanks + p.rank;
    }
    if (c->mc) {
      gth.mc_x = reinterpret_cast<uint4*>(c->mc + L.xg);
      gth.mc_y = reinterpret_cast<int32_t*>(c->mc + L.yg);
      gth.mc_flag = reinterpret_cast<uint32_t*>(c->mc + L.flags) + FLAG_GATHER * kMaxRanks + p.rank;
    }
    yg = reinterpret_cast<const int32_t*>(c->symm[p.rank] + L.yg);
    gather_fused = c->fused_gather;
    if (!gather_fused)
      PROFILED(K_GATHER, s, (launch(c, bridge_gather_kernel, dim3(gth.parts), dim3(256), 0, s, gth,
                                    env_int("WHALE_GATHER_DBG", 0))));
  }
  // ---- A3 logits GEMM with fused row statistics
  if (ES == 2 && p.f1) {
    // F1: logits + statistics + dX partials U in one pass over W_r (fwd_dx_sm100.cuh)
    F1Args a{};
    a.Bt = static_cast<int>(p.Bt);
    a.D = static_cast<int>(p.D);
    a.Dq = p.f1_Dq;
    a.C_r = static_cast<int>(p.Cr);
    a.num_tiles = p.fwd.n_blocks;
    a.stages = p.f1_stages;
    a.s2 = p.f1_s2;
    a.split_issue = env_int("WHALE_F1_SPLIT", 1);
    a.class_offset = p.o_r;
    a.labels = yg;
    a.bias = bias;
    a.m_tile = wsp<float>(c, L.m_tile);
    a.s_tile = wsp<float>(c, L.s_tile);
    a.zy = wsp<float>(c, L.zy);
    a.a_tile = pred != nullptr ? wsp<int32_t>(c, L.a_tile) : nullptr;  // top-1 only when asked for
    a.mx_tile = wsp<float>(c, L.mx_tile);
    a.upart = wsp<float>(c, L.upart);
    a.uref = wsp<float>(c, L.uref);
    a.dev_epoch = dev_epoch;
    a.err = err;
    a.debug = env_int("WHALE_F1_DBG", 0);
    if (p.world > 1) {
      a.wait_flags = reinterpret_cast<const uint32_t*>(c->symm[p.rank] + L.flags) + FLAG_GATHER * kMaxRanks;
      a.wait_count = p.world;
      a.wait_mult = static_cast<uint32_t>(gather_grid(p));
      a.gather_on = gather_fused ? 1 : 0;
      a.gather = gth;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.f1_ncl * kF1KC);
    cfg.blockDim = dim3(kF1Threads);
    cfg.dynamicSmemBytes = p.f1_smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kF1KC;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    c->cur_kbit = 8;  // PDL bit of the logits / F1 launch
    cfg.numAttrs = pdl_for(c) ? 2 : 1;
    PROFILED(K_LOGITS, s, ([&]() -> whale_status_t {
               CUDA_TRY(cudaLaunchKernelEx(&cfg, splitfc_fwd_dx_kernel, c->tmW_f1, c->tmX_f1, c->tmP_f1, a));
               return WHALE_OK;
             }()));
  } else {
    GemmArgs a = base_args(p.fwd, static_cast<int>(p.Bt), static_cast<int>(p.Cr));
    a.dev_epoch = dev_epoch;
    a.labels = yg;
    a.bias = bias;
    a.a_tile = pred != nullptr ? wsp<int32_t>(c, L.a_tile) : nullptr;  // top-1 only when asked for
    a.class_offset = p.o_r;
    a.m_tile = wsp<float>(c, L.m_tile);
    a.s_tile = wsp<float>(c, L.s_tile);
    a.zy = wsp<float>(c, L.zy);
    a.err = err;
    if (p.fwd.p_direct) {
      a.p_direct = c->ws + L.P;
      a.p_ld = static_cast<long long>(p.ldp);
    }
    a.b_keep = c->w_l2 ? 1 : 0;
    if (p.world > 1) {
      a.wait_flags = reinterpret_cast<const uint32_t*>(c->symm[p.rank] + L.flags) + FLAG_GATHER * kMaxRanks;
      a.wait_count = p.world;
      a.wait_mult = static_cast<uint32_t>(gather_grid(p));  // one increment per gather piece
      a.gather_on = gather_fused ? 1 : 0;
      a.gather = gth;
    }
    c->cur_kbit = 8;
    PROFILED(K_LOGITS, s,
             (launch_gemm<EPI_FWD_STATS, false, false, ES>(c, ES == 2 ? 0 : 3, p.fwd, c->tmX_fwd,
                                                           c->tmW_fwd, c->tmP_store, a, s)));
  }
  // ---- A4 + A5 statistics (exchange), combine, loss; A6 either in place (P~ -> G) or, with
  //      the G-fused backward, as the per-(row, tile) factor table the backward applies
  {
    StatsArgs a{};
    a.m_tile = wsp<float>(c, L.m_tile);
    a.s_tile = wsp<float>(c, L.s_tile);
    a.zy_r = wsp<float>(c, L.zy);
    a.y = yg;
    a.T = p.fwd.n_blocks;
    a.Bt = static_cast<int>(p.Bt);
    a.B = static_cast<int>(p.B);
    a.row0 = static_cast<int>(p.Boff[p.rank]);
    a.rank = p.rank;
    a.world = p.world;
    a.o_r = p.o_r;
    a.C_r = p.Cr;
    a.C = p.C;
    if (p.world > 1) {
      for (int r = 0; r < p.world; ++r) a.peer_stats.p[r] = c->symm[r] + L.stats;
      a.my_stats = reinterpret_cast<float4*>(c->symm[p.rank] + L.stats);
    }
    a.dev_epoch = dev_epoch;
    a.lse = wsp<float>(c, L.lse);
    a.row_loss_all = wsp<float>(c, L.row_loss);
    a.loss = loss;
    a.row_loss_local = row_loss;
    a.counter = counters + CNT_STATS;
    a.err = err;
    a.a_tile = pred != nullptr ? wsp<int32_t>(c, L.a_tile) : nullptr;  // top-1 only when asked for
    a.mx_tile = p.f1 ? wsp<float>(c, L.mx_tile) : nullptr;
    a.pred_local = pred;
    a.prob_local = prob;
    // every rewrite CTA re-reads its row's T tile partials (8T bytes): size the chunk so that
    // this stays <= ~10% of the chunk's P~ read+write traffic (4096 B per vector of the 128
    // threads); F1 (B_tot <= 32, 128-class tiles): the re-read comes from L2 and the grid is
    // short (B_tot rows) -> small chunks for enough loads in flight
    a.grad_vecs = static_cast<int>(std::min<int64_t>(64, std::max<int64_t>(4, (p.fwd.n_blocks * 10 + 511) / 512)));
    if (p.f1) a.grad_vecs = env_int("WHALE_F1_GV", 4);
    const int64_t chunk = static_cast<int64_t>(kStatsThreads) * a.grad_vecs * (16 / ES);
    int gy = 1;  // CTAs per row: the statistics CTA (+ G-rewrite CTAs)
    if (c->gfuse) {
      a.gscale = wsp<float>(c, L.gscale);  // NEXT-4b: the backward forms G from P~ itself
      a.chunks = 0;
    } else {
      a.chunks = cdiv(p.Cr, chunk);
      // ranks sharing one device (emulation): keep the grid to a few CTAs per SM of this rank
      const int cap = c->shared_device ? std::max(1, 2 * p.sms / static_cast<int>(p.Bt)) : a.chunks;
      gy = 1 + std::max(1, std::min(a.chunks, cap));
    }
    const float inv_bt = static_cast<float>(1.0 / static_cast<double>(p.Bt));
    void* P = static_cast<void*>(c->ws + L.P);
    if (p.world == 1) {
      // A4-A6 fused: lse, loss and G (or its factors) in one pass (no exchange needed)
      PROFILED(K_STATS, s,
               (c->cur_kbit = 1, launch(c, stats_grad_kernel<ES>, dim3(gy, p.Bt), dim3(kStatsThreads), 0, s, a, P,
                       static_cast<long long>(p.ldp), p.fwd.BN, inv_bt)));
    } else {
      // A4-A6 fused with the per-row cross-GPU exchange (chunk-0 CTAs of every row first)
      // one row per CTA; ranks sharing a device: a few row CTAs (they spin on the peers'
      // records, and spinning CTAs must not crowd out the peers' persistent kernels)
      const int gx = c->shared_device ? std::max(1, std::min(static_cast<int>(p.Bt), p.sms / 8)) : static_cast<int>(p.Bt);
      if (c->shared_device) gy = std::min(gy, 2);
      PROFILED(K_STATS, s,
               (c->cur_kbit = 1, launch(c, stats_grad_multi_kernel<ES>, dim3(gx, gy), dim3(kStatsThreads), 0, s, a, P,
                       static_cast<long long>(p.ldp), p.fwd.BN, inv_bt)));
    }
  }
  return WHALE_OK;
}

extern "C" whale_status_t whale_splitfc_forward(whale_splitfc_ctx* ctx, const void* x_local,
                                                const int32_t* labels_local, const void* w_shard, float* loss,
                                                float* row_loss, void* stream) {
  return whale_splitfc_forward_ex(ctx, x_local, labels_local, w_shard, nullptr, loss, row_loss, nullptr, nullptr,
                                  stream);
}

extern "C" whale_status_t whale_splitfc_forward_ex(whale_splitfc_ctx* ctx, const void* x_local,
                                                   const int32_t* labels_local, const void* w_shard,
                                                   const void* bias_shard, float* loss, float* row_loss,
                                                   int32_t* pred_local, float* prob_local, void* stream) {
  if (!ctx || !w_shard || !loss) return fail(WHALE_ERR_INVALID_ARG, "NULL argument");
  if (ctx->p.B > 0 && (!x_local || !labels_local)) return fail(WHALE_ERR_INVALID_ARG, "NULL x_local / labels_local");
  if (prob_local && !pred_local) return fail(WHALE_ERR_INVALID_ARG, "prob_local requires pred_local");
  if (reinterpret_cast<uintptr_t>(x_local) % 16 || reinterpret_cast<uintptr_t>(w_shard) % 16)
    return fail(WHALE_ERR_INVALID_ARG, "x_local / w_shard must be 16-byte aligned");
  ctx->epoch += 1;
  auto s = static_cast<cudaStream_t>(stream);
  if (ctx->have_fwd) {
    // the previous forward had no backward (forward-only step): end that step's epoch
    uint32_t* dev_epoch = wsp<unsigned>(ctx, ctx->p.L.counters) + CNT_EPOCH;
    whale_status_t sb = launch(ctx, epoch_bump_kernel, dim3(1), dim3(32), 0, s, dev_epoch);
    if (sb != WHALE_OK) return sb;
  }
  whale_status_t st =
      ctx->p.es == 2
          ? forward_impl<2>(ctx, x_local, labels_local, w_shard, bias_shard, loss, row_loss, pred_local, prob_local, s)
          : forward_impl<4>(ctx, x_local, labels_local, w_shard, bias_shard, loss, row_loss, pred_local, prob_local, s);
  if (st == WHALE_OK) ctx->have_fwd = true;
  return st;
}


// Destination of the dX rows this rank sends to owner q (A8 reduce-scatter).  Unicast: slot
// `rank` of q's receive slab (an NVLink store).  NVLS (multicast mapping present): slot q of
// THIS rank's own slab (a local store) -- the owner later reads slot q of every rank summed in
// the NVSwitch (multimem.ld_reduce).  Expressed as the base the kernels index with
// [rank * B_slab + row] * D, so the push code is the same for both.
static uint8_t* rs_dst_base(const whale_splitfc_ctx* c, int q) {
  const Plan& p = c->p;
  if (!c->nvls_rs) return c->symm[q] + p.L.dxrecv;
  const int64_t slab = static_cast<int64_t>(p.Bmax) * p.D * 4;
  return c->symm[p.rank] + p.L.dxrecv + (static_cast<int64_t>(q) - p.rank) * slab;
}

// ============================================================================ backward
template <int ES>
static whale_status_t backward_impl(whale_splitfc_ctx* c, const void* w, void* dx_local, void* dw, float* db,
                                    const float* grad_scale, cudaStream_t s) {
  const Plan& p = c->p;
  const Layout& L = p.L;
  unsigned* counters = wsp<unsigned>(c, L.counters);
  int* err = reinterpret_cast<int*>(counters + CNT_ERR);
  uint32_t* dev_epoch = counters + CNT_EPOCH;
  const int32_t* yg = p.world == 1 ? c->y_fwd : reinterpret_cast<const int32_t*>(c->symm[p.rank] + L.yg);
  {
    whale_status_t st = ensure_w_maps(c, w);
    if (st != WHALE_OK) return st;
  }
  if (dw != c->dw_cached) {
    whale_status_t st = map3d_out(&c->tmDW, dw, p.D, p.Cr, 1, p.dw_bf16 ? 2 : 4);
    if (st != WHALE_OK) return st;
    c->dw_cached = dw;
  }
  // ---- A6 G = (softmax - onehot) / B_tot was produced by the forward's fused stats kernel
  // ---- NEXT-4 bias gradient db_r = sum_i G_r[i, :] (fixed row order, two passes)
  if (db != nullptr) {
    constexpr int V = 16 / ES;
    const int chunks = cdiv(p.Bt, kDbRows);
    float* part = wsp<float>(c, L.dbpart);
    DbFused fz{};
    if (c->gfuse) {  // the buffer still holds P~: form G on the fly (same arithmetic as the rewrite)
      fz.gscale = wsp<float>(c, L.gscale);
      fz.y = yg;
      fz.o_r = p.o_r;
      fz.T = p.fwd.n_blocks;
      fz.BN = p.fwd.BN;
      fz.inv_bt = static_cast<float>(1.0 / static_cast<double>(p.Bt));
    }
    PROFILED(K_DB, s,
             (launch(c, bias_grad_part_kernel<ES>, dim3(cdiv(cdiv(p.Cr, V), 128), chunks), dim3(128), 0, s,
                     static_cast<const void*>(c->ws + L.P), static_cast<long long>(p.ldp), static_cast<int>(p.Bt),
                     static_cast<long long>(p.Cr), part, fz)));
    PROFILED(K_DB, s,
             (launch(c, bias_grad_sum_kernel, dim3(std::max(1, std::min(cdiv(p.Cr, 256), 4 * p.sms))), dim3(256), 0,
                     s, static_cast<const float*>(part), chunks, static_cast<long long>(p.Cr), db, grad_scale)));
  }
  // ---- A8 args: fused split-K fixup; N = 1 writes dX, N > 1 pushes rows to their owners
  GemmArgs ax = base_args(p.dx, static_cast<int>(p.Bt), static_cast<int>(p.D));
  ax.err = err;
  ax.grad_scale = grad_scale;
  ax.part = wsp<float>(c, L.dxpart);
  ax.st_out = wsp<float>(c, L.dxpart);
  ax.tile_cnt = wsp<uint32_t>(c, L.tile_cnt);
  ax.done_cnt = counters + CNT_DONE;
  ax.dev_epoch = dev_epoch;
  ax.bump_epoch = 1;  // the dX launch (or the fused launch) ends the step
  ax.rs_signal = p.world > 1 ? 1 : 0;
  ax.B = static_cast<int>(p.Bmax);
  for (int r = 0; r <= p.world; ++r) ax.row_off[r] = static_cast<int>(p.Boff[r]);
  ax.rank = p.rank;
  ax.world = p.world;
  if (p.world == 1) {
    ax.fix_mode = FIX_LOCAL;
    ax.out = dx_local;
  } else {
    ax.fix_mode = FIX_PUSH;
    for (int r = 0; r < p.world; ++r) {
      ax.recv.p[r] = rs_dst_base(c, r);
      ax.rs_flags.p[r] = reinterpret_cast<uint32_t*>(c->symm[r] + L.flags) + FLAG_RS * kMaxRanks + p.rank;
    }
  }
  if (ES == 2 && p.f1 && !c->fused_bwd) {
    // ---- A8 from the forward's U partials: dX = (1/B_tot)(sum_cl e^{ref - lse} U_cl - W_y)
    //      (with the fused backward these are work units of the backward kernel instead)
    RowSplit rs{};
    PeerPtrs recv{};
    for (int r = 0; r <= p.world; ++r) rs.off[r] = static_cast<int>(p.Boff[r]);
    if (p.world > 1)
      for (int r = 0; r < p.world; ++r) recv.p[r] = rs_dst_base(c, r);
    PROFILED(K_DX, s,
             (launch(c, dx_combine_kernel<2>, dim3(cdiv(p.D / 4, 32), static_cast<unsigned>(p.Bt)), dim3(256), 0,
                     s, static_cast<const float*>(wsp<float>(c, L.upart)),
                     static_cast<const float*>(wsp<float>(c, L.uref)), p.f1_ncl, static_cast<int>(p.Bt),
                     static_cast<int>(p.D), static_cast<const float*>(wsp<float>(c, L.lse)), yg,
                     static_cast<long long>(p.o_r), static_cast<long long>(p.Cr), w,
                     static_cast<float>(1.0 / static_cast<double>(p.Bt)), dx_local, recv, rs, p.rank, p.world,
                     static_cast<int>(p.Bmax), grad_scale)));
  }
  if (ES == 2 && c->fused_bwd) {
    // ---- A7 + A8 in one persistent launch: dX units first (one per CTA), then dW tiles
    //      (F1: dX came from the forward -> dW tiles only)
    BwdArgs b{};
    b.dx = ax;
    b.dw = base_args(p.dw, static_cast<int>(p.Cr), static_cast<int>(p.D));
    b.dw.dev_epoch = dev_epoch;
    // dW tiles N-fastest: CTAs running together share one G^T class block (read from HBM
    // once) across all D-column blocks; M-fastest re-read G once per column block (c5: 16x)
    b.dw.n_fastest = g_dw_m_fastest ? 0 : 1;
    b.dw.err = err;
    b.ux = p.f1 ? 0 : p.dx.num_tiles;
    b.tw = p.dw.num_tiles;
    if (p.f1) {  // F1: dX = (1/B_tot)(sum_cl e^{ref - lse} U_cl - W_y) as the schedule's last units
      CombineArgs& cb = b.cb;
      cb.upart = wsp<float>(c, L.upart);
      cb.uref = wsp<float>(c, L.uref);
      cb.ncl = p.f1_ncl;
      cb.Bt = static_cast<int>(p.Bt);
      cb.D = static_cast<int>(p.D);
      cb.parts = cdiv(p.D, kCombineCols);
      cb.lse = wsp<float>(c, L.lse);
      cb.y = yg;
      cb.o_r = p.o_r;
      cb.C_r = p.Cr;
      cb.w = w;
      cb.inv_bt = static_cast<float>(1.0 / static_cast<double>(p.Bt));
      cb.dx_out = dx_local;
      for (int r = 0; r <= p.world; ++r) cb.row_off[r] = static_cast<int>(p.Boff[r]);
      if (p.world > 1)
        for (int r = 0; r < p.world; ++r) cb.recv.p[r] = rs_dst_base(c, r);
      cb.rank = p.rank;
      cb.world = p.world;
      cb.Bslab = static_cast<int>(p.Bmax);
      cb.grad_scale = grad_scale;
      b.tc = static_cast<int>(p.Bt) * cb.parts;
    }
    if (c->gfuse) {  // NEXT-4b: the transformer warps turn each P~ operand stage into G
      GFuse& gf = b.gf;
      gf.gscale = wsp<float>(c, L.gscale);
      gf.y = yg;
      gf.o_r = p.o_r;
      gf.C_r = p.Cr;
      gf.T = p.fwd.n_blocks;
      gf.fwd_bn = p.fwd.BN;
      gf.Bt = static_cast<int>(p.Bt);
      gf.inv_bt = static_cast<float>(1.0 / static_cast<double>(p.Bt));
    }
    b.row_bulk = c->row_bulk ? 1 : 0;
    b.dw_bf16 = p.dw_bf16 ? 1 : 0;
    b.dw_ptr = dw;
    b.dw_ld = static_cast<int>(p.D);
    b.stages = c->bwd_stages;
    b.stage_bytes = c->bwd_stage_bytes;
    b.epi_bufs = c->bwd_epi_bufs;
    b.sched_cnt = counters + CNT_SCHED;
    b.w_last_use = c->w_l2 ? 1 : 0;
    if (p.world > 1 && c->fused_reduce) {  // A8 owner side in the backward's tail
      b.red_on = 1;
      b.red_recv = reinterpret_cast<const float4*>(c->symm[p.rank] + L.dxrecv);
      b.red_mc = c->nvls_rs ? reinterpret_cast<const float4*>(c->mc + L.dxrecv + static_cast<size_t>(p.rank) * p.Bmax * p.D * 4)
                            : nullptr;
      b.red_flags = reinterpret_cast<const uint32_t*>(c->symm[p.rank] + L.flags) + FLAG_RS * kMaxRanks;
      b.red_out = dx_local;
      b.red_B = static_cast<int>(p.B);
      b.red_Bslab = static_cast<int>(p.Bmax);
    }
    if (c->bwd_pair) {  // CTA pairs: units are pair tiles, the grid is 2-CTA clusters
      b.ux = p.dx.num_tiles / 2;
      b.tw = p.dw.num_tiles / 2;
      const int grid = 2 * std::min(b.ux + b.tw, p.sms / 2);
      auto kern = p.dw_bf16 ? splitfc_bwd_kernel<2, true, true> : splitfc_bwd_kernel<2, false, true>;
      {
        const whale_status_t st = ensure_smem_attr(kern, p.dw_bf16 ? 19 : 18);
        if (st != WHALE_OK) return st;
      }
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(kBwdThreads);
      cfg.dynamicSmemBytes = c->bwd_smem;
      cfg.stream = s;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      c->cur_kbit = 2;
      cfg.numAttrs = pdl_for(c) ? 2 : 1;
      PROFILED(K_BWD, s, ([&]() -> whale_status_t {
                 CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, c->tmG_dx, c->tmW_dx, c->tmDxPart, c->tmG_dw, c->tmX_dw,
                                             c->tmDW, b));
                 return WHALE_OK;
               }()));
    } else {
      const int grid = std::min(b.ux + b.tw + b.tc, p.sms);
      auto kern = p.dw_bf16 ? splitfc_bwd_kernel<2, true> : splitfc_bwd_kernel<2, false>;
      {
        const whale_status_t st = ensure_smem_attr(kern, p.dw_bf16 ? 9 : 8);
        if (st != WHALE_OK) return st;
      }
      PROFILED(K_BWD, s,
               (c->cur_kbit = 2, launch(c, kern, dim3(grid), dim3(kBwdThreads), c->bwd_smem, s, c->tmG_dx, c->tmW_dx, c->tmDxPart,
                       c->tmG_dw, c->tmX_dw, c->tmDW, b)));
    }
  } else if constexpr (ES == 2) {
    // ---- A7 dW_r = G_r^T X  (A = G^T MN-major, B = X MN-major); on the F1 path dX came from
    //      the combine kernel above, so this launch ends the step
    {
      GemmArgs a = base_args(p.dw, static_cast<int>(p.Cr), static_cast<int>(p.D));
      a.dev_epoch = dev_epoch;
      a.err = err;
      a.grad_scale = grad_scale;
      a.st_out = static_cast<float*>(dw);
      if (p.f1) {
        a.bump_epoch = 1;
        a.done_cnt = ax.done_cnt;
        a.rs_signal = ax.rs_signal;
        a.rs_flags = ax.rs_flags;
        a.world = p.world;
      }
      PROFILED(K_DW, s,
               (launch_gemm<EPI_STORE_F32, true, true, 2>(c, 1, p.dw, c->tmG_dw, c->tmX_dw, c->tmDW, a, s)));
    }
    // ---- A8 dX = G_r W_r  (A = G K-major, B = W_r MN-major), split-K + fused fixup
    if (!p.f1)
      PROFILED(K_DX, s,
               (launch_gemm<EPI_STORE_F32, false, true, 2>(c, 2, p.dx, c->tmG_dx, c->tmW_dx, c->tmDxPart, ax, s)));
  } else {
    // kind::tf32 accepts K-major operands only (plain 128B swizzle): transpose G, X, W_r.
    const void* xg = p.world == 1 ? c->x_fwd : static_cast<const void*>(c->symm[p.rank] + L.xg);
    auto tr = [&](const void* src, long long sld, void* dst, long long dld, int64_t R, int64_t Cc) -> whale_status_t {
      return launch(c, transpose_f32_kernel, dim3(cdiv(Cc, 32), cdiv(R, 32)), dim3(32, 32), 0, s,
                    static_cast<const float*>(src), sld, static_cast<float*>(dst), dld, static_cast<int>(R),
                    static_cast<int>(Cc));
    };
    PROFILED(K_TRANSPOSE, s, (tr(c->ws + L.P, p.ldp, c->ws + L.GT, L.ld_bt, p.Bt, p.Cr)));
    PROFILED(K_TRANSPOSE, s, (tr(xg, p.D, c->ws + L.XT, L.ld_bt, p.Bt, p.D)));
    PROFILED(K_TRANSPOSE, s, (tr(w, p.D, c->ws + L.WT, p.ldp, p.Cr, p.D)));
    {
      GemmArgs a = base_args(p.dw, static_cast<int>(p.Cr), static_cast<int>(p.D));
      a.dev_epoch = dev_epoch;
      a.err = err;
      a.grad_scale = grad_scale;
      a.st_out = static_cast<float*>(dw);
      PROFILED(K_DW, s, (launch_gemm<EPI_STORE_F32, false, false, 4>(c, 4, p.dw, c->tmGT, c->tmXT, c->tmDW, a, s)));
    }
    PROFILED(K_DX, s,
             (launch_gemm<EPI_STORE_F32, false, false, 4>(c, 5, p.dx, c->tmG_dx, c->tmWT, c->tmDxPart, ax, s)));
  }
  // ---- A8 owner side of the reduce-scatter (N > 1), unless the fused backward did it
  if (p.world > 1 && !(ES == 2 && c->fused_bwd && c->fused_reduce)) {
    const int64_t own = p.B * p.D / 4;
    const int g2 = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(cdiv(own, 256), c->shared_device ? std::max(1, p.sms / 8) : 2 * p.sms)));
    const uint32_t* my_flags = reinterpret_cast<const uint32_t*>(c->symm[p.rank] + L.flags) + FLAG_RS * kMaxRanks;
    // NVLS: slot `rank` of every rank's slab, summed in the switch (multicast view)
    const float4* mc_mine =
        c->nvls_rs ? reinterpret_cast<const float4*>(c->mc + L.dxrecv + static_cast<size_t>(p.rank) * p.Bmax * p.D * 4)
                   : nullptr;
    PROFILED(K_RS_REDUCE, s,
             (c->cur_kbit = 4, launch(c, dx_reduce_kernel<ES>, dim3(g2), dim3(256), 0, s,
                     reinterpret_cast<const float4*>(c->symm[p.rank] + L.dxrecv), static_cast<int>(p.B),
                     static_cast<int>(p.Bmax), static_cast<int>(p.D), p.world, my_flags, static_cast<const uint32_t*>(dev_epoch), dx_local,
                     err, mc_mine)));
  }
  return WHALE_OK;
}

extern "C" whale_status_t whale_splitfc_backward(whale_splitfc_ctx* ctx, const void* w_shard, void* dx_local,
                                                 void* dw_shard, void* stream) {
  return whale_splitfc_backward_ex(ctx, w_shard, dx_local, dw_shard, nullptr, stream);
}

extern "C" whale_status_t whale_splitfc_backward_ex(whale_splitfc_ctx* ctx, const void* w_shard, void* dx_local,
                                                    void* dw_shard, float* db_shard, void* stream) {
  return whale_splitfc_backward_scaled(ctx, w_shard, dx_local, dw_shard, db_shard, nullptr, stream);
}

extern "C" whale_status_t whale_splitfc_backward_scaled(whale_splitfc_ctx* ctx, const void* w_shard, void* dx_local,
                                                        void* dw_shard, float* db_shard, const float* grad_scale,
                                                        void* stream) {
  if (!ctx || !w_shard || !dw_shard) return fail(WHALE_ERR_INVALID_ARG, "NULL argument");
  if (ctx->p.B > 0 && !dx_local) return fail(WHALE_ERR_INVALID_ARG, "NULL dx_local");
  if (!ctx->have_fwd) return fail(WHALE_ERR_STATE, "backward called before forward");
  if (reinterpret_cast<uintptr_t>(dx_local) % 16 || reinterpret_cast<uintptr_t>(dw_shard) % 16)
    return fail(WHALE_ERR_INVALID_ARG, "dx_local / dw_shard must be 16-byte aligned");
  auto s = static_cast<cudaStream_t>(stream);
  whale_status_t st = ctx->p.es == 2 ? backward_impl<2>(ctx, w_shard, dx_local, dw_shard, db_shard, grad_scale, s)
                                     : backward_impl<4>(ctx, w_shard, dx_local, dw_shard, db_shard, grad_scale, s);
  if (st == WHALE_OK) ctx->have_fwd = false;
  return st;
}

extern "C" whale_status_t whale_splitfc_check(whale_splitfc_ctx* ctx, void* stream) {
  if (!ctx) return fail(WHALE_ERR_INVALID_ARG, "NULL ctx");
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  int* err = reinterpret_cast<int*>(wsp<unsigned>(ctx, ctx->p.L.counters) + CNT_ERR);
  int h = 0;
  CUDA_TRY(cudaMemcpy(&h, err, sizeof(int), cudaMemcpyDeviceToHost));
  if (h) CUDA_TRY(cudaMemset(err, 0, sizeof(int)));
  if (h & ERR_LABEL) return fail(WHALE_ERR_LABEL, "a label is outside [0, C)");
  if (h & (ERR_COMM | ERR_SPLITK))
    return fail(WHALE_ERR_COMM, "a wait timed out (error bits 0x%x:%s%s%s%s); destroy and re-create the context on every rank",
                h, (h & ERR_AT_GATHER) ? " bridge-gather flags" : "", (h & ERR_AT_STATS) ? " statistics records" : "",
                (h & ERR_AT_RS) ? " reduce-scatter flags" : "", (h & ERR_SPLITK) ? " split-K counters" : "");
  return WHALE_OK;
}

// ============================================================================ introspection
extern "C" int32_t whale_splitfc_launches_per_step(const whale_splitfc_ctx* ctx) {
  if (!ctx) return 0;
  // N = 1: logits, stats+grad, dW, dX;  N > 1: + gather, + dX owner reduce
  int base = ctx->p.world == 1 ? 4 : 6;
  if (ctx->fused_bwd) base -= 1;  // dW + dX share one launch (F1: dW tiles + dX combine units)
  if (ctx->p.world > 1 && ctx->fused_gather) base -= 1;  // the gather runs in the logits / F1 prologue
  if (ctx->p.world > 1 && ctx->fused_bwd && ctx->fused_reduce && ctx->p.es == 2) base -= 1;  // owner reduce in the backward
  // F1 unfused: the combine kernel replaces the dX GEMM (same count)
  return base + (ctx->p.es == 4 ? 3 : 0);  // fp32 path: operand transposes
}

extern "C" whale_status_t whale_splitfc_profile_enable(whale_splitfc_ctx* ctx, int32_t enable) {
  if (!ctx) return fail(WHALE_ERR_INVALID_ARG, "NULL ctx");
  ctx->profile = enable != 0;
  return WHALE_OK;
}

extern "C" whale_status_t whale_splitfc_profile_read(whale_splitfc_ctx* ctx, char* names, size_t names_len,
                                                     double* total_ms, int64_t* launches, int32_t max_kinds,
                                                     int32_t* n_kinds) {
  if (!ctx) return fail(WHALE_ERR_INVALID_ARG, "NULL ctx");
  for (auto& r : ctx->prof) {
    CUDA_TRY(cudaEventSynchronize(r.b));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, r.a, r.b));
    ctx->prof_ms[r.kind] += ms;
    ctx->prof_n[r.kind] += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  ctx->prof.clear();
  std::string nm;
  const int n = std::min<int>(K_NUM, max_kinds);
  for (int k = 0; k < n; ++k) {
    if (total_ms) total_ms[k] = ctx->prof_ms[k];
    if (launches) launches[k] = ctx->prof_n[k];
    nm += kKindNames[k];
    if (k + 1 < n) nm += ";";
    ctx->prof_ms[k] = 0;
    ctx->prof_n[k] = 0;
  }
  if (names && names_len) {
    strncpy(names, nm.c_str(), names_len - 1);
    names[names_len - 1] = 0;
  }
  if (n_kinds) *n_kinds = n;
  return WHALE_OK;
}

extern "C" whale_status_t whale_splitfc_config(const whale_splitfc_ctx* ctx, char* buf, size_t buf_len) {
  if (!ctx || !buf) return fail(WHALE_ERR_INVALID_ARG, "NULL argument");
  const Plan& p = ctx->p;
  auto g = [](const GemmCfg& c) {
    char b[320];
    snprintf(b, sizeof(b),
             "{\"BN\":%d,\"bk\":%d,\"m_blocks\":%d,\"n_blocks\":%d,\"splits\":%d,\"num_kb\":%d,\"kb_per_split\":%d,"
             "\"tiles\":%d,\"stages\":%d,\"epi_bufs\":%d,\"smem\":%d,\"grid\":%d,\"cluster\":%d}",
             c.BN, c.bk, c.m_blocks, c.n_blocks, c.splits, c.num_kb, c.kb_per_split, c.num_tiles, c.stages, c.epi_bufs,
             c.smem, c.grid, c.cluster);
    return std::string(b);
  };
  char head[320];
  snprintf(head, sizeof(head),
           "{\"rank\":%d,\"world\":%d,\"B\":%lld,\"Bt\":%lld,\"D\":%lld,\"C\":%lld,\"C_r\":%lld,\"o_r\":%lld,"
           "\"ldp\":%lld,\"sms\":%d,\"es\":%d,\"pdl\":%d,",
           p.rank, p.world, (long long)p.B, (long long)p.Bt, (long long)p.D, (long long)p.C, (long long)p.Cr,
           (long long)p.o_r, (long long)p.ldp, p.sms, p.es, ctx->pdl ? 1 : 0);
  std::string s = std::string(head) + "\"fwd\":" + g(p.fwd) + ",\"dw\":" + g(p.dw) + ",\"dx\":" + g(p.dx) +
                  ",\"off_P\":" + std::to_string(p.L.P) + ",\"off_m_tile\":" + std::to_string(p.L.m_tile) +
                  ",\"off_s_tile\":" + std::to_string(p.L.s_tile) + ",\"off_lse\":" + std::to_string(p.L.lse) +
                  ",\"off_dxpart\":" + std::to_string(p.L.dxpart) + ",\"f1\":" + std::to_string(p.f1 ? 1 : 0) +
                  ",\"f1_clusters\":" + std::to_string(p.f1_ncl) + ",\"f1_stages\":" + std::to_string(p.f1_stages) +
                  ",\"nvls\":" + std::to_string(ctx->mc != nullptr ? 1 : 0) +
                  ",\"nvls_rs\":" + std::to_string(ctx->nvls_rs ? 1 : 0) +
                  ",\"fused_bwd\":" + std::to_string(ctx->fused_bwd ? 1 : 0) +
                  ",\"bwd_pair\":" + std::to_string(ctx->bwd_pair ? 1 : 0) +
                  ",\"bwd_stages\":" + std::to_string(ctx->bwd_stages) +
                  ",\"bwd_epi_bufs\":" + std::to_string(ctx->bwd_epi_bufs) +
                  ",\"fused_gather\":" + std::to_string(ctx->fused_gather ? 1 : 0) +
                  ",\"w_l2\":" + std::to_string(ctx->w_l2 ? 1 : 0) +
                  ",\"local_bytes\":" + std::to_string(p.L.local_total) +
                  ",\"symm_bytes\":" + std::to_string(p.L.symm_total) + "}";
  if (s.size() + 1 > buf_len) return fail(WHALE_ERR_INVALID_ARG, "buffer too small (%zu)", s.size() + 1);
  memcpy(buf, s.c_str(), s.size() + 1);
  return WHALE_OK;
}

// Internal (not in the public header): debug timestamps written by kernels run with
// WHALE_GATHER_DBG & 16.  Synchronises the device.
extern "C" int whale_debug_timestamps(unsigned long long* out, int n) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(out, g_dbg_ts, sizeof(unsigned long long) * std::min(n, 32)) != cudaSuccess) return -1;
  return 0;
}

// Internal: device-side kernel windows (see TraceScope).  enable != 0 clears and arms the
// tracer; whale_debug_trace_read copies [16][2] (start, end) ns and re-arms (clears).
extern "C" int whale_debug_trace_enable(int enable) {
  unsigned int on = enable ? 1u : 0u;
  unsigned long long init[16][2];
  for (int k = 0; k < 16; ++k) {
    init[k][0] = ~0ull;
    init[k][1] = 0ull;
  }
  if (cudaMemcpyToSymbol(g_trace, init, sizeof(init)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(g_trace_on, &on, sizeof(on)) != cudaSuccess) return -1;
  return 0;
}
extern "C" int whale_debug_trace_read(unsigned long long* out) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * 32) != cudaSuccess) return -1;
  return whale_debug_trace_enable(1);
}

// Internal (not in the public header): how many KC-CTA clusters of the F1 kernel with
// `smem` dynamic bytes can be co-resident on this device (cudaOccupancyMaxActiveClusters).
extern "C" int whale_debug_f1_max_clusters(int smem) {
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, splitfc_fwd_dx_kernel) != cudaSuccess) return -1;
  if (cudaFuncSetAttribute(splitfc_fwd_dx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSmemLimit - static_cast<int>(fa.sharedSizeBytes)) != cudaSuccess)
    return -2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(kF1Threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kF1KC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, splitfc_fwd_dx_kernel, &cfg) != cudaSuccess) return -3;
  return n;
}

// Internal: read the logits debug timeline (160 CTAs x {entry, after prologue, last load issued,
// last MMA commit, first accumulator in the epilogue, epilogue done}; WHALE_EPI_DEBUG=16).
extern "C" int whale_debug_gemm_timeline(unsigned long long* out) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  return cudaMemcpyFromSymbol(out, g_gemm_cta, sizeof(g_gemm_cta)) == cudaSuccess ? 0 : -2;
}

// Internal: read the backward debug timeline (160 CTAs x {start, dX unit done, epilogue done,
// GEMM units}; WHALE_EPI_DEBUG=16).  Synchronises the device.
extern "C" int whale_debug_bwd_timeline(unsigned long long* out) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  return cudaMemcpyFromSymbol(out, g_bwd_cta, sizeof(g_bwd_cta)) == cudaSuccess ? 0 : -2;
}

// Internal: read the F1 debug timeline (64 periods x 16 stamps, then 160 CTAs x {entry, start, end,
// after cluster sync, exit}, ns).  Synchronises the device.
extern "C" int whale_debug_f1_timeline(unsigned long long* out) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(out, g_f1_ts, sizeof(g_f1_ts)) != cudaSuccess) return -2;
  return cudaMemcpyFromSymbol(out + 1024, g_f1_cta, sizeof(g_f1_cta)) == cudaSuccess ? 0 : -3;
}
