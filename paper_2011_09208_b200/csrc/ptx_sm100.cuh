// Thin inline-PTX wrappers for sm_100a: mbarrier, TMA (cp.async.bulk.tensor), tcgen05
// (TMEM alloc / MMA / commit / ld), UMMA shared-memory & instruction descriptors, and
// system-scope flag operations used by the NVLink exchange kernels.
//
// Only PTX that exists on sm_100a is used (no tcgen05.ld.red, no wgmma).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace whale {

// Timing experiments that SKIP work (results wrong: no A loads, no MMAs, no stores, no
// peer stores ...) exist only in builds with -DWHALE_TIMING_EXPERIMENTS (scripts/); the
// product library compiles them out.  Timestamp-only debug modes stay runtime switches.
#ifdef WHALE_TIMING_EXPERIMENTS
#define WHALE_SKIP(bits) (bits)
#else
#define WHALE_SKIP(bits) 0
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ spin guards
// Every spin loop is bounded (wall clock, %globaltimer).
//  * Waits on OTHER ranks or other CTAs (flags, LL words, split-K counters) give up after
//    g_wait_timeout_ns: they set the error bit in the workspace error word and return, the
//    kernel finishes its (now meaningless) work and still raises its own flags, so peers
//    are not left spinning; whale_splitfc_check() then reports WHALE_ERR_COMM.  Once the
//    error word holds a wait-timeout bit, later waits of the same step give up at once.
//  * Waits inside one CTA (mbarriers of the TMA / MMA pipelines) cannot time out unless
//    the kernel itself is broken; those trap (after the peer timeout + 10 s, as they may
//    legitimately sit behind a peer wait of the same kernel) instead of hanging.
__device__ unsigned long long g_wait_timeout_ns = 300ull * 1000000000ull;  // set by whale_splitfc_create
__device__ __forceinline__ unsigned long long wall_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Error word bits (workspace; whale_splitfc_check decodes them).  A timed-out wait raises
// ERR_COMM or ERR_SPLITK plus the bit of its site.
enum ErrBits : int {
  ERR_LABEL = 1,          // a label outside [0, C)
  ERR_COMM = 8,           // a wait on another rank timed out
  ERR_SPLITK = 16,        // a split-K fixup counter wait (this rank's own CTAs) timed out
  ERR_AT_GATHER = 32,     //   ... on the bridge all-gather flags (logits / F1 kernel)
  ERR_AT_STATS = 64,      //   ... on the statistics records (stats kernel)
  ERR_AT_RS = 128,        //   ... on the dX reduce-scatter flags (owner reduce)
};
constexpr int kErrWaitMask = ERR_COMM | ERR_SPLITK;
struct SpinGuard {
  unsigned long long start;
  unsigned n = 0;
  __device__ __forceinline__ SpinGuard() : start(wall_ns()) {}
  // true: stop waiting (timed out now, or an earlier wait of this step already did)
  __device__ __forceinline__ bool expired(int* err_word, int code) {
    if ((++n & 63u) != 0u) return false;  // poll the clock / error word every 64 spins
    if (err_word && (*reinterpret_cast<volatile int*>(err_word) & kErrWaitMask)) return true;
    if (wall_ns() - start > *reinterpret_cast<volatile unsigned long long*>(&g_wait_timeout_ns)) {
      if (err_word) atomicOr(err_word, code);
      return true;
    }
    return false;
  }
  // intra-CTA pipeline waits: a timeout is an internal bug -> trap
  __device__ __forceinline__ void check_internal() {
    if ((++n & 1023u) != 0u) return;
    // a peer wait upstream may legitimately take the whole peer timeout first
    if (wall_ns() - start > *reinterpret_cast<volatile unsigned long long*>(&g_wait_timeout_ns) + 10000000000ull)
      __trap();
  }
};

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe (never suspends the thread): for issuers that poll several barriers.
__device__ __forceinline__ bool mbar_test(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  SpinGuard g;
  while (!mbar_try_wait(a, parity)) g.check_internal();
}

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const void* map, uint64_t* bar, int c0, int c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_store_2d(const void* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const void* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// 1-D bulk copy shared -> global (16-byte aligned addresses, bytes % 16 == 0), bulk_group.
__device__ __forceinline__ void bulk_store_1d(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------------ tcgen05 / TMEM
__device__ __forceinline__ void tmem_alloc(uint32_t* holder_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(holder_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 inputs, fp32 accumulate); one thread issues.
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// kind::tf32 (fp32 storage, tf32 multiply, fp32 accumulate)
__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// Same, arriving on the mbarrier at the same smem offset in every CTA of `mask` (cluster).
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// ------------------------------------------------------------------ clusters
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ncluster_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Cluster barrier without release semantics: no MEMBAR, so it does not wait for this
// thread's outstanding global stores (F1's exit barrier took ~12 us with .release while the
// CTA's U write-out drained).  Use only where nothing but the barrier itself is ordered.
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
// TMA load multicast to the same smem offset (and mbarrier offset) of every CTA in `mask`.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const void* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// ------------------------------------------------------------------ CTA pairs (cta_group::2)
// A pair of CTAs in one cluster (same TPC) runs ONE M = 256 MMA: CTA r holds rows [128 r, +128)
// of A and columns [N/2 r, +N/2) of B in its own shared memory (at the same offsets), and its
// half of the accumulator (128 lanes x N columns) in its own TMEM.  Only CTA 0 issues the MMA.
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* holder_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(holder_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_tf32_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (once the pair's prior MMAs complete) on the mbarrier at this offset in every CTA of mask.
__device__ __forceinline__ void umma_commit_pair_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// TMA load into this CTA's smem whose completion bytes count on the mbarrier `bar_cluster`
// (a shared::cluster address -- the pair leader's barrier).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* map, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote_release(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}

// 32 lanes x 32b, 32 consecutive columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version field = 1.
//   K-major: 8-row x 128-byte swizzle atoms stacked along M/N at SBO; LBO unused (16 B).
//   MN-major: 64-element x 8-K-row atoms; LBO = stride between atoms along M/N,
//             SBO = stride between 8-row groups along K.
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor for kind::f16 (fmt 1 = bf16) / kind::tf32 (fmt 2), fp32 accumulator.
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N, bool a_mn, bool b_mn, uint32_t fmt) {
  return (1u << 4)                                   // D format F32
         | (fmt << 7) | (fmt << 10)                  // A, B format
         | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16)
         | (static_cast<uint32_t>(N >> 3) << 17)     // N >> 3
         | (static_cast<uint32_t>(M >> 4) << 24);    // M >> 4
}

// ------------------------------------------------------------------ flags (NVLink exchange)
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Remote counter increment with release semantics (orders this thread's prior writes,
// and -- after a CTA barrier -- the CTA's, before the count becomes visible to the peer).
__device__ __forceinline__ void red_add_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Relaxed remote increment: callers order their data with an explicit fence.sc.sys first
// (measured: a release-red costs ~3.5 us each on NVLink; fence + relaxed reds ~2.5 us total).
__device__ __forceinline__ void red_add_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// NVLS multimem (NVSwitch multicast): one store / reduction reaches the same offset in every
// rank's buffer of a multicast object; `mc` is an address inside the multicast mapping.
__device__ __forceinline__ void multimem_st_v4(void* mc, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void multimem_st_u32(void* mc, uint32_t v) {
  asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}
__device__ __forceinline__ void multimem_red_add_release_u32(void* mc, uint32_t v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}
// Load of the same 16 bytes from every rank's buffer, summed in the NVSwitch.
__device__ __forceinline__ float4 multimem_ld_reduce_add_v4f32(const void* mc) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}
__device__ __forceinline__ void multimem_red_add_relaxed_u32(void* mc, uint32_t v) {
  asm volatile("multimem.red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}

// LL protocol word: {data (low 32), flag (high 32)} written by one aligned 64-bit store, which
// is single-copy atomic -- the reader validates the data by its flag half (NCCL's LL idea).
__device__ __forceinline__ void st_relaxed_sys_v2(uint2* p, uint32_t data, uint32_t flag) {
  const unsigned long long w = (static_cast<unsigned long long>(flag) << 32) | data;
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Spin until the LL word carries `flag`; returns its data half (on a timeout: whatever the
// word holds, with `code` raised in the error word).
__device__ __forceinline__ uint32_t wait_ll(const uint2* p, uint32_t flag, int* err_word, int code) {
  unsigned long long w = ld_relaxed_sys_u64(p);
  if (static_cast<uint32_t>(w >> 32) != flag) {
    SpinGuard g;
    do {
      __nanosleep(20);
      if (g.expired(err_word, code)) break;
      w = ld_relaxed_sys_u64(p);
    } while (static_cast<uint32_t>(w >> 32) != flag);
  }
  return static_cast<uint32_t>(w);
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Wait until *p >= epoch (monotonic epochs); gives up (error word) after the wait timeout.
__device__ __forceinline__ void wait_flag_geq(const uint32_t* p, uint32_t epoch, int* err_word, int code) {
  if (static_cast<int32_t>(ld_acquire_sys(p) - epoch) >= 0) return;
  SpinGuard g;
  while (static_cast<int32_t>(ld_acquire_sys(p) - epoch) < 0) {
    __nanosleep(40);  // many CTAs may poll: keep L2 / NVLink free for the incoming data
    if (g.expired(err_word, code)) return;
  }
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Programmatic dependent launch: wait for the preceding grid's memory, and let the next
// grid be scheduled early (its own griddepcontrol.wait keeps it correct).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Named barrier over a subset of warps (id > 0; id 0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ device-side tracer
// Per kernel kind: earliest CTA start and latest CTA end on the device clock (globaltimer),
// accumulated with atomicMin/Max when g_trace_on (whale_debug_trace*); no cost when off.
__device__ unsigned int g_trace_on;
__device__ unsigned long long g_trace[16][2];
__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct TraceScope {
  int kind;
  bool on;
  __device__ __forceinline__ explicit TraceScope(int k) : kind(k), on(false) {
    if (threadIdx.x == 0 && threadIdx.y == 0 && *(volatile unsigned int*)&g_trace_on) {
      on = true;
      atomicMin(&g_trace[kind][0], gtime_ns());
    }
  }
  __device__ __forceinline__ ~TraceScope() {
    if (on) atomicMax(&g_trace[kind][1], gtime_ns());
  }
};

constexpr int kMaxRanks = 8;
struct PeerPtrs {
  void* p[kMaxRanks];
};
struct PeerFlags {
  uint32_t* p[kMaxRanks];
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ DSMEM (cluster shared memory)
// Address of the same smem location in CTA `rank` of this cluster (shared::cluster window).
__device__ __forceinline__ uint32_t mapa_smem(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// 16-byte asynchronous store into a peer CTA's smem; completes `bytes` on the peer's mbarrier.
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, uint32_t remote_bar, uint32_t a, uint32_t b,
                                            uint32_t c, uint32_t d) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(remote_addr),
      "r"(a), "r"(b), "r"(c), "r"(d), "r"(remote_bar)
      : "memory");
}
// 4-byte asynchronous store into a peer CTA's smem; completes 4 bytes on the peer's mbarrier.
__device__ __forceinline__ void st_async_u32(uint32_t remote_addr, uint32_t remote_bar, uint32_t v) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(remote_addr), "r"(v),
               "r"(remote_bar)
               : "memory");
}
// Arrive on a peer CTA's mbarrier and raise its expected transaction bytes (relaxed: the bytes
// themselves come with their own complete_tx, e.g. st.async).
__device__ __forceinline__ void mbar_arrive_expect_tx_remote(uint32_t remote_bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(remote_bar), "r"(tx)
               : "memory");
}
// Arrive on an mbarrier of a peer CTA.  Relaxed: used only to say "I have consumed the data
// you wrote into my smem" after the values were loaded into registers (and a CTA barrier),
// which needs no memory ordering; .release would emit a GPU-scope MEMBAR that waits for
// every outstanding global store of the thread (microseconds under load).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
// Wait with acquire at cluster scope (data written by peer CTAs before their arrive / st.async).
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait_cluster(a, parity)) return;
  SpinGuard g;
  while (!mbar_try_wait_cluster(a, parity)) g.check_internal();
}

// 32 lanes x 32b, 32 consecutive columns <- 32 registers per thread.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 32 lanes x 32b, 16 consecutive columns <-> 16 registers per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// ------------------------------------------------------------------ A2 bridge all-gather parts
// The bridge all-gather of the feature rows ("concatenation in batch
// dimension") as `parts` equal pieces: piece j copies vectors [j*per, (j+1)*per) of this rank's
// rows X_r (and its labels) to row offset R_r of every rank's gathered buffer, then raises
// flag[GATHER][rank] by one on every rank.  A consumer waits for flag >= epoch * parts for
// every source rank.  `parts` depends only on (B_max, D), so it is the same on every rank.
// The pieces run either in the stand-alone bridge_gather_kernel (one block each) or in the
// prologue of the kernel that consumes the gathered rows (the logits GEMM / F1), by its
// otherwise idle epilogue warps -- the all-gather fused into the GEMM that reads it.
struct GatherArgs {
  const uint4* x_local;  // [B_r x D] rows of this rank (16-byte vectors)
  const int32_t* y_local;
  int64_t x_vecs;        // B_r * D * es / 16
  int B;                 // B_r
  int row_off;           // R_r
  int64_t row_vecs;      // D * es / 16
  int rank, world, parts;
  PeerPtrs dst_x, dst_y;  // gathered X / y slab base on each rank
  PeerFlags flags;        // &flag[GATHER][rank] on each rank
  uint4* mc_x;            // NVLS multicast views (or NULL): one multimem op reaches every rank
  int32_t* mc_y;
  uint32_t* mc_flag;
};

// Piece `part` by `nthr` threads (thread index `t`); the caller then runs
// gather_signal() from ONE of those threads after a barrier over all `nthr` of them.
__device__ __forceinline__ void gather_copy(const GatherArgs& g, int part, int t, int nthr) {
  const int64_t per = (g.x_vecs + g.parts - 1) / g.parts;
  const int64_t v0 = static_cast<int64_t>(part) * per, v1 = v0 + per < g.x_vecs ? v0 + per : g.x_vecs;
  const int64_t off_vec = static_cast<int64_t>(g.row_off) * g.row_vecs;
  const int yper = (g.B + g.parts - 1) / g.parts;
  const int y0 = part * yper, y1 = y0 + yper < g.B ? y0 + yper : g.B;
  if (g.mc_x != nullptr) {
    for (int64_t v = v0 + t; v < v1; v += nthr) multimem_st_v4(g.mc_x + off_vec + v, __ldg(g.x_local + v));
    for (int i = y0 + t; i < y1; i += nthr) multimem_st_u32(g.mc_y + g.row_off + i, static_cast<uint32_t>(g.y_local[i]));
    return;
  }
  for (int64_t v = v0 + t; v < v1; v += nthr) {
    const uint4 val = __ldg(g.x_local + v);
#pragma unroll
    for (int p = 0; p < kMaxRanks; ++p)
      if (p < g.world) reinterpret_cast<uint4*>(g.dst_x.p[p])[off_vec + v] = val;
  }
  for (int i = y0 + t; i < y1; i += nthr) {
    const int32_t y = g.y_local[i];
#pragma unroll
    for (int p = 0; p < kMaxRanks; ++p)
      if (p < g.world) reinterpret_cast<int32_t*>(g.dst_y.p[p])[g.row_off + i] = y;
  }
}
// After a barrier over the copying threads: one fence.sc.sys orders all of their stores
// (cumulativity through the barrier) before the relaxed flag increments.
__device__ __forceinline__ void gather_signal(const GatherArgs& g, int npieces) {
  __threadfence_system();
  if (g.mc_x != nullptr) {
    multimem_red_add_relaxed_u32(g.mc_flag, static_cast<uint32_t>(npieces));  // on every rank at once
  } else {
    for (int p = 0; p < g.world; ++p) red_add_relaxed_sys(g.flags.p[p], static_cast<uint32_t>(npieces));
  }
}

}  // namespace whale
