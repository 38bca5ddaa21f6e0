/*
 * whale_splitfc.h -- C-ABI of the B200-native split-FC softmax cross-entropy library
 * (the hot path of Whale's hybrid strategy, arXiv 2011.09208).
 *
 * The method (Example 2 "Hybrid of replicate and split"):
 *     with wh.replicate(total_gpu): features = ResNet50(inputs)      # DP backbone
 *     with wh.split(total_gpu):     logits = FC(features)            # MP classifier
 *                                   predictions = Softmax(logits)
 * The FC weight W [C x D] (class-major) is split along the class dimension (sharding
 * pattern SP1, "shards the second input tensor in the second tensor
 * dimension"); rank r owns classes [o_r, o_r + C_r).  The bridge layer "gathers the
 * outputs from different batches for concatenation in batch dimension":
 * every rank sees X = concat_r X_r (rank order).  The loss is softmax cross-entropy,
 * mean over the global batch B_tot = world * B (reading R1).
 *
 * Conventions:
 *   - All functions are extern "C"; no C++ or CUDA types cross the boundary.  Streams
 *     are passed as `void*` (a cudaStream_t; NULL = legacy default stream).
 *   - Device pointers are raw CUDA device addresses; host pointers are ordinary memory.
 *   - The caller owns every buffer (inputs, outputs, workspaces).  The library never
 *     allocates device memory; it owns only host state inside a context.
 *   - Status codes are returned synchronously for argument/shape errors.  Errors found
 *     on the device (a label outside [0, C), a peer timeout) set a word in the
 *     workspace that whale_splitfc_check() reads.  The library never aborts.
 *   - whale_last_error() returns a thread-local message for the last non-OK status.
 *   - Multi-GPU: all ranks must issue the same sequence of forward/backward calls
 *     (collective semantics, like NCCL).
 */
#ifndef WHALE_SPLITFC_H_
#define WHALE_SPLITFC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  WHALE_OK = 0,
  WHALE_ERR_INVALID_ARG = 1, /* NULL pointer, non-positive size, rank out of range, ... */
  WHALE_ERR_UNSPLITTABLE = 2, /* C < world, or a shard would receive 0 classes */
  WHALE_ERR_UNSUPPORTED = 3,  /* D % 8 != 0, world > 8, dtype combination, no sm_100 device */
  WHALE_ERR_STATE = 4,        /* backward before forward, workspace too small */
  WHALE_ERR_LABEL = 5,        /* a label outside [0, C) (device-detected, via whale_splitfc_check) */
  WHALE_ERR_CUDA = 6,         /* a CUDA runtime/driver call failed */
  WHALE_ERR_COMM = 7          /* a peer flag wait timed out (device-detected) */
} whale_status_t;

typedef enum { WHALE_BF16 = 0, WHALE_F32 = 1 } whale_dtype_t;

/*
 * whale_splitfc_plan -- class-shard sizes (pure host function; no CUDA; thread-safe).
 *
 * PAPER.md:920 (§3.3.1): for a split TaskGraph Whale "balances the FLOP of a partitioned
 * operation through uneven sharding in splitting dimension"; the load ratio is
 * "initialized in proportional to the device's computing capacity",
 * the minimiser of Formula 1 when memory does not bind.
 *
 *   num_classes    C >= 1
 *   world_size     N in [1, 8]
 *   capacity       [N] integer capacity weights (> 0), or NULL for an even split
 *   shard_counts   out [N]: C_r; sum = C; every C_r >= 1
 *   shard_offsets  out [N]: o_r = C_0 + ... + C_{r-1}
 *
 * Rounding: Hamilton / largest remainder in exact integers, leftover classes
 * to the largest remainders, ties to the lower rank (R4/R5).  Deterministic:
 * every rank computes the identical plan.
 * Errors: WHALE_ERR_INVALID_ARG (N out of range, NULL outputs, a weight of 0),
 *         WHALE_ERR_UNSPLITTABLE (C < N, or some C_r would be 0).
 */
whale_status_t whale_splitfc_plan(int64_t num_classes, int32_t world_size, const uint32_t* capacity,
                                  int64_t* shard_counts, int64_t* shard_offsets);

/*
 * whale_splitfc_plan_mem -- class-shard sizes under per-device memory caps (pure host
 * function; deterministic; thread-safe).
 *
 * Algorithm 1, "Memory-Constraint Load Balancing", subject to the
 * constraint of Formula 1, L_i * TG_mem <= DM_i: start from the
 * proportional plan above; while some device is over its memory and some device has room,
 * shift classes from the device with the highest memory utilisation (peak) to the free
 * device with the lowest (FLOP utilisation, memory utilisation) (valley); each shift moves
 * min(peak overload, valley headroom) whole classes.
 *
 *   mem_bytes        [N] memory available to the FC shard on each device, or NULL (no cap:
 *                    identical to whale_splitfc_plan)
 *   bytes_per_class  device bytes one class costs (e.g. 6*D for a bf16 W row + fp32 dW row)
 *   fixed_bytes      bytes every device needs regardless of its shard (workspaces)
 *   capacity, outputs as whale_splitfc_plan.
 * Ties go to the lower rank; exact integer/rational arithmetic (R13).
 * Errors: as whale_splitfc_plan; WHALE_ERR_INVALID_ARG if bytes_per_class == 0;
 *         WHALE_ERR_UNSPLITTABLE if a device stays over its cap (infeasible) or ends with 0
 *         classes.
 */
whale_status_t whale_splitfc_plan_mem(int64_t num_classes, int32_t world_size, const uint32_t* capacity,
                                      const uint64_t* mem_bytes, uint64_t bytes_per_class, uint64_t fixed_bytes,
                                      int64_t* shard_counts, int64_t* shard_offsets);

/*
 * Context descriptor.  Layouts (all row-major, leading dimension = row length):
 *   X_r   [B x D]    x_dtype      this rank's DP rows (the backbone's output)
 *   y_r   [B]        int32        global class ids in [0, C)
 *   W_r   [C_r x D]  x_dtype      rows [o_r, o_r + C_r) of the class-major weight W
 *   dX_r  [B x D]    x_dtype      d loss / d X_r (includes the 1/B_tot of the mean)
 *   dW_r  [C_r x D]  dw_dtype     d loss / d W_r: WHALE_F32, or WHALE_BF16 (with bf16 operands;
 *                                 fp32 accumulation, one RN-even rounding at the store)
 * x_dtype = WHALE_BF16 runs bf16 x bf16 -> fp32 on tcgen05 kind::f16; WHALE_F32 runs
 * fp32 storage on tcgen05 kind::tf32 (R11).
 *
 * Multi-GPU (world > 1): `peer_symm_ptrs[p]` is rank p's symmetric buffer as mapped in
 * THIS process (e.g. torch symmetric-memory buffer_ptrs), each of `symm_bytes` >= the
 * size returned by whale_splitfc_workspace_size; the caller must zero every rank's buffer
 * and barrier before the first forward.  world == 1 ignores both.
 */
typedef struct whale_splitfc_desc {
  int32_t rank;
  int32_t world_size;
  int64_t local_batch; /* B = B_rank, this rank's DP rows (must equal batch_counts[rank] if given) */
  int64_t feature_dim; /* D, multiple of 8 */
  int64_t num_classes; /* C */
  const int64_t* shard_counts;  /* [world] from whale_splitfc_plan (host memory) */
  const int64_t* shard_offsets; /* [world] */
  whale_dtype_t x_dtype;
  whale_dtype_t dw_dtype;
  void* const* peer_symm_ptrs; /* [world] device addresses (host array), NULL if world == 1 */
  size_t symm_bytes;
  void* local_workspace; /* device, 256-byte aligned */
  size_t local_workspace_bytes;
  /* NEXT-3 (hardware-aware replicate): per-rank DP batch
   * [world] (host memory, identical on every rank), or NULL = local_batch on every rank.
   * Rank r's rows are rows [B_0 + ... + B_{r-1}, ... + B_r) of the gathered batch (rank
   * order); B_r may be 0 when world > 1 (that rank then only serves its class shard);
   * sum B_r >= 1.  whale_splitfc_plan(B_tot, world, capacity) gives the proportional split. */
  const int64_t* batch_counts;
  /* NVLS (NVLink SHARP) multicast address of the symmetric buffer (world > 1), or NULL: one
   * multimem store then reaches the same offset in every rank's buffer through the NVSwitch.
   * Used for the bridge all-gather (A2) of X_r, y_r and its flags (the B200
   * form of the all-gather the paper's bridge inserts); NULL keeps the
   * unicast peer stores.  With WHALE_NVLS_RS=1 the dX reduce-scatter (A8) goes through the
   * switch as well: every rank stores its rows for owner q in slot q of its OWN receive slab
   * and the owner reads all ranks' slot at once with multimem.ld_reduce (parity-green and
   * run-to-run reproducible at N = 2; off by default: measured slower than the unicast
   * pushes + rank-ordered sum, which stays the default). */
  void* multicast_ptr;
} whale_splitfc_desc;

typedef struct whale_splitfc_ctx whale_splitfc_ctx;

/* Bytes of symmetric (peer-mapped) and local device workspace the descriptor needs.
 * Pointers in the descriptor may be NULL for this query. */
whale_status_t whale_splitfc_workspace_size(const whale_splitfc_desc* desc, size_t* symm_bytes,
                                            size_t* local_bytes);

/* Validate the descriptor, pick tile configurations, encode TMA descriptors for the
 * workspace.  Host-side only apart from reading device attributes. */
whale_status_t whale_splitfc_create(const whale_splitfc_desc* desc, whale_splitfc_ctx** out);

/*
 * Forward (collective; stream-ordered; no host synchronisation):
 *   A2 bridge all-gather of X_r, y_r -> X [B_tot x D], y [B_tot]
 *   A3 logits GEMM Z_r = X W_r^T with the row max / sum-exp fused in its epilogue
 *   A4 cross-shard combine m = max_r m_r, s = sum_r s_r e^{m_r - m} over NVLink
 *   A5 loss = (1/B_tot) sum_i (m_i + ln s_i - z_{i,y_i})
 *   x_local  [B x D] device; labels_local [B] int32 device; w_shard [C_r x D] device
 *   loss     device float scalar (identical bits on every rank)
 *   row_loss device [B] per-row loss of this rank's rows, or NULL
 * With bf16 operands, B_tot <= 32 and D % 256 == 0, D <= 2048 the forward also accumulates
 * the dX partials U = sum_t P~_t W_t (one pass over W_r) and the backward only
 * finishes them -- same results, W_r read once per step.
 * Saves y, P~ and the statistics in the workspace for the following backward; X is saved
 * there too when world_size > 1 (the gathered batch).  At world_size 1 X is NOT copied: the
 * backward reads x_local itself, so it must stay valid and unmodified until the matching
 * backward has run (stream order).
 */
whale_status_t whale_splitfc_forward(whale_splitfc_ctx* ctx, const void* x_local, const int32_t* labels_local,
                                     const void* w_shard, float* loss, float* row_loss, void* stream);

/*
 * Backward of the last forward (collective):
 *   A6 G_r = (softmax - onehot) / B_tot on this shard's classes (one-hot only where the
 *      label is owned by this shard)
 *   A7 dW_r = G_r^T X   (no communication: the FC shard is updated locally)
 *   A8 dX = sum_r G_r W_r, reduce-scattered to the DP owners (bridge backward)
 *   dx_local [B x D] device (overwritten); dw_shard [C_r x D] device (overwritten)
 * WHALE_ERR_STATE if no forward preceded it.
 */
whale_status_t whale_splitfc_backward(whale_splitfc_ctx* ctx, const void* w_shard, void* dx_local,
                                      void* dw_shard, void* stream);

/*
 * NEXT-4 extensions: the FC bias and the predictions of Example 2
 * (`logits = FC(features)`, `predictions = Softmax(logits)`).
 *   bias_shard  [C_r] device, x_dtype, or NULL: logits = X W_r^T + b_r (a Dense layer with
 *               bias; the 782 MB FC size of PAPER.md:71 suggests one, R2)
 *   pred_local  [B] int32 device or NULL: top-1 class of each of this rank's rows (argmax of
 *               the softmax over ALL classes; ties -> lowest class id)
 *   prob_local  [B] float device or NULL (requires pred_local): its softmax probability
 * whale_splitfc_forward(...) == whale_splitfc_forward_ex(..., NULL bias, ..., NULL, NULL).
 */
whale_status_t whale_splitfc_forward_ex(whale_splitfc_ctx* ctx, const void* x_local, const int32_t* labels_local,
                                        const void* w_shard, const void* bias_shard, float* loss, float* row_loss,
                                        int32_t* pred_local, float* prob_local, void* stream);
/*   db_shard    [C_r] fp32 device or NULL: d loss / d b_r = sum over the global batch of G_r
 * whale_splitfc_backward(...) == whale_splitfc_backward_ex(..., NULL). */
whale_status_t whale_splitfc_backward_ex(whale_splitfc_ctx* ctx, const void* w_shard, void* dx_local,
                                         void* dw_shard, float* db_shard, void* stream);

/*
 * whale_splitfc_backward_scaled -- the backward with the upstream gradient folded in (the
 * autograd path: d(total)/d(loss) arrives as a device scalar, "utilized to
 * compute gradients for model parameters"):
 *   grad_scale  device float scalar g, or NULL (= 1): dX_r, dW_r and db_r are multiplied by g
 *               inside the kernels that store them (no extra pass)
 * The other arguments are those of whale_splitfc_backward_ex; with dw_dtype == WHALE_BF16 in the
 * descriptor dW_r is written in bf16 (rounded once from the fp32 accumulator, after g).
 * whale_splitfc_backward_ex(...) == whale_splitfc_backward_scaled(..., NULL, stream).
 */
whale_status_t whale_splitfc_backward_scaled(whale_splitfc_ctx* ctx, const void* w_shard, void* dx_local,
                                             void* dw_shard, float* db_shard, const float* grad_scale, void* stream);

/* Synchronise `stream` and surface device-detected errors (WHALE_ERR_LABEL, WHALE_ERR_COMM);
 * clears the error word. */
whale_status_t whale_splitfc_check(whale_splitfc_ctx* ctx, void* stream);

whale_status_t whale_splitfc_destroy(whale_splitfc_ctx* ctx);

/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char* whale_last_error(void);

/*
 * Introspection / profiling (used by bench.py and the tests):
 *   whale_splitfc_launches_per_step: kernels launched by one forward + backward.
 *   whale_splitfc_profile_enable: when on, every library kernel launch is bracketed by
 *     CUDA events on the launching stream.
 *   whale_splitfc_profile_read: synchronises, then returns per-kernel-kind totals:
 *     names (';'-separated into `names` of `names_len` bytes), total ms and launch count
 *     per kind (arrays of `max_kinds`), and the number of kinds in *n_kinds; resets.
 *   whale_splitfc_config: the chosen tile configuration as a JSON string in `buf`.
 */
int32_t whale_splitfc_launches_per_step(const whale_splitfc_ctx* ctx);
whale_status_t whale_splitfc_profile_enable(whale_splitfc_ctx* ctx, int32_t enable);
whale_status_t whale_splitfc_profile_read(whale_splitfc_ctx* ctx, char* names, size_t names_len, double* total_ms,
                                          int64_t* launches, int32_t max_kinds, int32_t* n_kinds);
whale_status_t whale_splitfc_config(const whale_splitfc_ctx* ctx, char* buf, size_t buf_len);

#ifdef __cplusplus
}
#endif

#endif /* WHALE_SPLITFC_H_ */
