/*
 * bgmf.h -- C ABI of libbgmf.so, the B200 (sm_100a) implementation of the
 * blocked-SGD matrix-factorization hot path of the reference `blockmf`
 * package (arXiv 2304.13724).  Paths below are relative to
 * /root/reference/pkg/src/blockmf/.
 *
 * Conventions
 *   - plain pointers and sizes only; every host buffer is caller-owned and is
 *     only read/written during the call; device buffers are owned by the
 *     context (bgmf_ctx) or, for bgmf_bind_factors, by the caller;
 *   - return 0 (BGMF_OK) on success, a negative BGMF_ERR_* code otherwise, with
 *     a message from bgmf_last_error(ctx) (ctx may be NULL for the stateless
 *     entry points: the message is then thread-local);
 *   - numeric divergence is NOT an error code: like the reference
 *     (_kernels.py:5-7,49-50) it is reported through out-parameters
 *     (bad_entry / bad_iter >= 0, sse_after = NaN);
 *   - one host thread per context at a time; distinct contexts (and the
 *     stateless calls, which use a thread-local scratch context) may be used
 *     concurrently from different threads.  The GIL is released by ctypes.
 */
#ifndef BGMF_H
#define BGMF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BGMF_OK 0
#define BGMF_ERR_CUDA (-1)   /* CUDA runtime error (message has details) */
#define BGMF_ERR_ARG (-2)    /* invalid argument (shape, range, NULL)    */
#define BGMF_ERR_STATE (-3)  /* call order: e.g. run_step before partition */
#define BGMF_ERR_DATA (-4)   /* dataset violates its contract (index range) */
#define BGMF_ERR_NOMEM (-5)  /* device allocation failed                  */

typedef struct bgmf_ctx bgmf_ctx;

/* ABI version (major*100 + minor). */
int bgmf_version(void);

/* Create a context on CUDA device `device`.  `stream` is a cudaStream_t to
 * launch on (NULL: the context creates its own non-blocking stream). */
int bgmf_create(int device, void* stream, bgmf_ctx** out);
void bgmf_destroy(bgmf_ctx* ctx);
const char* bgmf_last_error(const bgmf_ctx* ctx);

/* Tunables (B200 knobs; none changes the reference's semantics):
 *   "exact"      0/1   1 = fp64 sequential-per-block kernels, bit-identical to
 *                      the reference (_kernels.py fastmath=False order);
 *                      0 = fp32 warp-per-rating lossless kernels (default).
 *   "min_chunk"  int   minimum ratings per worker group in fast mode
 *                      (bounds per-block concurrency on small blocks; 256).
 *   "sparse_min_chunk" int  floor of the per-group chunk on sparse blocks
 *                      (density <= 1/8), where concurrency per block is
 *                      instead capped at "col_ratio" (0.6) x block columns
 *                      (default 32; 0 = always min_chunk).
 *   "col_ratio"  float see sparse_min_chunk.
 *   "l2_wave_bytes" int  fast mode: a stratum whose V blocks exceed this many
 *                      bytes runs as sequential waves of blocks that fit (so
 *                      the V traffic stays in L2; default 48 MiB, 0 = off).
 *   "stagger"    0/1/2 chunk-length rule in fast mode: 2 (default) rounds the
 *                      chunk up to 8*q with q odd so concurrent groups start
 *                      at staggered columns on dense rows (no lockstep V
 *                      collisions); 1 = next prime; 0 = as computed.
 *   "timing"     0/1   record CUDA events around every kernel launch.
 *   "warps_per_sm" int resident-warp target used to size chunks (0 = occupancy).
 *   "bulk_red"   0/1   1 = each rating's V-row delta leaves through the TMA
 *                      engine (cp.reduce.async.bulk add.f32 from a shared-
 *                      memory ring); 0 = per-lane red.global.add.v4 (default,
 *                      measured faster: both bound by the SM->L2 interface).
 *   "sse_wide"   0/1   1 = post-sweep SSE with several ratings' rows in flight
 *                      per group (measured slower on C4).
 *   "sse_async"  0/1   1 (default) = post-sweep SSE streams the V rows of the
 *                      next 4 ratings of each group through a per-lane
 *                      cp.async shared-memory ring; 0 = the sweep's
 *                      register-pipelined walk (one row in flight).
 *   "fused"      -1/0/1  1 = one cooperative launch per outer step (all
 *                      strata, sweeps and SSE passes separated by grid
 *                      barriers); 0 = one launch per stratum sweep / SSE pass;
 *                      -1 = auto (default): fused when a stratum holds at most
 *                      "fused_max_batch" ratings (default 0: measured on B200,
 *                      the per-stratum launches win at every config size).
 *   "ordered"    -1/0/1  -1 (default) = route batches whose chunked order would
 *                      distort the reference (dense blocks, chunks shorter
 *                      than a row, >1 group per V row) to the ordered stratum
 *                      kernel (every update in stored order, deterministic);
 *                      1 = always when it fits; 0 = never.
 *   "ord_row_split", "ord_col_conc"  float  the routing thresholds above
 *                      (1.0 / 1.0; ring ranks use ord_col_conc 6).
 *   "ord_stage_ratings" int, "ord_fill_ctas" int, "ord_warp" 0/1  ordered
 *                      kernel stage size (1024), CTAs per SM, one group per warp.
 *   "pdl"        0/1   programmatic dependent launch between sweep and SSE (1).
 *   "conv_graph" 0/1   ConvergeEachBlock steps as a CUDA graph with device-side
 *                      while-nodes (1) instead of host-driven sweeps.
 *   "no_val8"    0/1   streamed ratings never use 1-byte value codes.
 *   "spread"     0/1   partial sweep waves dealt evenly over a full wave of
 *                      CTAs (1).
 *   "u_prefetch" -1/0/1  L2 prefetch of upcoming runs' U rows: -1 (default)
 *                      when the mean run is < 1.5 ratings, 1 on, 0 off.
 *   "nt_download" 0/1  the model's fp32 -> fp64 widening into the caller's
 *                      arrays uses non-temporal stores (1).
 *   "u_ring"     -1/0/1  U rows of upcoming runs through a cp.async ring: -1
 *                      (default) when the partition's ratings-per-user CV > 1
 *                      (skewed users), 1 on, 0 off.
 *   Measured slower and kept off: "fuse_sse",
 *   "dyn_split" (int D), "snap" (int cap). */
int bgmf_set_option(bgmf_ctx* ctx, const char* key, double value);

/* Bucket the ratings into the I x J block grid on the GPU.
 * Replaces BlockedDataset.__init__ (partition.py:112-136) and make_grid /
 * split_bounds (partition.py:18-71): balanced slabs, entries sorted by
 * (block, row, col) with ties in input order -- bit-exact with np.lexsort.
 * rows/cols are global int64 indices, vals fp64 (RatingsDataset layout,
 * core.py:53-108).  Returns BGMF_ERR_DATA when an index is outside n x m. */
int bgmf_partition(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols,
                   const double* vals, int64_t nnz, int64_t n, int64_t m,
                   int grid_i, int grid_j);

/* bgmf_partition of the entries whose row lies in [row_lo, row_hi) only (the
 * rest are range-checked and dropped while the host threads narrow the
 * upload): a multi-GPU rank's U-row shard, without a host-side gather.  The
 * grid is still the full n x m one; exported `order` indices refer to the
 * kept entries in input order. */
int bgmf_partition_rows(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols,
                        const double* vals, int64_t nnz, int64_t n, int64_t m,
                        int grid_i, int grid_j, int64_t row_lo, int64_t row_hi);

/* Benchmark / test inputs (not part of the reference path): generate the
 * synthetic low-rank workload of paper_2304_13724_b200/workloads.py
 * (Feistel-sampled cells -- identical integers to workloads.feistel_cells --
 * and counter-based normals for the values) directly on the device and
 * partition it as bgmf_partition would.  Used for C5 (2e9 ratings), whose
 * host-side generation is impractical. */
int bgmf_synth_partition(bgmf_ctx* ctx, int64_t n, int64_t m, int64_t nnz,
                         uint64_t seed, int grid_i, int grid_j);
/* Same generator, ratings [start, start+nnz) copied to host arrays. */
int bgmf_synth(int64_t n, int64_t m, int64_t nnz, int64_t start, uint64_t seed,
               int64_t* rows, int64_t* cols, double* vals);

/* Copy the partition back (any pointer may be NULL):
 *   offsets[I*J+1]    BlockedDataset._offsets            (partition.py:134-136)
 *   order[nnz]        source index of each sorted entry (values = vals[order],
 *                     BlockedDataset._values, partition.py:131)
 *   lrows/lcols[nnz]  block-local coordinates (BlockedDataset._rows/_cols,
 *                     partition.py:125-130). */
int bgmf_partition_export(bgmf_ctx* ctx, int64_t* offsets, int64_t* order,
                          int32_t* lrows, int32_t* lcols);

/* The device-resident values in partition order, widened to fp64 (fast mode
 * holds fp32, exact mode fp64): what the kernels read for BlockedDataset._values
 * (partition.py:131).  Device-resident partitions only (BGMF_ERR_STATE when
 * the ratings stream from host memory). */
int bgmf_partition_values(bgmf_ctx* ctx, double* vals);

/* Out-of-core partitions keep their pinned host layout; when a context is
 * destroyed those buffers stay registered in a process-wide cache (up to a
 * quarter of physical memory) for the next out-of-core partition, like a
 * caching host allocator.  This unregisters and unmaps all of them. */
int bgmf_release_host_cache(void);

/* Upload U (n x k) and V (m x k), row-major fp64 as FactorModel.u/.v
 * (core.py:139-176).  Fast mode stores fp32 rows padded to a multiple of 4. */
int bgmf_set_factors(bgmf_ctx* ctx, const double* u, const double* v,
                     int64_t n, int64_t m, int k);
/* Download the factors into caller fp64 buffers (n x k, m x k). */
int bgmf_get_factors(bgmf_ctx* ctx, double* u, double* v);

/* Zero-fill a caller-owned host buffer with one write per 4 KiB page (OpenMP
 * threads), faulting its pages in.  Thread-safe and context-free: the
 * trainer runs it on a side thread over the not-yet-written fp64 factor
 * arrays while the epochs run, so bgmf_get_factors's widening does not pay
 * first-touch page faults. */
int bgmf_host_prefault(void* p, int64_t bytes);

/* init_factors on the device (core.py:179-193), bit-identical to numpy:
 * draws of the PCG64 stream whose seeded 128-bit (state, inc) -- numpy's
 * default_rng(seed).bit_generator.state -- are passed as hi/lo halves;
 * u = draws[0 : n*k] / sqrt(k), v = the next m*k draws / sqrt(k). */
int bgmf_init_factors(bgmf_ctx* ctx, uint64_t state_hi, uint64_t state_lo,
                      uint64_t inc_hi, uint64_t inc_lo, int64_t n, int64_t m,
                      int k);

/* Use caller-owned device factor buffers (fp32, row stride kp >= k, kp % 4 ==
 * 0, zero padding) instead of context-owned ones -- e.g. torch tensors that
 * NCCL moves between GPUs.  Fast mode only. */
int bgmf_bind_factors(bgmf_ctx* ctx, void* u_dev, void* v_dev, int64_t n,
                      int64_t m, int k, int kp);

/* One outer step (trainer.py:125-158): for each batch (plan_step order,
 * scheduler.py:45-75) run `inner_iters` SGD sweeps over every block of the
 * batch concurrently, then each block's post-sweep SSE (_kernels.py:56).
 *   plan[batch_off[t] .. batch_off[t+1]) = flat block ids bi*J+bj of batch t
 *   sse_out[I*J]  per-block post-sweep SSE (blocks not in the plan: 0)
 *   bad_out[3]    {plan position, entry, inner iteration} of the first
 *                 diverged block in plan order, or {-1,-1,-1}.
 * Equivalent to `_kernels.sgd_sweeps` on every block of the plan followed by
 * the trainer's merge.  Synchronous: returns after sse_out is on the host. */
int bgmf_run_step(bgmf_ctx* ctx, const int32_t* plan, const int32_t* batch_off,
                  int nbatch, int inner_iters, double alpha, double beta,
                  double* sse_out, int64_t* bad_out);

/* Converge mode (ConvergeEachBlock, kernel.py:108-126, _kernels.py:62-100):
 * every block of every batch sweeps until its RMSE improvement < tol or
 * `cap` sweeps.  iters_out[I*J] sweeps used, capped_out[I*J] 0/1. */
int bgmf_run_step_converge(bgmf_ctx* ctx, const int32_t* plan,
                           const int32_t* batch_off, int nbatch, double tol,
                           int64_t cap, double alpha, double beta,
                           double* sse_out, int64_t* iters_out,
                           int32_t* capped_out, int64_t* bad_out);

/* SSE of the current factors over all partitioned training entries
 * (metrics.py:39-52 numerator, for AdaptiveDecreasing's RMSE_0). */
int bgmf_train_sse(bgmf_ctx* ctx, double* sse_out);

/* Held-out set for per-step test RMSE (HoldoutEvaluator, metrics.py:55-81):
 * global int64 rows/cols, fp64 values, cold[count] (1 = predict `fallback`). */
int bgmf_holdout_set(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols,
                     const double* vals, const uint8_t* cold, int64_t count,
                     double fallback);
int bgmf_holdout_sse(bgmf_ctx* ctx, double* sse_out);

/* Out-of-core mode (C5; PAPER.md:190,196,294 -- data larger than HBM): move the
 * partitioned ratings to pinned host memory and keep only `nslots` device
 * slots of `slot_ratings` ratings each (12 B per rating).  Every later
 * bgmf_run_step streams each stratum's blocks through the slot ring on a side
 * stream while the previous piece computes; factors stay resident.  A slot
 * must hold the largest block.  Fast mode, fixed schedules. */
int bgmf_stream_ratings(bgmf_ctx* ctx, int64_t slot_ratings, int nslots);
/* Out-of-core partition (replaces bgmf_partition + bgmf_stream_ratings when
 * the partition itself must not exceed device_budget bytes of HBM): row
 * blocks in chunks, each partitioned on the device exactly as
 * bgmf_partition does, straight into the pinned streaming layout; then
 * nslots device slots of slot_ratings ratings.  Same ordering, offsets and
 * errors as bgmf_partition (reference partition.py:112-136).  Only rows in
 * [row_lo, row_hi) are kept (row_hi < 0: n) -- a ring rank's shard, as
 * bgmf_partition_rows; every entry is still range-checked. */
int bgmf_partition_ooc(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols,
                       const double* vals, int64_t nnz, int64_t n, int64_t m, int grid_i,
                       int grid_j, int64_t device_budget, int64_t slot_ratings, int nslots,
                       int64_t row_lo, int64_t row_hi);
/* Device memory of the stream-ordered pool every context allocates from:
 * out2 = {bytes in use now, high-water mark}; reset = 1 restarts the mark. */
int bgmf_mem_stats(bgmf_ctx* ctx, int64_t* out2, int reset);
/* Rating bytes streamed host->device since the context was created. */
int bgmf_stream_stats(bgmf_ctx* ctx, double* h2d_bytes);

/* nsteps outer steps in one call (fast mode, no host decision between them:
 * train_blocked with early stopping off and a fixed inner schedule).  Step s
 * runs plan block ids plans[...] cut by batch_offs[...] (both concatenated
 * over the steps; step s has nbatch[s] batches, nbatch[s] + 1 offsets) with
 * inner_iters[s] sweeps; sse_out[s * I*J + b] = block b's post-sweep SSE of
 * step s.  All steps are enqueued back to back with one synchronisation at
 * the end.  bad_out = {step, block id, entry, iteration} of the first
 * diverged step, or -1s (later steps' results are then meaningless, as after
 * the reference's DivergenceError).  step_ms (optional): device time of each
 * step. */
int bgmf_run_steps(bgmf_ctx* ctx, int nsteps, const int32_t* plans,
                   const int32_t* batch_offs, const int32_t* nbatch,
                   const int32_t* inner_iters, double alpha, double beta,
                   double* sse_out, int64_t* bad_out, float* step_ms);

/* Asynchronous outer step (fast mode), for callers that interleave their own
 * work between strata -- the multi-GPU ring trainer moves V blocks with NCCL
 * on the same stream between batches (trainer.py:138-152 barrier analog).
 * step_begin reserves work-table slots for up to max_blocks block launches
 * and zeroes the per-block SSEs; each step_batch enqueues its strata (same
 * arguments as bgmf_run_step) without a host sync; step_end synchronises and
 * returns sse_out[I*J] (blocks not run: 0) and bad_out = {block id, entry,
 * iteration} of the first diverged block in submission order, or -1s. */
int bgmf_step_begin(bgmf_ctx* ctx, int max_blocks);
int bgmf_step_batch(bgmf_ctx* ctx, const int32_t* plan, const int32_t* batch_off,
                    int nbatch, int inner_iters, double alpha, double beta);
int bgmf_step_end(bgmf_ctx* ctx, double* sse_out, int64_t* bad_out);
/* bgmf_step_end without a host round trip (the ring trainer's batched
 * epochs): the step's per-block SSEs (fp64 [I*J]) and its raw divergence
 * word go to caller DEVICE memory, stream-ordered; nothing waits.  The word
 * is all ones when clean, else (plan position in submission order << 48) |
 * (iteration << 32) | entry. */
int bgmf_step_end_async(bgmf_ctx* ctx, double* d_sse_out, uint64_t* d_bad_out);

/* One outer step of the synchronized row-sharded baseline trainer (CPMF,
 * baselines.py:100-182, `train_sync_parallel`) on a context partitioned 1 x 1
 * with factors set: shard w = entries [shard_edges[w], shard_edges[w+1]) of
 * the row-major partition (whole rows, edges from split_bounds), updating U
 * in place and a private copy of V; the copies' deltas are then summed onto V
 * in shard order (one shard works on V directly).  sse_out[w] = the shard's
 * post-sweep SSE; bad_out = {shard, entry within the shard, iteration} of the
 * first diverged shard in shard order, or -1s.  Exact mode is bit-identical
 * with the reference; fast mode chunks each shard over worker groups (fp32). */
int bgmf_run_sync_parallel_step(bgmf_ctx* ctx, const int64_t* shard_edges,
                                int nshards, double alpha, double beta,
                                double* sse_out, int64_t* bad_out);

/* Accumulated kernel time since the last reset (requires "timing"=1):
 * out[0] sgd ms, out[1] sse ms, out[2] sgd launches, out[3] sse launches,
 * out[4] algorithmic bytes of the timed sgd launches (ratings*(12+16k)). */
int bgmf_kernel_stats(bgmf_ctx* ctx, double* out5, int reset);

/* ---- stateless drop-ins for the reference's native loops ---------------
 * Same arguments and results as the numba functions they replace; all
 * arrays are host memory, u/v are updated in place.  Computed on the GPU
 * in fp64 sequential order (bit-identical with the reference). */

/* _kernels.py:31-59 sgd_sweeps(rows, cols, vals, u, v, alpha, beta, iters) */
int bgmf_sgd_sweeps(const int64_t* rows, const int64_t* cols,
                    const double* vals, int64_t count, double* u,
                    int64_t u_rows, double* v, int64_t v_rows, int k,
                    double alpha, double beta, int iters, double* sse_before,
                    double* sse_after, int64_t* bad_entry, int64_t* bad_iter);

/* _kernels.py:62-100 sgd_converge(rows, cols, vals, u, v, alpha, beta, tol, cap) */
int bgmf_sgd_converge(const int64_t* rows, const int64_t* cols,
                      const double* vals, int64_t count, double* u,
                      int64_t u_rows, double* v, int64_t v_rows, int k,
                      double alpha, double beta, double tol, int64_t cap,
                      double* sse_before, double* sse_after,
                      int64_t* iters_used, int32_t* capped,
                      int64_t* bad_entry, int64_t* bad_iter);

/* _kernels.py:103-140 gradient_steps(rows, cols, vals, u, v, alpha, beta,
 * iters): full-batch block gradient descent (the kernel behind
 * kernel.batch_gradient_block, kernel.py:142-158).  Same arguments and
 * results as bgmf_sgd_sweeps; bit-identical (fp64, reference order). */
int bgmf_gradient_steps(const int64_t* rows, const int64_t* cols,
                        const double* vals, int64_t count, double* u,
                        int64_t u_rows, double* v, int64_t v_rows, int k,
                        double alpha, double beta, int iters,
                        double* sse_before, double* sse_after,
                        int64_t* bad_entry, int64_t* bad_iter);

/* kernel.block_gradients / block_objective (kernel.py:161-179), pure:
 * gu = beta*u + sum_entries (-2e) v[c] (accumulated in entry order, like
 * np.add.at), gv likewise (gu / gv may be NULL); *sse = sum e^2 and
 * *sq_norms = |u|^2 + |v|^2, so objective = sse + beta/2 * sq_norms. */
int bgmf_block_gradients(const int64_t* rows, const int64_t* cols,
                         const double* vals, int64_t count, const double* u,
                         int64_t u_rows, const double* v, int64_t v_rows, int k,
                         double beta, double* gu, double* gv, double* sse,
                         double* sq_norms);

/* _kernels.py:16-28 block_sse(rows, cols, vals, u, v) */
int bgmf_block_sse(const int64_t* rows, const int64_t* cols,
                   const double* vals, int64_t count, const double* u,
                   int64_t u_rows, const double* v, int64_t v_rows, int k,
                   double* sse);

/* FactorModel.predict (core.py:163-165): out[i] = u[rows[i]] . v[cols[i]] */
int bgmf_predict(const double* u, int64_t n, const double* v, int64_t m, int k,
                 const int64_t* rows, const int64_t* cols, int64_t count,
                 double* out);

/* rmse / HoldoutEvaluator numerator (metrics.py:51,78-80): sum of squared
 * errors, cold[i] != 0 predicts `fallback` (cold may be NULL). */
int bgmf_sse(const double* u, int64_t n, const double* v, int64_t m, int k,
             const int64_t* rows, const int64_t* cols, const double* vals,
             const uint8_t* cold, double fallback, int64_t count, double* sse);

/* Peer transport of the multi-GPU ring (no reference counterpart; replaces
 * an NCCL send/recv pair per V-block move, distributed.py).  Ranks map each
 * other's V buffers and flag words once through CUDA IPC (also between
 * processes sharing one GPU); a move is then a copy straight into the
 * receiver's rows plus a release-store of a sequence number into its flag,
 * and the receiver's stream waits (acquire) for that number before its next
 * sweep -- all stream-ordered, no host round trip per batch.
 *   bgmf_peer_alloc  -- zeroed, IPC-exportable device memory owned by ctx
 *                       (freed by bgmf_destroy);
 *   bgmf_peer_handle -- BGMF_PEER_HANDLE_BYTES of IPC handle for such a base;
 *   bgmf_peer_open   -- map a peer's handle (unmapped by bgmf_destroy);
 *   bgmf_peer_push   -- on ctx's stream, one kernel: copy `bytes` src -> dst
 *                       (a peer address; both 16-byte aligned), fence every
 *                       store system-wide, then *peer_flag = value (release,
 *                       system scope);
 *   bgmf_peer_wait   -- on ctx's stream: block later work until *flag >= value
 *                       (wrap-safe comparison). */
#define BGMF_PEER_HANDLE_BYTES 64
int bgmf_peer_alloc(bgmf_ctx* ctx, int64_t bytes, void** out);
int bgmf_peer_handle(bgmf_ctx* ctx, void* base, uint8_t* handle_out);
int bgmf_peer_open(bgmf_ctx* ctx, const uint8_t* handle, void** out);
int bgmf_peer_push(bgmf_ctx* ctx, void* dst, const void* src, int64_t bytes,
                   uint32_t* peer_flag, uint32_t value);
int bgmf_peer_wait(bgmf_ctx* ctx, const uint32_t* flag, uint32_t value);
/* Bounded waits: a wait gives up (and records why) once *abort_word != 0 or
 * after timeout_s; bgmf_peer_abort sets a peer's abort word (a failing rank
 * calls it for every peer); bgmf_peer_error returns 0, 1 (a wait timed out)
 * or 2 (a peer aborted), synchronising ctx's stream. */
int bgmf_peer_config(bgmf_ctx* ctx, const uint32_t* abort_word, double timeout_s);
int bgmf_peer_abort(bgmf_ctx* ctx, uint32_t* peer_abort_word);
int bgmf_peer_error(bgmf_ctx* ctx, int* out);

/* Measurement only (no reference counterpart): the SM<->L2 ceiling of the
 * sweep's access pattern on `device` -- `ratings` random 512-byte rows of an
 * L2-resident rows x 128 fp32 matrix, read (mode 0), read + reduce-added into
 * other random rows (mode 1, the sweep's V traffic) or reduce-added only
 * (mode 2), two reads + one reduce (mode 3), or even warps mode 1 and odd
 * warps mode 0 over as many rows again (mode 4), groups of 8 lanes,
 * 256-thread CTAs x ctas_per_sm per SM.  Best
 * kernel time of 3 timed launches in *ms_out. */
int bgmf_probe_l2(int device, int64_t rows, int64_t ratings, int mode,
                  int ctas_per_sm, double* ms_out);
/* DSMEM variant of the probe (V block of `rows` x 128 fp32 spread over a
 * cluster of cs CTAs): mode 5 remote row read + fp32 atomic row add, 6 the
 * same within the CTA's own slice, 7 remote reads only. */
int bgmf_probe_dsmem(int device, int64_t rows, int64_t ratings, int mode, int cs,
                     int ctas_per_sm, double* ms_out);

#ifdef __cplusplus
}
#endif

#endif /* BGMF_H */
