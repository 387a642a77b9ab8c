// bgmf_internal.cuh -- shared declarations of libbgmf.so (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/bgmf.h"

namespace bgmf {

constexpr unsigned kFull = 0xffffffffu;

// One block of one batch (fast path).  Entries [begin, end) of the
// partition arrays are cut into chunks of chunk_len; chunk c of the batch
// belongs to the work item whose [first_chunk, first_chunk + nchunks)
// contains c.
struct BlockWork {
  int64_t begin, end;           // entry range in the partition arrays
  int64_t row_start, col_start; // factor slice offsets (rows of U / V)
  int32_t chunk_len;            // ratings per worker group
  int32_t first_chunk;          // exclusive prefix of chunk counts in batch
  int32_t block_id;             // bi * J + bj
  int32_t pos;                  // position in the step plan
  // device-side ConvergeEachBlock (run_step_converge_fast): the block's
  // active flag (its chunks do nothing once it is 0) and the current
  // iteration; nullptr everywhere else
  const int32_t* active;
  const int32_t* iter;
};

// Divergence record: smaller = earlier in the reference's order
// (plan position, then inner iteration, then entry).
__host__ __device__ inline unsigned long long pack_bad(int64_t pos, int64_t iter,
                                                       int64_t entry) {
  return ((unsigned long long)pos << 48) | ((unsigned long long)(iter & 0xFFFF) << 32) |
         (unsigned long long)(entry & 0xFFFFFFFFll);
}
constexpr unsigned long long kNoBad = ~0ull;

struct TimedLaunch {
  cudaEvent_t a, b;
  int kind;        // 0 sgd, 1 sse
  double bytes;    // algorithmic bytes (sgd)
};

}  // namespace bgmf

struct bgmf_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int num_sms = 148;

  // options
  bool exact = false;
  int min_chunk = 256;
  int stagger = 2;       // chunk-length rule (stagger_chunk)
  int sparse_min_chunk = 32;  // block_chunk: floor on sparse blocks (0: always min_chunk)
  double col_ratio = 0.6;     // block_chunk: concurrent groups per block column (see there)
  int64_t l2_wave_bytes = 48ll << 20;  // l2_waves: V bytes swept at once (0: whole strata)
  bool timing = false;
  int warps_per_sm = 0;
  bool bulk_red = false;  // V deltas via TMA bulk reduce (measured slower: SM->L2 bound)
  bool sse_wide = false;  // post-sweep SSE with D ratings in flight (measured slower)
  bool sse_async = true;  // post-sweep SSE through a per-lane cp.async ring (sse_async_kernel)
  bool conv_graph = true;  // ConvergeEachBlock loop as a CUDA-graph WHILE node (chunked path)
  void* d_cstate = nullptr;  // its per-block state (ConvState, flags, iteration)
  int cstate_cap = 0;
  std::map<std::string, cudaGraphExec_t> conv_graphs;  // instantiated converge graphs per batch
  bool pdl = true;        // programmatic dependent launch between sweep / SSE kernels
  int u_ring = -1;        // sweep: U rows of upcoming runs via a cp.async smem ring:
                          // 1 on, 0 off, -1 when the users are skewed (row_cv)
  double row_cv = 0.0;    // coefficient of variation of ratings per user (partition)
  bool fuse_sse = false;  // last sweep + SSE in one launch (sweep_sse_kernel; measured slower)
  unsigned* d_fuse = nullptr;  // sweep_sse_kernel's per-work-item counters
  int dyn_split = 1;           // sweep: chunks cut D ways, taken from a ticket counter
  unsigned* d_dyn = nullptr;   // its two self-resetting counters (allocated with the option)
  int u_prefetch = -1;         // sweep/SSE L2 prefetch of upcoming runs' U rows: 1 on, 0 off,
                               // -1 when runs are short (upf_route)
  bool upf_on = false;         // resolved for the current partition
  int64_t upf_key = -1;        // partition the resolution belongs to
  bool spread = true;          // sweep: partial waves dealt evenly over a full wave of CTAs
  bool nt_download = true;     // model download: non-temporal fp64 stores
  int snap_cap = 0;            // sweep: chunk edges moved to the end of a run within this many ratings
  int fused = -1;      // 1: one cooperative launch per step, 0: per stratum, -1 auto
  int groups_key = -1;                // sweep_groups() cache
  int64_t groups_cache = 0;
  int64_t fused_max_batch = 0;  // auto: fuse when a stratum has <= this many ratings

  // grid + partition
  int64_t n = 0, m = 0, nnz = 0;
  int I = 0, J = 0;
  int rbits = 0, cbits = 0;              // bits of a block-local row / col index
  std::vector<int64_t> row_bounds, col_bounds, h_offsets;
  bool partitioned = false;
  int32_t* d_lrow = nullptr;
  int32_t* d_lcol = nullptr;
  float* d_val = nullptr;
  double* d_val64 = nullptr;
  uint32_t* d_order = nullptr;

  // factors
  int k = 0, kp = 0;
  // peer transport (peer.cu): IPC-exportable buffers and mapped peer buffers
  std::vector<void*> peer_owned, peer_opened;
  unsigned int* d_push_done = nullptr;  // CTA-completion counter of peer_push_kernel
  unsigned int* d_peer_err = nullptr;   // peer waits: 1 timed out, 2 aborted by a peer
  const unsigned int* peer_abort = nullptr;  // this rank's abort word (its flag page)
  unsigned long long peer_timeout_ns = 120ull * 1000000000ull;
  bool have_factors = false, bound = false;
  float* d_u = nullptr;
  float* d_v = nullptr;
  double* d_u64 = nullptr;
  double* d_v64 = nullptr;

  // step scratch
  double* d_sse = nullptr;               // [I*J]
  unsigned long long* d_bad = nullptr;   // [1]
  bgmf::BlockWork* d_work = nullptr;
  void* d_priv = nullptr;                // sync-parallel private V copies
  size_t priv_bytes = 0;
  bgmf::BlockWork* h_work = nullptr;     // pinned
  size_t work_cap = 0;
  bool in_step = false;                  // between bgmf_step_begin / _end
  int w_cursor = 0;                      // next free work-table slot of the step
  int w_limit = 0;                       // end of the step's half of the work table
  // steps ended with bgmf_step_end_async alternate between the two halves of
  // the pinned work table; ws_done[h] marks the end of the last step that
  // used half h (its H2D copies read the pinned table when the stream gets
  // there, so the half is rewritten only after that event)
  int ws_half = 0;
  cudaEvent_t ws_done[2] = {nullptr, nullptr};
  bool ws_pending[2] = {false, false};
  std::vector<int32_t> submitted;        // block id of every submitted plan position
  int step_pos0 = 0;                     // submitted.size() when the current step began
  double* h_sse = nullptr;               // pinned [I*J]
  unsigned long long* h_bad = nullptr;   // pinned [1]

  // holdout
  int32_t* d_hrow = nullptr;
  int32_t* d_hcol = nullptr;
  float* d_hval = nullptr;
  double* d_hval64 = nullptr;
  uint8_t* d_hcold = nullptr;
  int64_t hcount = 0;
  double hfallback = 0.0;
  double* d_partials = nullptr;          // eval partial sums
  double* h_scalar = nullptr;            // pinned

  // out-of-core streaming (stream.cu)
  bool streaming = false;
  int nslots = 0;
  int64_t slot_cap = 0;                  // ratings per device slot
  // pinned host copy of the partition, blocks laid out so that every batch
  // of the rotating plan is contiguous (diagonals when I == J); packed
  // 4-byte (lrow << cbits | lcol) records when they fit (8 B per rating)
  bool packed = false;
  bool no_val8 = false;                  // option: keep fp32 values in the streamed records
  bool val8 = false;                     // values are integers 0..255: 1-byte codes in
                                         // h_val and the slots (records 5 B instead of 8)
  int32_t* h_lrow = nullptr;             // or the packed records
  int32_t* h_lcol = nullptr;             // unused when packed
  float* h_val = nullptr;
  uint32_t* h_order = nullptr;
  std::vector<int64_t> h_pos;            // host start of each block
  std::vector<int32_t*> s_lrow, s_lcol;  // device slots
  std::vector<float*> s_val;
  std::vector<cudaEvent_t> ev_copied, ev_consumed;
  cudaStream_t copy_stream = nullptr;
  double h2d_bytes = 0;                  // streamed this context (stats)
  int ooc_chunks = 0;                    // chunks of the last out-of-core partition
  int64_t piece_seq = 0;                 // pieces streamed by asynchronous steps (slot rotation)

  // ordered sweep (ordered.cu): column ranks, row pointers, row flags
  int ord_mode = -1;                     // 1: ordered where possible, 0: never, -1: auto
  int64_t ord_stage_ratings = 1024;      // target ratings per stage (slab CTA)
  int ord_fill_ctas = 1;                 // stages per SM when filling the GPU
  int ord_warp = 1;                      // one group per warp (ordered_shape)
  bool ord_ready = false;
  uint32_t ord_gen = 1;                  // row-flag generation of the next sweep
  int32_t* d_qrank = nullptr;            // [nnz] rank of the entry within its column
  int32_t* d_rowptr = nullptr;           // per block: h + 1 row starts (block-relative)
  std::vector<int64_t> h_rp;             // offset of each block's row pointers
  uint32_t* d_rflag = nullptr;           // [n] tag of the last visit of each U row
  uint32_t* d_obar = nullptr;            // per launched block: two barrier counters
  double* d_opart = nullptr;             // per stage: SSE partial
  int64_t* d_conv = nullptr;             // per block: converge iters_used, capped
  double* d_esq = nullptr;               // exact mode: per-entry squared residuals
  double ord_row_split = 1.0;            // auto: ordered when chunks < this many mean rows
  double ord_col_conc = 1.0;             // auto: ... or > this many groups per V row (<= 0: off)
  std::map<uint64_t, int> ord_cap;       // (kp, smem) -> co-resident CTAs

  // timing
  std::vector<bgmf::TimedLaunch> events;
  size_t events_used = 0;
  double t_sgd_ms = 0, t_sse_ms = 0, t_bytes = 0;
  int64_t n_sgd = 0, n_sse = 0;
};

namespace bgmf {

// The streamed record format as the kernels' `cbits` argument: -1 = SoA
// int32 row / int32 col / fp32 value; else packed (row << cbits | col) records,
// bit 8 set when the values are 1-byte codes (val8).
inline int stream_cbits(const bgmf_ctx* c) {
  return c->packed ? (c->cbits | (c->val8 ? 0x100 : 0)) : -1;
}
inline int64_t val_bytes(const bgmf_ctx* c) { return c->val8 ? 1 : 4; }

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync)
// whose release threshold bgmf_create raises to "never": a second train call
// reuses the first one's pages instead of re-mapping GBs through the driver
// (cudaMalloc/cudaFree of the partition temporaries cost 2-500 ms per call on
// the B200 hosts, profiles/r01_e2e_phases.txt).
template <class T>
inline cudaError_t dmalloc(T** p, size_t bytes, cudaStream_t s) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), bytes, s);
}
inline void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

// Chunk length used by the fast paths.  Groups start their chunks at entry
// c*len of a block; when len is a multiple of a row length (dense rows, all
// with the same column order) every group walks the same columns in lockstep
// and their V updates collide on every rating (drift 0.08 RMSE on a dense
// 64x64 block).  mode 1: the smallest prime >= cl; mode 2: 8*q with q odd
// (>= cl): stagger for every even row length >= 16 while chunk starts stay
// 32-byte aligned for the L-wide triple loads.
inline int64_t stagger_chunk(int64_t cl, int mode) {
  if (mode == 2) {
    int64_t q = (cl + 7) / 8;
    if ((q & 1) == 0) ++q;
    return 8 * q;
  }
  if (mode != 1) return cl;
  if (cl < 3) return cl < 2 ? 2 : cl;
  for (int64_t p = cl | 1;; p += 2) {
    bool prime = true;
    for (int64_t d = 3; d * d <= p; d += 2)
      if (p % d == 0) { prime = false; break; }
    if (prime) return p;
  }
}

// error helpers --------------------------------------------------------
int fail(bgmf_ctx* ctx, int code, const std::string& msg);
int cuda_fail(bgmf_ctx* ctx, cudaError_t e, const char* what);

#define BGMF_CK(ctx, call)                                   \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return bgmf::cuda_fail((ctx), _e, #call); \
  } while (0)

// BGMF_PROFILE=1: stream-synchronised wall-clock marks on stderr (host
// phases of the e2e path); free when the variable is unset.
void prof_mark(bgmf_ctx* ctx, const char* what);

// partition.cu
int partition_device(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols,
                     const double* vals, int64_t nnz, int64_t n, int64_t m, int I, int J,
                     bool dev_in = false, int64_t row_lo = 0, int64_t row_hi = -1);

// hostio.cu -- host <-> device through the process-wide pinned staging pool
int64_t staged_upload(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols,
                      const double* vals, int64_t nnz, int64_t n, int64_t m, int32_t* d_r,
                      int32_t* d_c, void* d_v, bool v64, int* rc, int64_t row_lo,
                      int64_t row_hi, int64_t* kept);
int download_rows(bgmf_ctx* c, const float* d, double* h, int64_t rows, int k, int kp);
// process-wide cache of small pinned host buffers (hostio.cu)
cudaError_t pinned_alloc(void** p, size_t bytes);
void pinned_free(void* p);
// GB-sized pinned arrays: THP-backed + cudaHostRegister; freed off-thread
cudaError_t big_pinned_alloc(void** p, size_t bytes, int threads = 0);
void big_pinned_free(void* p);
void big_pinned_trim();
void* big_host_alloc(size_t bytes);
void big_host_free(void* p);
void big_host_release(void* p, size_t bytes);
int staged_h2d(bgmf_ctx* ctx, void* dst, const void* src, size_t bytes);
int upload_rows(bgmf_ctx* c, const double* h, float* d, int64_t rows, int k, int kp);

// synth.cu (benchmark / test input generator)
int synth_lowrank_device(bgmf_ctx* ctx, int64_t n, int64_t m, int64_t nnz, int64_t start,
                         uint64_t seed, int64_t* rows, int64_t* cols, double* vals);

// sgd.cu
int run_step_fast(bgmf_ctx* ctx, const int32_t* plan, const int32_t* batch_off,
                  int nbatch, int iters, float alpha, float beta);
int run_step_exact(bgmf_ctx* ctx, const int32_t* plan, const int32_t* batch_off,
                   int nbatch, int iters, double alpha, double beta);
int step_begin(bgmf_ctx* c, int max_blocks);
int step_batch(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off, int nbatch, int iters,
               float alpha, float beta);
int step_end(bgmf_ctx* c, double* sse_out, int64_t* bad_out);
int step_end_async(bgmf_ctx* c, double* d_sse_out, unsigned long long* d_bad_out);
// wait until no asynchronous step's work-table copy is pending (sgd.cu)
void drain_async_steps(bgmf_ctx* c);
// drop the cached converge graphs (they capture device pointers)
void conv_graphs_release(bgmf_ctx* c);
// unmap peer buffers, free IPC-exportable ones (peer.cu)
void peer_release(bgmf_ctx* c);
int run_steps(bgmf_ctx* c, int nsteps, const int32_t* plans, const int32_t* offs,
              const int32_t* nbatch, const int32_t* iters, float alpha, float beta,
              double* sse_out, int64_t* bad_out, float* ms_out);
int run_sync_parallel_step(bgmf_ctx* c, const int64_t* edges, int nshards, double alpha,
                           double beta, double* sse_out, int64_t* bad_out);
int run_step_converge_exact(bgmf_ctx* ctx, const int32_t* plan, const int32_t* batch_off,
                            int nbatch, double tol, int64_t cap, double alpha, double beta,
                            int64_t* iters_out, int32_t* capped_out);
int run_step_converge_fast(bgmf_ctx* ctx, const int32_t* plan, const int32_t* batch_off,
                           int nbatch, double tol, int64_t cap, double alpha, double beta,
                           int64_t* iters_out, int32_t* capped_out);
int train_sse_fast(bgmf_ctx* ctx, double* out);
int train_sse_exact(bgmf_ctx* ctx, double* out);
int ensure_step_scratch(bgmf_ctx* ctx, size_t nwork);
int64_t fast_groups(bgmf_ctx* ctx);
bool chunked_splits_rows(bgmf_ctx* ctx, const int32_t* plan, int q0, int q1, double factor,
                         double max_col_conc);
int launch_piece(bgmf_ctx* ctx, const BlockWork* d_work, int nwork, int chunks,
                 const int32_t* lrow, const int32_t* lcol, const float* val, int iters,
                 float alpha, float beta, double ratings, int cbits);
int launch_piece_sweep(bgmf_ctx* ctx, const BlockWork* d_work, int nwork, int chunks,
                       const int32_t* lrow, const int32_t* lcol, const float* val, float alpha,
                       float beta, int it, int cbits);
int run_step_stream_converge(bgmf_ctx* ctx, const int32_t* plan, const int32_t* batch_off,
                             int nbatch, double tol, int64_t cap, double alpha, double beta,
                             int64_t* iters_out, int32_t* capped_out);

// ordered.cu -- order-faithful stratum sweep (V slabs in shared memory)
void order_release(bgmf_ctx* ctx);
int ensure_order_index(bgmf_ctx* ctx);
bool ordered_block_ok(bgmf_ctx* ctx, int b);
bool use_ordered(bgmf_ctx* ctx, const int32_t* plan, int q0, int q1, bool converge = false);
bool order_risky(bgmf_ctx* ctx, const int32_t* plan, int q0, int q1);
int run_batch_ordered(bgmf_ctx* ctx, const int32_t* plan, int q0, int q1, int pos_base,
                      int iters, float alpha, float beta, bool conv = false, double tol = 0.0,
                      double alpha64 = 0.0, double beta64 = 0.0);
int run_shards_ordered(bgmf_ctx* ctx, const int32_t* r0, const int32_t* r1,
                       const int64_t* edges, int nshards, float* vpriv, float alpha, float beta,
                       double* sse_dev);

// stream.cu -- out-of-core: ratings in pinned host memory, device slot ring
int stream_enable(bgmf_ctx* ctx, int64_t slot_ratings, int nslots);
int stream_slots(bgmf_ctx* ctx, int64_t slot_ratings, int nslots);
__global__ void values_to_codes(const float* __restrict__ v, int64_t n, uint8_t* __restrict__ out);
// out-of-core partition (partition.cu): chunks of row blocks under `budget`
// bytes of HBM straight into the pinned streaming layout
int partition_ooc(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols, const double* vals,
                  int64_t nnz, int64_t n, int64_t m, int I, int J, int64_t budget,
                  int64_t slot_ratings, int nslots, int64_t row_lo = 0, int64_t row_hi = -1);
void stream_free(bgmf_ctx* ctx);
int stream_export(bgmf_ctx* ctx, int64_t* order, int32_t* lrows, int32_t* lcols);
int run_step_stream(bgmf_ctx* ctx, const int32_t* plan, const int32_t* batch_off, int nbatch,
                    int iters, float alpha, float beta);
int stream_batch(bgmf_ctx* ctx, const int32_t* plan, const int32_t* batch_off, int nbatch,
                 int iters, float alpha, float beta, int pos0);
// single-block exact kernel used by the stateless drop-ins
int block_exact(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols, const double* vals,
                int64_t count, double* u, int64_t u_rows, double* v, int64_t v_rows, int k,
                double alpha, double beta, int mode, int iters, double tol, int64_t cap,
                double* out6);

// gradient.cu -- verification kernels (_kernels.gradient_steps, kernel.py:161-179)
int gradient_steps(bgmf_ctx* c, const int64_t* rows, const int64_t* cols, const double* vals,
                   int64_t count, double* u, int64_t nu, double* v, int64_t nv, int k,
                   double alpha, double beta, int iters, double* out4);
int block_gradients(bgmf_ctx* c, const int64_t* rows, const int64_t* cols, const double* vals,
                    int64_t count, const double* u, int64_t nu, const double* v, int64_t nv,
                    int k, double beta, double* gu, double* gv, double* out2);

// init.cu
int init_factors_device(bgmf_ctx* ctx, uint64_t shi, uint64_t slo, uint64_t ihi, uint64_t ilo,
                        int64_t n, int64_t m, int k);

// eval.cu
int eval_sse_f32(bgmf_ctx* ctx, const int32_t* rows, const int32_t* cols, const float* vals,
                 const uint8_t* cold, double fallback, int64_t count, double* out);
int eval_sse_f64(bgmf_ctx* ctx, const double* u, const double* v, int k, const int32_t* rows,
                 const int32_t* cols, const double* vals, const uint8_t* cold, double fallback,
                 int64_t count, double* out);
int predict_f64(bgmf_ctx* ctx, const double* u, const double* v, int k, const int32_t* rows,
                const int32_t* cols, int64_t count, double* out_dev);

// timing
void record_begin(bgmf_ctx* ctx, int kind, double bytes, TimedLaunch** slot);
void record_end(bgmf_ctx* ctx, TimedLaunch* slot);
void harvest_timing(bgmf_ctx* ctx);

}  // namespace bgmf
