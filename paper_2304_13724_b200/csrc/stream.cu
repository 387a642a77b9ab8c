// stream.cu -- out-of-core epoch: the partitioned ratings live in pinned host
// memory and stream through a ring of device slots (the
// paper's motivating case).  Factors stay resident.
//
// Host layout.  For square grids the host copy is re-laid out by diagonal:
// batch t of step s is the diagonal d = (s + t) mod P (blocks ((j+d) mod P, j),
// j ascending -- exactly plan_step's order), so every batch, and every piece
// of it, is ONE contiguous range: one cudaMemcpyAsync per array per piece.
// When a block-local (row, col) fits 32 bits the records are packed as
// (row << cbits | col) + fp32 value: 8 B per rating instead of 12 over PCIe.
//
// A step is cut into "pieces": consecutive blocks of one batch whose ratings
// fit one slot.  Blocks of a batch own disjoint U/V slices, so any grouping
// of a batch's blocks into sequential pieces is the same algorithm, and a
// block's post-sweep SSE can run right after its own sweep.  Piece p uses slot
// p % nslots: a side stream copies piece p+1.. (H2D from pinned memory) while
// the compute stream sweeps piece p; events order "slot copied" -> "sweep" ->
// "slot free for the next copy".

#include <cstring>

#include "bgmf_internal.cuh"

namespace bgmf {

void stream_free(bgmf_ctx* c) {
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  for (auto p : c->s_lrow) dfree(p, c->stream);
  for (auto p : c->s_lcol) dfree(p, c->stream);
  for (auto p : c->s_val) dfree(p, c->stream);
  for (auto e : c->ev_copied) cudaEventDestroy(e);
  for (auto e : c->ev_consumed) cudaEventDestroy(e);
  c->s_lrow.clear(); c->s_lcol.clear(); c->s_val.clear();
  c->ev_copied.clear(); c->ev_consumed.clear();
  big_pinned_free(c->h_lrow);
  big_pinned_free(c->h_lcol);
  big_pinned_free(c->h_val);
  big_pinned_free(c->h_order);
  c->h_lrow = c->h_lcol = nullptr;
  c->h_val = nullptr;
  c->h_order = nullptr;
  c->h_pos.clear();
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  c->copy_stream = nullptr;
  c->streaming = false;
  c->packed = false;
  c->nslots = 0;
  c->slot_cap = 0;
}

namespace {

__global__ void pack_records(const int32_t* __restrict__ lrow, const int32_t* __restrict__ lcol,
                             int64_t n, int cbits, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)(((uint32_t)lrow[i] << cbits) | (uint32_t)lcol[i]);
}

// 1-byte value codes: every value an integer in 0..255 (rating scales:
// MovieLens 1..5, Netflix 1..5), so (float)code is the value bit for bit.
__global__ void byte_values_check(const float* __restrict__ v, int64_t n, int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float x = v[i];
    if (!(x >= 0.f && x <= 255.f && x == rintf(x))) *bad = 1;
  }
}

}  // namespace

__global__ void values_to_codes(const float* __restrict__ v, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)v[i];
}

int stream_enable(bgmf_ctx* c, int64_t slot_ratings, int nslots) {
  if (!c->partitioned) return fail(c, BGMF_ERR_STATE, "bgmf_partition has not been called");
  if (c->exact) return fail(c, BGMF_ERR_STATE, "streaming is fast-mode only");
  if (c->streaming) return fail(c, BGMF_ERR_STATE, "already streaming");
  if (nslots < 2 || nslots > 8) return fail(c, BGMF_ERR_ARG, "nslots must be in [2, 8]");
  const int nb = c->I * c->J;
  int64_t max_block = 0;
  for (int b = 0; b < nb; ++b) {
    const int64_t cnt = c->h_offsets[b + 1] - c->h_offsets[b];
    if (cnt > max_block) max_block = cnt;
  }
  if (slot_ratings < max_block || slot_ratings < 1)
    return fail(c, BGMF_ERR_ARG, "slot smaller than the largest block (" +
                                     std::to_string(max_block) + " ratings)");
  cudaStream_t s = c->stream;
  c->packed = c->rbits + c->cbits <= 32;
  // host block order: diagonals of the rotating plan for square grids
  std::vector<int> order;
  order.reserve(nb);
  if (c->I == c->J) {
    for (int d = 0; d < c->I; ++d)
      for (int j = 0; j < c->J; ++j) order.push_back(((j + d) % c->I) * c->J + j);
  } else {
    for (int b = 0; b < nb; ++b) order.push_back(b);
  }
  c->h_pos.assign(nb, 0);
  int64_t pos = 0;
  for (int b : order) {
    c->h_pos[b] = pos;
    pos += c->h_offsets[b + 1] - c->h_offsets[b];
  }
  const size_t N = (size_t)(c->nnz > 0 ? c->nnz : 1);
  c->val8 = false;
  if (c->packed && c->nnz > 0) {  // 1-byte value codes when every value allows
    int* d_bad = nullptr;
    int h_bad = 0;
    BGMF_CK(c, dmalloc(&d_bad, sizeof(int), s));
    BGMF_CK(c, cudaMemsetAsync(d_bad, 0, sizeof(int), s));
    byte_values_check<<<c->num_sms * 8, 256, 0, s>>>(c->d_val, c->nnz, d_bad);
    BGMF_CK(c, cudaMemcpyAsync(&h_bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    BGMF_CK(c, cudaStreamSynchronize(s));
    dfree(d_bad, s);
    c->val8 = h_bad == 0 && !c->no_val8;
    if (c->val8) {  // codes in place of the fp32 values
      uint8_t* codes = nullptr;
      BGMF_CK(c, dmalloc(&codes, N, s));
      values_to_codes<<<c->num_sms * 8, 256, 0, s>>>(c->d_val, c->nnz, codes);
      BGMF_CK(c, cudaGetLastError());
      BGMF_CK(c, cudaStreamSynchronize(s));
      dfree(c->d_val, s);
      c->d_val = reinterpret_cast<float*>(codes);
    }
  }
  BGMF_CK(c, big_pinned_alloc((void**)&c->h_lrow, N * 4));
  if (!c->packed) BGMF_CK(c, big_pinned_alloc((void**)&c->h_lcol, N * 4));
  BGMF_CK(c, big_pinned_alloc((void**)&c->h_val, N * val_bytes(c)));
  BGMF_CK(c, big_pinned_alloc((void**)&c->h_order, N * 4));
  if (c->packed && c->nnz > 0) {  // pack in place of the (no longer needed) lrow
    int32_t* rec = nullptr;
    BGMF_CK(c, dmalloc(&rec, N * 4, c->stream));
    pack_records<<<c->num_sms * 8, 256, 0, s>>>(c->d_lrow, c->d_lcol, c->nnz, c->cbits, rec);
    BGMF_CK(c, cudaGetLastError());
    BGMF_CK(c, cudaStreamSynchronize(s));
    dfree(c->d_lrow, c->stream);
    c->d_lrow = rec;
  }
  for (int b : order) {  // D2H block by block into the diagonal layout
    const int64_t lo = c->h_offsets[b], cnt = c->h_offsets[b + 1] - lo, dst = c->h_pos[b];
    if (cnt == 0) continue;
    BGMF_CK(c, cudaMemcpyAsync(c->h_lrow + dst, c->d_lrow + lo, cnt * 4, cudaMemcpyDeviceToHost, s));
    if (!c->packed)
      BGMF_CK(c, cudaMemcpyAsync(c->h_lcol + dst, c->d_lcol + lo, cnt * 4, cudaMemcpyDeviceToHost,
                                 s));
    BGMF_CK(c, cudaMemcpyAsync(reinterpret_cast<char*>(c->h_val) + dst * val_bytes(c),
                               reinterpret_cast<const char*>(c->d_val) + lo * val_bytes(c),
                               cnt * val_bytes(c), cudaMemcpyDeviceToHost, s));
    BGMF_CK(c, cudaMemcpyAsync(c->h_order + dst, c->d_order + lo, cnt * 4, cudaMemcpyDeviceToHost,
                               s));
  }
  BGMF_CK(c, cudaStreamSynchronize(s));
  dfree(c->d_lrow, c->stream); dfree(c->d_lcol, c->stream); dfree(c->d_val, c->stream); dfree(c->d_order, c->stream);
  c->d_lrow = c->d_lcol = nullptr;
  c->d_val = nullptr;
  c->d_order = nullptr;
  return stream_slots(c, slot_ratings, nslots);
}

// The device slot ring and the copy stream of the streaming path.
int stream_slots(bgmf_ctx* c, int64_t slot_ratings, int nslots) {
  c->slot_cap = slot_ratings;
  c->nslots = nslots;
  for (int i = 0; i < nslots; ++i) {
    int32_t *a = nullptr, *b = nullptr;
    float* v = nullptr;
    BGMF_CK(c, dmalloc(&a, (size_t)slot_ratings * 4, c->stream));
    if (!c->packed) BGMF_CK(c, dmalloc(&b, (size_t)slot_ratings * 4, c->stream));
    BGMF_CK(c, dmalloc(&v, (size_t)slot_ratings * 4, c->stream));
    c->s_lrow.push_back(a);
    c->s_lcol.push_back(b);
    c->s_val.push_back(v);
    cudaEvent_t e1, e2;
    BGMF_CK(c, cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    BGMF_CK(c, cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
    c->ev_copied.push_back(e1);
    c->ev_consumed.push_back(e2);
  }
  BGMF_CK(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  c->streaming = true;
  return BGMF_OK;
}

// Host copies for bgmf_partition_export while streaming (partitioned order).
int stream_export(bgmf_ctx* c, int64_t* order, int32_t* lrows, int32_t* lcols) {
  if (!order && !lrows && !lcols) return BGMF_OK;  // offsets only (the trainer's call)
  const int nb = c->I * c->J;
  const uint32_t cmask = c->cbits >= 32 ? 0xFFFFFFFFu : ((1u << c->cbits) - 1u);
#pragma omp parallel for schedule(dynamic, 1)
  for (int b = 0; b < nb; ++b) {
    const int64_t lo = c->h_offsets[b], cnt = c->h_offsets[b + 1] - lo, src = c->h_pos[b];
    for (int64_t i = 0; i < cnt; ++i) {
      if (c->packed) {
        const uint32_t rc = (uint32_t)c->h_lrow[src + i];
        if (lrows) lrows[lo + i] = (int32_t)(rc >> c->cbits);
        if (lcols) lcols[lo + i] = (int32_t)(rc & cmask);
      } else {
        if (lrows) lrows[lo + i] = c->h_lrow[src + i];
        if (lcols) lcols[lo + i] = c->h_lcol[src + i];
      }
      if (order) order[lo + i] = (int64_t)c->h_order[src + i];
    }
  }
  return BGMF_OK;
}

namespace {

struct Piece {
  int w0, nw, chunks;  // work-table range
  int slot;
  double ratings;
};

}  // namespace

// Cut every batch into pieces that fit a slot (and one L2 wave); slot-relative
// work items into h_work[0, *w).  Pieces never span batches.
static int build_pieces(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off, int nbatch,
                        std::vector<Piece>& pieces, int* w_out, int w_base = 0, int pos0 = 0,
                        int64_t slot_seq = 0) {
  const int nb = c->I * c->J;
  const int64_t groups = fast_groups(c);
  int w = w_base;
  for (int t = 0; t < nbatch; ++t) {
    // the ordered kernel does not stream: where the chunked sweep would
    // distort the reference order (order_risky) each block is one chunk --
    // one group walks it in stored order (exact but for the next rating's V
    // row being read one update early when two consecutive ratings share a
    // column)
    const bool seq = c->ord_mode != 0 && order_risky(c, plan, batch_off[t], batch_off[t + 1]);
    int q = batch_off[t];
    while (q < batch_off[t + 1]) {
      int q_end = q;
      int64_t fill = 0;
      double vbytes = 0;
      int nonempty = 0;
      while (q_end < batch_off[t + 1]) {
        const int b = plan[q_end];
        if (b < 0 || b >= nb) return fail(c, BGMF_ERR_ARG, "plan block id out of range");
        const int64_t cnt = c->h_offsets[b + 1] - c->h_offsets[b];
        if (fill + cnt > c->slot_cap) break;
        // one L2-resident wave per piece (l2_waves, sgd.cu)
        const int bj = b % c->J;
        const double vb = (double)(c->col_bounds[bj + 1] - c->col_bounds[bj]) * c->kp * 4.0;
        if (c->l2_wave_bytes > 0 && q_end > q && vbytes + vb > (double)c->l2_wave_bytes) break;
        vbytes += vb;
        fill += cnt;
        nonempty += cnt > 0;
        ++q_end;
      }
      const int64_t slots = groups - nonempty > 0 ? groups - nonempty : 1;
      int64_t cl = (fill + slots - 1) / slots;
      if (cl < c->min_chunk) cl = c->min_chunk;
      cl = stagger_chunk(cl, c->stagger);
      Piece pc{w, 0, 0, (int)((slot_seq + (int64_t)pieces.size()) % c->nslots), 0.0};
      int64_t off = 0;
      for (int qq = q; qq < q_end; ++qq) {
        const int b = plan[qq];
        const int64_t cnt = c->h_offsets[b + 1] - c->h_offsets[b];
        if (cnt == 0) continue;
        const int64_t bl = seq ? cnt : (cl < cnt ? cl : cnt);
        BlockWork& bw = c->h_work[w++];
        bw.begin = off;
        bw.end = off + cnt;
        bw.row_start = c->row_bounds[b / c->J];
        bw.col_start = c->col_bounds[b % c->J];
        bw.chunk_len = (int32_t)bl;
        bw.first_chunk = pc.chunks;
        bw.block_id = b;
        bw.pos = pos0 + qq;
        bw.active = nullptr;
        bw.iter = nullptr;
        pc.chunks += (int)((cnt + bl - 1) / bl);
        pc.ratings += (double)cnt;
        off += cnt;
      }
      pc.nw = w - pc.w0;
      pieces.push_back(pc);
      q = q_end;
    }
  }
  *w_out = w;
  return BGMF_OK;
}

int run_step_stream(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off, int nbatch,
                    int iters, float alpha, float beta) {
  cudaStream_t s = c->stream, cs = c->copy_stream;
  const int nb = c->I * c->J;
  const int total = batch_off[nbatch];
  int rc = ensure_step_scratch(c, (size_t)total);
  if (rc) return rc;
  // 1. pieces and their slot-relative work items
  std::vector<Piece> pieces;
  int w = 0;
  if ((rc = build_pieces(c, plan, batch_off, nbatch, pieces, &w))) return rc;

  if (w > 0)
    BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work, sizeof(BlockWork) * w,
                               cudaMemcpyHostToDevice, s));
  BGMF_CK(c, cudaMemsetAsync(c->d_sse, 0, sizeof(double) * nb, s));
  BGMF_CK(c, cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  // the copy stream must not overwrite a slot before the work table is in place
  cudaEvent_t ready;
  BGMF_CK(c, cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  BGMF_CK(c, cudaEventRecord(ready, s));
  BGMF_CK(c, cudaStreamWaitEvent(cs, ready, 0));

  // one H2D per array for a run of host-contiguous blocks
  auto copy_run = [&](int sl, int64_t dst, int64_t src, int64_t cnt) -> int {
    BGMF_CK(c, cudaMemcpyAsync(c->s_lrow[sl] + dst, c->h_lrow + src, cnt * 4,
                               cudaMemcpyHostToDevice, cs));
    if (!c->packed)
      BGMF_CK(c, cudaMemcpyAsync(c->s_lcol[sl] + dst, c->h_lcol + src, cnt * 4,
                                 cudaMemcpyHostToDevice, cs));
    BGMF_CK(c, cudaMemcpyAsync(reinterpret_cast<char*>(c->s_val[sl]) + dst * val_bytes(c),
                               reinterpret_cast<const char*>(c->h_val) + src * val_bytes(c),
                               cnt * val_bytes(c), cudaMemcpyHostToDevice, cs));
    c->h2d_bytes += (double)((c->packed ? 4 : 8) + val_bytes(c)) * (double)cnt;
    return BGMF_OK;
  };

  // 2. pipeline: copy piece p on the side stream, compute it on the main one
  for (size_t p = 0; p < pieces.size(); ++p) {
    const Piece& pc = pieces[p];
    const int sl = pc.slot;
    if (p >= (size_t)c->nslots) BGMF_CK(c, cudaStreamWaitEvent(cs, c->ev_consumed[sl], 0));
    int64_t run_dst = 0, run_src = -1, run_cnt = 0;
    for (int i = 0; i < pc.nw; ++i) {
      const BlockWork& bw = c->h_work[pc.w0 + i];
      const int64_t src = c->h_pos[bw.block_id];
      const int64_t cnt = bw.end - bw.begin;
      if (run_src >= 0 && src == run_src + run_cnt && bw.begin == run_dst + run_cnt) {
        run_cnt += cnt;  // extends the contiguous run
        continue;
      }
      if (run_src >= 0 && (rc = copy_run(sl, run_dst, run_src, run_cnt))) break;
      run_dst = bw.begin;
      run_src = src;
      run_cnt = cnt;
    }
    if (!rc && run_src >= 0) rc = copy_run(sl, run_dst, run_src, run_cnt);
    if (rc) { cudaEventDestroy(ready); return rc; }
    BGMF_CK(c, cudaEventRecord(c->ev_copied[sl], cs));
    BGMF_CK(c, cudaStreamWaitEvent(s, c->ev_copied[sl], 0));
    rc = launch_piece(c, c->d_work + pc.w0, pc.nw, pc.chunks, c->s_lrow[sl], c->s_lcol[sl],
                      c->s_val[sl], iters, alpha, beta, pc.ratings, stream_cbits(c));
    if (rc) { cudaEventDestroy(ready); return rc; }
    BGMF_CK(c, cudaEventRecord(c->ev_consumed[sl], s));
  }
  BGMF_CK(c, cudaMemcpyAsync(c->h_sse, c->d_sse, sizeof(double) * nb, cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaStreamSynchronize(s));
  cudaEventDestroy(ready);
  if (c->timing) harvest_timing(c);
  return BGMF_OK;
}

// One batch of an asynchronous step (the multi-GPU ring, sgd.cu step_batch)
// on a streaming context: the batch's pieces go through the slot ring with the
// copy stream running ahead, nothing waits on the host.  Work items go to the
// step's reserved work-table range at c->w_cursor; slots rotate with a
// context-wide piece counter, and a piece always waits until its slot's
// previous occupant has been swept (ev_consumed; a no-op for a fresh slot).
int stream_batch(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off, int nbatch,
                 int iters, float alpha, float beta, int pos0) {
  cudaStream_t s = c->stream, cs = c->copy_stream;
  std::vector<Piece> pieces;
  int w_end = c->w_cursor;
  int rc = build_pieces(c, plan, batch_off, nbatch, pieces, &w_end, c->w_cursor, pos0,
                        c->piece_seq);
  if (rc) return rc;
  if (w_end > c->w_limit)
    return fail(c, BGMF_ERR_ARG, "more blocks than reserved by bgmf_step_begin");
  if (w_end > c->w_cursor)
    BGMF_CK(c, cudaMemcpyAsync(c->d_work + c->w_cursor, c->h_work + c->w_cursor,
                               sizeof(BlockWork) * (w_end - c->w_cursor), cudaMemcpyHostToDevice,
                               s));
  for (const Piece& pc : pieces) {
    const int sl = pc.slot;
    BGMF_CK(c, cudaStreamWaitEvent(cs, c->ev_consumed[sl], 0));
    int64_t run_dst = 0, run_src = -1, run_cnt = 0;
    auto copy_run = [&](int64_t dst, int64_t src, int64_t cnt) -> int {
      BGMF_CK(c, cudaMemcpyAsync(c->s_lrow[sl] + dst, c->h_lrow + src, cnt * 4,
                                 cudaMemcpyHostToDevice, cs));
      if (!c->packed)
        BGMF_CK(c, cudaMemcpyAsync(c->s_lcol[sl] + dst, c->h_lcol + src, cnt * 4,
                                   cudaMemcpyHostToDevice, cs));
      BGMF_CK(c, cudaMemcpyAsync(reinterpret_cast<char*>(c->s_val[sl]) + dst * val_bytes(c),
                                 reinterpret_cast<const char*>(c->h_val) + src * val_bytes(c),
                                 cnt * val_bytes(c), cudaMemcpyHostToDevice, cs));
      c->h2d_bytes += (double)((c->packed ? 4 : 8) + val_bytes(c)) * (double)cnt;
      return BGMF_OK;
    };
    for (int i = 0; i < pc.nw && !rc; ++i) {
      const BlockWork& bw = c->h_work[pc.w0 + i];
      const int64_t src = c->h_pos[bw.block_id];
      const int64_t cnt = bw.end - bw.begin;
      if (run_src >= 0 && src == run_src + run_cnt && bw.begin == run_dst + run_cnt) {
        run_cnt += cnt;
        continue;
      }
      if (run_src >= 0) rc = copy_run(run_dst, run_src, run_cnt);
      run_dst = bw.begin;
      run_src = src;
      run_cnt = cnt;
    }
    if (!rc && run_src >= 0) rc = copy_run(run_dst, run_src, run_cnt);
    if (rc) return rc;
    BGMF_CK(c, cudaEventRecord(c->ev_copied[sl], cs));
    BGMF_CK(c, cudaStreamWaitEvent(s, c->ev_copied[sl], 0));
    rc = launch_piece(c, c->d_work + pc.w0, pc.nw, pc.chunks, c->s_lrow[sl], c->s_lcol[sl],
                      c->s_val[sl], iters, alpha, beta, pc.ratings, stream_cbits(c));
    if (rc) return rc;
    BGMF_CK(c, cudaEventRecord(c->ev_consumed[sl], s));
  }
  c->piece_seq += (int64_t)pieces.size();
  c->w_cursor = w_end;
  return BGMF_OK;
}

// ConvergeEachBlock while streaming (_kernels.py:62-100 per block): piece by
// piece, the piece's ratings are copied into a slot once, then its blocks
// sweep until their RMSE improves by less than tol (or cap sweeps), each
// iteration one sweep launch over the still-active blocks plus an SSE
// measurement read back to the host -- the in-core run_step_converge_fast
// loop on slot-resident data.  Synchronous (no copy/compute overlap): the
// per-iteration host decision dominates anyway.
int run_step_stream_converge(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off,
                             int nbatch, double tol, int64_t cap, double alpha, double beta,
                             int64_t* iters_out, int32_t* capped_out) {
  cudaStream_t s = c->stream;
  const int nb = c->I * c->J;
  const int total = batch_off[nbatch];
  int rc = ensure_step_scratch(c, 2 * (size_t)(total > 0 ? total : 1));
  if (rc) return rc;
  std::vector<Piece> pieces;
  int w = 0;
  if ((rc = build_pieces(c, plan, batch_off, nbatch, pieces, &w))) return rc;
  for (int b = 0; b < nb; ++b) { iters_out[b] = 0; capped_out[b] = 0; }
  std::vector<double> sse_final(nb, 0.0);
  unsigned long long best = kNoBad;
  const int cb = stream_cbits(c);
  BGMF_CK(c, cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  for (const Piece& pc : pieces) {
    const int sl = 0;
    for (int i = 0; i < pc.nw; ++i) {  // the piece's blocks into slot 0
      const BlockWork& bw = c->h_work[pc.w0 + i];
      const int64_t src = c->h_pos[bw.block_id], cnt = bw.end - bw.begin;
      BGMF_CK(c, cudaMemcpyAsync(c->s_lrow[sl] + bw.begin, c->h_lrow + src, cnt * 4,
                                 cudaMemcpyHostToDevice, s));
      if (!c->packed)
        BGMF_CK(c, cudaMemcpyAsync(c->s_lcol[sl] + bw.begin, c->h_lcol + src, cnt * 4,
                                   cudaMemcpyHostToDevice, s));
      BGMF_CK(c, cudaMemcpyAsync(reinterpret_cast<char*>(c->s_val[sl]) + bw.begin * val_bytes(c),
                                 reinterpret_cast<const char*>(c->h_val) + src * val_bytes(c),
                                 cnt * val_bytes(c),
                                 cudaMemcpyHostToDevice, s));
      c->h2d_bytes += (double)((c->packed ? 4 : 8) + val_bytes(c)) * (double)cnt;
    }
    std::vector<char> active(pc.nw, 1);
    std::vector<double> prev(pc.nw, 0.0);
    int n_active = pc.nw;
    // active blocks' work items (slot offsets unchanged) at h_work[w, ...)
    auto upload_active = [&](int* nw, int* chunks) -> int {
      *nw = 0;
      *chunks = 0;
      for (int i = 0; i < pc.nw; ++i) {
        if (!active[i]) continue;
        BlockWork bw = c->h_work[pc.w0 + i];
        bw.first_chunk = *chunks;
        *chunks += (int)((bw.end - bw.begin + bw.chunk_len - 1) / bw.chunk_len);
        c->h_work[w + (*nw)++] = bw;
      }
      if (*nw > 0)
        BGMF_CK(c, cudaMemcpyAsync(c->d_work + w, c->h_work + w, sizeof(BlockWork) * (*nw),
                                   cudaMemcpyHostToDevice, s));
      return BGMF_OK;
    };
    auto measure = [&](int nw, int chunks) -> int {  // SSE of the active blocks
      BGMF_CK(c, cudaMemsetAsync(c->d_sse, 0, sizeof(double) * nb, s));
      int r2 = launch_piece(c, c->d_work + w, nw, chunks, c->s_lrow[sl], c->s_lcol[sl],
                            c->s_val[sl], 0, (float)alpha, (float)beta, 0.0, cb);
      if (r2) return r2;
      BGMF_CK(c, cudaMemcpyAsync(c->h_sse, c->d_sse, sizeof(double) * nb,
                                 cudaMemcpyDeviceToHost, s));
      BGMF_CK(c, cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, s));
      BGMF_CK(c, cudaStreamSynchronize(s));
      return BGMF_OK;
    };
    int nw = 0, chunks = 0;
    if ((rc = upload_active(&nw, &chunks)) || (rc = measure(nw, chunks))) return rc;
    for (int i = 0; i < pc.nw; ++i) {
      const BlockWork& bw = c->h_work[pc.w0 + i];
      prev[i] = std::sqrt(c->h_sse[bw.block_id] / (double)(bw.end - bw.begin));
    }
    int64_t it = 0;
    while (n_active > 0 && it < cap) {
      if ((rc = upload_active(&nw, &chunks))) return rc;
      if ((rc = launch_piece_sweep(c, c->d_work + w, nw, chunks, c->s_lrow[sl], c->s_lcol[sl],
                                   c->s_val[sl], (float)alpha, (float)beta, (int)(it & 0xFFFF),
                                   cb)))
        return rc;
      ++it;
      if ((rc = measure(nw, chunks))) return rc;
      for (int i = 0; i < pc.nw; ++i) {
        if (!active[i]) continue;
        const BlockWork& bw = c->h_work[pc.w0 + i];
        const int64_t cnt = bw.end - bw.begin;
        const double cur = c->h_sse[bw.block_id];
        iters_out[bw.block_id] = it;
        sse_final[bw.block_id] = cur;
        const double now = std::sqrt(cur / (double)cnt);
        if (!std::isfinite(cur)) {
          const unsigned long long key = pack_bad(bw.pos, it - 1, cnt - 1);
          if (key < best) best = key;
          active[i] = 0; --n_active;
        } else if (prev[i] - now < tol) {
          active[i] = 0; --n_active;
        } else {
          prev[i] = now;
        }
      }
      if (*c->h_bad != kNoBad) break;
    }
    for (int i = 0; i < pc.nw; ++i)
      if (active[i]) capped_out[c->h_work[pc.w0 + i].block_id] = 1;
    if (*c->h_bad != kNoBad) break;
  }
  for (int b = 0; b < nb; ++b) c->h_sse[b] = sse_final[b];
  if (*c->h_bad < best) best = *c->h_bad;
  *c->h_bad = best;
  return BGMF_OK;
}

}  // namespace bgmf
