// libbgs host runtime: context, workspace arena, transports (NCCL / in-process device group),
// and the C ABI entry points of include/bgs.h.  Orchestration only; every step of the path
// runs in the kernels of project.cu, sort.cu, raster.cu, project_bwd.cu, route.cu and
// importance.cu.  There is no CPU fallback: without a CUDA device every call fails.
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "bgs_internal.cuh"

using namespace bgs;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct Transport;
struct BatchState;

}  // namespace

struct bgs_ctx;
namespace {
void destroy_batch(bgs_ctx* c);  // NEXT-2 batch state (defined with bgs_batch_step)
}  // namespace

// bgs_stage_times: project, route, sort, raster_fwd, loss, raster_bwd, route_reverse, project_bwd,
// importance
constexpr int kStages = 9;

struct bgs_ctx {
  int rank = 0, world = 1, device = 0;
  std::shared_ptr<Transport> tr;
  std::string err;
  int64_t launches = 0;
  int64_t host_syncs = 0;  // times an ABI call blocked the host on the device (bgs_host_sync_count)
  int64_t collectives = 0;  // transport collectives issued (bgs_batch_stats)
  bool capturing = false;         // a CUDA graph capture is open on this ctx's work: ensure() must not grow
  bool grew_in_capture = false;   // ... and it had to (the batch then runs eagerly)
  BatchState* batch = nullptr;    // NEXT-2 batched step (bgs_batch_step), created on first use
  // view state
  CameraK cam{};
  int T = 0;
  int stage = 0;  // 1 projected, 2 routed, 3 sorted, 4 fwd, 5 bwd, 6 reversed
  int64_t n_local = 0, F = 0, P_all = 0, R = 0, D = 0, P = 0, n_lod = 0, n_act = 0;
  int t_begin = 0, t_end = 0, n_passes = 0, fallback = 0;
  int raster_split = 0;  // heavy tiles split over two CTAs in the last forward (the backward reuses it)
  int imp_parity = 0;  // which half of imp_hist the next world-1 importance call uses
  bool colored = false;  // the last projection ran k_color (its Jacobian feeds bgs_project_bwd)
  int pend_gate = 0, pend_fb_num = 0, pend_fb_den = 1;  // gate of the enqueued projection (project_finish)
  const Rec* recv = nullptr;  // == recs at world 1
  Acc* acc_local = nullptr;   // == acc at world 1
  // arena
  DevBuf counters, recs, rec_lidx, tile_diff, tile_pairs, owner, runinfo, dest_mask, block_counts, totals,
      send_base, send, recvbuf, keys[2], vals[2], digit_hist, pass_ctrl, status, ranges, acc, rev, accl, imp_state,
      imp_hist, imp_total, scr_rgb, scr_t, scr_n, scr_dl, xchg_counts, aux, tile_perm, cand, wbuf, cmask,
      loss_img, loss_part, loss_sums, scr_tgt, scr_loss, scr_in2,
      scr_dlsup,  // supervised steps' dL/dC (never one of the host-upload double buffers)
      bucket_cur,  // per-tile write cursors of the bucket sort
      jdir,  // per local record: k_color's colour Jacobian wrt the view direction + clamp bits (a11 input)
      imp_cand, imp_gath;  // world > 1 importance: this rank's crossing-bin candidates, all ranks' gathered
  // NEXT-1 simplification scratch (selection keys / state / histograms, keep masks, row exchange)
  DevBuf sel_keys, sel_state, sel_hist, masks, sblocks, new_gid, rows_send, rows_recv, dcnt;
  unsigned long long* h_counters = nullptr;  // pinned
  int64_t* h_misc = nullptr;                 // pinned scratch for routing sizes
  cudaEvent_t ev_counters = nullptr;         // counters copied to the host (bgs_project)
  cudaEvent_t ev_geom = nullptr;             // geometry kernels done (bgs_project)
  cudaStream_t side = nullptr;               // carries the counters copy off the working stream
  cudaStream_t hi = nullptr;                 // high-priority stream for the latency-bound stages (view steps)
  cudaEvent_t ev_hi_fork = nullptr, ev_hi_join = nullptr;
  bool stage_timing = false, stage_recorded = false;  // bgs_set_stage_timing / bgs_stage_times
  cudaStream_t h2d = nullptr, d2h = nullptr;          // host-buffer step: copy streams
  cudaEvent_t ev_in = nullptr, ev_dl = nullptr, ev_fwd = nullptr, ev_out = nullptr;
  // host-buffer steps: the uploaded input (dL/dC or the target) alternates between two buffers, so
  // a view's upload waits only for the view two steps back that read the same buffer
  cudaEvent_t ev_in_free[2] = {nullptr, nullptr};
  int in_parity = 0;
  cudaEvent_t stage_ev[kStages + 1] = {};
  std::vector<int64_t> send_cnt, recv_cnt, send_off, recv_off;
};

namespace {

// The ABI's stream argument: NULL selects the calling thread's per-thread default stream
// (cudaStreamPerThread), never the legacy default stream; it is still ordered with
// legacy-stream work of the same process (the per-thread stream is a blocking stream).
inline cudaStream_t as_stream(void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
}

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) return fail(ctx, BGS_ERR_CUDA, #call, cudaGetErrorString(e_)); \
  } while (0)

#define CK_CTX(c, call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) return fail(c, BGS_ERR_CUDA, #call, cudaGetErrorString(e_)); \
  } while (0)

#define CKS(call)                                   \
  do {                                              \
    bgs_status s_ = (call);                         \
    if (s_ != BGS_OK) return s_;                    \
  } while (0)

bgs_status fail(bgs_ctx* ctx, bgs_status st, const char* what, const char* detail = "") {
  if (ctx) ctx->err = std::string(what) + (detail && *detail ? std::string(": ") + detail : std::string());
  return st;
}

bgs_status launched(bgs_ctx* ctx, int n = 1) {
  ctx->launches += n;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, BGS_ERR_CUDA, "kernel launch", cudaGetErrorString(e));
  return BGS_OK;
}

// The ABI's host synchronisations, counted (bgs_host_sync_count)
cudaError_t host_sync(bgs_ctx* ctx, cudaStream_t s) {
  ++ctx->host_syncs;
  return cudaStreamSynchronize(s);
}
cudaError_t host_sync_event(bgs_ctx* ctx, cudaEvent_t e) {
  ++ctx->host_syncs;
  return cudaEventSynchronize(e);
}

bgs_status ensure(bgs_ctx* ctx, DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (bytes <= b.cap) return BGS_OK;
  if (ctx->capturing) {  // a graph is being captured: growing (cudaFree / cudaMalloc) is not allowed
    ctx->grew_in_capture = true;
    return fail(ctx, BGS_ERR_CAPACITY, "arena growth needed during graph capture");
  }
  if (b.p) {
    cudaError_t e = cudaFree(b.p);
    if (e != cudaSuccess) return fail(ctx, BGS_ERR_CUDA, "cudaFree", cudaGetErrorString(e));
  }
  // 1.5x headroom: per-view sizes vary by 2-3x across a camera set, and every regrowth is a
  // cudaFree + cudaMalloc in the middle of a step
  size_t want = bytes + bytes / 2 + 4096;
  cudaError_t e = cudaMalloc(&b.p, want);
  if (e != cudaSuccess) {
    b.p = nullptr;
    b.cap = 0;
    char msg[128];
    snprintf(msg, sizeof msg, "arena grow to %zu bytes", want);
    return fail(ctx, BGS_ERR_CAPACITY, msg, cudaGetErrorString(e));
  }
  b.cap = want;
  return BGS_OK;
}

template <class T>
T* P_(DevBuf& b) {
  return static_cast<T*>(b.p);
}

// ---------------------------------------------------------------------------------------
// Transports
// ---------------------------------------------------------------------------------------
struct Transport {
  virtual ~Transport() = default;
  virtual bgs_status allreduce_i32(bgs_ctx* ctx, int32_t* buf, int64_t n, cudaStream_t s) = 0;
  virtual bgs_status allreduce_u64(bgs_ctx* ctx, unsigned long long* buf, int64_t n, cudaStream_t s) = 0;
  virtual bgs_status allreduce_f32(bgs_ctx* ctx, float* buf, int64_t n, cudaStream_t s) = 0;
  virtual bgs_status allreduce_f64(bgs_ctx* ctx, double* buf, int64_t n, cudaStream_t s) = 0;
  // device int64 [world] -> device int64 [world]: element d of send goes to rank d
  virtual bgs_status alltoall1(bgs_ctx* ctx, const int64_t* send, int64_t* recv, cudaStream_t s) = 0;
  virtual bgs_status alltoallv(bgs_ctx* ctx, const void* send, const int64_t* scnt, const int64_t* soff, void* recv,
                               const int64_t* rcnt, const int64_t* roff, size_t elem, cudaStream_t s) = 0;
  // device int64 [world][n] -> [world][n]: send[p n .. p n + n) goes to rank p (batched counts)
  virtual bgs_status alltoall_n(bgs_ctx* ctx, const int64_t* send, int64_t* recv, int n, cudaStream_t s) = 0;
  // ONE grouped exchange of nb segment sets (the views of a batch): for every view b and peer p,
  // send[b] + soff[b M + p] (scnt[b M + p] elements) goes to p, and recv[b] + roff[b M + k] gets
  // rcnt[b M + k] elements from k
  virtual bgs_status alltoallv_batch(bgs_ctx* ctx, int nb, const void* const* send, const int64_t* scnt,
                                     const int64_t* soff, void* const* recv, const int64_t* rcnt, const int64_t* roff,
                                     size_t elem, cudaStream_t s) = 0;
  // every rank's `bytes` bytes of send, concatenated in rank order into recv (world x bytes)
  virtual bgs_status allgather(bgs_ctx* ctx, const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  virtual bool capturable() const = 0;  // collectives may be recorded into a CUDA graph
};

bgs_status nccl_fail(bgs_ctx* ctx, ncclResult_t r, const char* what) {
  return fail(ctx, BGS_ERR_NCCL, what, ncclGetErrorString(r));
}

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  ~NcclTransport() override {
    if (comm) ncclCommDestroy(comm);
  }
  bgs_status allreduce_i32(bgs_ctx* ctx, int32_t* buf, int64_t n, cudaStream_t s) override {
    ++ctx->collectives;
    ncclResult_t r = ncclAllReduce(buf, buf, size_t(n), ncclInt32, ncclSum, comm, s);
    return r == ncclSuccess ? BGS_OK : nccl_fail(ctx, r, "ncclAllReduce");
  }
  bgs_status allreduce_u64(bgs_ctx* ctx, unsigned long long* buf, int64_t n, cudaStream_t s) override {
    ++ctx->collectives;
    ncclResult_t r = ncclAllReduce(buf, buf, size_t(n), ncclUint64, ncclSum, comm, s);
    return r == ncclSuccess ? BGS_OK : nccl_fail(ctx, r, "ncclAllReduce");
  }
  bgs_status allreduce_f32(bgs_ctx* ctx, float* buf, int64_t n, cudaStream_t s) override {
    ++ctx->collectives;
    ncclResult_t r = ncclAllReduce(buf, buf, size_t(n), ncclFloat32, ncclSum, comm, s);
    return r == ncclSuccess ? BGS_OK : nccl_fail(ctx, r, "ncclAllReduce");
  }
  bgs_status allreduce_f64(bgs_ctx* ctx, double* buf, int64_t n, cudaStream_t s) override {
    ++ctx->collectives;
    ncclResult_t r = ncclAllReduce(buf, buf, size_t(n), ncclFloat64, ncclSum, comm, s);
    return r == ncclSuccess ? BGS_OK : nccl_fail(ctx, r, "ncclAllReduce");
  }
  bgs_status alltoall1(bgs_ctx* ctx, const int64_t* send, int64_t* recv, cudaStream_t s) override {
    ++ctx->collectives;
    ncclResult_t r = ncclGroupStart();
    for (int p = 0; p < ctx->world && r == ncclSuccess; ++p) {
      r = ncclSend(send + p, 1, ncclInt64, p, comm, s);
      if (r == ncclSuccess) r = ncclRecv(recv + p, 1, ncclInt64, p, comm, s);
    }
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclSend/Recv counts");
    return r2 == ncclSuccess ? BGS_OK : nccl_fail(ctx, r2, "ncclGroupEnd");
  }
  bgs_status alltoallv(bgs_ctx* ctx, const void* send, const int64_t* scnt, const int64_t* soff, void* recv,
                       const int64_t* rcnt, const int64_t* roff, size_t elem, cudaStream_t s) override {
    ++ctx->collectives;
    ncclResult_t r = ncclGroupStart();
    for (int p = 0; p < ctx->world && r == ncclSuccess; ++p) {
      if (scnt[p] > 0)
        r = ncclSend(static_cast<const char*>(send) + soff[p] * elem, size_t(scnt[p]) * elem, ncclChar, p, comm, s);
      if (r == ncclSuccess && rcnt[p] > 0)
        r = ncclRecv(static_cast<char*>(recv) + roff[p] * elem, size_t(rcnt[p]) * elem, ncclChar, p, comm, s);
    }
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclSend/Recv records");
    return r2 == ncclSuccess ? BGS_OK : nccl_fail(ctx, r2, "ncclGroupEnd");
  }
  bgs_status alltoall_n(bgs_ctx* ctx, const int64_t* send, int64_t* recv, int n, cudaStream_t s) override {
    ++ctx->collectives;
    ncclResult_t r = ncclGroupStart();
    for (int p = 0; p < ctx->world && r == ncclSuccess; ++p) {
      r = ncclSend(send + size_t(p) * n, size_t(n), ncclInt64, p, comm, s);
      if (r == ncclSuccess) r = ncclRecv(recv + size_t(p) * n, size_t(n), ncclInt64, p, comm, s);
    }
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclSend/Recv batched counts");
    return r2 == ncclSuccess ? BGS_OK : nccl_fail(ctx, r2, "ncclGroupEnd");
  }
  bgs_status alltoallv_batch(bgs_ctx* ctx, int nb, const void* const* send, const int64_t* scnt, const int64_t* soff,
                             void* const* recv, const int64_t* rcnt, const int64_t* roff, size_t elem,
                             cudaStream_t s) override {
    ++ctx->collectives;
    const int M = ctx->world;
    ncclResult_t r = ncclGroupStart();
    for (int b = 0; b < nb && r == ncclSuccess; ++b)
      for (int p = 0; p < M && r == ncclSuccess; ++p) {
        const size_t i = size_t(b) * M + p;
        if (scnt[i] > 0)
          r = ncclSend(static_cast<const char*>(send[b]) + soff[i] * elem, size_t(scnt[i]) * elem, ncclChar, p, comm,
                       s);
        if (r == ncclSuccess && rcnt[i] > 0)
          r = ncclRecv(static_cast<char*>(recv[b]) + roff[i] * elem, size_t(rcnt[i]) * elem, ncclChar, p, comm, s);
      }
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclSend/Recv batched records");
    return r2 == ncclSuccess ? BGS_OK : nccl_fail(ctx, r2, "ncclGroupEnd");
  }
  bgs_status allgather(bgs_ctx* ctx, const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    ++ctx->collectives;
    ncclResult_t r = ncclAllGather(send, recv, bytes, ncclChar, comm, s);
    return r == ncclSuccess ? BGS_OK : nccl_fail(ctx, r, "ncclAllGather");
  }
  bool capturable() const override { return true; }
};

// In-process group of `world` contexts on one device (test transport).  Collectives are
// device-to-device copies / reduction kernels ordered by CUDA events; a host barrier orders
// the publication of pointers.  Each ctx is driven by its own host thread.
struct LocalGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;
  std::vector<const int64_t*> cnt, off;
  std::vector<const void* const*> bptr;  // batched exchange: per rank, its nb send pointers
  std::vector<cudaEvent_t> ready, done;
  explicit LocalGroup(int w) : world(w), ptr(w), cnt(w), off(w), bptr(w), ready(w), done(w) {
    for (int i = 0; i < w; ++i) {
      cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
    }
  }
  ~LocalGroup() {
    for (int i = 0; i < world; ++i) {
      cudaEventDestroy(ready[i]);
      cudaEventDestroy(done[i]);
    }
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalTransport : Transport {
  std::shared_ptr<LocalGroup> g;
  DevBuf tmp;  // reduction scratch
  explicit LocalTransport(std::shared_ptr<LocalGroup> grp) : g(std::move(grp)) {}
  ~LocalTransport() override {
    if (tmp.p) cudaFree(tmp.p);
  }
  template <class T, class L>
  bgs_status allreduce(bgs_ctx* ctx, T* buf, int64_t n, cudaStream_t s, L launch) {
    ++ctx->collectives;
    const int r = ctx->rank;
    CKS(ensure(ctx, tmp, size_t(n) * sizeof(T)));
    g->ptr[r] = buf;
    CK(cudaEventRecord(g->ready[r], s));
    g->barrier();
    PtrList pl{};
    pl.n = g->world;
    for (int k = 0; k < g->world; ++k) {
      pl.p[k] = g->ptr[k];
      CK(cudaStreamWaitEvent(s, g->ready[k], 0));
    }
    launch(pl, static_cast<T*>(tmp.p), n, s);
    CKS(launched(ctx));
    CK(cudaEventRecord(g->done[r], s));
    g->barrier();
    for (int k = 0; k < g->world; ++k) CK(cudaStreamWaitEvent(s, g->done[k], 0));
    CK(cudaMemcpyAsync(buf, tmp.p, size_t(n) * sizeof(T), cudaMemcpyDeviceToDevice, s));
    g->barrier();  // nobody republishes before everyone has queued its waits
    return BGS_OK;
  }
  bgs_status allreduce_i32(bgs_ctx* ctx, int32_t* buf, int64_t n, cudaStream_t s) override {
    return allreduce(ctx, buf, n, s, [](PtrList p, int32_t* d, int64_t nn, cudaStream_t ss) {
      launch_reduce_sum_i32(p, d, nn, ss);
    });
  }
  bgs_status allreduce_u64(bgs_ctx* ctx, unsigned long long* buf, int64_t n, cudaStream_t s) override {
    return allreduce(ctx, buf, n, s, [](PtrList p, unsigned long long* d, int64_t nn, cudaStream_t ss) {
      launch_reduce_sum_u64(p, d, nn, ss);
    });
  }
  bgs_status allreduce_f32(bgs_ctx* ctx, float* buf, int64_t n, cudaStream_t s) override {
    return allreduce(ctx, buf, n, s, [](PtrList p, float* d, int64_t nn, cudaStream_t ss) {
      launch_reduce_sum_f32(p, d, nn, ss);
    });
  }
  bgs_status allreduce_f64(bgs_ctx* ctx, double* buf, int64_t n, cudaStream_t s) override {
    return allreduce(ctx, buf, n, s, [](PtrList p, double* d, int64_t nn, cudaStream_t ss) {
      launch_reduce_sum_f64(p, d, nn, ss);
    });
  }
  bgs_status exchange(bgs_ctx* ctx, const void* send, const int64_t* scnt, const int64_t* soff, void* recv,
                      const int64_t* rcnt, const int64_t* roff, size_t elem, cudaStream_t s) {
    ++ctx->collectives;
    const int r = ctx->rank;
    g->ptr[r] = send;
    g->cnt[r] = scnt;
    g->off[r] = soff;
    CK(cudaEventRecord(g->ready[r], s));
    g->barrier();
    for (int k = 0; k < g->world; ++k) {
      CK(cudaStreamWaitEvent(s, g->ready[k], 0));
      const int64_t c = g->cnt[k][r];
      if (c != rcnt[k]) return fail(ctx, BGS_ERR_INTERNAL, "local exchange: count mismatch");
      if (c > 0)
        CK(cudaMemcpyAsync(static_cast<char*>(recv) + roff[k] * elem,
                           static_cast<const char*>(g->ptr[k]) + g->off[k][r] * elem, size_t(c) * elem,
                           cudaMemcpyDeviceToDevice, s));
    }
    CK(cudaEventRecord(g->done[r], s));
    g->barrier();
    for (int k = 0; k < g->world; ++k) CK(cudaStreamWaitEvent(s, g->done[k], 0));
    g->barrier();
    return BGS_OK;
  }
  bgs_status alltoall1(bgs_ctx* ctx, const int64_t* send, int64_t* recv, cudaStream_t s) override {
    std::vector<int64_t> one(ctx->world, 1), idx(ctx->world);
    for (int k = 0; k < ctx->world; ++k) idx[k] = k;
    return exchange(ctx, send, one.data(), idx.data(), recv, one.data(), idx.data(), sizeof(int64_t), s);
  }
  bgs_status alltoallv(bgs_ctx* ctx, const void* send, const int64_t* scnt, const int64_t* soff, void* recv,
                       const int64_t* rcnt, const int64_t* roff, size_t elem, cudaStream_t s) override {
    return exchange(ctx, send, scnt, soff, recv, rcnt, roff, elem, s);
  }
  bgs_status alltoall_n(bgs_ctx* ctx, const int64_t* send, int64_t* recv, int n, cudaStream_t s) override {
    std::vector<int64_t> cnt(ctx->world, n), idx(ctx->world);
    for (int k = 0; k < ctx->world; ++k) idx[k] = int64_t(k) * n;
    return exchange(ctx, send, cnt.data(), idx.data(), recv, cnt.data(), idx.data(), sizeof(int64_t), s);
  }
  bgs_status alltoallv_batch(bgs_ctx* ctx, int nb, const void* const* send, const int64_t* scnt, const int64_t* soff,
                             void* const* recv, const int64_t* rcnt, const int64_t* roff, size_t elem,
                             cudaStream_t s) override {
    ++ctx->collectives;
    const int r = ctx->rank, M = ctx->world;
    g->bptr[r] = send;
    g->cnt[r] = scnt;
    g->off[r] = soff;
    CK(cudaEventRecord(g->ready[r], s));
    g->barrier();
    for (int k = 0; k < M; ++k) CK(cudaStreamWaitEvent(s, g->ready[k], 0));
    for (int b = 0; b < nb; ++b)
      for (int k = 0; k < M; ++k) {
        const size_t mine = size_t(b) * M + k, theirs = size_t(b) * M + r;
        const int64_t c = g->cnt[k][theirs];
        if (c != rcnt[mine]) return fail(ctx, BGS_ERR_INTERNAL, "local batched exchange: count mismatch");
        if (c > 0)
          CK(cudaMemcpyAsync(static_cast<char*>(recv[b]) + roff[mine] * elem,
                             static_cast<const char*>(g->bptr[k][b]) + g->off[k][theirs] * elem, size_t(c) * elem,
                             cudaMemcpyDeviceToDevice, s));
      }
    CK(cudaEventRecord(g->done[r], s));
    g->barrier();
    for (int k = 0; k < M; ++k) CK(cudaStreamWaitEvent(s, g->done[k], 0));
    g->barrier();
    return BGS_OK;
  }
  bgs_status allgather(bgs_ctx* ctx, const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    std::vector<int64_t> cnt(ctx->world, int64_t(bytes)), zero(ctx->world, 0), roff(ctx->world);
    for (int k = 0; k < ctx->world; ++k) roff[k] = int64_t(k) * int64_t(bytes);
    return exchange(ctx, send, cnt.data(), zero.data(), recv, cnt.data(), roff.data(), 1, s);
  }
  bool capturable() const override { return false; }  // host barriers order the copies
};

// ---------------------------------------------------------------------------------------
bgs_status check_ctx(bgs_ctx* ctx) {
  if (!ctx) return BGS_ERR_INVALID_ARGUMENT;
  ctx->err.clear();
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return fail(ctx, BGS_ERR_CUDA, "cudaSetDevice", cudaGetErrorString(e));
  return BGS_OK;
}

bgs_status check_stream(bgs_ctx*, void*) { return BGS_OK; }

// NVTX range around every ABI stage (header-only NVTX v3: a no-op unless a tool such as Nsight
// Systems attaches; lets a timeline show the stages of each view / batch)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// View steps run their latency-bound stages (a1-a7, and a11 with BGS_PRIO=2) on a high-priority
// stream of the ctx, so that with views in flight their short kernels are scheduled ahead of the
// large compositing grids of the other views (BGS_PRIO=0: everything on the caller's stream)
int prio_mode() {
  const char* e = getenv("BGS_PRIO");
  return e ? atoi(e) : 1;
}

// a12 at world > 1: the coarse-histogram + all-gather path (two collectives per view) unless
// BGS_IMP=rounds selects the radix-round path (one all-reduce per round)
bool use_imp_rounds() {
  const char* e = getenv("BGS_IMP");
  return e && std::strcmp(e, "rounds") == 0;
}

// a12 at world 1: the cooperative single-launch path when BGS_IMP=coop, else the coarse path
bool use_imp_coop() {
  const char* e = getenv("BGS_IMP");
  return e && std::strcmp(e, "coop") == 0;
}

// a5-a7: the onesweep radix path (sort.cu); BGS_SORT=bucket selects the per-tile bucket sort
// (bucket.cu: bit-identical order, measured no faster -- DESIGN.md §12)
bool use_bucket_sort() {
  const char* e = getenv("BGS_SORT");
  return e && std::strcmp(e, "bucket") == 0;
}

bgs_status set_camera(bgs_ctx* ctx, const bgs_camera* c) {
  if (!c) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "camera is NULL");
  if (c->width <= 0 || c->height <= 0 || !(c->fx > 0) || !(c->fy > 0) || !(c->near_clip > 0))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "camera: width/height/fx/fy/near_clip must be > 0");
  CameraK& k = ctx->cam;
  k.fx = c->fx;
  k.fy = c->fy;
  k.cx = c->cx;
  k.cy = c->cy;
  k.W = c->width;
  k.H = c->height;
  k.TX = (c->width + kTile - 1) / kTile;
  k.TY = (c->height + kTile - 1) / kTile;
  if (k.TX > 255 || k.TY > 255) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "image too large (tiles per axis <= 255)");
  std::memcpy(k.R, c->R, sizeof k.R);
  std::memcpy(k.t, c->t, sizeof k.t);
  std::memcpy(k.campos, c->campos, sizeof k.campos);
  k.near_clip = c->near_clip;
  ctx->T = k.TX * k.TY;
  return BGS_OK;
}

bgs_status check_gaussians(bgs_ctx* ctx, const bgs_gaussians* g) {
  if (!g) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "gaussians is NULL");
  if (g->n_local < 0) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "n_local < 0");
  if (g->n_local > 0 && (!g->mean_opac || !g->quat || !g->scale || !g->sh || !g->lod))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "gaussian plane pointer is NULL");
  if (g->n_local >= (int64_t(1) << 31)) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "n_local >= 2^31");
  return BGS_OK;
}

}  // namespace

// =========================================================================================
// C ABI
// =========================================================================================
extern "C" {

bgs_status bgs_get_unique_id(void* out) {
  if (!out) return BGS_ERR_INVALID_ARGUMENT;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return BGS_ERR_NCCL;
  std::memcpy(out, &id, sizeof id);
  return BGS_OK;
}

static bgs_status ctx_alloc_common(bgs_ctx* c) {
  bgs_ctx* ctx = c;
  CK(cudaSetDevice(c->device));
  CK(cudaMallocHost(&c->h_counters, sizeof(unsigned long long) * C_NCOUNTERS));
  CK(cudaMallocHost(&c->h_misc, sizeof(int64_t) * 64));
  CKS(ensure(c, c->counters, sizeof(unsigned long long) * C_NCOUNTERS));
  return BGS_OK;
}

bgs_status bgs_ctx_create(int32_t rank, int32_t world, const void* uid, int32_t device, bgs_ctx** out) {
  if (!out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world) return BGS_ERR_INVALID_ARGUMENT;
  if (world > 1 && !uid) return BGS_ERR_INVALID_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return BGS_ERR_CUDA;  // no CPU fallback
  auto* c = new bgs_ctx();
  c->rank = rank;
  c->world = world;
  c->device = device;
  bgs_status st = ctx_alloc_common(c);
  if (st != BGS_OK) {
    bgs_ctx_destroy(c);
    return st;
  }
  if (world > 1) {
    auto t = std::make_shared<NcclTransport>();
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    if (ncclCommInitRank(&t->comm, world, id, rank) != ncclSuccess) {
      t->comm = nullptr;
      bgs_ctx_destroy(c);  // frees the pinned buffers and the arena allocated above
      return BGS_ERR_NCCL;
    }
    c->tr = t;
  }
  *out = c;
  return BGS_OK;
}

bgs_status bgs_ctx_create_local_group(int32_t world, int32_t device, bgs_ctx** out) {
  if (!out || world < 1 || world > kMaxWorld) return BGS_ERR_INVALID_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return BGS_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return BGS_ERR_CUDA;
  auto grp = std::make_shared<LocalGroup>(world);
  for (int r = 0; r < world; ++r) {
    auto* c = new bgs_ctx();
    c->rank = r;
    c->world = world;
    c->device = device;
    out[r] = c;
    if (ctx_alloc_common(c) != BGS_OK) {
      for (int k = 0; k <= r; ++k) {  // no partially created group is left behind
        bgs_ctx_destroy(out[k]);
        out[k] = nullptr;
      }
      return BGS_ERR_CUDA;
    }
    if (world > 1) c->tr = std::make_shared<LocalTransport>(grp);
  }
  return BGS_OK;
}

bgs_status bgs_ctx_destroy(bgs_ctx* c) {
  if (!c) return BGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  DevBuf* bufs[] = {&c->counters, &c->recs, &c->rec_lidx, &c->tile_diff, &c->tile_pairs, &c->owner, &c->runinfo,
                    &c->dest_mask, &c->block_counts, &c->totals, &c->send_base, &c->send, &c->recvbuf,
                    &c->keys[0], &c->keys[1], &c->vals[0], &c->vals[1], &c->digit_hist, &c->pass_ctrl, &c->status,
                    &c->ranges, &c->acc, &c->rev, &c->accl, &c->imp_state, &c->imp_hist, &c->imp_total,
                    &c->scr_rgb, &c->scr_t, &c->scr_n, &c->scr_dl, &c->xchg_counts, &c->aux, &c->tile_perm, &c->cand, &c->wbuf, &c->cmask, &c->loss_img, &c->loss_part, &c->loss_sums, &c->scr_tgt, &c->scr_loss, &c->scr_in2, &c->scr_dlsup, &c->bucket_cur, &c->jdir, &c->imp_cand, &c->imp_gath,
                    &c->sel_keys, &c->sel_state, &c->sel_hist, &c->masks, &c->sblocks, &c->new_gid, &c->rows_send,
                    &c->rows_recv, &c->dcnt};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  if (c->h_counters) cudaFreeHost(c->h_counters);
  if (c->h_misc) cudaFreeHost(c->h_misc);
  if (c->ev_counters) cudaEventDestroy(c->ev_counters);
  if (c->ev_geom) cudaEventDestroy(c->ev_geom);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->hi) cudaStreamDestroy(c->hi);
  if (c->ev_hi_fork) cudaEventDestroy(c->ev_hi_fork);
  if (c->ev_hi_join) cudaEventDestroy(c->ev_hi_join);
  for (cudaEvent_t e : c->stage_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {c->ev_in, c->ev_dl, c->ev_fwd, c->ev_out, c->ev_in_free[0], c->ev_in_free[1]})
    if (e) cudaEventDestroy(e);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  destroy_batch(c);
  c->tr.reset();
  delete c;
  return BGS_OK;
}

const char* bgs_last_error(const bgs_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

int64_t bgs_launch_count(const bgs_ctx* c) { return c ? c->launches : -1; }

int64_t bgs_host_sync_count(const bgs_ctx* c) { return c ? c->host_syncs : -1; }

bgs_status bgs_query(bgs_ctx* ctx, int64_t* out) {
  if (!ctx || !out) return BGS_ERR_INVALID_ARGUMENT;
  const int64_t v[BGS_Q_COUNT] = {ctx->n_local, ctx->n_lod, ctx->n_act, ctx->F, ctx->D, ctx->R, ctx->P,
                                  ctx->t_begin, ctx->t_end, ctx->fallback, ctx->n_passes, ctx->P_all,
                                  ctx->cam.W, ctx->cam.H};
  std::memcpy(out, v, sizeof v);
  return BGS_OK;
}

bgs_status bgs_debug_buffer(bgs_ctx* ctx, int32_t which, void** ptr, int64_t* bytes) {
  // test-only accessor: settle all queued work first (the selectors below are read with a
  // synchronous copy on the legacy stream, which does not wait for non-blocking streams)
  if (!ctx || !ptr || !bytes) return BGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  void* p = nullptr;
  int64_t b = 0;
  uint32_t sel = 0;
  if (which == 3 || which == 4) {
    if (ctx->stage < 3) return fail(ctx, BGS_ERR_CONTRACT, "sorted pairs requested before bgs_sort_tiles");
    // final ping-pong buffer selectors live on the device (keys: after the passes; values:
    // after the tie fix-up)
    cudaError_t e = cudaMemcpy(&sel, P_<uint32_t>(ctx->pass_ctrl) + (which == 3 ? kFinalSel : kValsSel), 4,
                               cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(ctx, BGS_ERR_CUDA, "debug_buffer", cudaGetErrorString(e));
  }
  switch (which) {
    case 0: p = ctx->recs.p; b = ctx->F * 48; break;
    case 1: p = ctx->rec_lidx.p; b = ctx->F * 4; break;
    case 2: p = ctx->world > 1 ? ctx->recvbuf.p : nullptr; b = ctx->world > 1 ? ctx->R * 48 : 0; break;
    case 3: p = ctx->keys[sel].p; b = ctx->P * 4; break;
    case 4: p = ctx->vals[sel].p; b = ctx->P * 4; break;
    case 5: p = ctx->ranges.p; b = int64_t(ctx->t_end - ctx->t_begin) * 8; break;
    case 6: p = ctx->acc.p; b = ctx->R * 48; break;
    case 7: p = ctx->acc_local; b = ctx->F * 48; break;
    case 8: p = ctx->owner.p; b = ctx->world > 1 ? int64_t(ctx->T) * 4 : 0; break;
    case 9: p = ctx->dest_mask.p; b = ctx->world > 1 ? ctx->F : 0; break;
    case 10: p = ctx->tile_pairs.p; b = ctx->world > 1 ? int64_t(ctx->T) * 4 : 0; break;
    case 11: p = ctx->counters.p; b = int64_t(C_NCOUNTERS) * 8; break;
    default: return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "unknown debug buffer");
  }
  *ptr = p;
  *bytes = b;
  return BGS_OK;
}

// ---------------------------------------------------------------------------------------
// a1 + a2
// ---------------------------------------------------------------------------------------
// a1 + a2 enqueued; the counters are on their way to the host (project_finish reads them).
static bgs_status project_enqueue(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam,
                                  const bgs_lod_gate* gate, const uint32_t* cull_column, uint32_t flags,
                                  int32_t* radius_out, void* stream) {
  CKS(check_gaussians(ctx, g));
  CKS(set_camera(ctx, cam));
  if (g->n_local > 0 && !radius_out) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "radius_out is NULL");
  cudaStream_t s = as_stream(stream);
  ctx->stage = 0;
  ctx->n_local = g->n_local;
  ProjectArgs a{};
  a.mean_opac = reinterpret_cast<const float4*>(g->mean_opac);
  a.quat = reinterpret_cast<const float4*>(g->quat);
  a.scale = reinterpret_cast<const float4*>(g->scale);
  a.sh = g->sh;
  a.lod = g->lod;
  a.cull = cull_column;
  a.bounds = reinterpret_cast<const float4*>(g->bounds);
  a.n = g->n_local;
  a.cam = ctx->cam;
  a.gate_enabled = 0;
  if (gate && gate->enabled) {
    if (!(gate->d0 > 0)) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "gate d0 must be > 0");
    if (gate->fallback_den <= 0 || gate->fallback_num < 0)
      return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "gate fallback ratio must be num >= 0, den > 0");
    a.gate_enabled = 1;
    a.l_max = gate->l_max;
    a.fb_num = gate->fallback_num;
    a.fb_den = gate->fallback_den;
    // D2[l] = (d0 * 2^(1/2 - l))^2 in double, rounded to float (Eq.4 threshold form, R18)
    for (int l = 0; l < 32; ++l) {
      const double v = gate->d0 * std::ldexp(std::sqrt(2.0), -l);
      a.D2[l] = static_cast<float>(v * v);
    }
  }
  a.no_color = (flags & BGS_NO_COLOR) ? 1 : 0;
  {
    // per-camera constants, float expressions identical to the per-Gaussian ones of the
    // oracle (IEEE binary32 on the host: same bits)
    const volatile float Wf = float(cam->width), Hf = float(cam->height);
    const float tan_fovx = (0.5f * Wf) / cam->fx;
    const float tan_fovy = (0.5f * Hf) / cam->fy;
    a.lim[0] = (Wf - cam->cx) / cam->fx + 0.3f * tan_fovx;
    a.lim[1] = cam->cx / cam->fx + 0.3f * tan_fovx;
    a.lim[2] = (Hf - cam->cy) / cam->fy + 0.3f * tan_fovy;
    a.lim[3] = cam->cy / cam->fy + 0.3f * tan_fovy;
    const double Lx = std::max(a.lim[0], a.lim[1]), Ly = std::max(a.lim[2], a.lim[3]);
    const double K = double(cam->fx) * cam->fx * (1.0 + Lx * Lx) + double(cam->fy) * cam->fy * (1.0 + Ly * Ly);
    a.cull_K = float(K * 1.0001);
  }
  a.rank = ctx->rank;
  a.world = ctx->world;
  a.radius = radius_out;
  CKS(ensure(ctx, ctx->recs, size_t(std::max<int64_t>(g->n_local, 1)) * sizeof(Rec)));
  CKS(ensure(ctx, ctx->rec_lidx, size_t(std::max<int64_t>(g->n_local, 1)) * 4));
  CKS(ensure(ctx, ctx->cand, size_t(std::max<int64_t>(g->n_local, 1)) * 4));
  if (!(flags & BGS_NO_COLOR)) CKS(ensure(ctx, ctx->jdir, size_t(std::max<int64_t>(g->n_local, 1)) * 48));
  a.jdir = P_<float4>(ctx->jdir);
  ctx->colored = !(flags & BGS_NO_COLOR);
  a.recs = P_<Rec>(ctx->recs);
  a.rec_lidx = P_<uint32_t>(ctx->rec_lidx);
  a.cand = P_<uint32_t>(ctx->cand);
  a.rec_cap = g->n_local;
  a.counters = P_<unsigned long long>(ctx->counters);
  CK(cudaMemsetAsync(ctx->counters.p, 0, sizeof(unsigned long long) * C_NCOUNTERS, s));
  a.tile_diff = nullptr;  // per-tile pair counts come from k_tile_count over the records (a3, a5)
  if (a.gate_enabled && a.n > 0) {
    launch_gate_count(a, s);
    CKS(launched(ctx));
  }
  if (a.n > 0) {
    launch_project(a, s);
    CKS(launched(ctx, 2));
  }
  // The counters (F, P_all, ...) are final once the geometry kernels are done: copy them out on a
  // side stream and wait on that copy only, while the colour kernel (next on the working stream,
  // not queued behind the copy) keeps the device busy during the host round trip (the one host
  // synchronisation of a world-1 step).
  if (!ctx->ev_counters) CK(cudaEventCreateWithFlags(&ctx->ev_counters, cudaEventDisableTiming));
  if (!ctx->ev_geom) CK(cudaEventCreateWithFlags(&ctx->ev_geom, cudaEventDisableTiming));
  if (!ctx->side) CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  CK(cudaEventRecord(ctx->ev_geom, s));
  CK(cudaStreamWaitEvent(ctx->side, ctx->ev_geom, 0));
  CK(cudaMemcpyAsync(ctx->h_counters, ctx->counters.p, sizeof(unsigned long long) * C_NCOUNTERS,
                     cudaMemcpyDeviceToHost, ctx->side));
  CK(cudaEventRecord(ctx->ev_counters, ctx->side));
  if (a.n > 0 && !a.no_color) {
    launch_color(a, s);
    CKS(launched(ctx));
  }
  ctx->pend_gate = a.gate_enabled;
  ctx->pend_fb_num = a.fb_num;
  ctx->pend_fb_den = a.fb_den;
  return BGS_OK;
}

// The projection counters, once the host copy of project_enqueue has landed (the caller waited on
// ev_counters): F, |A|, P_all, |L|, the fallback decision and the depth range (sort key layout).
static void project_finish(bgs_ctx* ctx) {
  ctx->F = int64_t(ctx->h_counters[C_F]);
  ctx->n_act = int64_t(ctx->h_counters[C_NACT]);
  ctx->P_all = int64_t(ctx->h_counters[C_PALL]);
  ctx->n_lod = ctx->pend_gate ? int64_t(ctx->h_counters[C_NLOD]) : ctx->n_local;
  ctx->fallback = ctx->pend_gate ? int((unsigned long long)ctx->pend_fb_den * ctx->h_counters[C_NLOD] >
                                       (unsigned long long)ctx->pend_fb_num * (unsigned long long)ctx->n_local)
                                 : 1;
  ctx->stage = 1;
}

bgs_status bgs_project(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam, const bgs_lod_gate* gate,
                       const uint32_t* cull_column, uint32_t flags, int32_t* radius_out, void* stream) {
  NvtxRange nvtx_("bgs_project");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  CKS(project_enqueue(ctx, g, cam, gate, cull_column, flags, radius_out, stream));
  CK(host_sync_event(ctx, ctx->ev_counters));
  project_finish(ctx);
  return BGS_OK;
}

// ---------------------------------------------------------------------------------------
// a3 + a4
// ---------------------------------------------------------------------------------------
bgs_status bgs_route(bgs_ctx* ctx, const int32_t* tile_owner_in, int32_t* tile_owner_out, int64_t* n_recv_out,
                     void* stream) {
  NvtxRange nvtx_("bgs_route");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (ctx->stage < 1) return fail(ctx, BGS_ERR_CONTRACT, "bgs_route before bgs_project");
  cudaStream_t s = as_stream(stream);
  const int M = ctx->world;
  if (M == 1) {
    ctx->recv = P_<Rec>(ctx->recs);
    ctx->R = ctx->F;
    ctx->D = ctx->F;
    ctx->t_begin = 0;
    ctx->t_end = ctx->T;
    ctx->P = ctx->P_all;
    if (tile_owner_out) CK(cudaMemsetAsync(tile_owner_out, 0, size_t(ctx->T) * 4, s));
    if (n_recv_out) *n_recv_out = ctx->R;
    ctx->stage = 2;
    return BGS_OK;
  }
  if (ctx->T > 16384) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "world > 1 supports at most 16384 tiles");
  const int T = ctx->T;
  // a3: per-tile pair counts -> all ranks -> owner map
  CKS(ensure(ctx, ctx->tile_pairs, size_t(T) * 4));
  CKS(ensure(ctx, ctx->owner, size_t(T) * 4));
  CKS(ensure(ctx, ctx->runinfo, 64 + size_t(M + 1) * 8));
  CK(cudaMemsetAsync(ctx->tile_pairs.p, 0, size_t(T) * 4, s));
  if (ctx->F > 0) {
    launch_tile_count(P_<Rec>(ctx->recs), ctx->F, nullptr, ctx->cam.TX, 0, T, P_<int32_t>(ctx->tile_pairs), s);
    CKS(launched(ctx));
  }
  CKS(ctx->tr->allreduce_i32(ctx, P_<int32_t>(ctx->tile_pairs), T, s));
  int32_t* run = P_<int32_t>(ctx->runinfo);
  long long* pown = reinterpret_cast<long long*>(P_<char>(ctx->runinfo) + 64);
  launch_owner_map(P_<int32_t>(ctx->tile_pairs), T, M, P_<int32_t>(ctx->owner), run, pown, tile_owner_in, s);
  CKS(launched(ctx));
  if (tile_owner_out) CK(cudaMemcpyAsync(tile_owner_out, ctx->owner.p, size_t(T) * 4, cudaMemcpyDeviceToDevice, s));
  // a4: destination masks, per-destination counts, count exchange
  const int64_t F = ctx->F;
  const int64_t nb = std::max<int64_t>(1, (F + kRouteBlock - 1) / kRouteBlock);
  CKS(ensure(ctx, ctx->dest_mask, size_t(std::max<int64_t>(F, 1))));
  CKS(ensure(ctx, ctx->block_counts, size_t(nb) * M * 4));
  CKS(ensure(ctx, ctx->totals, size_t(M) * 8));
  CKS(ensure(ctx, ctx->xchg_counts, size_t(M) * 8));
  CKS(ensure(ctx, ctx->send_base, size_t(M) * 8));
  CK(cudaMemsetAsync(ctx->totals.p, 0, size_t(M) * 8, s));
  if (F > 0) {
    launch_dest_count(ctx->recs.p ? P_<Rec>(ctx->recs) : nullptr, F, nullptr, P_<int32_t>(ctx->owner), ctx->cam.TX,
                      M, P_<uint8_t>(ctx->dest_mask), P_<uint32_t>(ctx->block_counts), s);
    CKS(launched(ctx));
    launch_block_scan(P_<uint32_t>(ctx->block_counts), F, nullptr, M, P_<unsigned long long>(ctx->totals), s);
    CKS(launched(ctx));
  }
  CKS(ctx->tr->alltoall1(ctx, P_<int64_t>(ctx->totals), P_<int64_t>(ctx->xchg_counts), s));
  int64_t* h = ctx->h_misc;  // [0,M) send, [M,2M) recv, [2M,4M) run, [4M,5M] pown + bad-map flag
  CK(cudaMemcpyAsync(h, ctx->totals.p, size_t(M) * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(h + M, ctx->xchg_counts.p, size_t(M) * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(h + 2 * M, run, size_t(2 * M) * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(h + 4 * M, pown, size_t(M + 1) * 8, cudaMemcpyDeviceToHost, s));
  CK(host_sync(ctx, s));
  if (h[5 * M]) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "tile_owner_in: not contiguous non-decreasing runs in [0, world)");
  ctx->send_cnt.assign(h, h + M);
  ctx->recv_cnt.assign(h + M, h + 2 * M);
  const int32_t* hrun = reinterpret_cast<const int32_t*>(h + 2 * M);
  ctx->t_begin = hrun[2 * ctx->rank];
  ctx->t_end = hrun[2 * ctx->rank + 1];
  ctx->P = h[4 * M + ctx->rank];
  ctx->send_off.assign(M, 0);
  ctx->recv_off.assign(M, 0);
  int64_t D = 0, R = 0;
  for (int d = 0; d < M; ++d) {
    ctx->send_off[d] = D;
    ctx->recv_off[d] = R;
    D += ctx->send_cnt[d];
    R += ctx->recv_cnt[d];
  }
  ctx->D = D;
  ctx->R = R;
  CKS(ensure(ctx, ctx->send, size_t(std::max<int64_t>(D, 1)) * sizeof(Rec)));
  CKS(ensure(ctx, ctx->recvbuf, size_t(std::max<int64_t>(R, 1)) * sizeof(Rec)));
  CK(cudaMemcpyAsync(ctx->send_base.p, ctx->send_off.data(), size_t(M) * 8, cudaMemcpyHostToDevice, s));
  if (F > 0) {
    launch_pack(P_<Rec>(ctx->recs), F, nullptr, P_<uint8_t>(ctx->dest_mask), P_<uint32_t>(ctx->block_counts), M,
                P_<int64_t>(ctx->send_base), P_<Rec>(ctx->send), s);
    CKS(launched(ctx));
  }
  CKS(ctx->tr->alltoallv(ctx, ctx->send.p, ctx->send_cnt.data(), ctx->send_off.data(), ctx->recvbuf.p,
                         ctx->recv_cnt.data(), ctx->recv_off.data(), sizeof(Rec), s));
  ctx->recv = P_<Rec>(ctx->recvbuf);
  if (n_recv_out) *n_recv_out = R;
  ctx->stage = 2;
  return BGS_OK;
}

// ---------------------------------------------------------------------------------------
// a5 + a6 + a7
// ---------------------------------------------------------------------------------------
bgs_status bgs_sort_tiles(bgs_ctx* ctx, void* stream) {
  NvtxRange nvtx_("bgs_sort_tiles");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (ctx->stage < 2) return fail(ctx, BGS_ERR_CONTRACT, "bgs_sort_tiles before bgs_route");
  cudaStream_t s = as_stream(stream);
  const int64_t P = ctx->P;
  if (P >= (int64_t(1) << 30)) return fail(ctx, BGS_ERR_CAPACITY, "more than 2^30 pairs in one view");
  const int nt = ctx->t_end - ctx->t_begin;
  int tbits = 0;
  while ((1 << tbits) < std::max(nt, 1)) ++tbits;
  // 32-bit key = (local tile << kd) | ((bits(depth) - lo) >> sd) (KeyLayout).  World 1: the
  // records are the received set and their depth range came back with the projection counters,
  // so the pass count is exact.  World > 1: the range of the received records is computed on
  // the device and 4 passes are launched; passes whose digit is constant skip on the device.
  const int kbits = ctx->world == 1 ? std::min(32, tbits + key_layout(ctx->h_counters[C_DLO],
                                                                      ctx->h_counters[C_DHI], tbits).nb)
                                    : 32;
  ctx->n_passes = std::max(1, (kbits + 7) / 8);
  SortArgs a{};
  a.recv = ctx->recv;
  a.n_recv = ctx->R;
  a.TX = ctx->cam.TX;
  a.t_begin = ctx->t_begin;
  a.t_end = ctx->t_end;
  for (int b = 0; b < 2; ++b) {
    CKS(ensure(ctx, ctx->keys[b], size_t(std::max<int64_t>(P, 1)) * 8));
    CKS(ensure(ctx, ctx->vals[b], size_t(std::max<int64_t>(P, 1)) * 4));
    a.keys[b] = P_<unsigned long long>(ctx->keys[b]);
    a.vals[b] = P_<uint32_t>(ctx->vals[b]);
  }
  a.cap = P;
  a.counters = P_<unsigned long long>(ctx->counters);
  CKS(ensure(ctx, ctx->pass_ctrl, 64 * 4));
  CKS(ensure(ctx, ctx->ranges, size_t(std::max(nt, 1)) * 8));
  a.pass_ctrl = P_<uint32_t>(ctx->pass_ctrl);
  a.n_passes = ctx->n_passes;
  a.tbits = tbits;
  a.ranges = P_<uint2>(ctx->ranges);
  CKS(ensure(ctx, ctx->aux, size_t(std::max<int64_t>(ctx->R, 1)) * 16));
  a.aux = P_<float4>(ctx->aux);
  CK(cudaMemsetAsync(ctx->pass_ctrl.p, 0, 64 * 4, s));  // buffer selectors 0: results in keys[0] / vals[0]
  if (use_bucket_sort()) {
    // bucket sizes: world 1 the rects' 2D difference array (bgs_project) prefix-summed; world > 1
    // the all-reduced a3 counts (exactly the pairs this owner receives per owned tile)
    if (ctx->world == 1) {
      if (ctx->T > 16384) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bucket sort supports at most 16384 tiles");
      CKS(ensure(ctx, ctx->tile_pairs, size_t(std::max(ctx->T, 1)) * 4));
      CK(cudaMemsetAsync(ctx->tile_pairs.p, 0, size_t(ctx->T) * 4, s));
      if (ctx->R > 0) {
        launch_tile_count(ctx->recv, ctx->R, nullptr, ctx->cam.TX, 0, ctx->T, P_<int32_t>(ctx->tile_pairs), s);
        CKS(launched(ctx));
      }
    }
    if (ctx->world > 1) {  // depth-bit range of the received records (world 1: from bgs_project)
      CK(cudaMemsetAsync(P_<unsigned long long>(ctx->counters) + C_DLO, 0, 16, s));
      if (ctx->R > 0) {
        launch_depth_range(ctx->recv, ctx->R, P_<unsigned long long>(ctx->counters), s);
        CKS(launched(ctx));
      }
    }
    CKS(ensure(ctx, ctx->bucket_cur, size_t(2 * std::max(nt, 1) + 3) * 4));  // cursors + work list
    CKS(ensure(ctx, ctx->tile_perm, size_t(std::max(nt, 1)) * 4));
    int64_t nl = 0;
    launch_bucket_sort(a, P_<int32_t>(ctx->tile_pairs), P_<uint32_t>(ctx->bucket_cur), P_<uint32_t>(ctx->tile_perm),
                       s, &nl);
    CKS(launched(ctx, int(nl)));
    ctx->n_passes = 0;
  } else {
  CKS(ensure(ctx, ctx->digit_hist, kMaxSortPasses * 256 * 4));
  const int64_t n_parts = std::max<int64_t>(1, (P + kViewSortPart - 1) / kViewSortPart);
  CKS(ensure(ctx, ctx->status, size_t(n_parts) * 256 * 4 * ctx->n_passes));
  a.digit_hist = P_<uint32_t>(ctx->digit_hist);
  a.status = P_<uint32_t>(ctx->status);
  CK(cudaMemsetAsync(ctx->digit_hist.p, 0, kMaxSortPasses * 256 * 4, s));
  CK(cudaMemsetAsync(P_<unsigned long long>(ctx->counters) + C_P, 0, 8, s));
  CK(cudaMemsetAsync(ctx->status.p, 0, size_t(n_parts) * 256 * 4 * ctx->n_passes, s));
  CK(cudaMemsetAsync(ctx->ranges.p, 0, size_t(std::max(nt, 1)) * 8, s));
  if (ctx->world > 1) {
    CK(cudaMemsetAsync(P_<unsigned long long>(ctx->counters) + C_DLO, 0, 16, s));
    if (ctx->R > 0) {
      launch_depth_range(ctx->recv, ctx->R, P_<unsigned long long>(ctx->counters), s);
      CKS(launched(ctx));
    }
  }
  if (ctx->R > 0) {
    launch_emit(a, s);
    CKS(launched(ctx));
  }
  int64_t nl = 0;
  launch_sort_passes(a, P, s, &nl, 4);
  CKS(launched(ctx, int(nl)));
  if (P > 0) {
    launch_ranges_fixup(a, P, s);
    CKS(launched(ctx));
  }
  CKS(ensure(ctx, ctx->tile_perm, size_t(std::max(nt, 1)) * 4));
  launch_tile_order(P_<uint2>(ctx->ranges), nt, P_<uint32_t>(ctx->tile_perm), s);
  CKS(launched(ctx));
  }
  ctx->stage = 3;
  return BGS_OK;
}

static RasterArgs raster_args(bgs_ctx* ctx) {
  RasterArgs a{};
  a.recv = ctx->recv;
  a.ranges = P_<uint2>(ctx->ranges);
  for (int b = 0; b < 2; ++b) {
    a.keys[b] = P_<unsigned long long>(ctx->keys[b]);
    a.vals[b] = P_<uint32_t>(ctx->vals[b]);
  }
  a.pass_ctrl = P_<uint32_t>(ctx->pass_ctrl);
  a.t_begin = ctx->t_begin;
  a.n_tiles = ctx->t_end - ctx->t_begin;
  a.TX = ctx->cam.TX;
  a.W = ctx->cam.W;
  a.H = ctx->cam.H;
  a.acc = P_<Acc>(ctx->acc);
  a.aux = P_<float4>(ctx->aux);
  a.tile_perm = P_<uint32_t>(ctx->tile_perm);
  a.cmask = P_<uint32_t>(ctx->cmask);
  a.no_color = ctx->colored ? 0 : 1;
  return a;
}

bgs_status bgs_raster_fwd(bgs_ctx* ctx, uint32_t flags, float* rgb, float* t_final, int32_t* n_contrib,
                          void* stream) {
  NvtxRange nvtx_("bgs_raster_fwd");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (ctx->stage < 3) return fail(ctx, BGS_ERR_CONTRACT, "bgs_raster_fwd before bgs_sort_tiles");
  if (!rgb || !t_final || !n_contrib) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "output image pointer is NULL");
  cudaStream_t s = as_stream(stream);
  CKS(ensure(ctx, ctx->acc, size_t(std::max<int64_t>(ctx->R, 1)) * sizeof(Acc)));
  CK(cudaMemsetAsync(ctx->acc.p, 0, size_t(std::max<int64_t>(ctx->R, 1)) * sizeof(Acc), s));
  // contributor masks: one word per (warp block, 32-entry chunk of its tile's list), chunk index
  // floor(range.x / 32) + lt + c is injective over (lt, c) (raster.cu), 8 warp blocks per tile
  CKS(ensure(ctx, ctx->cmask, size_t(kRasterSlots) * size_t(ctx->P / 32 + (ctx->t_end - ctx->t_begin) + 2) * 4));
  RasterArgs a = raster_args(ctx);
  if (a.n_tiles > 0) {
    ctx->raster_split = launch_raster_fwd(a, flags, rgb, t_final, n_contrib, s);
    CKS(launched(ctx));
  }
  ctx->stage = 4;
  return BGS_OK;
}

bgs_status bgs_raster_bwd(bgs_ctx* ctx, const float* dL, const float* t_final, const int32_t* n_contrib,
                          void* stream) {
  NvtxRange nvtx_("bgs_raster_bwd");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (ctx->stage < 4) return fail(ctx, BGS_ERR_CONTRACT, "bgs_raster_bwd before bgs_raster_fwd");
  if (!dL || !t_final || !n_contrib) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "image pointer is NULL");
  cudaStream_t s = as_stream(stream);
  RasterArgs a = raster_args(ctx);
  a.n_split = ctx->raster_split;
  if (a.n_tiles > 0) {
    launch_raster_bwd(a, dL, t_final, n_contrib, s);
    CKS(launched(ctx));
  }
  ctx->stage = 5;
  return BGS_OK;
}

bgs_status bgs_route_reverse(bgs_ctx* ctx, uint32_t flags, void* stream) {
  NvtxRange nvtx_("bgs_route_reverse");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (ctx->stage < 4) return fail(ctx, BGS_ERR_CONTRACT, "bgs_route_reverse before bgs_raster_fwd");
  cudaStream_t s = as_stream(stream);
  const int M = ctx->world;
  if (M == 1) {
    ctx->acc_local = P_<Acc>(ctx->acc);
    ctx->stage = 6;
    return BGS_OK;
  }
  if (flags & BGS_IMPORTANCE_ONLY) {  // 12-B (w, a) units instead of the 48-B accumulators
    CKS(ensure(ctx, ctx->rev, size_t(std::max<int64_t>(std::max(ctx->D, ctx->R), 1)) * sizeof(Acc)));
    CKS(ensure(ctx, ctx->accl, size_t(std::max<int64_t>(ctx->F, 1)) * sizeof(Acc)));
    // pack the received records' (w, a) into the tail of rev (R x 12 B fits behind D x 12 B: rev
    // holds max(D, R) 48-B units)
    char* packed = P_<char>(ctx->rev) + size_t(std::max<int64_t>(ctx->D, 1)) * 12;
    launch_pack_imp(P_<Acc>(ctx->acc), ctx->R, packed, s);
    CKS(launched(ctx));
    CKS(ctx->tr->alltoallv(ctx, packed, ctx->recv_cnt.data(), ctx->recv_off.data(), ctx->rev.p,
                           ctx->send_cnt.data(), ctx->send_off.data(), 12, s));
    if (ctx->F > 0) {
      launch_gather_imp(ctx->rev.p, ctx->F, P_<uint8_t>(ctx->dest_mask), P_<uint32_t>(ctx->block_counts), M,
                        P_<int64_t>(ctx->send_base), P_<Acc>(ctx->accl), s);
      CKS(launched(ctx));
    }
    ctx->acc_local = P_<Acc>(ctx->accl);
    ctx->stage = 6;
    return BGS_OK;
  }
  CKS(ensure(ctx, ctx->rev, size_t(std::max<int64_t>(ctx->D, 1)) * sizeof(Acc)));
  CKS(ensure(ctx, ctx->accl, size_t(std::max<int64_t>(ctx->F, 1)) * sizeof(Acc)));
  // transposed counts: what I received from k goes back to k; what I sent to d comes back from d
  CKS(ctx->tr->alltoallv(ctx, ctx->acc.p, ctx->recv_cnt.data(), ctx->recv_off.data(), ctx->rev.p,
                         ctx->send_cnt.data(), ctx->send_off.data(), sizeof(Acc), s));
  if (ctx->F > 0) {
    launch_gather_sum(P_<Acc>(ctx->rev), ctx->F, nullptr, P_<uint8_t>(ctx->dest_mask),
                      P_<uint32_t>(ctx->block_counts), M, P_<int64_t>(ctx->send_base), P_<Acc>(ctx->accl), s);
    CKS(launched(ctx));
  }
  ctx->acc_local = P_<Acc>(ctx->accl);
  ctx->stage = 6;
  return BGS_OK;
}

bgs_status bgs_project_bwd(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam,
                           const bgs_gaussian_grads* grads, void* stream) {
  NvtxRange nvtx_("bgs_project_bwd");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  CKS(check_gaussians(ctx, g));
  if (ctx->stage < 6) return fail(ctx, BGS_ERR_CONTRACT, "bgs_project_bwd before bgs_route_reverse");
  if (g->n_local != ctx->n_local) return fail(ctx, BGS_ERR_CONTRACT, "n_local differs from bgs_project's");
  if (!ctx->colored) return fail(ctx, BGS_ERR_CONTRACT, "bgs_project_bwd after a BGS_NO_COLOR projection");
  if (!grads || !grads->mean_opac || !grads->quat || !grads->scale || !grads->sh)
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "gradient pointer is NULL");
  if (!cam) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "camera is NULL");
  cudaStream_t s = as_stream(stream);
  ProjectBwdArgs a{};
  a.mean_opac = reinterpret_cast<const float4*>(g->mean_opac);
  a.quat = reinterpret_cast<const float4*>(g->quat);
  a.scale = reinterpret_cast<const float4*>(g->scale);
  a.sh = g->sh;
  a.rec_lidx = P_<uint32_t>(ctx->rec_lidx);
  a.acc = ctx->acc_local;
  a.jdir = P_<float4>(ctx->jdir);
  a.F = ctx->F;
  a.cam = ctx->cam;
  a.g_mean_opac = reinterpret_cast<float4*>(grads->mean_opac);
  a.g_quat = reinterpret_cast<float4*>(grads->quat);
  a.g_scale = reinterpret_cast<float4*>(grads->scale);
  a.g_sh = grads->sh;
  if (a.F > 0) {
    launch_project_bwd(a, s);
    CKS(launched(ctx));
  }
  return BGS_OK;
}

bgs_status bgs_importance(bgs_ctx* ctx, int64_t n_local, const int32_t* radius, const uint64_t* w_fixed,
                          const uint32_t* a_in, int32_t mass_num, int32_t mass_den, double* s_out, uint32_t* c_rad,
                          uint32_t* c_vis, uint32_t* cull_out, void* stream) {
  NvtxRange nvtx_("bgs_importance");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (n_local < 0 || !s_out || !c_rad || !c_vis || !cull_out)
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "importance outputs must be non-NULL");
  if (mass_den <= 0 || mass_num < 0 || mass_num > mass_den)
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "mass fraction must satisfy 0 <= num <= den, den > 0");
  const bool dense = w_fixed != nullptr;
  if (dense && (!a_in || !radius)) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "dense w_fixed needs a and radius");
  if (!dense && ctx->stage < 6) return fail(ctx, BGS_ERR_CONTRACT, "bgs_importance before bgs_route_reverse");
  if (!dense && n_local != ctx->n_local) return fail(ctx, BGS_ERR_CONTRACT, "stale n_local (S:384)");
  cudaStream_t s = as_stream(stream);
  ImportanceArgs a{};
  a.n_items = dense ? n_local : ctx->F;
  a.item_lidx = dense ? nullptr : P_<uint32_t>(ctx->rec_lidx);
  a.radius = radius;
  a.w_dense = reinterpret_cast<const unsigned long long*>(w_fixed);
  a.a_dense = a_in;
  a.acc = ctx->acc_local;
  a.n_local = n_local;
  a.rank = ctx->rank;
  a.world = ctx->world;
  a.s = s_out;
  a.c_rad = c_rad;
  a.c_vis = c_vis;
  a.cull = cull_out;
  CKS(ensure(ctx, ctx->wbuf, size_t(std::max<int64_t>(a.n_items, 1)) * 8));
  a.wbuf = P_<unsigned long long>(ctx->wbuf);
  const int WR = imp_w_rounds(), GR = imp_g_rounds();
  CKS(ensure(ctx, ctx->imp_state, kImpStateBytes));
  ImpState* st = static_cast<ImpState*>(ctx->imp_state.p);
  if (ctx->world == 1 && !use_imp_coop()) {
    // world 1: the coarse-histogram path without collectives or host reads -- every item with w > 0
    // in the crossing bin is gathered into a buffer of capacity n_items (an upper bound), then the
    // same exact single-CTA selection; five short kernels instead of a cooperative grid that holds
    // its SMs at grid barriers while other views are in flight
    const int64_t HW = imp_coarse_words();
    CKS(ensure(ctx, ctx->imp_hist, size_t(HW) * 8));
    CK(cudaMemsetAsync(ctx->imp_hist.p, 0, size_t(HW) * 8, s));
    const int64_t words = 2 + 2 * std::max<int64_t>(a.n_items, 1);
    CKS(ensure(ctx, ctx->imp_cand, size_t(words) * 8));
    CK(cudaMemsetAsync(ctx->imp_cand.p, 0, 16, s));
    unsigned long long* hist = P_<unsigned long long>(ctx->imp_hist);
    launch_fill_bits(cull_out, n_local, s);
    launch_imp_stats_coarse(a, hist, s);
    launch_imp_coarse_decide(st, hist, mass_num, mass_den, s);
    launch_imp_gather_cand(a, st, P_<unsigned long long>(ctx->imp_cand), s);
    launch_imp_select_cand(st, P_<unsigned long long>(ctx->imp_cand), 1, words, mass_num, mass_den, s);
    launch_imp_mark(a, st, s);
    return launched(ctx, 6);
  }
  if (ctx->world == 1) {
    // one cooperative launch; its histogram sets alternate between calls and each call zeroes
    // the other one, so only a freshly allocated pair is cleared here
    const size_t set_bytes = size_t(imp_set_words()) * 8;
    const bool fresh = ctx->imp_hist.cap < 2 * set_bytes;
    CKS(ensure(ctx, ctx->imp_hist, 2 * set_bytes));
    if (fresh) CK(cudaMemsetAsync(ctx->imp_hist.p, 0, 2 * set_bytes, s));
    CKS(ensure(ctx, ctx->cand, size_t(imp_cand_words(a.n_items)) * 4));
    unsigned long long* sets = P_<unsigned long long>(ctx->imp_hist);
    unsigned long long* cur = sets + (ctx->imp_parity ? imp_set_words() : 0);
    unsigned long long* nxt = sets + (ctx->imp_parity ? 0 : imp_set_words());
    ctx->imp_parity ^= 1;
    CK(launch_imp_coop(a, st, cur, nxt, P_<uint32_t>(ctx->cand), mass_num, mass_den, s));
    return launched(ctx, 1);
  }
  if (!use_imp_rounds()) {
    // two collectives per view (importance.cu): coarse histogram all-reduce, one host read of the
    // crossing bin's global count, candidate all-gather, exact select on every rank
    const int64_t HW = imp_coarse_words();
    CKS(ensure(ctx, ctx->imp_hist, size_t(HW) * 8));
    CK(cudaMemsetAsync(ctx->imp_hist.p, 0, size_t(HW) * 8, s));
    unsigned long long* hist = P_<unsigned long long>(ctx->imp_hist);
    launch_fill_bits(cull_out, n_local, s);
    launch_imp_stats_coarse(a, hist, s);
    CKS(launched(ctx, 2));
    CKS(ctx->tr->allreduce_u64(ctx, hist, HW, s));
    launch_imp_coarse_decide(st, hist, mass_num, mass_den, s);
    CKS(launched(ctx));
    CK(cudaMemcpyAsync(ctx->h_misc + 62, P_<char>(ctx->imp_state) + imp_state_ncand_offset(), 8,
                       cudaMemcpyDeviceToHost, s));
    CK(host_sync(ctx, s));
    const int64_t ncand = ctx->h_misc[62];
    if (ncand > 0) {
      const int64_t words = 2 + 2 * ncand;  // [count, pad, (w, gid) x cap]; cap = global count
      CKS(ensure(ctx, ctx->imp_cand, size_t(words) * 8));
      CKS(ensure(ctx, ctx->imp_gath, size_t(words) * 8 * ctx->world));
      // the whole block is all-gathered (fixed size); slots past this rank's count are zero
      CK(cudaMemsetAsync(ctx->imp_cand.p, 0, size_t(words) * 8, s));
      launch_imp_gather_cand(a, st, P_<unsigned long long>(ctx->imp_cand), s);
      CKS(launched(ctx));
      CKS(ctx->tr->allgather(ctx, ctx->imp_cand.p, ctx->imp_gath.p, size_t(words) * 8, s));
      launch_imp_select_cand(st, P_<unsigned long long>(ctx->imp_gath), ctx->world, words, mass_num, mass_den, s);
      CKS(launched(ctx));
    }
    launch_imp_mark(a, st, s);
    return launched(ctx);
  }
  CKS(ensure(ctx, ctx->imp_total, 65 * 8));  // total + 64-bin MSB histogram
  CKS(ensure(ctx, ctx->imp_hist, size_t(WR * 512 + GR * 256) * 8));
  CK(cudaMemsetAsync(ctx->imp_state.p, 0, kImpStateBytes, s));
  CK(cudaMemsetAsync(ctx->imp_total.p, 0, 65 * 8, s));
  CK(cudaMemsetAsync(ctx->imp_hist.p, 0, size_t(WR * 512 + GR * 256) * 8, s));
  unsigned long long* total = P_<unsigned long long>(ctx->imp_total);
  unsigned long long* hist = P_<unsigned long long>(ctx->imp_hist);
  int nl = 0;
  launch_fill_bits(cull_out, n_local, s);
  ++nl;
  launch_imp_stats(a, total, s);
  ++nl;
  if (ctx->world > 1) CKS(ctx->tr->allreduce_u64(ctx, total, 65, s));
  for (int r = 0; r < WR; ++r) {
    launch_imp_hist(a, st, r, hist + r * 512, s);
    if (ctx->world > 1) CKS(ctx->tr->allreduce_u64(ctx, hist + r * 512, 512, s));
    launch_imp_decide(st, total, r, hist + r * 512, mass_num, mass_den, s);
    nl += 2;
  }
  for (int r = 0; r < GR; ++r) {
    launch_imp_gid_hist(a, st, r, hist + WR * 512 + r * 256, s);
    if (ctx->world > 1) CKS(ctx->tr->allreduce_u64(ctx, hist + WR * 512 + r * 256, 256, s));
    launch_imp_gid_decide(st, r, hist + WR * 512 + r * 256, s);
    nl += 2;
  }
  launch_imp_mark(a, st, s);
  ++nl;
  CKS(launched(ctx, nl));
  return BGS_OK;
}

bgs_status bgs_shard_bounds(bgs_ctx* ctx, const bgs_gaussians* g, float* bounds_out, void* stream) {
  CKS(check_ctx(ctx));
  CKS(check_gaussians(ctx, g));
  if (g->n_local > 0 && !bounds_out) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bounds_out is NULL");
  launch_shard_bounds(reinterpret_cast<const float4*>(g->mean_opac), reinterpret_cast<const float4*>(g->scale),
                      g->n_local, reinterpret_cast<float4*>(bounds_out), as_stream(stream));
  return g->n_local > 0 ? launched(ctx) : BGS_OK;
}

bgs_status bgs_spatial_order(bgs_ctx* ctx, const float* mean_opac, int64_t n, uint32_t* perm_out, void* stream) {
  CKS(check_ctx(ctx));
  if (n < 0 || (n > 0 && (!mean_opac || !perm_out))) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "spatial_order args");
  if (n >= (int64_t(1) << 30)) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "spatial_order: n >= 2^30");
  if (n == 0) return BGS_OK;
  cudaStream_t s = as_stream(stream);
  ctx->stage = 0;  // reuses the sort scratch: the current view's intermediates are gone
  SortArgs a{};
  for (int b = 0; b < 2; ++b) {
    CKS(ensure(ctx, ctx->keys[b], size_t(n) * 8));
    CKS(ensure(ctx, ctx->vals[b], size_t(n) * 4));
    a.keys[b] = P_<unsigned long long>(ctx->keys[b]);
    a.vals[b] = P_<uint32_t>(ctx->vals[b]);
  }
  a.cap = n;
  a.n_passes = 6;  // 48-bit codes
  const int64_t n_parts = (n + kSortPart - 1) / kSortPart;
  CKS(ensure(ctx, ctx->digit_hist, kMaxSortPasses * 256 * 4));
  CKS(ensure(ctx, ctx->pass_ctrl, 64 * 4));
  CKS(ensure(ctx, ctx->status, size_t(n_parts) * 256 * 4 * a.n_passes));
  CKS(ensure(ctx, ctx->tile_diff, 64));  // bounding-box scratch
  a.counters = P_<unsigned long long>(ctx->counters);
  a.digit_hist = P_<uint32_t>(ctx->digit_hist);
  a.pass_ctrl = P_<uint32_t>(ctx->pass_ctrl);
  a.status = P_<uint32_t>(ctx->status);
  CK(cudaMemsetAsync(ctx->digit_hist.p, 0, kMaxSortPasses * 256 * 4, s));
  CK(cudaMemsetAsync(ctx->pass_ctrl.p, 0, 64 * 4, s));
  CK(cudaMemsetAsync(ctx->status.p, 0, size_t(n_parts) * 256 * 4 * a.n_passes, s));
  CK(cudaMemsetAsync(ctx->tile_diff.p, 0xff, 12, s));                       // min (ordered ints)
  CK(cudaMemsetAsync(P_<char>(ctx->tile_diff) + 12, 0, 12, s));             // max
  ctx->h_misc[63] = n;
  CK(cudaMemcpyAsync(P_<unsigned long long>(ctx->counters) + C_P, ctx->h_misc + 63, 8, cudaMemcpyHostToDevice, s));
  int64_t nl = 0;
  launch_spatial_order(reinterpret_cast<const float4*>(mean_opac), n, P_<unsigned int>(ctx->tile_diff), a, perm_out,
                       s, &nl);
  CKS(launched(ctx, int(nl)));
  CK(host_sync(ctx, s));  // h_misc is reused
  return BGS_OK;
}

// dl_ready: event the compositing backward waits for (dL/dC still arriving); fwd_done: event
// recorded once the image is final (the host path copies it out while the backward runs)
// the host-buffer steps' copy streams and events (created on first use)
static bgs_status copy_streams(bgs_ctx* ctx) {
  if (!ctx->h2d) {
    CK(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&ctx->ev_in, &ctx->ev_dl, &ctx->ev_fwd, &ctx->ev_out, &ctx->ev_in_free[0], &ctx->ev_in_free[1]})
      CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  return BGS_OK;
}

static bgs_status view_step_impl(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam,
                                 const bgs_lod_gate* gate, const uint32_t* cull_column, uint32_t flags,
                                 int32_t* radius_out, float* rgb, float* t_final, int32_t* n_contrib, const float* dL,
                                 const bgs_gaussian_grads* grads, const bgs_importance_out* imp, void* stream,
                                 cudaEvent_t dl_ready, cudaEvent_t fwd_done, const bgs_supervision* sup = nullptr,
                                 float* dL_sup = nullptr, cudaEvent_t loss_done = nullptr) {
  if (imp) flags |= BGS_IMPORTANCE;
  cudaStream_t s = as_stream(stream);
  // stage boundaries (bgs_stage_times): events on the working stream, recorded only when enabled
  auto mark = [&](int k) -> bgs_status {
    if (ctx->stage_timing) CK(cudaEventRecord(ctx->stage_ev[k], s));
    return BGS_OK;
  };
  if (ctx->stage_timing && !ctx->stage_ev[0])
    for (auto& e : ctx->stage_ev) CK(cudaEventCreate(&e));
  // latency-bound stages on the high-priority stream (not while stage events time the step)
  const int pm = ctx->stage_timing ? 0 : prio_mode();
  void* hs = stream;
  if (pm > 0) {
    if (!ctx->hi) {
      int least = 0, greatest = 0;
      CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      CK(cudaStreamCreateWithPriority(&ctx->hi, cudaStreamNonBlocking, greatest));
      CK(cudaEventCreateWithFlags(&ctx->ev_hi_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_hi_join, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ctx->ev_hi_fork, s));
    CK(cudaStreamWaitEvent(ctx->hi, ctx->ev_hi_fork, 0));
    hs = ctx->hi;
  }
  CKS(mark(0));
  CKS(bgs_project(ctx, g, cam, gate, cull_column, flags, radius_out, hs));
  CKS(mark(1));
  CKS(bgs_route(ctx, nullptr, nullptr, nullptr, hs));
  CKS(mark(2));
  CKS(bgs_sort_tiles(ctx, hs));
  if (pm > 0) {
    CK(cudaEventRecord(ctx->ev_hi_join, ctx->hi));
    CK(cudaStreamWaitEvent(s, ctx->ev_hi_join, 0));
  }
  CKS(mark(3));
  CKS(bgs_raster_fwd(ctx, flags, rgb, t_final, n_contrib, stream));
  if (fwd_done) CK(cudaEventRecord(fwd_done, s));
  CKS(mark(4));
  if (dl_ready) CK(cudaStreamWaitEvent(s, dl_ready, 0));  // dL/dC (or the target image) uploaded
  if (sup) {
    // NEXT-4: Eq.7 on the owned tiles gives this view's dL/dC; Eq.8 adds to the scale gradient
    CKS(bgs_loss_photo(ctx, rgb, sup->target, sup->lambda, sup->batch_inv, dL_sup, sup->loss_out, stream));
    if (sup->beta != 0.f)
      CKS(bgs_loss_scale(ctx, g, sup->beta, grads, sup->loss_out + 3, stream));
    else
      CK(cudaMemsetAsync(sup->loss_out + 3, 0, 2 * sizeof(double), s));  // {L_scale, |V|} = 0: not computed
    if (loss_done) CK(cudaEventRecord(loss_done, s));
    dL = dL_sup;
  }
  CKS(mark(5));
  if (dL) CKS(bgs_raster_bwd(ctx, dL, t_final, n_contrib, stream));
  CKS(mark(6));
  // no backward in this step (scoring sweep): only (w, a) travel back, 12 B per record
  CKS(bgs_route_reverse(ctx, dL ? 0u : uint32_t(BGS_IMPORTANCE_ONLY), stream));
  CKS(mark(7));
  if (dL && grads) {
    if (pm > 1) {
      CK(cudaEventRecord(ctx->ev_hi_fork, s));
      CK(cudaStreamWaitEvent(ctx->hi, ctx->ev_hi_fork, 0));
      CKS(bgs_project_bwd(ctx, g, cam, grads, ctx->hi));
      CK(cudaEventRecord(ctx->ev_hi_join, ctx->hi));
      CK(cudaStreamWaitEvent(s, ctx->ev_hi_join, 0));
    } else {
      CKS(bgs_project_bwd(ctx, g, cam, grads, stream));
    }
  }
  CKS(mark(8));
  if (imp)
    CKS(bgs_importance(ctx, g->n_local, radius_out, nullptr, nullptr, imp->mass_num, imp->mass_den, imp->s,
                       imp->c_rad, imp->c_vis, imp->cull_out, stream));
  CKS(mark(9));
  ctx->stage_recorded = ctx->stage_timing;
  return BGS_OK;
}

bgs_status bgs_view_step(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam, const bgs_lod_gate* gate,
                         const uint32_t* cull_column, uint32_t flags, int32_t* radius_out, float* rgb,
                         float* t_final, int32_t* n_contrib, const float* dL, const bgs_gaussian_grads* grads,
                         const bgs_importance_out* imp, void* stream) {
  NvtxRange nvtx_("bgs_view_step");
  return view_step_impl(ctx, g, cam, gate, cull_column, flags, radius_out, rgb, t_final, n_contrib, dL, grads, imp,
                        stream, nullptr, nullptr);
}

static bgs_status check_sup(bgs_ctx* ctx, const bgs_supervision* sup, bool need_target) {
  if (!sup) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "supervision is NULL");
  if ((need_target && !sup->target) || !sup->loss_out)
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "supervision target / loss_out is NULL");
  return BGS_OK;
}

bgs_status bgs_train_view_step(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam, const bgs_lod_gate* gate,
                               const uint32_t* cull_column, uint32_t flags, int32_t* radius_out,
                               const bgs_supervision* sup, float* rgb, float* t_final, int32_t* n_contrib,
                               float* dL_scratch, const bgs_gaussian_grads* grads, const bgs_importance_out* imp,
                               void* stream) {
  NvtxRange nvtx_("bgs_train_view_step");
  CKS(check_ctx(ctx));
  CKS(check_sup(ctx, sup, true));
  if (!dL_scratch) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "dL_scratch is NULL");
  return view_step_impl(ctx, g, cam, gate, cull_column, flags, radius_out, rgb, t_final, n_contrib, nullptr, grads,
                        imp, stream, nullptr, nullptr, sup, dL_scratch, nullptr);
}

bgs_status bgs_train_view_step_host_async(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam,
                                          const bgs_lod_gate* gate, const uint32_t* cull_column, uint32_t flags,
                                          int32_t* radius_out, const float* target_host, float lambda,
                                          float batch_inv, float beta, double* loss_host,
                                          const bgs_gaussian_grads* grads, const bgs_importance_out* imp,
                                          void* stream) {
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  CKS(set_camera(ctx, cam));
  if (!target_host || !loss_host) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "host target / loss pointer is NULL");
  cudaStream_t s = as_stream(stream);
  const size_t npix = size_t(ctx->cam.W) * ctx->cam.H;
  CKS(ensure(ctx, ctx->scr_rgb, npix * 12));
  CKS(ensure(ctx, ctx->scr_dlsup, npix * 12));
  CKS(ensure(ctx, ctx->scr_tgt, npix * 12));
  CKS(ensure(ctx, ctx->scr_t, npix * 4));
  CKS(ensure(ctx, ctx->scr_n, npix * 4));
  CKS(ensure(ctx, ctx->scr_loss, 8 * sizeof(double)));
  CKS(ensure(ctx, ctx->scr_in2, npix * 12));
  CKS(copy_streams(ctx));
  // target upload on its own copy engine into the buffer this ctx's view before last used (needed
  // only by the loss, after the forward); the loss download starts as soon as the loss is final,
  // overlapping the backward
  const int b = ctx->in_parity;
  ctx->in_parity ^= 1;
  float* tgt = P_<float>(b ? ctx->scr_in2 : ctx->scr_tgt);
  CK(cudaStreamWaitEvent(ctx->h2d, ctx->ev_in_free[b], 0));
  CK(cudaMemcpyAsync(tgt, target_host, npix * 12, cudaMemcpyHostToDevice, ctx->h2d));
  CK(cudaEventRecord(ctx->ev_dl, ctx->h2d));
  bgs_supervision sup{tgt, lambda, batch_inv, beta, P_<double>(ctx->scr_loss)};
  CKS(view_step_impl(ctx, g, cam, gate, cull_column, flags, radius_out, P_<float>(ctx->scr_rgb),
                     P_<float>(ctx->scr_t), P_<int32_t>(ctx->scr_n), nullptr, grads, imp, stream, ctx->ev_dl,
                     nullptr, &sup, P_<float>(ctx->scr_dlsup), ctx->ev_fwd));
  CK(cudaEventRecord(ctx->ev_in_free[b], s));
  CK(cudaStreamWaitEvent(ctx->d2h, ctx->ev_fwd, 0));
  CK(cudaMemcpyAsync(loss_host, ctx->scr_loss.p, 5 * sizeof(double), cudaMemcpyDeviceToHost, ctx->d2h));
  CK(cudaEventRecord(ctx->ev_out, ctx->d2h));
  CK(cudaStreamWaitEvent(s, ctx->ev_out, 0));
  return BGS_OK;
}

bgs_status bgs_set_stage_timing(bgs_ctx* ctx, int32_t enable) {
  CKS(check_ctx(ctx));
  ctx->stage_timing = enable != 0;
  ctx->stage_recorded = false;
  return BGS_OK;
}

bgs_status bgs_stage_times(bgs_ctx* ctx, float* ms_out) {
  CKS(check_ctx(ctx));
  if (!ms_out) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bgs_stage_times: ms_out is NULL");
  if (!ctx->stage_recorded) return fail(ctx, BGS_ERR_CONTRACT, "no bgs_view_step with stage timing enabled");
  CK(host_sync_event(ctx, ctx->stage_ev[kStages]));
  for (int k = 0; k < kStages; ++k) CK(cudaEventElapsedTime(ms_out + k, ctx->stage_ev[k], ctx->stage_ev[k + 1]));
  return BGS_OK;
}

bgs_status bgs_view_step_host_async(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam,
                                    const bgs_lod_gate* gate, const uint32_t* cull_column, uint32_t flags,
                                    int32_t* radius_out, const float* dL_host, float* rgb_host,
                                    const bgs_gaussian_grads* grads, const bgs_importance_out* imp, void* stream) {
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  CKS(set_camera(ctx, cam));
  if (!dL_host || !rgb_host) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "host image pointer is NULL");
  cudaStream_t s = as_stream(stream);
  const size_t npix = size_t(ctx->cam.W) * ctx->cam.H;
  CKS(ensure(ctx, ctx->scr_rgb, npix * 12));
  CKS(ensure(ctx, ctx->scr_dl, npix * 12));
  CKS(ensure(ctx, ctx->scr_t, npix * 4));
  CKS(ensure(ctx, ctx->scr_n, npix * 4));
  CKS(ensure(ctx, ctx->scr_in2, npix * 12));
  CKS(copy_streams(ctx));
  // dL/dC upload on its own copy engine, needed only by the compositing backward, into the buffer
  // this ctx's view before last read (two alternating buffers): it overlaps the previous view
  const int b = ctx->in_parity;
  ctx->in_parity ^= 1;
  float* dl = P_<float>(b ? ctx->scr_in2 : ctx->scr_dl);
  CK(cudaStreamWaitEvent(ctx->h2d, ctx->ev_in_free[b], 0));
  CK(cudaMemcpyAsync(dl, dL_host, npix * 12, cudaMemcpyHostToDevice, ctx->h2d));
  CK(cudaEventRecord(ctx->ev_dl, ctx->h2d));
  CKS(view_step_impl(ctx, g, cam, gate, cull_column, flags, radius_out, P_<float>(ctx->scr_rgb),
                     P_<float>(ctx->scr_t), P_<int32_t>(ctx->scr_n), dl, grads, imp, stream,
                     ctx->ev_dl, ctx->ev_fwd));
  CK(cudaEventRecord(ctx->ev_in_free[b], s));
  // the image is final after the forward: download it while the backward runs; the working
  // stream then waits for the download, so a sync of `stream` covers rgb_host
  CK(cudaStreamWaitEvent(ctx->d2h, ctx->ev_fwd, 0));
  CK(cudaMemcpyAsync(rgb_host, ctx->scr_rgb.p, npix * 12, cudaMemcpyDeviceToHost, ctx->d2h));
  CK(cudaEventRecord(ctx->ev_out, ctx->d2h));
  CK(cudaStreamWaitEvent(s, ctx->ev_out, 0));
  return BGS_OK;
}

bgs_status bgs_view_step_host(bgs_ctx* ctx, const bgs_gaussians* g, const bgs_camera* cam,
                              const bgs_lod_gate* gate, const uint32_t* cull_column, uint32_t flags,
                              int32_t* radius_out, const float* dL_host, float* rgb_host,
                              const bgs_gaussian_grads* grads, const bgs_importance_out* imp, void* stream) {
  CKS(bgs_view_step_host_async(ctx, g, cam, gate, cull_column, flags, radius_out, dL_host, rgb_host, grads, imp,
                               stream));
  CK(host_sync(ctx, as_stream(stream)));
  return BGS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// NEXT-2: the batched step.  B views of one training batch ("a
// mini-batch of B cameras") in ONE call: each view runs on an internal view slot (its own arena
// and stream, like a ctx per view in flight), the host reads sizes ONCE per batch (the projection
// counters and, at world > 1, the exchanged counts), and at world > 1 the batch makes one tile-cost
// all-reduce, one count exchange, ONE record all-to-all and ONE reverse all-to-all ("the
// batch's records concatenated into one exchange") instead of four collectives per view.
// BGS_GRAPH: everything after the host read is recorded as one CUDA graph (re-captured per batch,
// the executable updated in place) and launched with one call.
// ---------------------------------------------------------------------------------------
namespace {

constexpr int kMaxBatch = 16;

struct BatchState {
  std::vector<bgs_ctx*> slots;
  std::vector<cudaStream_t> streams, gstreams;  // per slot: eager work / graph-capture work
  std::vector<cudaEvent_t> done, gdone;
  cudaEvent_t fork = nullptr, gfork = nullptr;
  cudaStream_t cap = nullptr;                    // capture origin
  cudaGraphExec_t exec = nullptr;
  DevBuf pairs, tot_send, tot_recv;              // [B][T] int32, [M][B] int64 x 2
  int64_t* h = nullptr;                          // pinned host staging
  size_t h_words = 0;
  int64_t graph_launches = 0, graph_instantiations = 0, graph_fallbacks = 0, batches = 0;
  bool graph_unsupported = false;  // a capture failed for another reason than arena growth: stay eager
};

void destroy_batch(bgs_ctx* c) {
  BatchState* bs = c->batch;
  if (!bs) return;
  for (bgs_ctx* sl : bs->slots) {
    sl->tr.reset();
    bgs_ctx_destroy(sl);
  }
  for (auto v : {&bs->streams, &bs->gstreams})
    for (cudaStream_t st : *v) cudaStreamDestroy(st);
  for (auto v : {&bs->done, &bs->gdone})
    for (cudaEvent_t e : *v) cudaEventDestroy(e);
  if (bs->fork) cudaEventDestroy(bs->fork);
  if (bs->gfork) cudaEventDestroy(bs->gfork);
  if (bs->cap) cudaStreamDestroy(bs->cap);
  if (bs->exec) cudaGraphExecDestroy(bs->exec);
  for (DevBuf* b : {&bs->pairs, &bs->tot_send, &bs->tot_recv})
    if (b->p) cudaFree(b->p);
  if (bs->h) cudaFreeHost(bs->h);
  delete bs;
  c->batch = nullptr;
}

bgs_status batch_prepare(bgs_ctx* ctx, int B) {
  if (!ctx->batch) {
    ctx->batch = new BatchState();
    CK(cudaEventCreateWithFlags(&ctx->batch->fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->batch->gfork, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&ctx->batch->cap, cudaStreamNonBlocking));
  }
  BatchState& bs = *ctx->batch;
  while (int(bs.slots.size()) < B) {
    auto* c = new bgs_ctx();
    c->rank = ctx->rank;
    c->world = ctx->world;
    c->device = ctx->device;
    bs.slots.push_back(c);  // owned by the batch from here on (destroy_batch frees it)
    if (ctx_alloc_common(c) != BGS_OK) return fail(ctx, BGS_ERR_CUDA, "batch view slot", c->err.c_str());
    c->tr = ctx->tr;  // per-view collectives of a slot (a12 at world > 1) go through the parent's transport
    cudaStream_t st, gst;
    cudaEvent_t e, ge;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    bs.streams.push_back(st);
    CK(cudaStreamCreateWithFlags(&gst, cudaStreamNonBlocking));
    bs.gstreams.push_back(gst);
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    bs.done.push_back(e);
    CK(cudaEventCreateWithFlags(&ge, cudaEventDisableTiming));
    bs.gdone.push_back(ge);
  }
  const size_t words = size_t(kMaxWorld) * kMaxBatch * 8 + 64;
  if (bs.h_words < words) {
    if (bs.h) CK(cudaFreeHost(bs.h));
    bs.h = nullptr;
    CK(cudaMallocHost(&bs.h, words * sizeof(int64_t)));
    bs.h_words = words;
  }
  return BGS_OK;
}

// fork: streams[0..B) wait for `from`; join: `to` waits for every stream's last work
bgs_status fork_streams(bgs_ctx* ctx, cudaEvent_t ev, cudaStream_t from, const std::vector<cudaStream_t>& st, int B) {
  CK(cudaEventRecord(ev, from));
  for (int b = 0; b < B; ++b) CK(cudaStreamWaitEvent(st[b], ev, 0));
  return BGS_OK;
}
bgs_status join_streams(bgs_ctx* ctx, const std::vector<cudaEvent_t>& ev, const std::vector<cudaStream_t>& st,
                        cudaStream_t to, int B) {
  for (int b = 0; b < B; ++b) {
    CK(cudaEventRecord(ev[b], st[b]));
    CK(cudaStreamWaitEvent(to, ev[b], 0));
  }
  return BGS_OK;
}

// a3 + a4 for the whole batch at world > 1 (the counterpart of bgs_route): one all-reduce of the
// B x T tile pair counts, one exchange of the B x M per-destination totals, the ONE host read of the
// batch (projection counters, totals, owner runs), then one grouped all-to-all of every view's
// records.  All on stream s, after the slots' projections were joined into it.
bgs_status batch_route(bgs_ctx* ctx, int B, cudaStream_t s) {
  BatchState& bs = *ctx->batch;
  const int M = ctx->world;
  const int T = bs.slots[0]->T;
  for (int b = 1; b < B; ++b)
    if (bs.slots[b]->T != T || bs.slots[b]->cam.TX != bs.slots[0]->cam.TX)
      return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "batch views must share the image size (one tile grid)");
  if (T > 16384) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "world > 1 supports at most 16384 tiles");
  CKS(ensure(ctx, bs.pairs, size_t(B) * T * 4));
  CKS(ensure(ctx, bs.tot_send, size_t(M) * B * 8));
  CKS(ensure(ctx, bs.tot_recv, size_t(M) * B * 8));
  int32_t* pairs = P_<int32_t>(bs.pairs);
  CK(cudaMemsetAsync(pairs, 0, size_t(B) * T * 4, s));
  for (int b = 0; b < B; ++b) {
    bgs_ctx* sl = bs.slots[b];
    if (sl->n_local > 0) {  // the record count is on the device until the host read
      launch_tile_count(P_<Rec>(sl->recs), sl->n_local, P_<unsigned long long>(sl->counters) + C_F, sl->cam.TX, 0, T,
                        pairs + size_t(b) * T, s);
      CKS(launched(ctx));
    }
  }
  CKS(ctx->tr->allreduce_i32(ctx, pairs, int64_t(B) * T, s));  // collective 1 of the batch
  for (int b = 0; b < B; ++b) {  // each view's global counts: a3's costs and its owner's bucket sizes
    bgs_ctx* sl = bs.slots[b];
    CKS(ensure(sl, sl->tile_pairs, size_t(T) * 4));
    CK(cudaMemcpyAsync(sl->tile_pairs.p, pairs + size_t(b) * T, size_t(T) * 4, cudaMemcpyDeviceToDevice, s));
  }
  for (int b = 0; b < B; ++b) {
    bgs_ctx* sl = bs.slots[b];
    const int64_t cap = std::max<int64_t>(sl->n_local, 1);  // F is on the device until the host read
    const int64_t nb = (cap + kRouteBlock - 1) / kRouteBlock;
    CKS(ensure(sl, sl->owner, size_t(T) * 4));
    CKS(ensure(sl, sl->runinfo, 64 + size_t(M + 1) * 8));
    CKS(ensure(sl, sl->dest_mask, size_t(cap)));
    CKS(ensure(sl, sl->block_counts, size_t(nb) * M * 4));
    CKS(ensure(sl, sl->totals, size_t(M) * 8));
    CKS(ensure(sl, sl->send_base, size_t(M) * 8));
    int32_t* run = P_<int32_t>(sl->runinfo);
    long long* pown = reinterpret_cast<long long*>(P_<char>(sl->runinfo) + 64);
    launch_owner_map(pairs + size_t(b) * T, T, M, P_<int32_t>(sl->owner), run, pown, nullptr, s);
    const unsigned long long* F_dev = P_<unsigned long long>(sl->counters) + C_F;
    launch_dest_count(P_<Rec>(sl->recs), cap, F_dev, P_<int32_t>(sl->owner), sl->cam.TX, M, P_<uint8_t>(sl->dest_mask),
                      P_<uint32_t>(sl->block_counts), s);
    launch_block_scan(P_<uint32_t>(sl->block_counts), cap, F_dev, M, P_<unsigned long long>(sl->totals), s);
    CKS(launched(ctx, 3));
    // totals of view b for destination d -> tot_send[d B + b]
    CK(cudaMemcpy2DAsync(P_<int64_t>(bs.tot_send) + b, size_t(B) * 8, sl->totals.p, 8, 8, size_t(M),
                         cudaMemcpyDeviceToDevice, s));
  }
  CKS(ctx->tr->alltoall_n(ctx, P_<int64_t>(bs.tot_send), P_<int64_t>(bs.tot_recv), B, s));  // collective 2
  // the one host read of the batch
  int64_t* h = bs.h;  // [0, MB) send, [MB, 2MB) recv, then per view: run (M int64 = 2M int32), pown (M + 1)
  const size_t MB = size_t(M) * B;
  CK(cudaMemcpyAsync(h, bs.tot_send.p, MB * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(h + MB, bs.tot_recv.p, MB * 8, cudaMemcpyDeviceToHost, s));
  for (int b = 0; b < B; ++b) {
    bgs_ctx* sl = bs.slots[b];
    int64_t* hb = h + 2 * MB + size_t(b) * (2 * M + 1);
    CK(cudaMemcpyAsync(hb, sl->runinfo.p, size_t(2 * M) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hb + M, P_<char>(sl->runinfo) + 64, size_t(M + 1) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamWaitEvent(s, sl->ev_counters, 0));  // the slot's projection counters reached the host
  }
  CK(host_sync(ctx, s));
  int64_t* hbase = h + 2 * MB + size_t(B) * (2 * M + 1);  // send_base staging, B x M
  std::vector<const void*> sends(B);
  std::vector<void*> recvs(B);
  std::vector<int64_t> scnt(MB), soff(MB), rcnt(MB), roff(MB);
  for (int b = 0; b < B; ++b) {
    bgs_ctx* sl = bs.slots[b];
    project_finish(sl);
    const int64_t* hb = h + 2 * MB + size_t(b) * (2 * M + 1);
    const int32_t* hrun = reinterpret_cast<const int32_t*>(hb);
    sl->t_begin = hrun[2 * ctx->rank];
    sl->t_end = hrun[2 * ctx->rank + 1];
    sl->P = hb[M + ctx->rank];
    sl->send_cnt.assign(M, 0);
    sl->recv_cnt.assign(M, 0);
    sl->send_off.assign(M, 0);
    sl->recv_off.assign(M, 0);
    int64_t D = 0, R = 0;
    for (int d = 0; d < M; ++d) {
      sl->send_cnt[d] = h[size_t(d) * B + b];
      sl->recv_cnt[d] = h[MB + size_t(d) * B + b];
      sl->send_off[d] = D;
      sl->recv_off[d] = R;
      D += sl->send_cnt[d];
      R += sl->recv_cnt[d];
      scnt[size_t(b) * M + d] = sl->send_cnt[d];
      soff[size_t(b) * M + d] = sl->send_off[d];
      rcnt[size_t(b) * M + d] = sl->recv_cnt[d];
      roff[size_t(b) * M + d] = sl->recv_off[d];
      hbase[size_t(b) * M + d] = sl->send_off[d];
    }
    if (D != [&] { int64_t c = 0; for (int d = 0; d < M; ++d) c += sl->send_cnt[d]; return c; }() || sl->F < 0)
      return fail(ctx, BGS_ERR_INTERNAL, "batch route: inconsistent counts");
    sl->D = D;
    sl->R = R;
    CKS(ensure(sl, sl->send, size_t(std::max<int64_t>(D, 1)) * sizeof(Rec)));
    CKS(ensure(sl, sl->recvbuf, size_t(std::max<int64_t>(R, 1)) * sizeof(Rec)));
    CK(cudaMemcpyAsync(sl->send_base.p, hbase + size_t(b) * M, size_t(M) * 8, cudaMemcpyHostToDevice, s));
    if (sl->F > 0) {
      launch_pack(P_<Rec>(sl->recs), sl->F, nullptr, P_<uint8_t>(sl->dest_mask), P_<uint32_t>(sl->block_counts), M,
                  P_<int64_t>(sl->send_base), P_<Rec>(sl->send), s);
      CKS(launched(ctx));
    }
    sends[b] = sl->send.p;
    recvs[b] = sl->recvbuf.p;
  }
  CKS(ctx->tr->alltoallv_batch(ctx, B, sends.data(), scnt.data(), soff.data(), recvs.data(), rcnt.data(),
                               roff.data(), sizeof(Rec), s));  // collective 3: ONE exchange of the batch
  for (int b = 0; b < B; ++b) {
    bgs_ctx* sl = bs.slots[b];
    sl->recv = P_<Rec>(sl->recvbuf);
    sl->stage = 2;
  }
  return BGS_OK;
}

// a10 for the whole batch at world > 1: ONE grouped all-to-all of every view's accumulators back
// along the transposed counts, then each view's owner-ordered gather-sum.
bgs_status batch_reverse(bgs_ctx* ctx, int B, cudaStream_t s) {
  BatchState& bs = *ctx->batch;
  const int M = ctx->world;
  const size_t MB = size_t(M) * B;
  std::vector<const void*> sends(B);
  std::vector<void*> recvs(B);
  std::vector<int64_t> scnt(MB), soff(MB), rcnt(MB), roff(MB);
  for (int b = 0; b < B; ++b) {
    bgs_ctx* sl = bs.slots[b];
    CKS(ensure(sl, sl->rev, size_t(std::max<int64_t>(sl->D, 1)) * sizeof(Acc)));
    CKS(ensure(sl, sl->accl, size_t(std::max<int64_t>(sl->F, 1)) * sizeof(Acc)));
    for (int d = 0; d < M; ++d) {
      scnt[size_t(b) * M + d] = sl->recv_cnt[d];
      soff[size_t(b) * M + d] = sl->recv_off[d];
      rcnt[size_t(b) * M + d] = sl->send_cnt[d];
      roff[size_t(b) * M + d] = sl->send_off[d];
    }
    sends[b] = sl->acc.p;
    recvs[b] = sl->rev.p;
  }
  CKS(ctx->tr->alltoallv_batch(ctx, B, sends.data(), scnt.data(), soff.data(), recvs.data(), rcnt.data(),
                               roff.data(), sizeof(Acc), s));  // collective 4
  for (int b = 0; b < B; ++b) {
    bgs_ctx* sl = bs.slots[b];
    if (sl->F > 0) {
      launch_gather_sum(P_<Acc>(sl->rev), sl->F, nullptr, P_<uint8_t>(sl->dest_mask), P_<uint32_t>(sl->block_counts),
                        M, P_<int64_t>(sl->send_base), P_<Acc>(sl->accl), s);
      CKS(launched(ctx));
    }
    sl->acc_local = P_<Acc>(sl->accl);
    sl->stage = 6;
  }
  return BGS_OK;
}

// the view's Cull column: the caller's, else the slot's scratch (sized before the batch runs)
uint32_t* slot_cull(bgs_ctx* sl, const bgs_batch_view& v) {
  return v.cull_out ? v.cull_out : P_<uint32_t>(sl->scr_n);
}

// Phases of one view slot after the sizes are known (run on stream st).  World 1 runs them all per
// slot on its own stream; world > 1 runs the collective ones (loss reductions, a10, a12) batched or
// serialised on the parent stream, in view order on every rank.
enum : uint32_t { PH_FWD = 1, PH_LOSS = 2, PH_BWD = 4, PH_REV = 8, PH_PBWD = 16, PH_IMP = 32, PH_ALL = 63 };

bgs_status check_view_sup(bgs_ctx* ctx, const bgs_batch_view& v) {
  if (!v.sup) return BGS_OK;
  if (!v.sup->target || !v.sup->loss_out || !v.dL_scratch)
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "supervised batch view: target / loss_out / dL_scratch is NULL");
  return BGS_OK;
}

bgs_status slot_phases(bgs_ctx* sl, const bgs_gaussians* g, const bgs_batch_view& v, uint32_t flags,
                       const bgs_gaussian_grads* grads, const bgs_importance_out* imp, cudaStream_t st,
                       uint32_t ph) {
  const float* dL = v.sup ? v.dL_scratch : v.dL_drgb;
  if (ph & PH_FWD) {
    CKS(bgs_sort_tiles(sl, st));
    CKS(bgs_raster_fwd(sl, flags, v.rgb, v.t_final, v.n_contrib, st));
  }
  if ((ph & PH_LOSS) && v.sup) {  // NEXT-4 Eq.7 (+ Eq.8) writes this view's dL/dC
    const bgs_supervision& sp = *v.sup;
    CKS(bgs_loss_photo(sl, v.rgb, sp.target, sp.lambda, sp.batch_inv, v.dL_scratch, sp.loss_out, st));
    if (sp.beta != 0.f && grads)
      CKS(bgs_loss_scale(sl, g, sp.beta, grads, sp.loss_out + 3, st));
    else
      CK_CTX(sl, cudaMemsetAsync(sp.loss_out + 3, 0, 2 * sizeof(double), st));
  }
  if ((ph & PH_BWD) && dL) CKS(bgs_raster_bwd(sl, dL, v.t_final, v.n_contrib, st));
  if (ph & PH_REV) CKS(bgs_route_reverse(sl, dL ? 0u : uint32_t(BGS_IMPORTANCE_ONLY), st));
  if ((ph & PH_PBWD) && dL && grads) CKS(bgs_project_bwd(sl, g, &v.cam, grads, st));
  if ((ph & PH_IMP) && imp)
    CKS(bgs_importance(sl, g->n_local, v.radius_out, nullptr, nullptr, imp->mass_num, imp->mass_den, imp->s,
                       imp->c_rad, imp->c_vis, slot_cull(sl, v), st));
  return BGS_OK;
}

void clear_capture(bgs_ctx* ctx, int B) {
  for (int b = 0; b < B; ++b) ctx->batch->slots[b]->capturing = false;
  ctx->capturing = false;
}

// world 1, BGS_GRAPH: record the post-read part of all B views as one graph (slots forked from the
// capture stream), update the executable in place (or instantiate it), launch it on s.  Returns
// BGS_OK with *ran = false when the capture had to be abandoned (an arena must grow first, or a
// launch is not capturable): the caller then runs the same work eagerly.
bgs_status batch_graph(bgs_ctx* ctx, int B, const bgs_gaussians* g, const bgs_batch_view* views, uint32_t flags,
                       const bgs_gaussian_grads* grads, const bgs_importance_out* imp, cudaStream_t s, bool* ran) {
  BatchState& bs = *ctx->batch;
  *ran = false;
  if (bs.graph_unsupported) return BGS_OK;
  std::vector<int> parity(B);
  for (int b = 0; b < B; ++b) parity[b] = bs.slots[b]->imp_parity;
  CK(cudaStreamBeginCapture(bs.cap, cudaStreamCaptureModeThreadLocal));
  bgs_status st = BGS_OK;
  for (int b = 0; b < B; ++b) {
    bs.slots[b]->capturing = true;
    bs.slots[b]->grew_in_capture = false;
  }
  st = fork_streams(ctx, bs.gfork, bs.cap, bs.gstreams, B);
  for (int b = 0; b < B && st == BGS_OK; ++b) {
    st = slot_phases(bs.slots[b], g, views[b], flags, grads, imp, bs.gstreams[b], PH_ALL);
    if (st != BGS_OK) ctx->err = bs.slots[b]->err;
  }
  if (st == BGS_OK) st = join_streams(ctx, bs.gdone, bs.gstreams, bs.cap, B);
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(bs.cap, &graph);
  clear_capture(ctx, B);
  if (st != BGS_OK || ec != cudaSuccess || !graph) {
    if (graph) cudaGraphDestroy(graph);
    // streams that joined the failed capture are back to normal after EndCapture; any error the
    // failed capture left is cleared so the eager run starts clean
    (void)cudaGetLastError();
    bool grew = false;
    for (int b = 0; b < B; ++b) {
      grew |= bs.slots[b]->grew_in_capture;
      bs.slots[b]->imp_parity = parity[b];  // the captured importance calls never ran
      bs.slots[b]->err.clear();
    }
    ctx->err.clear();
    if (!grew) bs.graph_unsupported = true;
    ++bs.graph_fallbacks;
    return BGS_OK;
  }
  bool updated = false;
  if (bs.exec) {
    cudaGraphExecUpdateResultInfo info{};
    updated = cudaGraphExecUpdate(bs.exec, graph, &info) == cudaSuccess;
    if (!updated) {
      (void)cudaGetLastError();
      cudaGraphExecDestroy(bs.exec);
      bs.exec = nullptr;
    }
  }
  if (!bs.exec) {
    const cudaError_t ei = cudaGraphInstantiate(&bs.exec, graph, 0);
    if (ei != cudaSuccess) {
      cudaGraphDestroy(graph);
      bs.exec = nullptr;
      return fail(ctx, BGS_ERR_CUDA, "cudaGraphInstantiate", cudaGetErrorString(ei));
    }
    ++bs.graph_instantiations;
  }
  cudaGraphDestroy(graph);
  CK(cudaGraphLaunch(bs.exec, s));
  ++bs.graph_launches;
  for (int b = 0; b < B; ++b) ctx->launches += bs.slots[b]->launches, bs.slots[b]->launches = 0;
  *ran = true;
  return BGS_OK;
}

}  // namespace

extern "C" {

bgs_status bgs_batch_step(bgs_ctx* ctx, int32_t n_views, const bgs_gaussians* g, const bgs_lod_gate* gate,
                          uint32_t flags, const bgs_batch_view* views, const bgs_gaussian_grads* grads,
                          const bgs_importance_out* imp, void* stream) {
  NvtxRange nvtx_("bgs_batch_step");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  CKS(check_gaussians(ctx, g));
  const int B = n_views;
  if (B < 1 || B > kMaxBatch || !views) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "n_views must be in [1, 16]");
  bool any_sup = false;
  for (int b = 0; b < B; ++b) {
    const bgs_batch_view& v = views[b];
    if ((g->n_local > 0 && !v.radius_out) || !v.rgb || !v.t_final || !v.n_contrib)
      return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "batch view: radius / rgb / t_final / n_contrib pointer is NULL");
    CKS(check_view_sup(ctx, v));
    any_sup |= v.sup != nullptr;
  }
  if (imp && (!imp->s || !imp->c_rad || !imp->c_vis))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "importance s / c_rad / c_vis must be non-NULL");
  const bool graph = (flags & BGS_GRAPH) != 0 && ctx->world == 1;
  CKS(batch_prepare(ctx, B));
  BatchState& bs = *ctx->batch;
  cudaStream_t s = as_stream(stream);
  if (imp)
    for (int b = 0; b < B; ++b)
      if (!views[b].cull_out)
        CKS(ensure(bs.slots[b], bs.slots[b]->scr_n, size_t((g->n_local + 31) / 32 + 1) * 4));
  const uint32_t vflags = (flags & BGS_NO_COLOR) | (imp ? BGS_IMPORTANCE : 0u);
  ++bs.batches;
  // a1 + a2 of every view on its slot stream
  CKS(fork_streams(ctx, bs.fork, s, bs.streams, B));
  for (int b = 0; b < B; ++b) {
    bgs_ctx* sl = bs.slots[b];
    sl->err.clear();
    const bgs_status st = project_enqueue(sl, g, &views[b].cam, gate, views[b].cull_column, vflags,
                                          views[b].radius_out, bs.streams[b]);
    if (st != BGS_OK) return fail(ctx, st, "batch view projection", sl->err.c_str());
  }
  CKS(join_streams(ctx, bs.done, bs.streams, s, B));
  if (ctx->world == 1) {
    // the one host read of the batch: every view's projection counters
    for (int b = 0; b < B; ++b) CK(cudaEventSynchronize(bs.slots[b]->ev_counters));
    ++ctx->host_syncs;
    for (int b = 0; b < B; ++b) {
      project_finish(bs.slots[b]);
      CKS(bgs_route(bs.slots[b], nullptr, nullptr, nullptr, s));  // identity at world 1 (no work)
    }
    bool ran = false;
    if (graph) CKS(batch_graph(ctx, B, g, views, vflags, grads, imp, s, &ran));
    if (!ran) {
      CKS(fork_streams(ctx, bs.fork, s, bs.streams, B));
      for (int b = 0; b < B; ++b) {
        const bgs_status st = slot_phases(bs.slots[b], g, views[b], vflags, grads, imp, bs.streams[b], PH_ALL);
        if (st != BGS_OK) return fail(ctx, st, "batch view", bs.slots[b]->err.c_str());
      }
      CKS(join_streams(ctx, bs.done, bs.streams, s, B));
    }
  } else {
    CKS(batch_route(ctx, B, s));
    // per-slot work on the slot streams; phases with collectives on s, view order (same on every rank)
    auto par = [&](uint32_t ph) -> bgs_status {
      CKS(fork_streams(ctx, bs.fork, s, bs.streams, B));
      for (int b = 0; b < B; ++b) {
        const bgs_status st = slot_phases(bs.slots[b], g, views[b], vflags, grads, imp, bs.streams[b], ph);
        if (st != BGS_OK) return fail(ctx, st, "batch view", bs.slots[b]->err.c_str());
      }
      return join_streams(ctx, bs.done, bs.streams, s, B);
    };
    auto ser = [&](uint32_t ph) -> bgs_status {
      for (int b = 0; b < B; ++b) {
        const bgs_status st = slot_phases(bs.slots[b], g, views[b], vflags, grads, imp, s, ph);
        if (st != BGS_OK) return fail(ctx, st, "batch view", bs.slots[b]->err.c_str());
      }
      return BGS_OK;
    };
    CKS(par(PH_FWD));
    if (any_sup) CKS(ser(PH_LOSS));  // the loss's image and sum all-reduces
    CKS(par(PH_BWD));
    CKS(batch_reverse(ctx, B, s));
    CKS(par(PH_PBWD));
    if (imp) CKS(ser(PH_IMP));  // a12's selection rounds are collectives
  }
  // the slots' launches and collectives are the batch's
  for (int b = 0; b < B; ++b) {
    ctx->launches += bs.slots[b]->launches;
    bs.slots[b]->launches = 0;
    ctx->collectives += bs.slots[b]->collectives;
    bs.slots[b]->collectives = 0;
    ctx->host_syncs += bs.slots[b]->host_syncs;
    bs.slots[b]->host_syncs = 0;
  }
  return BGS_OK;
}

bgs_status bgs_batch_view_ctx(bgs_ctx* ctx, int32_t b, bgs_ctx** out) {
  if (!ctx || !out) return BGS_ERR_INVALID_ARGUMENT;
  if (!ctx->batch || b < 0 || b >= int32_t(ctx->batch->slots.size()))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "no such batch view slot (run bgs_batch_step first)");
  *out = ctx->batch->slots[b];
  return BGS_OK;
}

bgs_status bgs_batch_stats(bgs_ctx* ctx, int64_t* out) {
  if (!ctx || !out) return BGS_ERR_INVALID_ARGUMENT;
  const BatchState* bs = ctx->batch;
  const int64_t v[6] = {ctx->host_syncs, ctx->collectives, bs ? bs->batches : 0, bs ? bs->graph_launches : 0,
                        bs ? bs->graph_instantiations : 0, bs ? bs->graph_fallbacks : 0};
  std::memcpy(out, v, sizeof v);
  return BGS_OK;
}

}  // extern "C"


extern "C" {

// ---------------------------------------------------------------------------------------
// NEXT-4 supervision: Eq.7 photometric loss + gradient on the owned tiles, Eq.8 regulariser
// ---------------------------------------------------------------------------------------
bgs_status bgs_loss_photo(bgs_ctx* ctx, const float* rgb, const float* target, float lambda, float batch_inv,
                          float* dL_drgb, double* out, void* stream) {
  NvtxRange nvtx_("bgs_loss_photo");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (ctx->stage < 4) return fail(ctx, BGS_ERR_CONTRACT, "bgs_loss_photo before bgs_raster_fwd");
  if (!rgb || !target || !dL_drgb || !out) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "loss pointer is NULL");
  if (!(lambda >= 0.f && lambda <= 1.f)) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "lambda outside [0, 1]");
  cudaStream_t s = as_stream(stream);
  const int W = ctx->cam.W, H = ctx->cam.H;
  const size_t plane = size_t(W) * H;
  const float* x = rgb;
  if (ctx->world > 1) {
    // the owned pixels of every rank summed into one full image (x + 0 = x: every rank holds
    // the same bits), so windows across ownership boundaries match the single-GPU loss
    CKS(ensure(ctx, ctx->loss_img, 3 * plane * 4));
    CK(cudaMemsetAsync(ctx->loss_img.p, 0, 3 * plane * 4, s));
    launch_owned_copy(rgb, W, H, ctx->cam.TX, ctx->t_begin, ctx->t_end, P_<float>(ctx->loss_img), s);
    CKS(launched(ctx));
    CKS(ctx->tr->allreduce_f32(ctx, P_<float>(ctx->loss_img), int64_t(3 * plane), s));
    x = P_<float>(ctx->loss_img);
  }
  const int64_t nb = loss_n_blocks(W, H);
  CKS(ensure(ctx, ctx->loss_part, size_t(nb) * sizeof(double2)));
  CKS(ensure(ctx, ctx->loss_sums, 8 * sizeof(double)));
  LossArgs a{};
  a.x = x;
  a.y = target;
  a.dL = dL_drgb;
  a.partials = P_<double2>(ctx->loss_part);
  a.W = W;
  a.H = H;
  a.TX = ctx->cam.TX;
  a.t_begin = ctx->t_begin;
  a.t_end = ctx->t_end;
  const double n_elem = 3.0 * double(plane);
  a.k_l1 = float(double(batch_inv) * (1.0 - double(lambda)) / n_elem);
  a.k_ssim = float(double(batch_inv) * double(lambda) / n_elem);
  // normalised 1-D window, sigma 1.5 (computed in double, rounded once)
  double gw[11], gs = 0.0;
  for (int k = 0; k < 11; ++k) gs += (gw[k] = std::exp(-double((k - 5) * (k - 5)) / (2.0 * 1.5 * 1.5)));
  for (int k = 0; k < 11; ++k) a.g[k] = float(gw[k] / gs);
  launch_loss_photo(a, s);
  CKS(launched(ctx));
  double* sums = P_<double>(ctx->loss_sums);
  launch_loss_sums(a.partials, int(nb), sums, s);
  CKS(launched(ctx));
  if (ctx->world > 1) CKS(ctx->tr->allreduce_f64(ctx, sums, 2, s));
  launch_loss_finish(sums, n_elem, double(lambda), out, s);
  CKS(launched(ctx));
  return BGS_OK;
}

bgs_status bgs_loss_scale(bgs_ctx* ctx, const bgs_gaussians* g, float beta, const bgs_gaussian_grads* grads,
                          double* out, void* stream) {
  NvtxRange nvtx_("bgs_loss_scale");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  CKS(check_gaussians(ctx, g));
  if (ctx->stage < 1) return fail(ctx, BGS_ERR_CONTRACT, "bgs_loss_scale before bgs_project");
  if (!out || !grads || !grads->scale) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "loss_scale pointer is NULL");
  cudaStream_t s = as_stream(stream);
  const int64_t F = ctx->F;  // this view's records = the local visible set (radius > 0)
  const uint32_t* lidx = P_<uint32_t>(ctx->rec_lidx);
  const int nb = scale_n_blocks(F);
  CKS(ensure(ctx, ctx->loss_part, size_t(nb) * sizeof(double2)));
  CKS(ensure(ctx, ctx->loss_sums, 8 * sizeof(double)));
  double* sums = P_<double>(ctx->loss_sums) + 4;
  launch_scale_sum(reinterpret_cast<const float4*>(g->scale), lidx, F, P_<double2>(ctx->loss_part), s);
  CKS(launched(ctx));
  launch_loss_sums(P_<double2>(ctx->loss_part), nb, sums, s);
  CKS(launched(ctx));
  if (ctx->world > 1) CKS(ctx->tr->allreduce_f64(ctx, sums, 2, s));
  launch_scale_finish(sums, out, s);
  CKS(launched(ctx));
  if (F > 0) {
    launch_scale_grad(reinterpret_cast<const float4*>(g->scale), lidx, F, sums, beta, grads->scale, s);
    CKS(launched(ctx));
  }
  return BGS_OK;
}

// ---------------------------------------------------------------------------------------
// NEXT-3: fused Adam on the owned shard (adam.cu)
// ---------------------------------------------------------------------------------------
bgs_status bgs_adam_step(bgs_ctx* ctx, const bgs_train_params* p, const bgs_gaussian_grads* grads,
                         const bgs_gaussians_out* act, const uint32_t* visible, const bgs_adam_hparams* h,
                         void* stream) {
  NvtxRange nvtx_("bgs_adam_step");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (!p || !grads || !act || !h) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "adam: NULL argument");
  if (p->n_local < 0) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "adam: n_local < 0");
  if (h->step < 1) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "adam: step must be >= 1");
  if (!(h->beta1 >= 0.0 && h->beta1 < 1.0 && h->beta2 >= 0.0 && h->beta2 < 1.0))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "adam: betas outside [0, 1)");
  if (p->n_local == 0) return BGS_OK;
  if (act->capacity < p->n_local) return fail(ctx, BGS_ERR_CAPACITY, "adam: act capacity < n_local");
  const float* planes[] = {p->mean_logit, p->quat_raw, p->log_scale, p->sh, p->m[0], p->m[1], p->m[2], p->m[3],
                           p->v[0], p->v[1], p->v[2], p->v[3], grads->mean_opac, grads->quat, grads->scale,
                           grads->sh, act->mean_opac, act->quat, act->scale, act->sh};
  for (const float* q : planes)
    if (!q) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "adam: plane pointer is NULL");
  AdamArgs a{};
  a.n = p->n_local;
  float* raw[3] = {p->mean_logit, p->quat_raw, p->log_scale};
  float* gr[3] = {grads->mean_opac, grads->quat, grads->scale};
  float* ac[3] = {act->mean_opac, act->quat, act->scale};
  for (int k = 0; k < 3; ++k) {
    a.p[k] = reinterpret_cast<float4*>(raw[k]);
    a.m[k] = reinterpret_cast<float4*>(p->m[k]);
    a.v[k] = reinterpret_cast<float4*>(p->v[k]);
    a.g[k] = reinterpret_cast<float4*>(gr[k]);
    a.act[k] = reinterpret_cast<float4*>(ac[k]);
  }
  a.sh_p = p->sh;
  a.sh_m = p->m[3];
  a.sh_v = p->v[3];
  a.sh_g = grads->sh;
  a.sh_act = act->sh;
  a.visible = visible;
  a.lr_mean = h->lr_mean;
  a.lr_opacity = h->lr_opacity;
  a.lr_quat = h->lr_quat;
  a.lr_scale = h->lr_scale;
  a.lr_sh_dc = h->lr_sh_dc;
  a.lr_sh_rest = h->lr_sh_rest;
  a.b1 = float(h->beta1);
  a.b2 = float(h->beta2);
  a.om1 = float(1.0 - h->beta1);
  a.om2 = float(1.0 - h->beta2);
  a.eps = float(h->eps);
  a.c1 = float(1.0 / (1.0 - std::pow(h->beta1, double(h->step))));
  a.c2 = float(1.0 / (1.0 - std::pow(h->beta2, double(h->step))));
  launch_adam(a, as_stream(stream));
  CKS(launched(ctx, 2));
  return BGS_OK;
}

// ---------------------------------------------------------------------------------------
// NEXT-3: density control (densify.cu)
// ---------------------------------------------------------------------------------------
bgs_status bgs_visibility_mask(bgs_ctx* ctx, int64_t n_local, const int32_t* radius, uint32_t* mask, void* stream) {
  CKS(check_ctx(ctx));
  if (n_local < 0 || (n_local > 0 && (!radius || !mask)))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "visibility_mask: radius and mask must be non-NULL");
  launch_visibility_or(radius, n_local, mask, as_stream(stream));
  return n_local > 0 ? launched(ctx) : BGS_OK;
}

bgs_status bgs_densify_accumulate(bgs_ctx* ctx, int64_t n_local, const double* phi, float* stat, uint32_t* count,
                                  void* stream) {
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (ctx->stage < 6) return fail(ctx, BGS_ERR_CONTRACT, "bgs_densify_accumulate before bgs_route_reverse");
  if (n_local != ctx->n_local) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "densify: n_local differs from the view's");
  if (ctx->F > 0 && (!stat || !count)) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "densify: stat / count NULL");
  DensifyAccArgs a{};
  a.F = ctx->F;
  a.lidx = P_<uint32_t>(ctx->rec_lidx);
  a.recs = P_<Rec>(ctx->recs);
  a.acc = ctx->acc_local;
  a.phi = phi;
  a.half_w = 0.5f * float(ctx->cam.W);
  a.half_h = 0.5f * float(ctx->cam.H);
  a.stat = stat;
  a.count = count;
  if (a.F > 0) {
    launch_densify_accumulate(a, as_stream(stream));
    CKS(launched(ctx));
  }
  return BGS_OK;
}

static bool planes_ok(const bgs_train_params* p) {
  if (!p->mean_logit || !p->quat_raw || !p->log_scale || !p->sh) return false;
  for (int k = 0; k < 4; ++k)
    if (!p->m[k] || !p->v[k]) return false;
  return true;
}

bgs_status bgs_densify_apply(bgs_ctx* ctx, const bgs_train_params* in, const uint8_t* lod_in, const float* stat,
                             const uint32_t* count, const bgs_densify_params* dp, const bgs_train_params* out,
                             uint8_t* lod_out, const bgs_gaussians_out* act_out, int64_t* n_out, void* stream) {
  NvtxRange nvtx_("bgs_densify_apply");
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (!in || !out || !dp || !n_out) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "densify: NULL argument");
  if (in->n_local < 0) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "densify: n_local < 0");
  if (!(dp->split_div > 0.f)) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "densify: split_div must be > 0");
  *n_out = 0;
  if (in->n_local == 0) return BGS_OK;
  if (!planes_ok(in) || !planes_ok(out) || !lod_in || !lod_out || !stat || !count)
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "densify: plane pointer is NULL");
  if (act_out && (!act_out->mean_opac || !act_out->quat || !act_out->scale || !act_out->sh))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "densify: act_out plane pointer is NULL");
  cudaStream_t s = as_stream(stream);
  DensifyArgs a{};
  a.n = in->n_local;
  a.rank = ctx->rank;
  a.world = ctx->world;
  const float* ip[3] = {in->mean_logit, in->quat_raw, in->log_scale};
  float* op[3] = {out->mean_logit, out->quat_raw, out->log_scale};
  for (int k = 0; k < 3; ++k) {
    a.p_in[k] = reinterpret_cast<const float4*>(ip[k]);
    a.m_in[k] = reinterpret_cast<const float4*>(in->m[k]);
    a.v_in[k] = reinterpret_cast<const float4*>(in->v[k]);
    a.p_out[k] = reinterpret_cast<float4*>(op[k]);
    a.m_out[k] = reinterpret_cast<float4*>(out->m[k]);
    a.v_out[k] = reinterpret_cast<float4*>(out->v[k]);
  }
  a.sh_in = in->sh;
  a.sh_m_in = in->m[3];
  a.sh_v_in = in->v[3];
  a.sh_out = out->sh;
  a.sh_m_out = out->m[3];
  a.sh_v_out = out->v[3];
  a.lod_in = lod_in;
  a.lod_out = lod_out;
  a.stat = stat;
  a.count = count;
  a.tau = dp->grad_threshold;
  if (!(dp->dense_extent > 0.f) || !(dp->min_opacity > 0.f && dp->min_opacity < 1.f))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "densify: dense_extent > 0 and 0 < min_opacity < 1 required");
  a.log_extent = float(std::log(double(dp->dense_extent)));
  a.logit_min = float(std::log(double(dp->min_opacity) / (1.0 - double(dp->min_opacity))));
  a.log_div = float(std::log(double(dp->split_div)));
  a.seed = dp->seed;
  if (dp->k_levels < 1 || dp->k_levels > 256)
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "densify: k_levels must be in [1, 256]");
  a.max_level = dp->k_levels - 1;
  if (act_out) {
    a.act[0] = reinterpret_cast<float4*>(act_out->mean_opac);
    a.act[1] = reinterpret_cast<float4*>(act_out->quat);
    a.act[2] = reinterpret_cast<float4*>(act_out->scale);
    a.sh_act = act_out->sh;
  }
  const int64_t nb = densify_n_blocks(a.n);
  CKS(ensure(ctx, ctx->dcnt, size_t(3 * nb + 8) * 4 + 64));
  a.block_counts = P_<uint32_t>(ctx->dcnt) + 16;
  a.totals = P_<unsigned long long>(ctx->dcnt);
  launch_densify_count(a, s);
  CKS(launched(ctx, 2));
  unsigned long long tot[3];
  CK(cudaMemcpyAsync(tot, a.totals, sizeof tot, cudaMemcpyDeviceToHost, s));
  CK(host_sync(ctx, s));
  const int64_t n_new = int64_t(tot[0] + tot[1] + 2 * tot[2]);
  *n_out = n_new;
  if (n_new > out->n_local || (act_out && n_new > act_out->capacity))
    return fail(ctx, BGS_ERR_CAPACITY, "densify: new shard exceeds the output capacity");
  launch_densify_emit(a, s);
  CKS(launched(ctx));
  return BGS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// NEXT-1: phi, scheduled simplification passes, index-parity redistribution (simplify.cu)
// ---------------------------------------------------------------------------------------
namespace {

// sum of n host values over the ranks (small scratch in dcnt[0, 8)); synchronises the stream
bgs_status sum_over_ranks(bgs_ctx* ctx, unsigned long long* vals, int n, cudaStream_t s) {
  if (ctx->world == 1) return BGS_OK;
  CKS(ensure(ctx, ctx->dcnt, 64 * 8));
  unsigned long long* d = P_<unsigned long long>(ctx->dcnt);
  CK(cudaMemcpyAsync(d, vals, size_t(n) * 8, cudaMemcpyHostToDevice, s));
  CKS(ctx->tr->allreduce_u64(ctx, d, n, s));
  CK(cudaMemcpyAsync(vals, d, size_t(n) * 8, cudaMemcpyDeviceToHost, s));
  CK(host_sync(ctx, s));
  return BGS_OK;
}

// keep = top of (key desc, global id asc) over all ranks: the first k items (count mode) or the
// smallest prefix with den * mass >= num * total (mass mode)
bgs_status run_select(bgs_ctx* ctx, int64_t n, const unsigned long long* key, int mass, long long num, long long den,
                      unsigned long long k, uint8_t* keep, cudaStream_t s) {
  const int R = sel_rounds(), GR = sel_gid_rounds();
  const size_t hw = size_t(R) * 512 + size_t(GR) * 256 + 8;
  CKS(ensure(ctx, ctx->sel_state, sel_state_bytes()));
  CKS(ensure(ctx, ctx->sel_hist, hw * 8));
  CK(cudaMemsetAsync(ctx->sel_state.p, 0, sel_state_bytes(), s));
  CK(cudaMemsetAsync(ctx->sel_hist.p, 0, hw * 8, s));
  unsigned long long* hist = P_<unsigned long long>(ctx->sel_hist);
  unsigned long long* total = hist + size_t(R) * 512 + size_t(GR) * 256;
  void* st = ctx->sel_state.p;
  int nl = 0;
  launch_sel_total(n, key, mass, total, s);
  ++nl;
  if (ctx->world > 1) CKS(ctx->tr->allreduce_u64(ctx, total, 1, s));
  for (int r = 0; r < R; ++r) {
    launch_sel_hist(n, key, st, r, hist + r * 512, s);
    if (ctx->world > 1) CKS(ctx->tr->allreduce_u64(ctx, hist + r * 512, 512, s));
    launch_sel_decide(st, total, r, hist + r * 512, mass, num, den, k, s);
    nl += 2;
  }
  for (int r = 0; r < GR; ++r) {
    unsigned long long* h = hist + size_t(R) * 512 + size_t(r) * 256;
    launch_sel_gid_hist(n, key, st, r, ctx->rank, ctx->world, h, s);
    if (ctx->world > 1) CKS(ctx->tr->allreduce_u64(ctx, h, 256, s));
    launch_sel_gid_decide(st, r, h, s);
    nl += 2;
  }
  launch_sel_mark(n, key, st, ctx->rank, ctx->world, keep, s);
  return launched(ctx, nl + 1);
}

}  // namespace

extern "C" {

bgs_status bgs_score_phi(bgs_ctx* ctx, int64_t n_local, const uint32_t* c_rad, const uint32_t* c_vis, double* phi,
                         void* stream) {
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (n_local < 0 || (n_local > 0 && (!c_rad || !c_vis || !phi)))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bgs_score_phi: arguments");
  launch_phi(n_local, c_rad, c_vis, phi, as_stream(stream));
  return n_local > 0 ? launched(ctx) : BGS_OK;
}

bgs_status bgs_prune_stochastic(bgs_ctx* ctx, int64_t n_local, const double* s_score, int64_t keep_count,
                                uint64_t seed, uint8_t* keep_out, void* stream) {
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (n_local < 0 || (n_local > 0 && (!s_score || !keep_out)))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bgs_prune_stochastic: arguments");
  if (n_local >= (int64_t(1) << 32) / ctx->world) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "global ids exceed 32 bits");
  cudaStream_t s = as_stream(stream);
  unsigned long long N = (unsigned long long)n_local;
  CKS(sum_over_ranks(ctx, &N, 1, s));
  if (keep_count <= 0 || (unsigned long long)keep_count >= N) {
    launch_fill_u8(n_local, keep_out, keep_count <= 0 ? 0 : 1, s);
    CKS(n_local > 0 ? launched(ctx) : BGS_OK);
    CK(host_sync(ctx, s));
    return BGS_OK;
  }
  CKS(ensure(ctx, ctx->sel_keys, size_t(std::max<int64_t>(n_local, 1)) * 8));
  unsigned long long* key = P_<unsigned long long>(ctx->sel_keys);
  launch_keys_race(n_local, s_score, (unsigned long long)seed, ctx->rank, ctx->world, key, s);
  CKS(n_local > 0 ? launched(ctx) : BGS_OK);
  CKS(run_select(ctx, n_local, key, 0, 0, 1, (unsigned long long)keep_count, keep_out, s));
  CK(host_sync(ctx, s));
  return BGS_OK;
}

bgs_status bgs_prune_mass_cut(bgs_ctx* ctx, int64_t n_local, const double* s_score, int32_t num, int32_t den,
                              uint8_t* keep_out, int32_t* all_zero_out, void* stream) {
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (n_local < 0 || (n_local > 0 && (!s_score || !keep_out)))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bgs_prune_mass_cut: arguments");
  if (den <= 0 || num <= 0 || num > den) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "mass cut needs 0 < num <= den");
  if (n_local >= (int64_t(1) << 32) / ctx->world) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "global ids exceed 32 bits");
  cudaStream_t s = as_stream(stream);
  if (all_zero_out) *all_zero_out = 0;
  CKS(ensure(ctx, ctx->sel_keys, size_t(std::max<int64_t>(n_local, 1)) * 8));
  CKS(ensure(ctx, ctx->dcnt, 64 * 8));
  unsigned long long* key = P_<unsigned long long>(ctx->sel_keys);
  unsigned long long* cnt = P_<unsigned long long>(ctx->dcnt) + 8;  // [0] positive count, [1] total mass
  CK(cudaMemsetAsync(cnt, 0, 16, s));
  launch_keys_mass(n_local, s_score, key, s);
  launch_keep_positive(n_local, s_score, keep_out, cnt, s);  // keep = (s > 0): the num == den answer
  launch_sel_total(n_local, key, 1, cnt + 1, s);
  CKS(n_local > 0 ? launched(ctx, 3) : BGS_OK);
  unsigned long long h[2] = {0, 0};
  CK(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, s));
  CK(host_sync(ctx, s));
  CKS(sum_over_ranks(ctx, h, 2, s));
  if (num == den && h[0] > 0) return BGS_OK;  // every s > 0 is kept
  if (h[1] == 0) {
    // all-zero scores: only the forced first element (global id 0 = local 0 of rank 0)
    launch_fill_u8(n_local, keep_out, 0, s);
    CKS(n_local > 0 ? launched(ctx) : BGS_OK);
    if (ctx->rank == 0 && n_local > 0) CK(cudaMemsetAsync(keep_out, 1, 1, s));
    if (all_zero_out) *all_zero_out = 1;
    CK(host_sync(ctx, s));
    return BGS_OK;
  }
  CKS(run_select(ctx, n_local, key, 1, num, den, 0, keep_out, s));
  CK(host_sync(ctx, s));
  return BGS_OK;
}

bgs_status bgs_shard_sizes(bgs_ctx* ctx, int64_t n_local, int64_t* sizes_out) {
  CKS(check_ctx(ctx));
  if (!sizes_out || n_local < 0) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bgs_shard_sizes: arguments");
  const int M = ctx->world;
  if (M > 64) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bgs_shard_sizes: world > 64");
  std::vector<unsigned long long> sz(size_t(M), 0ull);
  sz[size_t(ctx->rank)] = (unsigned long long)n_local;
  CKS(sum_over_ranks(ctx, sz.data(), M, ctx->side ? ctx->side : nullptr));
  for (int d = 0; d < M; ++d) sizes_out[d] = int64_t(sz[size_t(d)]);
  return BGS_OK;
}

bgs_status bgs_redistribute(bgs_ctx* ctx, const bgs_gaussians* in, const uint8_t* keep, const bgs_gaussians_out* out,
                            int64_t* n_out, void* stream) {
  CKS(check_ctx(ctx));
  CKS(check_stream(ctx, stream));
  if (!in || !out || !n_out || in->n_local < 0 || (in->n_local > 0 && (!keep || !in->mean_opac || !in->quat ||
                                                                     !in->scale || !in->sh)))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bgs_redistribute: arguments");
  cudaStream_t s = as_stream(stream);
  const int M = ctx->world, rank = ctx->rank;
  const int64_t n = in->n_local;
  // every rank's shard size (one-hot sums).  The global order is gid = j M + m over slices padded
  // to the largest shard (rows j >= n_m are absent, i.e. not kept), so shards left unequal by
  // density control redistribute as well (P:170 skew-triggered rebalancing)
  if (M > 64) return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bgs_redistribute: world > 64");
  std::vector<unsigned long long> sz(size_t(M), 0ull);
  sz[size_t(rank)] = (unsigned long long)n;
  CKS(sum_over_ranks(ctx, sz.data(), M, s));
  int64_t n_max = 0;
  for (unsigned long long v : sz) n_max = std::max<int64_t>(n_max, int64_t(v));
  const int64_t N = n_max * M;
  const int64_t wpr = (n_max + 31) / 32;  // mask words per rank
  CKS(ensure(ctx, ctx->masks, size_t(std::max<int64_t>((M + 1) * wpr, 1)) * 4));
  uint32_t* masks = P_<uint32_t>(ctx->masks);
  CK(cudaMemsetAsync(masks, 0, size_t((M + 1) * wpr) * 4, s));
  int nl = 0;
  if (M == 1) {
    launch_pack_bits(n, keep, masks, s);
    nl += n > 0;
  } else {
    // allgather of the keep masks: own bits in slot M, gathered into slots [0, M)
    launch_pack_bits(n, keep, masks + size_t(M) * wpr, s);
    nl += n > 0;
    std::vector<int64_t> scnt(M, wpr), soff(M, 0), rcnt(M, wpr), roff(M);
    for (int d = 0; d < M; ++d) roff[d] = d * wpr;
    CKS(ctx->tr->alltoallv(ctx, masks + size_t(M) * wpr, scnt.data(), soff.data(), masks, rcnt.data(), roff.data(), 4,
                           s));
  }
  const int64_t nb = std::max<int64_t>(1, (N + 255) / 256);
  CKS(ensure(ctx, ctx->sblocks, size_t(nb) * 4));
  CKS(ensure(ctx, ctx->new_gid, size_t(std::max<int64_t>(n, 1)) * 4));
  CKS(ensure(ctx, ctx->dcnt, 64 * 8));
  unsigned long long* dc = P_<unsigned long long>(ctx->dcnt);
  CK(cudaMemsetAsync(dc + 16, 0, 48 * 8, s));
  uint32_t* new_gid = P_<uint32_t>(ctx->new_gid);
  launch_new_ids(N, masks, wpr, M, rank, P_<uint32_t>(ctx->sblocks), dc + 16, n, new_gid, s);
  nl += N > 0 ? 3 : 0;
  unsigned long long kept = 0;
  CK(cudaMemcpyAsync(&kept, dc + 16, 8, cudaMemcpyDeviceToHost, s));
  CK(host_sync(ctx, s));
  const int64_t nk = int64_t(kept);
  const int64_t mine = nk > rank ? (nk - rank + M - 1) / M : 0;
  *n_out = mine;
  if (mine > out->capacity) return fail(ctx, BGS_ERR_CAPACITY, "bgs_redistribute: new shard exceeds out->capacity");
  if (mine > 0 && (!out->mean_opac || !out->quat || !out->scale || !out->sh))
    return fail(ctx, BGS_ERR_INVALID_ARGUMENT, "bgs_redistribute: output arrays");
  if (M == 1) {
    launch_scatter_direct(n, new_gid, *in, *out, out->capacity, s);
    CKS(launched(ctx, nl + (n > 0)));
    CK(host_sync(ctx, s));
    return BGS_OK;
  }
  // per-destination counts -> exchange -> pack 256-B rows -> one all-to-all -> scatter
  unsigned long long* scnt_d = dc + 24;
  int64_t* rcnt_d = reinterpret_cast<int64_t*>(dc + 32);
  int64_t* base_d = reinterpret_cast<int64_t*>(dc + 40);
  unsigned long long* cursor = dc + 48;
  launch_dest_hist(n, new_gid, M, scnt_d, s);
  nl += n > 0;
  CKS(ctx->tr->alltoall1(ctx, reinterpret_cast<const int64_t*>(scnt_d), rcnt_d, s));
  std::vector<int64_t> scnt(M), rcnt(M), soff(M), roff(M);
  CK(cudaMemcpyAsync(scnt.data(), scnt_d, size_t(M) * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(rcnt.data(), rcnt_d, size_t(M) * 8, cudaMemcpyDeviceToHost, s));
  CK(host_sync(ctx, s));
  int64_t D = 0, R = 0;
  for (int d = 0; d < M; ++d) {
    soff[d] = D;
    roff[d] = R;
    D += scnt[d];
    R += rcnt[d];
  }
  if (R != mine) return fail(ctx, BGS_ERR_INTERNAL, "bgs_redistribute: received rows != new shard size");
  const size_t row = param_row_bytes();
  CKS(ensure(ctx, ctx->rows_send, size_t(std::max<int64_t>(D, 1)) * row));
  CKS(ensure(ctx, ctx->rows_recv, size_t(std::max<int64_t>(R, 1)) * row));
  CK(cudaMemcpyAsync(base_d, soff.data(), size_t(M) * 8, cudaMemcpyHostToDevice, s));
  launch_pack_rows(n, new_gid, M, base_d, cursor, *in, ctx->rows_send.p, s);
  nl += n > 0;
  CKS(ctx->tr->alltoallv(ctx, ctx->rows_send.p, scnt.data(), soff.data(), ctx->rows_recv.p, rcnt.data(), roff.data(),
                         row, s));
  launch_unpack_rows(R, ctx->rows_recv.p, *out, out->capacity, s);
  nl += R > 0;
  CKS(launched(ctx, nl));
  CK(host_sync(ctx, s));
  return BGS_OK;
}

}  // extern "C"
