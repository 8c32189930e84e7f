// tabi_api.cu -- host side of the C ABI declared in include/tabi.h.
//
// tabi_pack enqueues the whole pipeline on one stream with no host round trip
// between kernels:  [H2D] -> reset -> K1 proxies -> K2 sort -> prep (slot
// layout, area bound, raster tiles) -> fused wave kernel (K3 footprints + K3b
// pair offsets + K4 fold & push of a wave of candidates, one cooperative
// launch; split K3/K3b/K4 kernels with TABI_FUSED=0) -> [hybrid tail] -> K5
// select/scatter -> [D2H placements] + D2H status/records -> one sync.  The
// whole search is captured once as a CUDA graph and replayed: further waves
// (only when every candidate of a wave fails) run in a WHILE node whose
// condition select_kernel sets on the device -- no host round trip between
// waves.  tabi_pack_async returns right after the graph launch.
// If a device-side capacity check fails (footprint slots or lock-pair lists
// larger than the current buffers), the context grows those buffers and
// re-runs from the slot layout; sizes persist, so steady-state calls never
// retry.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <thread>
#include <vector>
#include <cstdlib>
#include <cstring>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "tabi_internal.cuh"

using namespace tabi;

// NVTX range for the host-side phases of a call (header-only NVTX3: free
// unless a profiler is attached)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

// Everything a captured first-wave graph bakes in: if any of it changes, the
// graph is re-captured.
struct GraphKey {
  const void* xy;
  const void* start;
  const void* out;
  int32_t n;
  int64_t V;
  int on_device;
  float rx, ry;
  tabi_spec spec;
  int B, fused;
  int64_t gen;
  char sort_env;  // TABI_SORT (test knob) is read at capture time
  bool operator==(const GraphKey& o) const {
    return xy == o.xy && start == o.start && out == o.out && n == o.n && V == o.V &&
           on_device == o.on_device && rx == o.rx && ry == o.ry && B == o.B && fused == o.fused &&
           gen == o.gen && sort_env == o.sort_env && memcmp(&spec, &o.spec, sizeof(tabi_spec)) == 0;
  }
};

// The arguments of a pending asynchronous pack (tabi_pack_async), kept for
// tabi_pack_wait's re-run after a capacity overflow.
struct PendArgs {
  const float* xy;
  const int32_t* start;
  int32_t n;
  float rx, ry;
  tabi_spec spec;
  tabi_placement* out;
  void* stream;
};

// Batch-mode workspace (tabi_pack_many): chart-indexed arrays for every atlas
// of the batch, per-atlas status / results, the work queue, and one set of
// per-candidate buffers per persistent CTA.  Grows to the largest batch seen.
struct ManyWs {
  int64_t cap_N = 0, cap_V = 0, cap_A = 0, cap_q = 0;
  int32_t cap_k = 0, nmax = 0, G = 0;
  int64_t col_cap = 0, row_cap = 0, pair_cap = 0;
  // chart-indexed
  float* d_xy = nullptr;          // staging for host-mode outlines (2V floats)
  int32_t* d_start = nullptr;     // staging for host-mode chart offsets (N + 1)
  int32_t* qx = nullptr;
  int32_t* qy = nullptr;
  Proxies P{};
  int32_t *perm = nullptr, *colofs = nullptr, *rowofs = nullptr, *hsorted = nullptr;
  int32_t *tstart = nullptr, *tix = nullptr;
  tabi_placement* d_out = nullptr;
  // atlas-indexed: abase (A + 1) | order (A) | res (2A floats) in one upload
  int32_t* d_small = nullptr;
  int32_t* h_small = nullptr;     // pinned
  Status* sts = nullptr;
  AtlasRes* res = nullptr;        // device; followed by nothing
  Status* h_sts = nullptr;        // pinned copies
  AtlasRes* h_res = nullptr;
  int32_t* q = nullptr;           // [cap_q] queue + [4] control words at the end
  // per persistent CTA
  uint32_t *dcol = nullptr, *drow = nullptr;
  int32_t *wd = nullptr, *hd = nullptr, *off = nullptr, *scratch = nullptr, *X = nullptr, *Y = nullptr;
  uint8_t *lock = nullptr, *mir = nullptr;
  Cand* cands = nullptr;
  int32_t* cand_bad = nullptr;
  unsigned long long* cycles = nullptr;   // [3] batch kernel phase cycles
  int64_t* area = nullptr;                // [G][nmax] lazy batch mode
  unsigned long long h_cycles[3] = {0, 0, 0};
  int64_t cycles_cap = 0;
  std::vector<unsigned long long> h_cta;  // per CTA: start, last item end (ns)
  int32_t* solo_start = nullptr;  // rebased chart offsets of a solo atlas (device mode)
  // pinned host staging for host-mode inputs / outputs
  float* h_xy = nullptr;          // 2V floats + N + 1 ints
  int64_t h_cap = 0;
  tabi_placement* h_out = nullptr;
  int64_t h_out_cap = 0;
  cudaEvent_t span[2] = {nullptr, nullptr};
  cudaEvent_t stage[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // TABI_TIMING
  cudaStream_t copy_stream = nullptr;  // host mode: chunked outline upload
  cudaEvent_t chunk_ev[9] = {};
  void release() {
    void* ds[] = {d_xy, d_start, qx, qy, P.w, P.h, P.area2, P.xmin, P.ymin, P.pose, P.prerot, P.sl,
                  P.obb_j, P.obb, perm, colofs, rowofs, hsorted, tstart, tix, d_out, d_small, sts,
                  res, q, dcol, drow, wd, hd, off, scratch, X, Y, lock, mir, cands, cand_bad,
                  solo_start, cycles, area};
    for (void* p : ds)
      if (p) cudaFree(p);
    void* hs[] = {h_small, h_sts, h_res, h_xy, h_out};
    for (void* p : hs)
      if (p) cudaFreeHost(p);
    for (auto& e : span)
      if (e) cudaEventDestroy(e);
    for (auto& e : stage)
      if (e) cudaEventDestroy(e);
    for (auto& e : chunk_ev)
      if (e) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
  }
};

struct tabi_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int32_t max_n = 0;
  int64_t max_v = 0;
  int32_t max_side = 0;
  // inputs / proxies
  float* d_xy = nullptr;
  int32_t* d_start = nullptr;
  int32_t* d_qx = nullptr;
  int32_t* d_qy = nullptr;
  Proxies P{};
  uint64_t* keys = nullptr;
  uint64_t* keys2 = nullptr;
  int32_t* perm = nullptr;
  int32_t* perm2 = nullptr;
  int32_t* colofs = nullptr;
  int32_t* rowofs = nullptr;
  int32_t* hsorted = nullptr;
  const uint64_t* sorted_keys = nullptr;  // keys in sorted order (chunked sort), else nullptr
  PrepSync* prep_sync = nullptr;          // multi-CTA slot layout's look-back state (zeroed once)
  tabi_placement* d_out = nullptr;
  Status* d_status = nullptr;
  Status* h_status = nullptr;  // pinned
  // per-candidate buffers (sized for cand_M candidates)
  int32_t cand_M = 0;
  int32_t* wd = nullptr;
  int32_t* hd = nullptr;
  int32_t* off = nullptr;
  uint8_t* lockbits = nullptr;
  int32_t* cand_bad = nullptr;
  int32_t* big_list = nullptr;  // (candidate, chart) items too large for K3's tile buffer
  int32_t* rdy = nullptr;       // fused kernel: per (wave slot, tile) ready flags
  int32_t* tstart = nullptr;    // fused kernel: raster tile boundaries [N + 1]
  int32_t* tix = nullptr;       // fused kernel: tile of each sorted position [N]
  // hybrid prefix tail state per candidate
  int32_t* t_state = nullptr;
  int32_t* t_r0 = nullptr;
  int32_t* t_p = nullptr;
  int32_t* t_iter = nullptr;
  int32_t* t_fsave = nullptr;
  int32_t fstride = 0;
  int32_t* X = nullptr;
  int32_t* Y = nullptr;
  uint8_t* mir = nullptr;
  Cand* cands = nullptr;
  Cand* h_cands = nullptr;  // pinned
  uint32_t* dcol = nullptr;
  uint32_t* drow = nullptr;
  int64_t col_cap = 0, row_cap = 0;  // entries per candidate
  int32_t* scratch = nullptr;
  int64_t pair_cap = 0;
  // pinned host staging
  float* h_xy = nullptr;
  int32_t* h_start = nullptr;
  tabi_placement* h_out = nullptr;
  // last pack (introspection)
  int32_t last_n = 0, last_M = 0, last_k = 0, last_g = 0, last_fused = 0;
  std::string err;
  // first-wave CUDA graph (tabi_pack) and the buffer generation it was captured on
  cudaGraphExec_t gexec = nullptr;
  GraphKey gkey{};
  int g_launches = 0;
  int64_t alloc_gen = 0;
  cudaError_t last_cuda = cudaSuccess;
  bool fused_off = false;  // the cooperative launch was refused once: split kernels from now on
  Validator val;           // tabi_validate scratch (N3)
  cudaEvent_t span[2] = {nullptr, nullptr};  // tabi_info.device_ms
  ManyWs many;             // tabi_pack_many
  cudaStream_t cap_stream = nullptr;  // captures the graph's wave-loop body
  cudaStream_t cap_stream2 = nullptr; // captures the hybrid tail's rounds-loop body
  cudaStream_t fork_stream = nullptr; // proxy_kernel beside the sizes -> sort -> slot layout chain
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int g_body = 0;                     // kernels per wave of the graph's loop body
  bool loop_off = false;              // the graph's device wave loop failed once
  bool pend = false;                  // an asynchronous pack is in flight
  PendArgs pend_args{};
};

#define CK(call)                                              \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) {                                  \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_); \
      ctx->last_cuda = e_;                                    \
      return TABI_ECUDA;                                      \
    }                                                         \
  } while (0)

constexpr size_t kStatusPad = (sizeof(Status) + 63) & ~(size_t)63;

template <class T>
static cudaError_t dalloc(T** p, size_t count) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  return cudaMalloc((void**)p, sizeof(T) * (count ? count : 1));
}

static void dfree_all(tabi_ctx* ctx) {
  void* ps[] = {ctx->d_xy, ctx->d_start, ctx->d_qx, ctx->d_qy, ctx->P.w, ctx->P.h, ctx->P.area2,
                ctx->P.xmin, ctx->P.ymin, ctx->P.pose, ctx->P.prerot, ctx->P.sl, ctx->P.obb_j, ctx->P.obb,
                ctx->keys, ctx->keys2, ctx->perm, ctx->perm2, ctx->colofs, ctx->rowofs,
                ctx->hsorted, ctx->d_out, ctx->d_status, ctx->prep_sync, ctx->wd, ctx->hd, ctx->off,
                ctx->lockbits, ctx->cand_bad, ctx->big_list, ctx->rdy, ctx->tstart, ctx->tix, ctx->X, ctx->Y, ctx->mir,
                ctx->dcol, ctx->t_state, ctx->t_r0, ctx->t_p, ctx->t_iter,
                ctx->t_fsave,
                ctx->drow, ctx->scratch};  // cands / h_cands live inside the status blocks
  for (void* p : ps)
    if (p) cudaFree(p);
  ctx->val.release();
  ctx->many.release();
  for (auto& e : ctx->span)
    if (e) cudaEventDestroy(e);
  void* hs[] = {ctx->h_status, ctx->h_xy, ctx->h_start, ctx->h_out};
  for (void* p : hs)
    if (p) cudaFreeHost(p);
}

extern "C" const char* tabi_status_str(tabi_status s) {
  switch (s) {
    case TABI_OK: return "ok";
    case TABI_EINVAL: return "invalid argument";
    case TABI_NO_FIT: return "no candidate scale fits";
    case TABI_ECUDA: return "CUDA error";
    case TABI_ECAPACITY: return "capacity exceeded";
    case TABI_PENDING: return "pending";
  }
  return "unknown";
}

extern "C" const char* tabi_last_error(tabi_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

extern "C" tabi_status tabi_ctx_create(tabi_ctx** out, int cuda_device, int32_t max_charts,
                                       int64_t max_vertices, int32_t max_atlas_side) {
  if (!out || max_charts < 1 || max_vertices < 3 || max_atlas_side < 1 ||
      max_atlas_side > TABI_MAX_ATLAS_SIDE)
    return TABI_EINVAL;
  tabi_ctx* ctx = new tabi_ctx();
  *out = nullptr;
  ctx->device = cuda_device;
  ctx->max_n = max_charts;
  ctx->max_v = max_vertices;
  ctx->max_side = max_atlas_side;
  auto fail = [&]() {
    dfree_all(ctx);
    delete ctx;
    return TABI_ECUDA;
  };
  if (cudaSetDevice(cuda_device) != cudaSuccess) return fail();
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) return fail();
  if (cudaStreamCreateWithFlags(&ctx->fork_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess)
    return fail();
  if (cudaEventCreate(&ctx->span[0]) != cudaSuccess || cudaEventCreate(&ctx->span[1]) != cudaSuccess)
    return fail();
  const size_t N = (size_t)max_charts, V = (size_t)max_vertices;
  // d_xy / h_xy: outline (2V floats) followed by the chart offsets (N + 1 ints)
  bool ok = dalloc(&ctx->d_xy, 2 * V + N + 1) == cudaSuccess &&
            dalloc(&ctx->d_start, 1) == cudaSuccess &&
            dalloc(&ctx->d_qx, V) == cudaSuccess && dalloc(&ctx->d_qy, V) == cudaSuccess &&
            dalloc(&ctx->P.w, N) == cudaSuccess && dalloc(&ctx->P.h, N) == cudaSuccess &&
            dalloc(&ctx->P.area2, N) == cudaSuccess && dalloc(&ctx->P.xmin, N) == cudaSuccess &&
            dalloc(&ctx->P.ymin, N) == cudaSuccess && dalloc(&ctx->P.pose, N) == cudaSuccess &&
            dalloc(&ctx->P.prerot, N) == cudaSuccess &&
            dalloc(&ctx->P.sl, N * 4 * TABI_KMAX) == cudaSuccess &&
            dalloc(&ctx->P.obb_j, N) == cudaSuccess && dalloc(&ctx->P.obb, 4 * N) == cudaSuccess &&
            dalloc(&ctx->keys, N) == cudaSuccess && dalloc(&ctx->keys2, N) == cudaSuccess &&
            dalloc(&ctx->perm, N) == cudaSuccess && dalloc(&ctx->perm2, N) == cudaSuccess &&
            dalloc(&ctx->colofs, N) == cudaSuccess && dalloc(&ctx->rowofs, N) == cudaSuccess &&
            dalloc(&ctx->hsorted, N) == cudaSuccess && dalloc(&ctx->d_out, N) == cudaSuccess &&
            dalloc(&ctx->tstart, N + 1) == cudaSuccess && dalloc(&ctx->tix, N) == cudaSuccess &&
            dalloc(&ctx->d_status, 1) == cudaSuccess && dalloc(&ctx->prep_sync, 1) == cudaSuccess &&
            cudaMemset(ctx->prep_sync, 0, sizeof(PrepSync)) == cudaSuccess;
  if (!ok) return fail();
  if (cudaMallocHost((void**)&ctx->h_status, sizeof(Status)) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->h_xy, sizeof(float) * (2 * V + N + 1)) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->h_start, sizeof(int32_t)) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->h_out, sizeof(tabi_placement) * N) != cudaSuccess)
    return fail();
  // initial footprint slot capacity per candidate (grows on demand)
  ctx->col_cap = ((int64_t)N * 96 + 4 * (int64_t)max_atlas_side) & ~(int64_t)3;  // 16-B aligned per candidate
  ctx->row_cap = ctx->col_cap;
  ctx->pair_cap = (int64_t)N * 2 + 1024;
  *out = ctx;
  return TABI_OK;
}

extern "C" void tabi_ctx_destroy(tabi_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  dfree_all(ctx);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->cap_stream2) cudaStreamDestroy(ctx->cap_stream2);
  if (ctx->fork_stream) cudaStreamDestroy(ctx->fork_stream);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  delete ctx;
}

static tabi_status ensure_candidates(tabi_ctx* ctx, int32_t M, bool regrow_cols, bool regrow_pairs) {
  const size_t N = (size_t)ctx->max_n;
  if (M > ctx->cand_M) {
    CK(dalloc(&ctx->wd, (size_t)M * N));
    CK(dalloc(&ctx->hd, (size_t)M * N));
    CK(dalloc(&ctx->off, (size_t)M * N));
    CK(dalloc(&ctx->lockbits, (size_t)M * N));
    CK(dalloc(&ctx->cand_bad, (size_t)M));
    CK(dalloc(&ctx->big_list, (size_t)M * N));
    // ready flags + boundary arrival counters + per-slot completed-tile counts
    CK(dalloc(&ctx->rdy, 2 * (size_t)M * N + 2 * (size_t)M));
    ctx->fstride = ((ctx->max_side + 2 * 64 + 4) + 31) & ~31;
    CK(dalloc(&ctx->t_state, (size_t)M));
    CK(dalloc(&ctx->t_r0, (size_t)M));
    CK(dalloc(&ctx->t_p, (size_t)M));
    CK(dalloc(&ctx->t_iter, (size_t)M));
    CK(dalloc(&ctx->t_fsave, (size_t)M * ctx->fstride));
    CK(dalloc(&ctx->X, (size_t)M * N));
    CK(dalloc(&ctx->Y, (size_t)M * N));
    CK(dalloc(&ctx->mir, (size_t)M * N));
    // status block and candidate records in ONE allocation (device and pinned
    // host) so a wave's results come back with a single D2H copy
    {
      const size_t bytes = kStatusPad + sizeof(Cand) * (size_t)M;
      cudaFree(ctx->d_status);
      ctx->d_status = nullptr;
      CK(cudaMalloc((void**)&ctx->d_status, bytes));
      ctx->cands = (Cand*)((char*)ctx->d_status + kStatusPad);
      cudaFreeHost(ctx->h_status);
      ctx->h_status = nullptr;
      CK(cudaMallocHost((void**)&ctx->h_status, bytes));
      ctx->h_cands = (Cand*)((char*)ctx->h_status + kStatusPad);
    }
    regrow_cols = regrow_pairs = true;
    ctx->cand_M = M;
  }
  if (regrow_cols || regrow_pairs) ctx->alloc_gen++;  // captured graphs hold stale pointers
  const int32_t Mc = ctx->cand_M;
  if (regrow_cols) {
    CK(dalloc(&ctx->dcol, (size_t)Mc * ctx->col_cap));
    CK(dalloc(&ctx->drow, (size_t)Mc * ctx->row_cap));
  }
  if (regrow_pairs) CK(dalloc(&ctx->scratch, (size_t)Mc * (6 * N + 3 * (size_t)ctx->pair_cap)));
  return TABI_OK;
}

// A wave hit the device-side capacity check: grow the footprint slots and / or
// the lock-pair lists to what it reported (with headroom; sizes persist).
static tabi_status grow_for(tabi_ctx* ctx, const Status& st, int32_t M) {
  bool cols = false, pairs = false;
  if (st.capacity & 1) {
    ctx->col_cap = ((int64_t)st.cols_total + (st.cols_total >> 2) + 1024) & ~(int64_t)3;
    ctx->row_cap = ((int64_t)st.rows_total + (st.rows_total >> 2) + 1024) & ~(int64_t)3;
    cols = true;
  }
  if (st.capacity & 2) {
    ctx->pair_cap = (int64_t)st.pad[0] * 2 + 1024;
    pairs = true;
  }
  return ensure_candidates(ctx, M, cols, pairs);
}

static bool spec_ok(const tabi_spec* s) {
  return s && s->atlas_w >= 1 && s->atlas_h >= 1 && s->atlas_w <= TABI_MAX_ATLAS_SIDE &&
         s->atlas_h <= TABI_MAX_ATLAS_SIDE && s->gutter >= 0 && s->gutter <= 64 &&
         s->scale_count >= 1 && s->scale_count <= TABI_MAX_SCALES && s->local_aabb_count >= 1 &&
         s->local_aabb_count <= TABI_MAX_LOCAL_AABBS && s->t_opt_bp >= -1 &&
         s->t_opt_bp <= 10000 && (s->flags & ~63u) == 0;
}

namespace {
struct Timer {
  bool on = false;
  cudaEvent_t ev[9];
  int n = 0;
  void init(bool enable) {
    on = enable;
    if (on)
      for (auto& e : ev) cudaEventCreate(&e);
  }
  void mark(cudaStream_t s) {
    if (on && n < 9) cudaEventRecord(ev[n++], s);
  }
  void finish(tabi_info* info) {
    if (!on) return;
    cudaEventSynchronize(ev[n - 1]);
    for (int i = 0; i + 1 < n && i < 8; i++) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      if (info) info->stage_ms[i] = ms;
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
};
}  // namespace

static tabi_status pack_impl(tabi_ctx* ctx, const float* xy, const int32_t* chart_start,
                             int32_t n, float res_x, float res_y, const tabi_spec* spec,
                             tabi_placement* out, tabi_info* info, int on_device, void* stream,
                             bool async = false);
static tabi_status finish_pack(tabi_ctx* ctx, int32_t n, int32_t M, int32_t k, int32_t g,
                               int on_device, tabi_placement* out, tabi_info* info, int launches,
                               Timer& tm);

extern "C" tabi_status tabi_pack(tabi_ctx* ctx, const float* xy, const int32_t* chart_start,
                                 int32_t n, float res_x, float res_y, const tabi_spec* spec,
                                 tabi_placement* out, tabi_info* info, int on_device,
                                 void* stream) {
  Nvtx nv_("tabi_pack");
  if (!ctx) return TABI_EINVAL;
  if (ctx->pend) {
    ctx->err = "an asynchronous pack is pending on this context (tabi_pack_wait first)";
    return TABI_EINVAL;
  }
  ctx->last_cuda = cudaSuccess;
  tabi_status st = pack_impl(ctx, xy, chart_start, n, res_x, res_y, spec, out, info, on_device,
                             stream);
  if (st == TABI_ECUDA && ctx->last_cuda == cudaErrorCooperativeLaunchTooLarge && !ctx->fused_off) {
    // the GPU cannot hold the fused wave kernel's grid right now (shared
    // device, MPS limits): same result from the split kernels
    cudaGetLastError();
    ctx->fused_off = true;
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
    st = pack_impl(ctx, xy, chart_start, n, res_x, res_y, spec, out, info, on_device, stream);
  }
  return st;
}

extern "C" tabi_status tabi_pack_async(tabi_ctx* ctx, const float* xy, const int32_t* chart_start,
                                       int32_t n, float res_x, float res_y, const tabi_spec* spec,
                                       tabi_placement* out, void* stream) {
  Nvtx nv_("tabi_pack_async");
  if (!ctx) return TABI_EINVAL;
  if (ctx->pend) {
    ctx->err = "an asynchronous pack is already pending on this context";
    return TABI_EINVAL;
  }
  ctx->last_cuda = cudaSuccess;
  return pack_impl(ctx, xy, chart_start, n, res_x, res_y, spec, out, nullptr, 1, stream, true);
}

extern "C" tabi_status tabi_pack_query(tabi_ctx* ctx) {
  if (!ctx || !ctx->pend) return TABI_EINVAL;
  const cudaError_t e = cudaEventQuery(ctx->span[1]);
  if (e == cudaErrorNotReady) return TABI_PENDING;
  if (e != cudaSuccess) {
    ctx->err = std::string("cudaEventQuery: ") + cudaGetErrorString(e);
    return TABI_ECUDA;
  }
  return TABI_OK;
}

extern "C" tabi_status tabi_pack_wait(tabi_ctx* ctx, tabi_info* info) {
  Nvtx nv_("tabi_pack_wait");
  if (!ctx || !ctx->pend) return TABI_EINVAL;
  ctx->pend = false;
  const PendArgs a = ctx->pend_args;
  if (info) {
    memset(info, 0, sizeof(*info));
    info->bad_chart = -1;
    info->fused = ctx->last_fused;
  }
  CK(cudaEventSynchronize(ctx->span[1]));
  const Status st = *ctx->h_status;
  if (st.bad_chart != INT32_MAX) {
    if (info) info->bad_chart = st.bad_chart;
    return TABI_EINVAL;
  }
  if (st.capacity & 4) return TABI_ECAPACITY;
  if (st.capacity) {  // grow, then the same pack synchronously
    const tabi_status ts = grow_for(ctx, st, a.spec.scale_count);
    if (ts != TABI_OK) return ts;
    return tabi_pack(ctx, a.xy, a.start, a.n, a.rx, a.ry, &a.spec, a.out, info, 1, a.stream);
  }
  const int launches = ctx->g_launches + ctx->g_body * st.wave + 4 * st.rounds_run;
  Timer tm;
  return finish_pack(ctx, a.n, a.spec.scale_count, a.spec.local_aabb_count, a.spec.gutter, 1, a.out,
                     info, launches, tm);
}

extern "C" tabi_status tabi_validate(tabi_ctx* ctx, const float* xy, const int32_t* chart_start,
                                     int32_t n, float res_x, float res_y, int32_t W, int32_t H,
                                     int32_t g, const tabi_placement* placements,
                                     tabi_validation* out, int on_device, void* stream) {
  Nvtx nv_("tabi_validate");
  if (!ctx || !out) return TABI_EINVAL;
  memset(out, 0, sizeof(*out));
  out->bad_chart = -1;
  if (!xy || !chart_start || !placements || n < 1 || W < 1 || H < 1 || W > 65536 ||
      H > 65536 || g < 0 || g > 64)
    return TABI_EINVAL;
  if (n > ctx->max_n) return TABI_ECAPACITY;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
  int64_t V = 0;
  if (on_device) {
    int32_t v = 0;
    CK(cudaMemcpyAsync(&v, chart_start + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    V = v;
  } else {
    V = chart_start[n];
    for (int32_t c = 0; c < n; c++)
      if (chart_start[c + 1] - chart_start[c] < 3) {
        out->bad_chart = c;
        return TABI_EINVAL;
      }
  }
  if (V < 3) return TABI_EINVAL;
  int launches = 0;
  const int st = ctx->val.run(xy, chart_start, n, res_x, res_y, W, H, g, placements,
                              on_device != 0, V, s, out, &launches, &ctx->err);
  out->gpu_launches = launches;
  return (tabi_status)st;
}

static tabi_status pack_impl(tabi_ctx* ctx, const float* xy, const int32_t* chart_start,
                             int32_t n, float res_x, float res_y, const tabi_spec* spec,
                             tabi_placement* out, tabi_info* info, int on_device, void* stream,
                             bool async) {
  if (!ctx) return TABI_EINVAL;
  if (info) {
    memset(info, 0, sizeof(*info));
    info->bad_chart = -1;
  }
  if (!xy || !chart_start || !out || n < 1 || !spec_ok(spec)) return TABI_EINVAL;
  if (n > ctx->max_n || spec->atlas_w > ctx->max_side || spec->atlas_h > ctx->max_side)
    return TABI_ECAPACITY;
  // D23 policy: t_opt = 0 for <= 10,000 charts, 1 % of H above
  const int32_t t_opt = spec->t_opt_bp >= 0 ? spec->t_opt_bp : (n > 10000 ? 100 : 0);
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
  int launches = 0;
  Timer tm;
  const char* tenv = getenv("TABI_TIMING");
  tm.init(tenv && tenv[0] == '1');
  tm.mark(s);

  const float* d_xy = xy;
  const int32_t* d_start = chart_start;
  if (!on_device) {
    const int64_t V = chart_start[n];
    if (chart_start[0] != 0 || V < 3) {
      if (info) info->bad_chart = 0;
      return TABI_EINVAL;
    }
    for (int32_t c = 0; c < n; c++)
      if (chart_start[c + 1] - chart_start[c] < 3) {
        if (info) info->bad_chart = c;
        return TABI_EINVAL;
      }
    if (V > ctx->max_v) return TABI_ECAPACITY;
    // outline and chart offsets staged back to back: one H2D copy (enqueued
    // with the first wave)
    memcpy(ctx->h_xy, xy, sizeof(float) * 2 * V);
    memcpy(ctx->h_xy + 2 * V, chart_start, sizeof(int32_t) * (n + 1));
    d_xy = ctx->d_xy;
    d_start = (const int32_t*)(ctx->d_xy + 2 * V);
  }
  tm.mark(s);
  const int32_t M = spec->scale_count;
  tabi_status ts = ensure_candidates(ctx, M, false, false);
  if (ts != TABI_OK) return ts;

  PackParams pp;
  pp.n = n;
  pp.k = spec->local_aabb_count;
  pp.M = M;
  pp.g = spec->gutter;
  pp.W = spec->atlas_w;
  pp.H = spec->atlas_h;
  pp.Wp = spec->atlas_w + 2 * spec->gutter;
  pp.Hp = spec->atlas_h + 2 * spec->gutter;
  pp.flags = spec->flags;
  pp.t_opt = t_opt;
  pp.mode = 0;
  pp.tail = 0;
  pp.early = t_opt == 0 ? 1 : 0;  // sequential: the smallest successful slot wins outright
  pp.T.state = ctx->t_state;
  pp.T.r0 = ctx->t_r0;
  pp.T.p = ctx->t_p;
  pp.T.iter = ctx->t_iter;
  pp.T.fsave = ctx->t_fsave;
  pp.T.fstride = ctx->fstride;

  // Candidate waves: prep_kernel computes the area
  // bound m_hi (every m above it must fail); wave w evaluates m_hi - w*B - j,
  // j < B, all in parallel.  The first wave containing a success holds the
  // largest successful m, so later waves are skipped -- the result equals the
  // exhaustive search.  A further wave costs one host round trip.
  const char* wenv = getenv("TABI_WAVE");
  int B = wenv ? atoi(wenv) : 16;
  if (B < 1 || B > M) B = M;
  pp.B = B;
  // fused wave kernel: needs B packer CTAs plus rasterizer CTAs co-resident
  const char* fenv = getenv("TABI_FUSED");
  const int fgrid = fused_grid(ctx->device);
  const bool fused = !(fenv && fenv[0] == '0') && !ctx->fused_off && fgrid >= B + 8 &&
                     fused_fits(pp.k);
  if (info) info->fused = fused ? 1 : 0;
  ctx->last_fused = fused ? 1 : 0;
  // ready flags + arrival counters + per-slot completed-tile counts + per-slot
  // "failed" flags (rasterizers drop a failed candidate's remaining tiles)
  const int64_t nrdy = fused ? 2 * (int64_t)B * n + 2 * B : 0;

  tabi_placement* d_out = on_device ? out : ctx->d_out;
  const int64_t V_in = on_device ? 0 : (int64_t)chart_start[n];
  int wave = 0;
  // The pack is enqueued in three parts on s:
  //  prologue  [H2D] + fresh status + proxies + sort + slot layout (full), or
  //            fresh status + slot layout only (a capacity retry keeps the
  //            proxies and the order);
  //  body      one candidate wave: [reset] + the fused wave kernel (or the
  //            split K3/K3b/K4 kernels) + [hybrid tail] + select;
  //  epilogue  [D2H placements] + D2H status and candidate records.
  // Append a WHILE node with condition h to the graph being captured on
  // stream sm (after everything captured so far); returns its body graph.
  auto add_while = [&](cudaStream_t sm, cudaGraphConditionalHandle h,
                       cudaGraph_t& body) -> cudaError_t {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaGraph_t cg = nullptr;
    cudaError_t ce = cudaStreamGetCaptureInfo(sm, &cs, nullptr, &cg, &deps, &ndeps);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn = nullptr;
    if (ce == cudaSuccess) ce = cudaGraphAddNode(&cn, cg, deps, ndeps, &cp);
    if (ce == cudaSuccess)
      ce = cudaStreamUpdateCaptureDependencies(sm, &cn, 1, cudaStreamSetCaptureDependencies);
    body = ce == cudaSuccess ? cp.conditional.phGraph_out[0] : nullptr;
    return ce;
  };
  auto enqueue_prologue = [&](bool full, int& nl) -> tabi_status {
    bool prep_done = false;
    if (full && !on_device)
      CK(cudaMemcpyAsync(ctx->d_xy, ctx->h_xy, sizeof(float) * 2 * V_in + sizeof(int32_t) * (n + 1),
                         cudaMemcpyHostToDevice, s));
    // (prep_kernel zeroes the fused kernel's flags for the T tiles it lays out)
    launch_reset(ctx->d_status, 2, ctx->cands, ctx->t_state, ctx->cand_bad, M, ctx->rdy, 0, s);
    nl++;
    // Fork: the order and the slot layout need only w, h and the area
    // (sizes_kernel), so they run while proxy_kernel computes the slices and
    // OBBs on a second stream (joined before the candidate waves); not with
    // the prerotation (its w, h follow the OBB angle) or under TABI_TIMING
    // (stage times stay sequential).  Above 4096 charts only: measured C4
    // (20,000 charts) 1.141 -> 1.129 ms, while C3 (1,572) and C2 (214) gained
    // nothing (the graph's fork / join costs what the shorter chain saves).
    // TABI_PROXY_FORK=0 / 1: test knob (off / on at any size).
    const char* fenv2 = getenv("TABI_PROXY_FORK");
    const bool fork = full && !(pp.flags & TABI_F_PREROTATE) && !tm.on &&
                      (fenv2 ? fenv2[0] == '1' : n > 4096);
    if (full) {
      ctx->sorted_keys = nullptr;  // (set by launch_sort when its ranks write them)
      if (fork) {
        CK(cudaEventRecord(ctx->ev_fork, s));
        CK(cudaStreamWaitEvent(ctx->fork_stream, ctx->ev_fork, 0));
        launch_proxies(d_xy, d_start, n, res_x, res_y, pp.k, pp.flags, ctx->d_qx, ctx->d_qy,
                       ctx->max_v, ctx->P, ctx->d_status, ctx->fork_stream,
                       AtlasMap{nullptr, 1, nullptr}, V_in, true);
        launch_sizes(d_xy, d_start, n, res_x, res_y, ctx->max_v, ctx->P, ctx->d_status, s);
        nl += 2;
      } else {
        launch_proxies(d_xy, d_start, n, res_x, res_y, pp.k, pp.flags,
                       ctx->d_qx, ctx->d_qy, ctx->max_v, ctx->P, ctx->d_status, s,
                       AtlasMap{nullptr, 1, nullptr}, V_in);
        nl++;
      }
      tm.mark(s);
      if (launch_sort_prep(ctx->P, ctx->perm, pp, ctx->colofs, ctx->rowofs, ctx->hsorted,
                           ctx->tstart, ctx->tix, ctx->d_status, fused ? ctx->rdy : nullptr, s)) {
        nl++;
        prep_done = true;
      } else {
        nl += launch_sort(ctx->P, n, ctx->keys, ctx->keys2, ctx->perm, ctx->perm2, ctx->d_status, s,
                          &ctx->sorted_keys);
      }
      tm.mark(s);
    }
    if (!prep_done) {
      launch_prep(ctx->P, ctx->perm, pp, ctx->colofs, ctx->rowofs, ctx->hsorted, ctx->tstart,
                  ctx->tix, ctx->d_status, fused ? ctx->rdy : nullptr, s, ctx->sorted_keys,
                  ctx->prep_sync);
      nl++;
    }
    if (fork) {  // join: the waves need the slices and OBBs
      CK(cudaEventRecord(ctx->ev_join, ctx->fork_stream));
      CK(cudaStreamWaitEvent(s, ctx->ev_join, 0));
    }
    return TABI_OK;
  };
  // reset_mode: -1 none (wave 0 after the prologue), 0 the next wave; with
  // use_h, select also sets the graph's wave-loop condition h
  auto enqueue_body = [&](int reset_mode, int& nl, cudaGraphConditionalHandle h,
                          int use_h) -> tabi_status {
    if (reset_mode >= 0) {
      launch_reset(ctx->d_status, reset_mode, ctx->cands, ctx->t_state, ctx->cand_bad, M, ctx->rdy,
                   nrdy, s);
      nl++;
    }
    if (fused) {
      // K3 + K3b + K4 as one cooperative persistent launch
      tm.mark(s);
      tm.mark(s);
      CK(launch_fused(fgrid, ctx->P, ctx->perm, pp, ctx->colofs, ctx->rowofs, ctx->dcol,
                      ctx->drow, ctx->wd, ctx->hd, ctx->off, ctx->lockbits, ctx->hsorted,
                      ctx->cand_bad, ctx->rdy, ctx->tstart, ctx->tix, ctx->scratch, ctx->pair_cap, ctx->X, ctx->Y,
                      ctx->mir, ctx->cands, ctx->d_status, s));
      nl++;
    } else {
      launch_profiles(ctx->P, ctx->perm, pp, ctx->colofs, ctx->rowofs, (int16_t*)ctx->dcol,
                      (int16_t*)ctx->drow, ctx->wd, ctx->hd, ctx->cand_bad, ctx->big_list,
                      ctx->d_status, s);
      nl += 2;  // K3 tiles, K3 large charts
      tm.mark(s);
      launch_offsets(pp, ctx->colofs, ctx->rowofs, (const int16_t*)ctx->drow, ctx->wd, ctx->hd,
                     ctx->off, ctx->lockbits, ctx->cand_bad, ctx->d_status, s);
      nl++;
      tm.mark(s);
      launch_pack(pp, ctx->colofs, ctx->rowofs, ctx->dcol, ctx->drow, ctx->wd, ctx->hd, ctx->off,
                  ctx->lockbits, ctx->hsorted, ctx->cand_bad, ctx->scratch, ctx->pair_cap, ctx->X,
                  ctx->Y, ctx->mir, ctx->cands, ctx->d_status, s);
      nl++;
    }
    if (t_opt > 0) {
      // hybrid prefix tail for the candidates K4 switched: rows and
      // sigma, then re-rasterize / re-lay rounds until every row fits (at most
      // 9), then the prefix rows.  In the graph the rounds are a WHILE node
      // whose condition the last CTA of tail_prepare / tail_layout sets, so
      // they stop at the round that fits; the host-driven loop enqueues 9
      // (the kernels of a finished candidate exit at once).
      PackParams pt = pp;
      pt.tail = 1;
      // (the exact tail, R6, keeps the footprints at m/M: no re-rasterization)
      const bool exact = (pp.flags & TABI_F_EXACT_TAIL) != 0;
      const bool rloop = use_h && !exact;
      cudaGraphConditionalHandle hr = 0;
      if (rloop) {
        cudaStreamCaptureStatus cs;
        cudaGraph_t cg = nullptr;
        CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, nullptr, nullptr));
        CK(cudaGraphConditionalHandleCreate(&hr, cg, 0, cudaGraphCondAssignDefault));
      }
      launch_tail_prepare(pp, ctx->perm, ctx->P.area2, ctx->wd, ctx->off, ctx->scratch,
                          ctx->pair_cap, ctx->cands, ctx->d_status, s, hr, rloop ? 1 : 0);
      nl++;
      auto round = [&](int use_r) -> tabi_status {
        CK(cudaMemsetAsync(&ctx->d_status->pad[1], 0, sizeof(int32_t), s));
        launch_profiles(ctx->P, ctx->perm, pt, ctx->colofs, ctx->rowofs, (int16_t*)ctx->dcol,
                        (int16_t*)ctx->drow, ctx->wd, ctx->hd, ctx->cand_bad, ctx->big_list,
                        ctx->d_status, s);
        launch_offsets(pt, ctx->colofs, ctx->rowofs, (const int16_t*)ctx->drow, ctx->wd, ctx->hd,
                       ctx->off, ctx->lockbits, ctx->cand_bad, ctx->d_status, s);
        launch_tail_layout(pt, ctx->wd, ctx->off, ctx->scratch, ctx->pair_cap, ctx->d_status, s, hr,
                           use_r);
        return TABI_OK;
      };
      if (rloop) {
        if (!ctx->cap_stream2) CK(cudaStreamCreateWithFlags(&ctx->cap_stream2, cudaStreamNonBlocking));
        const cudaStream_t ms = s;
        cudaGraph_t body = nullptr;
        CK(add_while(s, hr, body));
        s = ctx->cap_stream2;
        cudaError_t ce = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                                       cudaStreamCaptureModeThreadLocal);
        tabi_status es = TABI_OK;
        if (ce == cudaSuccess) {
          es = round(1);
          cudaGraph_t bg = nullptr;
          const cudaError_t e2 = cudaStreamEndCapture(s, &bg);
          if (ce == cudaSuccess) ce = e2;
        }
        s = ms;
        if (es != TABI_OK) return es;
        CK(ce);
        // (the rounds' 4 kernels each are counted from Status::rounds_run)
      } else {
        const int rounds = exact ? 0 : 9;
        for (int r = 0; r < rounds; r++) {
          const tabi_status es = round(0);
          if (es != TABI_OK) return es;
          nl += 4;
        }
      }
      PackParams pm = pp;
      pm.mode = 1;
      launch_pack(pm, ctx->colofs, ctx->rowofs, ctx->dcol, ctx->drow, ctx->wd, ctx->hd, ctx->off,
                  ctx->lockbits, ctx->hsorted, ctx->cand_bad, ctx->scratch, ctx->pair_cap, ctx->X,
                  ctx->Y, ctx->mir, ctx->cands, ctx->d_status, s);
      nl++;
    }
    tm.mark(s);
    launch_select(pp, ctx->P, ctx->perm, ctx->wd, ctx->hd, ctx->X, ctx->Y, ctx->mir, ctx->cands,
                  d_out, ctx->d_status, s, h, use_h);
    nl++;
    tm.mark(s);
    CK(cudaGetLastError());
    return TABI_OK;
  };
  auto enqueue_epilogue = [&]() -> tabi_status {
    if (!on_device)  // placements (valid if some wave held the winner)
      CK(cudaMemcpyAsync(ctx->h_out, ctx->d_out, sizeof(tabi_placement) * n, cudaMemcpyDeviceToHost,
                         s));
    // status + candidate records: one contiguous block, one copy
    CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, kStatusPad + sizeof(Cand) * M,
                       cudaMemcpyDeviceToHost, s));
    return TABI_OK;
  };

  // The common case runs as ONE CUDA graph, captured once per (pointers,
  // sizes, spec, buffer generation) and relaunched with one call: the
  // prologue, candidate wave 0, a WHILE node whose body is one further wave,
  // and the epilogue.  Each wave's select_kernel decides on the device
  // whether another wave is needed (it sets the node's condition), so a
  // multi-wave scale search has no host round trip and the host syncs once;
  // in the common case the loop body never runs.  Test knobs (TABI_GRAPH=0,
  // TABI_TIMING=1) and capacity retries use the host-driven loop below, which
  // enqueues the same kernels wave by wave.
  const char* genv = getenv("TABI_GRAPH");
  const bool use_graph = !tm.on && !(genv && genv[0] == '0');
  if (async && !use_graph) {
    ctx->err = "asynchronous packs need the graph path (TABI_GRAPH / TABI_TIMING unset)";
    return TABI_EINVAL;
  }
  // bound: every wave but the last evaluates >= 1 candidate (<= M waves), plus
  // at most 8 capacity retries; reaching it is an internal error, not NO_FIT
  const int max_attempts = M + 10;
  bool finished = false;
  for (int attempt = 0; attempt < max_attempts; attempt++) {
    pp.col_cap = ctx->col_cap;
    pp.row_cap = ctx->row_cap;
    const bool first = attempt == 0;
    const bool device_loop = first && use_graph && !ctx->loop_off;
    if (device_loop) {
      char sort_env = 0;  // test knobs read while enqueuing: part of the key
      for (const char* p = getenv("TABI_SORT"); p && *p; p++) sort_env = (char)(sort_env * 31 + *p);
      for (const char* p = getenv("TABI_PROXY_LANES"); p && *p; p++)
        sort_env = (char)(sort_env * 37 + *p);
      // host mode: the graph reads the context's own staging buffers, so the
      // caller's pointers are not part of what it bakes in
      GraphKey key{on_device ? (const void*)xy : nullptr, on_device ? (const void*)chart_start : nullptr,
                   on_device ? (const void*)out : nullptr, n, V_in, on_device, res_x, res_y, *spec, B,
                   fused ? 1 : 0, ctx->alloc_gen, sort_env};
      if (!ctx->gexec || !(key == ctx->gkey)) {
        // Only the caller's device pointers changed (same sizes, spec and
        // buffers): the re-captured graph has the same topology, so the
        // instantiated graph is updated in place (cudaGraphExecUpdate) rather
        // than re-instantiated.
        GraphKey kp = key;
        kp.xy = ctx->gkey.xy;
        kp.start = ctx->gkey.start;
        kp.out = ctx->gkey.out;
        const bool try_update = ctx->gexec && kp == ctx->gkey;
        if (ctx->gexec && !try_update) {
          cudaGraphExecDestroy(ctx->gexec);
          ctx->gexec = nullptr;
        }
        Nvtx nv_cap(try_update ? "graph capture + update" : "graph capture + instantiate");
        if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
        cudaGraph_t g = nullptr;
        int npro = 0, nbody = 0;
        // capture on the context's own streams (the caller's may be the legacy
        // default stream, which cannot be captured); launched on the caller's
        const cudaStream_t user_s = s;
        s = ctx->stream;
        const cudaError_t be = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        if (be != cudaSuccess) s = user_s;
        CK(be);
        tabi_status es = enqueue_prologue(true, npro);
        cudaError_t ce = cudaSuccess;
        cudaStreamCaptureStatus cs;
        cudaGraph_t cg = nullptr;
        cudaGraphConditionalHandle h = 0;
        if (es == TABI_OK) {
          ce = cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, nullptr, nullptr);
          // (default 0 at every launch: a wave that stops early leaves it so)
          if (ce == cudaSuccess) ce = cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault);
          if (ce == cudaSuccess) es = enqueue_body(-1, npro, h, 1);
        }
        if (es == TABI_OK && ce == cudaSuccess) {
          // WHILE node after wave 0; its body captured from a second stream
          cudaGraph_t body = nullptr;
          ce = add_while(s, h, body);
          if (ce == cudaSuccess) {
            const cudaStream_t ms = s;
            s = ctx->cap_stream;
            ce = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal);
            if (ce == cudaSuccess) {
              es = enqueue_body(0, nbody, h, 1);
              cudaGraph_t bg = nullptr;
              const cudaError_t e2 = cudaStreamEndCapture(s, &bg);
              if (ce == cudaSuccess) ce = e2;
            }
            s = ms;
          }
          if (es == TABI_OK && ce == cudaSuccess) es = enqueue_epilogue();
        }
        const cudaError_t ee = cudaStreamEndCapture(s, &g);
        s = user_s;
        if (ce == cudaSuccess) ce = ee;
        if (es != TABI_OK && es != TABI_ECUDA) {
          if (g) cudaGraphDestroy(g);
          return es;
        }
        cudaError_t ie = ce;
        if (es == TABI_ECUDA && ie == cudaSuccess)
          ie = ctx->last_cuda != cudaSuccess ? ctx->last_cuda : cudaErrorUnknown;
        if (ie == cudaSuccess && try_update) {
          cudaGraphExecUpdateResultInfo ui;
          if (cudaGraphExecUpdate(ctx->gexec, g, &ui) != cudaSuccess) {
            cudaGetLastError();  // (topology not updatable here: instantiate anew)
            cudaGraphExecDestroy(ctx->gexec);
            ctx->gexec = nullptr;
          }
        } else if (ctx->gexec) {
          cudaGraphExecDestroy(ctx->gexec);
          ctx->gexec = nullptr;
        }
        if (ie == cudaSuccess && !ctx->gexec) ie = cudaGraphInstantiate(&ctx->gexec, g, 0);
        if (g) cudaGraphDestroy(g);
        if (ie != cudaSuccess) {
          // no conditional-node graph here (driver, cooperative launch in a
          // loop body, ...): the host-driven loop from now on
          cudaGetLastError();
          if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
          ctx->gexec = nullptr;
          ctx->loop_off = true;
          ctx->err = std::string("device wave loop unavailable: ") + cudaGetErrorString(ie);
          if (async) return TABI_ECUDA;
          attempt--;
          continue;
        }
        ctx->gkey = key;
        ctx->g_launches = npro;
        ctx->g_body = nbody;
      }
      Nvtx nv_l("graph launch: proxies, sort, every candidate wave, results");
      CK(cudaEventRecord(ctx->span[0], s));
      CK(cudaGraphLaunch(ctx->gexec, s));
    } else {
      Nvtx nv_w(wave == 0 ? (first ? "host-driven wave 0" : "capacity retry, wave 0")
                          : "host-driven further wave");
      int nl = 0;
      if (first) CK(cudaEventRecord(ctx->span[0], s));
      if (wave == 0) {
        const tabi_status es = enqueue_prologue(first, nl);
        if (es != TABI_OK) return es;
      }
      const tabi_status es = enqueue_body(wave == 0 ? -1 : 0, nl, 0, 0);
      if (es != TABI_OK) return es;
      const tabi_status ee = enqueue_epilogue();
      if (ee != TABI_OK) return ee;
      launches += nl;
    }
    CK(cudaEventRecord(ctx->span[1], s));  // device span: first enqueued op .. last copy
    if (device_loop && async) {
      // return after enqueueing; tabi_pack_wait finishes (or re-runs on a
      // capacity overflow) -- the caller keeps its buffers until then
      ctx->pend = true;
      ctx->pend_args = PendArgs{xy, chart_start, n, res_x, res_y, *spec, out, stream};
      return TABI_OK;
    }
    {
      Nvtx nv_s("wait for the device");
      CK(cudaStreamSynchronize(s));
    }
    const Status st = *ctx->h_status;
    if (device_loop) launches += ctx->g_launches + ctx->g_body * st.wave + 4 * st.rounds_run;
    if (st.bad_chart != INT32_MAX) {
      if (info) info->bad_chart = st.bad_chart;
      return TABI_EINVAL;
    }
    if (st.capacity & 4) return TABI_ECAPACITY;  // vertex range beyond max_vertices
    if (!st.capacity) {
      finished = true;
      if (device_loop) break;  // the device decided the waves
      // Continue while an unevaluated (lower) candidate could still beat the
      // best area-weighted scale found: V(m) <= A_tot * m * 2^20 (p <= m 2^20/M);
      // in sequential mode any success stops the search (select_kernel's rule).
      const int next_m = st.pad[2] - (st.b0 + wave * B);  // top of wave + 1 (see wave_m)
      if (next_m < 1) break;
      if (st.winner > 0) {
        const i128 Atot = (i128)(((unsigned __int128)st.atot_hi << 64) | st.atot_lo);
        const Cand& c = ctx->h_cands[st.winner - 1];
        const bool tail = c.switched_at >= 0;
        const i128 Ap = tail ? (i128)(((unsigned __int128)c.apre_hi << 64) | c.apre_lo) : 0;
        const i128 bestV = (Atot - Ap) * st.winner * ((i128)1 << 20) + Ap * c.p * M;
        if (Atot * next_m * ((i128)1 << 20) <= bestV) break;
      }
      finished = false;
      wave++;
      continue;
    }
    wave = 0;
    // grow and retry from the slot layout (proxies and order are kept)
    ts = grow_for(ctx, st, M);
    if (ts != TABI_OK) return ts;
    tm.n = 3;  // re-time the retried stages
    if (attempt >= 8) return TABI_ECAPACITY;
  }
  if (!finished) {
    ctx->err = "candidate wave loop did not terminate";
    return TABI_ECUDA;
  }
  return finish_pack(ctx, n, M, pp.k, pp.g, on_device, out, info, launches, tm);
}

// After the last wave: the winner's record -> tabi_info, placements (host mode)
// -> the caller's buffer.
static tabi_status finish_pack(tabi_ctx* ctx, int32_t n, int32_t M, int32_t k, int32_t g,
                               int on_device, tabi_placement* out, tabi_info* info, int launches,
                               Timer& tm) {
  ctx->last_n = n;
  ctx->last_M = M;
  ctx->last_k = k;
  ctx->last_g = g;
  const int32_t win = ctx->h_status->winner;
  if (win == 0) {
    if (info) info->gpu_launches = launches;
    return TABI_NO_FIT;
  }
  if (!on_device) memcpy(out, ctx->h_out, sizeof(tabi_placement) * n);  // copied with the status
  tm.finish(info);
  if (info) {
    float dms = 0.f;
    if (cudaEventElapsedTime(&dms, ctx->span[0], ctx->span[1]) == cudaSuccess) info->device_ms = dms;
    const Cand& c = ctx->h_cands[win - 1];
    info->scale_index = win;
    // D26: every map is a similarity, so the per-triangle L2 stretch is 1/s
    // (P:1028); area-weighted RMS over sequential (m/M) and tail (p/2^20) charts
    if (c.switched_at < 0) {
      info->l2_stretch = (double)M / (double)win;
    } else {
      const i128 At = (i128)(((unsigned __int128)ctx->h_status->atot_hi << 64) | ctx->h_status->atot_lo);
      const i128 Ap = (i128)(((unsigned __int128)c.apre_hi << 64) | c.apre_lo);
      const double fs = (double)(At - Ap) / (double)At, fp = (double)Ap / (double)At;
      const double a = (double)M / (double)win, b = (double)(1 << 20) / (double)c.p;
      info->l2_stretch = sqrt(fs * a * a + fp * b * b);
    }
    info->rows = c.rows;
    info->knees_found = c.knees_found;
    info->knee_rows = c.knee_rows;
    info->prefix_rows = c.prefix_rows;
    info->gpu_launches = launches;
    info->work_pack = (int64_t)ctx->h_status->work_pack;
    info->work_profile = (int64_t)ctx->h_status->work_prof;
  }
  return TABI_OK;
}

// ---- many atlases on one GPU: one device pipeline (tabi_pack_many) ----------

template <class T>
static cudaError_t grow(T** p, int64_t count) {
  return dalloc(p, (size_t)(count > 0 ? count : 1));
}

static tabi_status many_ensure(tabi_ctx* ctx, int64_t N, int64_t V, int32_t A, int32_t k,
                               int32_t nmax, int32_t M, int32_t side) {
  ManyWs& w = ctx->many;
  if (!w.span[0]) {
    CK(cudaEventCreate(&w.span[0]));
    CK(cudaEventCreate(&w.span[1]));
    for (auto& e : w.stage) CK(cudaEventCreate(&e));
  }
  const int32_t G = many_grid(ctx->device);
  if (G < 1) {
    ctx->err = "batch kernel cannot be resident";
    return TABI_ECUDA;
  }
  if (N > w.cap_N || k > w.cap_k || A > w.cap_A) {
    const int64_t n = std::max(N, w.cap_N), kk = std::max<int64_t>(k, w.cap_k);
    const int64_t a = std::max<int64_t>(A, w.cap_A);
    CK(grow(&w.P.w, n)); CK(grow(&w.P.h, n)); CK(grow(&w.P.area2, n));
    CK(grow(&w.P.xmin, n)); CK(grow(&w.P.ymin, n)); CK(grow(&w.P.pose, n));
    CK(grow(&w.P.prerot, n)); CK(grow(&w.P.sl, n * 4 * kk)); CK(grow(&w.P.obb_j, n));
    CK(grow(&w.P.obb, 4 * n)); CK(grow(&w.perm, n)); CK(grow(&w.colofs, n));
    CK(grow(&w.rowofs, n)); CK(grow(&w.hsorted, n)); CK(grow(&w.tix, n));
    CK(grow(&w.tstart, n + a + 1)); CK(grow(&w.d_out, n)); CK(grow(&w.d_start, n + 1));
    w.cap_N = n;
    w.cap_k = (int32_t)kk;
  }
  if (V > w.cap_V) {
    CK(grow(&w.qx, V)); CK(grow(&w.qy, V)); CK(grow(&w.d_xy, 2 * V));
    w.cap_V = V;
  }
  if (A > w.cap_A || (int64_t)A * M > w.cap_q) {
    const int64_t a = std::max<int64_t>(A, w.cap_A);
    const int64_t qc = std::max<int64_t>((int64_t)A * M, w.cap_q);
    CK(grow(&w.d_small, 4 * a + 1));
    CK(grow(&w.sts, a));
    CK(grow(&w.res, a));
    CK(grow(&w.q, qc + 4));
    CK(grow(&w.tstart, w.cap_N + a + 1));
    if (w.h_small) cudaFreeHost(w.h_small);
    if (w.h_sts) cudaFreeHost(w.h_sts);
    if (w.h_res) cudaFreeHost(w.h_res);
    w.h_small = nullptr; w.h_sts = nullptr; w.h_res = nullptr;
    CK(cudaMallocHost((void**)&w.h_small, sizeof(int32_t) * (4 * a + 1)));
    CK(cudaMallocHost((void**)&w.h_sts, sizeof(Status) * a));
    CK(cudaMallocHost((void**)&w.h_res, sizeof(AtlasRes) * a));
    w.cap_A = a;
    w.cap_q = qc;
  }
  const int64_t col0 = ((int64_t)nmax * 96 + 4 * (int64_t)side + 1024) & ~(int64_t)3;
  const int64_t pair0 = 2 * (int64_t)nmax + 1024;
  const bool cta = nmax > w.nmax || G != w.G || col0 > w.col_cap || pair0 > w.pair_cap;
  if (cta || !w.dcol) {
    w.nmax = std::max(nmax, w.nmax);
    w.G = G;
    w.col_cap = std::max(col0, w.col_cap);
    w.row_cap = std::max(col0, w.row_cap);
    w.pair_cap = std::max(pair0, w.pair_cap);
    const int64_t nm = w.nmax;
    CK(grow(&w.dcol, (int64_t)G * w.col_cap));
    CK(grow(&w.drow, (int64_t)G * w.row_cap));
    CK(grow(&w.wd, G * nm)); CK(grow(&w.hd, G * nm)); CK(grow(&w.off, G * nm));
    CK(grow(&w.X, G * nm)); CK(grow(&w.Y, G * nm));
    CK(grow(&w.lock, G * nm)); CK(grow(&w.mir, G * nm));
    CK(grow(&w.scratch, (int64_t)G * (6 * nm + 3 * w.pair_cap)));
    CK(grow(&w.cands, G)); CK(grow(&w.cand_bad, G));
    CK(grow(&w.area, G * nm));
  }
  if (w.cycles_cap < 3 + 2 * (int64_t)w.G) {
    CK(grow(&w.cycles, 3 + 2 * (int64_t)w.G));
    w.cycles_cap = 3 + 2 * (int64_t)w.G;
    w.h_cta.assign(2 * (size_t)w.G, 0ull);
  }
  return TABI_OK;
}

// Grow the per-CTA footprint slots / pair lists to what a capacity-flagged
// atlas needed (the slot totals are in its status block).
static tabi_status many_grow_cta(tabi_ctx* ctx, const Status& st) {
  ManyWs& w = ctx->many;
  const int64_t G = w.G, nm = w.nmax;
  if (st.capacity & 1) {
    w.col_cap = std::max<int64_t>(w.col_cap, ((int64_t)st.cols_total + (st.cols_total >> 2) + 1024) & ~(int64_t)3);
    w.row_cap = std::max<int64_t>(w.row_cap, ((int64_t)st.rows_total + (st.rows_total >> 2) + 1024) & ~(int64_t)3);
    CK(grow(&w.dcol, G * w.col_cap));
    CK(grow(&w.drow, G * w.row_cap));
  }
  if (st.capacity & 2) {
    w.pair_cap = std::max<int64_t>(w.pair_cap, (int64_t)st.pad[0] * 2 + 1024);
    CK(grow(&w.scratch, G * (6 * nm + 3 * w.pair_cap)));
  }
  return TABI_OK;
}

static bool host_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

extern "C" tabi_status tabi_pack_many(tabi_ctx* ctx, int32_t A, const float* xy,
                                      const int32_t* chart_start, const int32_t* atlas_start,
                                      const float* res_xy, const tabi_spec* spec,
                                      tabi_placement* out, tabi_info* infos,
                                      int32_t* atlas_status, tabi_batch_info* binfo, int on_device,
                                      void* stream) {
  Nvtx nv_("tabi_pack_many");
  if (!ctx) return TABI_EINVAL;
  if (binfo) memset(binfo, 0, sizeof(*binfo));
  if (A < 1 || !xy || !chart_start || !atlas_start || !out || !spec_ok(spec)) return TABI_EINVAL;
  if (atlas_start[0] != 0) return TABI_EINVAL;
  for (int32_t a = 0; a < A; a++)
    if (atlas_start[a + 1] < atlas_start[a]) return TABI_EINVAL;
  const int64_t N = atlas_start[A];
  if (N < 1 || spec->atlas_w > ctx->max_side || spec->atlas_h > ctx->max_side) {
    return N < 1 ? TABI_EINVAL : TABI_ECAPACITY;
  }
  ctx->last_cuda = cudaSuccess;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
  std::vector<tabi_status> stv(A, TABI_OK);
  std::vector<tabi_info> inf(A);
  for (auto& i : inf) {
    memset(&i, 0, sizeof(i));
    i.bad_chart = -1;
  }
  // atlases the device batch takes: 1 <= n <= kManyMaxCharts and a sequential
  // search (t_opt resolves to 0; P:418 gives 0 for every atlas this small);
  // the others ("solo") go through tabi_pack one by one, largest first
  std::vector<int32_t> order, solo;
  int32_t nmax = 1;
  for (int32_t a = 0; a < A; a++) {
    const int32_t n = atlas_start[a + 1] - atlas_start[a];
    const int32_t t = spec->t_opt_bp >= 0 ? spec->t_opt_bp : (n > 10000 ? 100 : 0);
    if (n < 1) {
      stv[a] = TABI_EINVAL;
    } else if (n <= kManyMaxCharts && t == 0) {
      order.push_back(a);
      nmax = std::max(nmax, n);
    } else {
      solo.push_back(a);
    }
  }
  // LPT: the largest atlases first, so the queue's tail holds small items
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
    return atlas_start[x + 1] - atlas_start[x] > atlas_start[y + 1] - atlas_start[y];
  });
  const int32_t E = (int32_t)order.size();
  int launches = 0;
  float dev_ms = 0.f;
  float stage_ms[4] = {0.f, 0.f, 0.f, 0.f};
  int32_t evaluated = 0;
  int64_t work_pack = 0, work_prof = 0;
  bool lazy_used = false;
  const char* tenv = getenv("TABI_TIMING");
  const bool timing = tenv && tenv[0] == '1';
  if (E > 0) {
    int64_t V = 0;
    if (on_device) {
      int32_t v = 0;
      CK(cudaMemcpyAsync(&v, chart_start + N, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      V = v;
    } else {
      V = chart_start[N];
      if (chart_start[0] != 0) return TABI_EINVAL;
    }
    if (V < 3) return TABI_EINVAL;
    const int32_t M = spec->scale_count;
    tabi_status ts = many_ensure(ctx, N, V, A, spec->local_aabb_count, nmax, M,
                                 std::max(spec->atlas_w, spec->atlas_h));
    if (ts != TABI_OK) return ts;
    ManyWs& w = ctx->many;
    Nvtx nv_b("tabi_pack_many: enqueue inputs, proxies, sort + slots, batch kernel, results");
    CK(cudaEventRecord(w.span[0], s));
    const float* d_xy = xy;
    const int32_t* d_start = chart_start;
    // host mode: the outlines go up in chunks on a copy stream, each chunk's
    // proxies starting as soon as it lands (the copy of chunk j + 1 overlaps
    // the proxies of chunk j); pinned caller memory is copied directly,
    // pageable memory via staging
    const float* xy_src = xy;
    const char* chenv = getenv("TABI_UPLOAD_CHUNKS");  // test knob: 1..8 (default 8)
    const int nch_max = chenv ? std::min(8, std::max(1, atoi(chenv))) : 8;
    const int nch = on_device ? 1 : (N >= 8 * 2048 ? nch_max : 1);
    int32_t cbound[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j <= nch; j++) cbound[j] = (int32_t)((int64_t)N * j / nch);
    if (!on_device) {
      if (!host_pinned(xy)) {
        if (w.h_cap < 2 * V) {
          if (w.h_xy) cudaFreeHost(w.h_xy);
          w.h_xy = nullptr;
          CK(cudaMallocHost((void**)&w.h_xy, sizeof(float) * 2 * V));
          w.h_cap = 2 * V;
        }
        memcpy(w.h_xy, xy, sizeof(float) * 2 * V);
        xy_src = w.h_xy;
      }
      CK(cudaMemcpyAsync(w.d_start, chart_start, sizeof(int32_t) * (N + 1), cudaMemcpyHostToDevice, s));
      d_xy = w.d_xy;
      d_start = w.d_start;
      if (!w.copy_stream) {
        CK(cudaStreamCreateWithFlags(&w.copy_stream, cudaStreamNonBlocking));
        for (auto& e : w.chunk_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
      // (the copy stream starts after everything before this call on s)
      CK(cudaEventRecord(w.chunk_ev[8], s));
      CK(cudaStreamWaitEvent(w.copy_stream, w.chunk_ev[8], 0));
      for (int j = 0; j < nch; j++) {
        const int64_t v0 = chart_start[cbound[j]], v1 = chart_start[cbound[j + 1]];
        if (v1 > v0)
          CK(cudaMemcpyAsync(w.d_xy + 2 * v0, xy_src + 2 * v0, sizeof(float) * 2 * (v1 - v0),
                             cudaMemcpyHostToDevice, w.copy_stream));
        CK(cudaEventRecord(w.chunk_ev[j], w.copy_stream));
      }
    }
    // abase (A + 1) | order (E) | res (2A floats): one upload
    int32_t* hs = w.h_small;
    memcpy(hs, atlas_start, sizeof(int32_t) * (A + 1));
    for (int32_t i = 0; i < E; i++) hs[A + 1 + i] = order[i];  // item (a, r = 0)
    float* hr = (float*)(hs + 2 * A + 1);
    for (int32_t a = 0; a < A; a++) {
      hr[2 * a] = res_xy ? res_xy[2 * a] : 1.0f;
      hr[2 * a + 1] = res_xy ? res_xy[2 * a + 1] : 1.0f;
    }
    CK(cudaMemcpyAsync(w.d_small, hs, sizeof(int32_t) * (4 * (size_t)A + 1), cudaMemcpyHostToDevice, s));
    const int32_t* d_abase = w.d_small;
    const int32_t* d_order = w.d_small + A + 1;
    const float* d_res = (const float*)(w.d_small + 2 * A + 1);
    int32_t* qctl = w.q + w.cap_q;
    PackParams pp;
    memset(&pp, 0, sizeof(pp));
    pp.n = 0;
    pp.k = spec->local_aabb_count;
    pp.M = M;
    pp.g = spec->gutter;
    pp.W = spec->atlas_w;
    pp.H = spec->atlas_h;
    pp.Wp = spec->atlas_w + 2 * spec->gutter;
    pp.Hp = spec->atlas_h + 2 * spec->gutter;
    pp.flags = spec->flags;
    pp.B = 1;
    pp.col_cap = w.col_cap;
    pp.row_cap = w.row_cap;
    pp.early = 1;  // a rank stops at its next row once a lower rank (larger m) won
    // Ranks in flight per atlas: one atlas's top-down chain is sequential (up
    // to 16 candidates of a 2,000-chart atlas in C5), which sets the batch's
    // critical path when the GPU has more CTAs than the batch has atlases to
    // keep them busy.  K = round(sqrt(6 G / E)) ranks of each atlas start at
    // once when E < 4 G / 3, else 1 (1 for the 512- and 256-atlas shares of
    // C5 on one / two GPUs, 3 for 128, 4 for 64, 5 for 32), a CTA whose rank
    // failed then continuing with the atlas's next rank; a rank above the
    // winner is wasted work, so more is not better.  Measured on C5 subsets
    // (kernel ms by K): 128 atlases 7.1 / 4.7 / 5.6 / 6.7 (K = 1 / 3 / 4 /
    // 6), 64: 7.0 / 3.4 / 3.2 / 3.7 (1 / 3 / 4 / 6), 32: 2.9 / 2.5 / 2.3 /
    // 2.7 (3 / 4 / 6 / 8); 256: 7.4 / 7.7 (1 / 2).  TABI_MANY_INFLIGHT
    // overrides.
    const char* ienv = getenv("TABI_MANY_INFLIGHT");
    int32_t inflight = 1;
    if (ienv) inflight = atoi(ienv);
    else if (3 * (int64_t)E < 4 * (int64_t)w.G)
      inflight = (int32_t)lround(sqrt(6.0 * w.G / std::max(E, 1)));
    inflight = std::max<int32_t>(1, std::min<int32_t>(inflight, std::min<int32_t>(16, M)));
    const int32_t qcap = (int32_t)std::min<int64_t>(w.cap_q, (int64_t)E * M);
    launch_many_reset(w.sts, w.res, A, d_order, E, w.q, qcap, qctl, inflight, s);
    if (binfo) binfo->ranks_in_flight = inflight;
    CK(cudaMemsetAsync(w.cycles, 0, 3 * sizeof(unsigned long long), s));
    if (timing) CK(cudaEventRecord(w.stage[0], s));
    for (int j = 0; j < nch; j++) {
      if (!on_device) CK(cudaStreamWaitEvent(s, w.chunk_ev[j], 0));
      // (nverts scaled to the chunk's end keeps the lane-group choice of the whole batch)
      launch_proxies(d_xy, d_start, cbound[j + 1], 1.0f, 1.0f, pp.k, pp.flags, w.qx, w.qy, w.cap_V,
                     w.P, w.sts, s, AtlasMap{d_abase, A, d_res, cbound[j]},
                     V * cbound[j + 1] / N);
    }
    if (timing) CK(cudaEventRecord(w.stage[1], s));
    launch_many_sort_prep(w.P, d_abase, A, w.perm, pp, w.colofs, w.rowofs, w.hsorted, w.tstart,
                          w.tix, w.sts, s);
    if (timing) CK(cudaEventRecord(w.stage[2], s));
    ManyArgs ma;
    ma.P = w.P;
    ma.abase = d_abase;
    ma.perm = w.perm;
    ma.colofs = w.colofs;
    ma.rowofs = w.rowofs;
    ma.hsorted = w.hsorted;
    ma.sts = w.sts;
    ma.res = w.res;
    ma.out = on_device ? out : w.d_out;
    ma.q = w.q;
    ma.qctl = qctl;
    ma.qcap = qcap;
    {
      const char* cenv = getenv("TABI_MANY_CARRY");  // test knob: 1 = continue the atlas even at K = 1
      ma.inflight = inflight;
      // a CTA continues its atlas's chain itself while the batch has fewer
      // atlases than 2 G (measured: 256 C5 atlases 8.1 -> 7.4 ms); with more,
      // failures requeue at the tail so the chains interleave (512: 13.2 ->
      // 12.9 ms)
      ma.carry = (inflight > 1 || E < 2 * w.G || (cenv && cenv[0] == '1')) ? 1 : 0;
      if (cenv && cenv[0] == '0') ma.carry = inflight > 1 ? 1 : 0;
      // Idle speculation: once the queue is drained, an idle CTA starts the
      // next rank of an undecided atlas (up to 2 in flight per atlas) instead
      // of waiting -- the batch's tail is the top-down chains of its last
      // atlases.  Needs carry mode (no rank is requeued, so a queue index past
      // the tail is never filled).  Measured on C5 (kernel ms, same box):
      // 9.93 without, 9.83 carry alone, 9.16 / 9.13 / 9.17 with 2 / 3 / 4
      // ranks (load-balance tail 1.40 -> 0.53 / 0.30 / 0.18 ms, 4,017 ->
      // 4,131 / 4,208 / 4,278 items).  TABI_MANY_SPEC: test knob (0 = off).
      const char* senv = getenv("TABI_MANY_SPEC");
      ma.spec = senv ? atoi(senv) : 2;
      if (ma.spec > 1) ma.carry = 1;
      ma.order = d_order;
      ma.E = E;
    }
    ma.dcol = w.dcol;
    ma.drow = w.drow;
    ma.wd = w.wd;
    ma.hd = w.hd;
    ma.off = w.off;
    ma.lock = w.lock;
    ma.scratch = w.scratch;
    ma.X = w.X;
    ma.Y = w.Y;
    ma.mir = w.mir;
    ma.cands = w.cands;
    ma.cand_bad = w.cand_bad;
    ma.cycles = w.cycles;
    ma.area = w.area;
    {  // lazy raster + area test (R8); TABI_LAZY=0 / TABI_EARLY_FAIL=0 switch them off
      const char* le = getenv("TABI_LAZY");
      const char* fe = getenv("TABI_EARLY_FAIL");
      ma.lazy = !(le && le[0] == '0') && many_lazy_ok(pp.k, pp.g, pp.Wp);
      ma.early_fail = ma.lazy && !(fe && fe[0] == '0') && !(pp.flags & TABI_F_ADJACENT_LOCKS_ONLY);
      lazy_used = ma.lazy != 0;
      // positions rasterized beyond the fold's need: 0 (the lazy raster
      // still takes whole 64-chart tiles); measured on C5: 0 / 32 / 64 / 96 /
      // 160 -> 9.35 / 9.42 / 9.74 / 9.75 / 10.42 ms (a failing candidate
      // rasterizes fewer charts it never reaches).  TABI_LZ_AHEAD: test knob
      const char* ae = getenv("TABI_LZ_AHEAD");
      ma.ahead = ae ? atoi(ae) : 0;
      if (ma.ahead < 0) ma.ahead = 0;
    }
    ma.nmax = w.nmax;
    ma.pair_cap = w.pair_cap;
    CK(launch_many(w.G, pp, ma, s));
    if (timing) CK(cudaEventRecord(w.stage[3], s));
    launches = 4;
    if (!on_device) {
      tabi_placement* dst = out;
      if (!host_pinned(out)) {
        if (w.h_out_cap < N) {
          if (w.h_out) cudaFreeHost(w.h_out);
          w.h_out = nullptr;
          CK(cudaMallocHost((void**)&w.h_out, sizeof(tabi_placement) * N));
          w.h_out_cap = N;
        }
        dst = w.h_out;
      }
      CK(cudaMemcpyAsync(dst, w.d_out, sizeof(tabi_placement) * N, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaMemcpyAsync(w.h_sts, w.sts, sizeof(Status) * A, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(w.h_res, w.res, sizeof(AtlasRes) * A, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(w.h_cycles, w.cycles, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(w.h_cta.data(), w.cycles + 3, 2 * (size_t)w.G * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(w.span[1], s));
    CK(cudaStreamSynchronize(s));
    cudaEventElapsedTime(&dev_ms, w.span[0], w.span[1]);
    if (timing) {
      cudaEventElapsedTime(&stage_ms[0], w.span[0], w.stage[0]);
      for (int i = 1; i < 4; i++) cudaEventElapsedTime(&stage_ms[i], w.stage[i - 1], w.stage[i]);
    }
    const bool staged = !on_device && !host_pinned(out);
    for (int32_t i = 0; i < E; i++) {
      const int32_t a = order[i];
      const Status& st = w.h_sts[a];
      const AtlasRes& R = w.h_res[a];
      evaluated += R.evaluated;
      work_pack += (int64_t)st.work_pack;
      work_prof += (int64_t)st.work_prof;
      if (st.bad_chart != INT32_MAX) {
        stv[a] = TABI_EINVAL;
        inf[a].bad_chart = st.bad_chart;
      } else if (st.capacity & 4) {
        stv[a] = TABI_ECAPACITY;
      } else if (st.capacity) {  // slots / pair lists too small: grow, then solo
        ts = many_grow_cta(ctx, st);
        if (ts != TABI_OK) return ts;
        solo.push_back(a);
      } else if (R.winner > 0) {
        tabi_info& f = inf[a];
        f.scale_index = R.winner;
        f.l2_stretch = (double)M / (double)R.winner;  // D26: uniform scale m/M
        f.rows = R.rows;
        f.knees_found = R.knees_found;
        f.knee_rows = R.knee_rows;
        const int32_t c0 = atlas_start[a], n = atlas_start[a + 1] - c0;
        if (staged) memcpy(out + c0, w.h_out + c0, sizeof(tabi_placement) * n);
      } else {
        stv[a] = TABI_NO_FIT;
      }
    }
  }
  // solo atlases (hybrid tail, more than kManyMaxCharts charts, or a capacity
  // retry) through the single-pack path, atlas-local chart offsets
  Nvtx nv_solo("tabi_pack_many: solo atlases via tabi_pack");
  for (int32_t a : solo) {
    const int32_t c0 = atlas_start[a], n = atlas_start[a + 1] - c0;
    const float rx = res_xy ? res_xy[2 * a] : 1.0f, ry = res_xy ? res_xy[2 * a + 1] : 1.0f;
    std::vector<int32_t> loc(n + 1);
    if (on_device) {
      CK(cudaMemcpyAsync(loc.data(), chart_start + c0, sizeof(int32_t) * (n + 1),
                         cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    } else {
      memcpy(loc.data(), chart_start + c0, sizeof(int32_t) * (n + 1));
    }
    const int32_t v0 = loc[0];
    for (auto& v : loc) v -= v0;
    if (on_device) {
      ManyWs& w = ctx->many;
      if (!w.solo_start || w.cap_N < n + 1) CK(grow(&w.solo_start, std::max<int64_t>(n + 1, w.cap_N + 1)));
      CK(cudaMemcpyAsync(w.solo_start, loc.data(), sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, s));
      stv[a] = tabi_pack(ctx, xy + 2 * (int64_t)v0, w.solo_start, n, rx, ry, spec, out + c0, &inf[a],
                         1, s);
    } else {
      stv[a] = tabi_pack(ctx, xy + 2 * (int64_t)v0, loc.data(), n, rx, ry, spec, out + c0, &inf[a],
                         0, s);
    }
    launches += inf[a].gpu_launches;
  }
  tabi_status ret = TABI_OK;
  for (int32_t a = 0; a < A; a++) {
    if (atlas_status) atlas_status[a] = stv[a];
    if (infos) infos[a] = inf[a];
    if (ret == TABI_OK && stv[a] != TABI_OK && stv[a] != TABI_NO_FIT) ret = stv[a];
  }
  if (binfo) {
    binfo->device_ms = dev_ms;
    binfo->gpu_launches = launches;
    binfo->candidates_evaluated = evaluated;
    binfo->solo_atlases = (int32_t)solo.size();
    binfo->batched_atlases = E;
    for (int i = 0; i < 4; i++) binfo->stage_ms[i] = stage_ms[i];
    binfo->work_pack = work_pack;
    binfo->work_profile = work_prof;
    for (int i = 0; i < 3; i++) binfo->cycles[i] = E > 0 ? (int64_t)ctx->many.h_cycles[i] : 0;
    // load balance of the batch kernel: how long the last CTAs ran after the
    // median CTA finished its last item, and the mean busy fraction
    const ManyWs& w = ctx->many;
    if (E > 0 && w.G > 0 && (int64_t)w.h_cta.size() >= 2 * (int64_t)w.G) {
      unsigned long long t0 = ~0ull, t1 = 0;
      std::vector<unsigned long long> ends(w.G);
      for (int g = 0; g < w.G; g++) {
        t0 = std::min(t0, w.h_cta[2 * g]);
        t1 = std::max(t1, w.h_cta[2 * g + 1]);
        ends[g] = w.h_cta[2 * g + 1];
      }
      std::sort(ends.begin(), ends.end());
      double busy = 0.0;
      for (int g = 0; g < w.G; g++) busy += (double)(w.h_cta[2 * g + 1] - w.h_cta[2 * g]);
      if (t1 > t0) {
        binfo->tail_ms = (float)((double)(t1 - ends[w.G / 2]) * 1e-6);
        binfo->busy_frac = (float)(busy / ((double)w.G * (double)(t1 - t0)));
      }
    }
    if (lazy_used) binfo->cycles[2] = std::max<int64_t>(0, binfo->cycles[2] - binfo->cycles[0] - binfo->cycles[1]);
  }
  return ret;
}

// ---- batches over several GPUs --------------------------------

extern "C" tabi_status tabi_shard_plan(int32_t n_atlases, const int32_t* n_charts, int32_t n_gpus,
                                       int32_t* assignment) {
  if (n_atlases < 0 || n_gpus < 1 || (n_atlases > 0 && (!n_charts || !assignment)))
    return TABI_EINVAL;
  std::vector<int32_t> order(n_atlases);
  std::vector<double> cost(n_atlases);
  for (int32_t i = 0; i < n_atlases; i++) {
    order[i] = i;
    const double n = n_charts[i] > 0 ? (double)n_charts[i] : 0.0;
    cost[i] = n * (1.0 + std::log2(n + 1.0));  // sort + per-row work estimate
  }
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return cost[a] > cost[b]; });
  std::vector<double> load(n_gpus, 0.0);
  for (int32_t i : order) {
    int32_t g = 0;
    for (int32_t q = 1; q < n_gpus; q++)
      if (load[q] < load[g]) g = q;
    assignment[i] = g;
    load[g] += cost[i];
  }
  return TABI_OK;
}

extern "C" tabi_status tabi_pack_batch(tabi_ctx* const* ctxs, int32_t n_gpus, int32_t n_atlases,
                                       const float* const* xy, const int32_t* const* chart_start,
                                       const int32_t* n_charts, const float* res_xy,
                                       const tabi_spec* specs, tabi_placement* const* out,
                                       tabi_info* infos) {
  Nvtx nv_("tabi_pack_batch");
  if (!ctxs || n_gpus < 1 || n_atlases < 0) return TABI_EINVAL;
  if (n_atlases == 0) return TABI_OK;
  if (!xy || !chart_start || !n_charts || !specs || !out) return TABI_EINVAL;
  std::vector<int32_t> asg(n_atlases);
  tabi_status st = tabi_shard_plan(n_atlases, n_charts, n_gpus, asg.data());
  if (st != TABI_OK) return st;
  std::vector<tabi_status> res(n_atlases, TABI_OK);
  std::vector<tabi_status> gst(n_gpus, TABI_OK);
  // One host thread per GPU.  Its atlases are grouped by spec; each group is
  // gathered back to back into the context's pinned staging and packed by
  // ONE tabi_pack_many call (device batch pipeline), then scattered to out[i].
  std::vector<std::thread> th;
  for (int32_t g = 0; g < n_gpus; g++) {
    th.emplace_back([&, g]() {
      Nvtx nv_g("tabi_pack_batch: one GPU's atlases");
      tabi_ctx* ctx = ctxs[g];
      std::vector<int32_t> mine;
      for (int32_t i = 0; i < n_atlases; i++)
        if (asg[i] == g) mine.push_back(i);
      std::vector<char> used(mine.size(), 0);
      for (size_t u = 0; u < mine.size(); u++) {
        if (used[u]) continue;
        std::vector<int32_t> grp;  // atlases with the same spec as mine[u]
        for (size_t v = u; v < mine.size(); v++)
          if (!used[v] && memcmp(&specs[mine[v]], &specs[mine[u]], sizeof(tabi_spec)) == 0) {
            grp.push_back(mine[v]);
            used[v] = 1;
          }
        const int32_t A = (int32_t)grp.size();
        std::vector<int32_t> abase(A + 1, 0);
        std::vector<float> rxy(2 * (size_t)A);
        int64_t V = 0;
        bool bad = false;
        for (int32_t j = 0; j < A; j++) {
          const int32_t i = grp[j];
          abase[j + 1] = abase[j] + n_charts[i];
          if (n_charts[i] < 1 || chart_start[i][0] != 0) bad = true;
          else V += chart_start[i][n_charts[i]];
          rxy[2 * j] = res_xy ? res_xy[2 * i] : 1.0f;
          rxy[2 * j + 1] = res_xy ? res_xy[2 * i + 1] : 1.0f;
        }
        if (bad) {  // malformed atlas: pack one by one so each gets its own status
          for (int32_t i : grp) {
            const float rx = res_xy ? res_xy[2 * i] : 1.0f, ry = res_xy ? res_xy[2 * i + 1] : 1.0f;
            res[i] = tabi_pack(ctx, xy[i], chart_start[i], n_charts[i], rx, ry, &specs[i], out[i],
                               infos ? &infos[i] : nullptr, 0, nullptr);
          }
          continue;
        }
        const int64_t N = abase[A];
        ManyWs& w = ctx->many;
        if (cudaSetDevice(ctx->device) != cudaSuccess) { gst[g] = TABI_ECUDA; return; }
        if (w.h_cap < 2 * V) {
          if (w.h_xy) cudaFreeHost(w.h_xy);
          w.h_xy = nullptr;
          w.h_cap = 0;
          if (cudaMallocHost((void**)&w.h_xy, sizeof(float) * 2 * V) != cudaSuccess) {
            gst[g] = TABI_ECUDA;
            return;
          }
          w.h_cap = 2 * V;
        }
        if (w.h_out_cap < N) {
          if (w.h_out) cudaFreeHost(w.h_out);
          w.h_out = nullptr;
          w.h_out_cap = 0;
          if (cudaMallocHost((void**)&w.h_out, sizeof(tabi_placement) * N) != cudaSuccess) {
            gst[g] = TABI_ECUDA;
            return;
          }
          w.h_out_cap = N;
        }
        std::vector<int32_t> cs(N + 1);
        int64_t vo = 0;
        for (int32_t j = 0; j < A; j++) {
          const int32_t i = grp[j], n = n_charts[i];
          const int32_t nv = chart_start[i][n];
          memcpy(w.h_xy + 2 * vo, xy[i], sizeof(float) * 2 * (size_t)nv);
          for (int32_t c = 0; c < n; c++) cs[abase[j] + c] = (int32_t)vo + chart_start[i][c];
          vo += nv;
        }
        cs[N] = (int32_t)vo;
        std::vector<tabi_info> inf(A);
        std::vector<int32_t> ast(A);
        tabi_placement* hout = w.h_out;
        const tabi_status r = tabi_pack_many(ctx, A, w.h_xy, cs.data(), abase.data(), rxy.data(),
                                             &specs[grp[0]], hout, inf.data(), ast.data(), nullptr,
                                             0, nullptr);
        if (r == TABI_ECUDA) { gst[g] = r; return; }
        for (int32_t j = 0; j < A; j++) {
          const int32_t i = grp[j];
          res[i] = (tabi_status)ast[j];
          if (infos) infos[i] = inf[j];
          if (ast[j] == TABI_OK)
            memcpy(out[i], hout + abase[j], sizeof(tabi_placement) * (size_t)n_charts[i]);
        }
      }
    });
  }
  for (auto& t : th) t.join();
  for (int32_t g = 0; g < n_gpus; g++)
    if (gst[g] != TABI_OK) return gst[g];
  for (int32_t i = 0; i < n_atlases; i++)
    if (res[i] != TABI_OK && res[i] != TABI_NO_FIT) return res[i];
  return TABI_OK;
}

// ---- introspection ---------------------------------------------------------

extern "C" tabi_status tabi_debug_proxies(tabi_ctx* ctx, tabi_proxy_dbg* out) {
  if (!ctx || !out || ctx->last_n < 1) return TABI_EINVAL;
  const int n = ctx->last_n, k = ctx->last_k;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  int32_t *w = new int32_t[n], *h = new int32_t[n], *xm = new int32_t[n], *ym = new int32_t[n];
  int32_t *oj = new int32_t[n], *sl = new int32_t[(size_t)n * 4 * k];
  int64_t *a2 = new int64_t[n], *ob = new int64_t[4 * (size_t)n];
  uint8_t* pose = new uint8_t[n];
  uint8_t* pre = new uint8_t[n];
  cudaMemcpy(pre, ctx->P.prerot, n, cudaMemcpyDeviceToHost);
  cudaMemcpy(w, ctx->P.w, 4 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(h, ctx->P.h, 4 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(xm, ctx->P.xmin, 4 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(ym, ctx->P.ymin, 4 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(oj, ctx->P.obb_j, 4 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(sl, ctx->P.sl, sizeof(int32_t) * (size_t)n * 4 * k, cudaMemcpyDeviceToHost);
  cudaMemcpy(a2, ctx->P.area2, 8 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(ob, ctx->P.obb, 32 * (size_t)n, cudaMemcpyDeviceToHost);
  cudaMemcpy(pose, ctx->P.pose, n, cudaMemcpyDeviceToHost);
  for (int c = 0; c < n; c++) {
    tabi_proxy_dbg& d = out[c];
    memset(&d, 0, sizeof(d));
    d.w = w[c]; d.h = h[c]; d.area2 = a2[c]; d.xmin = xm[c]; d.ymin = ym[c];
    d.rot90 = pose[c] & 1; d.fx = (pose[c] >> 1) & 1; d.fy = (pose[c] >> 2) & 1; d.k = k;
    for (int j = 0; j < k; j++) {
      d.top[j] = sl[(size_t)c * 4 * k + j];
      d.bot[j] = sl[(size_t)c * 4 * k + k + j];
      d.left[j] = sl[(size_t)c * 4 * k + 2 * k + j];
      d.right[j] = sl[(size_t)c * 4 * k + 3 * k + j];
    }
    d.obb_j = oj[c];
    d.prerot = pre[c];
    d.umin = ob[4 * c]; d.umax = ob[4 * c + 1]; d.vmin = ob[4 * c + 2]; d.vmax = ob[4 * c + 3];
  }
  delete[] w; delete[] h; delete[] xm; delete[] ym; delete[] oj; delete[] sl;
  delete[] a2; delete[] ob; delete[] pose; delete[] pre;
  CK(cudaGetLastError());
  return TABI_OK;
}

extern "C" tabi_status tabi_debug_perm(tabi_ctx* ctx, int32_t* perm) {
  if (!ctx || !perm || ctx->last_n < 1) return TABI_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpy(perm, ctx->perm, sizeof(int32_t) * ctx->last_n, cudaMemcpyDeviceToHost));
  return TABI_OK;
}

extern "C" tabi_status tabi_debug_candidates(tabi_ctx* ctx, tabi_cand_dbg* out) {
  if (!ctx || !out || ctx->last_n < 1) return TABI_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpy(out, ctx->cands, sizeof(Cand) * ctx->last_M, cudaMemcpyDeviceToHost));
  return TABI_OK;
}

extern "C" tabi_status tabi_debug_profile(tabi_ctx* ctx, int32_t m, int32_t s, int32_t* wd_hd,
                                          int32_t* dtop, int32_t* dbot, int32_t* dleft,
                                          int32_t* dright) {
  if (!ctx || ctx->last_n < 1 || m < 1 || m > ctx->last_M || s < 0 || s >= ctx->last_n)
    return TABI_EINVAL;
  CK(cudaSetDevice(ctx->device));
  const int64_t b = (int64_t)(m - 1) * ctx->last_n + s;
  int32_t Wd, Hd, co, ro, bad;
  CK(cudaMemcpy(&Wd, ctx->wd + b, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&Hd, ctx->hd + b, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&co, ctx->colofs + s, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&ro, ctx->rowofs + s, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&bad, ctx->cand_bad + (m - 1), 4, cudaMemcpyDeviceToHost));
  Cand cd;
  CK(cudaMemcpy(&cd, ctx->cands + (m - 1), sizeof(Cand), cudaMemcpyDeviceToHost));
  wd_hd[0] = Wd;
  wd_hd[1] = Hd;
  // candidate not evaluated (outside the searched waves) or skipped because a
  // chart exceeds the atlas at this scale: no footprints
  if (bad || !cd.evaluated) return TABI_NO_FIT;
  uint32_t* c = new uint32_t[Wd];
  uint32_t* r = new uint32_t[Hd];
  cudaMemcpy(c, ctx->dcol + (int64_t)(m - 1) * ctx->col_cap + co, 4 * (size_t)Wd, cudaMemcpyDeviceToHost);
  cudaMemcpy(r, ctx->drow + (int64_t)(m - 1) * ctx->row_cap + ro, 4 * (size_t)Hd, cudaMemcpyDeviceToHost);
  for (int i = 0; i < Wd; i++) { dtop[i] = (int32_t)(c[i] & 0xffff); dbot[i] = (int32_t)(c[i] >> 16); }
  for (int i = 0; i < Hd; i++) { dleft[i] = (int32_t)(r[i] & 0xffff); dright[i] = (int32_t)(r[i] >> 16); }
  delete[] c;
  delete[] r;
  CK(cudaGetLastError());
  return TABI_OK;
}

extern "C" tabi_status tabi_debug_trace(tabi_ctx* ctx, int64_t* out16) {
  if (!ctx || !out16 || ctx->last_n < 1) return TABI_EINVAL;
  const Status& st = *ctx->h_status;
  const unsigned long long t0 = st.tr[0];
  const bool f = ctx->last_fused != 0;
  out16[0] = f && st.tr[1] > t0 ? (int64_t)(st.tr[1] - t0) : 0;
  out16[1] = f && st.tr[2] > t0 ? (int64_t)(st.tr[2] - t0) : 0;
  out16[2] = (int64_t)st.tr[3];
  out16[3] = (int64_t)st.tr[4];
  out16[4] = (int64_t)st.tr[5];
  out16[5] = ctx->last_fused;
  for (int i = 0; i < 10; i++) out16[6 + i] = (int64_t)st.ph[i];
  return TABI_OK;
}

extern "C" tabi_status tabi_debug_trace_raster(tabi_ctx* ctx, int64_t* out16) {
  if (!ctx || !out16 || ctx->last_n < 1) return TABI_EINVAL;
  const Status& st = *ctx->h_status;
  for (int i = 0; i < 8; i++) out16[i] = (int64_t)st.rph[i];
  for (int i = 0; i < 8; i++)
    out16[8 + i] = st.tfirst[i] > st.tr[0] && st.tfirst[i] != 0 ? (int64_t)(st.tfirst[i] - st.tr[0]) : 0;
  return TABI_OK;
}

extern "C" tabi_status tabi_debug_latency_floor(int cuda_device, double* out8) {
  if (!out8) return TABI_EINVAL;
  return latency_floor(cuda_device, out8) == 0 ? TABI_OK : TABI_ECUDA;
}

extern "C" tabi_status tabi_debug_offsets(tabi_ctx* ctx, int32_t m, int32_t* off, uint8_t* lockbits) {
  if (!ctx || ctx->last_n < 1 || m < 1 || m > ctx->last_M) return TABI_EINVAL;
  CK(cudaSetDevice(ctx->device));
  const int64_t b = (int64_t)(m - 1) * ctx->last_n;
  CK(cudaMemcpy(off, ctx->off + b, sizeof(int32_t) * ctx->last_n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(lockbits, ctx->lockbits + b, ctx->last_n, cudaMemcpyDeviceToHost));
  return TABI_OK;
}
