// k_pack.cu -- K4: balanced fold-and-push for every candidate scale in ONE
// launch (one CTA per candidate, "one work group per scale factor"),
// and K5: scale selection + placement scatter.
//
// Per candidate the CTA runs Alg. 4 row by row with the frontline
// F (one int32 per dilated atlas column) resident in shared memory:
//   Alg. 2 knee refinement (block arg-max/min over F)
//   Alg. 3 fold of both HC settings as two block-wide exclusive
//   scans + first-overflow min-reductions
//   non-adjacent lock pairs of the row (D15)
//   push: max over covered columns of F - TopEdge
//   Alg. 1 fixpoint over the lock pairs
//   score: max over covered columns of Y + BottomEdge
//   hierarchical selection, commit (shared atomicMax into F),
//   FindKnee (block max of the height drop)
//
// Data movement: a row is processed in windows of up to kRW charts.  Per
// window the charts' scalars (fold positions, widths, footprint offsets) go to
// shared memory and their column footprints -- contiguous in HBM because the
// slots follow the sorted order -- are staged with ONE TMA bulk copy
// (cp.async.bulk + mbarrier) into shared memory.  Push, score and commit are
// then flattened over the window's (chart, column) pairs: each thread walks a
// contiguous run of columns, so all 512 threads work regardless of chart
// sizes and no warp waits on per-chart global-load chains.
//
// Selection is decided before pushing where the paper allows it: the
// horizontal-compaction choice depends only on the fold's row end (P:304
// "enable horizontal compacting if it allows more charts to fit"), so each
// fold pushes 2 directions instead of 4 configurations, with identical
// results.
#include "k3_dev.cuh"

namespace tabi {
namespace {

constexpr int kNT = 512;
constexpr int kNW = kNT / 32;
constexpr int kRW = 2048;          // charts per row window
constexpr int kPWN = 1024;         // sorted positions in the fold's position window
constexpr int kPairSm = 512;       // lock pairs of a row kept in shared memory
constexpr int kMaxDynSmem = 227 * 1024 - 1024;  // leave room for static Smem
#ifndef TABI_PACK_NT
#define TABI_PACK_NT 512
#endif
// The packer role runs on the first kPT threads of its CTA with a named
// barrier (the other threads of a kNT-thread CTA leave at once).
constexpr int kPT = TABI_PACK_NT;
constexpr int kPW = kPT / 32;
static_assert(kPT % 32 == 0 && kPT <= kNT, "packer threads");
__device__ __forceinline__ void pk_sync() {
  if (kPT == kNT) __syncthreads();
  else asm volatile("bar.sync 1, %0;" ::"n"(kPT) : "memory");
}
// barrier + OR of a per-thread predicate over the packer's threads
__device__ __forceinline__ bool pk_sync_or(bool v) {
  if (kPT == kNT) return __syncthreads_or(v ? 1 : 0) != 0;
  unsigned r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n bar.red.or.pred q, 1, %2, p;\n"
      " selp.u32 %0, 1, 0, q;\n}\n"
      : "=r"(r)
      : "r"(v ? 1u : 0u), "n"(kPT)
      : "memory");
  return r != 0;
}

struct Smem {
  int32_t scan[2][kNW + 1];
  int32_t row_start, fmax, fail, rows, knees_found, knee_rows;
  int32_t knee_valid, knee_ltr, knee_left, knee_right;
  int32_t nk, conc_max;
  int32_t endv[4];      // (fold f, hc) -> row end, index f * 2 + hc
  int32_t fmin[4];
  int32_t done;
  int32_t hcsel[2], knee_ok, end_cfg[4];
  int32_t newmax[4];
  int32_t changed, npairs, pair_overflow;
  int32_t sel_cfg;
  int32_t win_s0, win_e, pglobal, a0;
  int32_t pf_out, pf_a0, pf_a1;  // row-top footprint prefetch (words [pf_a0, pf_a1))
  int32_t fold_hi, next_a0;      // fold's scanned end; colofs of the next row start (or -1)
  int32_t changed3[3];           // Alg. 1 rotating change flags
  int32_t abort;                 // sequential fused mode: a higher candidate won
  int32_t pw_b, pw_e, pw_c0, pw_c1;  // fold position window (see pw_fill)
  int32_t w_fold;                    // W.* hold the fold's scalars of the row start
  int32_t prefix_rows, switched;
  int32_t r_done;                // lazy raster: sorted positions [0, r_done) rasterized
  unsigned long long knee_key;
  long long sumF, placed;        // lazy + early fail: sum of F, 2 x area of the placed charts
  unsigned long long work;
  alignas(8) uint64_t mbar;
};

__host__ __device__ __forceinline__ size_t r16(size_t b) { return (b + 15) & ~(size_t)15; }

__device__ __forceinline__ unsigned char* carve(unsigned char*& p, size_t bytes) {
  unsigned char* r = p;
  p += r16(bytes);
  return r;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
// 1-D TMA: global -> shared, completion counted in bytes on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

__device__ __forceinline__ void block_scan2(int32_t a, int32_t b, int32_t& ea, int32_t& eb,
                                            int32_t& ta, int32_t& tb, Smem& S) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int32_t ia = warp_incl_sum(a, lane), ib = warp_incl_sum(b, lane);
  if (lane == 31) { S.scan[0][wid] = ia; S.scan[1][wid] = ib; }
  pk_sync();
  if (wid == 0) {
    const int32_t va = lane < kPW ? S.scan[0][lane] : 0, vb = lane < kPW ? S.scan[1][lane] : 0;
    const int32_t xa = warp_incl_sum(va, lane), xb = warp_incl_sum(vb, lane);
    if (lane < kPW) { S.scan[0][lane] = xa - va; S.scan[1][lane] = xb - vb; }
    if (lane == 31) { S.scan[0][kPW] = xa; S.scan[1][kPW] = xb; }
  }
  pk_sync();
  ea = S.scan[0][wid] + ia - a;
  eb = S.scan[1][wid] + ib - b;
  ta = S.scan[0][kPW];
  tb = S.scan[1][kPW];
  pk_sync();
}

struct Win {                 // shared-memory window of one row
  int32_t* rx0;              // fold position without HC (= prefix of widths)
  int32_t* rx1;              // fold position with HC
  int32_t* rwd;              // dilated width
  int32_t* rco;              // footprint offset (colofs, absolute; see pr_base)
  int32_t* rY;               // [4][kRW] vertical offsets per configuration
  int32_t* rbot;             // (unused: a chart's largest BottomEdge is its Hd, see the push)
  int32_t* rhs;              // unscaled heights (FindKnee), written by the fold
  uint8_t* rlk;              // adjacent-pair lock bits (Alg. 1), written by the fold
  uint32_t* prof;            // staged column footprints
  int32_t prof_cap;
};

// Walk the flattened (chart, column) pairs [t, tend) of the window; body(i, j)
// gets the window chart index i and column j; seg(i, first) is called when a
// run enters chart i (first = the run starts at column 0), fin(i) when it leaves.
template <class Enter, class Body, class Leave>
__device__ __forceinline__ void walk(const Win& w, int nwin, Enter enter, Body body, Leave leave) {
  const int32_t base0 = w.rx0[0];
  const int32_t T = w.rx0[nwin - 1] - base0 + w.rwd[nwin - 1];
  // run length per thread, forced odd: lanes then hit F / the staged footprints
  // at addresses C apart, i.e. 32 distinct shared-memory banks per warp access
  const int32_t C = ((T + kPT - 1) / kPT) | 1;
  int32_t t = threadIdx.x * C;
  const int32_t tend = min(T, t + C);
  if (t >= tend) return;
  int lo = 0, hi = nwin - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (w.rx0[mid] - base0 <= t) lo = mid;
    else hi = mid - 1;
  }
  int i = lo;
  while (t < tend) {
    const int32_t j0 = t - (w.rx0[i] - base0);
    const int32_t j1 = min(w.rwd[i], j0 + (tend - t));
    enter(i, j0, j1);
    for (int32_t j = j0; j < j1; j++) body(i, j);
    leave(i);
    t += j1 - j0;
    i++;
  }
}

// Fused-mode readiness: tile t (charts [t*tcf, (t+1)*tcf)) of wave slot j is
// published by a rasterizer CTA: rdy = 1 footprints written, 2 also the
// adjacent-pair offsets/locks of the pairs ending in the tile.
struct Ready {
  int32_t* flags;        // [B][T] or nullptr (non-fused: everything precomputed)
  int32_t T;             // tiles
  const int32_t* tstart; // [T + 1] first sorted position of each tile
  const int32_t* tix;    // [n] tile of each sorted position
};

// Batch mode, lazy: the packer rasterizes the footprints (and the adjacent
// pairs) itself, a few rows ahead of its fold, in the staging buffer it does
// not use before the last chart is rasterized -- so a candidate that fails
// never rasterizes the charts it does not reach.  With early_fail, a row end
// also checks that the charts still to place can fit below the frontline
// (their polygon area <= the free area sum_x (H' - F[x])): the method's
// packings are overlap-free, so a candidate failing this test fails anyway
// (R8).
struct LazyRaster {
  Proxies P;             // at the atlas's chart offset
  const int32_t* perm;   // sorted position -> atlas-local chart
  int32_t* cbad;         // the candidate's "a chart does not fit" flag
  int64_t* area;         // [n] 2 x polygon area by sorted position (written here)
  k3::Scale sc;
  int32_t ahead;         // positions rasterized beyond the one the fold needs
  int32_t early_fail;
  int64_t atot;          // 2 x the atlas's total polygon area (fits int64 for n <= 2048)
  unsigned long long* cycles;  // [2]: SM cycles in the lazy raster, in its pair offsets
};
#ifndef TABI_LZ_TC
#define TABI_LZ_TC 64
#endif
constexpr int kLzTC = TABI_LZ_TC;  // charts per lazy raster tile (the whole CTA, 8 threads per chart)

__device__ __forceinline__ int32_t atom_add_acq_rel(int32_t* p, int32_t v) {
  int32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(int32_t* p, int32_t v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// a release pattern: one fence, then relaxed adds (a release per add would
// fence each one)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_add_relaxed(int32_t* p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Lazy raster step (batch mode): the packer's threads rasterize the sorted
// positions [done, target) in kLzTC-chart tiles into the candidate's buffers
// (footprints, widths / heights, 2 x polygon areas) and compute the adjacent
// pairs that end in them.  Not inlined: its register working set then does
// not add to the packer's (no spills in the row loop).  Returns the new end.
__device__ __noinline__ int lazy_tiles(const LazyRaster& lz, const PackParams& pp,
                                       const int32_t* __restrict__ colofs,
                                       const int32_t* __restrict__ rowofs, uint32_t* dcol,
                                       uint32_t* drow, int32_t* wd, int32_t* hd, int32_t* off,
                                       uint8_t* lock, int slot, int done, int target,
                                       unsigned char* scratch, int32_t scratch_words) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, n = pp.n;
  unsigned char* p = scratch;  // the packer's staging buffer (idle until the last tile)
  k3::ChartK3* CH = (k3::ChartK3*)carve(p, sizeof(k3::ChartK3) * kLzTC);
  int32_t* cells = (int32_t*)carve(p, 4 * kLzTC);
  int32_t* cpre = (int32_t*)carve(p, 4 * (kLzTC + 1));
  int32_t* opre = (int32_t*)carve(p, 4 * (kLzTC + 1));
  int32_t* big = (int32_t*)carve(p, 4 * kLzTC);
  int32_t* misc = (int32_t*)carve(p, 32);
  int32_t* tabs = (int32_t*)carve(p, (size_t)4 * kLzTC * 4 * pp.k);
  // the rest of the staging buffer holds a tile's dilated row footprints, so
  // its internal pairs read shared memory (g <= kDilMax)
  uint32_t* rstash = (uint32_t*)p;
  const int32_t rcap = scratch_words - (int32_t)((p - scratch) / 4);
  const bool stash = pp.g <= k3::kDilMax && rcap > 0;
  long long c0 = tid == 0 ? clock64() : 0, cpair = 0;
  while (done < target) {  // (uniform)
    const int s0 = done, nt = min(kLzTC, n - s0);
    k3::tile_raster<kLzTC, kPT, 1>(lz.P, lz.perm, pp, colofs, rowofs, dcol, drow, wd, hd, lz.cbad,
                                   slot, s0, lz.sc, CH, cells, cpre, opre, &misc[1], big, tabs,
                                   nullptr, nt, tid, [] { pk_sync(); }, k3::NoMark(),
                                   stash ? rstash : nullptr, rcap);
    const bool stashed = stash && cpre[nt] <= rcap;
    if (tid < nt) lz.area[s0 + tid] = lz.P.area2[lz.perm[s0 + tid]];
    // pairs (s, s + 1) that end in this tile, and the last chart's zero entry
    const long long cp = tid == 0 ? clock64() : 0;
    const int plo = max(0, s0 - 1), phi = s0 + nt == n ? n - 1 : s0 + nt - 2;
    for (int q = plo + wid; q <= phi; q += kPW) {
      const int a = q - s0;
      if (stashed && a >= 0 && a + 1 < nt && CH[a].small && CH[a + 1].small) {
        const int64_t b = (int64_t)slot * n + q;
        k3::pair_rows(rstash + cpre[a], rstash + cpre[a + 1], CH[a].hs + 2 * pp.g,
                      CH[a + 1].hs + 2 * pp.g, CH[a].ws + 2 * pp.g, off + b, lock + b, lane);
      } else {
        k3::pair_offset(pp, rowofs, drow, wd, hd, off, lock, slot, q, lane);
      }
    }
    pk_sync();
    if (tid == 0) cpair += clock64() - cp;
    done = s0 + nt;
  }
  if (tid == 0) {
    const long long dt = clock64() - c0;
    atomicAdd(lz.cycles, (unsigned long long)(dt - cpair));
    atomicAdd(lz.cycles + 1, (unsigned long long)cpair);
  }
  return done;
}

// The footprint/offset arrays are not __restrict__ here: in fused mode other
// CTAs write them during the launch, so they must not go through the
// non-coherent load path.
__device__ __forceinline__ void packer(PackParams pp, const int32_t* __restrict__ colofs,
            const int32_t* __restrict__ rowofs,
            const uint32_t* dcol, const uint32_t* drow,
            const int32_t* wd_all, const int32_t* hd_all,
            const int32_t* off_all, const uint8_t* lock_all,
            const int32_t* __restrict__ hsorted, const int32_t* cand_bad,
            int32_t* scratch, int64_t pair_cap, int32_t* Xo_all, int32_t* Yo_all, uint8_t* mir_all,
            Cand* cands, Status* st, int32_t prof_cap, int m, int slot, int jslot, Ready rd,
            unsigned char* dsm, const bool lazy = false, const LazyRaster lzv = LazyRaster{}) {
  const LazyRaster* lz = lazy ? &lzv : nullptr;
  // m: the candidate scale m/M; slot: its index in the per-candidate arrays
  // (m - 1 for a single pack, the CTA's own buffers in batch mode); jslot: its
  // wave slot (ready flags, early exit)
  __shared__ Smem S;
  __shared__ int32_t ready_upto;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid >= kPT) return;
  const int n = pp.n, Wp = pp.Wp, Hp = pp.Hp;
  // (decided by thread 0 for the whole packer: in batch mode another CTA
  // evaluating a rank of the same atlas may set the capacity bits meanwhile)
  __shared__ int32_t pk_bad;
  if (tid == 0) pk_bad = (*(volatile int32_t*)&st->bad_chart != INT32_MAX ||
                          *(volatile int32_t*)&st->capacity != 0) ? 1 : 0;
  pk_sync();
  if (pk_bad) return;
  // fused mode: tiles [0, ready_upto] of this slot are known to be published
  if (tid == 0) ready_upto = -1;
  // sequential mode: a higher candidate already succeeded, so this one cannot
  // win -- its remaining tiles may never be rasterized; stop
  auto beaten = [&]() -> bool {
    return pp.early && *(volatile int32_t*)&st->win_j < jslot;
  };
  // Fold-side readiness: block until position s (and its pair offset) is
  // published, then take whatever further tiles are already published (no
  // waiting).  Returns the last sorted position the fold may scan, so the
  // packer runs right behind the rasterizers instead of a whole scan chunk
  // behind them.
  // Warp 0 probes 32 flags per step with relaxed loads; each lane then
  // fences (acquire pattern: relaxed load + fence.acq_rel, which also drops
  // the SM's L1 so later plain loads see the published data).
  __shared__ int32_t ready_lim;
  if (tid == 0) ready_lim = -1;
  auto wait_ready = [&](int s) -> int {
    if (!rd.flags || ready_upto == rd.T - 1) return n - 1;  // (no tile-index loads)
    const int t_need = rd.tix[min(s + 1, n - 1)];
    // probe as far as the published prefix reaches (32 flags per step): once
    // every tile is in, later calls take the fast path above
    const int t_cap = rd.T - 1;
    // enough is known ready: no probe (a probe's fence also empties the L1
    // that keeps the row's scalars warm between rows) -- except every 4th row,
    // so the known-ready prefix catches up with the raster and reaches the
    // all-ready fast path (which also enables the row-top prefetch)
    if (ready_upto >= rd.tix[min(s + 64, n - 1)] && (S.rows & 3) != 0) return ready_lim;
    if (wid == 0) {
      const int32_t* fl = rd.flags + (int64_t)jslot * rd.T;
      int up = ready_upto;
      const unsigned long long t0 = up < t_need && lane == 0 ? gtime() : 0ull;
      const bool blocked = up < t_need;
      while (true) {
        const int tt = up + 1 + lane;
        int32_t f = 2;
        if (tt <= t_cap && tt < rd.T)
          asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(fl + tt) : "memory");
        else
          f = 0;
        const unsigned ok = __ballot_sync(0xffffffffu, f >= 2);
        const int adv = ok == 0xffffffffu ? 32 : __ffs(~ok) - 1;  // consecutive ready tiles
        up += adv;
        if (up >= t_need && adv < 32) break;
        if (up >= t_cap || up + 1 >= rd.T) break;
        if (adv == 0) {
          if (__shfl_sync(0xffffffffu, beaten() ? 1 : 0, 0)) break;  // uniform: lane 0 decides
          __nanosleep(64);
        }
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      if (lane == 0) {
        if (blocked) atomicAdd(&st->tr[3], gtime() - t0);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // TMA reads follow
        ready_upto = up;
        ready_lim = up == rd.T - 1 ? n - 1 : rd.tstart[up + 1] - 2;
        if (up < t_need) { S.abort = 1; ready_lim = -2; }  // beaten while waiting
      }
    }
    pk_sync();
    return ready_lim;
  };
  const int64_t cb = (int64_t)slot * n;
  const int32_t* wd = wd_all + cb;
  const int32_t* hd = hd_all + cb;
  const int32_t* off = off_all + cb;
  const uint8_t* lk = lock_all + cb;
  const uint32_t* col = dcol + (int64_t)slot * pp.col_cap;
  const uint32_t* row = drow + (int64_t)slot * pp.row_cap;
  int32_t* sc = scratch + (int64_t)slot * (6 * (int64_t)n + 3 * pair_cap);
  int32_t* xs0 = sc;
  int32_t* xs1 = sc + n;
  int32_t* Yc = sc + 2 * (int64_t)n;  // [4][n]
  int32_t* pa = sc + 6 * (int64_t)n;
  int32_t* pb = pa + pair_cap;
  int32_t* plk = pb + pair_cap;
  int32_t* Xo = Xo_all + cb;
  int32_t* Yo = Yo_all + cb;
  uint8_t* mir = mir_all + cb;
  const bool adj_only = (pp.flags & TABI_F_ADJACENT_LOCKS_ONLY) != 0;
  const bool no_hc = (pp.flags & TABI_F_NO_HC) != 0;
  const bool no_bal = (pp.flags & TABI_F_NO_BALANCE) != 0;
  const bool ef = lz && lz->early_fail;  // batch mode: the area test at every row end
  const int32_t cols_total = st->cols_total;

  // dynamic shared memory: F | window scalars | staged footprints
  int32_t* F = (int32_t*)dsm;
  const int32_t f_words = (Wp + 3) & ~3;
  Win W;
  W.rx0 = F + f_words;
  W.rx1 = W.rx0 + kRW;
  W.rwd = W.rx1 + kRW;
  W.rco = W.rwd + kRW;
  W.rY = W.rco + kRW;
  W.rbot = W.rY + 4 * kRW;
  W.rhs = W.rbot + kRW;
  W.rlk = (uint8_t*)(W.rhs + kRW);
  struct {
    int32_t *p0, *p1, *wd, *co, *hs;
    uint8_t* lk;
  } PW;
  PW.p0 = (int32_t*)(W.rlk + kRW);
  PW.p1 = PW.p0 + kPWN;
  PW.wd = PW.p1 + kPWN;
  PW.co = PW.wd + kPWN;
  PW.hs = PW.co + kPWN;
  PW.lk = (uint8_t*)(PW.hs + kPWN);
  struct {  // the row's first kPairSm lock pairs (D15) in shared memory
    int32_t *a, *b;
    uint8_t* lk;
  } SP;
  SP.a = (int32_t*)(PW.lk + kPWN);
  SP.b = SP.a + kPairSm;
  SP.lk = (uint8_t*)(SP.b + kPairSm);
  W.prof = (uint32_t*)(SP.lk + kPairSm);
  W.prof_cap = prof_cap;

  const bool prefix_mode = pp.mode == 1;  // D24 steps 3-4: push the prefix-folded rows
  int32_t* qrow = sc + 5 * (int64_t)n;    // prefix row id per sorted position (tail)
  const int32_t* rend = sc + 4 * (int64_t)n;  // prefix row: last position, by its first (tail)
  if (prefix_mode) {
    if (pp.T.state[slot] != TAIL_READY) return;
  } else if ((!rd.flags && !lz && cand_bad[slot]) || (rd.flags && cand_too_big(pp, st, m))) {
    // a chart exceeds the dilated atlas at this scale (fused mode: decided
    // from the largest chart at once, and the rasterizers drop the slot)
    if (tid == 0) {
      cands[slot] = Cand{0, 0, 0, 0, 0, 0, 0, 1, -1, 0, 0ull, 0ull};
      if (rd.flags) *(volatile int32_t*)(rd.flags + 2 * (int64_t)pp.B * n + pp.B + jslot) = 1;
    }
    return;
  }
  if (!prefix_mode && !rd.flags) {  // work accounting: footprint entries K3 produced
    unsigned long long pe = 0;
    #pragma unroll 1  // (cold or short: keep the code small)
    for (int s = tid; s < n; s += kPT) pe += (unsigned long long)(wd[s] + hd[s]);
    for (int o = 16; o > 0; o >>= 1) pe += __shfl_xor_sync(0xffffffffu, pe, o);
    if (lane == 0) atomicAdd(&st->work_prof, pe);
  }
  int32_t* fsave = pp.T.fsave + (int64_t)slot * pp.T.fstride;
  #pragma unroll 1  // (cold or short: keep the code small)
  for (int x = tid; x < Wp; x += kPT) F[x] = prefix_mode ? fsave[x] : 0;  // top
  if (tid == 0) {
    S.row_start = 0; S.fmax = 0; S.fail = 0; S.rows = 0; S.knees_found = 0; S.knee_rows = 0;
    S.next_a0 = 0; S.fold_hi = 0; S.pf_out = 0; S.abort = 0;
    S.pw_b = 0; S.pw_e = 0; S.pw_c0 = 0; S.pw_c1 = 0; S.w_fold = 0;
    for (int q = 0; q < 4; q++) S.fmin[q] = INT32_MAX;
    S.knee_valid = 0; S.knee_ltr = 0; S.knee_left = 0; S.knee_right = 0;
    S.work = 0ull;
    S.knee_key = 0ull;
    S.prefix_rows = 0;
    S.switched = 0;
    S.r_done = 0;
    S.sumF = 0;
    S.placed = 0;
    if (prefix_mode) {  // continue from the state saved at the switch
      const Cand cd = cands[slot];
      S.row_start = pp.T.r0[slot];
      S.next_a0 = S.row_start < n ? colofs[S.row_start] : -1;  // the first prefix row's prefetch
      S.fmax = cd.score; S.rows = cd.rows; S.knees_found = cd.knees_found;
      S.knee_rows = cd.knee_rows;
    }
    mbar_init(&S.mbar);
  }
  pk_sync();
  uint32_t phase = 0;
  unsigned long long wk = 0;  // frontline column visits by this thread
  // row-phase timing (thread 0, SM clock cycles), compiled in only for the
  // trace build (-DTABI_PHASE_TRACE, tools/fused_trace.py)
  unsigned long long ph[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#ifdef TABI_PHASE_TRACE
  long long t_last = clock64();
  auto phase_mark = [&](int i) {
    if (tid == 0) {
      const long long t = clock64();
      ph[i] += (unsigned long long)(t - t_last);
      t_last = t;
    }
  };
#else
  auto phase_mark = [](int) {};
#endif

  // Stage window [ws0, we) of the current row (no-op if already staged).
  // A row's footprints are prefetched by one TMA copy issued at the top of the
  // row (before the knee update and the fold), covering the published slots
  // from the row start up to a cap; the first stage() of the row consumes it
  // if its window lies inside (else drains it and copies the exact window).
  bool pf_pending = false;  // uniform: a prefetch copy is in flight
  int32_t wj = INT32_MAX;   // thread 0: last seen st->win_j
  // the staged window and where its footprints are (every thread keeps the
  // same copy: no shared-memory handshake)
  int32_t win_s0 = -1, win_e = -1, g_a0 = 0;
  bool g_pg = false;
  auto stage = [&](int ws0, int we) {
    if (win_s0 == ws0 && win_e == we) return;
    const int nwin = we - ws0;
    // the fold already wrote the scalars of the row's first kRW charts
    // (positions below S.fold_hi), footprint offsets included
    const bool fw = !prefix_mode && ws0 == S.row_start;
    // (only while W still holds the fold's scalars: a later window of a long
    // row overwrites them)
    const bool have = fw && nwin <= kRW && S.w_fold != 0;
    const int32_t c0 = have ? W.rco[0] : colofs[ws0];
    const int32_t c1 = we >= n ? cols_total
                               : (fw && we < S.fold_hi && nwin < kRW) ? W.rco[nwin] : colofs[we];
    const int32_t a0 = c0 & ~3, a1 = (c1 + 3) & ~3;
    const bool pg = (a1 - a0) > W.prof_cap;
    const bool hit = pf_pending && c0 >= S.pf_a0 && c1 <= S.pf_a1;
    win_s0 = ws0;
    win_e = we;
    g_pg = hit ? false : pg;
    g_a0 = hit ? S.pf_a0 : a0;
    if (have && hit) {
      // the fold wrote the window's scalars and the row-top prefetch holds its
      // footprints: nothing in shared memory changes, so no barrier -- every
      // thread waits for the copy on the mbarrier
      mbar_wait(&S.mbar, phase);
      phase ^= 1u;
      pf_pending = false;
      return;
    }
    pk_sync();  // previous readers of the window buffers are done
    #pragma unroll 1  // (cold or short: keep the code small)
    for (int k = tid; k < nwin && !have; k += kPT) {
      const int s = ws0 + k;
      W.rx0[k] = xs0[s];
      W.rx1[k] = xs1[s];
      W.rwd[k] = wd[s];
      W.rco[k] = colofs[s];
    }
    if (pf_pending) {  // consume (hit) or drain (miss) the row-top prefetch
      mbar_wait(&S.mbar, phase);
      phase ^= 1u;
      pf_pending = false;
    }
    if (!hit && !pg && tid == 0) bulk_g2s(W.prof, col + a0, (uint32_t)(a1 - a0) * 4u, &S.mbar);
    if (tid == 0 && !have) S.w_fold = 0;
    if (!hit && !pg) {
      mbar_wait(&S.mbar, phase);
      phase ^= 1u;
    }
    pk_sync();
  };

  // Lazy raster (batch mode): make sorted positions [0, s + 2 + ahead) have
  // their footprints, widths / heights and pair offsets; returns the last
  // position whose pair offset is valid (the fold's scan limit).
  auto lazy_fill = [&](int s) -> int {
    const int target = min(n, max(S.r_done, s + 2) + lz->ahead);
    if (S.r_done < target) {
      const int done = lazy_tiles(*lz, pp, colofs, rowofs, (uint32_t*)dcol, (uint32_t*)drow,
                                  (int32_t*)wd_all, (int32_t*)hd_all, (int32_t*)off_all,
                                  (uint8_t*)lock_all, slot, S.r_done, target,
                                  (unsigned char*)W.prof, W.prof_cap);
      if (tid == 0) S.r_done = done;
      pk_sync();
      return done >= n ? n - 1 : done - 2;
    }
    const int d0 = S.r_done;
    pk_sync();  // (every thread has read S.r_done before a later call changes it)
    return d0 >= n ? n - 1 : d0 - 2;
  };

  // Position window for the fold (non-prefix mode): sorted positions
  // [S.pw_b, S.pw_e) with the exclusive prefix sums of widths (p0) and of the
  // compaction offsets (p1) from S.pw_b, and the per-position scalars the row
  // window needs.  Filled (or appended to) by block scans over published
  // positions only; only its first chunk may wait for the rasterizers.
  // mode 0: a new window at `from` (prefix frame restarts at 0); 1: append at
  // S.pw_e; 2: slide -- a new window at `from` = S.pw_e that keeps the prefix
  // frame (a row longer than the window continues in the same frame).
  auto pw_fill = [&](int from, int mode) -> bool {
    const bool append = mode == 1;
    int count = append ? S.pw_e - S.pw_b : 0;
    const int count0 = count;
    const int b0 = append ? S.pw_b : from;
    int32_t c0 = mode ? S.pw_c0 : 0, c1 = mode ? S.pw_c1 : 0;
    int base = append ? S.pw_e : from;
    int lim = -1;
    while (count < kPWN && base < n) {
      if (base > lim) {
        if (count > count0) break;  // only the first chunk waits
        lim = lz ? lazy_fill(base) : wait_ready(base);
        if (lim == -2) return false;  // beaten (S.abort)
#ifdef TABI_PHASE_TRACE
        if (rd.flags && jslot == 0 && base == 0 && tid == 0) st->tfirst[2] = gtime();
#endif
      }
      const int cnt = min(min(kPT, lim - base + 1), kPWN - count);
      const int s = base + tid;
      const bool valid = tid < cnt;
      const int32_t w_s = valid ? wd[s] : 0;
      const int32_t a1 = valid ? off[s] : 0;
      // fused mode: a chart that cannot fit the dilated atlas at this scale
      // makes the candidate fail (it must be placed in some row)
      if ((rd.flags || lz) && valid && (w_s > Wp || hd[s] > Hp)) S.fail = 1;
      int32_t e0, e1, t0, t1;
      block_scan2(w_s, a1, e0, e1, t0, t1, S);
      if (valid) {
        const int i = count + tid;
        PW.p0[i] = c0 + e0;
        PW.p1[i] = c1 + e1;
        PW.wd[i] = w_s;
        PW.co[i] = colofs[s];
        PW.hs[i] = hsorted[s];
        PW.lk[i] = lk[s];
      }
      c0 += t0;
      c1 += t1;
      count += cnt;
      base += cnt;
    }
    pk_sync();
    if (tid == 0) {
      S.pw_b = b0;
      S.pw_e = b0 + count;
      S.pw_c0 = c0;
      S.pw_c1 = c1;
    }
    pk_sync();
    return true;
  };

  while (true) {
    const int32_t rs = S.row_start;
    if (rs >= n || S.fail || S.abort) break;
    // ---- D23 switch to prefix folding ("when no more knees are
    // detected and the height of the tallest chart in the row decreases below
    // a threshold t_opt"), checked before each row, latched: save the state,
    // the tail kernels take over. ------------------------------------------
    if (!prefix_mode && pp.t_opt > 0 && !S.knee_valid) {
      const int64_t hs0 = ceildiv((int64_t)hsorted[rs] * m, (int64_t)pp.M * TABI_UNITS);
      if (hs0 * 10000 < (int64_t)pp.t_opt * pp.H) {
        // (a candidate with a chart too big for the atlas never gets here: the
        // split path checks cand_bad first, the fused packer cand_too_big)
        #pragma unroll 1  // (cold or short: keep the code small)
        for (int x = tid; x < Wp; x += kPT) fsave[x] = F[x];
        if (tid == 0) {
          pp.T.state[slot] = TAIL_LAYOUT;
          pp.T.r0[slot] = rs;
          pp.T.iter[slot] = 0;
          cands[slot] = Cand{0, S.fmax, S.rows, S.knees_found, S.knee_rows, 0, 0, 1, rs, 0,
                              0ull, 0ull};
          S.switched = 1;
        }
        pk_sync();
        break;
      }
    }
    // sequential fused mode: has a higher candidate won?  Loaded here, used at
    // the row end, so the load's latency hides behind the row
    // (batch mode: a lower rank of the same atlas, i.e. a larger m, won)
    if (tid == 0 && (rd.flags || lz) && pp.early) wj = *(volatile int32_t*)&st->win_j;
    // ---- footprint prefetch for this row (consumed by the push's stage) ----
    // (no global loads on thread 0's path: the row start's slot offset was
    // kept from the previous row's fold; in fused mode only once every tile
    // is published)
    if (tid == 0) {
      S.pf_out = 0;
      // every tile of this candidate published?  (one acquire load of the
      // slot's completed-tile count; the fold's window fills probe far less
      // often than once a row)
      if (rd.flags && ready_lim != n - 1 &&
          ld_acquire(rd.flags + 2 * (int64_t)pp.B * n + jslot) >= 2 * rd.T) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // TMA reads follow
        ready_upto = rd.T - 1;
        ready_lim = n - 1;
      }
#ifdef TABI_NO_PREFETCH
      const bool all = false;  // experiment: measure the row without the prefetch
#else
      const bool all = lz ? S.r_done >= n : !rd.flags || ready_lim == n - 1;
#endif
      if (all && S.next_a0 >= 0) {
        const int32_t a0 = S.next_a0 & ~3;
        const int32_t a1 = min((cols_total + 3) & ~3, a0 + min(W.prof_cap, 4 * f_words));
        if (a1 > a0) {
          bulk_g2s(W.prof, col + a0, (uint32_t)(a1 - a0) * 4u, &S.mbar);
          S.pf_out = 1; S.pf_a0 = a0; S.pf_a1 = a1;
        }
      }
    }
    // ---- Alg. 2 UpdateKneeLocation ---------------------------
    if (S.knee_valid) {
      const int32_t left = S.knee_left, right = S.knee_right, ltr = S.knee_ltr;
      const bool degenerate = ltr ? (right >= Wp) : (left <= 0);
      if (tid == 0) S.nk = ltr ? left - 1 : right;
      pk_sync();
      if (!degenerate) {
        const int32_t ref = ltr ? F[right] : F[left - 1];
        #pragma unroll 1  // (cold or short: keep the code small)
        for (int x = left + tid; x < right; x += kPT) {
          if (F[x] >= ref) {
            if (ltr) atomicMax(&S.nk, x);
            else atomicMin(&S.nk, x);
          }
        }
      }
      pk_sync();
      if (tid == 0) {
        if (degenerate) {
          S.knee_valid = 0;
        } else if (ltr) {
          if (S.nk + 1 == left) S.knee_valid = 0;  // collapsed: discard (D20)
          else S.knee_right = S.nk + 1;
        } else {
          if (S.nk == right) S.knee_valid = 0;
          else S.knee_left = S.nk;
        }
        S.conc_max = INT32_MIN;
      }
      pk_sync();
    }
    phase_mark(0);
    const int32_t kv = S.knee_valid;
    const int32_t ka = kv ? (S.knee_ltr ? S.knee_right : 0) : 0;  // knee fold region [ka, kb)
    const int32_t kb = kv ? (S.knee_ltr ? Wp : S.knee_left) : 0;
    if (kv) {
      int32_t mx = INT32_MIN;
      #pragma unroll 1  // (cold or short: keep the code small)
      for (int x = ka + tid; x < kb; x += kPT) mx = max(mx, F[x]);
      mx = warp_max(mx);
      if (lane == 0) atomicMax(&S.conc_max, mx);
    }
    // ---- level 1 of the hierarchical choice: HC iff it fits more,
    // by thread 0 once the fold's row ends are known ---------------------------
    auto hc_select = [&]() {
      S.hcsel[0] = (!no_hc && S.endv[1] > S.endv[0]) ? 1 : 0;
      S.hcsel[1] = (!no_hc && S.endv[3] > S.endv[2]) ? 1 : 0;
      if (prefix_mode) { S.hcsel[0] = 1; S.hcsel[1] = 0; }  // HC always on in the tail
      const int32_t ea = S.endv[S.hcsel[0]];
      const int32_t ek = S.endv[2 + S.hcsel[1]];
      S.knee_ok = kv && ek >= rs;
      S.end_cfg[0] = S.end_cfg[1] = ea;
      S.end_cfg[2] = S.end_cfg[3] = ek;
      if (ea < rs) S.fail = 1;  // first chart wider than the atlas (D22)
      for (int q = 0; q < 4; q++) S.newmax[q] = INT32_MIN;
      S.npairs = 0;
      S.pair_overflow = 0;
    };
    // ---- Alg. 3 FoldRow for both HC settings and both folds --------------
    // (no barrier here: in the non-prefix fold only thread 0 reads these
    // before the fold's own barriers)
    if (tid < 4) S.endv[tid] = INT32_MIN;
    if (tid == 0) S.done = 0;
    win_s0 = win_e = -1;
    bool anylock = true;   // some adjacent pair the row may hold has a lock bit (else Alg. 1 is a no-op)
    bool anypl = false;    // some non-adjacent (D15) pair of the row is locked
    if (prefix_mode) pk_sync();
    if (prefix_mode) {
      // prefix rows were laid out by the tail kernels (positions in xs0/xs1,
      // and each row's last position by its first: rend, written by
      // tail_layout / the exact tail's row search)
      if (tid == 0) {
        const int32_t e = rend[rs];
        S.endv[0] = S.endv[1] = e;
        S.endv[2] = S.endv[3] = rs - 1;
        S.done = 1;
      }
    } else {
      // Fold over the position window: its exclusive prefix sums of widths
      // and offsets were scanned when the window was filled, so a row's fold
      // positions are differences (x(s) = P(s) - P(rs)) -- no block scan and no
      // global loads while the row start stays inside the window.
      bool beaten = false;
      if (rs < S.pw_b || rs >= S.pw_e) beaten = !pw_fill(rs, 0);
      // the row start's prefixes (the frame stays fixed while the row is folded)
      const int32_t r0 = beaten ? 0 : PW.p0[rs - S.pw_b], r1 = beaten ? 0 : PW.p1[rs - S.pw_b];
      int sc = rs;  // next position to examine
      bool lockv = false;  // this thread saw a lock bit among the row's candidate pairs
      while (!beaten) {
        const int pb = S.pw_b, pe = S.pw_e;
        // (S.fmin[] are INT32_MAX here: reset by thread 0 after each use)
        for (; sc < pe; sc = min(sc + kPT, pe)) {  // (sc ends at pe: an append resumes there)
          const int s = sc + tid;
          if (s < pe) {
            const int i = s - pb;
            const int32_t w_s = PW.wd[i], x0 = PW.p0[i] - r0, x1 = PW.p1[i] - r1;
            xs0[s] = x0;
            xs1[s] = x1;
            if (s - rs < kRW) {  // the row's window scalars, straight into smem
              W.rx0[s - rs] = x0;
              W.rx1[s - rs] = x1;
              W.rwd[s - rs] = w_s;
              W.rco[s - rs] = PW.co[i];
              W.rhs[s - rs] = PW.hs[i];
              W.rlk[s - rs] = PW.lk[i];
              lockv |= PW.lk[i] != 0;
#pragma unroll
              for (int q = 0; q < 4; q++) W.rY[q * kRW + (s - rs)] = INT32_MIN;  // push init
            }
            if (x0 + w_s > Wp) atomicMin(&S.fmin[0], s);
            if (x1 + w_s > Wp) atomicMin(&S.fmin[1], s);
            if (x0 + w_s > kb - ka) atomicMin(&S.fmin[2], s);
            if (x1 + w_s > kb - ka) atomicMin(&S.fmin[3], s);
          }
          anylock = pk_sync_or(lockv);  // (lockv is sticky: the last chunk's OR covers all)
          if (tid == 0) {
            for (int q = 0; q < 4; q++) {
              if (S.endv[q] == INT32_MIN && S.fmin[q] != INT32_MAX) S.endv[q] = S.fmin[q] - 1;
              S.fmin[q] = INT32_MAX;
            }
            const int hi = min(sc + kPT, pe);
            if (S.endv[1] != INT32_MIN || hi >= n) {
              for (int q = 0; q < 4; q++)
                if (S.endv[q] == INT32_MIN) S.endv[q] = n - 1;
              S.done = 1;
              S.fold_hi = hi;  // W.* hold positions [rs, min(fold_hi, rs + kRW))
              S.w_fold = 1;
              hc_select();  // published by the barrier below
            }
          }
          pk_sync();
          if (S.done) break;
        }
        if (S.done) break;
        // the row reaches past the window: append, or slide it on when full
        const bool full = S.pw_e - S.pw_b >= kPWN;
        beaten = !pw_fill(S.pw_e, full ? 2 : 1);
      }
    }  // !prefix_mode
    // (the row-top prefetch flag: published by the fold's barriers; set before
    // any exit so the end of the packer drains a copy still in flight)
    pf_pending = S.pf_out != 0;
    if (S.abort) break;  // beaten while waiting for tiles (set before a barrier)
    phase_mark(1);
    // (the non-prefix fold ran hc_select in its last step, before a barrier)
    if (prefix_mode) {
      if (tid == 0) hc_select();
      pk_sync();
    }
    if (S.fail) break;
    const int32_t knee_ok = S.knee_ok;
    const int32_t hc0 = S.hcsel[0], hc1 = S.hcsel[1];
    const int32_t endA = S.end_cfg[0], endK = S.end_cfg[2];
    const int ncfg = knee_ok ? 4 : 2;
    // prefix rows: FastAtlas fixes the direction in advance (one L->R row,
    // then two R->L) and HC is on, so a prefix row pushes,
    // relaxes and scores ONE configuration (pdir) instead of both directions
#ifndef TABI_PREFIX_ONECFG
#define TABI_PREFIX_ONECFG 1
#endif
    const int pdir = TABI_PREFIX_ONECFG && prefix_mode ? ((S.prefix_rows % 3 == 0) ? 0 : 1) : -1;
    // A row of at most kRW charts (the normal case) is one window: its Y
    // values then live in shared memory from push to commit, and the fold's
    // window scalars (W.rx1, W.rwd) serve the lock-pair scan; longer rows
    // round-trip through HBM per window.
    const bool one = endA - rs + 1 <= kRW;
    const bool useW = one && !prefix_mode;
    // ---- D15: non-adjacent lock pairs of the row (HC folds only) ----------
    const int32_t R = max(hc0 ? endA : -1, (knee_ok && hc1) ? endK : -1);
    if (!adj_only && R > rs) {
      // pair-list slots by warp-aggregated atomics: the list's order is
      // immaterial (each pair's lock bits and Alg. 1's fixpoint do not depend
      // on it), so no block scan
      for (int base = rs; base <= R; base += kPT) {
        const int a = base + tid;
        int32_t cnt = 0;
        if (a <= R && useW) {
          const int32_t xa = W.rx1[a - rs], wa = W.rwd[a - rs];
          for (int b = a + 2; b <= R && W.rx1[b - rs] - xa < wa; b++) cnt++;
        } else if (a <= R) {
          const int32_t xa = xs1[a], wa = wd[a];
          for (int b = a + 2; b <= R && xs1[b] - xa < wa; b++) cnt++;
        }
        const int32_t inc = warp_incl_sum(cnt, lane);
        const int32_t wtot = __shfl_sync(0xffffffffu, inc, 31);
        int32_t wbase = 0;
        if (lane == 31 && wtot > 0) wbase = atomicAdd(&S.npairs, wtot);
        wbase = __shfl_sync(0xffffffffu, wbase, 31);
        if (a <= R && cnt > 0) {
          int32_t p = wbase + inc - cnt;
          for (int b = a + 2; b < a + 2 + cnt; b++, p++) {
            if (p < kPairSm) {  // the row's first pairs stay in shared memory
              SP.a[p] = a;
              SP.b[p] = b;
            } else if (p < pair_cap) {
              pa[p] = a;
              pb[p] = b;
            }
          }
        }
      }
      pk_sync();
      if (S.npairs > pair_cap) {  // (uniform)
        if (tid == 0) {
          S.pair_overflow = 1;
          S.fail = 1;
          atomicOr(&st->capacity, 2);
          atomicMax(&st->pad[0], S.npairs);
        }
        pk_sync();
        break;
      }
      const int32_t np = S.npairs;
      bool plv = false;
      for (int p = wid; p < np; p += kPW) {
        const int a = p < kPairSm ? SP.a[p] : pa[p], b = p < kPairSm ? SP.b[p] : pb[p];
        bool la, lb;
        const int32_t dx = useW ? W.rx1[b - rs] - W.rx1[a - rs] : xs1[b] - xs1[a];
        warp_locks(row + rowofs[a], row + rowofs[b], hd[a], hd[b], dx, lane, la, lb);
        if (lane == 0) {
          const uint8_t bits = (la ? 1 : 0) | (lb ? 2 : 0);
          if (p < kPairSm) SP.lk[p] = bits;
          else plk[p] = bits;
          plv |= bits != 0;
        }
      }
      if (np > 0) anypl = pk_sync_or(plv);  // (np is uniform: no pairs, no barrier)
    }
    const int32_t np = S.npairs;
    phase_mark(2);

    // per-configuration geometry of chart (window index i, sorted s): X
    auto cfgX = [&](int cfg, int i) -> int32_t {
      const int f = cfg >> 1, dir = cfg & 1;
      const int hc = f ? hc1 : hc0;
      const int32_t xl = hc ? W.rx1[i] : W.rx0[i];
      const int32_t Wd = W.rwd[i];
      return dir ? (f ? kb : Wp) - xl - Wd : (f ? ka : 0) + xl;
    };

    // A chart's largest BottomEdge is its dilated height Hd (the footprint
    // contains the chart, whose lowest point lies in some column, and never
    // exceeds Hd; D11, D13 -- checked on the oracle's footprints), so the
    // score max_j (Y + BottomEdge_j) of a chart is Y + Hd: the push needs no
    // BottomEdge reduction.  One-window rows load Hd here, consumed by the
    // score (the load's latency hides behind the push).
    const int32_t hd_mine = (one && tid <= endA - rs) ? hd[rs + tid] : 0;
    // ---- push: Y = max over covered columns of F - TopEdge ----
    for (int ws0 = rs; ws0 <= endA; ws0 += kRW) {
      const int we = min(endA + 1, ws0 + kRW), nwin = we - ws0;
      stage(ws0, we);
      if (!(ws0 == rs && one && !prefix_mode)) {  // (else the fold initialised them)
        for (int k = tid; k < nwin; k += kPT) {
#pragma unroll
          for (int q = 0; q < 4; q++) W.rY[q * kRW + k] = INT32_MIN;
        }
        pk_sync();
      }
      phase_mark(8);
      const uint32_t* pr = g_pg ? col : W.prof - g_a0;
      // flattened (chart, column) runs (see walk()); per chart segment the
      // configurations' frontline pointers are set once and the column loop is
      // specialised on 2 / 4 configurations (L->R reads F[X + j], R->L reads
      // F[X + Wd - 1 - j])
      {
        const int32_t base0 = W.rx0[0];
        const int32_t T = W.rx0[nwin - 1] - base0 + W.rwd[nwin - 1];
        const int32_t C = ((T + kPT - 1) / kPT) | 1;
        int32_t t = tid * C;
        const int32_t tend = min(T, t + C);
        int i = 0;
        if (t < tend) {
          int lo = 0, hi = nwin - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (W.rx0[mid] - base0 <= t) lo = mid;
            else hi = mid - 1;
          }
          i = lo;
        }
        while (t < tend) {
          const int32_t Wd = W.rwd[i];
          const int32_t j0 = t - (W.rx0[i] - base0);
          const int32_t j1 = min(Wd, j0 + (tend - t));
          const uint32_t* pc = pr + W.rco[i];
          const int32_t* f0 = F + cfgX(0, i);
          const int32_t* f1 = F + cfgX(1, i) + Wd - 1;
          int32_t m0 = INT32_MIN, m1 = INT32_MIN, m2 = INT32_MIN, m3 = INT32_MIN;
          const bool four = knee_ok && ws0 + i <= endK;
          if (four) {
            const int32_t* f2 = F + cfgX(2, i);
            const int32_t* f3 = F + cfgX(3, i) + Wd - 1;
            #pragma unroll 4
            for (int32_t j = j0; j < j1; j++) {
              const int32_t top = lo16(pc[j]);
              m0 = max(m0, f0[j] - top);
              m1 = max(m1, f1[-j] - top);
              m2 = max(m2, f2[j] - top);
              m3 = max(m3, f3[-j] - top);
            }
          } else if (pdir >= 0) {  // prefix row: its one direction (m0 holds it)
            const int32_t* fp = pdir ? f1 : f0;
            const int32_t step = pdir ? -1 : 1;
            #pragma unroll 4
            for (int32_t j = j0; j < j1; j++) m0 = max(m0, fp[step * j] - lo16(pc[j]));
          } else {
            #pragma unroll 4
            for (int32_t j = j0; j < j1; j++) {
              const int32_t top = lo16(pc[j]);
              m0 = max(m0, f0[j] - top);
              m1 = max(m1, f1[-j] - top);
            }
          }
          wk += (unsigned long long)((four ? 4 : pdir >= 0 ? 1 : 2) * (j1 - j0));
          if (pdir >= 0) {
            atomicMax(&W.rY[pdir * kRW + i], m0);
          } else {
            atomicMax(&W.rY[i], m0);
            atomicMax(&W.rY[kRW + i], m1);
          }
          if (four) {
            atomicMax(&W.rY[2 * kRW + i], m2);
            atomicMax(&W.rY[3 * kRW + i], m3);
          }
          t += j1 - j0;
          i++;
        }
      }
      pk_sync();
      if (one) continue;  // Y stays in shared memory for Alg. 1, score and commit
      for (int k = tid; k < nwin; k += kPT) {
        const int s = ws0 + k;
        const int na = (knee_ok && s <= endK) ? 4 : 2;
        for (int q = 0; q < na; q++) __stcg(&Yc[(int64_t)q * n + s], W.rY[q * kRW + k]);
      }
      pk_sync();
    }
    phase_mark(3);
    // ---- Alg. 1 CorrectYOffsets over adjacent + non-adjacent pairs ---------
    {
      int c0 = hc0 ? 0 : 2, c1 = (knee_ok && hc1) ? 4 : 2;  // HC configs [c0, c1)
      if (pdir >= 0) { c0 = pdir; c1 = pdir + 1; }  // (prefix rows: HC on, one direction)
      // (no lock bit among the row's pairs: every pass would change nothing)
      if (!one || prefix_mode) anylock = true;
      if (c1 > c0 && (anylock || anypl)) {
        const int32_t per = (endA - rs) + (adj_only ? 0 : np);  // adjacent pairs + list
        const int nitems = (c1 - c0) * per;
        // item -> (Ya, Yb, lock bits); with <= 2 items per thread they are
        // resolved once and kept in registers across the fixpoint iterations
        auto item = [&](int it, int32_t*& Ya, int32_t*& Yb, int& bits) -> bool {
          const int cfg = c0 + it / per;
          const int q = it % per;
          const int32_t endc = S.end_cfg[cfg];
          int a, b;
          if (q < endA - rs) {
            a = rs + q;
            b = a + 1;
            if (b > endc) return false;
            bits = useW ? W.rlk[a - rs] : lk[a];
          } else {
            const int p = q - (endA - rs);
            a = p < kPairSm ? SP.a[p] : pa[p];
            b = p < kPairSm ? SP.b[p] : pb[p];
            if (b > endc) return false;
            bits = p < kPairSm ? SP.lk[p] : plk[p];
          }
          Ya = one ? &W.rY[cfg * kRW + (a - rs)] : &Yc[(int64_t)cfg * n + a];
          Yb = one ? &W.rY[cfg * kRW + (b - rs)] : &Yc[(int64_t)cfg * n + b];
          return bits != 0;
        };
        auto relax = [&](int32_t* Ya, int32_t* Yb, int bits, int flag) {
          const int32_t ya = one ? *(volatile int32_t*)Ya : __ldcg(Ya);
          const int32_t yb = one ? *(volatile int32_t*)Yb : __ldcg(Yb);
          bool ch = false;
          if ((bits & 1) && ya < yb) { atomicMax(Ya, yb); ch = true; }
          if ((bits & 2) && yb < ya) { atomicMax(Yb, ya); ch = true; }
          return ch;
        };
        const bool cached = nitems <= 2 * kPT;
        int32_t *ya0 = nullptr, *yb0 = nullptr, *ya1 = nullptr, *yb1 = nullptr;
        int bits0 = 0, bits1 = 0;
        bool v0 = false, v1 = false;
        if (cached) {
          if (tid < nitems) v0 = item(tid, ya0, yb0, bits0);
          if (tid + kPT < nitems) v1 = item(tid + kPT, ya1, yb1, bits1);
        }
        // one barrier per pass, which also ORs the threads' "raised something"
        // (the items read only values published before Alg. 1: no setup barrier)
        for (int iter = 0;; iter++) {
          bool ch = false;
          if (cached) {
            if (v0) ch |= relax(ya0, yb0, bits0, 0);
            if (v1) ch |= relax(ya1, yb1, bits1, 0);
          } else {
            for (int it = tid; it < nitems; it += kPT) {
              int32_t *Ya, *Yb;
              int bits;
              if (item(it, Ya, Yb, bits)) ch |= relax(Ya, Yb, bits, 0);
            }
          }
          const bool any = pk_sync_or(ch);
#ifdef TABI_PHASE_TRACE
          if (tid == 0 && jslot == 0) atomicAdd(&st->rph[7], 1ull);  // Alg. 1 passes
#endif
          if (!any) break;
        }
      }
    }
    phase_mark(4);
    // ---- score: max over covered columns of Y + BottomEdge ----
    // Y is constant per chart, so the max over its columns is Y + the chart's
    // largest BottomEdge = Y + Hd (see the push): one pass over the row's
    // charts instead of a column walk.  Multi-window rows walk.
    {
      int32_t nm[4] = {INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN};
      if (one) {
        const int nwin = endA - rs + 1;
        for (int k = tid; k < nwin; k += kPT) {
          const int na = (knee_ok && rs + k <= endK) ? 4 : 2;
          const int32_t hdk = k == tid ? hd_mine : hd[rs + k];
          for (int q = 0; q < na; q++) nm[q] = max(nm[q], W.rY[q * kRW + k] + hdk);
        }
      }
      for (int ws0 = rs; ws0 <= endA && !one; ws0 += kRW) {
        const int we = min(endA + 1, ws0 + kRW), nwin = we - ws0;
        stage(ws0, we);
        for (int k = tid; k < nwin && !one; k += kPT) {
          const int s = ws0 + k;
          const int na = (knee_ok && s <= endK) ? 4 : 2;
          for (int q = 0; q < na; q++) W.rY[q * kRW + k] = __ldcg(&Yc[(int64_t)q * n + s]);
        }
        pk_sync();
        const uint32_t* pr = g_pg ? col : W.prof - g_a0;
        int32_t Yv[4];
        int nact = 0;
        walk(
            W, nwin,
            [&](int i, int32_t, int32_t) {
              nact = (knee_ok && ws0 + i <= endK) ? 4 : 2;
              for (int q = 0; q < 4; q++) Yv[q] = q < nact ? W.rY[q * kRW + i] : 0;
            },
            [&](int i, int32_t j) {
              const int32_t bot = hi16(pr[W.rco[i] + j]);
#pragma unroll
              for (int q = 0; q < 4; q++)
                if (q < nact) nm[q] = max(nm[q], Yv[q] + bot);
              wk += nact;
            },
            [&](int) {});
        pk_sync();
      }
      for (int q = 0; q < ncfg; q++) {
        const int32_t v = warp_max(nm[q]);
        if (lane == 0) atomicMax(&S.newmax[q], v);
      }
    }
    pk_sync();
    phase_mark(5);
    // ---- hierarchical selection -----------------------------------
    // (every thread: the inputs were published by the score's barrier and stay
    // unchanged until the row end, where thread 0 stores the new maximum)
    int cfg;
    int32_t fmax_new;
    {
      const int32_t sw0 = max(S.fmax, S.newmax[0]), sw1 = max(S.fmax, S.newmax[1]);
      int d0 = sw1 < sw0 ? 1 : 0;   // ties -> left to right
      if (no_bal) d0 = S.rows & 1;  // static alternation (ablation)
      // prefix rows: FastAtlas alternation, one L->R row then two R->L
      if (prefix_mode) d0 = (S.prefix_rows % 3 == 0) ? 0 : 1;
      cfg = d0;
      if (knee_ok) {
        const int32_t sk0 = max(S.conc_max, S.newmax[2]), sk1 = max(S.conc_max, S.newmax[3]);
        const int d1 = sk1 < sk0 ? 1 : 0;
        const int32_t swk = max(S.fmax, S.newmax[2 + d1]);
        if (swk <= (d0 ? sw1 : sw0) - 1) cfg = 2 + d1;  // "at least marginally smaller"
      }
      fmax_new = max(S.fmax, S.newmax[cfg]);
    }
    // ---- commit: F <- max(F, Y + BottomEdge); record placements ------------
    const int f = cfg >> 1, dir = cfg & 1;
    const int32_t endS = S.end_cfg[cfg];
    // prefix rows: the next row's slot offset for its row-top prefetch (the
    // load's latency hides behind the commit walk)
    const int32_t pf_next = (prefix_mode && tid == 0 && endS + 1 < n) ? colofs[endS + 1] : -1;
    // ---- FindKnee after an atlas-fold row: the height
    // drops of the row's charts, issued here so their loads overlap the commit
    // walk (the commit's last barrier publishes S.knee_key) ------------------
    if (f == 0 && !no_bal && !prefix_mode) {
      for (int t = rs + tid; t < endS; t += kPT) {
        const int32_t h0 = useW ? W.rhs[t - rs] : hsorted[t];
        const int32_t h1 = useW ? W.rhs[t + 1 - rs] : hsorted[t + 1];
        const int64_t d = (int64_t)h0 - h1;
        if (10 * d >= (int64_t)pp.H * TABI_UNITS && 5 * d >= h0) {
          const unsigned long long key =
              ((unsigned long long)d << 32) | (unsigned long long)(0x7fffffff - t);
          atomicMax(&S.knee_key, key);
        }
      }
    }
    if (ef) {  // 2 x polygon area of the row's charts (published by the walk's barrier)
      long long pa = 0;
      for (int t = rs + tid; t <= endS; t += kPT) pa += lz->area[t];
      pa = warp_sum64(pa);
      if (lane == 0 && pa) atomicAdd((unsigned long long*)&S.placed, (unsigned long long)pa);
    }
    for (int ws0 = rs; ws0 <= endS; ws0 += kRW) {
      const int we = min(endA + 1, ws0 + kRW), nwin = min(we, endS + 1) - ws0;
      stage(ws0, we);
      if (!one) {
        for (int k = tid; k < nwin; k += kPT) W.rY[k] = __ldcg(&Yc[(int64_t)cfg * n + ws0 + k]);
        pk_sync();
      }
      phase_mark(9);
      const uint32_t* pr = g_pg ? col : W.prof - g_a0;
      const int32_t* rYc = one ? W.rY + cfg * kRW : W.rY;
      int32_t* const Fs = F;
      long long dsum = 0;  // early fail: this thread's increase of sum_x F[x]
      walk(
          W, nwin,
          [&](int i, int32_t j0, int32_t j1) {
            const int32_t Xc = cfgX(cfg, i), Yv = rYc[i], Wd = W.rwd[i];
            if (j0 == 0) {
              const int s = ws0 + i;
              Xo[s] = Xc;
              Yo[s] = Yv;
              mir[s] = (uint8_t)dir;
            }
            // the whole run of this chart at once: F <- max(F, Y + BottomEdge)
            const uint32_t* pc = pr + W.rco[i];
            if (ef) {  // each raise returns the value it replaced: the increases telescope
              int32_t* fp = dir ? Fs + Xc + Wd - 1 : Fs + Xc;
              const int step = dir ? -1 : 1;
              for (int32_t j = j0; j < j1; j++) {
                const int32_t v = Yv + hi16(pc[j]);
                const int32_t o = atomicMax(fp + step * j, v);
                if (v > o) dsum += v - o;
              }
            } else if (dir) {
              int32_t* fp = Fs + Xc + Wd - 1;
              #pragma unroll 4
              for (int32_t j = j0; j < j1; j++) atomicMax(fp - j, Yv + hi16(pc[j]));
            } else {
              int32_t* fp = Fs + Xc;
              #pragma unroll 4
              for (int32_t j = j0; j < j1; j++) atomicMax(fp + j, Yv + hi16(pc[j]));
            }
            wk += (unsigned long long)(j1 - j0);
          },
          [&](int, int32_t) {}, [&](int) {});
      if (ef) {
        dsum = warp_sum64(dsum);
        if (lane == 0 && dsum) atomicAdd((unsigned long long*)&S.sumF, (unsigned long long)dsum);
      }
      pk_sync();
    }
    phase_mark(6);
    if (tid == 0) {
      if (prefix_mode) S.prefix_rows++;
      else S.rows++;
#ifdef TABI_PHASE_TRACE
      if (rd.flags && jslot == 0 && S.rows == 1 && !prefix_mode) st->tfirst[3] = gtime();
#endif
      if (f == 1) S.knee_rows++;
      S.fmax = fmax_new;
      if (f == 0 && !no_bal && !prefix_mode) {
        if (S.knee_key != 0ull) {
          const int t = 0x7fffffff - (int)(S.knee_key & 0xffffffffull);
          S.knee_valid = 1;
          S.knee_ltr = dir == 0;
          const int32_t xk = useW ? cfgX(cfg, t - rs) : Xo[t];
          S.knee_left = xk;
          S.knee_right = xk + (useW ? W.rwd[t - rs] : wd[t]);
          S.knees_found++;
        } else {
          S.knee_valid = 0;
        }
        S.knee_key = 0ull;  // (consumed: the next FindKnee starts from zero)
      }
      if (S.fmax > Hp) S.fail = 1;  // overflow below the atlas bottom
      S.row_start = endS + 1;
      if (ef && !S.fail && S.row_start < n) {
        // R8: the charts still to place lie below the frontline, disjoint, in
        // [F(x), H') per column: their polygon area (2 x area in units^2 at
        // scale 1, x (m / (M 256))^2 / 2) cannot exceed sum_x (H' - F[x])
        const i128 rem = (i128)(lz->atot - S.placed);
        const i128 freeA = (i128)Wp * Hp - S.sumF;
        const i128 SCm2 = (i128)pp.M * TABI_UNITS * pp.M * TABI_UNITS;
        if (rem * m * m > 2 * SCm2 * freeA) S.fail = 1;
      }
      if ((rd.flags || lz) && pp.early && wj < jslot) S.abort = 1;  // checked at the next row start
      const int nx = endS + 1;  // the next row's slot offset, if this fold saw it
      S.next_a0 = prefix_mode ? pf_next
                  : (S.w_fold && nx < n && nx < S.fold_hi && nx - rs < kRW) ? W.rco[nx - rs] : -1;
    }
    pk_sync();
    phase_mark(7);
  }
  if (pf_pending) {  // a failed row left its prefetch in flight: let it land first
    mbar_wait(&S.mbar, phase);
    phase ^= 1u;
  }
  if (tid == 0)
    for (int i = 0; i < 10; i++) atomicAdd(&st->ph[i], ph[i]);
  for (int o = 16; o > 0; o >>= 1) wk += __shfl_xor_sync(0xffffffffu, wk, o);
  if (lane == 0) atomicAdd(&st->work_pack, wk);
  if (rd.flags && tid == 0) atomicMax(&st->tr[2], gtime());
  if (rd.flags && S.fail && tid == 0) {
    // fused mode: this candidate's remaining tiles are no longer needed -- the
    // rasterizers drop them (a hint: a relaxed flag read at each item fetch)
    *(volatile int32_t*)(rd.flags + 2 * (int64_t)pp.B * n + pp.B + jslot) = 1;
  }
  // a beaten candidate stays "not evaluated" (its record keeps the reset zeros)
  if (tid == 0 && !S.switched && !S.abort) {
    Cand cd{S.fail ? 0 : 1, S.fmax, S.rows, S.knees_found, S.knee_rows, 0, 0, 1, -1, 0, 0ull, 0ull};
    // sequential fused mode: announce the success so lower candidates stop
    if (!S.fail && rd.flags && pp.early) atomicMin(&st->win_j, jslot);
    if (prefix_mode) {  // keep the tail's area (written by the layout kernel)
      const Cand prev = cands[slot];
      cd.prefix_rows = S.prefix_rows;
      cd.p = pp.T.p[slot];
      cd.switched_at = pp.T.r0[slot];
      cd.apre_lo = prev.apre_lo;
      cd.apre_hi = prev.apre_hi;
    }
    cands[slot] = cd;
  }
}

__global__ void __launch_bounds__(kNT, 1)
pack_kernel(PackParams pp, const int32_t* __restrict__ colofs, const int32_t* __restrict__ rowofs,
            const uint32_t* __restrict__ dcol, const uint32_t* __restrict__ drow,
            const int32_t* __restrict__ wd_all, const int32_t* __restrict__ hd_all,
            const int32_t* __restrict__ off_all, const uint8_t* __restrict__ lock_all,
            const int32_t* __restrict__ hsorted, const int32_t* __restrict__ cand_bad,
            int32_t* scratch, int64_t pair_cap, int32_t* Xo_all, int32_t* Yo_all, uint8_t* mir_all,
            Cand* cands, Status* st, int32_t prof_cap) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int m = wave_m(pp, st->wave, st->pad[2], st->b0, blockIdx.x);
  if (m == 0) return;
  packer(pp, colofs, rowofs, dcol, drow, wd_all, hd_all, off_all, lock_all, hsorted, cand_bad,
         scratch, pair_cap, Xo_all, Yo_all, mir_all, cands, st, prof_cap, m, m - 1, blockIdx.x,
         Ready{nullptr, 0, nullptr, nullptr}, dsm);
}

// ---- fused persistent kernel: one cooperative launch per candidate wave ----
// CTAs [0, B) are packers (one candidate each); every other CTA runs kRG
// independent raster groups of kRGT threads (named barriers 1..kRG), each
// taking tiles of kTCF sorted charts of one candidate from a work queue in
// sorted (tile-major) order: footprints, then the adjacent-pair offsets and
// locks.  Each tile is published with a release flag that the packers acquire
// before reading it.  K3/K3b thus run on the SMs the packers leave idle and
// overlap with the row loop; no host round trip inside the wave.  Several
// groups per SM hide the latency of one group's setup / barrier phases the
// way several resident CTAs do in the split kernels.
#ifndef TABI_TOP_FIRST
#define TABI_TOP_FIRST 0
#endif
// sequential mode: 1 queues the top candidate's tiles before the others'; 0
// (default) tile-major for every slot, as in hybrid mode -- the top
// candidate often fails (C3 at rho 1.5: 0.303 -> 0.292 ms)
constexpr bool kTopFirst = TABI_TOP_FIRST != 0;
constexpr int kRG = kFusedGroups;   // raster groups per CTA
constexpr int kRGT = kNT / kRG;     // threads per group (8 per chart in setup)
constexpr int kTCF = kRGT / 8;      // charts per raster tile
constexpr int kRGW = kRGT / 32;    // warps per group
constexpr int kRawF = 16384 / kRG;  // raw cells per group chunk (64 KB per CTA)
static_assert(kTCF * 8 == kRGT, "setup maps 8 threads to a chart");
static_assert(kTCF >= kFusedTileCharts, "prep_kernel's tiles must fit a raster group");

struct GroupSync {
  int id;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kRGT) : "memory");
  }
};

struct RasterArgs {
  Proxies P;
  const int32_t* perm;
  int32_t* wd;
  int32_t* hd;
  int32_t* off;
  uint8_t* lock;
  int32_t* cand_bad;
  uint32_t* dcol;
  uint32_t* drow;
  int32_t* rdy;
  const int32_t* tstart;  // [T + 1] tile boundaries (prep_kernel)
  const int32_t* tix;     // [n] tile of each sorted position
};


// per-group carve of the dynamic shared memory
__host__ __device__ __forceinline__ size_t group_bytes(int k) {
  return r16(sizeof(k3::ChartK3) * kTCF) + r16(4 * kTCF) + 2 * r16(4 * (kTCF + 1)) +
         r16(4 * kTCF) + r16(32) + r16(4 * (2 * kRGW + 4)) + r16((size_t)4 * kTCF * 4 * k) + r16(4 * (size_t)kRawF);
}


__global__ void __launch_bounds__(kNT, 1)
fused_kernel(PackParams pp, const int32_t* __restrict__ colofs, const int32_t* __restrict__ rowofs,
             const int32_t* __restrict__ hsorted, int32_t* scratch, int64_t pair_cap,
             int32_t* Xo_all, int32_t* Yo_all, uint8_t* mir_all, Cand* cands, Status* st,
             int32_t prof_cap, RasterArgs ra) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int T = st->ntiles;
  // wave slots in use: prep_kernel narrows wave 0 (Status::b0); the CTAs of
  // unused slots rasterize instead
  const int Bw = st->wave == 0 ? st->b0 : pp.B;
  if (threadIdx.x == 0) atomicMin(&st->tr[0], gtime());
  if ((int)blockIdx.x < Bw) {
    const int m = wave_m(pp, st->wave, st->pad[2], st->b0, blockIdx.x);
    if (m == 0) return;
    packer(pp, colofs, rowofs, ra.dcol, ra.drow, ra.wd, ra.hd, ra.off, ra.lock, hsorted,
           ra.cand_bad, scratch, pair_cap, Xo_all, Yo_all, mir_all, cands, st, prof_cap, m, m - 1,
           blockIdx.x, Ready{ra.rdy, T, ra.tstart, ra.tix}, dsm);
    return;
  }
  // ---- rasterizer role ----
  if (st->bad_chart != INT32_MAX || st->capacity) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int grp = tid / kRGT, gt = tid % kRGT, gw = gt >> 5;
  const GroupSync gsync{1 + grp};
  const int k = pp.k;
  unsigned char* p = dsm + group_bytes(k) * grp;
  k3::ChartK3* CH = (k3::ChartK3*)carve(p, sizeof(k3::ChartK3) * kTCF);
  int32_t* cells = (int32_t*)carve(p, 4 * kTCF);
  int32_t* cpre = (int32_t*)carve(p, 4 * (kTCF + 1));
  int32_t* opre = (int32_t*)carve(p, 4 * (kTCF + 1));
  int32_t* big = (int32_t*)carve(p, 4 * kTCF);
  int32_t* misc = (int32_t*)carve(p, 32);
  int32_t* red = (int32_t*)carve(p, 4 * (2 * kRGW + 4));  // group reductions (big pairs)
  int32_t* tabs = (int32_t*)carve(p, (size_t)4 * kTCF * 4 * k);
  uint32_t* raw = (uint32_t*)carve(p, 4 * (size_t)kRawF);
  p = dsm + group_bytes(k) * kRG;  // per-warp large-chart state
  k3::ChartK3* CW = (k3::ChartK3*)carve(p, sizeof(k3::ChartK3) * kNW);
  int32_t* wtab = (int32_t*)carve(p, (size_t)4 * kNW * 4 * k);
  const int32_t m_hi = st->pad[2];
  const int NB = T * Bw;
  const int64_t SCm = (int64_t)pp.M * TABI_UNITS;
#ifdef TABI_PHASE_TRACE
  unsigned long long rph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long rt = clock64();
  auto rmark = [&](int i) {
    if (gt == 0) {
      const long long t1 = clock64();
      rph[i] += (unsigned long long)(t1 - rt);
      rt = t1;
    }
  };
#else
  auto rmark = [](int) {};
#endif
  // the first G items go to the G raster groups statically (no queue round
  // trip before the first -- most urgent -- tiles); the queue hands out the rest
  const int G = ((int)gridDim.x - Bw) * kRG;
  // (constant for the launch: loaded once -- the loop's atomics would make
  // the compiler reload them every tile)
  const int32_t wave = st->wave, b0 = st->b0;
  int32_t* const done_cnt0 = ra.rdy + 2 * (int64_t)pp.B * pp.n;
  // Tile-major over the wave's slots (kTopFirst: in sequential mode the
  // highest candidate's tiles first, then the others tile-major).
  auto item_tj = [&](int it, int& t, int& j) {
    if (!(kTopFirst && pp.early) || Bw == 1) {
      t = it / Bw;
      j = it % Bw;
    } else if (it < T) {
      t = it;
      j = 0;
    } else {
      t = (it - T) / (Bw - 1);
      j = 1 + (it - T) % (Bw - 1);
    }
  };
  // (leader) an item's drop hint and tile bounds: items of a candidate that
  // failed (its packer has exited), and in sequential mode of candidates below
  // a successful one, are dropped -- the top candidate's (slot 0) never are
  auto probe = [&](int it, int& drop, int32_t& ts0, int32_t& ts1) {
    drop = 1;
    ts0 = ts1 = 0;
    if (it >= NB) return;
    int t, j;
    item_tj(it, t, j);
    drop = (pp.early && j > 0 && *(volatile int32_t*)&st->win_j < j) ||
           *(volatile int32_t*)(done_cnt0 + pp.B + j) != 0;
    ts0 = ra.tstart[t];
    ts1 = ra.tstart[t + 1];
  };
  int first_it = ((int)blockIdx.x - Bw) * kRG + grp;
  // the claimer (lane 0 of the group's last warp) claims the next item during
  // a tile's pair phase and leaves it, its drop hint and its tile bounds in
  // misc[0], misc[4..6] with misc[7] = 1; the leader (gt == 0) claims at the
  // loop top only when nothing was left there
  const int gclaim = 32 * (kRGW - 1);
  static_assert(kRGW >= 2, "pair phase: warp 0 boundary pairs, the rest internal pairs");
  if (gt == 0) misc[7] = 0;
  while (true) {
    if (gt == 0) {
      if (misc[7] == 0) {  // the first item, or the one after a dropped item
        const int it0 = first_it >= 0 ? first_it : G + atomicAdd(&st->work_next, 1);
        int drop;
        int32_t ts0, ts1;
        probe(it0, drop, ts0, ts1);
        misc[0] = it0;
        misc[4] = drop;
        misc[5] = ts0;
        misc[6] = ts1;
      }
      misc[7] = 0;
    }
    first_it = -1;
    gsync();
    const int it = misc[0];
    const bool dropped = misc[4] != 0;
    const int s0 = misc[5], nt = misc[6] - s0;
    rmark(0);
    if (it >= NB) {
      if (gt == 0) atomicMax(&st->tr[1], gtime());
#ifdef TABI_PHASE_TRACE
      if (gt == 0)
        for (int i = 0; i < 8; i++) atomicAdd(&st->rph[i], rph[i]);
#endif
      break;
    }
    int t, j;
    item_tj(it, t, j);
    const int m = dropped ? 0 : wave_m(pp, wave, m_hi, b0, j);
    if (m == 0) {
      gsync();  // (everyone has read misc before the leader rewrites it)
      continue;
    }
    const k3::Scale sc{m, SCm, 0};
    // (g <= kDilMax: the raw buffer is free and holds the tile's dilated row
    // footprints for its internal pair offsets)
    const bool stash = pp.g <= k3::kDilMax;
    k3::tile_raster<kTCF, kRGT, kRawF>(ra.P, ra.perm, pp, colofs, rowofs, ra.dcol, ra.drow, ra.wd,
                                       ra.hd, ra.cand_bad, m - 1, s0, sc, CH, cells, cpre, opre,
                                       &misc[1], big, tabs, raw, nt, gt, gsync,
                                       [&](int w) {
                                         if (w == 0) rmark(6);
#ifdef TABI_PHASE_TRACE
                                         if (gt == 0 && t == 0 && j == 0)
                                           st->tfirst[w == 0 ? 5 : 4] = gtime();
#endif
                                       },
                                       stash ? raw : nullptr, kRawF);
    const bool stashed = stash && cpre[nt] <= kRawF;
    rmark(1);
#ifdef TABI_PHASE_TRACE
    if (gt == 0 && t == 0 && j == 0) atomicMax(&st->tfirst[0], gtime());
#endif
    if (pp.g > k3::kDilMax) {  // (uniform; g <= kDilMax hands no chart to this pass)
      for (int ci = gw; ci < nt; ci += kRGW)
        if (big[ci])
          k3::big_chart(ra.P, ra.perm, pp, colofs, rowofs, ra.dcol, ra.drow, m - 1, s0 + ci, sc,
                        CW[wid], wtab + wid * 4 * k, lane);
      gsync();
    }
    rmark(2);
    // Adjacent pairs: the tile's internal pairs here; a boundary pair with a
    // neighbour tile is done by whichever of the two tiles publishes its
    // footprints second (arrival counter per boundary, acq_rel), so no tile
    // waits for another.  rdy[t] reaches 2 once the pairs (s, s + 1) of all
    // s in tile t are done: its internal pairs (+1) and its right boundary (+1;
    // the last tile adds its own zero entry instead).  Every contribution is
    // also added to the slot's done count (2 T once all of its tiles are
    // complete): each is a release pattern (fence + relaxed adds), so the
    // packers' one acquire load of the count that reads 2 T happens-after all
    // of them.
    int32_t* fl = ra.rdy + (int64_t)j * T;
    int32_t* arr = ra.rdy + (int64_t)pp.B * pp.n + (int64_t)j * T;  // boundary t | t+1
    int32_t* done_cnt = done_cnt0 + j;
    // both arrivals in one instruction (lane 0 left, lane 1 right boundary)
    int32_t arrived = 0;
    if (gt < 2 && (gt == 0 ? t > 0 : t < T - 1)) arrived = atom_add_acq_rel(arr + t - 1 + gt, 1);
    // claim the next item now: its queue round trip overlaps the pair offsets
    int nx_it = -1;
    if (gt == gclaim) nx_it = G + atomicAdd(&st->work_next, 1);
    if (gt == 0) atomicAdd(&st->tr[5], 1ull);  // tiles rasterized
    if (gw == kRGW - 1) {  // work accounting: footprint entries of the tile (from smem)
      unsigned long long pe = 0;
      for (int ci = lane; ci < nt; ci += 32)
        pe += (unsigned long long)(CH[ci].ws + CH[ci].hs + 4 * pp.g);
      for (int o = 16; o > 0; o >>= 1) pe += __shfl_xor_sync(0xffffffffu, pe, o);
      if (lane == 0) atomicAdd(&st->work_prof, pe);
    }
    // pairs with many shared rows (the tallest charts, first in the order and
    // first needed by the packers) go to the whole group, one after another;
    // the rest one warp each.  Only in tiles with fewer charts than half the
    // group's warps: otherwise warp-per-pair already keeps every warp busy.
    auto big_pair = [&](int s) {
      if (2 * nt > kRGW || s + 1 >= pp.n) return false;
      const int64_t b = (int64_t)(m - 1) * pp.n;  // boundary pairs: heights from HBM
      const int32_t ha = s >= s0 ? CH[s - s0].hs : ra.hd[b + s] - 2 * pp.g;
      const int32_t hb = s + 1 < s0 + nt ? CH[s + 1 - s0].hs : ra.hd[b + s + 1] - 2 * pp.g;
      return min(ha, hb) >= 512;
    };
    auto warp_pair = [&](int s) {
      const int a = s - s0;
      if (stashed && a >= 0 && a + 1 < nt && CH[a].small && CH[a + 1].small) {
        // both charts in this tile: their row footprints from shared memory
        const int64_t b = (int64_t)(m - 1) * pp.n + s;
        k3::pair_rows(raw + cpre[a], raw + cpre[a + 1], CH[a].hs + 2 * pp.g, CH[a + 1].hs + 2 * pp.g,
                      CH[a].ws + 2 * pp.g, ra.off + b, ra.lock + b, lane);
      } else {
        k3::pair_offset(pp, rowofs, ra.drow, ra.wd, ra.hd, ra.off, ra.lock, m - 1, s, lane);
      }
    };
    auto leave_next = [&]() {  // (claimer) the next item for the loop top
      if (gt == gclaim) {
        int drop;
        int32_t ts0, ts1;
        probe(nx_it, drop, ts0, ts1);
        misc[0] = nx_it;
        misc[4] = drop;
        misc[5] = ts0;
        misc[6] = ts1;
        misc[7] = 1;
      }
    };
    // (only tiles of fewer than kRGW / 2 charts can hold a big pair)
    const bool may_big = 2 * nt <= kRGW;
    // internal pairs (s, s + 1) of the tile (the last tile: up to the zero
    // entry of position n - 1)
    const int hi = (t == T - 1) ? pp.n - 1 : s0 + nt - 2;
    const int32_t vint = t == T - 1 ? 2 : 1;
    if (!may_big) {
      // warp 0: the boundary pairs this tile arrived second at (its lanes 0 / 1
      // hold the arrivals), each published as soon as it is done; the other
      // warps: the internal pairs, published together after the group barrier
      if (gw == 0) {
        const bool needL = t > 0 && __shfl_sync(0xffffffffu, arrived, 0) == 1;
        const bool needR = t < T - 1 && __shfl_sync(0xffffffffu, arrived, 1) == 1;
        __syncwarp();  // (orders the lanes' neighbour reads after lanes 0 / 1's acquires)
        for (int q = 0; q < 2; q++) {
          if (!(q == 0 ? needL : needR)) continue;
          warp_pair(q == 0 ? s0 - 1 : s0 + nt - 1);
          __syncwarp();
          if (lane == 0) {
            fence_acq_rel_gpu();
            red_add_relaxed(fl + (q == 0 ? t - 1 : t), 1);
            red_add_relaxed(done_cnt, 1);
          }
        }
      } else {
        for (int s = s0 + gw - 1; s <= hi; s += kRGW - 1) warp_pair(s);
      }
      leave_next();
      gsync();
      rmark(3);
#ifdef TABI_PHASE_TRACE
      if (gt == 0 && t == 0 && j == 0) st->tfirst[6] = gtime();
#endif
      if (gt == 0) {
        fence_acq_rel_gpu();
        red_add_relaxed(fl + t, vint);
        red_add_relaxed(done_cnt, vint);
      }
    } else {
      // few (tall) charts: wait for the arrivals, then every pair -- a tall
      // one by the whole group -- and publish them together
      if (gt < 2) misc[2 + gt] = arrived == 1 && (gt == 0 ? t > 0 : t < T - 1);
      leave_next();
      gsync();
      rmark(3);
#ifdef TABI_PHASE_TRACE
      if (gt == 0 && t == 0 && j == 0) st->tfirst[6] = gtime();
#endif
      const bool needL = misc[2] != 0, needR = misc[3] != 0;
      const int lo = needL ? s0 - 1 : s0;
      const int hh = needR ? s0 + nt - 1 : hi;
      for (int s = lo + gw; s <= hh; s += kRGW)
        if (!big_pair(s)) warp_pair(s);
      for (int s = lo; s <= hh; s++)
        if (big_pair(s))
          k3::pair_offset_group<kRGT>(pp, rowofs, ra.drow, ra.wd, ra.hd, ra.off, ra.lock, m - 1, s,
                                      gt, gsync, red);
      gsync();
      if (gt == 0) {
        const int32_t v = vint + (needR ? 1 : 0);
        fence_acq_rel_gpu();
        red_add_relaxed(fl + t, v);
        if (needL) red_add_relaxed(fl + t - 1, 1);
        red_add_relaxed(done_cnt, v + (needL ? 1 : 0));
      }
    }
    rmark(4);
#ifdef TABI_PHASE_TRACE
    if (gt == 0 && t == 0 && j == 0) st->tfirst[7] = gtime();
    if (gt == 0 && j == 0 && t <= 1) atomicMax(&st->tfirst[1], gtime());
#endif
    rmark(5);
  }
}

// ---- batch mode (tabi_pack_many): a persistent work queue of (atlas,
// candidate) items, one CTA per item, no cross-CTA waiting --------------------
// Item (a, r) evaluates m = m_hi(a) - r, m_hi the atlas's area bound.  The CTA
// rasterizes all of the atlas's footprints at m/M (tile_raster over 64-chart
// tiles, large charts warp by warp) into its own buffers, computes every
// adjacent pair's offset and locks (warp per pair), then runs the packer (the
// same Alg. 4 code as a single pack).  Success: m is the largest successful
// scale (every higher one was evaluated and failed, or is above the exact area
// bound -- SURVEY §3(iii)'s top-down order), so the CTA scatters the
// placements.  Failure: the item (a, r + 1) is appended to the queue.  A CTA
// that draws a ticket past the queue's end waits until the ticket is filled
// or every atlas is decided; items are only ever produced by running CTAs, so
// the queue cannot deadlock.  P:307 "one work group per scale factor" is the
// unit; the batch gives each GPU hundreds of them in flight.
// Batch-kernel rasterization: kBG independent groups of kBGT threads (named
// barriers 1..kBG), each taking every kBG-th tile of kBTC sorted charts, so
// one group's barrier / setup latency hides behind the others' work (the
// packer that follows uses the whole CTA).
#ifndef TABI_BATCH_RG
#define TABI_BATCH_RG 4
#endif
constexpr int kBG = TABI_BATCH_RG;
constexpr int kBGT = kNT / kBG;
constexpr int kBTC = kBGT / 8;
constexpr int kBGW = kBGT / 32;
constexpr int kBRaw = 16384 / kBG;
__host__ __device__ __forceinline__ size_t bgroup_bytes(int k) {
  return r16(sizeof(k3::ChartK3) * kBTC) + r16(4 * kBTC) + 2 * r16(4 * (kBTC + 1)) +
         r16(4 * kBTC) + r16(32) + r16((size_t)4 * kBTC * 4 * k) + r16(4 * (size_t)kBRaw);
}
struct BGroupSync {
  int id;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kBGT) : "memory");
  }
};

__device__ __forceinline__ int32_t ld_acquire_i(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_i(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Idle speculation (batch, carry mode): an undecided atlas of the LPT order
// with fewer than A.spec ranks in flight gets its next rank issued here (warp
// 0 scans 32 order positions per step; a hint skips the leading decided
// ones).  The rank counts as issued BEFORE it is taken, as a continuation is,
// so a completion can never decide the atlas while it is being taken; a taken
// index past the last candidate is completed at once (and decides the atlas
// if it was the last outstanding rank).  Returns the item for every lane, or
// -1.
__device__ __noinline__ int spec_pick(const ManyArgs& A, int lane) {
  const int h0 = *(volatile int32_t*)(A.qctl + 3);
  for (int p0 = h0; p0 < A.E; p0 += 32) {
    const int p = p0 + lane;
    bool dec = true, cand = false;
    int a = 0;
    if (p < A.E) {
      a = A.order[p];
      const AtlasRes& R = A.res[a];
      const Status* st = A.sts + a;
      dec = *(volatile int32_t*)&R.done != 0;
      const int32_t nr = *(volatile int32_t*)&R.next_r;
      cand = !dec && *(volatile int32_t*)&st->win_j == INT32_MAX &&
             *(volatile int32_t*)&st->bad_chart == INT32_MAX &&
             *(volatile int32_t*)&st->capacity == 0 &&
             *(volatile int32_t*)&R.issued - *(volatile int32_t*)&R.completed < A.spec &&
             st->pad[2] - nr >= 1 && nr < 256;
    }
    const unsigned dm = __ballot_sync(0xffffffffu, dec);
    if (lane == 0 && p0 == h0 && (dm & 1u)) {
      const int lead = dm == 0xffffffffu ? 32 : __ffs(~dm) - 1;
      atomicMax(A.qctl + 3, p0 + lead);
    }
    unsigned cm = __ballot_sync(0xffffffffu, cand);
    while (cm) {
      const int src = __ffs(cm) - 1;
      int v = -1;
      if (lane == src) {
        AtlasRes& R = A.res[a];
        Status* st = A.sts + a;
        atomicAdd(&R.issued, 1);
        const int nr = atomicAdd(&R.next_r, 1);
        if (st->pad[2] - nr >= 1 && nr < 256) {
          v = a | (nr << 20);
        } else {
          const int done_now = atomicAdd(&R.completed, 1) + 1;
          if (done_now == *(volatile int32_t*)&R.issued &&
              *(volatile int32_t*)&st->win_j == INT32_MAX && atomicCAS(&R.done, 0, 1) == 0) {
            __threadfence();
            atomicSub(A.qctl + 2, 1);
          }
        }
      }
      v = __shfl_sync(0xffffffffu, v, src);
      if (v >= 0) return v;
      cm &= cm - 1;
    }
  }
  return -1;
}

__global__ void __launch_bounds__(kNT, 1)
many_kernel(PackParams pp0, ManyArgs A, int32_t prof_cap) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ int32_t item_s, outcome_s, skip_s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gcta = blockIdx.x;
  int carry = -1;  // thread 0: the next rank of the atlas this CTA just failed
  const int64_t nm = A.nmax;
  uint32_t* dcol = A.dcol + (int64_t)gcta * pp0.col_cap;
  uint32_t* drow = A.drow + (int64_t)gcta * pp0.row_cap;
  int32_t* wd = A.wd + gcta * nm;
  int32_t* hd = A.hd + gcta * nm;
  int32_t* off = A.off + gcta * nm;
  uint8_t* lock = A.lock + gcta * nm;
  int32_t* scr = A.scratch + (int64_t)gcta * (6 * nm + 3 * A.pair_cap);
  int32_t* X = A.X + gcta * nm;
  int32_t* Y = A.Y + gcta * nm;
  uint8_t* mir = A.mir + gcta * nm;
  Cand* cand = A.cands + gcta;
  int32_t* cbad = A.cand_bad + gcta;
  const int k = pp0.k, g = pp0.g;
  const int64_t SCm = (int64_t)pp0.M * TABI_UNITS;
  // per-CTA timeline (globaltimer ns): start, end of its last item
  if (tid == 0) A.cycles[3 + 2 * gcta] = A.cycles[3 + 2 * gcta + 1] = gtime();
  while (true) {
    if (wid == 0) {
      int v = __shfl_sync(0xffffffffu, carry, 0);  // (carry lives in thread 0)
      if (v < 0) {
        int i = lane == 0 ? atomicAdd(&A.qctl[0], 1) : 0;
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i < A.qcap) {
          while (true) {
            int got = -1, stop = 0;
            if (lane == 0) {
              got = ld_acquire_i(A.q + i);
              if (got < 0) stop = ld_acquire_i(A.qctl + 2) == 0;  // every atlas decided
            }
            got = __shfl_sync(0xffffffffu, got, 0);
            stop = __shfl_sync(0xffffffffu, stop, 0);
            if (got >= 0) { v = got; break; }
            if (stop) break;
            // idle: in carry mode no rank is ever requeued, so an index at or
            // past the tail is never filled -- start the next rank of an
            // undecided atlas instead (speculation that costs an idle SM only)
            if (A.spec > 1 && i >= *(volatile int32_t*)(A.qctl + 1)) {
              v = spec_pick(A, lane);
              if (v >= 0) break;
            }
            __nanosleep(256);
          }
        }
      }
      if (lane == 0) {
      item_s = v;
      // a rank of an atlas already decided, or above a lower rank that won, is
      // skipped -- decided HERE, once, for the whole CTA (other CTAs change
      // these words concurrently, so per-thread reads could disagree)
      if (v >= 0) {
        const int a = v & 0xfffff, r = v >> 20;
        const Status* sa = A.sts + a;
        const int na = A.abase[a + 1] - A.abase[a];
        const bool bad_a = *(volatile int32_t*)&sa->bad_chart != INT32_MAX ||
                           *(volatile int32_t*)&sa->capacity != 0 || na < 1 || na > A.nmax;
        skip_s = bad_a ? 2
                 : (*(volatile int32_t*)&sa->win_j < r || *(volatile int32_t*)&A.res[a].done != 0) ? 1
                                                                                                  : 0;
      }
      }
    }
    __syncthreads();
    const int item = item_s;
    if (item < 0) break;
    const int a = item & 0xfffff, r = item >> 20;
    Status* st = A.sts + a;
    AtlasRes& R = A.res[a];
    const int c0 = A.abase[a], n = A.abase[a + 1] - c0;
    const int m = st->pad[2] - r;
    // an atlas problem (bad chart, capacity) decides the atlas; a rank past the
    // last candidate (m < 1), one above an already successful rank, or of a
    // decided atlas is not evaluated (m is fixed for the atlas)
    const bool bad = skip_s == 2;
    const bool dead = bad || m < 1 || skip_s != 0;
    PackParams pp = pp0;
    pp.n = n;
    Proxies P = A.P;
    P.w += c0; P.h += c0; P.area2 += c0; P.xmin += c0; P.ymin += c0; P.pose += c0;
    P.prerot += c0; P.sl += (int64_t)c0 * 4 * k; P.obb_j += c0; P.obb += 4 * (int64_t)c0;
    const int32_t* perm = A.perm + c0;
    const int32_t* colofs = A.colofs + c0;
    const int32_t* rowofs = A.rowofs + c0;
    long long tc0 = 0, tc1 = 0, tc2 = 0;  // thread 0: phase clocks (raster, pairs, packer)
    if (!dead) {
      // ---- footprints of every chart at m/M (K3, D11 + D13): all up front,
      // or (lazy) inside the packer as its fold reaches them (LazyRaster) ----
      if (tid == 0) { *cbad = 0; *cand = Cand{}; tc0 = clock64(); }
      __syncthreads();
      LazyRaster lzr;
      lzr.P = P;
      lzr.perm = perm;
      lzr.cbad = cbad;
      lzr.area = A.area + gcta * nm;
      lzr.sc = k3::Scale{m, SCm, 0};
      lzr.ahead = A.ahead;
      lzr.early_fail = A.early_fail;
      lzr.atot = (int64_t)st->atot_lo;
      lzr.cycles = A.cycles;
      if (!A.lazy) {
        const int grp = tid / kBGT, gt = tid % kBGT, gw = gt >> 5;
        const BGroupSync gsync{1 + grp};
        unsigned char* p = dsm + bgroup_bytes(k) * grp;
        k3::ChartK3* CH = (k3::ChartK3*)carve(p, sizeof(k3::ChartK3) * kBTC);
        int32_t* cells = (int32_t*)carve(p, 4 * kBTC);
        int32_t* cpre = (int32_t*)carve(p, 4 * (kBTC + 1));
        int32_t* opre = (int32_t*)carve(p, 4 * (kBTC + 1));
        int32_t* big = (int32_t*)carve(p, 4 * kBTC);
        int32_t* misc = (int32_t*)carve(p, 32);
        int32_t* tabs = (int32_t*)carve(p, (size_t)4 * kBTC * 4 * k);
        uint32_t* raw = (uint32_t*)carve(p, 4 * (size_t)kBRaw);
        p = dsm + bgroup_bytes(k) * kBG;
        k3::ChartK3* CW = (k3::ChartK3*)carve(p, sizeof(k3::ChartK3) * kNW);
        int32_t* wtab = (int32_t*)carve(p, (size_t)4 * kNW * 4 * k);
        const k3::Scale sc{m, SCm, 0};
        const int ntile = (n + kBTC - 1) / kBTC;
        unsigned long long pe = 0;  // work accounting: footprint entries (Wd + Hd)
        for (int t = grp; t < ntile; t += kBG) {
          const int s0 = t * kBTC, nt = min(kBTC, n - s0);
          k3::tile_raster<kBTC, kBGT, kBRaw>(P, perm, pp, colofs, rowofs, dcol, drow, wd, hd, cbad,
                                             0, s0, sc, CH, cells, cpre, opre, &misc[1], big, tabs,
                                             raw, nt, gt, gsync);
          for (int ci = gw; ci < nt; ci += kBGW)
            if (big[ci])
              k3::big_chart(P, perm, pp, colofs, rowofs, dcol, drow, 0, s0 + ci, sc, CW[wid],
                            wtab + wid * 4 * k, lane);
          if (gt < nt) pe += (unsigned long long)(CH[gt].ws + CH[gt].hs + 4 * g);
          // the tile's internal adjacent pairs (K3b, D14 + D15) while its rows
          // are hot in L2 -- warp per pair, both charts rasterized above
          for (int s = s0 + gw; s < s0 + nt - 1; s += kBGW)
            if (CH[s - s0].small && CH[s + 1 - s0].small)
              k3::pair_offset(pp, rowofs, drow, wd, hd, off, lock, 0, s, lane);
          gsync();
        }
        for (int o = 16; o > 0; o >>= 1) pe += __shfl_xor_sync(0xffffffffu, pe, o);
        if (lane == 0 && pe) atomicAdd(&st->work_prof, pe);
        __syncthreads();
      }
      // ---- the pairs across tile boundaries, and the last chart's zero entry --
      if (tid == 0) tc1 = clock64();
      if (!A.lazy && !*(volatile int32_t*)cbad) {
        const int ntile = (n + kBTC - 1) / kBTC;
        for (int b = wid; b < ntile; b += kNW)
          k3::pair_offset(pp, rowofs, drow, wd, hd, off, lock, 0, min(n - 1, (b + 1) * kBTC - 1),
                          lane);
      }
      __syncthreads();
      // ---- Alg. 4 for this candidate (K4) -----------------------------------
      if (tid == 0) tc2 = clock64();
      packer(pp, colofs, rowofs, dcol, drow, wd, hd, off, lock, A.hsorted + c0, cbad, scr,
             A.pair_cap, X, Y, mir, cand, st, prof_cap, m, 0, r, Ready{nullptr, 0, nullptr, nullptr},
             dsm, A.lazy != 0, lzr);
      __syncthreads();
    }
    if (tid == 0) {
      // Outcome.  Several ranks of one atlas may be in flight (A.inflight
      // initial items per atlas; a CTA whose rank failed continues with the
      // atlas's next unissued rank): the winner is the lowest successful rank
      // all of whose lower ranks failed -- the top-down search's result.
      const Cand cd = *cand;  // (written by this CTA before the barrier)
      int oc;  // 0 failed, 1 won, 2 atlas decided as bad, 3 not needed
      if (bad) oc = 2;
      else if (m < 1) oc = 0;
      else if (dead || *(volatile int32_t*)&st->win_j < r) oc = 3;  // (beaten)
      else oc = cd.success ? 1 : 0;
      if (!dead) {
        atomicAdd(&R.evaluated, 1);
        const long long t3 = clock64();
        atomicAdd(&A.cycles[0], (unsigned long long)(tc1 - tc0));
        atomicAdd(&A.cycles[1], (unsigned long long)(tc2 - tc1));
        atomicAdd(&A.cycles[2], (unsigned long long)(t3 - tc2));  // (lazy: raster inside, see below)
      }
      if (oc == 1) {
        // announce (higher ranks in flight stop at their next row), then wait
        // until every lower rank has failed -- or a lower rank won
        atomicMin(&st->win_j, r);
        while (true) {
          __threadfence();
          if (*(volatile int32_t*)&st->win_j < r || *(volatile int32_t*)&R.done != 0) { oc = 3; break; }
          bool all = true;
          for (int w = 0; w * 32 < r; w++) {
            const uint32_t mk = r - w * 32 >= 32 ? 0xffffffffu : ((1u << (r - w * 32)) - 1u);
            if ((*(volatile uint32_t*)&R.fail[w] & mk) != mk) all = false;
          }
          if (all) break;
          __nanosleep(256);
        }
        if (oc == 1) {
          R.winner = m;
          R.rows = cd.rows;
          R.knees_found = cd.knees_found;
          R.knee_rows = cd.knee_rows;
        }
      }
      carry = -1;
      if (oc == 0) {
        __threadfence();
        if (r < 256) atomicOr(&R.fail[r >> 5], 1u << (r & 31));
        // no rank has succeeded yet: this CTA continues with the atlas's next
        // rank (issued before this rank's completion is counted, below)
        if (*(volatile int32_t*)&st->win_j == INT32_MAX && *(volatile int32_t*)&R.done == 0) {
          const int nr = atomicAdd(&R.next_r, 1);
          if (st->pad[2] - nr >= 1 && nr < 256) {
            atomicAdd(&R.issued, 1);
            if (A.carry) {
              carry = a | (nr << 20);
            } else {
              // one rank in flight (many atlases per CTA): the next rank goes
              // to the queue's tail, so the atlases' chains interleave
              const int slot = atomicAdd(&A.qctl[1], 1);
              if (slot < A.qcap) st_release_i(A.q + slot, a | (nr << 20));
              else atomicOr(&st->capacity, 8);  // (cannot happen: E * M slots)
            }
          }
        }
      }
      outcome_s = oc;
    }
    __syncthreads();
    const int oc = outcome_s;
    if (oc == 1) {  // K5 for this atlas: placements in input order
      for (int s = tid; s < n; s += kNT) {
        const int c = perm[s];
        const uint8_t ps = P.pose[c];
        tabi_placement pl;
        pl.tx = X[s];
        pl.ty = Y[s];
        pl.scale_num = m;
        pl.scale_den = pp.M;
        pl.box_w = wd[s] - 2 * g;
        pl.box_h = hd[s] - 2 * g;
        pl.rot90 = ps & 1;
        pl.flip_x = (ps >> 1) & 1;
        pl.flip_y = (ps >> 2) & 1;
        pl.mirror_x = mir[s];
        pl.mode = 0;
        pl.prerot = P.prerot[c];
        pl.pad[0] = pl.pad[1] = 0;
        A.out[c0 + c] = pl;
      }
    }
    __syncthreads();  // (placements written before the atlas is announced)
    if (tid == 0) {
      // the atlas is decided once: by its winner, by a bad chart / capacity
      // overflow, or -- no rank succeeded -- by the completion that finds
      // every issued rank done (a rank issues its successor before its own
      // completion is counted, so nothing is issued after that point)
      bool decide = oc == 1 || oc == 2;
      const int done_now = atomicAdd(&R.completed, 1) + 1;
      if (!decide && carry < 0 && done_now == *(volatile int32_t*)&R.issued &&
          *(volatile int32_t*)&st->win_j == INT32_MAX)
        decide = true;
      if (decide && atomicCAS(&R.done, 0, 1) == 0) {
        __threadfence();
        atomicSub(&A.qctl[2], 1);
      }
      A.cycles[3 + 2 * gcta + 1] = gtime();
    }
  }
}

// K5: the largest successful m ("return the largest scale and packing
// that succeed"), then every chart's placement in input order.
__global__ void select_kernel(PackParams pp, const int32_t* __restrict__ perm,
                              const uint8_t* __restrict__ pose, const uint8_t* __restrict__ prerot,
                              const int32_t* __restrict__ wd_all,
                              const int32_t* __restrict__ hd_all, const int32_t* __restrict__ Xo,
                              const int32_t* __restrict__ Yo, const uint8_t* __restrict__ mir,
                              const Cand* __restrict__ cands, tabi_placement* out, Status* st,
                              cudaGraphConditionalHandle h, int use_h) {
  __shared__ int32_t win, wr0, wp;
  // this thread's chart and pose do not depend on the winner: their loads go
  // out first, beside the status and candidate loads (one latency, not three)
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = s < pp.n ? perm[s] : 0;
  const uint8_t ps = s < pp.n ? pose[c] : 0, prr = s < pp.n ? prerot[c] : 0;
  if (st->bad_chart != INT32_MAX || st->capacity) {
    if (use_h && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(h, 0u);
    return;
  }
  // Without a prefix tail anywhere V (below) is increasing in m, so the
  // winner is the largest successful m: one parallel pass (thread m - 1 reads
  // its candidate's two flags) and a shared max -- no serial loop, no int128.
  if (threadIdx.x == 0) win = 0;
  bool tl = false;
  int32_t best = 0;
  for (int i = threadIdx.x; i < pp.M; i += blockDim.x) {
    const Cand& cd = cands[i];
    tl |= cd.switched_at >= 0;
    if (cd.success) best = i + 1;
  }
  const bool any_tail = __syncthreads_or(tl ? 1 : 0) != 0;
  if (!any_tail) {
    if (best) atomicMax(&win, best);
    if (threadIdx.x == 0) { wr0 = pp.n; wp = 0; }
  } else if (threadIdx.x == 0) {
    // D25: the candidate with the largest area-weighted mean final scale,
    // V = A_seq * m * 2^20 + A_pre * p * M (exact, int128), ties -> larger m;
    // without a prefix tail this is the largest successful m.
    const i128 Atot = (i128)(((unsigned __int128)st->atot_hi << 64) | st->atot_lo);
    int32_t w = 0, r0 = pp.n, pw = 0;
    i128 bestV = -1;
    for (int m = 1; m <= pp.M; m++) {
      const Cand& cd = cands[m - 1];
      if (!cd.success) continue;
      const bool tail = cd.switched_at >= 0;
      const i128 Ap = tail ? (i128)(((unsigned __int128)cd.apre_hi << 64) | cd.apre_lo) : 0;
      const i128 V = (Atot - Ap) * m * ((i128)1 << 20) + Ap * cd.p * pp.M;
      if (V >= bestV) {
        bestV = V;
        w = m;
        r0 = tail ? cd.switched_at : pp.n;
        pw = cd.p;
      }
    }
    win = w;
    wr0 = r0;
    wp = pw;
  }
  __syncthreads();
  const int32_t m = win;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->winner = m;
    // Device-side candidate-wave loop (a CUDA-graph WHILE node whose body is
    // the next wave, so a multi-wave scale search has no host round trip):
    // continue while an unevaluated lower candidate could still win.
    // Sequential mode: any success ends the search (the largest successful m
    // wins).  Hybrid mode (D25): a lower m can win only if its V(m) <= A_tot m
    // 2^20 (p <= m 2^20 / M) can exceed the best V found.
    if (use_h) {
      const int next_m = st->pad[2] - (st->b0 + st->wave * pp.B);  // top of the next wave
      bool go = next_m >= 1 && st->wave < pp.M;
      if (go && m > 0) {
        const i128 Atot = (i128)(((unsigned __int128)st->atot_hi << 64) | st->atot_lo);
        const Cand& c = cands[m - 1];
        const bool tail = c.switched_at >= 0;
        const i128 Ap = tail ? (i128)(((unsigned __int128)c.apre_hi << 64) | c.apre_lo) : 0;
        const i128 bestV = (Atot - Ap) * m * ((i128)1 << 20) + Ap * c.p * pp.M;
        if (Atot * next_m * ((i128)1 << 20) <= bestV) go = false;
      }
      cudaGraphSetConditional(h, go ? 1u : 0u);
    }
  }
  if (m == 0) return;
  if (s >= pp.n) return;
  const int64_t b = (int64_t)(m - 1) * pp.n + s;
  const bool tail = s >= wr0;  // tail chart: final scale p / 2^20 (D24) ...
  const bool ptail = tail && !(pp.flags & TABI_F_EXACT_TAIL);  // ... or m/M (R6)
  tabi_placement p;
  p.tx = Xo[b];
  p.ty = Yo[b];
  p.scale_num = ptail ? wp : m;
  p.scale_den = ptail ? (1 << 20) : pp.M;
  p.box_w = wd_all[b] - 2 * pp.g;
  p.box_h = hd_all[b] - 2 * pp.g;
  p.rot90 = ps & 1;
  p.flip_x = (ps >> 1) & 1;
  p.flip_y = (ps >> 2) & 1;
  p.mirror_x = mir[b];
  p.mode = tail ? 1 : 0;
  p.prerot = prr;
  p.pad[0] = p.pad[1] = 0;
  out[c] = p;
}

}  // namespace

void launch_pack(const PackParams& pp, const int32_t* colofs, const int32_t* rowofs,
                 const uint32_t* dcol, const uint32_t* drow, const int32_t* wd, const int32_t* hd,
                 const int32_t* off, const uint8_t* lockbits, const int32_t* hsorted,
                 const int32_t* cand_bad, int32_t* scratch, int64_t pair_cap, int32_t* X,
                 int32_t* Y, uint8_t* mir, Cand* cands, Status* st, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  ensure_dyn_smem((const void*)pack_kernel, kMaxDynSmem, attr);
  const int f_words = (pp.Wp + 3) & ~3;
  const size_t fixed = sizeof(int32_t) * ((size_t)f_words + 10 * (size_t)kRW + 5 * (size_t)kPWN +
                                         2 * (size_t)kPairSm) + kRW + kPWN + kPairSm;
  const int32_t prof_cap = (int32_t)(((size_t)kMaxDynSmem - fixed) / 4) & ~3;
  pack_kernel<<<pp.B, kNT, kMaxDynSmem, s>>>(pp, colofs, rowofs, dcol, drow, wd, hd, off, lockbits,
                                             hsorted, cand_bad, scratch, pair_cap, X, Y, mir,
                                             cands, st, prof_cap);
}

int fused_grid(int device) {
  // per-device cache, filled once; several host threads (tabi_pack_batch)
  // may race here, so the value is an atomic (-1 = not yet known) and the
  // computation is idempotent
  static std::atomic<int> cached[64] = {};
  static std::atomic<bool> have[64] = {};
  if (device < 0 || device >= 64) return 0;
  if (!have[device].load(std::memory_order_acquire)) {
    cudaFuncSetAttribute(fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
    int sms = 0, per = 0, coop = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fused_kernel, kNT, kMaxDynSmem);
    cached[device].store(coop ? sms * per : 0, std::memory_order_relaxed);
    have[device].store(true, std::memory_order_release);
  }
  return cached[device].load(std::memory_order_relaxed);
}


bool fused_fits(int k) {  // the rasterizer role's carve of the dynamic smem
  const size_t need = group_bytes(k) * kRG + r16(sizeof(k3::ChartK3) * kNW) +
                      r16((size_t)4 * kNW * 4 * k);
  return need <= (size_t)kMaxDynSmem;
}

cudaError_t launch_fused(int grid, const Proxies& P, const int32_t* perm, const PackParams& pp,
                         const int32_t* colofs, const int32_t* rowofs, uint32_t* dcol,
                         uint32_t* drow, int32_t* wd, int32_t* hd, int32_t* off, uint8_t* lockbits,
                         const int32_t* hsorted, int32_t* cand_bad, int32_t* rdy,
                         const int32_t* tstart, const int32_t* tix, int32_t* scratch,
                         int64_t pair_cap, int32_t* X, int32_t* Y, uint8_t* mir, Cand* cands,
                         Status* st, cudaStream_t s) {
  const int f_words = (pp.Wp + 3) & ~3;
  const size_t fixed = sizeof(int32_t) * ((size_t)f_words + 10 * (size_t)kRW + 5 * (size_t)kPWN +
                                         2 * (size_t)kPairSm) + kRW + kPWN + kPairSm;
  int32_t prof_cap = (int32_t)(((size_t)kMaxDynSmem - fixed) / 4) & ~3;
  RasterArgs ra{P, perm, wd, hd, off, lockbits, cand_bad, dcol, drow, rdy, tstart, tix};
  PackParams p = pp;
  void* args[] = {&p,       (void*)&colofs, (void*)&rowofs, (void*)&hsorted, &scratch, &pair_cap,
                  &X,       &Y,             &mir,           &cands,          &st,      &prof_cap,
                  &ra};
  return cudaLaunchCooperativeKernel((const void*)fused_kernel, dim3(grid), dim3(kNT), args,
                                     kMaxDynSmem, s);
}

bool many_lazy_ok(int k, int g, int Wp) {
  const int f_words = (Wp + 3) & ~3;
  const size_t fixed = sizeof(int32_t) * ((size_t)f_words + 10 * (size_t)kRW + 5 * (size_t)kPWN +
                                         2 * (size_t)kPairSm) + kRW + kPWN + kPairSm;
  const size_t prof = (((size_t)kMaxDynSmem - fixed) / 4 & ~(size_t)3) * 4;
  const size_t need = r16(sizeof(k3::ChartK3) * kLzTC) + r16(4 * kLzTC) + 2 * r16(4 * (kLzTC + 1)) +
                      r16(4 * kLzTC) + r16(32) + r16((size_t)4 * kLzTC * 4 * k);
  return g <= k3::kDilMax && need <= prof;
}

int many_grid(int device) {
  static std::atomic<int> cached[64] = {};
  static std::atomic<bool> have[64] = {};
  if (device < 0 || device >= 64) return 0;
  if (!have[device].load(std::memory_order_acquire)) {
    cudaFuncSetAttribute(many_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, many_kernel, kNT, kMaxDynSmem);
    cached[device].store(sms * (per > 0 ? per : 1), std::memory_order_relaxed);
    have[device].store(true, std::memory_order_release);
  }
  return cached[device].load(std::memory_order_relaxed);
}

cudaError_t launch_many(int grid, const PackParams& pp, const ManyArgs& a, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  ensure_dyn_smem((const void*)many_kernel, kMaxDynSmem, attr);
  const int f_words = (pp.Wp + 3) & ~3;
  const size_t fixed = sizeof(int32_t) * ((size_t)f_words + 10 * (size_t)kRW + 5 * (size_t)kPWN +
                                         2 * (size_t)kPairSm) + kRW + kPWN + kPairSm;
  const int32_t prof_cap = (int32_t)(((size_t)kMaxDynSmem - fixed) / 4) & ~3;
  many_kernel<<<grid, kNT, kMaxDynSmem, s>>>(pp, a, prof_cap);
  return cudaGetLastError();
}

void launch_select(const PackParams& pp, const Proxies& P, const int32_t* perm, const int32_t* wd,
                   const int32_t* hd, const int32_t* X, const int32_t* Y, const uint8_t* mir,
                   const Cand* cands, tabi_placement* out, Status* st, cudaStream_t s,
                   cudaGraphConditionalHandle h, int use_h) {
  const int blocks = (pp.n + 255) / 256;
  select_kernel<<<blocks, 256, 0, s>>>(pp, perm, P.pose, P.prerot, wd, hd, X, Y, mir, cands, out, st,
                                       h, use_h);
}

}  // namespace tabi
