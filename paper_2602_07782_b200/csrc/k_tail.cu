// k_tail.cu -- hybrid prefix-sum tail ("Performance Optimization",
// SURVEY D23-D25, reading R3).
//
// After K4 switched a candidate to prefix folding at sorted position r0 (its
// frontline saved), per candidate (one CTA each):
//   tail_prepare_kernel: exclusive prefix sum of the compaction offsets at the
//     candidate scale m/M over [r0, n) ("the prefix sum of the horizontal
//     offsets"), FastAtlas rows = floor(start / W'), widest row extent E,
//     the global intermediate scale p / 2^20 = (m/M) * min(1, W'/E),
//     and the tail's area for the area-weighted choice (D25);
//   [K3 / K3b in tail mode re-rasterize the tail at p / 2^20]
//   tail_layout_kernel: re-lay each row with an in-row (segmented) exclusive
//     scan of the new offsets; if the widest row still exceeds W', shrink p by
//     W'/E' and repeat (at most 8 times), else mark the candidate ready for
//     K4 in prefix-row mode.
// All scans are block-wide (warp shuffles + one shared pass per window).
#include "tabi_internal.cuh"

namespace tabi {
namespace {

constexpr int kT = 512;
constexpr int kW = kT / 32;

struct ScanSmem {
  int32_t s[3][kW + 1];
  int32_t mx[kW];
  unsigned long long a[2][kW];
  int32_t carry[3];
};

// Block-wide exclusive sums of a, b and inclusive max of c (one value each per
// thread), with window totals / max returned.
__device__ __forceinline__ void block_scan3(int32_t a, int32_t b, int32_t c, int32_t& ea,
                                            int32_t& eb, int32_t& ic, int32_t& ta, int32_t& tb,
                                            int32_t& mc, ScanSmem& S) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int32_t ia = warp_incl_sum(a, lane), ib = warp_incl_sum(b, lane);
  const int32_t xc = warp_incl_max(c, lane);
  if (lane == 31) { S.s[0][wid] = ia; S.s[1][wid] = ib; S.s[2][wid] = xc; }
  __syncthreads();
  if (wid == 0) {
    const int32_t va = lane < kW ? S.s[0][lane] : 0, vb = lane < kW ? S.s[1][lane] : 0;
    const int32_t vc = lane < kW ? S.s[2][lane] : INT32_MIN;
    const int32_t xa = warp_incl_sum(va, lane), xb = warp_incl_sum(vb, lane);
    const int32_t yc = warp_incl_max(vc, lane);
    int32_t pc = __shfl_up_sync(0xffffffffu, yc, 1);
    if (lane == 0) pc = INT32_MIN;
    if (lane < kW) { S.s[0][lane] = xa - va; S.s[1][lane] = xb - vb; S.s[2][lane] = pc; }
    if (lane == 31) { S.s[0][kW] = xa; S.s[1][kW] = xb; S.s[2][kW] = yc; }
  }
  __syncthreads();
  ea = S.s[0][wid] + ia - a;
  eb = S.s[1][wid] + ib - b;
  ic = max(S.s[2][wid], xc);
  ta = S.s[0][kW];
  tb = S.s[1][kW];
  mc = S.s[2][kW];
  __syncthreads();
}

// Like block_scan3 but c's result is the EXCLUSIVE max over the threads
// before this one (INT32_MIN for thread 0 of the block).
__device__ __forceinline__ void block_scan3x(int32_t a, int32_t b, int32_t c, int32_t& ea,
                                             int32_t& eb, int32_t& xc_ex, int32_t& ta, int32_t& tb,
                                             int32_t& mc, ScanSmem& S) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int32_t ia = warp_incl_sum(a, lane), ib = warp_incl_sum(b, lane);
  const int32_t xc = warp_incl_max(c, lane);
  int32_t xprev = __shfl_up_sync(0xffffffffu, xc, 1);
  if (lane == 0) xprev = INT32_MIN;
  if (lane == 31) { S.s[0][wid] = ia; S.s[1][wid] = ib; S.s[2][wid] = xc; }
  __syncthreads();
  if (wid == 0) {
    const int32_t va = lane < kW ? S.s[0][lane] : 0, vb = lane < kW ? S.s[1][lane] : 0;
    const int32_t vc = lane < kW ? S.s[2][lane] : INT32_MIN;
    const int32_t xa = warp_incl_sum(va, lane), xb = warp_incl_sum(vb, lane);
    const int32_t yc = warp_incl_max(vc, lane);
    int32_t pc = __shfl_up_sync(0xffffffffu, yc, 1);
    if (lane == 0) pc = INT32_MIN;
    if (lane < kW) { S.s[0][lane] = xa - va; S.s[1][lane] = xb - vb; S.s[2][lane] = pc; }
    if (lane == 31) { S.s[0][kW] = xa; S.s[1][kW] = xb; S.s[2][kW] = yc; }
  }
  __syncthreads();
  ea = S.s[0][wid] + ia - a;
  eb = S.s[1][wid] + ib - b;
  xc_ex = max(S.s[2][wid], xprev);
  ta = S.s[0][kW];
  tb = S.s[1][kW];
  mc = S.s[2][kW];
  __syncthreads();
}

// Scans over the tail [r0, n) take kIT consecutive positions per thread (a
// sequential scan in registers, then one block scan of the thread totals):
// kIT x fewer barrier-separated block scans than one position per thread.
constexpr int kIT = 8;

__device__ __forceinline__ int32_t block_max(int32_t v, ScanSmem& S) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) S.mx[wid] = v;
  __syncthreads();
  int32_t r = INT32_MIN;
  for (int w = 0; w < kW; w++) r = max(r, S.mx[w]);
  __syncthreads();
  return r;
}

// Device-side stop of the re-layout rounds (a CUDA-graph WHILE node around
// K3 + K3b + tail_layout): the last CTA of the grid to finish (fence +
// counter, the threadFenceReduction pattern) sets the node's condition to
// "some candidate of the wave still needs a round" -- TAIL_LAYOUT, whose
// iteration count tail_layout bounds by 8.
__device__ __forceinline__ void rounds_decide(const PackParams& pp, Status* st,
                                              cudaGraphConditionalHandle h, bool round) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  __threadfence();
  if (atomicAdd(&st->tail_cnt, 1) != (int)gridDim.x - 1) return;
  st->tail_cnt = 0;
  if (round) st->rounds_run++;
  __threadfence();
  bool go = false;
  if (st->bad_chart == INT32_MAX && !st->capacity) {
    for (int j = 0; j < (int)gridDim.x; j++) {
      const int m = wave_m(pp, st->wave, st->pad[2], st->b0, j);
      if (m != 0 && *(volatile int32_t*)&pp.T.state[m - 1] == TAIL_LAYOUT) go = true;
    }
  }
  cudaGraphSetConditional(h, go ? 1u : 0u);
}

__device__ __noinline__ void tail_prepare(const PackParams& pp, const int32_t* __restrict__ perm,
                                          const int64_t* __restrict__ area2,
                                          const int32_t* __restrict__ wd_all,
                                          const int32_t* __restrict__ off_all, int32_t* scratch,
                                          int64_t pair_cap, Cand* cands, int m) {
  __shared__ ScanSmem S;
  const int n = pp.n, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t Wp = pp.Wp;
  const int32_t r0 = pp.T.r0[m - 1];
  const int64_t cb = (int64_t)(m - 1) * n;
  const int32_t* wd = wd_all + cb;
  const int32_t* off = off_all + cb;
  int32_t* sc = scratch + (int64_t)(m - 1) * (6 * (int64_t)n + 3 * pair_cap);
  int32_t* qrow = sc + 5 * (int64_t)n;
  int32_t* start = sc + 4 * (int64_t)n;  // temporary: prefix sum at scale m
  if (pp.flags & TABI_F_EXACT_TAIL) {
    // R6: Alg. 3 with compaction at m/M, row by row.  Exclusive
    // prefix sums of the offsets (positions) and of the widths (the packer's
    // flattened column index) over [r0, n); then each row ends before the first
    // chart c with start(c) - start(a) + Wd(c) > W' -- one block-wide
    // first-violation search per row.  Every chart keeps scale m/M.
    __shared__ int32_t row_end[2], row_a;  // row_end alternates by pass (no reset race)
    int32_t* pwd = sc + 3 * (int64_t)n;
    int32_t* xs0 = sc;
    int32_t* xs1 = sc + n;
    int32_t c0 = 0, c1 = 0;
    for (int base = r0; base < n; base += kT) {
      const int s = base + tid;
      const int32_t a = (s < n && s + 1 < n) ? off[s] : 0;
      const int32_t b = s < n ? wd[s] : 0;
      int32_t ea, eb, ic, ta, tb, mc;
      block_scan3(a, b, 0, ea, eb, ic, ta, tb, mc, S);
      if (s < n) { start[s] = c0 + ea; pwd[s] = c1 + eb; }
      c0 += ta;
      c1 += tb;
    }
    if (tid == 0) row_a = r0;
    __syncthreads();
    int32_t row = 0;
    bool ok = true;
    while (true) {
      const int32_t a = row_a;
      if (a >= n) break;
      const int32_t sa = start[a], wa = pwd[a];
      int32_t end = n - 1;
      for (int base = a, pass = 0;; base += kT, pass ^= 1) {
        if (tid == 0) row_end[pass] = INT32_MAX;
        __syncthreads();
        const int s = base + tid;
        if (s < n && start[s] - sa + wd[s] > Wp) atomicMin(&row_end[pass], s);
        __syncthreads();
        const int32_t e = row_end[pass];
        if (e != INT32_MAX) { end = e - 1; break; }
        if (base + kT >= n) break;
      }
      if (end < a) { ok = false; break; }  // D22: the first chart does not fit
      for (int s = a + tid; s <= end; s += kT) {
        qrow[s] = row;
        xs1[s] = start[s] - sa;
        xs0[s] = pwd[s] - wa;
      }
      if (tid == 0) start[a] = end;  // (rend, read by the packer's prefix rows; start[a] is dead)
      row++;
      __syncthreads();
      if (tid == 0) row_a = end + 1;
      __syncthreads();
    }
    if (tid == 0) {
      pp.T.p[m - 1] = (int32_t)(((int64_t)m << 20) / pp.M);  // informational
      pp.T.state[m - 1] = ok ? TAIL_READY : TAIL_FAIL;
      cands[m - 1].apre_lo = 0ull;  // every chart keeps m/M: no area at another scale
      cands[m - 1].apre_hi = 0ull;
    }
    return;
  }
  // pass 1: start = exclusive scan of off over [r0, n); q = floor(start / W')
  int32_t carry = 0;
  for (int base = r0; base < n; base += kT * kIT) {
    const int s0 = base + tid * kIT;
    int32_t lx[kIT], tot = 0;
#pragma unroll
    for (int u = 0; u < kIT; u++) {
      const int s = s0 + u;
      lx[u] = tot;
      tot += (s < n && s + 1 < n) ? off[s] : 0;
    }
    int32_t ea, eb, ic, ta, tb, mc;
    block_scan3(tot, 0, 0, ea, eb, ic, ta, tb, mc, S);
#pragma unroll
    for (int u = 0; u < kIT; u++) {
      const int s = s0 + u;
      if (s < n) {
        start[s] = carry + ea + lx[u];
        qrow[s] = (int32_t)((int64_t)(carry + ea + lx[u]) / Wp);
      }
    }
    carry += ta;
  }
  __syncthreads();
  // pass 2: E = max over charts of (start - start of the row's first chart + Wd)
  int32_t fcarry = INT32_MIN, emax = INT32_MIN;
  i128 apre = 0;
  for (int base = r0; base < n; base += kT * kIT) {
    const int s0 = base + tid * kIT;
    int32_t lf = INT32_MIN;  // the thread's last row start among its positions
#pragma unroll
    for (int u = 0; u < kIT; u++) {
      const int s = s0 + u;
      if (s < n && (s == r0 || qrow[s] != qrow[s - 1])) lf = s;
    }
    int32_t ea, eb, fx, ta, tb, mc;
    block_scan3x(0, 0, lf, ea, eb, fx, ta, tb, mc, S);
    int32_t f = max(fcarry, fx);
#pragma unroll
    for (int u = 0; u < kIT; u++) {
      const int s = s0 + u;
      if (s < n) {
        if (s == r0 || qrow[s] != qrow[s - 1]) f = s;
        emax = max(emax, start[s] - start[f] + wd[s]);
        apre += area2[perm[s]];
      }
    }
    fcarry = max(fcarry, mc);
  }
  emax = block_max(emax, S);
  apre = warp_sum128(apre);
  if (lane == 0) {
    S.a[0][wid] = (unsigned long long)(uint64_t)apre;
    S.a[1][wid] = (unsigned long long)(uint64_t)(apre >> 64);
  }
  __syncthreads();
  if (tid == 0) {
    i128 A = 0;
    for (int w = 0; w < kW; w++) A += (i128)(((unsigned __int128)S.a[1][w] << 64) | S.a[0][w]);
    const i128 P20 = (i128)1 << 20;
    i128 p = ((i128)m * P20 * Wp) / ((i128)pp.M * emax);
    const i128 pm = ((i128)m * P20) / pp.M;  // sigma <= 1: intermediate DOWNscaling
    if (p > pm) p = pm;
    pp.T.p[m - 1] = (int32_t)p;
    if (p < 1) pp.T.state[m - 1] = TAIL_FAIL;
    cands[m - 1].apre_lo = (unsigned long long)(uint64_t)A;
    cands[m - 1].apre_hi = (unsigned long long)(uint64_t)(A >> 64);
  }
}

__global__ void __launch_bounds__(kT, 1)
tail_prepare_kernel(PackParams pp, const int32_t* __restrict__ perm, const int64_t* __restrict__ area2,
                    const int32_t* __restrict__ wd_all, const int32_t* __restrict__ off_all,
                    int32_t* scratch, int64_t pair_cap, Cand* cands, Status* st,
                    cudaGraphConditionalHandle h, int use_h) {
  if (st->bad_chart == INT32_MAX && !st->capacity) {
    const int m = wave_m(pp, st->wave, st->pad[2], st->b0, blockIdx.x);
    if (m != 0 && pp.T.state[m - 1] == TAIL_LAYOUT) tail_prepare(pp, perm, area2, wd_all, off_all, scratch, pair_cap, cands, m);
  }
  if (use_h) rounds_decide(pp, st, h, false);
}

__device__ __noinline__ void tail_layout(const PackParams& pp, const int32_t* __restrict__ wd_all,
                                         const int32_t* __restrict__ off_all, int32_t* scratch,
                                         int64_t pair_cap, int m) {
  __shared__ ScanSmem S;
  const int n = pp.n, tid = threadIdx.x;
  const int64_t Wp = pp.Wp;
  const int32_t r0 = pp.T.r0[m - 1];
  const int64_t cb = (int64_t)(m - 1) * n;
  const int32_t* wd = wd_all + cb;
  const int32_t* off = off_all + cb;
  int32_t* sc = scratch + (int64_t)(m - 1) * (6 * (int64_t)n + 3 * pair_cap);
  int32_t* xs0 = sc;
  int32_t* xs1 = sc + n;
  int32_t* poff = sc + 2 * (int64_t)n;  // temporary global prefix sums
  int32_t* pwd = sc + 3 * (int64_t)n;
  const int32_t* qrow = sc + 5 * (int64_t)n;
  int32_t* rend = sc + 4 * (int64_t)n;  // row's last position by its first (the packer's prefix rows)
  // global exclusive prefix sums of the new offsets and widths over [r0, n)
  int32_t c0 = 0, c1 = 0;
  for (int base = r0; base < n; base += kT * kIT) {
    const int s0 = base + tid * kIT;
    int32_t la[kIT], lb[kIT], sa = 0, sb = 0;
#pragma unroll
    for (int u = 0; u < kIT; u++) {
      const int s = s0 + u;
      la[u] = sa;
      lb[u] = sb;
      sa += (s < n && s + 1 < n) ? off[s] : 0;
      sb += s < n ? wd[s] : 0;
    }
    int32_t ea, eb, ic, ta, tb, mc;
    block_scan3(sa, sb, 0, ea, eb, ic, ta, tb, mc, S);
#pragma unroll
    for (int u = 0; u < kIT; u++) {
      const int s = s0 + u;
      if (s < n) { poff[s] = c0 + ea + la[u]; pwd[s] = c1 + eb + lb[u]; }
    }
    c0 += ta;
    c1 += tb;
  }
  __syncthreads();
  // row-relative positions: subtract the value at the row's first chart
  int32_t fcarry = INT32_MIN, emax = INT32_MIN;
  for (int base = r0; base < n; base += kT * kIT) {
    const int s0 = base + tid * kIT;
    int32_t lf = INT32_MIN;
#pragma unroll
    for (int u = 0; u < kIT; u++) {
      const int s = s0 + u;
      if (s < n && (s == r0 || qrow[s] != qrow[s - 1])) lf = s;
    }
    int32_t ea, eb, fx, ta, tb, mc;
    block_scan3x(0, 0, lf, ea, eb, fx, ta, tb, mc, S);
    int32_t f = max(fcarry, fx);
#pragma unroll
    for (int u = 0; u < kIT; u++) {
      const int s = s0 + u;
      if (s < n) {
        if (s == r0 || qrow[s] != qrow[s - 1]) f = s;
        const int32_t x = poff[s] - poff[f];
        xs1[s] = x;                // position with compaction (D24 step 2 re-lay)
        xs0[s] = pwd[s] - pwd[f];  // prefix of widths in the row (flattened index)
        emax = max(emax, x + wd[s]);
        if (s == n - 1 || qrow[s + 1] != qrow[s]) rend[f] = s;  // the row's last position
      }
    }
    fcarry = max(fcarry, mc);
  }
  emax = block_max(emax, S);
  if (tid == 0) {
    const int it = pp.T.iter[m - 1];
    if (emax <= Wp) {
      pp.T.state[m - 1] = TAIL_READY;
    } else if (it >= 8) {
      pp.T.state[m - 1] = TAIL_FAIL;
    } else {
      const int64_t p = ((int64_t)pp.T.p[m - 1] * Wp) / emax;
      pp.T.p[m - 1] = (int32_t)p;
      pp.T.iter[m - 1] = it + 1;
      if (p < 1) pp.T.state[m - 1] = TAIL_FAIL;
    }
  }
}

__global__ void __launch_bounds__(kT, 1)
tail_layout_kernel(PackParams pp, const int32_t* __restrict__ wd_all,
                   const int32_t* __restrict__ off_all, int32_t* scratch, int64_t pair_cap,
                   Status* st, cudaGraphConditionalHandle h, int use_h) {
  if (st->bad_chart == INT32_MAX && !st->capacity) {
    const int m = wave_m(pp, st->wave, st->pad[2], st->b0, blockIdx.x);
    if (m != 0 && pp.T.state[m - 1] == TAIL_LAYOUT) tail_layout(pp, wd_all, off_all, scratch, pair_cap, m);
  }
  if (use_h) rounds_decide(pp, st, h, true);
}

}  // namespace

void launch_tail_prepare(const PackParams& pp, const int32_t* perm, const int64_t* area2,
                         const int32_t* wd, const int32_t* off, int32_t* scratch, int64_t pair_cap,
                         Cand* cands, Status* st, cudaStream_t s, cudaGraphConditionalHandle h,
                         int use_h) {
  tail_prepare_kernel<<<pp.B, kT, 0, s>>>(pp, perm, area2, wd, off, scratch, pair_cap, cands, st, h,
                                          use_h);
}

void launch_tail_layout(const PackParams& pp, const int32_t* wd, const int32_t* off,
                        int32_t* scratch, int64_t pair_cap, Status* st, cudaStream_t s,
                        cudaGraphConditionalHandle h, int use_h) {
  tail_layout_kernel<<<pp.B, kT, 0, s>>>(pp, wd, off, scratch, pair_cap, st, h, use_h);
}

}  // namespace tabi
