// k_profile.cu -- K3: per-(chart, candidate) footprints; K3b: compaction
// offsets and lock flags of adjacent pairs.
//
// K3 evaluates TopEdge/BottomEdge for every texel column and the symmetric
// left/right edges for every texel row of every chart at every candidate
// scale m/M ("We evaluate TopEdge and BottomEdge using both
// proxies and use the result per-texel that provides the tightest bound"),
// rounded outward (D11), then applies the gutter as a Chebyshev dilation by g
// (D13).  One warp per (chart, candidate); lanes walk the columns/rows and
// store packed uint16 pairs coalesced; the dilation is an in-place window
// min/max over the warp's slot.
//
// OBB bound per column: the top boundary y_top(x) = max of a decreasing and an
// increasing line, minimised over the column's strip.  Its crossing point and
// crossing value are per-(chart, candidate) constants, so per column exactly
// one line matters (the increasing one right of the crossing, the decreasing
// one left of it): one exact division per bound per column, done by a
// double-precision estimate plus integer correction (fdiv_fast*) instead of an
// emulated int128 divide.
//
// K3b computes, per candidate and adjacent sorted pair, the horizontal
// compaction advance (a max-reduction of profile gaps over shared
// rows, D14) and the CannotMoveAbove flags (D15) with warp scans.
#include "tabi_internal.cuh"

namespace tabi {
namespace {

constexpr int kWarps = 8;

// In-place Chebyshev dilation of a slot holding raw (lo, hi) pairs at
// positions [2g, 2g + n0): out[i] = (min lo, max hi + 2g) over raw [i-2g, i].
__device__ void dilate_slot(uint32_t* slot, int32_t n0, int32_t g, int lane) {
  const int32_t nd = n0 + 2 * g;
  for (int base = 0; base < nd; base += 32) {
    const int i = base + lane;
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    if (i < nd) {
      const int q0 = max(0, i - 2 * g), q1 = min(i, n0 - 1);
      for (int q = q0; q <= q1; q++) {
        const uint32_t v = slot[q + 2 * g];
        lo = min(lo, lo16(v));
        hi = max(hi, hi16(v));
      }
    }
    __syncwarp();
    if (i < nd) slot[i] = (uint32_t)lo | ((uint32_t)(hi + 2 * g) << 16);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kWarps * 32)
profile_kernel(Proxies P, const int32_t* __restrict__ perm, PackParams pp,
               const int32_t* __restrict__ colofs, const int32_t* __restrict__ rowofs,
               uint32_t* dcol, uint32_t* drow, int32_t* wd_all, int32_t* hd_all, int32_t* cand_bad,
               const Status* st) {
  if (st->bad_chart != INT32_MAX || st->capacity) return;
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (item >= (int64_t)pp.n * pp.M) return;
  const int m = (int)(item / pp.n) + 1;
  const int s = (int)(item % pp.n);
  const int c = perm[s];
  const int64_t w = P.w[c], h = P.h[c], k = pp.k;
  const int64_t num = m, SC = (int64_t)pp.M * TABI_UNITS;
  const int64_t nw = num * w, nh = num * h;
  const int64_t ws = cdiv_fast(nw, SC), hs = cdiv_fast(nh, SC);
  const int32_t Wd = (int32_t)(ws + 2 * pp.g), Hd = (int32_t)(hs + 2 * pp.g);
  if (lane == 0) {
    wd_all[(int64_t)(m - 1) * pp.n + s] = Wd;
    hd_all[(int64_t)(m - 1) * pp.n + s] = Hd;
  }
  if (ws + 2 * pp.g > pp.Wp || hs + 2 * pp.g > pp.Hp) {  // cannot fit at this scale
    if (lane == 0) cand_bad[m - 1] = 1;
    return;
  }
  const int32_t* sl = P.sl + (int64_t)c * 4 * k;
  const int j8 = P.obb_j[c];
  uint32_t* col = dcol + (int64_t)(m - 1) * pp.col_cap + colofs[s];
  uint32_t* row = drow + (int64_t)(m - 1) * pp.row_cap + rowofs[s];
  // per-(chart, candidate) OBB constants (D11)
  const i128 C = kQC[j8], S = kQS[j8], N2 = C * C + S * S;
  const i128 umin = P.obb[4 * (int64_t)c], umax = P.obb[4 * (int64_t)c + 1];
  const i128 vmin = P.obb[4 * (int64_t)c + 2], vmax = P.obb[4 * (int64_t)c + 3];
  const i128 N2SC = N2 * SC;
  i128 xsT = 0, xsB = 0, ysL = 0, ysR = 0;
  int64_t starT = 0, starB = 0, starL = 0, starR = 0;
  if (j8 != 0) {
    xsT = num * (C * umin - S * vmin);
    starT = fdiv_fast128(num * (S * umin + C * vmin), N2SC);
    xsB = num * (C * umax - S * vmax);
    starB = cdiv_fast128(num * (S * umax + C * vmax), N2SC);
    ysL = num * (S * umin + C * vmax);
    starL = fdiv_fast128(num * (C * umin - S * vmax), N2SC);
    ysR = num * (S * umax + C * vmin);
    starR = cdiv_fast128(num * (C * umax - S * vmin), N2SC);
  }
  const i128 SSC = S * SC, CSC = C * SC;
  for (int64_t i = lane; i < ws; i += 32) {
    // local-AABB bound: slices whose scaled range openly overlaps [i, i+1]
    int64_t jl = fdiv_fast(i * SC * k, nw), jh = cdiv_fast((i + 1) * SC * k, nw) - 1;
    if (jl < 0) jl = 0;
    if (jh > k - 1) jh = k - 1;
    int64_t mt = INT64_MAX, mb = INT64_MIN;
    for (int64_t j = jl; j <= jh; j++) {
      if (num * j * w < (i + 1) * SC * k && num * (j + 1) * w > i * SC * k) {
        mt = min(mt, (int64_t)sl[j]);
        mb = max(mb, (int64_t)sl[k + j]);
      }
    }
    int64_t t = max((int64_t)0, fdiv_fast(num * mt, SC));
    int64_t b = min(hs, cdiv_fast(num * mb, SC));
    if (j8 != 0) {
      const i128 P0 = (i128)i * SC, P1 = (i128)min((i + 1) * SC, nw);
      const i128 P0N = P0 * N2, P1N = P1 * N2;
      int64_t ot, ob;
      if (P0N <= xsT && xsT <= P1N) ot = starT;
      else if (xsT < P0N) ot = fdiv_fast128(vmin * num + P0 * S, CSC);  // increasing part, at P0
      else ot = fdiv_fast128(umin * num - P1 * C, SSC);                 // decreasing part, at P1
      if (P0N <= xsB && xsB <= P1N) ob = starB;
      else if (xsB < P0N) ob = cdiv_fast128(umax * num - P0 * C, SSC);  // decreasing, at P0
      else ob = cdiv_fast128(vmax * num + P1 * S, CSC);                 // increasing, at P1
      t = max(t, ot);
      b = min(b, ob);
    }
    col[i + 2 * pp.g] = (uint32_t)t | ((uint32_t)b << 16);
  }
  for (int64_t r = lane; r < hs; r += 32) {
    int64_t jl = fdiv_fast(r * SC * k, nh), jh = cdiv_fast((r + 1) * SC * k, nh) - 1;
    if (jl < 0) jl = 0;
    if (jh > k - 1) jh = k - 1;
    int64_t ml = INT64_MAX, mr = INT64_MIN;
    for (int64_t j = jl; j <= jh; j++) {
      if (num * j * h < (r + 1) * SC * k && num * (j + 1) * h > r * SC * k) {
        ml = min(ml, (int64_t)sl[2 * k + j]);
        mr = max(mr, (int64_t)sl[3 * k + j]);
      }
    }
    int64_t l = max((int64_t)0, fdiv_fast(num * ml, SC));
    int64_t rr = min(ws, cdiv_fast(num * mr, SC));
    if (j8 != 0) {
      const i128 Q0 = (i128)r * SC, Q1 = (i128)min((r + 1) * SC, nh);
      const i128 Q0N = Q0 * N2, Q1N = Q1 * N2;
      int64_t ol, orr;
      if (Q0N <= ysL && ysL <= Q1N) ol = starL;
      else if (ysL < Q0N) ol = fdiv_fast128(Q0 * C - vmax * num, SSC);   // increasing, at Q0
      else ol = fdiv_fast128(umin * num - Q1 * S, CSC);                  // decreasing, at Q1
      if (Q0N <= ysR && ysR <= Q1N) orr = starR;
      else if (ysR < Q0N) orr = cdiv_fast128(umax * num - Q0 * S, CSC);  // decreasing, at Q0
      else orr = cdiv_fast128(Q1 * C - vmin * num, SSC);                 // increasing, at Q1
      l = max(l, ol);
      rr = min(rr, orr);
    }
    row[r + 2 * pp.g] = (uint32_t)l | ((uint32_t)rr << 16);
  }
  __syncwarp();
  dilate_slot(col, (int32_t)ws, pp.g, lane);
  dilate_slot(row, (int32_t)hs, pp.g, lane);
}

__global__ void __launch_bounds__(kWarps * 32)
offsets_kernel(PackParams pp, const int32_t* __restrict__ rowofs, const uint32_t* __restrict__ drow,
               const int32_t* __restrict__ wd_all, const int32_t* __restrict__ hd_all,
               int32_t* off_all, uint8_t* lock_all, const int32_t* __restrict__ cand_bad,
               const Status* st) {
  if (st->bad_chart != INT32_MAX || st->capacity) return;
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (item >= (int64_t)pp.n * pp.M) return;
  const int m = (int)(item / pp.n) + 1;
  const int s = (int)(item % pp.n);
  if (cand_bad[m - 1]) return;
  const int64_t base = (int64_t)(m - 1) * pp.n;
  if (s == pp.n - 1) {
    if (lane == 0) { off_all[base + s] = 0; lock_all[base + s] = 0; }
    return;
  }
  const int32_t Hda = hd_all[base + s], Hdb = hd_all[base + s + 1], Wda = wd_all[base + s];
  const uint32_t* ra = drow + (int64_t)(m - 1) * pp.row_cap + rowofs[s];
  const uint32_t* rb = drow + (int64_t)(m - 1) * pp.row_cap + rowofs[s + 1];
  const int rows = min(Hda, Hdb);
  int32_t off = 0;
  for (int j = lane; j < rows; j += 32) off = max(off, hi16(ra[j]) - lo16(rb[j]));
  off = warp_max(off);
  bool la = false, lb = false;
  if (off < Wda) warp_locks(ra, rb, Hda, Hdb, off, lane, la, lb);
  if (lane == 0) {
    off_all[base + s] = off;
    lock_all[base + s] = (uint8_t)((la ? 1 : 0) | (lb ? 2 : 0));
  }
}

}  // namespace

void launch_profiles(const Proxies& P, const int32_t* perm, const PackParams& pp,
                     const int32_t* colofs, const int32_t* rowofs, int16_t* dcol, int16_t* drow,
                     int32_t* wd, int32_t* hd, int32_t* cand_bad, const Status* st,
                     cudaStream_t s) {
  const int64_t items = (int64_t)pp.n * pp.M;
  const int blocks = (int)((items + kWarps - 1) / kWarps);
  profile_kernel<<<blocks, kWarps * 32, 0, s>>>(P, perm, pp, colofs, rowofs, (uint32_t*)dcol,
                                                 (uint32_t*)drow, wd, hd, cand_bad, st);
}

void launch_offsets(const PackParams& pp, const int32_t* colofs, const int32_t* rowofs,
                    const int16_t* drow, const int32_t* wd, const int32_t* hd, int32_t* off,
                    uint8_t* lockbits, const int32_t* cand_bad, const Status* st,
                    cudaStream_t s) {
  (void)colofs;
  const int64_t items = (int64_t)pp.n * pp.M;
  const int blocks = (int)((items + kWarps - 1) / kWarps);
  offsets_kernel<<<blocks, kWarps * 32, 0, s>>>(pp, rowofs, (const uint32_t*)drow, wd, hd, off,
                                                 lockbits, cand_bad, st);
}

}  // namespace tabi
