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
// Cost structure (what makes this kernel fast):
//  * local-AABB bound: each slice's scaled floor/ceil and the column range it
//    openly overlaps are computed once per (chart, candidate) by lanes j < k;
//    a column then takes min/max over its 1-2 slices found by a per-lane
//    pointer (columns of a lane increase monotonically) -- no division;
//  * OBB bound: y_top(x) = max(decreasing, increasing line) is minimised over
//    the column strip; the crossing point and value are per-(chart,
//    candidate) constants, so per column exactly one line is evaluated (left
//    of the crossing the decreasing one at the strip's right end, right of it
//    the increasing one at the left end): one exact division, done as a
//    multiply by a precomputed reciprocal plus an integer correction.
//
// K3b computes, per candidate and adjacent sorted pair, the horizontal
// compaction advance (a max-reduction of profile gaps over shared
// rows, D14) and the CannotMoveAbove flags (D15) with warp scans.
#include "tabi_internal.cuh"

namespace tabi {
namespace {

constexpr int kWarps = 8;

struct SliceTab {  // per-warp tables, one axis
  int32_t lo[TABI_KMAX];    // first texel column/row the slice openly overlaps
  int32_t hi[TABI_KMAX];    // last one
  int32_t flo[TABI_KMAX];   // floor(num * low bound / SC)
  int32_t chi[TABI_KMAX];   // ceil(num * high bound / SC)
};

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

// Slice table of one axis: slice j spans [j*ext/k, (j+1)*ext/k] (units), i.e.
// the scaled range [num*j*ext/(SC*k), num*(j+1)*ext/(SC*k)]; it openly
// overlaps texel t iff num*j*ext < (t+1)*SC*k and num*(j+1)*ext > t*SC*k, i.e.
// t in [floor(num*j*ext/(SC*k)), ceil(num*(j+1)*ext/(SC*k)) - 1].
__device__ void build_tab(SliceTab& T, const int32_t* blo, const int32_t* bhi, int64_t ext,
                          int64_t num, int64_t SC, int k, int lane) {
  const int64_t SCk = SC * k, nx = num * ext;
  for (int j = lane; j < k; j += 32) {
    T.lo[j] = (int32_t)fdiv_fast(nx * j, SCk);
    T.hi[j] = (int32_t)(cdiv_fast(nx * (j + 1), SCk) - 1);
    T.flo[j] = (int32_t)fdiv_fast(num * blo[j], SC);
    T.chi[j] = (int32_t)cdiv_fast(num * bhi[j], SC);
  }
  __syncwarp();
}

struct ObbLine {   // constants of one axis' OBB bounds at one scale
  i128 cross_lo, cross_hi;   // num * crossing numerator (compare with P * N2)
  int64_t star_lo, star_hi;  // bound values at the crossings (floor / ceil, scaled)
};

__global__ void __launch_bounds__(kWarps * 32, 2)
profile_kernel(Proxies P, const int32_t* __restrict__ perm, PackParams pp,
               const int32_t* __restrict__ colofs, const int32_t* __restrict__ rowofs,
               uint32_t* dcol, uint32_t* drow, int32_t* wd_all, int32_t* hd_all, int32_t* cand_bad,
               const Status* st) {
  __shared__ SliceTab tabs[kWarps][2];
  if (st->bad_chart != INT32_MAX || st->capacity) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t item = (int64_t)blockIdx.x * kWarps + wib;
  if (item >= (int64_t)pp.n * pp.M) return;
  const int m = (int)(item / pp.n) + 1;
  const int s = (int)(item % pp.n);
  const int c = perm[s];
  const int64_t w = P.w[c], h = P.h[c];
  const int k = pp.k;
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
  SliceTab& TX = tabs[wib][0];
  SliceTab& TY = tabs[wib][1];
  build_tab(TX, sl, sl + k, w, num, SC, k, lane);
  build_tab(TY, sl + 2 * k, sl + 3 * k, h, num, SC, k, lane);
  const int j8 = P.obb_j[c];
  uint32_t* col = dcol + (int64_t)(m - 1) * pp.col_cap + colofs[s];
  uint32_t* row = drow + (int64_t)(m - 1) * pp.row_cap + rowofs[s];
  // ---- OBB constants (D11): lines of the box in the (x, y) chart frame ----
  const int64_t C = kQC[j8], S = kQS[j8], N2 = C * C + S * S;
  const int64_t umin = P.obb[4 * (int64_t)c], umax = P.obb[4 * (int64_t)c + 1];
  const int64_t vmin = P.obb[4 * (int64_t)c + 2], vmax = P.obb[4 * (int64_t)c + 3];
  const i128 UMN = mul_wide(umin, num), UXN = mul_wide(umax, num);
  const i128 VMN = mul_wide(vmin, num), VXN = mul_wide(vmax, num);
  const int64_t DS = S * SC, DC = C * SC;          // divisors of the two lines
  const double rDS = 1.0 / (double)DS, rDC = 1.0 / (double)DC;
  ObbLine OX{}, OY{};
  if (j8 != 0) {
    const i128 N2SC = (i128)N2 * SC;
    OX.cross_lo = (i128)C * UMN - (i128)S * VMN;     // x* of the top boundary  (x num N2)
    OX.star_lo = fdiv_fast128((i128)S * UMN + (i128)C * VMN, N2SC);
    OX.cross_hi = (i128)C * UXN - (i128)S * VXN;     // x** of the bottom boundary
    OX.star_hi = cdiv_fast128((i128)S * UXN + (i128)C * VXN, N2SC);
    OY.cross_lo = (i128)S * UMN + (i128)C * VXN;     // y* of the left boundary
    OY.star_lo = fdiv_fast128((i128)C * UMN - (i128)S * VXN, N2SC);
    OY.cross_hi = (i128)S * UXN + (i128)C * VMN;     // y** of the right boundary
    OY.star_hi = cdiv_fast128((i128)C * UXN - (i128)S * VMN, N2SC);
  }
  // ---- columns: Top / Bottom -------------------------------------------------
  {
    int jp = 0;
    for (int64_t i = lane; i < ws; i += 32) {
      while (TX.hi[jp] < i) jp++;
      int32_t t = INT32_MAX, b = INT32_MIN;
      for (int j = jp; j < k && TX.lo[j] <= i; j++) {
        t = min(t, TX.flo[j]);
        b = max(b, TX.chi[j]);
      }
      int64_t T = max(0, t), B = min((int64_t)b, hs);
      if (j8 != 0) {
        const int64_t P0 = i * SC, P1 = min((i + 1) * SC, nw);
        const i128 P0N = mul_wide(P0, N2), P1N = mul_wide(P1, N2);
        int64_t ot, ob;
        if (P0N <= OX.cross_lo && OX.cross_lo <= P1N) ot = OX.star_lo;
        else if (OX.cross_lo < P0N) ot = fdiv_rcp(VMN + mul_wide(P0, S), DC, rDC);  // increasing line at P0
        else ot = fdiv_rcp(UMN - mul_wide(P1, C), DS, rDS);                         // decreasing line at P1
        if (P0N <= OX.cross_hi && OX.cross_hi <= P1N) ob = OX.star_hi;
        else if (OX.cross_hi < P0N) ob = cdiv_rcp(UXN - mul_wide(P0, C), DS, rDS);  // decreasing line at P0
        else ob = cdiv_rcp(VXN + mul_wide(P1, S), DC, rDC);                         // increasing line at P1
        T = max(T, ot);
        B = min(B, ob);
      }
      col[i + 2 * pp.g] = (uint32_t)T | ((uint32_t)B << 16);
    }
  }
  // ---- rows: Left / Right -----------------------------------------------------
  {
    int jp = 0;
    for (int64_t r = lane; r < hs; r += 32) {
      while (TY.hi[jp] < r) jp++;
      int32_t l = INT32_MAX, rr = INT32_MIN;
      for (int j = jp; j < k && TY.lo[j] <= r; j++) {
        l = min(l, TY.flo[j]);
        rr = max(rr, TY.chi[j]);
      }
      int64_t L = max(0, l), R = min((int64_t)rr, ws);
      if (j8 != 0) {
        const int64_t Q0 = r * SC, Q1 = min((r + 1) * SC, nh);
        const i128 Q0N = mul_wide(Q0, N2), Q1N = mul_wide(Q1, N2);
        int64_t ol, orr;
        if (Q0N <= OY.cross_lo && OY.cross_lo <= Q1N) ol = OY.star_lo;
        else if (OY.cross_lo < Q0N) ol = fdiv_rcp(mul_wide(Q0, C) - VXN, DS, rDS);  // increasing at Q0
        else ol = fdiv_rcp(UMN - mul_wide(Q1, S), DC, rDC);                         // decreasing at Q1
        if (Q0N <= OY.cross_hi && OY.cross_hi <= Q1N) orr = OY.star_hi;
        else if (OY.cross_hi < Q0N) orr = cdiv_rcp(UXN - mul_wide(Q0, S), DC, rDC);  // decreasing at Q0
        else orr = cdiv_rcp(mul_wide(Q1, C) - VMN, DS, rDS);                         // increasing at Q1
        L = max(L, ol);
        R = min(R, orr);
      }
      row[r + 2 * pp.g] = (uint32_t)L | ((uint32_t)R << 16);
    }
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
