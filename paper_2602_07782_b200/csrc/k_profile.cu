// k_profile.cu -- K3: per-(chart, candidate) footprints; K3b: compaction
// offsets and lock flags of adjacent pairs.
//
// K3 evaluates TopEdge/BottomEdge for every texel column and the symmetric
// left/right edges for every texel row of every chart at every candidate
// scale m/M ("We evaluate TopEdge and BottomEdge using both
// proxies and use the result per-texel that provides the tightest bound"),
// rounded outward (D11), then applies the gutter as a Chebyshev dilation by g
// (D13).  One warp per (chart, candidate); lanes walk the columns and rows
// (one merged index space, so narrow charts still fill the warp) and store
// packed uint16 pairs coalesced; the dilation is an in-place window min/max.
//
// Cost structure:
//  * local-AABB bound: each slice's scaled floor/ceil and the cell range it
//    openly overlaps are computed once per (chart, candidate) by lanes j < k;
//    a cell takes min/max over its 1-2 slices, found by a per-lane pointer
//    (a lane's cells increase monotonically) -- no division per cell;
//  * OBB bound: y_top(x) = max(decreasing, increasing line) minimised over the
//    cell's strip.  Which case applies (crossing inside / left / right) is an
//    integer compare of the cell index with per-(chart, candidate) crossing
//    indices; each line evaluated at a cell edge is floor((A + i*B)/D), an
//    int64 progression (LinDiv) whose 128-bit parts are split off once per
//    warp, lane-parallel.  So a cell costs two int64 multiply-corrects.
//
// K3b computes, per candidate and adjacent sorted pair, the horizontal
// compaction advance (a max-reduction of profile gaps over shared
// rows, D14) and the CannotMoveAbove flags (D15) with warp scans.
#include "tabi_internal.cuh"

namespace tabi {
namespace {

constexpr int kWarps = 8;

struct SliceTab {  // per-warp tables, one axis
  int32_t lo[TABI_KMAX];    // first texel cell the slice openly overlaps
  int32_t hi[TABI_KMAX];    // last one
  int32_t flo[TABI_KMAX];   // floor(num * low bound / SC)
  int32_t chi[TABI_KMAX];   // ceil(num * high bound / SC)
};

// Per-warp OBB constants.  Index q = axis * 2 + (0: low bound, 1: high bound);
// lines lin[axis * 4 + kind]: kind 0 low-bound line right of the crossing
// (evaluated at the cell's left edge), 1 low-bound line left of it (right
// edge, non-last cells), 2 / 3 the same for the high bound (negated floors).
struct ObbW {
  LinDiv lin[8];
  int64_t last[4];   // value at the clipped right edge of the last cell
  int64_t star[4];   // value at the crossing
  int64_t iA[4];     // crossing at or right of cell i's left edge  <=>  i <= iA
  int64_t iB[4];     // crossing at or left of cell i's right edge  <=>  i >= iB (non-last)
  int32_t lastB[4];  // same test for the last cell (edge = chart extent)
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
}

// Lane-parallel setup of the OBB constants (D11).  The box is
// {Umin <= xC + yS <= Umax, Vmin <= -xS + yC <= Vmax}; with num/SC scaling:
//  top    y_top(x)   = max((Umin - xC)/S, (Vmin + xS)/C)
//  bottom y_bot(x)   = min((Umax - xC)/S, (Vmax + xS)/C)
//  left   x_left(y)  = max((Umin - yS)/C, (yC - Vmax)/S)
//  right  x_right(y) = min((Umax - yS)/C, (yC - Vmin)/S)
__device__ void build_obb(ObbW& O, int64_t C, int64_t S, i128 UMN, i128 UXN, i128 VMN, i128 VXN,
                          int64_t SC, int64_t nw, int64_t nh, int lane) {
  const int64_t N2 = C * C + S * S, DS = S * SC, DC = C * SC;
  const i128 N2SC = (i128)N2 * SC;
  const int64_t SCS = SC * S, SCC = SC * C;
  if (lane < 8) {
    i128 A;
    int64_t B, D;
    switch (lane) {
      case 0: A = VMN; B = SCS; D = DC; break;               // top, increasing line at P0
      case 1: A = UMN - SCC; B = -SCC; D = DS; break;        // top, decreasing line at P1
      case 2: A = -UXN; B = SCC; D = DS; break;              // bottom, decreasing at P0 (neg)
      case 3: A = -VXN - SCS; B = -SCS; D = DC; break;       // bottom, increasing at P1 (neg)
      case 4: A = -VXN; B = SCC; D = DS; break;              // left, increasing at Q0
      case 5: A = UMN - SCS; B = -SCS; D = DC; break;        // left, decreasing at Q1
      case 6: A = -UXN; B = SCS; D = DC; break;              // right, decreasing at Q0 (neg)
      default: A = VMN - SCC; B = -SCC; D = DS; break;       // right, increasing at Q1 (neg)
    }
    O.lin[lane] = make_lindiv(A, B, D);
  } else if (lane < 12) {
    const int q = lane - 8;
    int64_t v;
    switch (q) {
      case 0: v = fdiv_fast128(UMN - mul_wide(nw, C), (i128)DS); break;
      case 1: v = cdiv_fast128(VXN + mul_wide(nw, S), (i128)DC); break;
      case 2: v = fdiv_fast128(UMN - mul_wide(nh, S), (i128)DC); break;
      default: v = cdiv_fast128(mul_wide(nh, C) - VMN, (i128)DS); break;
    }
    O.last[q] = v;
  } else if (lane < 16) {
    const int q = lane - 12;
    int64_t v;
    switch (q) {
      case 0: v = fdiv_fast128((i128)S * UMN + (i128)C * VMN, N2SC); break;
      case 1: v = cdiv_fast128((i128)S * UXN + (i128)C * VXN, N2SC); break;
      case 2: v = fdiv_fast128((i128)C * UMN - (i128)S * VXN, N2SC); break;
      default: v = cdiv_fast128((i128)C * UXN - (i128)S * VMN, N2SC); break;
    }
    O.star[q] = v;
  } else if (lane < 20) {
    const int q = lane - 16;
    i128 cross;
    switch (q) {
      case 0: cross = (i128)C * UMN - (i128)S * VMN; break;   // x* of the top boundary
      case 1: cross = (i128)C * UXN - (i128)S * VXN; break;   // x** of the bottom
      case 2: cross = (i128)S * UMN + (i128)C * VXN; break;   // y* of the left
      default: cross = (i128)S * UXN + (i128)C * VMN; break;  // y** of the right
    }
    O.iA[q] = fdiv_clamp128(cross, N2SC);
    O.iB[q] = -fdiv_clamp128(-cross, N2SC) - 1;
    O.lastB[q] = cross <= mul_wide(q < 2 ? nw : nh, N2);
  }
}

__global__ void __launch_bounds__(kWarps * 32, 2)
profile_kernel(Proxies P, const int32_t* __restrict__ perm, PackParams pp,
               const int32_t* __restrict__ colofs, const int32_t* __restrict__ rowofs,
               uint32_t* dcol, uint32_t* drow, int32_t* wd_all, int32_t* hd_all, int32_t* cand_bad,
               const Status* st) {
  __shared__ SliceTab tabs[kWarps][2];
  __shared__ ObbW obbs[kWarps];
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
  const SliceTab* TT = tabs[wib];
  build_tab(tabs[wib][0], sl, sl + k, w, num, SC, k, lane);
  build_tab(tabs[wib][1], sl + 2 * k, sl + 3 * k, h, num, SC, k, lane);
  const int j8 = P.obb_j[c];
  ObbW& O = obbs[wib];
  if (j8 != 0) {
    const int64_t C = kQC[j8], S = kQS[j8];
    const int64_t* ob = P.obb + 4 * (int64_t)c;
    build_obb(O, C, S, mul_wide(ob[0], num), mul_wide(ob[1], num), mul_wide(ob[2], num),
              mul_wide(ob[3], num), SC, nw, nh, lane);
  }
  __syncwarp();
  uint32_t* col = dcol + (int64_t)(m - 1) * pp.col_cap + colofs[s];
  uint32_t* row = drow + (int64_t)(m - 1) * pp.row_cap + rowofs[s];
  int jp = 0, ax_prev = 0;
  for (int64_t e = lane; e < ws + hs; e += 32) {
    const int ax = e >= ws ? 1 : 0;      // 0: column i (top/bottom), 1: row i (left/right)
    const int64_t i = ax ? e - ws : e;
    const int64_t cnt = ax ? hs : ws;
    const SliceTab& T = TT[ax];
    if (ax != ax_prev) { jp = 0; ax_prev = ax; }
    while (T.hi[jp] < i) jp++;
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    for (int j = jp; j < k && T.lo[j] <= i; j++) {
      lo = min(lo, T.flo[j]);
      hi = max(hi, T.chi[j]);
    }
    int64_t L = max(0, lo), H = min((int64_t)hi, ax ? ws : hs);
    if (j8 != 0) {
      const bool last = i == cnt - 1;
      const int q0 = 2 * ax, q1 = 2 * ax + 1;
      int64_t v;
      if (i <= O.iA[q0] && (last ? O.lastB[q0] != 0 : i >= O.iB[q0])) v = O.star[q0];
      else if (i > O.iA[q0]) v = lindiv_eval(O.lin[4 * ax + 0], i);
      else v = last ? O.last[q0] : lindiv_eval(O.lin[4 * ax + 1], i);
      L = max(L, v);
      if (i <= O.iA[q1] && (last ? O.lastB[q1] != 0 : i >= O.iB[q1])) v = O.star[q1];
      else if (i > O.iA[q1]) v = -lindiv_eval(O.lin[4 * ax + 2], i);
      else v = last ? O.last[q1] : -lindiv_eval(O.lin[4 * ax + 3], i);
      H = min(H, v);
    }
    (ax ? row : col)[i + 2 * pp.g] = (uint32_t)L | ((uint32_t)H << 16);
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
