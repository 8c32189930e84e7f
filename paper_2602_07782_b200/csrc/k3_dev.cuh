// k3_dev.cuh -- device-side footprint rasterization shared by the K3 kernels
// (k_profile.cu) and the fused persistent pack kernel (k_pack.cu).
// See k_profile.cu for the method (D11, D13).
#pragma once
#include "tabi_internal.cuh"

namespace tabi {
namespace k3 {

constexpr int kRaw = 8192;   // raw cells per chunk (32 KB)
constexpr int kDilMax = 2;   // gutters up to this use the fused raster + dilation pass
#ifndef TABI_RUN_MIN
#define TABI_RUN_MIN 1
#endif
constexpr int kRunMin = TABI_RUN_MIN | 1;  // shortest dilated-output run per thread
// Per-(chart, candidate) constants.  OBB index q = axis * 2 + (0 low, 1 high);
// lines lin[axis * 4 + kind]: kind 0 low-bound line right of the crossing
// (at the cell's low edge), 1 low-bound line left of it (high edge, non-last
// cells), 2 / 3 the same for the high bound (negated floors).
struct ObbC {
  LinDiv lin[8];
  int64_t last[4];   // value at the clipped high edge of the last cell
  int64_t star[4];   // value at the crossing
  // iA / iB are only compared with cell indices (< 2^30), so they are kept
  // clamped to +-2^30 (the same comparisons), in 32 bits
  int32_t iA[4];     // crossing at or beyond cell i's low edge  <=>  i <= iA
  int32_t iB[4];     // crossing at or before cell i's high edge <=>  i >= iB (non-last)
  int32_t lastB[4];  // same test for the last cell (edge = chart extent)
  int32_t starc[4], lastc[4];  // star / last clamped to +-2^30 (RawIter's bounds)
};

// v clamped to +-2^30: where a value is only compared with cell indices or
// texel values (both far smaller), the clamp changes no comparison
__device__ __forceinline__ int32_t clamp30(int64_t v) {
  return (int32_t)(v < -(1ll << 30) ? -(1ll << 30) : v > (1ll << 30) ? (1ll << 30) : v);
}

struct ChartK3 {
  int32_t s, c, ws, hs, j8, small;  // small: handled by the tile kernel
  int32_t col_o, row_o;             // slot offsets in dcol / drow (candidate base added)
  int64_t nw, nh;
  double rnw, rnh;                  // 1 / (num * w), 1 / (num * h)
  ObbC O;
};

// ---- setup jobs ---------------------------------------------------------
// Slice entry: scaled floor of the low bound / ceil of the high bound.
__device__ __forceinline__ void slice_job(int32_t* tab, const int32_t* blo, const int32_t* bhi, int j,
                                          int64_t num, int64_t SC, double rSC) {
  tab[2 * j] = (int32_t)fdiv_r64(num * blo[j], SC, rSC);
  tab[2 * j + 1] = (int32_t)(-fdiv_r64(-num * bhi[j], SC, rSC));
}


// OBB job r (0..7) of a chart: LinDiv r, one of last/star, one of iA/iB.  The
// box is {Umin <= xC + yS <= Umax, Vmin <= -xS + yC <= Vmax}; with num/SC:
//  top    y_top(x)   = max((Umin - xC)/S, (Vmin + xS)/C)
//  bottom y_bot(x)   = min((Umax - xC)/S, (Vmax + xS)/C)
//  left   x_left(y)  = max((Umin - yS)/C, (yC - Vmax)/S)
//  right  x_right(y) = min((Umax - yS)/C, (yC - Vmin)/S)
// The 8 jobs of a chart run on 8 lanes of one warp, so the job index only
// selects operands: every lane then runs the same three divisions (no 8-way
// divergence through per-job branches).
__device__ inline void obb_job(ObbC& O, int r, int64_t C, int64_t S, i128 UMN, i128 UXN, i128 VMN,
                               i128 VXN, int64_t SC, int64_t nw, int64_t nh) {
  const int64_t N2 = C * C + S * S, DS = S * SC, DC = C * SC;
  const i128 N2SC = (i128)N2 * SC;
  const double rDS = rcp_approx((double)DS), rDC = rcp_approx((double)DC);
  const double rN2SC = rcp_approx(i128_to_double(N2SC));
  const int64_t SCS = SC * S, SCC = SC * C;
  const int q = r & 3;
  {  // LinDiv r: f(i) = floor((A + i B) / D)
    const bool dc = r == 0 || r == 3 || r == 5 || r == 6;
    const int64_t D = dc ? DC : DS;
    const double rD = dc ? rDC : rDS;
    const i128 A0 = (r == 0 || r == 7) ? VMN : (r == 1 || r == 5) ? UMN : (r == 2 || r == 6) ? -UXN : -VXN;
    const int64_t Aoff = (r == 1 || r == 7) ? -SCC : (r == 3 || r == 5) ? -SCS : 0;
    const int64_t B = (r == 0 || r == 6) ? SCS : (r == 2 || r == 4) ? SCC : (r == 3 || r == 5) ? -SCS : -SCC;
    const i128 A = A0 + Aoff;
    LinDiv L;
    L.D = D;
    L.rcp = rD;
    L.qA = fdiv_r128(A, (i128)D, rD, false);
    L.rA = (int64_t)(A - mul_wide(L.qA, D));
    L.qB = fdiv_r64(B, D, rD);
    L.rB = B - L.qB * D;
    O.lin[r] = L;
  }
  // jobs 0-3: value at the last cell's clipped edge; 4-7: value at the
  // crossing.  Even q rounds down, odd q up: v = sg * floor(sg * num / den).
  {
    const int64_t sg = (q & 1) ? -1 : 1;
    i128 nm, den;
    double rden;
    if (r < 4) {
      const i128 X = q == 0 ? UMN : q == 1 ? VXN : q == 2 ? UMN : -VMN;
      const int64_t f = q < 2 ? nw : nh;
      const int64_t P = q == 0 ? -C : q == 1 ? S : q == 2 ? -S : C;
      nm = X + mul_wide(f, P);
      const bool ds = q == 0 || q == 3;
      den = ds ? DS : DC;
      rden = ds ? rDS : rDC;
    } else {
      const int64_t m1 = q < 2 ? S : C, m2 = q < 2 ? C : -S;
      const i128 X1 = (q & 1) ? UXN : UMN;
      const i128 X2 = q == 0 ? VMN : q == 1 ? VXN : q == 2 ? VXN : VMN;
      nm = (i128)m1 * X1 + (i128)m2 * X2;
      den = N2SC;
      rden = rN2SC;
    }
    const int64_t v = sg * fdiv_r128(sg > 0 ? nm : -nm, den, rden, false);
    if (r < 4) { O.last[q] = v; O.lastc[q] = clamp30(v); }
    else { O.star[q] = v; O.starc[q] = clamp30(v); }
  }
  {  // crossing x* / x** / y* / y**: i <= iA  (jobs 0-3), i >= iB (jobs 4-7)
    const int64_t m1 = q < 2 ? C : S;
    const int64_t m2 = q < 2 ? -S : C;
    const i128 X1 = (q & 1) ? UXN : UMN;
    const i128 X2 = q == 0 ? VMN : q == 1 ? VXN : q == 2 ? VXN : VMN;
    const i128 cross = (i128)m1 * X1 + (i128)m2 * X2;
    if (r < 4) {
      O.iA[q] = clamp30(fdiv_r128(cross, N2SC, rN2SC, true));
      O.lastB[q] = cross <= mul_wide(q < 2 ? nw : nh, N2);
    } else {
      O.iB[q] = clamp30(-fdiv_r128(-cross, N2SC, rN2SC, true) - 1);
    }
  }
}

// Raw (undilated) bounds of cell i on axis ax (0: column -> (Top, Bottom),
// 1: row -> (Left, Right)), packed lo | hi << 16.
__device__ __forceinline__ uint32_t raw_cell(const ChartK3& H, const int32_t* tab, int k, int ax,
                                             int64_t i, int64_t num, int64_t SC) {
  const int64_t nx = ax ? H.nh : H.nw;
  const double rnx = ax ? H.rnh : H.rnw;
  const int64_t SCk = SC * k;
  int64_t jl = fdiv_r64(i * SCk, nx, rnx);
  int64_t jh = -fdiv_r64(-(i + 1) * SCk, nx, rnx) - 1;
  if (jl < 0) jl = 0;
  if (jh > k - 1) jh = k - 1;
  const int32_t* t = tab + ax * 2 * k;
  int32_t lo = INT32_MAX, hi = INT32_MIN;
  for (int64_t j = jl; j <= jh; j++) {
    lo = min(lo, t[2 * j]);
    hi = max(hi, t[2 * j + 1]);
  }
  const int64_t cnt = ax ? H.hs : H.ws;
  int64_t L = max(0, lo), Hh = min((int64_t)hi, ax ? (int64_t)H.ws : (int64_t)H.hs);
  if (H.j8 != 0) {
    const ObbC& O = H.O;
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
    Hh = min(Hh, v);
  }
  return (uint32_t)L | ((uint32_t)Hh << 16);
}

// raw_cell for the consecutive cells i0 .. i0 + len - 1 of one axis, written
// to out[0 .. len).  Same values; the per-cell divisions become running
// quotients: the slice index bounds jl(i) = floor(i SCk / nx) and
// jh(i) = floor(((i + 1) SCk - 1) / nx) and the four OBB line progressions each
// advance by one add and one conditional carry per cell.
__device__ __forceinline__ void raw_run(const ChartK3& H, const int32_t* tab, int k, int ax,
                                        int64_t i0, int len, int64_t SC, uint32_t* out) {
  const int64_t nx = ax ? H.nh : H.nw;
  const double rnx = ax ? H.rnh : H.rnw;
  const int64_t SCk = SC * k;
  const int64_t dq = fdiv_r64(SCk, nx, rnx), dr = SCk - dq * nx;
  int64_t a = i0 * SCk;
  int64_t ql = fdiv_r64(a, nx, rnx), rl = a - ql * nx;
  a += SCk - 1;
  int64_t qh = fdiv_r64(a, nx, rnx), rh = a - qh * nx;
  const int32_t* t = tab + ax * 2 * k;
  const int64_t cnt = ax ? H.hs : H.ws;
  const int64_t ext = ax ? H.ws : H.hs;
  const bool obb = H.j8 != 0;
  const ObbC& O = H.O;
  const int q0 = 2 * ax, q1 = 2 * ax + 1;
  int64_t v[4] = {0, 0, 0, 0}, r[4] = {0, 0, 0, 0}, sq[4] = {0, 0, 0, 0}, sr[4] = {0, 0, 0, 0},
          D[4] = {1, 1, 1, 1};
  int64_t iA0 = 0, iA1 = 0, iB0 = 0, iB1 = 0, st0 = 0, st1 = 0, la0 = 0, la1 = 0;
  int32_t lb0 = 0, lb1 = 0;
  if (obb) {
#pragma unroll
    for (int p = 0; p < 4; p++) {
      const LinDiv& L = O.lin[4 * ax + p];
      lindiv_start(L, i0, v[p], r[p]);
      sq[p] = L.qB;
      sr[p] = L.rB;
      D[p] = L.D;
    }
    iA0 = O.iA[q0]; iA1 = O.iA[q1]; iB0 = O.iB[q0]; iB1 = O.iB[q1];
    st0 = O.star[q0]; st1 = O.star[q1]; la0 = O.last[q0]; la1 = O.last[q1];
    lb0 = O.lastB[q0]; lb1 = O.lastB[q1];
  }
  for (int c = 0; c < len; c++) {
    const int64_t i = i0 + c;
    const int64_t jl = ql < 0 ? 0 : ql, jh = qh > k - 1 ? k - 1 : qh;
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    for (int64_t j = jl; j <= jh; j++) {
      lo = min(lo, t[2 * j]);
      hi = max(hi, t[2 * j + 1]);
    }
    int64_t L = max(0, lo), Hh = min((int64_t)hi, ext);
    if (obb) {
      const bool last = i == cnt - 1;
      int64_t w;
      if (i <= iA0 && (last ? lb0 != 0 : i >= iB0)) w = st0;
      else if (i > iA0) w = v[0];
      else w = last ? la0 : v[1];
      L = max(L, w);
      if (i <= iA1 && (last ? lb1 != 0 : i >= iB1)) w = st1;
      else if (i > iA1) w = -v[2];
      else w = last ? la1 : -v[3];
      Hh = min(Hh, w);
#pragma unroll
      for (int p = 0; p < 4; p++) {
        v[p] += sq[p];
        r[p] += sr[p];
        if (r[p] >= D[p]) { r[p] -= D[p]; v[p]++; }
      }
    }
    out[c] = (uint32_t)L | ((uint32_t)Hh << 16);
    ql += dq; rl += dr;
    if (rl >= nx) { rl -= nx; ql++; }
    qh += dq; rh += dr;
    if (rh >= nx) { rh -= nx; qh++; }
  }
}

// raw_cell as an iterator over consecutive cells i0, i0 + 1, ... of one axis
// (same values as raw_run).  Each OBB bound is piecewise over the cells: the
// low (high) bound follows line 1 (3) below its crossing band, the crossing
// value star in the band [iB, iA], line 0 (2) past iA, and the last cell's
// own value if the last cell is not past iA.  The iterator keeps only the
// current piece of each bound -- a progression (a constant piece is one with
// zero step) and the cell index where the next piece starts -- and reads the
// next piece's constants from the chart's ObbC in shared memory there, so the
// per-cell loop carries few registers.
struct RawIter {
  const int32_t* t;
  const ObbC* O;
  int64_t nx, rl, rh;                // slice-index progressions: remainders mod nx
  int64_t dr;                        // SCk - dq * nx (SCk = SC k: 2^28 k in tail mode)
  int32_t dq, ql, qh, k, cnt, ext, i, ax;
  bool obb;
  // bound b (0 low, 1 high): value (the high bound's negated), clamped to
  // +-2^30 where only compared with cell indices / texel values (both far
  // smaller); its step, remainder, divisor; the cell where its piece ends
  int32_t v[2], sq[2], sw[2];
  int64_t r[2], sr[2], D[2];
  // bound b's piece containing cell `at`
  __device__ __forceinline__ void seg(int b, int32_t at) {
    const int q = 2 * ax + b;
    const int32_t iA = O->iA[q], iB = O->iB[q], last = cnt - 1;
    const bool line = at > iA || (at != last && at < iB);
    if (line) {  // floor((A + i B) / D) from cell `at` on
      const LinDiv& L = O->lin[4 * ax + 2 * b + (at > iA ? 0 : 1)];
      int64_t vv;
      lindiv_start(L, at, vv, r[b]);
      v[b] = clamp30(vv);
      sq[b] = (int32_t)L.qB;
      sr[b] = L.rB;
      D[b] = L.D;
      sw[b] = at > iA ? INT32_MAX : min(min(iB, iA + 1), last);
    } else {  // the crossing value, or the last cell's
      const int32_t c = at == last && O->lastB[q] == 0 ? O->lastc[q] : O->starc[q];
      v[b] = b ? -c : c;
      sq[b] = 0;
      r[b] = 0;
      sr[b] = 0;
      D[b] = 1;
      sw[b] = at == last ? INT32_MAX : min(iA + 1, last);
    }
  }
  __device__ __forceinline__ void init(const ChartK3& H, const int32_t* tab, int k_, int ax_,
                                       int32_t i0, int64_t SC) {
    k = k_;
    ax = ax_;
    nx = ax ? H.nh : H.nw;
    const double rnx = ax ? H.rnh : H.rnw;
    const int64_t SCk = SC * k;
    const int64_t q = fdiv_r64(SCk, nx, rnx);
    dq = (int32_t)q;
    dr = SCk - q * nx;
    const int64_t a = (int64_t)i0 * SCk;
    const int64_t f = fdiv_r64(a, nx, rnx);
    ql = (int32_t)f;
    rl = a - f * nx;
    // a + SCk - 1 = (ql + dq) nx + (rl + dr - 1), with rl + dr - 1 in [-1, 2 nx - 2]
    rh = rl + dr - 1;
    qh = ql + dq;
    if (rh < 0) { rh += nx; qh--; }
    else if (rh >= nx) { rh -= nx; qh++; }
    t = tab + ax * 2 * k;
    cnt = ax ? H.hs : H.ws;
    ext = ax ? H.ws : H.hs;
    i = i0;
    obb = H.j8 != 0;
    if (obb) {
      O = &H.O;
      seg(0, i0);
      seg(1, i0);
    }
  }
  // value of cell i (packed lo | hi << 16), then move to i + 1
  __device__ __forceinline__ uint32_t next() {
    const int32_t jl = ql < 0 ? 0 : ql, jh = qh > k - 1 ? k - 1 : qh;
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    const int2* t2 = reinterpret_cast<const int2*>(t);  // (lo, hi) of slice j: one 8-byte load
    for (int32_t j = jl; j <= jh; j++) {
      const int2 e = t2[j];
      lo = min(lo, e.x);
      hi = max(hi, e.y);
    }
    int32_t L = max(0, lo), Hh = min(hi, ext);
    if (obb) {
      L = max(L, v[0]);
      Hh = min(Hh, -v[1]);
#pragma unroll
      for (int b = 0; b < 2; b++) {
        v[b] += sq[b];
        r[b] += sr[b];
        if (r[b] >= D[b]) { r[b] -= D[b]; v[b]++; }
        if (i + 1 == sw[b]) seg(b, i + 1);
      }
    }
    ql += dq; rl += dr;
    if (rl >= nx) { rl -= nx; ql++; }
    qh += dq; rh += dr;
    if (rh >= nx) { rh -= nx; qh++; }
    i++;
    return (uint32_t)L | ((uint32_t)Hh << 16);
  }
};

// Raster and dilation fused (D11 + D13) for gutters g <= GMAX: the dilated
// outputs o0 .. o0 + len - 1 of one axis (Dlo(o) = min Lo(q), Dhi(o) = max
// Hi(q) + 2g over raw cells q in [o - 2g, o] within [0, n0)), written to
// dst[0 .. len), the raw cells kept in a (2g + 1)-entry register window
// instead of a shared-memory buffer.  A window entry packs lo | (0xffff - hi)
// << 16, so one per-halfword minimum (vminu2) takes both bounds.
template <int GMAX>
__device__ __forceinline__ void dil_run(const ChartK3& H, const int32_t* tab, int k, int ax,
                                        int32_t o0, int32_t len, int64_t SC, int g, uint32_t* dst,
                                        uint32_t* dst2 = nullptr) {
  constexpr int WN = 2 * GMAX + 1;
  const int32_t n0 = ax ? H.hs : H.ws;
  RawIter it;
  it.init(H, tab, k, ax, max(0, o0 - 2 * g), SC);
  uint32_t win[WN];  // raw cells o - 2g .. o at slots WN - 1 - 2g .. WN - 1 (sentinel: empty)
#pragma unroll
  for (int u = 0; u < WN; u++) win[u] = 0xffffffffu;
  for (int32_t q = o0 - 2 * g; q < o0 + len; q++) {
#pragma unroll
    for (int u = 0; u + 1 < WN; u++) win[u] = win[u + 1];
    uint32_t e = 0xffffffffu;
    if (q >= 0 && q < n0) {
      const uint32_t v = it.next();
      e = (v & 0xffffu) | ((0xffffu - (v >> 16)) << 16);
    }
    win[WN - 1] = e;
    if (q >= o0) {
      uint32_t m = win[WN - 1];
#pragma unroll
      for (int u = WN - 2; u >= 0; u--)
        if (WN - 1 - u <= 2 * g) m = __vminu2(m, win[u]);
      const uint32_t val = (m & 0xffffu) | ((0xffffu - (m >> 16) + 2 * g) << 16);
      dst[q - o0] = val;
      if (dst2) dst2[q - o0] = val;
    }
  }
}

// Setup of one chart by 8 cooperating threads r = 0..7 (rank r).
__device__ inline void chart_setup(ChartK3& H, int32_t* tab, const Proxies& P, int k, int64_t num,
                            int64_t SC, int r) {
  const int c = H.c;
  const int32_t* sl = P.sl + (int64_t)c * 4 * k;
  const double rSC = rcp_approx((double)SC);
  for (int idx = r; idx < 2 * k; idx += 8) {
    const int ax = idx >= k, j = ax ? idx - k : idx;
    slice_job(tab + ax * 2 * k, sl + 2 * ax * k, sl + 2 * ax * k + k, j, num, SC, rSC);
  }
  if (H.j8 != 0) {
    const int64_t* ob = P.obb + 4 * (int64_t)c;
    obb_job(H.O, r, kQC[H.j8], kQS[H.j8], mul_wide(ob[0], num), mul_wide(ob[1], num),
            mul_wide(ob[2], num), mul_wide(ob[3], num), SC, H.nw, H.nh);
  }
}

// Warp per large chart (raw cells > kRaw) from the compacted list; raw values
// go straight into the HBM slot, then an in-place dilation.
__device__ inline void dilate_slot(uint32_t* slot, int32_t n0, int32_t g, int lane) {
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

// Scale of candidate m: m/M, or in tail mode the prefix tail's p / 2^20 (D24).
struct Scale {
  int64_t num, SC;
  int32_t r0;  // first sorted position rasterized (tail mode), else 0
};

// Rasterize the footprints of the TC charts [s0, s0 + TC) at scale sc into the
// per-candidate arrays of index `slot` (m - 1 for a single pack) with
// TT threads (8 per chart during setup).  Charts that fit the dilated atlas but
// have more than kRaw raw cells are left for a warp-per-chart pass: their tile
// index is flagged in big[ci].  Writes wd/hd, the footprint slots, cand_bad.
struct NoMark {  // mark(0): setup done; mark(1): a chunk's raw pass done
  __device__ void operator()(int) const {}
};

template <int TC, int TT, int RAW, class Sync, class Mark = NoMark>
__device__ void tile_raster(const Proxies& P, const int32_t* __restrict__ perm, const PackParams& pp,
                            const int32_t* __restrict__ colofs, const int32_t* __restrict__ rowofs,
                            uint32_t* dcol, uint32_t* drow, int32_t* wd_all, int32_t* hd_all,
                            int32_t* cand_bad, int slot, int s0, Scale sc, ChartK3* CH,
                            int32_t* cells, int32_t* cpre, int32_t* opre, int32_t* chunk_end,
                            int32_t* big, int32_t* tabs, uint32_t* raw, int nt, int tid,
                            Sync sync, Mark setup_done = Mark(), uint32_t* rstash = nullptr,
                            int32_t rstash_cap = 0) {
  const int k = pp.k, g = pp.g;  // tile = sorted positions [s0, s0 + nt), nt <= TC
  const int64_t num = sc.num, SC = sc.SC;
  const double rSC = rcp_approx((double)SC);
  const int ci = tid >> 3, r = tid & 7;
  // g <= kDilMax: the fused raster+dilation pass has no raw buffer, so every
  // fitting chart is rasterized here (no large-chart hand-off)
  const int raw_cap = g <= kDilMax ? INT32_MAX : RAW;
  if (ci < TC && r == 0) {
    cells[ci] = 0;
    big[ci] = 0;
    CH[ci].small = 0;
  }
  if (ci < nt && r == 0 && s0 + ci >= sc.r0) {
    ChartK3& H = CH[ci];
    const int s = s0 + ci;
    const int c = perm[s];
    const int64_t w = P.w[c], h = P.h[c];
    H.s = s;
    H.c = c;
    H.nw = num * w;
    H.nh = num * h;
    H.ws = (int32_t)(-fdiv_r64(-H.nw, SC, rSC));
    H.hs = (int32_t)(-fdiv_r64(-H.nh, SC, rSC));
    H.rnw = rcp_approx((double)H.nw);
    H.rnh = rcp_approx((double)H.nh);
    H.j8 = P.obb_j[c];
    const int64_t b = (int64_t)slot * pp.n + s;
    wd_all[b] = H.ws + 2 * g;
    hd_all[b] = H.hs + 2 * g;
    const bool fits = H.ws + 2 * g <= pp.Wp && H.hs + 2 * g <= pp.Hp;
    if (!fits) cand_bad[slot] = 1;
    H.small = fits && (H.ws + H.hs <= raw_cap);
    big[ci] = fits && !H.small;
    H.col_o = colofs[s];
    H.row_o = rowofs[s];
    cells[ci] = H.small ? H.ws + H.hs : 0;
  }
  sync();
  if (ci < nt && CH[ci].small) chart_setup(CH[ci], tabs + ci * 4 * k, P, k, num, SC, r);
  sync();
  setup_done(0);
  uint32_t* colb = dcol + (int64_t)slot * pp.col_cap;
  uint32_t* rowb = drow + (int64_t)slot * pp.row_cap;
  if (g <= kDilMax) {
    // fused raster + dilation (dil_run): no raw buffer, every fitting chart of
    // the tile in one pass over its flattened dilated outputs (Wd + Hd each)
    // (with rstash: cpre = the prefix of the dilated row counts, and each
    // chart's row outputs also go to rstash + cpre[ci] -- the caller's pair
    // offsets then read shared memory; only if they all fit rstash_cap)
    // Runs: each chart axis (Wd column outputs, then Hd row outputs) is cut
    // into runs of at most R outputs and every thread takes one run, so a
    // run never crosses into another chart: each thread starts one iterator
    // and the warps' loops have (nearly) equal lengths.  R is the smallest
    // length (from ceil(outputs / TT) up) whose runs fit the TT threads --
    // some R <= max(Wd, Hd) does (2 runs per chart, 2 TC <= TT).
    // opre = the prefix of the charts' run counts.
    if (tid < 32) {
      const int lane = tid;
      int32_t nout = 0;
      for (int idx = lane; idx < nt; idx += 32)
        if (CH[idx].small) nout += CH[idx].ws + CH[idx].hs + 4 * g;
      nout = warp_sum(nout);
      int32_t R = max(kRunMin, (nout + TT - 1) / TT);
      while (true) {
        int32_t runs = 0;
        for (int idx = lane; idx < nt; idx += 32)
          if (CH[idx].small)
            runs += (CH[idx].ws + 2 * g + R - 1) / R + (CH[idx].hs + 2 * g + R - 1) / R;
        if (warp_sum(runs) <= TT) break;
        R += max(1, R >> 3);
      }
      int otot = 0, rtot = 0;
      if (lane == 0) { opre[0] = 0; cpre[0] = 0; *chunk_end = R; }
      for (int e = 0; e < nt; e += 32) {
        const int idx = e + lane;
        const bool sm = idx < nt && CH[idx].small;
        int io = sm ? (CH[idx].ws + 2 * g + R - 1) / R + (CH[idx].hs + 2 * g + R - 1) / R : 0;
        int ir = sm ? CH[idx].hs + 2 * g : 0;
        // (the pass covers fitting charts only; big[] stays 0 on this path)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int b = __shfl_up_sync(0xffffffffu, io, o);
          const int br = __shfl_up_sync(0xffffffffu, ir, o);
          if (lane >= o) { io += b; ir += br; }
        }
        if (idx < nt) { opre[idx + 1] = otot + io; cpre[idx + 1] = rtot + ir; }
        otot += __shfl_sync(0xffffffffu, io, 31);
        rtot += __shfl_sync(0xffffffffu, ir, 31);
      }
    }
    sync();
    setup_done(1);
    if (rstash && cpre[nt] > rstash_cap) rstash = nullptr;  // (uniform)
    const int32_t R = *chunk_end;
    if (tid < opre[nt]) {
      int lo = 0, hi = nt - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (opre[mid] <= tid) lo = mid;
        else hi = mid - 1;
      }
      const ChartK3& H = CH[lo];
      const int32_t Wd = H.ws + 2 * g, Hd = H.hs + 2 * g;
      const int32_t u = tid - opre[lo], ncol = (Wd + R - 1) / R;
      const int ax = u >= ncol;
      const int32_t o = (ax ? u - ncol : u) * R;
      const int32_t len = min(R, (ax ? Hd : Wd) - o);
      dil_run<kDilMax>(H, tabs + lo * 4 * k, k, ax, o, len, SC, g,
                       (ax ? rowb + H.row_o : colb + H.col_o) + o,
                       ax && rstash ? rstash + cpre[lo] + o : nullptr);
    }
    sync();
    return;
  }
  int cb = 0;
  while (cb < nt && cells[cb] == 0) cb++;
  while (cb < nt) {
    if (tid < 32) {  // warp 0 plans chunk [cb, ce): raw cells fit the buffer
      // 32 charts per step: inclusive scans of raw cells and dilated outputs;
      // "fits" is a prefix property (cells >= 0), so a ballot gives the count
      const int lane = tid;
      int e = cb, tot = 0, otot = 0;
      if (lane == 0) { cpre[0] = 0; opre[0] = 0; }
      while (e < nt) {
        const int idx = e + lane;
        const int c = idx < nt ? cells[idx] : RAW + 1;  // past the tile: never fits
        int ic = c, io = (idx < nt && c) ? c + 4 * g : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int a = __shfl_up_sync(0xffffffffu, ic, o);
          const int b = __shfl_up_sync(0xffffffffu, io, o);
          if (lane >= o) { ic += a; io += b; }
        }
        const unsigned fit = __ballot_sync(0xffffffffu, tot + ic <= RAW);
        const int nf = fit == 0xffffffffu ? 32 : __ffs(~fit) - 1;
        if (lane < nf) {
          cpre[e - cb + lane + 1] = tot + ic;
          opre[e - cb + lane + 1] = otot + io;
        }
        if (nf > 0) {
          tot += __shfl_sync(0xffffffffu, ic, nf - 1);
          otot += __shfl_sync(0xffffffffu, io, nf - 1);
        }
        e += nf;
        if (nf < 32) break;
      }
      if (lane == 0) *chunk_end = e;
    }
    sync();
    const int ce = *chunk_end, nc = ce - cb;
    const int32_t ncell = cpre[nc], nout = opre[nc];
    {  // raw pass: each thread a contiguous run of the flattened cells (odd
       // length: the runs' smem stores hit distinct banks), evaluated incrementally
      const int32_t R = ((ncell + TT - 1) / TT) | 1;
      int32_t e = tid * R;
      const int32_t e1 = min(ncell, e + R);
      if (e < e1) {
        int lo = 0, hi = nc - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (cpre[mid] <= e) lo = mid;
          else hi = mid - 1;
        }
        while (e < e1) {
          const ChartK3& H = CH[cb + lo];
          const int32_t x = e - cpre[lo];
          const int ax = x >= H.ws;
          const int32_t len = min(e1 - e, (ax ? H.ws + H.hs : H.ws) - x);
          raw_run(H, tabs + (cb + lo) * 4 * k, k, ax, ax ? x - H.ws : x, len, SC, raw + e);
          e += len;
          while (lo < nc - 1 && cpre[lo + 1] <= e) lo++;  // next chart with cells
        }
      }
    }
    sync();
    setup_done(1);
    for (int o = tid; o < nout; o += TT) {  // dilation over the flattened outputs
      int lo = 0, hi = nc - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (opre[mid] <= o) lo = mid;
        else hi = mid - 1;
      }
      const ChartK3& H = CH[cb + lo];
      const int32_t y = o - opre[lo];
      const int Wd = H.ws + 2 * g;
      const int ax = y >= Wd;
      const int32_t i = ax ? y - Wd : y;
      const int32_t n0 = ax ? H.hs : H.ws;
      const uint32_t* rr = raw + cpre[lo] + (ax ? H.ws : 0);
      const int q0 = max(0, i - 2 * g), q1 = min(i, n0 - 1);
      int32_t vl = INT32_MAX, vh = INT32_MIN;
      for (int q = q0; q <= q1; q++) {
        const uint32_t v = rr[q];
        vl = min(vl, lo16(v));
        vh = max(vh, hi16(v));
      }
      (ax ? rowb + H.row_o : colb + H.col_o)[i] = (uint32_t)vl | ((uint32_t)(vh + 2 * g) << 16);
    }
    sync();
    cb = ce;
    while (cb < nt && cells[cb] == 0) cb++;  // skip charts handled elsewhere
    sync();
  }
}

// One large chart (sorted position s, candidate m) by one warp: raw values
// straight into the HBM slot, then an in-place dilation.
__device__ inline void big_chart(const Proxies& P, const int32_t* __restrict__ perm, const PackParams& pp,
                          const int32_t* __restrict__ colofs, const int32_t* __restrict__ rowofs,
                          uint32_t* dcol, uint32_t* drow, int slot, int s, Scale sc, ChartK3& H,
                          int32_t* tab, int lane) {
  const int k = pp.k;
  const int64_t num = sc.num, SC = sc.SC;
  const double rSC = rcp_approx((double)SC);
  if (lane == 0) {
    const int c = perm[s];
    H.s = s;
    H.c = c;
    H.nw = num * P.w[c];
    H.nh = num * P.h[c];
    H.ws = (int32_t)(-fdiv_r64(-H.nw, SC, rSC));
    H.hs = (int32_t)(-fdiv_r64(-H.nh, SC, rSC));
    H.rnw = rcp_approx((double)H.nw);
    H.rnh = rcp_approx((double)H.nh);
    H.j8 = P.obb_j[c];
  }
  __syncwarp();
  if (lane < 8) chart_setup(H, tab, P, k, num, SC, lane);
  __syncwarp();
  uint32_t* col = dcol + (int64_t)slot * pp.col_cap + colofs[s];
  uint32_t* row = drow + (int64_t)slot * pp.row_cap + rowofs[s];
  for (int64_t e = lane; e < (int64_t)H.ws + H.hs; e += 32) {
    const int ax = e >= H.ws;
    const int64_t i = ax ? e - H.ws : e;
    (ax ? row : col)[i + 2 * pp.g] = raw_cell(H, tab, k, ax, i, num, SC);
  }
  __syncwarp();
  dilate_slot(col, H.ws, pp.g, lane);
  dilate_slot(row, H.hs, pp.g, lane);
  __syncwarp();
}

// Compaction advance off(s, s+1) and CannotMoveAbove bits of the adjacent
// pair, by one warp (D14, D15).  The footprint arrays
// are plain (coherent) loads: in the fused kernel another CTA wrote chart s.
// The pair from its two dilated row footprints ra, rb (HBM or shared memory)
// and sizes; stores off and the lock bits at *off_o, *lock_o.
__device__ __forceinline__ void pair_rows(const uint32_t* ra, const uint32_t* rb, int32_t Hda,
                                          int32_t Hdb, int32_t Wda, int32_t* off_o, uint8_t* lock_o,
                                          int lane) {
  const int rows = min(Hda, Hdb);
  int32_t off = 0;
  for (int j = lane; j < rows; j += 32) off = max(off, hi16(ra[j]) - lo16(rb[j]));
  off = warp_max(off);
  bool la = false, lb = false;
  if (off < Wda) warp_locks(ra, rb, Hda, Hdb, off, lane, la, lb);
  if (lane == 0) {
    *off_o = off;
    *lock_o = (uint8_t)((la ? 1 : 0) | (lb ? 2 : 0));
  }
}

__device__ __forceinline__ void pair_offset(const PackParams& pp, const int32_t* __restrict__ rowofs,
                                            const uint32_t* drow, const int32_t* wd_all,
                                            const int32_t* hd_all, int32_t* off_all,
                                            uint8_t* lock_all, int slot, int s, int lane) {
  const int64_t base = (int64_t)slot * pp.n;
  if (s == pp.n - 1) {
    if (lane == 0) { off_all[base + s] = 0; lock_all[base + s] = 0; }
    return;
  }
  const int32_t Hda = hd_all[base + s], Hdb = hd_all[base + s + 1], Wda = wd_all[base + s];
  const uint32_t* ra = drow + (int64_t)slot * pp.row_cap + rowofs[s];
  const uint32_t* rb = drow + (int64_t)slot * pp.row_cap + rowofs[s + 1];
  pair_rows(ra, rb, Hda, Hdb, Wda, off_all + base + s, lock_all + base + s, lane);
}

// pair_offset for a pair with many shared rows, by a whole group of TT
// threads: the gap maximum is a block reduction, and the lock tests' running
// prefix min / max over rows become one exclusive block scan of per-thread
// segment extrema followed by a walk of each segment -- the same predicates as
// warp_locks, evaluated by TT threads instead of one warp.  red: >= 2 * (TT /
// 32) + 1 ints of shared scratch.  s < n - 1.  Ends with a sync.
template <int TT, class Sync>
__device__ void pair_offset_group(const PackParams& pp, const int32_t* __restrict__ rowofs,
                                  const uint32_t* drow, const int32_t* wd_all,
                                  const int32_t* hd_all, int32_t* off_all, uint8_t* lock_all,
                                  int slot, int s, int tid, Sync sync, int32_t* red) {
  constexpr int NW = TT / 32;
  const int lane = tid & 31, w = tid >> 5;
  const int64_t base = (int64_t)slot * pp.n;
  const int32_t Hda = hd_all[base + s], Hdb = hd_all[base + s + 1], Wda = wd_all[base + s];
  const uint32_t* ra = drow + (int64_t)slot * pp.row_cap + rowofs[s];
  const uint32_t* rb = drow + (int64_t)slot * pp.row_cap + rowofs[s + 1];
  const int rows = min(Hda, Hdb);
  int32_t off = 0;
  for (int j = tid; j < rows; j += TT) off = max(off, hi16(ra[j]) - lo16(rb[j]));
  off = warp_max(off);
  if (lane == 0) red[w] = off;
  if (tid == 0) red[2 * NW] = 0;
  sync();
  off = 0;
  for (int i = 0; i < NW; i++) off = max(off, red[i]);
  sync();
  bool xa = false, xb = false;
  if (off < Wda) {
    const int L = (Hdb + TT - 1) / TT;  // rows [r0, r1) of this thread
    const int r0 = min(Hdb, tid * L), r1 = min(Hdb, r0 + L);
    int32_t smin = INT32_MAX, smax = INT32_MIN;
    for (int r = r0; r < r1; r++) {
      smin = min(smin, lo16(rb[r]));
      smax = max(smax, hi16(ra[r]));
    }
    const int32_t imin = warp_incl_min(smin, lane), imax = warp_incl_max(smax, lane);
    if (lane == 31) { red[w] = imin; red[NW + w] = imax; }
    sync();
    int32_t cmin = INT32_MAX, cmax = INT32_MIN, tmin = INT32_MAX;
    for (int i = 0; i < NW; i++) {
      if (i < w) { cmin = min(cmin, red[i]); cmax = max(cmax, red[NW + i]); }
      tmin = min(tmin, red[i]);
    }
    int32_t emin = __shfl_up_sync(0xffffffffu, imin, 1);
    int32_t emax = __shfl_up_sync(0xffffffffu, imax, 1);
    if (lane == 0) { emin = INT32_MAX; emax = INT32_MIN; }
    emin = min(emin, cmin);  // prefix over rows < r0
    emax = max(emax, cmax);
    for (int r = r0; r < r1; r++) {
      const int32_t lb_r = lo16(rb[r]), ra_r = hi16(ra[r]);
      if (r >= 1) {
        if (emin != INT32_MAX && ra_r > off + emin) xa = true;
        if (emax != INT32_MIN && off + lb_r < emax) xb = true;
      }
      emin = min(emin, lb_r);
      emax = max(emax, ra_r);
    }
    for (int r = Hdb + tid; r < Hda; r += TT)
      if (r >= 1 && hi16(ra[r]) > off + tmin) xa = true;
  }
  const bool any_a = __any_sync(0xffffffffu, xa), any_b = __any_sync(0xffffffffu, xb);
  if (lane == 0 && (any_a || any_b)) atomicOr(&red[2 * NW], (any_a ? 1 : 0) | (any_b ? 2 : 0));
  sync();
  if (tid == 0) {
    off_all[base + s] = off;
    lock_all[base + s] = (uint8_t)red[2 * NW];
  }
  sync();
}

}  // namespace k3
}  // namespace tabi
