// k_proxy.cu -- K1: per-chart proxies, one lane group (8, 16 or 32 lanes) per
// chart.
//
// Computes, for every chart ("compute the AABBs of all charts, rotate the
// boxes to be taller than they are wide ... two parallel passes which compute
// our shape approximations for each chart and determine each chart's
// orientation"):
//   snap to 1/256 texel -> AABB -> 90-degree normalization -> local AABBs
//    + merge -> orientation -> final pose (the
//   slices reflected, D8) -> approximate OBB over 8 angles.
// Lanes stride over vertices / edges (lane v: vertex v and edge (v, v+1));
// the snapped vertices stay in shared memory (charts of <= 64 vertices; larger
// ones use the HBM scratch); slice bounds are accumulated with shared-memory
// atomicMin/Max (commutative, so schedule-independent); reductions are REDUX
// instructions (64-bit sums as four 16-bit-chunk REDUX sums) or shuffles.  The group size trades
// per-chart latency (wide groups, few charts) against charts in flight (narrow
// groups, many small charts): 32 lanes below 4096 charts (a pack of a few
// thousand charts is latency-bound per chart), 16 below 8192, else 8.
// Output: proxy SoA in HBM.
#include <cstdlib>

#include "tabi_internal.cuh"

namespace tabi {
namespace {

constexpr int kBlock = 256;  // threads per block
constexpr int kVCap = 64;    // vertices per group kept in shared memory (larger charts: HBM scratch)

// Per-group shared scratch, k slices per axis (sized by k at launch).
struct Slices {
  int32_t *mlo0, *mlo1, *mhi0, *mhi1;  // x-slices top/bot, y-slices left/right (merged = D4, R7)
  int64_t* ob;                         // [8][4] OBB extents per angle
  int32_t *vx, *vy;                    // [kVCap] the chart's vertices (nv <= kVCap)
};

__host__ __device__ constexpr size_t slice_bytes(int k) {
  return (256 + (size_t)4 * 4 * k + (size_t)8 * kVCap + 15) & ~(size_t)15;
}

template <int G>
struct Group {
  int gl;         // lane within the group
  unsigned mask;  // the group's lanes
  __device__ void sync() const { __syncwarp(mask); }
  template <class T>
  __device__ T xorv(T v, int o) const { return __shfl_xor_sync(mask, v, o, G); }
  // 32-bit group reductions: one REDUX over the group's lanes (the mask)
  __device__ int32_t min32(int32_t v) const { return __reduce_min_sync(mask, v); }
  __device__ int32_t max32(int32_t v) const { return __reduce_max_sync(mask, v); }
  __device__ uint32_t sumu(uint32_t v) const { return __reduce_add_sync(mask, v); }
  // 64-bit sum modulo 2^64 from four independent 16-bit-chunk REDUX sums (each
  // chunk sum < 2^21): exact whenever the true sum fits int64, whatever the
  // lanes' partial sums did
  __device__ int64_t sum64_wrap(int64_t v) const {
    const uint64_t u = (uint64_t)v;
    const uint64_t c0 = sumu((uint32_t)(u & 0xffffu)), c1 = sumu((uint32_t)((u >> 16) & 0xffffu));
    const uint64_t c2 = sumu((uint32_t)((u >> 32) & 0xffffu)), c3 = sumu((uint32_t)(u >> 48));
    return (int64_t)(c0 + (c1 << 16) + (c2 << 32) + (c3 << 48));
  }
};

// floor(a / e) and the remainder, for 0 <= a <= 2^31, 1 <= e <= 2^25 and a
// quotient <= 64 (a = k * coordinate, e = the extent): the double estimate
// from e's reciprocal is off by far less than 1 / e, so truncation gives the
// quotient or one less, and one exact correction step settles it.
__device__ __forceinline__ uint32_t strip_div(uint32_t a, uint32_t e, double re, uint32_t& r) {
  uint32_t q = (uint32_t)((double)a * re);
  int64_t rr = (int64_t)a - (int64_t)((uint64_t)q * e);
  if (rr < 0) { q--; rr += e; }
  else if (rr >= (int64_t)e) { q++; rr -= e; }
  r = (uint32_t)rr;
  return q;
}

// D4: slice bounds along one axis.  A = coordinate that is sliced (x for
// x-slices, in [0, ext]), B = the bounded coordinate.  Strip j = closed range
// k*A in [j*ext, (j+1)*ext].  Lane v takes vertex v and edge (v, v+1): the
// vertex updates the strips holding it, the edge its crossings of the strip
// boundary lines strictly inside it (floored into top, ceiled into bottom).
template <int G>
__device__ void accumulate_slices(const Group<G>& g, const int32_t* A, const int32_t* B, int nv,
                                  int64_t ext, int k, int32_t* lo, int32_t* hi) {
  const uint32_t e = (uint32_t)ext;
  const double re = rcp_approx((double)ext);
  // one crossing y = ya + (L*ext - k*xa) * dy / den of line L with an edge
  // (xa, ya) -> (xa + dx, ya + dy), dx > 0: floored into the top bound and
  // ceiled into the bottom bound of strips L - 1 and L
  auto crossing = [&](int32_t L, int64_t xa, int64_t ya, int64_t dx, int64_t dy) {
    const int64_t den = (int64_t)k * dx;
    const double rd = rcp_approx((double)den);
    // |num| <= den * 2^25 < 2^57
    const int64_t num = ((int64_t)L * e - (int64_t)k * xa) * dy;
    int64_t q = (int64_t)floor((double)num * rd);
    int64_t r = num - q * den;
    while (r < 0) { q--; r += den; }
    while (r >= den) { q++; r -= den; }
    const int32_t yf = (int32_t)(ya + q), yc = yf + (r != 0 ? 1 : 0);
    atomicMin(&lo[L - 1], yf);
    atomicMax(&hi[L - 1], yc);
    atomicMin(&lo[L], yf);
    atomicMax(&hi[L], yc);
  };
  // vertex v: the closed strips holding it; edge (v, v+1): the range [L0, L0 +
  // cnt) of strip boundary lines L*ext strictly inside it (k*xa < L*ext <
  // k*xb, L in [1, k-1]) and its endpoints ordered by the sliced coordinate
  auto vertex_edge = [&](int v, int32_t& xa, int32_t& ya, int32_t& dx, int32_t& dy, int32_t& L0,
                         int32_t& cnt) {
    cnt = 0;
    const int u = v + 1 == nv ? 0 : v + 1;
    const int32_t av = A[v], bv = B[v], au = A[u], bu = B[u];
    uint32_t rv, ru;
    const int32_t qv = (int32_t)strip_div((uint32_t)k * (uint32_t)av, e, re, rv);
    const int32_t qu = (int32_t)strip_div((uint32_t)k * (uint32_t)au, e, re, ru);
    // closed strips holding vertex v: q (unless q = k) and q - 1 when on a line
    if (qv <= k - 1) { atomicMin(&lo[qv], bv); atomicMax(&hi[qv], bv); }
    if (rv == 0 && qv >= 1) { atomicMin(&lo[qv - 1], bv); atomicMax(&hi[qv - 1], bv); }
    if (av == au) return;
    const bool fw = av < au;
    const int32_t qa = fw ? qv : qu, qb = fw ? qu : qv;
    const uint32_t rb = fw ? ru : rv;
    L0 = max(qa + 1, 1);
    const int32_t L1 = min(rb == 0 ? qb - 1 : qb, k - 1);
    if (L0 > L1) return;
    cnt = L1 - L0 + 1;
    xa = fw ? av : au;
    ya = fw ? bv : bu;
    dx = (fw ? au : av) - xa;
    dy = (fw ? bu : bv) - ya;
  };
  if (nv <= G) {
    // one vertex / edge per lane, then the crossings of all edges spread over
    // the lanes (an edge may cross up to k - 1 lines while its neighbours
    // cross none): lane x takes flattened crossings x, x + G, ..., its edge
    // found by a binary search over the lanes' inclusive crossing counts and
    // the edge's values read from the owning lane by shuffles.  The bounds are
    // min / max atomics, so the assignment does not change the result.
    int32_t xa = 0, ya = 0, dx = 0, dy = 0, L0 = 0, cnt = 0;
    if (g.gl < nv) vertex_edge(g.gl, xa, ya, dx, dy, L0, cnt);
    int32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const int32_t t = __shfl_up_sync(g.mask, inc, o, G);
      if (g.gl >= o) inc += t;
    }
    const int32_t total = __shfl_sync(g.mask, inc, G - 1, G);
    for (int32_t x0 = 0; x0 < total; x0 += G) {  // (uniform over the group)
      const int32_t x = x0 + g.gl;
      int pos = 0;  // lanes whose inclusive count is <= x = the owning edge
#pragma unroll
      for (int s = G / 2; s >= 1; s >>= 1) {
        const int32_t iv = __shfl_sync(g.mask, inc, pos + s - 1, G);
        if (iv <= x) pos += s;
      }
      const int32_t ex = __shfl_sync(g.mask, inc - cnt, pos, G);
      const int32_t oL0 = __shfl_sync(g.mask, L0, pos, G);
      const int32_t oxa = __shfl_sync(g.mask, xa, pos, G), oya = __shfl_sync(g.mask, ya, pos, G);
      const int32_t odx = __shfl_sync(g.mask, dx, pos, G), ody = __shfl_sync(g.mask, dy, pos, G);
      if (x < total) crossing(oL0 + (x - ex), oxa, oya, odx, ody);
    }
    return;
  }
  for (int v = g.gl; v < nv; v += G) {
    int32_t xa, ya, dx, dy, L0, cnt;
    vertex_edge(v, xa, ya, dx, dy, L0, cnt);
    for (int32_t L = L0; L < L0 + cnt; L++) crossing(L, xa, ya, dx, dy);
  }
}

// D4 slices, then D5's merge.  D5 is the identity on D4's slices (DESIGN.md
// R7: each slice is the exact extent of the polygon in its closed strip, and
// the y-band holding a strip's topmost point always meets the strip, so the
// merged bound never moves); the merged slices are the accumulated ones --
// pinned by the oracle (which merges literally) in every parity test.
template <int G>
__device__ void merged_slices(const Group<G>& g, const Slices& S, const int32_t* X, const int32_t* Y,
                              int nv, int64_t w, int64_t h, int k) {
  for (int j = g.gl; j < k; j += G) {
    S.mlo0[j] = INT32_MAX; S.mhi0[j] = INT32_MIN;
    S.mlo1[j] = INT32_MAX; S.mhi1[j] = INT32_MIN;
  }
  g.sync();
  accumulate_slices(g, X, Y, nv, w, k, S.mlo0, S.mhi0);
  accumulate_slices(g, Y, X, nv, h, k, S.mlo1, S.mhi1);
  g.sync();
}

// round_half_even(a / 2^30)
__device__ __forceinline__ int64_t q30_round(int64_t a) {
  int64_t q = a >> 30;  // floor
  const int64_t r = a - (q << 30);
  if (r > ((int64_t)1 << 29) || (r == ((int64_t)1 << 29) && (q & 1))) q++;
  return q;
}

// D6's minimum-area angle (ties to the smaller j) of the group's polygon,
// reflected on the fly (x -> w - x if fx, y -> h - y if fy): lane = (G / 8) *
// angle + vertex subgroup; the per-angle extents go through S.ob and lane 0
// picks.  Returns the same j in every lane.
template <int G>
__device__ int obb_angle(const Group<G>& g, const int32_t* X, const int32_t* Y, int nv,
                         const Slices& S, int nj = 8, bool fx = false, bool fy = false,
                         int32_t w = 0, int32_t h = 0) {
  constexpr int VG = G / 8;
  const int j = g.gl / VG, vg = g.gl % VG;
  const int32_t C = (int32_t)kQC[j], Sn = (int32_t)kQS[j];
  int64_t u0 = INT64_MAX, u1 = INT64_MIN, v0 = INT64_MAX, v1 = INT64_MIN;
  for (int v = vg; v < nv; v += VG) {
    const int32_t x = fx ? w - X[v] : X[v], y = fy ? h - Y[v] : Y[v];
    // |x|, |y| <= 2^25, C, Sn <= 2^30: 32 x 32 -> 64-bit products
    const int64_t u = (int64_t)x * C + (int64_t)y * Sn, vv = (int64_t)y * C - (int64_t)x * Sn;
    u0 = u < u0 ? u : u0; u1 = u > u1 ? u : u1;
    v0 = vv < v0 ? vv : v0; v1 = vv > v1 ? vv : v1;
  }
#pragma unroll
  for (int o = 1; o < VG; o <<= 1) {
    int64_t t = g.xorv(u0, o); u0 = t < u0 ? t : u0;
    t = g.xorv(u1, o); u1 = t > u1 ? t : u1;
    t = g.xorv(v0, o); v0 = t < v0 ? t : v0;
    t = g.xorv(v1, o); v1 = t > v1 ? t : v1;
  }
  if (vg == 0) {
    S.ob[4 * j + 0] = u0; S.ob[4 * j + 1] = u1; S.ob[4 * j + 2] = v0; S.ob[4 * j + 3] = v1;
  }
  // arg-min over the angle lanes (lane j * VG), ties to the smaller j
  i128 area = (i128)(u1 - u0) * (i128)(v1 - v0);
  int bj = j;
  if (j >= nj) area = ~((i128)1 << 127);  // excluded angles: +infinity
#pragma unroll
  for (int o = VG; o < G; o <<= 1) {
    const uint64_t lo = g.xorv((uint64_t)area, o), hi = g.xorv((uint64_t)(area >> 64), o);
    const int oj = g.xorv(bj, o);
    const i128 oa = (i128)(((unsigned __int128)hi << 64) | lo);
    if (oa < area || (oa == area && oj < bj)) { area = oa; bj = oj; }
  }
  bj = __shfl_sync(g.mask, bj, 0, G);
  g.sync();  // S.ob complete before any reader
  return bj;
}

template <int G>
__global__ void __launch_bounds__(kBlock)
proxy_kernel(const float* __restrict__ xy, const int32_t* __restrict__ start, int32_t n, float rx,
             float ry, int k, uint32_t flags, int32_t* qx, int32_t* qy, int64_t max_v, Proxies P,
             Status* st, AtlasMap am, bool skip_wh) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int lane = threadIdx.x & 31, gib = threadIdx.x / G;
  Group<G> g;
  g.gl = lane % G;
  g.mask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane / G * G));
  const int c = am.c0 + blockIdx.x * (kBlock / G) + gib;
  if (c >= n) return;  // the whole group leaves together
  // batch mode (tabi_pack_many): chart c is global; its atlas a is the last
  // with abase[a] <= c (uniform per group), which owns the status block, the
  // resolution and the chart index reported on EINVAL
  int32_t cl = c;
  const int gl0 = g.gl;
  if (am.abase) {
    // G-ary search by the group (one probe per lane, a ballot per round: 2-3
    // dependent loads instead of log2(na)); invariant abase[lo] <= c, the
    // answer in [lo, hi]; the probes are monotone, so the ballot's popcount
    // locates the last true one
    int lo = 0, hi = am.na - 1;
    while (lo < hi) {  // (uniform over the group)
      const int step = (hi - lo + G) / G;
      const int idx = lo + gl0 * step;
      const bool p = idx <= hi && am.abase[idx] <= c;
      const int j = __popc(__ballot_sync(g.mask, p)) - 1;
      lo += j * step;
      hi = min(hi, lo + step - 1);
    }
    st += lo;
    cl = c - am.abase[lo];
    if (am.res) { rx = am.res[2 * lo]; ry = am.res[2 * lo + 1]; }
  }
  Slices S;
  {
    unsigned char* p = dsm + slice_bytes(k) * gib;
    S.ob = (int64_t*)p;  // 256 B, 8-byte aligned at the group's slot
    int32_t* i32 = (int32_t*)(p + 256);
    S.mlo0 = i32; S.mlo1 = i32 + k; S.mhi0 = i32 + 2 * k; S.mhi1 = i32 + 3 * k;
    S.vx = i32 + 4 * k;
    S.vy = S.vx + kVCap;
  }
  const int gl = g.gl;
  const int32_t a0 = start[c];
  const int nv = start[c + 1] - a0;
  // device-pointer inputs are not checked on the host: a vertex range outside
  // the context's snapped-coordinate scratch is a capacity error (bit 2),
  // raised before any write (tabi.h: TABI_ECAPACITY beyond max_vertices)
  if (a0 < 0 || (int64_t)a0 + (nv > 0 ? nv : 0) > max_v) {
    if (gl == 0) atomicOr(&st->capacity, 4);
    return;
  }
  if (nv < 3) {
    if (gl == 0) atomicMin(&st->bad_chart, cl);
    return;
  }
  // the chart's vertices: shared memory when they fit, else the HBM scratch
  const bool in_smem = nv <= kVCap;
  int32_t* X = in_smem ? S.vx : qx + a0;
  int32_t* Y = in_smem ? S.vy : qy + a0;
  // A1 snap: q = round_half_even(x * res * 256), exact product in double (D2)
  bool ok = true;
  int32_t xmn = INT32_MAX, xmx = INT32_MIN, ymn = INT32_MAX, ymx = INT32_MIN;
  // (one 8-byte load per vertex when the caller's buffer allows it)
  const bool al8 = ((uintptr_t)xy & 7u) == 0;
  const float2* xy2 = reinterpret_cast<const float2*>(xy) + a0;
  for (int v = gl; v < nv; v += G) {
    const float2 p = al8 ? xy2[v] : make_float2(xy[2 * ((int64_t)a0 + v)], xy[2 * ((int64_t)a0 + v) + 1]);
    double fx = (double)p.x * (double)rx * 256.0;
    double fy = (double)p.y * (double)ry * 256.0;
    if (!isfinite(fx) || !isfinite(fy) || fabs(fx) > (double)TABI_QMAX ||
        fabs(fy) > (double)TABI_QMAX) {
      ok = false;
      continue;
    }
    int32_t ix = (int32_t)__double2ll_rn(fx), iy = (int32_t)__double2ll_rn(fy);
    X[v] = ix;
    Y[v] = iy;
    xmn = min(xmn, ix); xmx = max(xmx, ix);
    ymn = min(ymn, iy); ymx = max(ymx, iy);
  }
  if (__ballot_sync(g.mask, !ok) != 0u) {
    if (gl == 0) atomicMin(&st->bad_chart, cl);
    return;
  }
  int prerot = 0;
  if (flags & TABI_F_PREROTATE) {
    // R4 pre-rotation (TABI_F_PREROTATE): the D6 minimum-area angle
    // of the snapped polygon, then every vertex moves to that OBB frame,
    // rounded half to even to 1/256 texel (tabi_placement step 0).
    g.sync();
    prerot = obb_angle(g, X, Y, nv, S);
    if (prerot) {
      const int64_t C = kQC[prerot], Sn = kQS[prerot];
      xmn = INT32_MAX; xmx = INT32_MIN; ymn = INT32_MAX; ymx = INT32_MIN;
      for (int v = gl; v < nv; v += G) {
        const int64_t x = X[v], y = Y[v];
        const int32_t u = (int32_t)q30_round(x * C + y * Sn);
        const int32_t t = (int32_t)q30_round(-x * Sn + y * C);
        X[v] = u;
        Y[v] = t;
        xmn = min(xmn, u); xmx = max(xmx, u);
        ymn = min(ymn, t); ymx = max(ymx, t);
      }
    }
  }
  xmn = g.min32(xmn); xmx = g.max32(xmx);
  ymn = g.min32(ymn); ymx = g.max32(ymx);
  int64_t w = (int64_t)xmx - xmn, h = (int64_t)ymx - ymn;
  // D3 90-degree normalization, (x, y) -> (h - y, x) iff w > h, folded into
  // the translation of the AABB to the origin (one pass; each lane rewrites
  // only its own vertices)
  const bool rot = w > h;
  for (int v = gl; v < nv; v += G) {
    const int32_t x = X[v] - xmn, y = Y[v] - ymn;
    X[v] = rot ? (int32_t)(h - y) : x;
    Y[v] = rot ? x : y;
  }
  if (rot) { const int64_t t = w; w = h; h = t; }
  g.sync();
  // D3 shoelace (2 x area), exact: |x|, |y| <= 2^25, so each term fits int64
  // and the sum (|2A| <= 2^51) is exact modulo 2^64; a rotation keeps |area|
  int64_t s2 = 0;
  for (int v = gl; v < nv; v += G) {
    const int u = (v + 1 == nv) ? 0 : v + 1;
    s2 += (int64_t)X[v] * Y[u] - (int64_t)X[u] * Y[v];
  }
  s2 = g.sum64_wrap(s2);
  if (s2 < 0) s2 = -s2;
  if (s2 == 0) {
    if (gl == 0) atomicMin(&st->bad_chart, cl);
    return;
  }
  // D4/D5 in the normalized pose, D7 orientation
  merged_slices(g, S, X, Y, nv, w, h, k);
  // empty-area sums: every term is in [0, 2^25] and k <= 64, so the sums fit
  // 32 unsigned bits
  uint32_t top = 0, bot = 0, left = 0, right = 0;
  for (int j = gl; j < k; j += G) {
    top += (uint32_t)S.mlo0[j];
    bot += (uint32_t)(h - S.mhi0[j]);
    left += (uint32_t)S.mlo1[j];
    right += (uint32_t)(w - S.mhi1[j]);
  }
  const int64_t TOP = g.sumu(top), BOT = g.sumu(bot);
  const int64_t LEFT = g.sumu(left), RIGHT = g.sumu(right);
  const bool fy = TOP > BOT;
  const int64_t D = LEFT - RIGHT;  // |10 D| < 2^35, k w <= 2^31: int64
  bool fx;
  if (10 * D > (int64_t)k * w) {
    fx = true;
  } else if (10 * (-D) > (int64_t)k * w) {
    fx = false;
  } else {
    // bottom-left vs bottom-right (D7): BL2 = 2 S_L + mid, BR2 = 2 S_R + mid
    // with the odd-k middle slice split 50/50, so BL2 > BR2 iff S_L > S_R
    // (each a sum of < 32 gaps <= 2^25: 32 bits)
    uint32_t sl = 0, sr = 0;
    for (int j = gl; j < k; j += G) {
      const uint32_t gap = (uint32_t)(fy ? S.mlo0[j] : (h - S.mhi0[j]));
      if (2 * j + 1 < k) sl += gap;
      else if (2 * j + 1 > k) sr += gap;
    }
    fx = g.sumu(sl) > g.sumu(sr);
  }
  // D8 final pose.  The slices of the reflected chart are the reflected
  // slices: x -> w - x maps x-strip j to strip k-1-j (closed strips, the same
  // crossings) and a floored left bound to w - (ceiled right bound); the merge
  // commutes with both maps.  So the final-pose merged slices are an index
  // mirror plus a value reflection of the ones just computed -- no second
  // slicing pass (tests compare every slice with the oracle, which re-slices).
  // The vertices are reflected on the fly by the OBB pass below.
  if (fx || fy) {
    constexpr int U = TABI_KMAX / G;  // slices per lane (k <= 64)
    int32_t t0[U], b0[U], l1[U], r1[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int j = gl + G * u;
      if (j >= k) continue;
      const int sx = fx ? k - 1 - j : j;  // x-slices are indexed along x
      const int sy = fy ? k - 1 - j : j;  // y-slices along y
      t0[u] = fy ? (int32_t)(h - S.mhi0[sx]) : S.mlo0[sx];
      b0[u] = fy ? (int32_t)(h - S.mlo0[sx]) : S.mhi0[sx];
      l1[u] = fx ? (int32_t)(w - S.mhi1[sy]) : S.mlo1[sy];
      r1[u] = fx ? (int32_t)(w - S.mlo1[sy]) : S.mhi1[sy];
    }
    g.sync();
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int j = gl + G * u;
      if (j >= k) continue;
      S.mlo0[j] = t0[u]; S.mhi0[j] = b0[u];
      S.mlo1[j] = l1[u]; S.mhi1[j] = r1[u];
    }
    g.sync();
  }
  int32_t* sl = P.sl + (int64_t)c * 4 * k;
  for (int j = gl; j < k; j += G) {
    sl[j] = S.mlo0[j];
    sl[k + j] = S.mhi0[j];
    sl[2 * k + j] = S.mlo1[j];
    sl[3 * k + j] = S.mhi1[j];
  }
  // D6 OBB of the final pose: minimum (Umax-Umin)(Vmax-Vmin) over 8 angles,
  // ties -> smaller j
  const int bj = obb_angle(g, X, Y, nv, S, (flags & TABI_F_NO_OBB) ? 1 : 8, fx, fy, (int32_t)w,
                           (int32_t)h);
  if (gl == 0) {
    if (!skip_wh) {  // (else written by sizes_kernel, which the order is waiting on)
      P.w[c] = (int32_t)w;
      P.h[c] = (int32_t)h;
      P.area2[c] = s2;
    }
    P.xmin[c] = xmn;
    P.ymin[c] = ymn;
    P.pose[c] = (uint8_t)((rot ? 1 : 0) | (fx ? 2 : 0) | (fy ? 4 : 0));
    P.prerot[c] = (uint8_t)prerot;
    P.obb_j[c] = bj;
    P.obb[4 * (int64_t)c + 0] = S.ob[4 * bj + 0];
    P.obb[4 * (int64_t)c + 1] = S.ob[4 * bj + 1];
    P.obb[4 * (int64_t)c + 2] = S.ob[4 * bj + 2];
    P.obb[4 * (int64_t)c + 3] = S.ob[4 * bj + 3];
  }
}

// The order's inputs alone (A1-A3's AABB, 90-degree normalization and area,
// no prerotation): the snapped extents w, h (swapped when w > h, D3) and the
// doubled area |shoelace| of the snapped polygon -- translation- and
// rotation-invariant, so the normalized polygon's exactly -- with the same
// capacity / bad-chart decisions as proxy_kernel.  One 8-lane group per chart;
// nothing is written but w, h, area2 and the status words.  Lets the sort
// start while proxy_kernel computes the slices and OBBs on a second stream.
__global__ void __launch_bounds__(kBlock)
sizes_kernel(const float* __restrict__ xy, const int32_t* __restrict__ start, int32_t n, float rx,
             float ry, int64_t max_v, Proxies P, Status* st) {
  constexpr int G = 8;
  const int lane = threadIdx.x & 31, gl = lane % G;
  const unsigned mask = ((1u << G) - 1u) << (lane / G * G);
  const int c = blockIdx.x * (kBlock / G) + threadIdx.x / G;
  if (c >= n) return;  // (the whole group)
  const int32_t a0 = start[c];
  const int nv = start[c + 1] - a0;
  if (a0 < 0 || (int64_t)a0 + (nv > 0 ? nv : 0) > max_v) {
    if (gl == 0) atomicOr(&st->capacity, 4);
    return;
  }
  if (nv < 3) {
    if (gl == 0) atomicMin(&st->bad_chart, c);
    return;
  }
  auto snap = [&](int v, int32_t& ix, int32_t& iy) -> bool {
    const double fx = (double)xy[2 * ((int64_t)a0 + v)] * (double)rx * 256.0;
    const double fy = (double)xy[2 * ((int64_t)a0 + v) + 1] * (double)ry * 256.0;
    if (!isfinite(fx) || !isfinite(fy) || fabs(fx) > (double)TABI_QMAX || fabs(fy) > (double)TABI_QMAX)
      return false;
    ix = (int32_t)__double2ll_rn(fx);
    iy = (int32_t)__double2ll_rn(fy);
    return true;
  };
  bool ok = true;
  int32_t xmn = INT32_MAX, xmx = INT32_MIN, ymn = INT32_MAX, ymx = INT32_MIN;
  int64_t s2 = 0;
  for (int v = gl; v < nv; v += G) {
    int32_t x, y, xu, yu;
    const bool okv = snap(v, x, y), oku = snap(v + 1 == nv ? 0 : v + 1, xu, yu);
    if (!okv || !oku) { ok = false; continue; }
    xmn = min(xmn, x); xmx = max(xmx, x);
    ymn = min(ymn, y); ymx = max(ymx, y);
    s2 += (int64_t)x * yu - (int64_t)xu * y;  // (exact modulo 2^64; |2A| < 2^51)
  }
  if (__ballot_sync(mask, !ok) != 0u) {
    if (gl == 0) atomicMin(&st->bad_chart, c);
    return;
  }
  xmn = __reduce_min_sync(mask, xmn); xmx = __reduce_max_sync(mask, xmx);
  ymn = __reduce_min_sync(mask, ymn); ymx = __reduce_max_sync(mask, ymx);
  const uint64_t u = (uint64_t)s2;
  const uint64_t c0 = __reduce_add_sync(mask, (uint32_t)(u & 0xffffu));
  const uint64_t c1 = __reduce_add_sync(mask, (uint32_t)((u >> 16) & 0xffffu));
  const uint64_t c2 = __reduce_add_sync(mask, (uint32_t)((u >> 32) & 0xffffu));
  const uint64_t c3 = __reduce_add_sync(mask, (uint32_t)(u >> 48));
  int64_t a2 = (int64_t)(c0 + (c1 << 16) + (c2 << 32) + (c3 << 48));
  if (a2 < 0) a2 = -a2;
  if (gl != 0) return;
  if (a2 == 0) {
    atomicMin(&st->bad_chart, c);
    return;
  }
  int64_t w = (int64_t)xmx - xmn, h = (int64_t)ymx - ymn;
  if (w > h) { const int64_t t = w; w = h; h = t; }
  P.w[c] = (int32_t)w;
  P.h[c] = (int32_t)h;
  P.area2[c] = a2;
}

template <int G>
void launch_g(const float* xy, const int32_t* start, int32_t n, float rx, float ry, int k,
              uint32_t flags, int32_t* qx, int32_t* qy, int64_t max_v, Proxies P, Status* st,
              AtlasMap am, cudaStream_t s, bool skip_wh) {
  constexpr int per_block = kBlock / G;
  const int blocks = (n - am.c0 + per_block - 1) / per_block;
  if (blocks < 1) return;
  const size_t smem = slice_bytes(k) * per_block;
  static std::atomic<unsigned long long> attr{0};  // k = 64 with 8-lane groups: 32 charts x 4.4 KB per block
  ensure_dyn_smem((const void*)proxy_kernel<G>, (int)(slice_bytes(TABI_KMAX) * per_block), attr);
  proxy_kernel<G><<<blocks, kBlock, smem, s>>>(xy, start, n, rx, ry, k, flags, qx, qy, max_v, P,
                                                st, am, skip_wh);
}

}  // namespace

void launch_sizes(const float* xy, const int32_t* start, int32_t n, float rx, float ry,
                  int64_t max_v, Proxies P, Status* st, cudaStream_t s) {
  constexpr int per_block = kBlock / 8;
  const int blocks = (n + per_block - 1) / per_block;
  if (blocks < 1) return;
  sizes_kernel<<<blocks, kBlock, 0, s>>>(xy, start, n, rx, ry, max_v, P, st);
}

void launch_proxies(const float* xy, const int32_t* start, int32_t n, float rx, float ry, int k,
                    uint32_t flags, int32_t* qx, int32_t* qy, int64_t max_v, Proxies P, Status* st,
                    cudaStream_t s, AtlasMap am, int64_t nverts, bool skip_wh) {
  const char* genv = getenv("TABI_PROXY_LANES");  // test knob: force 8 / 16 / 32
  const int forced = genv ? atoi(genv) : 0;
  // Lanes per chart.  Below 4096 charts a pack is latency-bound per chart: 32.
  // Above, the lanes of a warp's groups diverge whenever their charts' vertex
  // counts differ, so narrow groups pay off only for charts of a few vertices:
  // measured C4 (20,000 lightmap quads, 4.4 vertices per chart) best at 8, the
  // C5 batch (547 k TSS charts, 9.6 vertices) at 32 (2.9 ms vs 3.9 at 16, 4.8 at 8).
  const int64_t avg = nverts > 0 ? (nverts + n - 1) / n : 0;
  const int G = forced == 8 || forced == 16 || forced == 32 ? forced
                : n < 4096 ? 32 : avg >= 8 ? 32 : avg >= 6 ? 16 : n < 8192 ? 16 : 8;
  if (G == 32) launch_g<32>(xy, start, n, rx, ry, k, flags, qx, qy, max_v, P, st, am, s, skip_wh);
  else if (G == 16) launch_g<16>(xy, start, n, rx, ry, k, flags, qx, qy, max_v, P, st, am, s, skip_wh);
  else launch_g<8>(xy, start, n, rx, ry, k, flags, qx, qy, max_v, P, st, am, s, skip_wh);
}

}  // namespace tabi
