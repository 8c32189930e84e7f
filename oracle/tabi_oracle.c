/* oracle/tabi_oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain, slow, obviously-correct CPU oracle of TABI (arxiv 2602.07782).
 * "P:n" = /root/reference/PAPER.md line n; "Dn" = SURVEY.md §8(c) reading n;
 * "S:n" = SPEC.md line n (interfaces / hand examples only).
 *
 * Structure follows the paper's own order ("Algorithm Summary"):
 *   snap -> AABB + 90deg normalization -> local AABBs + merge -> orientation
 *   -> final pose -> OBB -> height sort -> for every candidate scale:
 *   profiles -> compacting offsets -> Alg. 4 row loop (Alg. 2, 3, 1) ->
 *   pick the largest successful scale.
 * No blocking, fusion or reordering: every candidate, every configuration
 * (all 4 or 8 of P:301) and every frontline copy (Alg. 4 line "Copy frontLine
 * to localFrontLine[j]") is evaluated literally.
 * Pins (tests/test_oracle_*.py, -m "not gpu"): SPEC / paper worked examples,
 * hand-derived goldens for every tightening step, closed forms (single chart,
 * equal-square prefix tails, exact-tail squares), brute-force optimal
 * packings, exact-rational clipping, invariants; no function is left
 * "parity unpinned".
 */
#include "oracle.h"

#include <limits.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

/* ---- exact integer helpers (b > 0) ------------------------------------- */
static int64_t fdiv64(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b) != 0 && a < 0) q--;
  return q;
}
static int64_t cdiv64(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b) != 0 && a > 0) q++;
  return q;
}
static i128 fdiv128(i128 a, i128 b) {
  i128 q = a / b;
  if ((a % b) != 0 && a < 0) q--;
  return q;
}
static i128 cdiv128(i128 a, i128 b) {
  i128 q = a / b;
  if ((a % b) != 0 && a > 0) q++;
  return q;
}
static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

/* D6 / SURVEY Appendix B: theta_j = j*pi/16 ("8 evenly spaced rotations
 * in the interval [0, 7pi/16]"), cos/sin rounded to Q30.  Literal constants,
 * never libm, so every platform sees the same rotation. */
static const int64_t OR_QC[8] = {1073741824, 1053110176, 992008094, 892783698,
                                 759250125,  596538995,  410903207, 209476638};
static const int64_t OR_QS[8] = {0,         209476638, 410903207, 596538995,
                                 759250125, 892783698, 992008094, 1053110176};

/* ---- D2: snap a coordinate to 1/256 texel, round half to even ---------- */
static int snap(float v, float res, int64_t* q) {
  double x = (double)v * (double)res * 256.0; /* exact: 24b x 24b mantissas */
  if (!isfinite(x) || fabs(x) > (double)OR_QMAX) return 0;
  *q = (int64_t)llrint(x);
  return 1;
}

/* ---- D4: local AABB slices along x ("dividing the chart into
 * intervals of equal width ... local AABBs for the slice"; "each vertex
 * and each edge ... assigns itself to one or more intervals").  Strip j is
 * the closed range k*x in [j*w, (j+1)*w].  lo[j] = floor(min y), hi[j] =
 * ceil(max y) over vertices in the strip and edge crossings of the strip's
 * boundary lines.  Called with (Y, X, h) for the y-slices. */
static void slices(const int64_t* X, const int64_t* Y, int nv, int64_t w, int k,
                   int32_t* lo, int32_t* hi) {
  for (int j = 0; j < k; j++) {
    lo[j] = INT32_MAX;
    hi[j] = INT32_MIN;
  }
  for (int v = 0; v < nv; v++) {
    for (int j = 0; j < k; j++) {
      if ((int64_t)j * w <= k * X[v] && k * X[v] <= (int64_t)(j + 1) * w) {
        if (Y[v] < lo[j]) lo[j] = (int32_t)Y[v];
        if (Y[v] > hi[j]) hi[j] = (int32_t)Y[v];
      }
    }
  }
  for (int v = 0; v < nv; v++) {
    int a = v, b = (v + 1) % nv;
    if (X[a] == X[b]) continue;
    if (X[a] > X[b]) { int t = a; a = b; b = t; }
    for (int L = 1; L < k; L++) {
      int64_t line = (int64_t)L * w;
      if (k * X[a] < line && line < k * X[b]) {
        int64_t num = (line - k * X[a]) * (Y[b] - Y[a]);
        int64_t den = (int64_t)k * (X[b] - X[a]);
        int64_t yf = Y[a] + fdiv64(num, den);
        int64_t yc = Y[a] + cdiv64(num, den);
        for (int j = L - 1; j <= L; j++) {
          if (yf < lo[j]) lo[j] = (int32_t)yf;
          if (yc > hi[j]) hi[j] = (int32_t)yc;
        }
      }
    }
  }
}

/* ---- D5: merge ("taking the tighter bound along each axis").  Each
 * x-slice is tightened by the y-slices whose x-range meets it, and vice
 * versa, both from the UNMERGED slices. */
static void merge(int k, int64_t w, int64_t h, const int32_t* top, const int32_t* bot,
                  const int32_t* left, const int32_t* right, int32_t* top2, int32_t* bot2,
                  int32_t* left2, int32_t* right2) {
  for (int j = 0; j < k; j++) {
    int64_t mn = INT64_MAX, mx = INT64_MIN;
    for (int i = 0; i < k; i++) {
      if ((int64_t)k * left[i] <= (int64_t)(j + 1) * w && (int64_t)k * right[i] >= (int64_t)j * w) {
        mn = min64(mn, fdiv64((int64_t)i * h, k));
        mx = max64(mx, cdiv64((int64_t)(i + 1) * h, k));
      }
    }
    top2[j] = (int32_t)max64(top[j], mn == INT64_MAX ? top[j] : mn);
    bot2[j] = (int32_t)min64(bot[j], mx == INT64_MIN ? bot[j] : mx);
  }
  for (int i = 0; i < k; i++) {
    int64_t mn = INT64_MAX, mx = INT64_MIN;
    for (int j = 0; j < k; j++) {
      if ((int64_t)k * top[j] <= (int64_t)(i + 1) * h && (int64_t)k * bot[j] >= (int64_t)i * h) {
        mn = min64(mn, fdiv64((int64_t)j * w, k));
        mx = max64(mx, cdiv64((int64_t)(j + 1) * w, k));
      }
    }
    left2[i] = (int32_t)max64(left[i], mn == INT64_MAX ? left[i] : mn);
    right2[i] = (int32_t)min64(right[i], mx == INT64_MIN ? right[i] : mx);
  }
}

static void merged_slices(const int64_t* X, const int64_t* Y, int nv, int64_t w, int64_t h,
                          int k, int32_t* top2, int32_t* bot2, int32_t* left2,
                          int32_t* right2) {
  int32_t top[OR_KMAX], bot[OR_KMAX], left[OR_KMAX], right[OR_KMAX];
  slices(X, Y, nv, w, k, top, bot);
  slices(Y, X, nv, h, k, left, right);
  merge(k, w, h, top, bot, left, right, top2, bot2, left2, right2);
}

/* ---- D7: orientation ("Computing Chart Orientations"). -------- */
static void orientation(int k, int64_t w, int64_t h, const int32_t* top, const int32_t* bot,
                        const int32_t* left, const int32_t* right, int32_t* fx,
                        int32_t* fy) {
  int64_t TOP = 0, BOT = 0, LEFT = 0, RIGHT = 0;
  for (int j = 0; j < k; j++) { TOP += top[j]; BOT += h - bot[j]; }
  for (int i = 0; i < k; i++) { LEFT += left[i]; RIGHT += w - right[i]; }
  /* "If the top area is greater than the bottom area, we reflect the chart
   * vertically"; slice areas share the factor w/k. */
  *fy = TOP > BOT;
  /* "a difference greater than 10% of the chart's AABB area":
   * (LEFT-RIGHT)*h/k > w*h/10  <=>  10*(LEFT-RIGHT) > k*w. */
  int64_t D = LEFT - RIGHT;
  if ((i128)10 * D > (i128)k * w) {
    *fx = 1;
  } else if ((i128)10 * (-D) > (i128)k * w) {
    *fx = 0;
  } else {
    /* bottom-left vs bottom-right empty area, split at the midline; with the
     * vertical reflection applied the bottom gaps are the old top gaps. */
    int64_t BL2 = 0, BR2 = 0;
    for (int j = 0; j < k; j++) {
      int64_t gap = *fy ? top[j] : (h - bot[j]);
      if (2 * j + 1 < k) BL2 += 2 * gap;
      else if (2 * j + 1 > k) BR2 += 2 * gap;
      else { BL2 += gap; BR2 += gap; } /* odd k: middle slice split 50/50 */
    }
    *fx = BL2 > BR2;
  }
}

/* ---- D6: approximate OBB. -------------------------------- */
static void obb(const int64_t* X, const int64_t* Y, int nv, int nj, or_proxy* p) {
  i128 best = -1;
  for (int j = 0; j < nj; j++) { /* nj = 1 under OR_F_NO_OBB: the AABB (j = 0) */
    int64_t umin = INT64_MAX, umax = INT64_MIN, vmin = INT64_MAX, vmax = INT64_MIN;
    for (int v = 0; v < nv; v++) {
      int64_t u = X[v] * OR_QC[j] + Y[v] * OR_QS[j];
      int64_t vv = -X[v] * OR_QS[j] + Y[v] * OR_QC[j];
      umin = min64(umin, u); umax = max64(umax, u);
      vmin = min64(vmin, vv); vmax = max64(vmax, vv);
    }
    i128 area = (i128)(umax - umin) * (i128)(vmax - vmin);
    if (best < 0 || area < best) { /* ties keep the smaller angle */
      best = area;
      p->obb_j = j;
      p->umin = umin; p->umax = umax; p->vmin = vmin; p->vmax = vmax;
    }
  }
}

/* ---- R4: pre-rotation ("We pre-rotate the UV charts to align their
 * tight bounding boxes with the major axes prior to packing"
 * "rotated by the negative of its approximate-OBB angle").  The angle is the
 * D6 minimum-area angle of the snapped polygon; the rotated coordinates are
 * the Q30 frame (u, v) = (x C + y S, -x S + y C) divided by 2^30, rounded
 * half to even, so the pipeline continues on an integer polygon. ---------- */
static int64_t q30_round(int64_t a) { /* round_half_even(a / 2^30) */
  int64_t q = a >> 30;                 /* floor */
  int64_t r = a - (q << 30);           /* in [0, 2^30) */
  if (r > ((int64_t)1 << 29) || (r == ((int64_t)1 << 29) && (q & 1))) q++;
  return q;
}

static int prerotate_angle(const int64_t* X, const int64_t* Y, int nv) {
  i128 best = -1;
  int bj = 0;
  for (int j = 0; j < 8; j++) {
    int64_t umin = INT64_MAX, umax = INT64_MIN, vmin = INT64_MAX, vmax = INT64_MIN;
    for (int v = 0; v < nv; v++) {
      int64_t u = X[v] * OR_QC[j] + Y[v] * OR_QS[j];
      int64_t vv = -X[v] * OR_QS[j] + Y[v] * OR_QC[j];
      umin = min64(umin, u); umax = max64(umax, u);
      vmin = min64(vmin, vv); vmax = max64(vmax, vv);
    }
    i128 area = (i128)(umax - umin) * (i128)(vmax - vmin);
    if (best < 0 || area < best) { best = area; bj = j; }  /* ties: smaller angle */
  }
  return bj;
}

static void prerotate(int64_t* X, int64_t* Y, int nv, int j) {
  for (int v = 0; v < nv; v++) {
    int64_t u = X[v] * OR_QC[j] + Y[v] * OR_QS[j];
    int64_t vv = -X[v] * OR_QS[j] + Y[v] * OR_QC[j];
    X[v] = q30_round(u);
    Y[v] = q30_round(vv);
  }
}

/* ---- A1-A5: one chart's proxy ------------------------------------------ */
static int chart_proxy(const float* xy, int nv, float rx, float ry, int k, uint32_t flags,
                       or_proxy* p) {
  const int prerot_on = (flags & OR_F_PREROTATE) != 0;
  memset(p, 0, sizeof(*p));
  if (nv < 3) return 0;
  int64_t* X = malloc(sizeof(int64_t) * nv);
  int64_t* Y = malloc(sizeof(int64_t) * nv);
  int ok = 1;
  for (int v = 0; v < nv && ok; v++) ok = snap(xy[2 * v], rx, &X[v]) && snap(xy[2 * v + 1], ry, &Y[v]);
  if (!ok) { free(X); free(Y); return 0; }
  if (prerot_on) {
    p->prerot = prerotate_angle(X, Y, nv);
    if (p->prerot) prerotate(X, Y, nv, p->prerot);
  }
  /* D3: AABB, translate to the origin ("compute the AABBs"). */
  int64_t xmin = X[0], xmax = X[0], ymin = Y[0], ymax = Y[0];
  for (int v = 1; v < nv; v++) {
    xmin = min64(xmin, X[v]); xmax = max64(xmax, X[v]);
    ymin = min64(ymin, Y[v]); ymax = max64(ymax, Y[v]);
  }
  for (int v = 0; v < nv; v++) { X[v] -= xmin; Y[v] -= ymin; }
  int64_t w = xmax - xmin, h = ymax - ymin;
  i128 s = 0;
  for (int v = 0; v < nv; v++) {
    int b = (v + 1) % nv;
    s += (i128)X[v] * Y[b] - (i128)X[b] * Y[v];
  }
  if (s < 0) s = -s;
  if (s == 0) { free(X); free(Y); return 0; }
  p->area2 = (int64_t)s;
  p->xmin = (int32_t)xmin;
  p->ymin = (int32_t)ymin;
  /* D3: "rotated by 90 degrees if necessary so that they are taller than they
   * are wide"; a square is not rotated.  (x,y) -> (h-y, x). */
  if (w > h) {
    for (int v = 0; v < nv; v++) {
      int64_t nx = h - Y[v], ny = X[v];
      X[v] = nx; Y[v] = ny;
    }
    int64_t t = w; w = h; h = t;
    p->rot90 = 1;
  }
  p->w = (int32_t)w;
  p->h = (int32_t)h;
  p->k = k;
  /* D4/D5 in the normalized pose, D7 orientation. */
  int32_t top[OR_KMAX], bot[OR_KMAX], left[OR_KMAX], right[OR_KMAX];
  merged_slices(X, Y, nv, w, h, k, top, bot, left, right);
  orientation(k, w, h, top, bot, left, right, &p->fx, &p->fy);
  /* D8: apply the reflections to the geometry, recompute every proxy in the
   * final pose ("stored proxies describe the chart in its final pose"). */
  for (int v = 0; v < nv; v++) {
    if (p->fx) X[v] = w - X[v];
    if (p->fy) Y[v] = h - Y[v];
  }
  merged_slices(X, Y, nv, w, h, k, p->top, p->bot, p->left, p->right);
  obb(X, Y, nv, (flags & OR_F_NO_OBB) ? 1 : 8, p);
  free(X);
  free(Y);
  return 1;
}

int or_build_proxies(const float* xy, const int32_t* start, int32_t n, float res_x,
                     float res_y, int32_t k, uint32_t flags, or_proxy* out, int32_t* bad_chart) {
  *bad_chart = -1;
  if (n < 1 || k < 1 || k > OR_KMAX) return OR_EINVAL;
  for (int32_t c = 0; c < n; c++) {
    int nv = start[c + 1] - start[c];
    if (!chart_proxy(xy + 2 * (int64_t)start[c], nv, res_x, res_y, k, flags, &out[c])) {
      *bad_chart = c;
      return OR_EINVAL;
    }
  }
  return OR_OK;
}

/* ---- D9: decreasing-height order ("sorted in decreasing height
 * order"), ties by wider first then chart index (stable). */
static const or_proxy* g_sort_px;
static int cmp_order(const void* A, const void* B) {
  int32_t a = *(const int32_t*)A, b = *(const int32_t*)B;
  const or_proxy *pa = &g_sort_px[a], *pb = &g_sort_px[b];
  if (pa->h != pb->h) return pa->h > pb->h ? -1 : 1;
  if (pa->w != pb->w) return pa->w > pb->w ? -1 : 1;
  return a < b ? -1 : (a > b);
}
void or_sort(const or_proxy* p, int32_t n, int32_t* perm) {
  for (int32_t i = 0; i < n; i++) perm[i] = i;
  g_sort_px = p;
  qsort(perm, n, sizeof(int32_t), cmp_order);
}

/* ---- D11: OBB bound on one column / row ------------------------------------
 * The chart lies in {Umin <= x*C + y*S <= Umax, Vmin <= -x*S + y*C <= Vmax}.
 * For x in the column's unscaled strip [P0/num, P1/num] the top boundary is
 * y_top(x) = max((Umin - x*C)/S, (Vmin + x*S)/C) (convex); its minimum over
 * the strip is at x* = (C*Umin - S*Vmin)/(C^2+S^2) if inside, else at the
 * nearer endpoint.  Value scaled by num/SC and floored ("rounded up" toward
 * the atlas top; D11). */
static int64_t obb_top(const or_proxy* p, i128 num, i128 SC, i128 P0, i128 P1) {
  i128 C = OR_QC[p->obb_j], S = OR_QS[p->obb_j], N2 = C * C + S * S;
  i128 xs = num * (C * p->umin - S * p->vmin);
  if (P0 * N2 <= xs && xs <= P1 * N2) return (int64_t)fdiv128(num * (S * p->umin + C * p->vmin), N2 * SC);
  i128 P = xs < P0 * N2 ? P0 : P1;
  i128 y1 = fdiv128(p->umin * num - P * C, S * SC);
  i128 y2 = fdiv128(p->vmin * num + P * S, C * SC);
  return (int64_t)(y1 > y2 ? y1 : y2);
}
/* bottom: y_bot(x) = min((Umax - x*C)/S, (Vmax + x*S)/C), concave, ceil'd. */
static int64_t obb_bot(const or_proxy* p, i128 num, i128 SC, i128 P0, i128 P1) {
  i128 C = OR_QC[p->obb_j], S = OR_QS[p->obb_j], N2 = C * C + S * S;
  i128 xs = num * (C * p->umax - S * p->vmax);
  if (P0 * N2 <= xs && xs <= P1 * N2) return (int64_t)cdiv128(num * (S * p->umax + C * p->vmax), N2 * SC);
  i128 P = xs < P0 * N2 ? P0 : P1;
  i128 y1 = cdiv128(p->umax * num - P * C, S * SC);
  i128 y2 = cdiv128(p->vmax * num + P * S, C * SC);
  return (int64_t)(y1 < y2 ? y1 : y2);
}
/* left: x_left(y) = max((Umin - y*S)/C, (y*C - Vmax)/S), convex, floored. */
static int64_t obb_left(const or_proxy* p, i128 num, i128 SC, i128 Q0, i128 Q1) {
  i128 C = OR_QC[p->obb_j], S = OR_QS[p->obb_j], N2 = C * C + S * S;
  i128 ys = num * (S * p->umin + C * p->vmax);
  if (Q0 * N2 <= ys && ys <= Q1 * N2) return (int64_t)fdiv128(num * (C * p->umin - S * p->vmax), N2 * SC);
  i128 Q = ys < Q0 * N2 ? Q0 : Q1;
  i128 x1 = fdiv128(p->umin * num - Q * S, C * SC);
  i128 x2 = fdiv128(Q * C - p->vmax * num, S * SC);
  return (int64_t)(x1 > x2 ? x1 : x2);
}
/* right: x_right(y) = min((Umax - y*S)/C, (y*C - Vmin)/S), concave, ceil'd. */
static int64_t obb_right(const or_proxy* p, i128 num, i128 SC, i128 Q0, i128 Q1) {
  i128 C = OR_QC[p->obb_j], S = OR_QS[p->obb_j], N2 = C * C + S * S;
  i128 ys = num * (S * p->umax + C * p->vmin);
  if (Q0 * N2 <= ys && ys <= Q1 * N2) return (int64_t)cdiv128(num * (C * p->umax - S * p->vmin), N2 * SC);
  i128 Q = ys < Q0 * N2 ? Q0 : Q1;
  i128 x1 = cdiv128(p->umax * num - Q * S, C * SC);
  i128 x2 = cdiv128(Q * C - p->vmin * num, S * SC);
  return (int64_t)(x1 < x2 ? x1 : x2);
}

/* ---- D11 + D13: TopEdge/BottomEdge per texel column and the
 * symmetric per-row left/right edges, at scale num/den, then the gutter as a
 * Chebyshev dilation by g in a grid shifted by g. */
int or_profile(const or_proxy* p, int64_t num, int64_t den, int32_t g, or_prof* out) {
  const int64_t SC = den * 256, k = p->k, w = p->w, h = p->h;
  int64_t ws = cdiv64(w * num, SC), hs = cdiv64(h * num, SC);
  int64_t* T = malloc(sizeof(int64_t) * ws);
  int64_t* B = malloc(sizeof(int64_t) * ws);
  int64_t* Lf = malloc(sizeof(int64_t) * hs);
  int64_t* R = malloc(sizeof(int64_t) * hs);
  for (int64_t i = 0; i < ws; i++) {
    /* local-AABB bound: slices whose scaled x-range openly overlaps [i, i+1] */
    int64_t mt = INT64_MAX, mb = INT64_MIN;
    for (int64_t j = 0; j < k; j++) {
      if (num * j * w < (i + 1) * SC * k && num * (j + 1) * w > i * SC * k) {
        mt = min64(mt, p->top[j]);
        mb = max64(mb, p->bot[j]);
      }
    }
    if (mt == INT64_MAX) { free(T); free(B); free(Lf); free(R); return 0; }
    int64_t t = max64(0, fdiv64(num * mt, SC));
    int64_t b = min64(hs, cdiv64(num * mb, SC));
    if (p->obb_j != 0) { /* OBB bound; j = 0 is the AABB itself */
      i128 P0 = (i128)i * SC, P1 = min64((i + 1) * SC, w * num);
      t = max64(t, obb_top(p, num, SC, P0, P1));
      b = min64(b, obb_bot(p, num, SC, P0, P1));
    }
    T[i] = t;
    B[i] = b;
  }
  for (int64_t r = 0; r < hs; r++) {
    int64_t ml = INT64_MAX, mr = INT64_MIN;
    for (int64_t i = 0; i < k; i++) {
      if (num * i * h < (r + 1) * SC * k && num * (i + 1) * h > r * SC * k) {
        ml = min64(ml, p->left[i]);
        mr = max64(mr, p->right[i]);
      }
    }
    if (ml == INT64_MAX) { free(T); free(B); free(Lf); free(R); return 0; }
    int64_t l = max64(0, fdiv64(num * ml, SC));
    int64_t rr = min64(ws, cdiv64(num * mr, SC));
    if (p->obb_j != 0) {
      i128 Q0 = (i128)r * SC, Q1 = min64((r + 1) * SC, h * num);
      l = max64(l, obb_left(p, num, SC, Q0, Q1));
      rr = min64(rr, obb_right(p, num, SC, Q0, Q1));
    }
    Lf[r] = l;
    R[r] = rr;
  }
  /* D13: Dtop(i) = min Top over [i-2g, i], Dbot(i) = max Bot + 2g, etc. */
  out->ws = (int32_t)ws;
  out->hs = (int32_t)hs;
  out->Wd = (int32_t)(ws + 2 * g);
  out->Hd = (int32_t)(hs + 2 * g);
  out->Dtop = malloc(sizeof(int32_t) * out->Wd);
  out->Dbot = malloc(sizeof(int32_t) * out->Wd);
  out->Dleft = malloc(sizeof(int32_t) * out->Hd);
  out->Dright = malloc(sizeof(int32_t) * out->Hd);
  for (int64_t i = 0; i < out->Wd; i++) {
    int64_t lo = max64(0, i - 2 * g), hi = min64(i, ws - 1);
    int64_t mn = INT64_MAX, mx = INT64_MIN;
    for (int64_t q = lo; q <= hi; q++) { mn = min64(mn, T[q]); mx = max64(mx, B[q]); }
    out->Dtop[i] = (int32_t)mn;
    out->Dbot[i] = (int32_t)(mx + 2 * g);
  }
  for (int64_t r = 0; r < out->Hd; r++) {
    int64_t lo = max64(0, r - 2 * g), hi = min64(r, hs - 1);
    int64_t mn = INT64_MAX, mx = INT64_MIN;
    for (int64_t q = lo; q <= hi; q++) { mn = min64(mn, Lf[q]); mx = max64(mx, R[q]); }
    out->Dleft[r] = (int32_t)mn;
    out->Dright[r] = (int32_t)(mx + 2 * g);
  }
  free(T); free(B); free(Lf); free(R);
  return 1;
}

void or_prof_free(or_prof* pr) {
  free(pr->Dtop); free(pr->Dbot); free(pr->Dleft); free(pr->Dright);
  pr->Dtop = pr->Dbot = pr->Dleft = pr->Dright = NULL;
}

/* ---- D14: horizontal compacting: with both charts top-aligned,
 * the smallest x advance from a to b such that no shared row overlaps,
 * i.e. the max over shared rows of the gap between a's right and b's left
 * boundary ("take the minimum distance between the piecewise constant
 * values", in advance form).  Compacting distance = Wd_a - result. */
int32_t or_offset(const or_prof* a, const or_prof* b) {
  int32_t off = 0;
  int32_t rows = a->Hd < b->Hd ? a->Hd : b->Hd;
  for (int32_t j = 0; j < rows; j++) {
    int32_t d = a->Dright[j] - b->Dleft[j];
    if (d > off) off = d;
  }
  return off;
}

/* ---- D15: CannotMoveAbove for a (left) and b (right) at relative advance
 * delta ("a chart can move up without potential intersection if no
 * rectangular segment formed by its piecewise constant boundary is below a
 * segment of the other chart's boundary").  Moving a up by t puts a's row r
 * beside b's row r - t < r; a is locked iff some such pair may overlap. */
void or_locks(const or_prof* a, const or_prof* b, int32_t delta, int32_t* a_locked,
              int32_t* b_locked) {
  *a_locked = 0;
  *b_locked = 0;
  for (int32_t r = 1; r < a->Hd && !*a_locked; r++) {
    int32_t lim = r < b->Hd ? r : b->Hd;
    for (int32_t rho = 0; rho < lim; rho++)
      if (a->Dright[r] > delta + b->Dleft[rho]) { *a_locked = 1; break; }
  }
  for (int32_t r = 1; r < b->Hd && !*b_locked; r++) {
    int32_t lim = r < a->Hd ? r : a->Hd;
    for (int32_t rho = 0; rho < lim; rho++)
      if (delta + b->Dleft[r] < a->Dright[rho]) { *b_locked = 1; break; }
  }
}

/* ---- Alg. 3 FoldRow: returns the last chart index in the row
 * (row_start - 1 if even the first chart does not fit); x_out[c] = offset. */
int32_t or_fold_row(int32_t n, int32_t row_start, int32_t fold_w, int32_t hc,
                    const int32_t* wd, const int32_t* off, int32_t* x_out) {
  int32_t c = row_start;
  int64_t curr = 0;
  while (c < n) {
    int64_t next = curr + wd[c];
    if (next > fold_w) return c - 1;
    x_out[c] = (int32_t)curr;
    if (hc) curr = curr + off[c]; /* nextLeftEdge - compactingDistance[c+1] */
    else curr = next;
    c++;
  }
  return n - 1;
}

/* ---- Alg. 1 CorrectYOffsets, over the D15 pair list. ------- */
void or_correct_y(int32_t npairs, const int32_t* pa, const int32_t* pb, const int32_t* lock_ab,
                  const int32_t* lock_ba, int32_t* y) {
  int violation;
  do {
    violation = 0;
    for (int32_t q = 0; q < npairs; q++) {
      int32_t a = pa[q], b = pb[q];
      if (lock_ab[q] && y[a] < y[b]) { violation = 1; y[a] = y[b]; }
      if (lock_ba[q] && y[b] < y[a]) { violation = 1; y[b] = y[a]; }
    }
  } while (violation);
}

/* ---- Alg. 2 UpdateKneeLocation + D20 discard rules.
 * Returns 0 if the knee is discarded. */
int or_update_knee(const int32_t* F, int32_t Wp, int32_t ltr, int32_t* left, int32_t* right) {
  if (ltr) {
    if (*right >= Wp) return 0;
    int32_t curr = F[*right];
    int32_t nk = *left - 1;
    for (int32_t x = *left; x < *right; x++)
      if (F[x] >= curr && x > nk) nk = x;
    if (nk + 1 == *left) return 0;
    *right = nk + 1;
    return 1;
  }
  if (*left <= 0) return 0;
  int32_t curr = F[*left - 1];
  int32_t nk = *right;
  for (int32_t x = *left; x < *right; x++)
    if (F[x] >= curr && x < nk) nk = x;
  if (nk == *right) return 0;
  *left = nk;
  return 1;
}

/* ---- FindKnee: the consecutive pair with the
 * largest height drop that is >= 10% of the atlas height and >= 20% of the
 * taller chart, unscaled heights.  Returns the taller chart's position in
 * the row, or -1. */
int32_t or_find_knee(int32_t nrow, const int64_t* h_units, int32_t atlas_h) {
  int32_t best = -1;
  int64_t bestd = -1;
  for (int32_t t = 0; t + 1 < nrow; t++) {
    int64_t d = h_units[t] - h_units[t + 1];
    if (10 * d >= (int64_t)atlas_h * 256 && 5 * d >= h_units[t] && d > bestd) {
      best = t;
      bestd = d;
    }
  }
  return best;
}

/* ---- pushing step of Alg. 4: a chart's vertical offset is the
 * max over the texels it covers of (frontline - TopEdge); for a right-to-left
 * row the chart geometry is reflected (D17). */
int32_t or_push_y(const int32_t* F, int32_t X, int32_t wd, const int32_t* Dtop, int32_t dir) {
  int32_t y = INT32_MIN;
  for (int32_t i = 0; i < wd; i++) {
    int32_t dt = dir == 0 ? Dtop[i] : Dtop[wd - 1 - i];
    int32_t v = F[X + i] - dt;
    if (v > y) y = v; /* atomicMax(offsets.y, frontline - TopEdge) */
  }
  return y;
}

/* ---- Alg. 4 for one candidate scale m/M --------------------- */
typedef struct {
  int32_t end;               /* rowEnd */
  int32_t a, b;              /* fold region [a, b) */
  int32_t* X;                /* atlas column of each chart's dilated footprint */
  int32_t* Y;
  int32_t* F;                /* localFrontLine */
  int32_t score, score_knee;
} or_config;

static void eval_config(or_config* cf, const or_prof* pr, const int32_t* wd, const int32_t* xloc,
                        int32_t row_start, int32_t dir, const int32_t* F, int32_t Wp,
                        uint32_t flags, int32_t** pair_buf, int32_t* pair_cap) {
  memcpy(cf->F, F, sizeof(int32_t) * Wp); /* Copy frontLine to localFrontLine[j] */
  for (int32_t s = row_start; s <= cf->end; s++) {
    /* "Reflect charts and chart x offsets" (Alg. 4) -- D17 */
    cf->X[s] = dir == 0 ? cf->a + xloc[s] : cf->b - xloc[s] - wd[s];
    cf->Y[s] = or_push_y(cf->F, cf->X[s], wd[s], pr[s].Dtop, dir);
  }
  /* D15 pair list: every a < b of the row whose dilated x-ranges overlap in
   * the (unreflected) fold frame. */
  int32_t np = 0;
  for (int32_t sa = row_start; sa <= cf->end; sa++) {
    for (int32_t sb = sa + 1; sb <= cf->end; sb++) {
      int32_t delta = xloc[sb] - xloc[sa];
      if (delta >= wd[sa]) continue;
      if ((flags & OR_F_ADJACENT_LOCKS_ONLY) && sb != sa + 1) continue;
      if (np + 1 > *pair_cap) {
        *pair_cap = 2 * (*pair_cap) + 16;
        for (int q = 0; q < 4; q++) pair_buf[q] = realloc(pair_buf[q], sizeof(int32_t) * (*pair_cap));
      }
      int32_t la, lb;
      or_locks(&pr[sa], &pr[sb], delta, &la, &lb);
      pair_buf[0][np] = sa;
      pair_buf[1][np] = sb;
      pair_buf[2][np] = la;
      pair_buf[3][np] = lb;
      np++;
    }
  }
  or_correct_y(np, pair_buf[0], pair_buf[1], pair_buf[2], pair_buf[3], cf->Y);
  for (int32_t s = row_start; s <= cf->end; s++) {
    for (int32_t i = 0; i < wd[s]; i++) {
      int32_t db = dir == 0 ? pr[s].Dbot[i] : pr[s].Dbot[wd[s] - 1 - i];
      int32_t v = cf->Y[s] + db;
      if (v > cf->F[cf->X[s] + i]) cf->F[cf->X[s] + i] = v; /* atomicMax(localFrontLine) */
    }
  }
  cf->score = INT32_MIN;
  for (int32_t x = 0; x < Wp; x++)
    if (cf->F[x] > cf->score) cf->score = cf->F[x];
  cf->score_knee = INT32_MIN;
  for (int32_t x = cf->a; x < cf->b; x++)
    if (cf->F[x] > cf->score_knee) cf->score_knee = cf->F[x];
}

static int tail_rows(const or_prof* pt, const int32_t* q, const int32_t* xl, int32_t n,
                     int32_t r0, const or_spec* spec, int32_t* F, int32_t* X, int32_t* Y,
                     uint8_t* mir, or_cand* cand);

/* ---- D24 prefix-sum tail ("Performance Optimization") --------
 * Remaining sorted charts [r0, n) at candidate m: FastAtlas-style fold of the
 * prefix sum of the horizontal OFFSETS (HC always on), rows cut at
 * multiples of W'; one global intermediate downscale s' = p / 2^20 (P:141
 * "all charts must undergo an intermediate scaling-down") re-rasterized and
 * re-laid per row until every row fits (at most 8 adjustments); rows placed
 * with the fixed FastAtlas alternation, one left-to-right row then two
 * right-to-left rows, pushed with locks, no knees.
 * Returns 1 on success (F, X, Y, mir, pr_tail filled for [r0, n)). */
static int prefix_tail(const or_proxy* px, const int32_t* perm, int32_t n, int32_t r0, int32_t m,
                       const or_spec* spec, const or_prof* pr, const int32_t* off, int32_t* F,
                       int32_t* X, int32_t* Y, uint8_t* mir, or_prof* pt, or_cand* cand) {
  const int32_t g = spec->gutter, M = spec->scale_count;
  const int64_t Wp = spec->atlas_w + 2 * g, Hp = spec->atlas_h + 2 * g;
  const int64_t P20 = (int64_t)1 << 20;
  /* step 1: prefix sum of offsets at scale m, rows = floor(start / W') */
  int32_t* q = malloc(sizeof(int32_t) * n);
  int64_t start = 0, Emax = 0, row_first_start = 0;
  for (int32_t c = r0; c < n; c++) {
    q[c] = (int32_t)(start / Wp);
    if (c == r0 || q[c] != q[c - 1]) row_first_start = start;
    int64_t e = start - row_first_start + pr[c].Wd;
    if (e > Emax) Emax = e;
    if (c + 1 < n) start += off[c];
  }
  /* step 2: global intermediate scale p / 2^20 = (m / M) * sigma with
   * sigma = min(1, W' / Emax) -- an intermediate DOWNscaling (
   * DESIGN.md reading R3 caps sigma at 1) */
  int64_t p = ((i128)m * P20 * Wp) / ((i128)M * Emax);
  const int64_t pm = ((i128)m * P20) / M;
  if (p > pm) p = pm;
  int32_t* xl = malloc(sizeof(int32_t) * n);
  int ok = 0;
  for (int iter = 0; iter <= 8; iter++) {
    if (p < 1) break;
    for (int32_t c = r0; c < n; c++) {
      or_prof_free(&pt[c]);
      or_profile(&px[perm[c]], p, P20, g, &pt[c]);
    }
    int64_t E2 = 0;
    for (int32_t c = r0; c < n; c++) {
      xl[c] = (c == r0 || q[c] != q[c - 1]) ? 0 : xl[c - 1] + or_offset(&pt[c - 1], &pt[c]);
      if (xl[c] + pt[c].Wd > E2) E2 = xl[c] + pt[c].Wd;
    }
    if (E2 <= Wp) { ok = 1; break; }
    if (iter == 8) break;
    p = (p * Wp) / E2;
  }
  cand->p = (int32_t)p;
  cand->switched_at = r0;
  if (ok) ok = tail_rows(pt, q, xl, n, r0, spec, F, X, Y, mir, cand);
  free(q);
  free(xl);
  return ok;
}

/* D24 steps 3-4 (and R6): the tail rows q[] in order, L->R iff row index % 3
 * == 0 (FastAtlas), positions xl[] in the row, pushed with locks (D15,
 * Alg. 1), no knees; fails if the frontline passes the atlas bottom. */
static int tail_rows(const or_prof* pt, const int32_t* q, const int32_t* xl, int32_t n,
                     int32_t r0, const or_spec* spec, int32_t* F, int32_t* X, int32_t* Y,
                     uint8_t* mir, or_cand* cand) {
  const int32_t g = spec->gutter;
  const int64_t Wp = spec->atlas_w + 2 * g, Hp = spec->atlas_h + 2 * g;
  int ok = 1;
  int32_t row_idx = 0;
  int32_t cap = 1, np;
  int32_t *qa = malloc(sizeof(int32_t)), *qb = malloc(sizeof(int32_t));
  int32_t *la = malloc(sizeof(int32_t)), *lb = malloc(sizeof(int32_t));
  for (int32_t a = r0; a < n;) {
    int32_t b = a;
    while (b + 1 < n && q[b + 1] == q[a]) b++;
    const int dir = (row_idx % 3 == 0) ? 0 : 1;
    for (int32_t c = a; c <= b; c++) {
      X[c] = dir == 0 ? xl[c] : (int32_t)Wp - xl[c] - pt[c].Wd;
      Y[c] = or_push_y(F, X[c], pt[c].Wd, pt[c].Dtop, dir);
      mir[c] = (uint8_t)dir;
    }
    np = 0;
    for (int32_t s1 = a; s1 <= b; s1++)
      for (int32_t s2 = s1 + 1; s2 <= b; s2++) {
        int32_t delta = xl[s2] - xl[s1];
        if (delta >= pt[s1].Wd) continue;
        if ((spec->flags & OR_F_ADJACENT_LOCKS_ONLY) && s2 != s1 + 1) continue;
        if (np + 1 > cap) {
          cap = 2 * cap + 8;
          qa = realloc(qa, sizeof(int32_t) * cap); qb = realloc(qb, sizeof(int32_t) * cap);
          la = realloc(la, sizeof(int32_t) * cap); lb = realloc(lb, sizeof(int32_t) * cap);
        }
        qa[np] = s1; qb[np] = s2;
        or_locks(&pt[s1], &pt[s2], delta, &la[np], &lb[np]);
        np++;
      }
    or_correct_y(np, qa, qb, la, lb, Y);
    int32_t score = 0;
    for (int32_t c = a; c <= b; c++)
      for (int32_t i = 0; i < pt[c].Wd; i++) {
        int32_t db = dir == 0 ? pt[c].Dbot[i] : pt[c].Dbot[pt[c].Wd - 1 - i];
        if (Y[c] + db > F[X[c] + i]) F[X[c] + i] = Y[c] + db;
      }
    for (int64_t x = 0; x < Wp; x++)
      if (F[x] > score) score = F[x];
    cand->prefix_rows++;
    cand->score = score;
    if (score > Hp) { ok = 0; break; }
    row_idx++;
    a = b + 1;
  }
  free(qa); free(qb); free(la); free(lb);
  return ok;
}

/* ---- R6 exact-greedy tail (TABI_F_EXACT_TAIL) ----------
 * Same switch (D23) and the same row placement as D24 steps 3-4, but the
 * remaining charts [r0, n) are folded exactly by Alg. 3 with horizontal
 * compaction (HC always on in the tail) at the candidate
 * scale m/M itself: a row never overflows, so there is no intermediate
 * downscale and every chart keeps scale m/M. */
static int exact_tail(int32_t n, int32_t r0, int32_t m, const or_spec* spec, const or_prof* pr,
                      const int32_t* wd, const int32_t* off, int32_t* F, int32_t* X, int32_t* Y,
                      uint8_t* mir, or_cand* cand) {
  const int32_t g = spec->gutter, M = spec->scale_count;
  const int32_t Wp = spec->atlas_w + 2 * g;
  int32_t* q = malloc(sizeof(int32_t) * n);
  int32_t* xl = malloc(sizeof(int32_t) * n);
  int ok = 1;
  int32_t row = 0;
  for (int32_t a = r0; a < n; row++) {
    const int32_t end = or_fold_row(n, a, Wp, 1, wd, off, xl);
    if (end < a) { ok = 0; break; } /* D22: the first chart does not fit */
    for (int32_t c = a; c <= end; c++) q[c] = row;
    a = end + 1;
  }
  cand->p = (int32_t)(((int64_t)m << 20) / M); /* informational: every chart keeps m/M */
  cand->switched_at = r0;
  if (ok) ok = tail_rows(pr, q, xl, n, r0, spec, F, X, Y, mir, cand);
  free(q);
  free(xl);
  return ok;
}

int or_pack_candidate(const or_proxy* px, const int32_t* perm, int32_t n, const or_spec* spec,
                      int32_t m, or_placement* out, or_cand* cand) {
  const int32_t g = spec->gutter, M = spec->scale_count;
  const int32_t Wp = spec->atlas_w + 2 * g, Hp = spec->atlas_h + 2 * g;
  const uint32_t flags = spec->flags;
  memset(cand, 0, sizeof(*cand));
  cand->switched_at = -1;
  or_prof* pr = calloc(n, sizeof(or_prof));
  int32_t* wd = malloc(sizeof(int32_t) * n);
  int32_t* off = calloc(n, sizeof(int32_t));
  int64_t* hu = malloc(sizeof(int64_t) * n);
  for (int32_t s = 0; s < n; s++) {
    or_profile(&px[perm[s]], m, M, g, &pr[s]);
    wd[s] = pr[s].Wd;
    hu[s] = px[perm[s]].h;
  }
  for (int32_t s = 0; s + 1 < n; s++) off[s] = or_offset(&pr[s], &pr[s + 1]);

  int32_t* F = calloc(Wp, sizeof(int32_t)); /* frontline starts at 0 = top */
  int32_t* X = malloc(sizeof(int32_t) * n);
  int32_t* Y = malloc(sizeof(int32_t) * n);
  uint8_t* mir = calloc(n, 1);
  int32_t* xloc[2][2];
  or_config cfg[2][2][2];
  for (int f = 0; f < 2; f++)
    for (int hc = 0; hc < 2; hc++) {
      xloc[f][hc] = malloc(sizeof(int32_t) * n);
      for (int d = 0; d < 2; d++) {
        cfg[f][hc][d].X = malloc(sizeof(int32_t) * n);
        cfg[f][hc][d].Y = malloc(sizeof(int32_t) * n);
        cfg[f][hc][d].F = malloc(sizeof(int32_t) * Wp);
      }
    }
  int32_t* pair_buf[4] = {NULL, NULL, NULL, NULL};
  int32_t pair_cap = 0;

  int knee_valid = 0, knee_ltr = 0;
  int32_t knee_left = 0, knee_right = 0;
  int32_t score = 0;
  int32_t row_start = 0;
  int fail = 0;
  /* D23: t_opt policy ("t_opt = 0% for inputs with up to 10,000 charts and
   * t_opt = 1% otherwise"), in basis points of the atlas height */
  const int32_t t_opt = spec->t_opt_bp >= 0 ? spec->t_opt_bp : (n > 10000 ? 100 : 0);
  or_prof* pt = calloc(n, sizeof(or_prof));  /* tail footprints at s' */
  int32_t r0 = n;
  while (row_start < n && !fail) {
    /* D23 switch to prefix folding "when no more knees are detected and the
     * height of the tallest chart in the row decreases below t_opt";
     * checked before each row, latched. */
    if (t_opt > 0 && !knee_valid &&
        cdiv64(hu[row_start] * m, (int64_t)M * 256) * 10000 < (int64_t)t_opt * spec->atlas_h) {
      r0 = row_start;
      cand->score = score;
      const int okt = (flags & OR_F_EXACT_TAIL)
                          ? exact_tail(n, r0, m, spec, pr, wd, off, F, X, Y, mir, cand)
                          : prefix_tail(px, perm, n, r0, m, spec, pr, off, F, X, Y, mir, pt, cand);
      if (!okt) fail = 1;
      score = cand->score;
      break;
    }
    if (knee_valid) knee_valid = or_update_knee(F, Wp, knee_ltr, &knee_left, &knee_right);
    int nf = knee_valid ? 2 : 1;
    for (int f = 0; f < nf; f++) {
      int32_t a = 0, b = Wp;
      if (f == 1) {
        a = knee_ltr ? knee_right : 0;
        b = knee_ltr ? Wp : knee_left;
      }
      for (int hc = 0; hc < 2; hc++) {
        int32_t end = or_fold_row(n, row_start, b - a, hc, wd, off, xloc[f][hc]);
        for (int d = 0; d < 2; d++) {
          or_config* cf = &cfg[f][hc][d];
          cf->end = end;
          cf->a = a;
          cf->b = b;
          if (end < row_start) continue;
          eval_config(cf, pr, wd, xloc[f][hc], row_start, d, F, Wp, flags, pair_buf, &pair_cap);
        }
      }
    }
    /* Hierarchical selection. Level 1: horizontal compacting iff it
     * fits more charts in the row (strictly). */
    int hcsel[2], dsel[2];
    for (int f = 0; f < nf; f++) {
      hcsel[f] = (!(flags & OR_F_NO_HC) && cfg[f][1][0].end > cfg[f][0][0].end) ? 1 : 0;
    }
    if (cfg[0][hcsel[0]][0].end < row_start) { fail = 1; break; } /* D22 */
    int knee_ok = nf == 2 && cfg[1][hcsel[1]][0].end >= row_start;
    /* Level 2: the direction with the smaller max frontline -- whole
     * frontline for the atlas fold, the knee concavity for the knee fold;
     * ties go left-to-right. */
    for (int f = 0; f < (knee_ok ? 2 : 1); f++) {
      or_config* L = &cfg[f][hcsel[f]][0];
      or_config* R = &cfg[f][hcsel[f]][1];
      int32_t kl = f == 0 ? L->score : L->score_knee;
      int32_t kr = f == 0 ? R->score : R->score_knee;
      dsel[f] = kr < kl ? 1 : 0;
    }
    if (flags & OR_F_NO_BALANCE) dsel[0] = cand->rows & 1; /* static alternation */
    /* Level 3: fold at the knee iff its max height is at least marginally
     * (>= 1 texel) smaller. */
    int fsel = 0;
    if (knee_ok && cfg[1][hcsel[1]][dsel[1]].score <= cfg[0][hcsel[0]][dsel[0]].score - 1) fsel = 1;
    or_config* ch = &cfg[fsel][hcsel[fsel]][dsel[fsel]];
    /* commit (Alg. 4: copy localFrontLine and offsets) */
    memcpy(F, ch->F, sizeof(int32_t) * Wp);
    for (int32_t s = row_start; s <= ch->end; s++) {
      X[s] = ch->X[s];
      Y[s] = ch->Y[s];
      mir[s] = (uint8_t)dsel[fsel];
    }
    cand->rows++;
    if (fsel == 1) cand->knee_rows++;
    if (fsel == 0 && !(flags & OR_F_NO_BALANCE)) {
      int32_t t = or_find_knee(ch->end - row_start + 1, hu + row_start, spec->atlas_h);
      knee_valid = t >= 0;
      if (knee_valid) {
        cand->knees_found++;
        knee_ltr = dsel[0] == 0;
        knee_left = X[row_start + t];
        knee_right = X[row_start + t] + wd[row_start + t];
      }
    }
    score = ch->score;
    if (score > Hp) fail = 1; /* overflow: frontline below the atlas bottom */
    row_start = ch->end + 1;
  }
  cand->score = score;
  cand->success = !fail;
  if (!fail && out) {
    for (int32_t s = 0; s < n; s++) {
      int32_t c = perm[s];
      or_placement* o = &out[c];
      memset(o, 0, sizeof(*o));
      const int tail = s >= r0;  /* tail chart: final scale p / 2^20 (D24) */
      const int ptail = tail && !(flags & OR_F_EXACT_TAIL);  /* R6 keeps m/M */
      o->tx = X[s];
      o->ty = Y[s];
      o->scale_num = ptail ? cand->p : m;
      o->scale_den = ptail ? (1 << 20) : M;
      o->box_w = ptail ? pt[s].ws : pr[s].ws;
      o->box_h = ptail ? pt[s].hs : pr[s].hs;
      o->rot90 = (uint8_t)px[c].rot90;
      o->prerot = (uint8_t)px[c].prerot;
      o->flip_x = (uint8_t)px[c].fx;
      o->flip_y = (uint8_t)px[c].fy;
      o->mirror_x = mir[s];
      o->mode = (uint8_t)tail;
    }
  }
  for (int32_t s = 0; s < n; s++) or_prof_free(&pt[s]);
  free(pt);
  for (int f = 0; f < 2; f++)
    for (int hc = 0; hc < 2; hc++) {
      free(xloc[f][hc]);
      for (int d = 0; d < 2; d++) {
        free(cfg[f][hc][d].X); free(cfg[f][hc][d].Y); free(cfg[f][hc][d].F);
      }
    }
  for (int q = 0; q < 4; q++) free(pair_buf[q]);
  for (int32_t s = 0; s < n; s++) or_prof_free(&pr[s]);
  free(pr); free(wd); free(off); free(hu); free(F); free(X); free(Y); free(mir);
  return cand->success;
}

static int spec_ok(const or_spec* s) {
  return s->atlas_w >= 1 && s->atlas_h >= 1 && s->atlas_w <= 16384 && s->atlas_h <= 16384 &&
         s->gutter >= 0 && s->gutter <= 64 && s->scale_count >= 1 && s->scale_count <= 256 &&
         s->local_aabb_count >= 1 && s->local_aabb_count <= OR_KMAX && s->t_opt_bp >= -1 &&
         s->t_opt_bp <= 10000 && (s->flags & ~63u) == 0;
}

/* ---- scale search + output ("return the largest scale and
 * packing that succeed"; "64 scales ranging from 1/64 to 64/64"). */
int or_pack(const float* xy, const int32_t* start, int32_t n, float res_x, float res_y,
            const or_spec* spec, or_placement* out, or_info* info, or_cand* cands) {
  memset(info, 0, sizeof(*info));
  info->bad_chart = -1;
  if (n < 1 || !spec_ok(spec)) return OR_EINVAL;
  for (int32_t c = 0; c < n; c++)
    if (start[c + 1] - start[c] < 3) { info->bad_chart = c; return OR_EINVAL; }
  or_proxy* px = malloc(sizeof(or_proxy) * n);
  int32_t* perm = malloc(sizeof(int32_t) * n);
  int st = or_build_proxies(xy, start, n, res_x, res_y, spec->local_aabb_count, spec->flags, px,
                            &info->bad_chart);
  if (st != OR_OK) { free(px); free(perm); return st; }
  or_sort(px, n, perm);
  const int32_t M = spec->scale_count;
  const i128 P20 = (i128)1 << 20;
  /* area-prefix by sorted position for the D25 weights */
  i128* apre = malloc(sizeof(i128) * (n + 1));
  apre[0] = 0;
  for (int32_t s = 0; s < n; s++) apre[s + 1] = apre[s] + px[perm[s]].area2;
  int32_t best = 0;
  i128 bestV = -1;
  or_cand bc;
  memset(&bc, 0, sizeof(bc));
  for (int32_t m = 1; m <= M; m++) {
    or_cand cd;
    or_pack_candidate(px, perm, n, spec, m, NULL, &cd);
    if (cands) cands[m - 1] = cd;
    if (!cd.success) continue;
    /* D25: the largest area-weighted mean final scale ("the candidate
     * scale factor S that maximizes the average final scale weighted by chart
     * area"); sequential candidates reduce to the largest m.  Exact:
     * V = A_seq * m * 2^20 + A_pre * p * M; ties go to the larger m. */
    /* R6: every chart keeps m/M, so the whole area counts at m */
    const int32_t r0 =
        (cd.switched_at >= 0 && !(spec->flags & OR_F_EXACT_TAIL)) ? cd.switched_at : n;
    const i128 V = apre[r0] * m * P20 + (apre[n] - apre[r0]) * (i128)cd.p * M;
    if (V >= bestV) { bestV = V; best = m; bc = cd; }
  }
  if (best == 0) { free(px); free(perm); free(apre); return OR_NO_FIT; }
  or_cand cd;
  or_pack_candidate(px, perm, n, spec, best, out, &cd);
  info->scale_index = best;
  {
    /* D26: every map is a similarity, so the per-triangle L2 stretch is 1/s;
     * area-weighted RMS over the charts. */
    const int32_t r0 =
        (bc.switched_at >= 0 && !(spec->flags & OR_F_EXACT_TAIL)) ? bc.switched_at : n;
    if (r0 == n) {
      info->l2_stretch = (double)M / (double)best;
    } else {
      const double fs = (double)apre[r0] / (double)apre[n];
      const double fp = (double)(apre[n] - apre[r0]) / (double)apre[n];
      const double a = (double)M / (double)best, b = (double)(1 << 20) / (double)bc.p;
      info->l2_stretch = sqrt(fs * a * a + fp * b * b);
    }
  }
  free(apre);
  info->rows = bc.rows;
  info->knees_found = bc.knees_found;
  info->knee_rows = bc.knee_rows;
  info->prefix_rows = bc.prefix_rows;
  free(px);
  free(perm);
  return OR_OK;
}
