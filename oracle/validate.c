/* oracle/validate.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Exact integer raster validator ("number of texels
 * covered by two or more charts ... when rendered with 1 pixel gutter
 * dilation").  Independent of the proxy/profile machinery: it re-derives the
 * pose from the raw polygon and the placement alone, maps every snapped vertex
 * to the atlas with exact rationals (common denominator D = den * 256), and
 * marks texel (i, r) covered iff the OPEN square (i, i+1) x (r, r+1) meets the
 * closed polygon: some edge crosses the open square, or the square's centre is
 * inside (then the whole open square is).  Counts:
 *   overlap    texels covered by >= 2 charts,
 *   gutter     texels covered by >= 2 charts after a g-Chebyshev dilation of
 *              each chart's coverage (atlas edges exempt),
 *   oob        covered texels outside [0, W) x [0, H),
 *   covered    atlas texels covered by >= 1 chart (occupancy metric).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

typedef __int128 i128;

static int vsnap(float v, float res, int64_t* q) {
  double x = (double)v * (double)res * 256.0;
  if (!isfinite(x) || fabs(x) > (double)OR_QMAX) return 0;
  *q = (int64_t)llrint(x);
  return 1;
}

/* Q30 cos / sin of j pi / 16 for the pre-rotation step. */
static const int64_t V_QC[8] = {1073741824, 1053110176, 992008094, 892783698,
                                759250125,  596538995,  410903207, 209476638};
static const int64_t V_QS[8] = {0,         209476638, 410903207, 596538995,
                                759250125, 892783698, 992008094, 1053110176};

static int64_t v_q30_round(int64_t a) { /* round_half_even(a / 2^30) */
  int64_t q = a >> 30;
  int64_t r = a - (q << 30);
  if (r > ((int64_t)1 << 29) || (r == ((int64_t)1 << 29) && (q & 1))) q++;
  return q;
}

/* Placement transform documented in include/tabi.h (tabi_placement). */
static int atlas_coords(const float* xy, int32_t nv, float rx, float ry, const or_placement* P,
                        int64_t* AX, int64_t* AY, int64_t* D) {
  int64_t xmin = 0, ymin = 0, xmax = 0, ymax = 0;
  for (int32_t v = 0; v < nv; v++) {
    int64_t x, y;
    if (!vsnap(xy[2 * v], rx, &x) || !vsnap(xy[2 * v + 1], ry, &y)) return 0;
    if (P->prerot) {  /* step 0: pre-rotation into the OBB frame, rounded (R4) */
      const int64_t u = x * V_QC[P->prerot] + y * V_QS[P->prerot];
      const int64_t t = -x * V_QS[P->prerot] + y * V_QC[P->prerot];
      x = v_q30_round(u);
      y = v_q30_round(t);
    }
    AX[v] = x;
    AY[v] = y;
    if (v == 0 || x < xmin) xmin = x;
    if (v == 0 || x > xmax) xmax = x;
    if (v == 0 || y < ymin) ymin = y;
    if (v == 0 || y > ymax) ymax = y;
  }
  int64_t w = xmax - xmin, h = ymax - ymin;
  if (P->rot90) { int64_t t = w; w = h; h = t; }
  *D = (int64_t)P->scale_den * 256;
  for (int32_t v = 0; v < nv; v++) {
    int64_t u = AX[v] - xmin, t = AY[v] - ymin;
    if (P->rot90) { int64_t nu = w - t, nt = u; u = nu; t = nt; }
    if (P->flip_x) u = w - u;
    if (P->flip_y) t = h - t;
    int64_t ux = u * P->scale_num, vy = t * P->scale_num;
    if (P->mirror_x) ux = (int64_t)P->box_w * (*D) - ux;
    AX[v] = (int64_t)P->tx * (*D) + ux;
    AY[v] = (int64_t)P->ty * (*D) + vy;
  }
  return 1;
}

/* n1/d1 < n2/d2 (or <=), d1, d2 > 0 */
static int rlt(i128 n1, i128 d1, i128 n2, i128 d2, int strict) {
  i128 l = n1 * d2, r = n2 * d1;
  return strict ? l < r : l <= r;
}

/* Does segment P->Q meet the open box (x0, x1) x (y0, y1)? */
static int seg_hits_open_box(int64_t px, int64_t py, int64_t qx, int64_t qy, int64_t x0,
                             int64_t x1, int64_t y0, int64_t y1) {
  /* t-interval constraints: lower bounds (num, den, open), upper bounds */
  i128 ln[3], ld[3], un[3], ud[3];
  int lo[3], uo[3], nl = 0, nu = 0;
  ln[nl] = 0; ld[nl] = 1; lo[nl++] = 0;
  un[nu] = 1; ud[nu] = 1; uo[nu++] = 0;
  int64_t d[2] = {qx - px, qy - py}, p[2] = {px, py}, a[2] = {x0, y0}, b[2] = {x1, y1};
  for (int ax = 0; ax < 2; ax++) {
    if (d[ax] == 0) {
      if (!(a[ax] < p[ax] && p[ax] < b[ax])) return 0;
      continue;
    }
    i128 dd = d[ax] > 0 ? d[ax] : -d[ax];
    i128 t_a = (i128)(a[ax] - p[ax]) * (d[ax] > 0 ? 1 : -1); /* (a - p)/d */
    i128 t_b = (i128)(b[ax] - p[ax]) * (d[ax] > 0 ? 1 : -1);
    if (d[ax] > 0) {
      ln[nl] = t_a; ld[nl] = dd; lo[nl++] = 1;
      un[nu] = t_b; ud[nu] = dd; uo[nu++] = 1;
    } else {
      ln[nl] = t_b; ld[nl] = dd; lo[nl++] = 1;
      un[nu] = t_a; ud[nu] = dd; uo[nu++] = 1;
    }
  }
  for (int i = 0; i < nl; i++)
    for (int j = 0; j < nu; j++)
      if (!rlt(ln[i], ld[i], un[j], ud[j], lo[i] || uo[j])) return 0;
  return 1;
}

/* even-odd point-in-polygon for a point strictly off the boundary */
static int inside(const int64_t* X, const int64_t* Y, int32_t nv, i128 cx, i128 cy, i128 scale) {
  int in = 0;
  for (int32_t v = 0; v < nv; v++) {
    int32_t u = (v + 1) % nv;
    i128 py = (i128)Y[v] * scale, qy = (i128)Y[u] * scale;
    if ((py > cy) != (qy > cy)) {
      i128 px = (i128)X[v] * scale, qx = (i128)X[u] * scale;
      /* x of the crossing: px + (cy - py) * (qx - px) / (qy - py) ; test cx < it */
      i128 num = (cy - py) * (qx - px), den = qy - py;
      i128 lhs = (cx - px) * den;
      if (den > 0 ? lhs < num : lhs > num) in = !in;
    }
  }
  return in;
}

int or_raster_chart(const float* xy, int32_t nv, float res_x, float res_y, const or_proxy* unused,
                    const or_placement* pl, int32_t x0, int32_t y0, int32_t nx, int32_t ny,
                    uint8_t* mask) {
  (void)unused;
  int64_t* AX = malloc(sizeof(int64_t) * nv);
  int64_t* AY = malloc(sizeof(int64_t) * nv);
  int64_t D;
  if (!atlas_coords(xy, nv, res_x, res_y, pl, AX, AY, &D)) { free(AX); free(AY); return 0; }
  memset(mask, 0, (size_t)nx * ny);
  for (int32_t r = 0; r < ny; r++) {
    int64_t ya = (int64_t)(y0 + r) * D, yb = ya + D;
    for (int32_t i = 0; i < nx; i++) {
      int64_t xa = (int64_t)(x0 + i) * D, xb = xa + D;
      int hit = 0;
      for (int32_t v = 0; v < nv && !hit; v++) {
        int32_t u = (v + 1) % nv;
        int64_t mnx = AX[v] < AX[u] ? AX[v] : AX[u], mxx = AX[v] < AX[u] ? AX[u] : AX[v];
        int64_t mny = AY[v] < AY[u] ? AY[v] : AY[u], mxy = AY[v] < AY[u] ? AY[u] : AY[v];
        if (mxx <= xa || mnx >= xb || mxy <= ya || mny >= yb) continue;
        hit = seg_hits_open_box(AX[v], AY[v], AX[u], AY[u], xa, xb, ya, yb);
      }
      if (!hit) hit = inside(AX, AY, nv, (i128)(2 * xa + D), (i128)(2 * ya + D), 2);
      mask[(size_t)r * nx + i] = (uint8_t)hit;
    }
  }
  free(AX);
  free(AY);
  return 1;
}

static int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b) != 0 && a < 0) q--;
  return q;
}
static int64_t ceildiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b) != 0 && a > 0) q++;
  return q;
}

int or_validate(const float* xy, const int32_t* start, int32_t n, float res_x, float res_y,
                int32_t W, int32_t H, int32_t g, const or_placement* pl, int64_t* counts) {
  counts[0] = counts[1] = counts[2] = counts[3] = 0;
  size_t A = (size_t)W * H;
  int32_t* last0 = malloc(sizeof(int32_t) * A);
  int32_t* lastg = malloc(sizeof(int32_t) * A);
  uint8_t* cnt0 = calloc(A, 1);
  uint8_t* cntg = calloc(A, 1);
  for (size_t i = 0; i < A; i++) last0[i] = lastg[i] = -1;
  int ok = 1;
  for (int32_t c = 0; c < n && ok; c++) {
    int32_t nv = start[c + 1] - start[c];
    const float* p = xy + 2 * (int64_t)start[c];
    int64_t* AX = malloc(sizeof(int64_t) * nv);
    int64_t* AY = malloc(sizeof(int64_t) * nv);
    int64_t D;
    ok = atlas_coords(p, nv, res_x, res_y, &pl[c], AX, AY, &D);
    int64_t mnx = AX[0], mxx = AX[0], mny = AY[0], mxy = AY[0];
    for (int32_t v = 1; v < nv; v++) {
      if (AX[v] < mnx) mnx = AX[v];
      if (AX[v] > mxx) mxx = AX[v];
      if (AY[v] < mny) mny = AY[v];
      if (AY[v] > mxy) mxy = AY[v];
    }
    free(AX);
    free(AY);
    if (!ok) break;
    int32_t x0 = (int32_t)floordiv(mnx, D), x1 = (int32_t)ceildiv(mxx, D);
    int32_t y0 = (int32_t)floordiv(mny, D), y1 = (int32_t)ceildiv(mxy, D);
    int32_t nx = x1 - x0, ny = y1 - y0;
    if (nx <= 0 || ny <= 0) continue;
    uint8_t* mask = malloc((size_t)nx * ny);
    or_raster_chart(p, nv, res_x, res_y, NULL, &pl[c], x0, y0, nx, ny, mask);
    for (int32_t r = 0; r < ny; r++)
      for (int32_t i = 0; i < nx; i++) {
        if (!mask[(size_t)r * nx + i]) continue;
        int32_t X = x0 + i, Y = y0 + r;
        if (X < 0 || Y < 0 || X >= W || Y >= H) { counts[2]++; continue; }
        size_t t = (size_t)Y * W + X;
        if (last0[t] != c) { last0[t] = c; if (cnt0[t] < 255) cnt0[t]++; }
        for (int32_t dy = -g; dy <= g; dy++)
          for (int32_t dx = -g; dx <= g; dx++) {
            int32_t XX = X + dx, YY = Y + dy;
            if (XX < 0 || YY < 0 || XX >= W || YY >= H) continue;
            size_t tt = (size_t)YY * W + XX;
            if (lastg[tt] != c) { lastg[tt] = c; if (cntg[tt] < 255) cntg[tt]++; }
          }
      }
    free(mask);
  }
  for (size_t i = 0; i < A; i++) {
    if (cnt0[i] >= 1) counts[3]++; /* covered: occupancy = covered / (W H) */
    if (cnt0[i] >= 2) counts[0]++;
    if (cntg[i] >= 2) counts[1]++;
  }
  free(last0); free(lastg); free(cnt0); free(cntg);
  return ok;
}
