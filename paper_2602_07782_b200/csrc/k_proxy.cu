// k_proxy.cu -- K1: per-chart proxies, one warp per chart.
//
// Computes, for every chart ("compute the AABBs of all charts, rotate the
// boxes to be taller than they are wide ... two parallel passes which compute
// our shape approximations for each chart and determine each chart's
// orientation"):
//   snap to 1/256 texel -> AABB -> 90-degree normalization -> local AABBs
//    + merge -> orientation -> final pose ->
//   local AABBs again -> approximate OBB over 8 angles.
// Lanes stride over vertices / edges; slice bounds are accumulated with
// shared-memory atomicMin/Max (commutative, so schedule-independent), merges
// and reductions use warp shuffles.  Output: proxy SoA in HBM.
#include "tabi_internal.cuh"

namespace tabi {
namespace {

constexpr int kWarps = 8;  // warps (charts) per block

struct WarpSlices {
  int32_t lo[2][TABI_KMAX];  // unmerged: [0] x-slices top, [1] y-slices left
  int32_t hi[2][TABI_KMAX];  //           [0] x-slices bot, [1] y-slices right
  int32_t mlo[2][TABI_KMAX]; // merged
  int32_t mhi[2][TABI_KMAX];
  int64_t fl[2][TABI_KMAX];  // floor(i * ext / k) for the other axis' slice edges
  int64_t cl[2][TABI_KMAX];  // ceil((i + 1) * ext / k)
  int64_t ob[8][4];          // OBB extents per angle: Umin, Umax, Vmin, Vmax
};

// D4: slice bounds along one axis.  A = coordinate that is sliced (x for
// x-slices), B = the bounded coordinate.  Strip j = closed range k*A in
// [j*ext, (j+1)*ext].
__device__ void accumulate_slices(const int32_t* A, const int32_t* B, int nv, int64_t ext, int k,
                                  int32_t* lo, int32_t* hi, int lane) {
  const double rext = rcp_approx((double)ext);
  for (int v = lane; v < nv; v += 32) {
    int64_t ka = (int64_t)k * A[v];
    int64_t jh = fdiv_r64(ka, ext, rext);            // floor(k*a/ext), a >= 0
    int64_t jl = -fdiv_r64(-ka, ext, rext) - 1;      // ceil(k*a/ext) - 1
    if (jl < 0) jl = 0;
    if (jh > k - 1) jh = k - 1;
    for (int64_t j = jl; j <= jh; j++) {
      if (j * ext <= ka && ka <= (j + 1) * ext) {
        atomicMin(&lo[j], B[v]);
        atomicMax(&hi[j], B[v]);
      }
    }
  }
  for (int v = lane; v < nv; v += 32) {
    int a = v, b = (v + 1 == nv) ? 0 : v + 1;
    int64_t xa = A[a], xb = A[b], ya = B[a], yb = B[b];
    if (xa == xb) continue;
    if (xa > xb) {
      int64_t t = xa; xa = xb; xb = t;
      t = ya; ya = yb; yb = t;
    }
    int64_t L0 = fdiv_r64((int64_t)k * xa, ext, rext) + 1;       // first line strictly right of xa
    int64_t L1 = -fdiv_r64(-(int64_t)k * xb, ext, rext) - 1;     // last line strictly left of xb
    if (L0 < 1) L0 = 1;
    if (L1 > k - 1) L1 = k - 1;
    for (int64_t L = L0; L <= L1; L++) {
      int64_t line = L * ext;
      if (!((int64_t)k * xa < line && line < (int64_t)k * xb)) continue;
      int64_t num = (line - (int64_t)k * xa) * (yb - ya);
      int64_t den = (int64_t)k * (xb - xa);
      int32_t yf = (int32_t)(ya + fdiv_fast(num, den));
      int32_t yc = (int32_t)(ya + cdiv_fast(num, den));
      atomicMin(&lo[L - 1], yf);
      atomicMax(&hi[L - 1], yc);
      atomicMin(&lo[L], yf);
      atomicMax(&hi[L], yc);
    }
  }
}

// D5 merge: x-slice j tightened by y-slices whose x-range meets strip j.
__device__ void merge_slices(WarpSlices& S, int64_t w, int64_t h, int k, int lane) {
  for (int i = lane; i < k; i += 32) {
    S.fl[0][i] = fdiv_fast((int64_t)i * h, k);
    S.cl[0][i] = cdiv_fast((int64_t)(i + 1) * h, k);
    S.fl[1][i] = fdiv_fast((int64_t)i * w, k);
    S.cl[1][i] = cdiv_fast((int64_t)(i + 1) * w, k);
  }
  __syncwarp();
  for (int j = lane; j < k; j += 32) {
    // x-slices
    int64_t mn = INT64_MAX, mx = INT64_MIN;
    for (int i = 0; i < k; i++) {
      if ((int64_t)k * S.lo[1][i] <= (int64_t)(j + 1) * w && (int64_t)k * S.hi[1][i] >= (int64_t)j * w) {
        const int64_t f = S.fl[0][i], c = S.cl[0][i];
        mn = f < mn ? f : mn;
        mx = c > mx ? c : mx;
      }
    }
    int64_t t = S.lo[0][j], b = S.hi[0][j];
    if (mn != INT64_MAX && mn > t) t = mn;
    if (mx != INT64_MIN && mx < b) b = mx;
    S.mlo[0][j] = (int32_t)t;
    S.mhi[0][j] = (int32_t)b;
    // y-slices
    mn = INT64_MAX;
    mx = INT64_MIN;
    for (int i = 0; i < k; i++) {
      if ((int64_t)k * S.lo[0][i] <= (int64_t)(j + 1) * h && (int64_t)k * S.hi[0][i] >= (int64_t)j * h) {
        const int64_t f = S.fl[1][i], c = S.cl[1][i];
        mn = f < mn ? f : mn;
        mx = c > mx ? c : mx;
      }
    }
    t = S.lo[1][j];
    b = S.hi[1][j];
    if (mn != INT64_MAX && mn > t) t = mn;
    if (mx != INT64_MIN && mx < b) b = mx;
    S.mlo[1][j] = (int32_t)t;
    S.mhi[1][j] = (int32_t)b;
  }
}

__device__ void merged_slices(WarpSlices& S, const int32_t* X, const int32_t* Y, int nv, int64_t w,
                              int64_t h, int k, int lane) {
  for (int j = lane; j < k; j += 32) {
    S.lo[0][j] = INT32_MAX; S.hi[0][j] = INT32_MIN;
    S.lo[1][j] = INT32_MAX; S.hi[1][j] = INT32_MIN;
  }
  __syncwarp();
  accumulate_slices(X, Y, nv, w, k, S.lo[0], S.hi[0], lane);
  accumulate_slices(Y, X, nv, h, k, S.lo[1], S.hi[1], lane);
  __syncwarp();
  merge_slices(S, w, h, k, lane);
  __syncwarp();
}

__global__ void __launch_bounds__(kWarps * 32)
proxy_kernel(const float* __restrict__ xy, const int32_t* __restrict__ start, int32_t n, float rx,
             float ry, int k, int32_t* qx, int32_t* qy, Proxies P, Status* st) {
  __shared__ WarpSlices smem[kWarps];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int c = blockIdx.x * kWarps + wib;
  if (c >= n) return;
  WarpSlices& S = smem[wib];
  const int32_t a0 = start[c];
  const int nv = start[c + 1] - a0;
  if (nv < 3) {
    if (lane == 0) atomicMin(&st->bad_chart, c);
    return;
  }
  int32_t* X = qx + a0;
  int32_t* Y = qy + a0;
  // A1 snap: q = round_half_even(x * res * 256), exact product in double (D2)
  bool ok = true;
  int32_t xmn = INT32_MAX, xmx = INT32_MIN, ymn = INT32_MAX, ymx = INT32_MIN;
  for (int v = lane; v < nv; v += 32) {
    double fx = (double)xy[2 * (int64_t)(a0 + v)] * (double)rx * 256.0;
    double fy = (double)xy[2 * (int64_t)(a0 + v) + 1] * (double)ry * 256.0;
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
  if (!__all_sync(0xffffffffu, ok)) {
    if (lane == 0) atomicMin(&st->bad_chart, c);
    return;
  }
  xmn = warp_min(xmn); xmx = warp_max(xmx);
  ymn = warp_min(ymn); ymx = warp_max(ymx);
  int64_t w = (int64_t)xmx - xmn, h = (int64_t)ymx - ymn;
  __syncwarp();
  for (int v = lane; v < nv; v += 32) { X[v] -= xmn; Y[v] -= ymn; }
  __syncwarp();
  // D3 shoelace (2 x area), exact
  i128 s2 = 0;
  for (int v = lane; v < nv; v += 32) {
    int u = (v + 1 == nv) ? 0 : v + 1;
    s2 += (i128)((int64_t)X[v] * Y[u] - (int64_t)X[u] * Y[v]);
  }
  s2 = warp_sum128(s2);
  if (s2 < 0) s2 = -s2;
  if (s2 == 0) {
    if (lane == 0) atomicMin(&st->bad_chart, c);
    return;
  }
  // D3 90-degree normalization: (x, y) -> (h - y, x) iff w > h
  const bool rot = w > h;
  if (rot) {
    for (int v = lane; v < nv; v += 32) {
      int32_t nx = (int32_t)(h - Y[v]), ny = X[v];
      X[v] = nx;
      Y[v] = ny;
    }
    int64_t t = w; w = h; h = t;
  }
  __syncwarp();
  // D4/D5 in the normalized pose, D7 orientation
  merged_slices(S, X, Y, nv, w, h, k, lane);
  // empty-area sums: every term is in [0, 2^25] and k <= 64, so the sums fit
  // 32 unsigned bits and reduce in hardware (REDUX)
  uint32_t top = 0, bot = 0, left = 0, right = 0;
  for (int j = lane; j < k; j += 32) {
    top += (uint32_t)S.mlo[0][j];
    bot += (uint32_t)(h - S.mhi[0][j]);
    left += (uint32_t)S.mlo[1][j];
    right += (uint32_t)(w - S.mhi[1][j]);
  }
  const int64_t TOP = __reduce_add_sync(0xffffffffu, top), BOT = __reduce_add_sync(0xffffffffu, bot);
  const int64_t LEFT = __reduce_add_sync(0xffffffffu, left);
  const int64_t RIGHT = __reduce_add_sync(0xffffffffu, right);
  const bool fy = TOP > BOT;
  const int64_t D = LEFT - RIGHT;
  bool fx;
  if ((i128)10 * D > (i128)k * w) {
    fx = true;
  } else if ((i128)10 * (-D) > (i128)k * w) {
    fx = false;
  } else {
    int64_t BL2 = 0, BR2 = 0;
    for (int j = lane; j < k; j += 32) {
      int64_t gap = fy ? S.mlo[0][j] : (h - S.mhi[0][j]);
      if (2 * j + 1 < k) BL2 += 2 * gap;
      else if (2 * j + 1 > k) BR2 += 2 * gap;
      else { BL2 += gap; BR2 += gap; }
    }
    BL2 = warp_sum64(BL2);
    BR2 = warp_sum64(BR2);
    fx = BL2 > BR2;
  }
  // D8 final pose.  The slices of the reflected chart are the reflected
  // slices: x -> w - x maps x-strip j to strip k-1-j (closed strips, the same
  // crossings) and a floored left bound to w - (ceiled right bound); the merge
  // commutes with both maps.  So the final-pose merged slices are an index
  // mirror plus a value reflection of the ones just computed -- no second
  // slicing pass (tests compare every slice with the oracle, which re-slices).
  if (fx || fy) {
    __syncwarp();
    for (int v = lane; v < nv; v += 32) {
      if (fx) X[v] = (int32_t)(w - X[v]);
      if (fy) Y[v] = (int32_t)(h - Y[v]);
    }
    int32_t t0[2], b0[2], l1[2], r1[2];  // k <= 64: two slices per lane
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int j = lane + 32 * u;
      if (j >= k) continue;
      const int sx = fx ? k - 1 - j : j;  // x-slices are indexed along x
      const int sy = fy ? k - 1 - j : j;  // y-slices along y
      t0[u] = fy ? (int32_t)(h - S.mhi[0][sx]) : S.mlo[0][sx];
      b0[u] = fy ? (int32_t)(h - S.mlo[0][sx]) : S.mhi[0][sx];
      l1[u] = fx ? (int32_t)(w - S.mhi[1][sy]) : S.mlo[1][sy];
      r1[u] = fx ? (int32_t)(w - S.mlo[1][sy]) : S.mhi[1][sy];
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int j = lane + 32 * u;
      if (j >= k) continue;
      S.mlo[0][j] = t0[u]; S.mhi[0][j] = b0[u];
      S.mlo[1][j] = l1[u]; S.mhi[1][j] = r1[u];
    }
    __syncwarp();
  }
  int32_t* sl = P.sl + (int64_t)c * 4 * k;
  for (int j = lane; j < k; j += 32) {
    sl[j] = S.mlo[0][j];
    sl[k + j] = S.mhi[0][j];
    sl[2 * k + j] = S.mlo[1][j];
    sl[3 * k + j] = S.mhi[1][j];
  }
  // D6 OBB: minimum (Umax-Umin)(Vmax-Vmin) over 8 angles, ties -> smaller j.
  // All 8 angles at once: lane = 4 * angle + vertex group, so the extents are
  // reduced over 4 lanes (2 shuffle steps) instead of 32 lanes per angle.
  {
    const int j = lane >> 2, g = lane & 3;
    const int64_t C = kQC[j], Sn = kQS[j];
    int64_t u0 = INT64_MAX, u1 = INT64_MIN, v0 = INT64_MAX, v1 = INT64_MIN;
    for (int v = g; v < nv; v += 4) {
      const int64_t x = X[v], y = Y[v];
      const int64_t u = x * C + y * Sn, vv = -x * Sn + y * C;
      u0 = u < u0 ? u : u0; u1 = u > u1 ? u : u1;
      v0 = vv < v0 ? vv : v0; v1 = vv > v1 ? vv : v1;
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      int64_t t = __shfl_xor_sync(0xffffffffu, u0, o); u0 = t < u0 ? t : u0;
      t = __shfl_xor_sync(0xffffffffu, u1, o); u1 = t > u1 ? t : u1;
      t = __shfl_xor_sync(0xffffffffu, v0, o); v0 = t < v0 ? t : v0;
      t = __shfl_xor_sync(0xffffffffu, v1, o); v1 = t > v1 ? t : v1;
    }
    if (g == 0) {
      S.ob[j][0] = u0; S.ob[j][1] = u1; S.ob[j][2] = v0; S.ob[j][3] = v1;
    }
    __syncwarp();
  }
  if (lane == 0) {
    i128 best = -1;
    int bj = 0;
    for (int j = 0; j < 8; j++) {
      const i128 area = (i128)(S.ob[j][1] - S.ob[j][0]) * (i128)(S.ob[j][3] - S.ob[j][2]);
      if (best < 0 || area < best) { best = area; bj = j; }
    }
    const int64_t bu0 = S.ob[bj][0], bu1 = S.ob[bj][1], bv0 = S.ob[bj][2], bv1 = S.ob[bj][3];
    P.w[c] = (int32_t)w;
    P.h[c] = (int32_t)h;
    P.area2[c] = (int64_t)s2;
    P.xmin[c] = xmn;
    P.ymin[c] = ymn;
    P.pose[c] = (uint8_t)((rot ? 1 : 0) | (fx ? 2 : 0) | (fy ? 4 : 0));
    P.obb_j[c] = bj;
    P.obb[4 * (int64_t)c + 0] = bu0;
    P.obb[4 * (int64_t)c + 1] = bu1;
    P.obb[4 * (int64_t)c + 2] = bv0;
    P.obb[4 * (int64_t)c + 3] = bv1;
  }
}

}  // namespace

void launch_proxies(const float* xy, const int32_t* start, int32_t n, float rx, float ry, int k,
                    int32_t* qx, int32_t* qy, Proxies P, Status* st, cudaStream_t s) {
  int blocks = (n + kWarps - 1) / kWarps;
  proxy_kernel<<<blocks, kWarps * 32, 0, s>>>(xy, start, n, rx, ry, k, qx, qy, P, st);
}

}  // namespace tabi
