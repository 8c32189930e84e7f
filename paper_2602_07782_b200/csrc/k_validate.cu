// k_validate.cu -- N3: GPU raster validator and atlas metrics.
//
// P:85 / P:353 count "texels covered by two or more charts" with 1-pixel
// gutter dilation; S:545-553 fix the conservative rule: texel (i, r) is
// covered by a chart iff the OPEN square (i, i+1) x (r, r+1) meets the closed
// polygon placed by its tabi_placement (include/tabi.h, steps 0-6).  Counts
// are exact (integer geometry, i128 where products need it):
//   overlap  atlas texels covered by >= 2 charts
//   gutter   atlas texels covered by >= 2 charts after each chart's in-atlas coverage is
//            dilated by g (Chebyshev), atlas edges exempt
//   oob      covered texels outside [0, W) x [0, H)
//   covered  atlas texels covered by >= 1 chart (occupancy = covered / (W H))
// and the L2 stretch: every chart map is a similarity with scale
// s_c = num / den, so each triangle's stretch is 1/s_c and the area-weighted
// RMS is sqrt(sum A_c / s_c^2 / sum A_c), A_c the snapped outline's area.
//
// Pipeline (all on the context stream):
//   V1 coords  one warp per chart: snap, step 0-6 in exact integers with the
//              common denominator D = den * 256, the texel bbox, the area;
//   V2 scan    one CTA: prefix sums of the bbox areas (plain and g-dilated) and
//              the deterministic stretch sums;
//   V3 raster  flat over every (chart, dilated-bbox texel): coverage byte into
//              the chart's mask, 2-bit saturating counters per atlas texel
//              (seen-once / seen-twice; one chart visits a texel once);
//   V4/V5      separable Chebyshev dilation of each mask (row pass, column
//              pass), the column pass feeding the gutter counters;
//   V6 count   popcounts of the counter words.
// Masks live in HBM (one byte per dilated bbox texel); the counters are
// 2 bits per atlas texel, 8 MB for 4096^2.
#include <cstdio>
#include <cstring>

#include "tabi_internal.cuh"

namespace tabi {
namespace {

constexpr int kThreads = 256;

struct VChart {
  int64_t D;          // common denominator den * 256 of this chart's coordinates
  int32_t x0, y0;     // texel bbox origin
  int32_t nx, ny;     // texel bbox size (0 if degenerate)
  int64_t area2;      // 2 x snapped outline area, 1/256^2 texel units
  double inv_s2;      // (den / num)^2
};

// Q30 cos / sin of j pi / 16 (D6) for step 0.
__constant__ int64_t vQC[8] = {1073741824, 1053110176, 992008094, 892783698,
                               759250125,  596538995,  410903207, 209476638};
__constant__ int64_t vQS[8] = {0,         209476638, 410903207, 596538995,
                               759250125, 892783698, 992008094, 1053110176};

__device__ __forceinline__ int64_t rhe_q30(int64_t a) {  // round_half_even(a / 2^30)
  const int64_t fl = a >> 30, rem = a & ((1ll << 30) - 1);
  const int64_t half = 1ll << 29;
  return fl + ((rem > half || (rem == half && (fl & 1))) ? 1 : 0);
}

__device__ __forceinline__ int64_t wmin64(int64_t v) {
  for (int o = 16; o; o >>= 1) { const int64_t t = __shfl_xor_sync(~0u, v, o); v = t < v ? t : v; }
  return v;
}
__device__ __forceinline__ int64_t wmax64(int64_t v) {
  for (int o = 16; o; o >>= 1) { const int64_t t = __shfl_xor_sync(~0u, v, o); v = t > v ? t : v; }
  return v;
}

// V1: one warp per chart.
__global__ void __launch_bounds__(kThreads)
v_coords_kernel(const float* __restrict__ xy, const int32_t* __restrict__ start, int32_t n,
                float rx, float ry, const tabi_placement* __restrict__ pl, int64_t* AX,
                int64_t* AY, VChart* ch, int32_t* bad) {
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  if (c >= n) return;
  const int32_t a0 = start[c], nv = start[c + 1] - a0;
  const tabi_placement P = pl[c];
  bool ok = nv >= 3 && P.scale_num > 0 && P.scale_den > 0 && P.prerot < 8;
  int64_t xmn = INT64_MAX, xmx = INT64_MIN, ymn = INT64_MAX, ymx = INT64_MIN;
  // snap (D2) + step 0; the snapped coordinates are parked in AX/AY
  for (int v = lane; v < nv && ok; v += 32) {
    const double fx = (double)xy[2 * (int64_t)(a0 + v)] * (double)rx * 256.0;
    const double fy = (double)xy[2 * (int64_t)(a0 + v) + 1] * (double)ry * 256.0;
    if (!(fabs(fx) <= (double)TABI_QMAX) || !(fabs(fy) <= (double)TABI_QMAX)) { ok = false; break; }
    int64_t x = __double2ll_rn(fx), y = __double2ll_rn(fy);
    if (P.prerot) {
      const int64_t C = vQC[P.prerot], S = vQS[P.prerot];
      const int64_t u = rhe_q30(x * C + y * S), t = rhe_q30(y * C - x * S);
      x = u;
      y = t;
    }
    AX[a0 + v] = x;
    AY[a0 + v] = y;
    xmn = min(xmn, x); xmx = max(xmx, x);
    ymn = min(ymn, y); ymx = max(ymx, y);
  }
  if (__any_sync(~0u, !ok)) {
    if (lane == 0) {
      atomicMin(bad, c);
      ch[c] = VChart{1, 0, 0, 0, 0, 0, 0.0};
    }
    return;
  }
  xmn = wmin64(xmn); xmx = wmax64(xmx); ymn = wmin64(ymn); ymx = wmax64(ymx);
  __syncwarp();
  // area of the snapped outline before step 0 (the chart's own area)
  int64_t s2 = 0;
  for (int v = lane; v < nv; v += 32) {
    const int u = v + 1 == nv ? 0 : v + 1;
    const int64_t x0 = __double2ll_rn((double)xy[2 * (int64_t)(a0 + v)] * (double)rx * 256.0);
    const int64_t y0 = __double2ll_rn((double)xy[2 * (int64_t)(a0 + v) + 1] * (double)ry * 256.0);
    const int64_t x1 = __double2ll_rn((double)xy[2 * (int64_t)(a0 + u)] * (double)rx * 256.0);
    const int64_t y1 = __double2ll_rn((double)xy[2 * (int64_t)(a0 + u) + 1] * (double)ry * 256.0);
    s2 += x0 * y1 - x1 * y0;
  }
  for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(~0u, s2, o);
  // steps 1-6: posed, scaled, mirrored, translated; denominator D
  const int64_t w0 = xmx - xmn, h0 = ymx - ymn;
  const int64_t w = P.rot90 ? h0 : w0, h = P.rot90 ? w0 : h0;
  const int64_t D = (int64_t)P.scale_den * 256;
  int64_t bx0 = INT64_MAX, bx1 = INT64_MIN, by0 = INT64_MAX, by1 = INT64_MIN;
  for (int v = lane; v < nv; v += 32) {
    int64_t u = AX[a0 + v] - xmn, t = AY[a0 + v] - ymn;
    if (P.rot90) { const int64_t nu = w - t; t = u; u = nu; }
    if (P.flip_x) u = w - u;
    if (P.flip_y) t = h - t;
    int64_t X = u * P.scale_num, Y = t * P.scale_num;
    if (P.mirror_x) X = (int64_t)P.box_w * D - X;
    X += (int64_t)P.tx * D;
    Y += (int64_t)P.ty * D;
    AX[a0 + v] = X;
    AY[a0 + v] = Y;
    bx0 = min(bx0, X); bx1 = max(bx1, X); by0 = min(by0, Y); by1 = max(by1, Y);
  }
  bx0 = wmin64(bx0); bx1 = wmax64(bx1); by0 = wmin64(by0); by1 = wmax64(by1);
  if (lane == 0) {
    VChart r;
    r.D = D;
    r.x0 = (int32_t)floordiv(bx0, D);
    r.y0 = (int32_t)floordiv(by0, D);
    const int64_t nx = ceildiv(bx1, D) - r.x0, ny = ceildiv(by1, D) - r.y0;
    r.nx = nx > 0 && ny > 0 ? (int32_t)nx : 0;
    r.ny = nx > 0 && ny > 0 ? (int32_t)ny : 0;
    r.area2 = s2 < 0 ? -s2 : s2;
    const double q = (double)P.scale_den / (double)P.scale_num;
    r.inv_s2 = q * q;
    ch[c] = r;
  }
}

// V2: exclusive scans of the plain and dilated bbox areas, stretch sums; one
// CTA, fixed reduction order (deterministic).
__global__ void __launch_bounds__(1024)
v_scan_kernel(const VChart* __restrict__ ch, int32_t n, int32_t g, int64_t* ofs_d, int64_t* tot,
              double* sums) {
  __shared__ int64_t sd[1024];
  __shared__ double sa[1024], sw[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int per = (n + T - 1) / T;
  const int b = min(n, t * per), e = min(n, b + per);
  int64_t acc = 0;
  double A = 0.0, Wt = 0.0;
  for (int c = b; c < e; c++) {
    const VChart r = ch[c];
    acc += r.nx > 0 ? (int64_t)(r.nx + 2 * g) * (r.ny + 2 * g) : 0;
    A += (double)r.area2;
    Wt += (double)r.area2 * r.inv_s2;
  }
  sd[t] = acc;
  sa[t] = A;
  sw[t] = Wt;
  __syncthreads();
  for (int o = 1; o < T; o <<= 1) {  // Hillis-Steele inclusive scan
    const int64_t v = t >= o ? sd[t - o] : 0;
    __syncthreads();
    sd[t] += v;
    __syncthreads();
  }
  int64_t run = sd[t] - acc;
  for (int c = b; c < e; c++) {
    const VChart r = ch[c];
    ofs_d[c] = run;
    run += r.nx > 0 ? (int64_t)(r.nx + 2 * g) * (r.ny + 2 * g) : 0;
  }
  if (t == T - 1) {
    ofs_d[n] = sd[t];
    tot[0] = sd[t];
  }
  for (int o = T / 2; o; o >>= 1) {  // fixed-shape tree: deterministic
    __syncthreads();
    if (t < o) { sa[t] += sa[t + o]; sw[t] += sw[t + o]; }
  }
  if (t == 0) { sums[0] = sa[0]; sums[1] = sw[0]; }
}

// chart owning flat index f: largest c with ofs[c] <= f (charts with empty
// boxes have ofs[c] == ofs[c + 1] and are skipped by the upper-bound search)
__device__ __forceinline__ int owner(const int64_t* ofs, int32_t n, int64_t f) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ofs[mid] <= f) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// exact: does segment p->q meet the open box (x0, x1) x (y0, y1)?
// Parametrize p + t (q - p), t in [0, 1].  Per axis with d != 0 the box is the
// open t-interval between (a - p)/d and (b - p)/d; with d == 0 the coordinate
// must lie strictly inside.  Non-empty iff every lower bound is below every
// upper bound (strictly unless both are the closed 0 / 1).
__device__ bool seg_meets_open_box(int64_t px, int64_t py, int64_t qx, int64_t qy, int64_t x0,
                                   int64_t x1, int64_t y0, int64_t y1) {
  const int64_t dx = qx - px, dy = qy - py;
  // lower / upper numerators over a positive per-axis denominator
  i128 lx = 0, ux = 0, ly = 0, uy = 0;
  int64_t ex = 1, ey = 1;
  bool hx = false, hy = false;
  if (dx == 0) {
    if (!(x0 < px && px < x1)) return false;
  } else {
    hx = true;
    ex = dx > 0 ? dx : -dx;
    lx = dx > 0 ? (i128)(x0 - px) : (i128)(px - x1);
    ux = dx > 0 ? (i128)(x1 - px) : (i128)(px - x0);
  }
  if (dy == 0) {
    if (!(y0 < py && py < y1)) return false;
  } else {
    hy = true;
    ey = dy > 0 ? dy : -dy;
    ly = dy > 0 ? (i128)(y0 - py) : (i128)(py - y1);
    uy = dy > 0 ? (i128)(y1 - py) : (i128)(py - y0);
  }
  // lower bounds {0 (closed), lx/ex, ly/ey (open)}; upper {1 (closed), ux/ex, uy/ey (open)}
  if (hx) {
    if (!(lx < ex)) return false;       // lx/ex < 1
    if (!(0 < ux)) return false;        // 0 < ux/ex
    if (hy) {
      if (!(lx * ey < uy * ex)) return false;
      if (!(ly * ex < ux * ey)) return false;
    }
  }
  if (hy) {
    if (!(ly < ey)) return false;
    if (!(0 < uy)) return false;
  }
  return true;  // lx < ux and ly < uy hold since x0 < x1, y0 < y1
}

// even-odd test of the point (cx, cy) / 2 against the polygon scaled by 2;
// the point is a texel centre, which lies off every edge when no edge meets
// the open texel square.
__device__ bool centre_inside(const int64_t* X, const int64_t* Y, int nv, int64_t cx2,
                              int64_t cy2) {
  bool in = false;
  int64_t px = 2 * X[nv - 1], py = 2 * Y[nv - 1];
  for (int v = 0; v < nv; v++) {
    const int64_t qx = 2 * X[v], qy = 2 * Y[v];
    if ((py > cy2) != (qy > cy2)) {
      // crossing x = px + (cy2 - py) (qx - px) / (qy - py); centre left of it?
      const i128 num = (i128)(cy2 - py) * (qx - px);
      const i128 lhs = (i128)(cx2 - px) * (qy - py);
      if (qy > py ? lhs < num : lhs > num) in = !in;
    }
    px = qx;
    py = qy;
  }
  return in;
}

__device__ __forceinline__ void mark2(uint32_t* grid, int64_t t) {
  uint32_t* w = grid + (t >> 4);
  const uint32_t b = 1u << (2 * (t & 15));
  const uint32_t old = atomicOr(w, b);
  if (old & b) atomicOr(w, b << 1);
}

// V3: coverage of every dilated-bbox texel of every chart.
__global__ void __launch_bounds__(kThreads)
v_raster_kernel(const int32_t* __restrict__ start, int32_t n, const VChart* __restrict__ ch,
                const int64_t* __restrict__ ofs, const int64_t* __restrict__ tot,
                const int64_t* __restrict__ AX, const int64_t* __restrict__ AY, int32_t g,
                int32_t W, int32_t H, uint8_t* mask, uint32_t* grid0,
                unsigned long long* oob) {
  const int64_t total = *tot;
  uint32_t my_oob = 0;
  for (int64_t f = (int64_t)blockIdx.x * kThreads + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * kThreads) {
    const int c = owner(ofs, n, f);
    const VChart r = ch[c];
    const int64_t loc = f - ofs[c];
    const int32_t sx = r.nx + 2 * g;
    const int32_t i = (int32_t)(loc % sx) - g, j = (int32_t)(loc / sx) - g;
    bool hit = false;
    if (i >= 0 && j >= 0 && i < r.nx && j < r.ny) {
      const int32_t a0 = start[c], nv = start[c + 1] - a0;
      const int64_t* X = AX + a0;
      const int64_t* Y = AY + a0;
      const int64_t xa = (int64_t)(r.x0 + i) * r.D, xb = xa + r.D;
      const int64_t ya = (int64_t)(r.y0 + j) * r.D, yb = ya + r.D;
      int64_t px = X[nv - 1], py = Y[nv - 1];
      for (int v = 0; v < nv && !hit; v++) {
        const int64_t qx = X[v], qy = Y[v];
        const bool skip = (px <= xa && qx <= xa) || (px >= xb && qx >= xb) ||
                          (py <= ya && qy <= ya) || (py >= yb && qy >= yb);
        if (!skip) hit = seg_meets_open_box(px, py, qx, qy, xa, xb, ya, yb);
        px = qx;
        py = qy;
      }
      if (!hit) hit = centre_inside(X, Y, nv, 2 * xa + r.D, 2 * ya + r.D);
      if (hit) {
        const int32_t ax = r.x0 + i, ay = r.y0 + j;
        if (ax < 0 || ay < 0 || ax >= W || ay >= H) {
          my_oob++;
          hit = false;  // only in-atlas coverage is dilated (it is what gets rendered)
        } else {
          mark2(grid0, (int64_t)ay * W + ax);
        }
      }
    }
    mask[f] = hit ? 1 : 0;
  }
  for (int o = 16; o; o >>= 1) my_oob += __shfl_xor_sync(~0u, my_oob, o);
  if ((threadIdx.x & 31) == 0 && my_oob) atomicAdd(oob, (unsigned long long)my_oob);
}

// V4: row pass of the Chebyshev dilation (OR over dx in [-g, g]).
__global__ void __launch_bounds__(kThreads)
v_dilate_rows(int32_t n, const VChart* __restrict__ ch, const int64_t* __restrict__ ofs,
              const int64_t* __restrict__ tot, int32_t g, const uint8_t* __restrict__ mask,
              uint8_t* rows) {
  const int64_t total = *tot;
  for (int64_t f = (int64_t)blockIdx.x * kThreads + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * kThreads) {
    const int c = owner(ofs, n, f);
    const VChart r = ch[c];
    const int64_t loc = f - ofs[c];
    const int32_t sx = r.nx + 2 * g;
    const int32_t i = (int32_t)(loc % sx);
    const int64_t row0 = f - i;
    uint8_t v = 0;
    for (int32_t d = max(0, i - g); d <= min(sx - 1, i + g) && !v; d++) v = mask[row0 + d];
    rows[f] = v;
  }
}

// V5: column pass; dilated texels inside the atlas feed the gutter counters.
__global__ void __launch_bounds__(kThreads)
v_dilate_cols(int32_t n, const VChart* __restrict__ ch, const int64_t* __restrict__ ofs,
              const int64_t* __restrict__ tot, int32_t g, int32_t W, int32_t H,
              const uint8_t* __restrict__ rows, uint32_t* gridg) {
  const int64_t total = *tot;
  for (int64_t f = (int64_t)blockIdx.x * kThreads + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * kThreads) {
    const int c = owner(ofs, n, f);
    const VChart r = ch[c];
    const int64_t loc = f - ofs[c];
    const int32_t sx = r.nx + 2 * g, sy = r.ny + 2 * g;
    const int32_t i = (int32_t)(loc % sx), j = (int32_t)(loc / sx);
    uint8_t v = 0;
    for (int32_t d = max(0, j - g); d <= min(sy - 1, j + g) && !v; d++)
      v = rows[ofs[c] + (int64_t)d * sx + i];
    if (!v) continue;
    const int32_t ax = r.x0 - g + i, ay = r.y0 - g + j;
    if (ax < 0 || ay < 0 || ax >= W || ay >= H) continue;
    mark2(gridg, (int64_t)ay * W + ax);
  }
}

// V6: covered = seen-once bits of grid0, overlap = seen-twice bits of grid0,
// gutter = seen-twice bits of gridg.
__global__ void __launch_bounds__(kThreads)
v_count_kernel(const uint32_t* __restrict__ grid0, const uint32_t* __restrict__ gridg,
               int64_t words, unsigned long long* out) {
  uint32_t cov = 0, ov = 0, gu = 0;
  for (int64_t k = (int64_t)blockIdx.x * kThreads + threadIdx.x; k < words;
       k += (int64_t)gridDim.x * kThreads) {
    const uint32_t a = grid0[k], b = gridg[k];
    cov += __popc(a & 0x55555555u);
    ov += __popc(a & 0xaaaaaaaau);
    gu += __popc(b & 0xaaaaaaaau);
  }
  for (int o = 16; o; o >>= 1) {
    cov += __shfl_xor_sync(~0u, cov, o);
    ov += __shfl_xor_sync(~0u, ov, o);
    gu += __shfl_xor_sync(~0u, gu, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (cov) atomicAdd(out + 0, (unsigned long long)cov);
    if (ov) atomicAdd(out + 1, (unsigned long long)ov);
    if (gu) atomicAdd(out + 2, (unsigned long long)gu);
  }
}

template <class T>
cudaError_t grow(T** p, int64_t* cap, int64_t need) {
  if (need <= *cap) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  const int64_t c = need + need / 4 + 64;
  cudaError_t e = cudaMalloc((void**)p, sizeof(T) * (size_t)c);
  if (e == cudaSuccess) *cap = c;
  return e;
}

}  // namespace

void Validator::release() {
  cudaFree(xy); cudaFree(start); cudaFree(pl); cudaFree(AX); cudaFree(AY); cudaFree((void*)ch);
  cudaFree(ofs); cudaFree(mask); cudaFree(rows); cudaFree(grid); cudaFree(misc);
  cudaFreeHost(h_misc);
  *this = Validator{};
}

int Validator::run(const float* xy_in, const int32_t* start_in, int32_t n, float rx, float ry,
                   int32_t W, int32_t H, int32_t g, const tabi_placement* pl_in, bool on_device,
                   int64_t nverts, cudaStream_t s, tabi_validation* out, int* launches,
                   std::string* err) {
  auto ck = [&](cudaError_t e) {
    if (e != cudaSuccess && err) *err = cudaGetErrorString(e);
    return e == cudaSuccess;
  };
  *launches = 0;
  VChart* chp = (VChart*)ch;
  const bool okg = ck(grow(&AX, &cap_ax, nverts)) && ck(grow(&AY, &cap_ay, nverts)) &&
                   ck(grow(&chp, &cap_ch, (int64_t)n)) && ck(grow(&ofs, &cap_ofs, (int64_t)n + 1));
  ch = chp;
  if (!okg) return TABI_ECUDA;
  if (!misc) {
    if (!ck(cudaMalloc(&misc, 256)) || !ck(cudaMallocHost(&h_misc, 256))) return TABI_ECUDA;
  }
  const float* d_xy = xy_in;
  const int32_t* d_start = start_in;
  const tabi_placement* d_pl = pl_in;
  if (!on_device) {
    if (!ck(grow(&xy, &cap_xy, 2 * nverts)) || !ck(grow(&start, &cap_s, (int64_t)n + 1)) ||
        !ck(grow(&pl, &cap_pl, (int64_t)n)))
      return TABI_ECUDA;
    ck(cudaMemcpyAsync(xy, xy_in, sizeof(float) * 2 * nverts, cudaMemcpyHostToDevice, s));
    ck(cudaMemcpyAsync(start, start_in, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, s));
    ck(cudaMemcpyAsync(pl, pl_in, sizeof(tabi_placement) * n, cudaMemcpyHostToDevice, s));
    d_xy = xy;
    d_start = start;
    d_pl = pl;
  }
  // misc layout: [0] bad chart (int32), [8] total (int64), [16] sums (2 double),
  // [32] oob, [40] covered, [48] overlap, [56] gutter (u64)
  int32_t* bad = (int32_t*)misc;
  int64_t* tot = (int64_t*)(misc + 8);
  double* sums = (double*)(misc + 16);
  unsigned long long* cnt = (unsigned long long*)(misc + 32);
  ck(cudaMemsetAsync(misc, 0, 64, s));
  ck(cudaMemsetAsync(bad, 0x7f, 4, s));
  v_coords_kernel<<<(n * 32 + kThreads - 1) / kThreads, kThreads, 0, s>>>(
      d_xy, d_start, n, rx, ry, d_pl, AX, AY, chp, bad);
  v_scan_kernel<<<1, 1024, 0, s>>>(chp, n, g, ofs, tot, sums);
  *launches += 2;
  ck(cudaMemcpyAsync(h_misc, misc, 32, cudaMemcpyDeviceToHost, s));
  if (!ck(cudaStreamSynchronize(s))) return TABI_ECUDA;
  const int32_t hbad = *(int32_t*)h_misc;
  if (hbad != 0x7f7f7f7f) {
    out->bad_chart = hbad;
    return TABI_EINVAL;
  }
  const int64_t total = *(int64_t*)(h_misc + 8);
  const double* hs = (const double*)(h_misc + 16);
  const int64_t words = ((int64_t)W * H + 15) / 16;
  if (!ck(grow(&mask, &cap_m, total)) || !ck(grow(&rows, &cap_r, total)) ||
      !ck(grow(&grid, &cap_g, 2 * words)))
    return TABI_ECUDA;
  uint32_t* grid0 = grid;
  uint32_t* gridg = grid + words;
  ck(cudaMemsetAsync(grid, 0, sizeof(uint32_t) * 2 * words, s));
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int blocks_t = (int)std::min<int64_t>((total + kThreads - 1) / kThreads, (int64_t)sms * 8);
  const int blocks_w = (int)std::min<int64_t>((words + kThreads - 1) / kThreads, (int64_t)sms * 8);
  if (total > 0) {
    v_raster_kernel<<<blocks_t, kThreads, 0, s>>>(d_start, n, chp, ofs, tot, AX, AY, g, W, H, mask,
                                                  grid0, cnt);
    v_dilate_rows<<<blocks_t, kThreads, 0, s>>>(n, chp, ofs, tot, g, mask, rows);
    v_dilate_cols<<<blocks_t, kThreads, 0, s>>>(n, chp, ofs, tot, g, W, H, rows, gridg);
    *launches += 3;
  }
  if (words > 0) {
    v_count_kernel<<<std::max(blocks_w, 1), kThreads, 0, s>>>(grid0, gridg, words, cnt + 1);
    *launches += 1;
  }
  ck(cudaMemcpyAsync(h_misc + 32, misc + 32, 32, cudaMemcpyDeviceToHost, s));
  if (!ck(cudaStreamSynchronize(s))) return TABI_ECUDA;
  const unsigned long long* hc = (const unsigned long long*)(h_misc + 32);
  out->oob = (int64_t)hc[0];
  out->covered = (int64_t)hc[1];
  out->overlap = (int64_t)hc[2];
  out->gutter = (int64_t)hc[3];
  out->occupancy = (W > 0 && H > 0) ? (double)out->covered / ((double)W * (double)H) : 0.0;
  out->l2_stretch = hs[0] > 0 ? sqrt(hs[1] / hs[0]) : 0.0;
  out->bad_chart = -1;
  return TABI_OK;
}

}  // namespace tabi
