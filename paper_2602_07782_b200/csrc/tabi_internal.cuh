// tabi_internal.cuh -- device helpers and the context layout of the CUDA path.
//
// Integer model: coordinates are snapped once to
// 1/256 texel (int32), all later geometry is exact int64 / int128 with
// directed rounding, so the GPU reproduces the paper's method bit for bit
// under the readings listed in DESIGN.md.  Nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tabi.h"

typedef __int128 i128;

#define TABI_KMAX 64
#define TABI_QMAX (1 << 24)
#define TABI_UNITS 256

namespace tabi {

// ---- exact division with directed rounding (divisor > 0) -------------------
__host__ __device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b) != 0 && a < 0) q--;
  return q;
}
__host__ __device__ __forceinline__ int64_t ceildiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b) != 0 && a > 0) q++;
  return q;
}
__device__ __forceinline__ i128 floordiv128(i128 a, i128 b) {
  i128 q = a / b;
  if ((a % b) != 0 && a < 0) q--;
  return q;
}
__device__ __forceinline__ i128 ceildiv128(i128 a, i128 b) {
  i128 q = a / b;
  if ((a % b) != 0 && a > 0) q++;
  return q;
}

// Exact floor/ceil division from a double-precision estimate plus integer
// correction (no emulated 64/128-bit divide).  Exact for any operands: the
// correction loops run until the remainder is in [0, b); with |a/b| < 2^50
// the estimate is already within one unit so they run at most once or twice.
// 1/b to ~1 ulp without the fp64 divide routine: MUFU.RCP in fp32, then two
// Newton steps in fp64.  Only ever used as an estimate that an exact integer
// correction follows, so its last bits do not matter.
__device__ __forceinline__ double rcp_approx(double b) {
  double r = (double)__frcp_rn((float)b);
  r = r * (2.0 - b * r);
  r = r * (2.0 - b * r);
  return r;
}
__device__ __forceinline__ int64_t fdiv_fast(int64_t a, int64_t b) {
  int64_t q = (int64_t)floor((double)a * rcp_approx((double)b));
  int64_t r = a - q * b;
  while (r < 0) { q--; r += b; }
  while (r >= b) { q++; r -= b; }
  return q;
}
__device__ __forceinline__ int64_t cdiv_fast(int64_t a, int64_t b) { return -fdiv_fast(-a, b); }
__device__ __forceinline__ double i128_to_double(i128 a) {
  return (double)(int64_t)(a >> 64) * 18446744073709551616.0 + (double)(uint64_t)a;
}
__device__ __forceinline__ int64_t fdiv_fast128(i128 a, i128 b) {
  int64_t q = (int64_t)floor(i128_to_double(a) * rcp_approx(i128_to_double(b)));
  i128 r = a - (i128)q * b;
  while (r < 0) { q--; r += b; }
  while (r >= b) { q++; r -= b; }
  return q;
}
__device__ __forceinline__ int64_t cdiv_fast128(i128 a, i128 b) { return -fdiv_fast128(-a, b); }
// 64 x 64 -> 128-bit signed product with two native multiplies.
__device__ __forceinline__ i128 mul_wide(int64_t a, int64_t b) {
  const uint64_t lo = (uint64_t)a * (uint64_t)b;
  const int64_t hi = __mul64hi(a, b);
  return (i128)(((unsigned __int128)(uint64_t)hi << 64) | lo);
}
// floor(a / b), b > 0 fits int64, from a precomputed reciprocal 1/b and an
// exact integer correction.
__device__ __forceinline__ int64_t fdiv_rcp(i128 a, int64_t b, double rcp) {
  int64_t q = (int64_t)floor(i128_to_double(a) * rcp);
  i128 r = a - mul_wide(q, b);
  while (r < 0) { q--; r += b; }
  while (r >= (i128)b) { q++; r -= b; }
  return q;
}
__device__ __forceinline__ int64_t cdiv_rcp(i128 a, int64_t b, double rcp) {
  return -fdiv_rcp(-a, b, rcp);
}
// floor(a / b) clamped to [-2^40, 2^40] (callers compare it with small indices).
__device__ __forceinline__ int64_t fdiv_clamp128(i128 a, i128 b) {
  const double est = i128_to_double(a) * rcp_approx(i128_to_double(b));
  if (est > 1099511627776.0) return 1099511627776LL;
  if (est < -1099511627776.0) return -1099511627776LL;
  return fdiv_fast128(a, b);
}

// f(i) = floor((A + i*B) / D) for i >= 0 as an int64 progression:
// A = qA*D + rA, B = qB*D + rB (0 <= rA, rB < D), so
// f(i) = qA + i*qB + floor((rA + i*rB) / D) with a small int64 numerator.
struct LinDiv {
  int64_t qA, rA, qB, rB, D;
  double rcp;
};
__device__ __forceinline__ LinDiv make_lindiv(i128 A, int64_t B, int64_t D) {
  LinDiv L;
  L.D = D;
  L.rcp = rcp_approx((double)D);
  L.qA = fdiv_fast128(A, (i128)D);
  L.rA = (int64_t)(A - mul_wide(L.qA, D));
  L.qB = fdiv_fast(B, D);
  L.rB = B - L.qB * D;
  return L;
}
// floor(a / b) for int64 a, b > 0 from a precomputed reciprocal (exact).
__device__ __forceinline__ int64_t fdiv_r64(int64_t a, int64_t b, double rcp) {
  int64_t q = (int64_t)floor((double)a * rcp);
  int64_t r = a - q * b;
  while (r < 0) { q--; r += b; }
  while (r >= b) { q++; r -= b; }
  return q;
}
// floor(a / b) for i128 a and i128 b > 0 from a reciprocal; result clamped to
// [-2^40, 2^40] when clamp is set (for index comparisons).
__device__ __forceinline__ int64_t fdiv_r128(i128 a, i128 b, double rcp, bool clamp) {
  const double est = floor(i128_to_double(a) * rcp);
  if (clamp) {
    if (est > 1099511627776.0) return 1099511627776LL;
    if (est < -1099511627776.0) return -1099511627776LL;
  }
  int64_t q = (int64_t)est;
  i128 r = a - (i128)q * b;
  while (r < 0) { q--; r += b; }
  while (r >= b) { q++; r -= b; }
  return q;
}
// Start a running evaluation at i: v = f(i), r = (rA + i*rB) mod D; then
// lindiv_step moves to i + 1 with one add and one conditional carry (rB < D).
// rA + i rB is formed in 128 bits: in the hybrid tail the scale denominator is
// 2^20 x 256, so D = S x 2^28 reaches 2^58 and i rB overflows int64 from a
// few dozen cells on (the prefix tail's large charts, found by the random
// parity sweep tests/test_gpu_fuzz.py).
__device__ __forceinline__ void lindiv_start(const LinDiv& L, int64_t i, int64_t& v, int64_t& r) {
  // int64 whenever i D < 2^62 (then rA + i rB < 2^63): every sequential-mode
  // scale, and the tail's small charts
  const uint64_t iD = (uint64_t)i * (uint64_t)L.D;
  if (i >= 0 && __umul64hi((uint64_t)i, (uint64_t)L.D) == 0 && iD < (1ull << 62)) {
    const int64_t N = L.rA + i * L.rB;
    int64_t t = (int64_t)((double)N * L.rcp);
    int64_t rr = N - t * L.D;
    while (rr < 0) { t--; rr += L.D; }
    while (rr >= L.D) { t++; rr -= L.D; }
    v = L.qA + i * L.qB + t;
    r = rr;
    return;
  }
  const i128 N = (i128)L.rA + (i128)i * L.rB;
  int64_t t = (int64_t)(i128_to_double(N) * L.rcp);
  i128 rr = N - (i128)t * L.D;
  while (rr < 0) { t--; rr += L.D; }
  while (rr >= L.D) { t++; rr -= L.D; }
  v = L.qA + i * L.qB + t;
  r = (int64_t)rr;
}
__device__ __forceinline__ int64_t lindiv_eval(const LinDiv& L, int64_t i) {
  int64_t v, r;
  lindiv_start(L, i, v, r);
  return v;
}

// ---- warp reductions (full warp) ------------------------------------------
__device__ __forceinline__ int32_t warp_max(int32_t v) {
  return __reduce_max_sync(0xffffffffu, v);
}
__device__ __forceinline__ int32_t warp_min(int32_t v) {
  return __reduce_min_sync(0xffffffffu, v);
}
__device__ __forceinline__ int32_t warp_sum(int32_t v) {
  return __reduce_add_sync(0xffffffffu, v);
}
__device__ __forceinline__ int64_t warp_max64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t > v ? t : v;
  }
  return v;
}
__device__ __forceinline__ int64_t warp_min64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t < v ? t : v;
  }
  return v;
}
__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ i128 warp_sum128(i128 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t lo = (uint64_t)v, hi = (uint64_t)(v >> 64);
    lo = __shfl_xor_sync(0xffffffffu, lo, o);
    hi = __shfl_xor_sync(0xffffffffu, hi, o);
    v += (i128)(((unsigned __int128)hi << 64) | lo);
  }
  return v;
}
// inclusive warp scans
__device__ __forceinline__ int32_t warp_incl_sum(int32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
__device__ __forceinline__ int32_t warp_incl_min(int32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = t < v ? t : v;
  }
  return v;
}
__device__ __forceinline__ int32_t warp_incl_max(int32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = t > v ? t : v;
  }
  return v;
}

// Q30 rotation table for the 8 OBB angles theta_j = j*pi/16, j = 0..7
// ("8 evenly spaced rotations in the interval [0, 7pi/16]").
// Rounded cos/sin * 2^30 written as literals so no libm result enters the
// geometry (reading R6).
__constant__ const int64_t kQC[8] = {1073741824LL, 1053110176LL, 992008094LL, 892783698LL,
                                      759250125LL,  596538995LL,  410903207LL, 209476638LL};
__constant__ const int64_t kQS[8] = {0LL,          209476638LL, 410903207LL, 596538995LL,
                                      759250125LL,  892783698LL, 992008094LL, 1053110176LL};

// Footprint entries are two uint16 packed in a uint32: columns (Dtop | Dbot << 16),
// rows (Dleft | Dright << 16).
__device__ __forceinline__ int32_t lo16(uint32_t v) { return (int32_t)(v & 0xffffu); }
__device__ __forceinline__ int32_t hi16(uint32_t v) { return (int32_t)(v >> 16); }

// D15 CannotMoveAbove for the pair (a, b), a before b in the sorted line and
// b's footprint starting `delta` columns right of a's (top-aligned).  Moving a
// up by t puts a's row r beside b's row r - t < r; a is locked iff for some
// r >= 1, a's right edge there passes b's left edge of some row above r
// ("no rectangular segment ... is below a segment of the other chart's
// boundary").  Requires Hda >= Hdb (sorted by height).  Whole warp calls.
__device__ __forceinline__ void warp_locks(const uint32_t* ra, const uint32_t* rb, int32_t Hda,
                                           int32_t Hdb, int32_t delta, int lane, bool& la,
                                           bool& lb) {
  bool xa = false, xb = false;
  int32_t cmin_b = INT32_MAX, cmax_a = INT32_MIN;
  for (int base = 0; base < Hdb; base += 32) {
    const int r = base + lane;
    const bool valid = r < Hdb;
    const int32_t lb_r = valid ? lo16(rb[r]) : INT32_MAX;
    const int32_t ra_r = valid ? hi16(ra[r]) : INT32_MIN;
    const int32_t imin = warp_incl_min(lb_r, lane);
    const int32_t imax = warp_incl_max(ra_r, lane);
    int32_t emin = __shfl_up_sync(0xffffffffu, imin, 1);
    int32_t emax = __shfl_up_sync(0xffffffffu, imax, 1);
    if (lane == 0) { emin = INT32_MAX; emax = INT32_MIN; }
    emin = min(emin, cmin_b);
    emax = max(emax, cmax_a);
    if (valid && r >= 1) {
      if (emin != INT32_MAX && ra_r > delta + emin) xa = true;
      if (emax != INT32_MIN && delta + lb_r < emax) xb = true;
    }
    cmin_b = min(cmin_b, __shfl_sync(0xffffffffu, imin, 31));
    cmax_a = max(cmax_a, __shfl_sync(0xffffffffu, imax, 31));
  }
  for (int r = Hdb + lane; r < Hda; r += 32) {
    if (r >= 1 && hi16(ra[r]) > delta + cmin_b) xa = true;
  }
  la = __any_sync(0xffffffffu, xa);
  lb = __any_sync(0xffffffffu, xb);
}

// ---- device-side per-pack state -------------------------------------------
// Proxy SoA (final pose).  Slices: sl[c * 4k + {0: top, 1: bot, 2: left, 3: right} * k + j]
struct Proxies {
  int32_t* w;
  int32_t* h;
  int64_t* area2;
  int32_t* xmin;
  int32_t* ymin;
  uint8_t* pose;     // bit0 rot90, bit1 fx, bit2 fy
  uint8_t* prerot;   // pre-rotation angle index (TABI_F_PREROTATE), 0 = none
  int32_t* sl;
  int32_t* obb_j;
  int64_t* obb;      // [c*4 + {umin, umax, vmin, vmax}]
};

// Fused-kernel raster tiles (prep_kernel / k_pack.cu): at most
// kFusedTileCharts sorted charts and about kFusedTileCells footprint cells.
#ifndef TABI_FUSED_RG
#define TABI_FUSED_RG 1
#endif
constexpr int kFusedGroups = TABI_FUSED_RG;  // independent raster groups per CTA
constexpr int kFusedTileCharts = 64 / kFusedGroups;
#ifndef TABI_TILE_CELLS
#define TABI_TILE_CELLS 4096
#endif
constexpr int kFusedTileCells = TABI_TILE_CELLS / kFusedGroups;
#ifndef TABI_HEAD_CELLS
// quarter-size tiles for the first 16 K footprint cells (the tallest charts,
// which the first rows need): with a narrow first wave most raster CTAs are
// free at the start, and the first row's wait drops (C3: -10 us; measured
// 16 K < 32 K < 64 K < 128 K; with 16 candidates per wave it did not pay)
#define TABI_HEAD_CELLS 16384
#endif
constexpr int kFusedHeadCells = TABI_HEAD_CELLS;  // quarter-size tiles below this prefix

struct Status {       // device-side status block, copied back once per pack
  int32_t bad_chart;  // INT32_MAX if none
  int32_t capacity;   // bit 0: footprint slots, bit 1: lock-pair lists exceed the buffers
                      // (grow + retry); bit 2: a vertex range beyond max_vertices
  int32_t winner;     // winning m (0 = none)
  int32_t cols_total, rows_total;
  int32_t pad[3];
  int32_t work_next;  // fused kernel: raster work-queue head
  int32_t ntiles;     // fused kernel: raster tiles (prep_kernel)
  int32_t win_j;      // fused, sequential mode: smallest wave slot that succeeded
  int32_t b0;         // wave 0's candidate slots in use (prep_kernel; <= B)
  int32_t wave;       // current candidate wave (reset_kernel / wave_ctl_kernel advance it)
  int32_t tail_cnt;   // hybrid tail kernels: CTAs done (the last one decides the rounds loop)
  int32_t rounds_run; // hybrid tail: re-layout rounds run by the graph's rounds loop
  int32_t st_pad2;
  int32_t wmax, hmax; // largest chart width / height (units; prep_kernel): a
                      // candidate whose scaled largest chart exceeds the dilated
                      // atlas fails at once (cand_too_big)
  unsigned long long work_pack;  // K4 frontline column visits (push + score + commit)
  unsigned long long work_prof;  // K3 footprint entries (sum over candidates of Wd + Hd)
  unsigned long long atot_lo, atot_hi;  // total 2 x area (int128) for D25 / D26
  // fused-kernel trace (%globaltimer ns): [0] first CTA start, [1] last raster
  // group end, [2] last packer end, [3] packer ns spent waiting for tiles,
  // [4] raster ns spent waiting for the left tile, [5] tiles rasterized
  unsigned long long tr[6];
  // K4 row-phase time (SM cycles, thread 0 of every packer, summed; only in a
  // -DTABI_PHASE_TRACE build): knee update,
  // fold, HC choice + lock pairs, push, Alg. 1, score, select + commit, FindKnee
  unsigned long long ph[10];  // + [8] push staging, [9] commit staging
  // fused rasterizer per-item phases (SM cycles, summed; trace build only):
  // queue fetch, footprints (tile_raster), large charts, accounting,
  // boundary arrivals, pair offsets, publish
  unsigned long long rph[8];
  // first-row timeline of wave slot 0 (%globaltimer, trace build): [0] its
  // tile 0 footprints done, [1] tile 0 published, [2] packer 0's first fold
  // unblocked, [3] packer 0's first row done
  unsigned long long tfirst[8];  // + [4..7] its tile 0: fetched, setup, pairs start, pairs end
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Per-candidate result record (mirrors tabi_cand_dbg).
struct Cand {
  int32_t success, score, rows, knees_found, knee_rows, prefix_rows, p, evaluated;
  int32_t switched_at, reserved;
  unsigned long long apre_lo, apre_hi;  // 2 x area of the prefix-folded tail (D25), int128
};

// Batch mode (tabi_pack_many): the outcome of one atlas.
struct AtlasRes {
  int32_t winner;      // largest successful m, 0 = none (NO_FIT or not decided)
  int32_t rows, knees_found, knee_rows;
  int32_t evaluated;   // candidates evaluated (top-down from the area bound)
  int32_t done;        // 1 once decided (success or every candidate failed)
  int32_t next_r;      // next rank (m = m_hi - r) to issue
  int32_t issued;      // ranks issued (the initial in-flight ones + continuations)
  int32_t completed;   // ranks finished (failed, won, or not needed)
  int32_t pad;
  uint32_t fail[8];    // bit r: rank r failed (r < 256)
};
constexpr int kManyMaxCharts = 2048;  // per atlas in the device batch (one-CTA sort)

// Hybrid prefix tail state per candidate (DESIGN.md §1 A12).
enum { TAIL_NONE = 0, TAIL_LAYOUT = 1, TAIL_READY = 2, TAIL_FAIL = 3 };
struct TailBufs {
  int32_t* state;   // [M] TAIL_*
  int32_t* r0;      // [M] first prefix-folded sorted position
  int32_t* p;       // [M] intermediate scale numerator over 2^20
  int32_t* iter;    // [M] layout adjustments made
  int32_t* fsave;   // [M][fstride] frontline at the switch
  int32_t fstride;
};

struct PackParams {
  int32_t n, k, M, g, W, H, Wp, Hp;
  uint32_t flags;
  int32_t B;                  // candidates per wave: m = m_hi - wave * B - j, j < B (wave:
                              // Status::wave)
  int32_t t_opt;              // effective t_opt (basis points of H), 0 = sequential only
  int32_t mode;               // K4: 0 sequential rows (may switch), 1 prefix rows
  int32_t tail;               // K3 / K3b: 1 = rasterize tail charts at p / 2^20
  int32_t early;              // fused, sequential mode: candidate-major raster order and
                              // early exit once a higher candidate has succeeded
  int64_t col_cap, row_cap;   // per-candidate footprint slot capacity (entries)
  TailBufs T;
};

// Candidate j of the current wave (0 if below 1).  m_hi = st->pad[2] is the
// area bound computed by prep_kernel.
// Candidate of wave slot j: wave 0 evaluates the b0 candidates m_hi, m_hi - 1,
// ... (b0 <= B, chosen by prep_kernel); wave w >= 1 the next B below.
// The wave index lives in the status block (Status::wave): the device-side
// wave loop advances it without a host round trip.
__host__ __device__ __forceinline__ int wave_m(const PackParams& pp, int32_t wave, int32_t m_hi,
                                               int32_t b0, int j) {
  if (wave == 0 && j >= b0) return 0;
  const int m = m_hi - (wave == 0 ? 0 : b0 + (wave - 1) * pp.B) - j;
  return m >= 1 ? m : 0;
}

// Does candidate m's largest chart exceed the dilated atlas?  The rasterizers'
// per-chart test (cand_bad: ceil(w m / (M 256)) + 2g > W' or the same for h)
// on the largest width and height, which decides it for every chart.
__device__ __forceinline__ bool cand_too_big(const PackParams& pp, const Status* st, int m) {
  const int64_t SC = (int64_t)pp.M * TABI_UNITS;
  const int64_t ws = ((int64_t)st->wmax * m + SC - 1) / SC;
  const int64_t hs = ((int64_t)st->hmax * m + SC - 1) / SC;
  return ws + 2 * pp.g > pp.Wp || hs + 2 * pp.g > pp.Hp;
}

}  // namespace tabi

// Launch wrappers (defined in the .cu files)
namespace tabi {
// Batch mode (tabi_pack_many): charts of na atlases back to back, atlas a owning
// the global charts [abase[a], abase[a+1]) with status block st[a] and
// resolution res[2a..2a+1] (nullptr: rx, ry).  abase == nullptr: one atlas.
struct AtlasMap {
  const int32_t* abase;
  int32_t na;
  const float* res;
  int32_t c0;  // first chart of this launch (charts [c0, n)); 0 for one launch
};
// max_v: capacity of qx/qy; a chart's vertex range outside [0, max_v) sets
// Status::capacity bit 2 (-> TABI_ECAPACITY) before anything is written
void launch_proxies(const float* xy, const int32_t* start, int32_t n, float rx, float ry, int k,
                    uint32_t flags, int32_t* qx, int32_t* qy, int64_t max_v, Proxies P, Status* st,
                    cudaStream_t s, AtlasMap am = AtlasMap{nullptr, 1, nullptr},
                    int64_t nverts = 0, bool skip_wh = false);
// w, h, area2 and the status words alone (single pack, no prerotation): the
// order's inputs, so the sort can overlap proxy_kernel (skip_wh) on a second
// stream
void launch_sizes(const float* xy, const int32_t* start, int32_t n, float rx, float ry,
                  int64_t max_v, Proxies P, Status* st, cudaStream_t s);  // total vertices if known (picks the lane group)
// Status / per-wave state reset (k_sort.cu), one launch; see reset_kernel.
void launch_reset(Status* st, int mode, Cand* cands, int32_t* t_state, int32_t* cand_bad, int M,
                  int32_t* rdy, int64_t nrdy, cudaStream_t s);
// D9 sort: bitonic in smem (N <= 4096), rank sort (N <= 2^17), else radix.
// Returns the number of kernels launched.
int launch_sort(const Proxies& P, int32_t n, uint64_t* keys, uint64_t* keys2, int32_t* perm,
                int32_t* perm2, const Status* st, cudaStream_t s,
                const uint64_t** sorted_keys = nullptr);
// N <= 2048 and no TABI_SORT knob: sort + prep in one launch (returns false otherwise)
bool launch_sort_prep(const Proxies& P, int32_t* perm, const PackParams& pp, int32_t* colofs,
                      int32_t* rowofs, int32_t* hsorted, int32_t* tstart, int32_t* tix, Status* st,
                      int32_t* rdy, cudaStream_t s);  // rdy: zeroed for the fused wave, or nullptr
// Multi-CTA slot layout (prep_multi_kernel): decoupled look-back state,
// never reset (flags carry an epoch).  <= kPrepMaxBlocks blocks of 4096
// sorted positions (N <= 2^17).
constexpr int kPrepMaxBlocks = 32;
struct PrepSync {
  int32_t epoch;
  int32_t f1[kPrepMaxBlocks], f2[kPrepMaxBlocks];
  int32_t c[kPrepMaxBlocks], r[kPrepMaxBlocks], t[kPrepMaxBlocks];
  int32_t wm[kPrepMaxBlocks], hm[kPrepMaxBlocks];
  unsigned long long alo[kPrepMaxBlocks], ahi[kPrepMaxBlocks];
};
void launch_prep(const Proxies& P, const int32_t* perm, const PackParams& pp, int32_t* colofs,
                 int32_t* rowofs, int32_t* hsorted, int32_t* tstart, int32_t* tix, Status* st,
                 int32_t* rdy, cudaStream_t s, const uint64_t* sorted_keys = nullptr, PrepSync* ps = nullptr);
void launch_profiles(const Proxies& P, const int32_t* perm, const PackParams& pp,
                     const int32_t* colofs, const int32_t* rowofs, int16_t* dcol, int16_t* drow,
                     int32_t* wd, int32_t* hd, int32_t* cand_bad, int32_t* big_list, Status* st,
                     cudaStream_t s);
void launch_offsets(const PackParams& pp, const int32_t* colofs, const int32_t* rowofs,
                    const int16_t* drow, const int32_t* wd, const int32_t* hd, int32_t* off,
                    uint8_t* lockbits, const int32_t* cand_bad, const Status* st,
                    cudaStream_t s);
void launch_pack(const PackParams& pp, const int32_t* colofs, const int32_t* rowofs,
                 const uint32_t* dcol, const uint32_t* drow, const int32_t* wd, const int32_t* hd,
                 const int32_t* off, const uint8_t* lockbits, const int32_t* hsorted,
                 const int32_t* cand_bad, int32_t* scratch, int64_t pair_cap, int32_t* X,
                 int32_t* Y, uint8_t* mir, Cand* cands, Status* st, cudaStream_t s);
// Fused persistent wave kernel (k_pack.cu): K3 + K3b + K4 in one cooperative
// launch.  fused_grid = co-resident CTAs (0 if cooperative launch is
// unsupported); the ready flags are [B][n] (at most n tiles).
int fused_grid(int device);
bool fused_fits(int k);
cudaError_t launch_fused(int grid, const Proxies& P, const int32_t* perm, const PackParams& pp,
                         const int32_t* colofs, const int32_t* rowofs, uint32_t* dcol,
                         uint32_t* drow, int32_t* wd, int32_t* hd, int32_t* off, uint8_t* lockbits,
                         const int32_t* hsorted, int32_t* cand_bad, int32_t* rdy,
                         const int32_t* tstart, const int32_t* tix, int32_t* scratch,
                         int64_t pair_cap, int32_t* X, int32_t* Y, uint8_t* mir, Cand* cands,
                         Status* st, cudaStream_t s);
// Batch mode (tabi_pack_many): sort + slot layout per atlas
// (one CTA each), queue reset, and the persistent pack kernel in which each
// CTA takes (atlas, candidate) items -- rasterizes the atlas's footprints at
// that scale, computes its pair offsets and runs Alg. 4, all in its own
// buffers -- pushing the next lower candidate on failure (top-down search,
// exact) and scattering the placements on success.
struct ManyArgs {
  Proxies P;                      // global (chart-indexed)
  const int32_t* abase;           // [A + 1] first global chart of each atlas
  const int32_t* perm;            // per atlas at abase[a]: sorted position -> atlas-local chart
  const int32_t* colofs;
  const int32_t* rowofs;
  const int32_t* hsorted;
  Status* sts;                    // [A]
  AtlasRes* res;                  // [A]
  tabi_placement* out;            // global (chart-indexed)
  int32_t* q;                     // [qcap] items a | r << 20 (r = candidates below m_hi), -1 empty
  int32_t* qctl;                  // head, tail, atlases pending
  int32_t qcap;
  // per-CTA buffers, CTA g at g * (stride)
  uint32_t* dcol;                 // [G][col_cap]
  uint32_t* drow;                 // [G][row_cap]
  int32_t* wd;                    // [G][nmax] (also hd, off, X, Y below)
  int32_t* hd;
  int32_t* off;
  uint8_t* lock;
  int32_t* scratch;               // [G][6 nmax + 3 pair_cap]
  int32_t* X;
  int32_t* Y;
  uint8_t* mir;
  Cand* cands;                    // [G]
  int32_t* cand_bad;              // [G]
  unsigned long long* cycles;     // [3] SM cycles summed over items: raster, pairs, packer;
                                  // then [G][2] per CTA: start, end of its last item (ns)
  int64_t* area;                  // [G][nmax] lazy mode: 2 x polygon area by sorted position
  int32_t lazy;                   // rasterize on demand inside the packer (many_lazy_ok)
  int32_t inflight;               // ranks of one atlas in flight at once (K >= 1)
  int32_t carry;                  // a CTA whose rank failed continues with the next rank
                                  // (else the next rank goes to the queue's tail)
  int32_t spec;                   // > 1: idle CTAs start ranks of undecided atlases, up to
                                  // this many in flight per atlas (carry mode only)
  const int32_t* order;           // [E] the batched atlases, LPT order
  int32_t E;
  int32_t early_fail;             // lazy mode: the row-end area test (R8)
  int32_t ahead;                  // lazy mode: positions rasterized beyond the fold's need
  int32_t nmax;
  int64_t pair_cap;
};
// queue: ranks 0 .. inflight - 1 of every atlas, interleaved in `order`
void launch_many_reset(Status* sts, AtlasRes* res, int32_t A, const int32_t* order, int32_t E,
                       int32_t* q, int32_t qcap, int32_t* qctl, int32_t inflight, cudaStream_t s);
void launch_many_sort_prep(const Proxies& P, const int32_t* abase, int32_t A, int32_t* perm,
                          const PackParams& pp, int32_t* colofs, int32_t* rowofs, int32_t* hsorted,
                          int32_t* tstart, int32_t* tix, Status* sts, cudaStream_t s);
int many_grid(int device);  // persistent CTAs (one per SM)
// the lazy batch raster fits the packer's staging buffer at this k and W' (and g <= 2)
bool many_lazy_ok(int k, int g, int Wp);
// k_floor.cu: packer building-block latencies in ns (tabi_debug_latency_floor)
int latency_floor(int device, double* out8);
cudaError_t launch_many(int grid, const PackParams& pp, const ManyArgs& a, cudaStream_t s);
// K5; with use_h it also sets the graph's wave-loop condition (see
// select_kernel)
void launch_select(const PackParams& pp, const Proxies& P, const int32_t* perm, const int32_t* wd,
                   const int32_t* hd, const int32_t* X, const int32_t* Y, const uint8_t* mir,
                   const Cand* cands, tabi_placement* out, Status* st, cudaStream_t s,
                   cudaGraphConditionalHandle h = 0, int use_h = 0);
}  // namespace tabi

namespace tabi {
// (with use_h: the last CTA sets the rounds loop's condition h -- "some
// candidate still needs a re-layout round")
void launch_tail_prepare(const PackParams& pp, const int32_t* perm, const int64_t* area2,
                         const int32_t* wd, const int32_t* off, int32_t* scratch, int64_t pair_cap,
                         Cand* cands, Status* st, cudaStream_t s, cudaGraphConditionalHandle h = 0,
                         int use_h = 0);
void launch_tail_layout(const PackParams& pp, const int32_t* wd, const int32_t* off,
                        int32_t* scratch, int64_t pair_cap, Status* st, cudaStream_t s,
                        cudaGraphConditionalHandle h = 0, int use_h = 0);
}  // namespace tabi

#include <atomic>
#include <string>
namespace tabi {
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute is per device, and batch mode drives several devices from
// several host threads.
inline void ensure_dyn_smem(const void* fn, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done.fetch_or(bit, std::memory_order_acq_rel);
}

// N3 GPU validator (k_validate.cu): device scratch that grows on demand and
// persists across calls on one context.
struct Validator {
  float* xy = nullptr;
  int32_t* start = nullptr;
  tabi_placement* pl = nullptr;
  int64_t *AX = nullptr, *AY = nullptr;
  void* ch = nullptr;
  int64_t* ofs = nullptr;
  uint8_t *mask = nullptr, *rows = nullptr;
  uint32_t* grid = nullptr;
  unsigned char* misc = nullptr;
  unsigned char* h_misc = nullptr;  // pinned
  int64_t cap_xy = 0, cap_s = 0, cap_pl = 0, cap_ax = 0, cap_ay = 0, cap_ch = 0, cap_ofs = 0;
  int64_t cap_m = 0, cap_r = 0, cap_g = 0;
  void release();
  // counts for n charts placed by pl (host or device pointers); returns a
  // tabi_status; fills out (bad_chart on EINVAL) and the launch count
  int run(const float* xy, const int32_t* start, int32_t n, float rx, float ry, int32_t W,
          int32_t H, int32_t g, const tabi_placement* pl, bool on_device, int64_t nverts,
          cudaStream_t s, tabi_validation* out, int* launches, std::string* err);
};
}  // namespace tabi
