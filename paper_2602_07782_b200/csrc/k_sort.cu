// k_sort.cu -- K2: decreasing-height order + footprint slot layout.
//
// P:139 "sorted in decreasing height order"; ties by the wider chart, then by
// chart index.  Three exact paths by N:
//   N <= 2048    bitonic network in registers of one CTA (shuffles below
//                distance 64) on the packed unique keys (h, w, index);
//   N <= 2^17    chunked: every CTA sorts 2048 (key, index) pairs the same way,
//                then each element's rank = its rank in its chunk + binary-
//                search counts in the other chunks, and a scatter;
//                (test knobs: the smem bitonic for N <= 4096 and an O(N^2)
//                rank count, both exact);
//   larger       STABLE LSD radix sort on ((hmax - h) << bw) | (wmax - w) with
//                the chart index as payload, one CTA of 1024 threads: per-tile
//                digit ranks from warp match masks + per-warp digit counts.
//
// prep_kernel then lays out, per sorted position, the int16 footprint slots
// every candidate uses (slot = footprint at the largest scale, clipped to the
// dilated atlas) with a block-wide exclusive scan, and flags the pack for a
// capacity retry if the slots do not fit the current buffers.
#include <cstdlib>
#include <cstring>

#include "tabi_internal.cuh"

namespace tabi {
namespace {

constexpr int kT = 1024;
constexpr int kW = kT / 32;

__device__ __forceinline__ int bits_of(uint64_t v) { return v == 0 ? 0 : 64 - __clzll(v); }

__global__ void __launch_bounds__(kT, 1)
sort_kernel(const int32_t* __restrict__ hh, const int32_t* __restrict__ ww, int32_t n, uint64_t* keys,
            uint64_t* keys2, int32_t* perm, int32_t* perm2, const Status* st) {
  __shared__ int32_t wcnt[kW][256];
  __shared__ int32_t base[256];
  __shared__ int32_t run[256];
  __shared__ int32_t tot[256];
  __shared__ int32_t red[2][kW];
  if (st->bad_chart != INT32_MAX) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int32_t hm = 0, wm = 0;
  for (int i = tid; i < n; i += kT) {
    hm = max(hm, hh[i]);
    wm = max(wm, ww[i]);
  }
  hm = warp_max(hm);
  wm = warp_max(wm);
  if (lane == 0) { red[0][wid] = hm; red[1][wid] = wm; }
  __syncthreads();
  hm = 0;
  wm = 0;
  for (int i = 0; i < kW; i++) { hm = max(hm, red[0][i]); wm = max(wm, red[1][i]); }
  const int bw = bits_of((uint64_t)wm);
  const int nbits = bits_of((uint64_t)hm) + bw;
  for (int i = tid; i < n; i += kT) {
    keys[i] = ((uint64_t)(hm - hh[i]) << bw) | (uint64_t)(wm - ww[i]);
    perm[i] = i;
  }
  __syncthreads();
  uint64_t* kin = keys;
  uint64_t* kout = keys2;
  int32_t* pin = perm;
  int32_t* pout = perm2;
  const int passes = (nbits + 7) / 8;
  for (int p = 0; p < passes; p++) {
    const int sh = 8 * p;
    for (int d = tid; d < 256; d += kT) { base[d] = 0; run[d] = 0; }
    __syncthreads();
    for (int i = tid; i < n; i += kT) atomicAdd(&base[(kin[i] >> sh) & 255], 1);
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the 256-bin histogram, 8 bins per lane
      int32_t v[8], s = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) { v[q] = base[lane * 8 + q]; s += v[q]; }
      int32_t ex = warp_incl_sum(s, lane) - s;
#pragma unroll
      for (int q = 0; q < 8; q++) { base[lane * 8 + q] = ex; ex += v[q]; }
    }
    for (int t0 = 0; t0 < n; t0 += kT) {
      const int i = t0 + tid;
      const bool valid = i < n;
      const uint64_t key = valid ? kin[i] : 0;
      const int32_t pv = valid ? pin[i] : 0;
      const int d = valid ? (int)((key >> sh) & 255) : 256;
      for (int q = tid; q < kW * 256; q += kT) (&wcnt[0][0])[q] = 0;
      __syncthreads();
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      if (valid && rank == 0) wcnt[wid][d] = __popc(peers);
      __syncthreads();
      for (int dd = tid; dd < 256; dd += kT) {  // exclusive prefix over warps (stable)
        int32_t s = 0;
        for (int w = 0; w < kW; w++) {
          const int32_t cnt = wcnt[w][dd];
          wcnt[w][dd] = s;
          s += cnt;
        }
        tot[dd] = s;
      }
      __syncthreads();
      if (valid) {
        const int32_t dest = base[d] + run[d] + wcnt[wid][d] + rank;
        kout[dest] = key;
        pout[dest] = pv;
      }
      __syncthreads();
      for (int dd = tid; dd < 256; dd += kT) run[dd] += tot[dd];
    }
    __syncthreads();
    uint64_t* tk = kin; kin = kout; kout = tk;
    int32_t* tp = pin; pin = pout; pout = tp;
  }
  if (pin != perm) {
    for (int i = tid; i < n; i += kT) perm[i] = pin[i];
  }
}

// Block-wide exclusive scan of two int32 values (one per thread), kT threads.
__device__ __forceinline__ void block_scan2(int32_t a, int32_t b, int32_t& ea, int32_t& eb,
                                            int32_t& ta, int32_t& tb, int32_t (*sh)[kW + 1]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t ia = warp_incl_sum(a, lane), ib = warp_incl_sum(b, lane);
  if (lane == 31) { sh[0][wid] = ia; sh[1][wid] = ib; }
  __syncthreads();
  if (wid == 0) {
    int32_t va = sh[0][lane], vb = sh[1][lane];
    int32_t xa = warp_incl_sum(va, lane), xb = warp_incl_sum(vb, lane);
    sh[0][lane] = xa - va;
    sh[1][lane] = xb - vb;
    if (lane == 31) { sh[0][kW] = xa; sh[1][kW] = xb; }
  }
  __syncthreads();
  ea = sh[0][wid] + ia - a;
  eb = sh[1][wid] + ib - b;
  ta = sh[0][kW];
  tb = sh[1][kW];
  __syncthreads();
}

// ---- small and medium N: comparison sorts on unique keys -------------------
// D9 order (h desc, w desc, index asc) as one unsigned key per chart; w, h <
// 2^26 units (|coordinate| <= 2^24), so (2^26-1-h, 2^26-1-w, index) packs in
// 64 bits for N <= 4096 and the packed keys are unique: any correct sort gives
// the stable order.
#ifndef TABI_B0_HYBRID
#define TABI_B0_HYBRID 4
#endif
#ifndef TABI_B0_FILL
#define TABI_B0_FILL 55  // wave 0 reaches down to the scale filling this % of the atlas
#endif
constexpr int kBitonicMax = 4096;
constexpr int kRankMax = 1 << 17;
constexpr int kRankT = 256;   // rank sort: keys i per block
constexpr int kRankJ = 1024;  // rank sort: keys j per block (shared-memory tile)

__device__ __forceinline__ uint64_t order_key(int32_t h, int32_t w) {
  return ((uint64_t)(0x3ffffffu - (uint32_t)h) << 26) | (uint64_t)(0x3ffffffu - (uint32_t)w);
}

// N <= 4096: bitonic sort of the packed keys in shared memory, one CTA.
__global__ void __launch_bounds__(kT, 1)
bitonic_kernel(const int32_t* __restrict__ hh, const int32_t* __restrict__ ww, int32_t n,
               int32_t* perm, const Status* st) {
  __shared__ uint64_t key[kBitonicMax];
  if (st->bad_chart != INT32_MAX) return;
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = threadIdx.x; i < P; i += kT)
    key[i] = i < n ? (order_key(hh[i], ww[i]) << 12) | (uint64_t)i : ~0ull;
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += kT) {
        const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const uint64_t a = key[lo], b = key[hi];
        if ((a > b) == ((lo & size) == 0)) { key[lo] = b; key[hi] = a; }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += kT) perm[i] = (int32_t)(key[i] & 0xfffu);
}

// N <= 2048: the same bitonic network with each thread holding elements 2t
// and 2t + 1 in registers: the compare-exchange stages of element distance
// <= 32 are warp shuffles (partner thread t ^ (stride / 2), same slot) with no
// barrier; only distances >= 64 go through shared memory.
// Returns the sorted keys in shared memory (valid after a barrier): a
// following slot layout reads each position's (h, w, chart) from them instead
// of a dependent perm -> proxy load chain.
__device__ __forceinline__ const uint64_t* bitonic_reg_body(const int32_t* __restrict__ hh,
                                                            const int32_t* __restrict__ ww,
                                                            int32_t n, int32_t* perm) {
  __shared__ uint64_t key[2 * kT];
  const int t = threadIdx.x;
  uint64_t v[2];
#pragma unroll
  for (int s = 0; s < 2; s++) {
    const int i = 2 * t + s;
    v[s] = i < n ? (order_key(hh[i], ww[i]) << 12) | (uint64_t)i : ~0ull;
  }
  int P = 2;
  while (P < n) P <<= 1;  // sorting [0, P) suffices: the rest are sentinels
  for (int size = 2; size <= P; size <<= 1) {
    int stride = size >> 1;
    if (stride >= 64) {
      key[2 * t] = v[0];
      key[2 * t + 1] = v[1];
      __syncthreads();
      for (; stride >= 64; stride >>= 1) {
        const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const uint64_t a = key[lo], b = key[hi];
        if ((a > b) == ((lo & size) == 0)) { key[lo] = b; key[hi] = a; }
        __syncthreads();
      }
      v[0] = key[2 * t];
      v[1] = key[2 * t + 1];
    }
    const bool asc = ((2 * t) & size) == 0;
    for (; stride >= 2; stride >>= 1) {
      const int d = stride >> 1;
      const bool keep_min = (((2 * t) & stride) == 0) == asc;
#pragma unroll
      for (int s = 0; s < 2; s++) {
        const uint64_t p = __shfl_xor_sync(0xffffffffu, v[s], d);
        v[s] = keep_min ? (p < v[s] ? p : v[s]) : (p > v[s] ? p : v[s]);
      }
    }
    if ((v[0] > v[1]) == asc) {  // stride 1: the thread's own pair
      const uint64_t x = v[0];
      v[0] = v[1];
      v[1] = x;
    }
  }
#pragma unroll
  for (int s = 0; s < 2; s++) {
    const int i = 2 * t + s;
    if (i < n) perm[i] = (int32_t)(v[s] & 0xfffu);
    key[i] = v[s];  // (own slots only: the last smem pass read just these)
  }
  return key;
}

__global__ void __launch_bounds__(kT, 1)
bitonic_reg_kernel(const int32_t* __restrict__ hh, const int32_t* __restrict__ ww, int32_t n,
                   int32_t* perm, const Status* st) {
  if (st->bad_chart != INT32_MAX) return;
  bitonic_reg_body(hh, ww, n, perm);
}

// 2048 < N <= 2^17: each CTA sorts a chunk of 2048 (key, index) pairs with the
// register bitonic network above, then every element's final position is its
// rank in its own chunk plus, for every other chunk, the number of pairs
// below it (binary searches, 16 chunks at a time in lockstep so their loads
// overlap).  Pairs are unique (the index), so the ranks are a permutation.
constexpr int kChunk = 2 * kT;
__device__ __forceinline__ bool pair_lt(uint64_t ka, int32_t ia, uint64_t kb, int32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(kT, 1)
chunk_sort_kernel(const int32_t* __restrict__ hh, const int32_t* __restrict__ ww, int32_t n,
                  uint64_t* ck, int32_t* ci, const Status* st) {
  __shared__ uint64_t key[kChunk];
  __shared__ int32_t idx[kChunk];
  if (st->bad_chart != INT32_MAX) return;
  const int t = threadIdx.x, base = blockIdx.x * kChunk, cn = min(kChunk, n - base);
  uint64_t v[2];
  int32_t x[2];
#pragma unroll
  for (int s = 0; s < 2; s++) {
    const int i = 2 * t + s;
    v[s] = i < cn ? order_key(hh[base + i], ww[base + i]) : ~0ull;
    x[s] = i < cn ? base + i : INT32_MAX;
  }
  int P = 2;
  while (P < cn) P <<= 1;
  for (int size = 2; size <= P; size <<= 1) {
    int stride = size >> 1;
    if (stride >= 64) {
      key[2 * t] = v[0]; key[2 * t + 1] = v[1];
      idx[2 * t] = x[0]; idx[2 * t + 1] = x[1];
      __syncthreads();
      for (; stride >= 64; stride >>= 1) {
        const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const uint64_t a = key[lo], b = key[hi];
        const int32_t ia = idx[lo], ib = idx[hi];
        if (pair_lt(b, ib, a, ia) == ((lo & size) == 0)) {
          key[lo] = b; key[hi] = a;
          idx[lo] = ib; idx[hi] = ia;
        }
        __syncthreads();
      }
      v[0] = key[2 * t]; v[1] = key[2 * t + 1];
      x[0] = idx[2 * t]; x[1] = idx[2 * t + 1];
      __syncthreads();
    }
    const bool asc = ((2 * t) & size) == 0;
    for (; stride >= 2; stride >>= 1) {
      const int d = stride >> 1;
      const bool keep_min = (((2 * t) & stride) == 0) == asc;
#pragma unroll
      for (int s = 0; s < 2; s++) {
        const uint64_t p = __shfl_xor_sync(0xffffffffu, v[s], d);
        const int32_t px = __shfl_xor_sync(0xffffffffu, x[s], d);
        const bool plt = pair_lt(p, px, v[s], x[s]);
        if (keep_min == plt) { v[s] = p; x[s] = px; }
      }
    }
    if (pair_lt(v[1], x[1], v[0], x[0]) == asc) {
      const uint64_t tv = v[0]; v[0] = v[1]; v[1] = tv;
      const int32_t tx = x[0]; x[0] = x[1]; x[1] = tx;
    }
  }
#pragma unroll
  for (int s = 0; s < 2; s++) {
    const int i = 2 * t + s;
    if (i < cn) { ck[base + i] = v[s]; ci[base + i] = x[s]; }
  }
}

// Each block holds kT consecutive pairs of one chunk; the other chunks pass
// through shared memory one after another (the next one's loads are issued
// before the current one is searched), and every pair adds its lower bound in
// each of them -- an 11-step binary search in shared memory instead of global
// loads.
__global__ void __launch_bounds__(kT)
chunk_rank_kernel(const uint64_t* __restrict__ ck, const int32_t* __restrict__ ci, int32_t n,
                  int32_t* perm, uint64_t* skeys, const Status* st) {
  __shared__ uint64_t sk[kChunk];
  __shared__ int32_t si[kChunk];
  if (st->bad_chart != INT32_MAX) return;
  const int e = blockIdx.x * kT + threadIdx.x;
  const bool valid = e < n;
  const uint64_t k = valid ? ck[e] : 0ull;
  const int32_t i = valid ? ci[e] : 0;
  const int c = (int)(blockIdx.x * kT) / kChunk;  // (kChunk = 2 kT: one chunk per block)
  const int nother = (n + kChunk - 1) / kChunk - 1;
  int rank = e - c * kChunk;
  uint64_t rk[2];
  int32_t ri[2];
  auto fetch = [&](int q) {  // the q-th chunk other than c, padded with sentinels
    const int b = (q < c ? q : q + 1) * kChunk, len = min(kChunk, n - b);
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int x = threadIdx.x + u * kT;
      rk[u] = x < len ? ck[b + x] : ~0ull;
      ri[u] = x < len ? ci[b + x] : INT32_MAX;
    }
  };
  if (nother > 0) fetch(0);
  for (int q = 0; q < nother; q++) {
    __syncthreads();  // (the previous chunk's searches are done)
#pragma unroll
    for (int u = 0; u < 2; u++) {
      sk[threadIdx.x + u * kT] = rk[u];
      si[threadIdx.x + u * kT] = ri[u];
    }
    __syncthreads();
    if (q + 1 < nother) fetch(q + 1);
    // number of pairs below (k, i): binary lifting over the 2,048 sorted slots
    int pos = 0;
#pragma unroll
    for (int stp = kChunk / 2; stp >= 1; stp >>= 1)
      if (pair_lt(sk[pos + stp - 1], si[pos + stp - 1], k, i)) pos += stp;
    if (pair_lt(sk[pos], si[pos], k, i)) pos++;  // (pos <= kChunk - 1 here)
    rank += pos;
  }
  if (valid) {
    perm[rank] = i;
    skeys[rank] = k;  // the keys in sorted order: the slot layout reads (h, w) from them
  }
}

// N <= 2^17: rank of key i = #{j : (key_j, j) < (key_i, i)}, counted over a 2-D
// grid of (i block, j tile) with one atomicAdd per thread and tile, then a
// scatter perm[rank[i]] = i.
__global__ void __launch_bounds__(kRankT)
rank_count_kernel(const int32_t* __restrict__ hh, const int32_t* __restrict__ ww, int32_t n,
                  int32_t* rank, const Status* st) {
  __shared__ uint64_t tile[kRankJ];
  if (st->bad_chart != INT32_MAX) return;
  const int i = blockIdx.x * kRankT + threadIdx.x;
  const int j0 = blockIdx.y * kRankJ, m = min(kRankJ, n - j0);
  for (int q = threadIdx.x; q < m; q += kRankT) tile[q] = order_key(hh[j0 + q], ww[j0 + q]);
  __syncthreads();
  if (i >= n) return;
  const uint64_t ki = order_key(hh[i], ww[i]);
  const int lim = min(m, i - j0);  // tile entries with index j < i (ties count)
  int cnt = 0;
  int q = 0;
  for (; q < lim; q++) cnt += tile[q] <= ki;
  for (; q < m; q++) cnt += tile[q] < ki;
  if (cnt) atomicAdd(&rank[i], cnt);
}

__global__ void rank_scatter_kernel(const int32_t* __restrict__ rank, int32_t n, int32_t* perm,
                                    const Status* st) {
  if (st->bad_chart != INT32_MAX) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) perm[rank[i]] = i;
}

__device__ __forceinline__ void st_release_flag(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire_flag(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Fused-kernel raster tiles: consecutive sorted charts with tile key
// floor(slot prefix / kFusedTileCells) + floor(s / kFusedTileCharts) --
// non-decreasing in s, so equal keys are runs of <= kFusedTileCharts charts
// holding about kFusedTileCells footprint cells (the tallest charts come first
// and get small tiles, so their tiles are not the long pole every packer waits
// on); the first kFusedHeadCells cells (the tallest charts, which every packer
// needs first) are cut into quarter-size tiles so the first rows start early.
__device__ __forceinline__ int32_t fused_tile_id(int64_t cum, int s) {
  const int64_t q4 = kFusedTileCells / 4;
  const int64_t cell_key = cum < kFusedHeadCells
                               ? cum / q4
                               : kFusedHeadCells / q4 + (cum - kFusedHeadCells) / kFusedTileCells;
  return (int32_t)(cell_key + s / kFusedTileCharts);
}

// Scale bounds from the total polygon area (warp 0, every lane gets them).
// R2: sequential mode only -- every chart keeps m/M, so a successful
// (overlap-free, in-bounds) packing needs (m/M)^2 A <= W H; in units (2*area,
// 1/256 texel): m^2 * A2 <= 2 * 65536 * W * H * M^2.  In hybrid mode the prefix
// tail's intermediate downscale (D24) can make a candidate above that bound
// succeed, so the search starts at M.  m_hi = the largest m <= M passing it
// (monotone in m: lane l of round r tests m = M - 32 r - l; the lowest passing
// lane wins).  Wave 0's width b0: the candidates from m_hi down to the scale
// at which the charts would fill TABI_B0_FILL % of the atlas (TSS sets pack at
// ~60 %) -- below that a success is unlikely, and a narrower first wave leaves
// the top candidate's chain with less contention.  Later waves take B each
// and the wave loop's stopping rule (select_kernel; hybrid mode: the V bound
// of D25) is unchanged, so the result is the exhaustive search's either way.
// m_lo = 1 + the largest m' < m_hi below the fill level (monotone), else 1.
__device__ __forceinline__ void scale_bounds(const PackParams& pp, i128 tot, int lane, int& m_hi,
                                             int& b0) {
  const i128 rhs = (i128)2 * 65536 * pp.W * pp.H * (i128)pp.M * pp.M;
  m_hi = 0;
  for (int base = 0; base < pp.M && m_hi == 0; base += 32) {  // (uniform)
    const int m = pp.M - base - lane;
    const unsigned ok =
        __ballot_sync(0xffffffffu, m >= 1 && (pp.t_opt > 0 || (i128)m * m * tot <= rhs));
    if (ok) m_hi = pp.M - base - (__ffs(ok) - 1);
  }
  b0 = pp.B;
  if (pp.B > 2 && m_hi >= 1) {
    int m_lo = 0;
    for (int base = 1; base < m_hi && m_lo == 0; base += 32) {  // (uniform)
      const int mp = m_hi - base - lane;
      const unsigned lowr = __ballot_sync(
          0xffffffffu, mp >= 1 && (i128)100 * mp * mp * tot < (i128)TABI_B0_FILL * rhs);
      if (lowr) m_lo = m_hi - base - (__ffs(lowr) - 1) + 1;
    }
    if (m_lo == 0) m_lo = 1;
    b0 = min(pp.B, max(2, m_hi - m_lo + 1));
    // hybrid mode: the prefix tail's downscale absorbs the overflow that
    // fails a sequential candidate, so the top candidates usually succeed
    // and then win (D25) -- a first wave of TABI_B0_HYBRID; the device
    // loop's V bound decides whether lower ones still need a wave
    if (pp.t_opt > 0) b0 = min(b0, TABI_B0_HYBRID);
  }
}

// Footprint slots: column slot of sorted position s = min(ceil(w/256) + 2g, W'),
// row slot = min(ceil(h/256) + 2g, H') -- the footprint at the largest scale
// (m = M, scale 1) bounds every candidate's (w_s is monotone in m).
__device__ __forceinline__ void prep_body(const int32_t* __restrict__ hh,
                                          const int32_t* __restrict__ ww, const int64_t* area2,
                                          const int32_t* perm, const PackParams& pp, int32_t* colofs,
                                          int32_t* rowofs, int32_t* hsorted, int32_t* tstart,
                                          int32_t* tix, Status* st, int32_t* rdy,
                                          const uint64_t* skey = nullptr, int skey_shift = 12) {
  __shared__ int32_t sh[2][kW + 1];
  __shared__ unsigned long long asum[2][kW];
  __shared__ int32_t ext_max[2][kW];
  // Area bound on the candidate scales: the packed charts are disjoint and
  // inside the atlas, so (m/M)^2 * sum(area) <= W*H for any candidate that can
  // succeed; in units (2*area, 1/256 texel): m^2 * A2 <= 2 * 65536 * W * H * M^2.
  {
    i128 a = 0;
    int32_t wm = 0, hm = 0;
    for (int i = threadIdx.x; i < pp.n; i += kT) {
      a += area2[i];
      wm = max(wm, ww[i]);
      hm = max(hm, hh[i]);
    }
    a = warp_sum128(a);
    wm = warp_max(wm);
    hm = warp_max(hm);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
      asum[0][wid] = (unsigned long long)(uint64_t)a;
      asum[1][wid] = (unsigned long long)(uint64_t)(a >> 64);
      ext_max[0][wid] = wm;
      ext_max[1][wid] = hm;
    }
    __syncthreads();
    if (wid == 0) {  // warp 0: the totals, then the scale bounds by ballots
      i128 tot = (i128)(((unsigned __int128)asum[1][lane] << 64) | asum[0][lane]);
      tot = warp_sum128(tot);
      const int32_t wmx = warp_max(ext_max[0][lane]), hmx = warp_max(ext_max[1][lane]);
      int m_hi, b0;
      scale_bounds(pp, tot, lane, m_hi, b0);
      if (lane == 0) {
      st->wmax = wmx;
      st->hmax = hmx;
      st->pad[2] = m_hi;
      st->b0 = b0;
      st->atot_lo = (unsigned long long)(uint64_t)tot;
      st->atot_hi = (unsigned long long)(uint64_t)(tot >> 64);
      }
    }
  }
  // Chunks of kE * kT sorted positions: the slot sizes are loaded coalesced
  // into shared memory, then thread t runs over its kE consecutive positions
  // with running sums -- two block-wide scans per chunk (slot prefixes, then
  // tile starts) instead of two per kT positions.
  constexpr int kE = 4;
  constexpr int kCh = kE * kT;
  __shared__ uint16_t scw[kCh], srh[kCh];  // slot sizes <= W', H'
  static_assert(TABI_MAX_ATLAS_SIDE + 2 * 64 <= 65535, "slot sizes fit 16 bits (gutter <= 64)");
  __shared__ int32_t last_id;
  auto hw_at = [&](int s, int32_t& h, int32_t& w) {
    if (skey) {  // the sorted key holds (h, w): no dependent global loads
      const uint64_t k = skey[s] >> skey_shift;  // order_key(h, w) [<< 12 | index]
      h = (int32_t)(0x3ffffffu - (uint32_t)((k >> 26) & 0x3ffffffu));
      w = (int32_t)(0x3ffffffu - (uint32_t)(k & 0x3ffffffu));
    } else {
      const int c = perm[s];
      w = ww[c];
      h = hh[c];
    }
  };
  // Fused-kernel raster tiles: consecutive sorted charts with tile key
  // floor(slot prefix / kFusedTileCells) + floor(s / kFusedTileCharts) --
  // non-decreasing in s, so equal keys are runs of <= kFusedTileCharts
  // charts holding about kFusedTileCells footprint cells (the tallest
  // charts come first and get small tiles, so their tiles are not the long
  // pole every packer waits on).
  // the first kFusedHeadCells cells (the tallest charts, which every packer
  // needs first) are cut into quarter-size tiles so the first rows start early
  auto tile_id = [&](int64_t cum, int s) -> int32_t { return fused_tile_id(cum, s); };
  int32_t carry_c = 0, carry_r = 0, carry_t = 0, prev_id = -1;  // prev_id: the tile of the
                                                                 // previous chunk's last position
  for (int base = 0; base < pp.n; base += kCh) {
    const int cn = min(kCh, pp.n - base);
#pragma unroll
    for (int u = 0; u < kE; u++) {
      const int x = u * kT + threadIdx.x;
      if (x < cn) {
        int32_t h, w;
        hw_at(base + x, h, w);
        const int64_t wd = ceildiv(w, TABI_UNITS) + 2 * pp.g;
        const int64_t hd = ceildiv(h, TABI_UNITS) + 2 * pp.g;
        scw[x] = (uint16_t)(wd < pp.Wp ? wd : pp.Wp);
        srh[x] = (uint16_t)(hd < pp.Hp ? hd : pp.Hp);
        hsorted[base + x] = h;
      }
    }
    __syncthreads();
    const int q0 = min(cn, (int)threadIdx.x * kE), q1 = min(cn, q0 + kE);
    int32_t sc = 0, sr = 0;
    for (int q = q0; q < q1; q++) {
      sc += scw[q];
      sr += srh[q];
    }
    int32_t ec, er, tc, tr;
    block_scan2(sc, sr, ec, er, tc, tr, sh);
    ec += carry_c;
    er += carry_r;
    int32_t pid = q0 == 0 ? prev_id
                  : q0 < q1 ? tile_id((int64_t)ec + er - scw[q0 - 1] - srh[q0 - 1], base + q0 - 1)
                            : 0;
    int32_t nf = 0;
    {
      int64_t cum = (int64_t)ec + er;
      int32_t p = pid;
      for (int q = q0; q < q1; q++) {
        const int32_t id = tile_id(cum, base + q);
        nf += id != p;
        p = id;
        cum += scw[q] + srh[q];
      }
    }
    int32_t ef, e2, tf, t2;
    block_scan2(nf, 0, ef, e2, tf, t2, sh);
    {
      int32_t c = ec, r = er, tt = carry_t + ef - 1;
      for (int q = q0; q < q1; q++) {
        const int s = base + q;
        const int32_t id = tile_id((int64_t)c + r, s);
        if (id != pid) tstart[++tt] = s;
        colofs[s] = c;
        rowofs[s] = r;
        tix[s] = tt;
        c += scw[q];
        r += srh[q];
        pid = id;
      }
      if (q0 < q1 && q1 == cn) last_id = pid;
    }
    carry_c += tc;
    carry_r += tr;
    carry_t += tf;
    __syncthreads();
    prev_id = last_id;
  }
  if (threadIdx.x == 0) {
    st->cols_total = carry_c;
    st->rows_total = carry_r;
    st->ntiles = carry_t;
    tstart[carry_t] = pp.n;
    // +4: the TMA bulk copy of a row window rounds its end up to 16 bytes
    if ((int64_t)carry_c + 4 > pp.col_cap || (int64_t)carry_r + 4 > pp.row_cap) st->capacity |= 1;
  }
  if (rdy) {  // fused wave 0: the ready flags, arrival counters, completed-tile
              // counts and failed flags of the T tiles (the reset kernel leaves them to us)
    const int64_t bt = (int64_t)pp.B * carry_t, bn = (int64_t)pp.B * pp.n;
    for (int64_t q = threadIdx.x; q < bt; q += kT) {
      rdy[q] = 0;
      rdy[bn + q] = 0;
    }
    for (int q = threadIdx.x; q < 2 * pp.B; q += kT) rdy[2 * bn + q] = 0;
  }
}

__global__ void __launch_bounds__(kT, 1)
prep_kernel(const int32_t* __restrict__ hh, const int32_t* __restrict__ ww, const int64_t* area2,
            const int32_t* perm, PackParams pp, int32_t* colofs, int32_t* rowofs, int32_t* hsorted,
            int32_t* tstart, int32_t* tix, Status* st, int32_t* rdy, const uint64_t* skeys) {
  if (st->bad_chart != INT32_MAX) return;
  prep_body(hh, ww, area2, perm, pp, colofs, rowofs, hsorted, tstart, tix, st, rdy, skeys, 0);
}

// 4096 < N <= 2^17: the same layout by one CTA per 4096 sorted positions with
// decoupled look-back (the carries of a block are the published aggregates
// of all lower blocks, read in parallel by warp 0 -- no serial chain): pass 1
// slot-size sums (and the blocks' area / extent partials), pass 2 tile-start
// counts.  Every block of the grid is resident (<= 32 blocks), and a block
// waits only for lower ones.  Flags carry an epoch (PrepSync::epoch + 1,
// read by every block at its start; the last block -- which has seen every
// block's pass-1 flag, so every block has read the epoch -- advances it), so
// nothing is reset between packs.  The last block finishes the totals: the
// scale bounds, the tile end, the capacity test and the fused wave-0 flags.
__global__ void __launch_bounds__(kT, 1)
prep_multi_kernel(const int32_t* __restrict__ hh, const int32_t* __restrict__ ww,
                  const int64_t* area2, const int32_t* perm, PackParams pp, int32_t* colofs,
                  int32_t* rowofs, int32_t* hsorted, int32_t* tstart, int32_t* tix, Status* st,
                  int32_t* rdy, const uint64_t* skey, PrepSync* ps) {
  if (st->bad_chart != INT32_MAX) return;
  constexpr int kE = 4;
  constexpr int kCh = kE * kT;
  __shared__ int32_t sh[2][kW + 1];
  __shared__ unsigned long long asum[2][kW];
  __shared__ int32_t ext_max[2][kW];
  __shared__ uint16_t scw[kCh], srh[kCh];
  __shared__ int32_t s_ep, s_cc, s_cr, s_ct;
  const int b = blockIdx.x, nb = gridDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool last = b == nb - 1;
  if (tid == 0) s_ep = *(volatile int32_t*)&ps->epoch + 1;
  const int base = b * kCh, cn = min(kCh, pp.n - base);
  auto hw_at = [&](int s, int32_t& h, int32_t& w) {
    if (skey) {  // the sorted key holds (h, w): no dependent global loads
      const uint64_t k = skey[s];
      h = (int32_t)(0x3ffffffu - (uint32_t)((k >> 26) & 0x3ffffffu));
      w = (int32_t)(0x3ffffffu - (uint32_t)(k & 0x3ffffffu));
    } else {
      const int c = perm[s];
      w = ww[c];
      h = hh[c];
    }
  };
  // this block's share of the area / extent reductions (by chart index)
  {
    i128 a = 0;
    int32_t wm = 0, hm = 0;
    for (int i = base + tid; i < base + cn; i += kT) {
      a += area2[i];
      wm = max(wm, ww[i]);
      hm = max(hm, hh[i]);
    }
    a = warp_sum128(a);
    wm = warp_max(wm);
    hm = warp_max(hm);
    if (lane == 0) {
      asum[0][wid] = (unsigned long long)(uint64_t)a;
      asum[1][wid] = (unsigned long long)(uint64_t)(a >> 64);
      ext_max[0][wid] = wm;
      ext_max[1][wid] = hm;
    }
  }
  // slot sizes of the block's sorted positions (as prep_body)
#pragma unroll
  for (int u = 0; u < kE; u++) {
    const int x = u * kT + tid;
    if (x < cn) {
      int32_t h, w;
      hw_at(base + x, h, w);
      const int64_t wd = ceildiv(w, TABI_UNITS) + 2 * pp.g;
      const int64_t hd = ceildiv(h, TABI_UNITS) + 2 * pp.g;
      scw[x] = (uint16_t)(wd < pp.Wp ? wd : pp.Wp);
      srh[x] = (uint16_t)(hd < pp.Hp ? hd : pp.Hp);
      hsorted[base + x] = h;
    }
  }
  __syncthreads();
  const int q0 = min(cn, tid * kE), q1 = min(cn, q0 + kE);
  int32_t sc = 0, sr = 0;
  for (int q = q0; q < q1; q++) {
    sc += scw[q];
    sr += srh[q];
  }
  int32_t ec, er, tc, tr;
  block_scan2(sc, sr, ec, er, tc, tr, sh);
  const int32_t ep = s_ep;
  // pass 1: publish the block's aggregate, then the lower blocks' carries
  if (wid == 0) {
    i128 a = (i128)(((unsigned __int128)asum[1][lane] << 64) | asum[0][lane]);
    a = warp_sum128(a);
    const int32_t wm = warp_max(ext_max[0][lane]), hm = warp_max(ext_max[1][lane]);
    if (lane == 0) {
      ps->c[b] = tc;
      ps->r[b] = tr;
      ps->alo[b] = (unsigned long long)(uint64_t)a;
      ps->ahi[b] = (unsigned long long)(uint64_t)(a >> 64);
      ps->wm[b] = wm;
      ps->hm[b] = hm;
      __threadfence();
      st_release_flag(&ps->f1[b], ep);
    }
    int32_t cc = 0, cr = 0;
    i128 at = 0;
    int32_t wmx = 0, hmx = 0;
    if (lane < b) {
      while (ld_acquire_flag(&ps->f1[lane]) != ep) __nanosleep(32);
      cc = ps->c[lane];
      cr = ps->r[lane];
      at = (i128)(((unsigned __int128)ps->ahi[lane] << 64) | ps->alo[lane]);
      wmx = ps->wm[lane];
      hmx = ps->hm[lane];
    }
    cc = warp_sum(cc);
    cr = warp_sum(cr);
    if (lane == 0) { s_cc = cc; s_cr = cr; }
    if (last) {  // every block's partials: the area bound, extents, wave-0 width
      at = warp_sum128(at) + a;
      wmx = max(warp_max(wmx), wm);
      hmx = max(warp_max(hmx), hm);
      int m_hi, b0;
      scale_bounds(pp, at, lane, m_hi, b0);
      if (lane == 0) {
        st->wmax = wmx;
        st->hmax = hmx;
        st->pad[2] = m_hi;
        st->b0 = b0;
        st->atot_lo = (unsigned long long)(uint64_t)at;
        st->atot_hi = (unsigned long long)(uint64_t)(at >> 64);
        ps->epoch = ep;  // (every block has read the epoch: all pass-1 flags seen)
      }
    }
  }
  __syncthreads();
  ec += s_cc;
  er += s_cr;
  // the tile of the position before this block's first one
  int32_t prev_id = -1;
  if (base > 0) {
    int32_t h, w;
    hw_at(base - 1, h, w);
    const int64_t wd = min(ceildiv(w, TABI_UNITS) + 2 * pp.g, (int64_t)pp.Wp);
    const int64_t hd = min(ceildiv(h, TABI_UNITS) + 2 * pp.g, (int64_t)pp.Hp);
    prev_id = fused_tile_id((int64_t)s_cc + s_cr - wd - hd, base - 1);
  }
  int32_t pid = q0 == 0 ? prev_id
                : q0 < q1 ? fused_tile_id((int64_t)ec + er - scw[q0 - 1] - srh[q0 - 1], base + q0 - 1)
                          : 0;
  int32_t nf = 0;
  {
    int64_t cum = (int64_t)ec + er;
    int32_t p = pid;
    for (int q = q0; q < q1; q++) {
      const int32_t id = fused_tile_id(cum, base + q);
      nf += id != p;
      p = id;
      cum += scw[q] + srh[q];
    }
  }
  int32_t ef, e2, tf, t2;
  block_scan2(nf, 0, ef, e2, tf, t2, sh);
  // pass 2: tile-start counts
  if (wid == 0) {
    if (lane == 0) {
      ps->t[b] = tf;
      __threadfence();
      st_release_flag(&ps->f2[b], ep);
    }
    int32_t ct = 0;
    if (lane < b) {
      while (ld_acquire_flag(&ps->f2[lane]) != ep) __nanosleep(32);
      ct = ps->t[lane];
    }
    ct = warp_sum(ct);
    if (lane == 0) s_ct = ct;
  }
  __syncthreads();
  const int32_t carry_t = s_ct;
  {
    int32_t c = ec, r = er, tt = carry_t + ef - 1;
    for (int q = q0; q < q1; q++) {
      const int s = base + q;
      const int32_t id = fused_tile_id((int64_t)c + r, s);
      if (id != pid) tstart[++tt] = s;
      colofs[s] = c;
      rowofs[s] = r;
      tix[s] = tt;
      c += scw[q];
      r += srh[q];
      pid = id;
    }
  }
  if (!last) return;
  const int32_t cols = s_cc + tc, rows = s_cr + tr, ntiles = carry_t + tf;
  if (tid == 0) {
    st->cols_total = cols;
    st->rows_total = rows;
    st->ntiles = ntiles;
    tstart[ntiles] = pp.n;
    // +4: the TMA bulk copy of a row window rounds its end up to 16 bytes
    if ((int64_t)cols + 4 > pp.col_cap || (int64_t)rows + 4 > pp.row_cap) st->capacity |= 1;
  }
  if (rdy) {  // fused wave 0 (as prep_body)
    const int64_t bt = (int64_t)pp.B * ntiles, bn = (int64_t)pp.B * pp.n;
    for (int64_t q = tid; q < bt; q += kT) {
      rdy[q] = 0;
      rdy[bn + q] = 0;
    }
    for (int q = tid; q < 2 * pp.B; q += kT) rdy[2 * bn + q] = 0;
  }
}

// N <= 2048: order and slot layout in one launch (the block that sorted reads
// its own permutation after a barrier).
__global__ void __launch_bounds__(kT, 1)
sort_prep_kernel(const int32_t* __restrict__ hh, const int32_t* __restrict__ ww,
                 const int64_t* area2, int32_t* perm, PackParams pp, int32_t* colofs,
                 int32_t* rowofs, int32_t* hsorted, int32_t* tstart, int32_t* tix, Status* st,
                 int32_t* rdy) {
  if (st->bad_chart != INT32_MAX) return;
  const uint64_t* skey = bitonic_reg_body(hh, ww, pp.n, perm);
  __syncthreads();
  prep_body(hh, ww, area2, perm, pp, colofs, rowofs, hsorted, tstart, tix, st, rdy, skey);
}

// Batch mode (tabi_pack_many): one CTA per atlas -- its order (register
// bitonic, N <= 2048) and slot layout, written at the atlas's chart offset
// (tile arrays at offset + atlas index: one more tstart entry per atlas).
__global__ void __launch_bounds__(kT, 1)
many_sort_prep_kernel(Proxies P, const int32_t* __restrict__ abase, int32_t* perm, PackParams pp,
                      int32_t* colofs, int32_t* rowofs, int32_t* hsorted, int32_t* tstart,
                      int32_t* tix, Status* sts) {
  const int a = blockIdx.x;
  const int c0 = abase[a], n = abase[a + 1] - c0;
  Status* st = sts + a;
  if (n < 1 || n > 2 * kT || st->bad_chart != INT32_MAX || st->capacity) return;
  PackParams q = pp;
  q.n = n;
  const uint64_t* skey = bitonic_reg_body(P.h + c0, P.w + c0, n, perm + c0);
  __syncthreads();
  prep_body(P.h + c0, P.w + c0, P.area2 + c0, perm + c0, q, colofs + c0, rowofs + c0,
            hsorted + c0, tstart + c0 + a, tix + c0, st, nullptr, skey);
}

// Batch mode: per-atlas status blocks and results, and the pack work queue
// (items [0, E) = the batched atlases in `order`, candidate offset 0; the
// rest empty).
__global__ void many_reset_kernel(Status* sts, AtlasRes* res, int32_t A, const int32_t* order,
                                  int32_t E, int32_t* q, int32_t qcap, int32_t* qctl, int32_t K) {
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t a = t0; a < A; a += stride) {
    uint32_t* w = (uint32_t*)(sts + a);
    for (size_t i = 0; i < sizeof(Status) / 4; i++) w[i] = 0;
    sts[a].bad_chart = INT32_MAX;
    sts[a].win_j = INT32_MAX;
    AtlasRes z{};
    z.next_r = K;
    z.issued = K;
    res[a] = z;
  }
  // item i: atlas order[i / K], rank i % K (the largest atlases first, each
  // with K ranks in flight)
  for (int64_t i = t0; i < qcap; i += stride)
    q[i] = i < (int64_t)E * K ? order[i / K] | (int32_t)((i % K) << 20) : -1;
  if (t0 == 0) {
    qctl[0] = 0;      // head
    qctl[1] = E * K;  // tail
    qctl[2] = E;      // atlases not yet decided
    qctl[3] = 0;      // idle speculation: order positions below are decided
  }
}

// One launch instead of a status upload plus a string of memsets.
// mode 2: initialise the status block (bad_chart = none, trace start = max)
// and zero the candidate records and hybrid-tail states;
// always: zero per-wave state (cand_bad, large-chart list, raster queue head,
// fused ready flags / arrival counters).
__global__ void reset_kernel(Status* st, int mode, Cand* cands, int32_t* t_state,
                             int32_t* cand_bad, int M, int32_t* rdy, int64_t nrdy) {
  // mode 2: fresh status (wave 0); 0: the next wave (the wave index advances)
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (t0 == 0) {
    if (mode == 2) {
      uint32_t* w = (uint32_t*)st;
      for (size_t i = 0; i < sizeof(Status) / 4; i++) w[i] = 0;
      st->bad_chart = INT32_MAX;
      st->tr[0] = ~0ull;
      st->win_j = INT32_MAX;
    } else {
      if (mode == 0) st->wave++;
      st->pad[1] = 0;
      st->work_next = 0;
      st->win_j = INT32_MAX;
    }
  }
  if (mode == 1 || mode == 2) {
    int32_t* cw = (int32_t*)cands;
    for (int64_t i = t0; i < (int64_t)M * (int64_t)(sizeof(Cand) / 4); i += stride) cw[i] = 0;
    for (int64_t i = t0; i < M; i += stride) t_state[i] = 0;
  }
  for (int64_t i = t0; i < M; i += stride) cand_bad[i] = 0;
  for (int64_t i = t0; i < nrdy; i += stride) rdy[i] = 0;
}

}  // namespace

void launch_reset(Status* st, int mode, Cand* cands, int32_t* t_state, int32_t* cand_bad, int M,
                  int32_t* rdy, int64_t nrdy, cudaStream_t s) {
  const int64_t work = nrdy > (int64_t)M * 16 ? nrdy : (int64_t)M * 16;
  int blocks = (int)((work + 255) / 256);
  if (blocks > 296) blocks = 296;
  reset_kernel<<<blocks, 256, 0, s>>>(st, mode, cands, t_state, cand_bad, M, rdy, nrdy);
}

int launch_sort(const Proxies& P, int32_t n, uint64_t* keys, uint64_t* keys2, int32_t* perm,
                int32_t* perm2, const Status* st, cudaStream_t s, const uint64_t** sorted_keys) {
  if (sorted_keys) *sorted_keys = nullptr;
  // TABI_SORT=bitonic|chunk|rank|radix forces a path (tests cover all four)
  const char* force = getenv("TABI_SORT");
  const bool want_rank = force && strcmp(force, "rank") == 0;
  const bool want_radix = force && strcmp(force, "radix") == 0;
  const bool want_chunk = force && strcmp(force, "chunk") == 0;
  if (n <= 2 * kT && !want_rank && !want_radix && !want_chunk &&
      !(force && strcmp(force, "bitonic") == 0)) {
    bitonic_reg_kernel<<<1, kT, 0, s>>>(P.h, P.w, n, perm, st);
    return 1;
  }
  if (n <= kBitonicMax && force && strcmp(force, "bitonic") == 0) {
    bitonic_kernel<<<1, kT, 0, s>>>(P.h, P.w, n, perm, st);
    return 1;
  }
  if (n <= kRankMax && !want_radix && !want_rank) {
    // chunked bitonic + merge ranks (ck in keys, ci in perm2)
    const int nch = (n + kChunk - 1) / kChunk;
    chunk_sort_kernel<<<nch, kT, 0, s>>>(P.h, P.w, n, keys, perm2, st);
    chunk_rank_kernel<<<(n + kT - 1) / kT, kT, 0, s>>>(keys, perm2, n, perm, keys2, st);
    if (sorted_keys) *sorted_keys = keys2;
    return 2;
  }
  if (n <= kRankMax && !want_radix) {
    int32_t* rank = (int32_t*)keys2;
    cudaMemsetAsync(rank, 0, sizeof(int32_t) * (size_t)n, s);
    rank_count_kernel<<<dim3((n + kRankT - 1) / kRankT, (n + kRankJ - 1) / kRankJ), kRankT, 0, s>>>(
        P.h, P.w, n, rank, st);
    rank_scatter_kernel<<<(n + 255) / 256, 256, 0, s>>>(rank, n, perm, st);
    return 2;
  }
  sort_kernel<<<1, kT, 0, s>>>(P.h, P.w, n, keys, keys2, perm, perm2, st);
  return 1;
}

bool launch_sort_prep(const Proxies& P, int32_t* perm, const PackParams& pp, int32_t* colofs,
                      int32_t* rowofs, int32_t* hsorted, int32_t* tstart, int32_t* tix, Status* st,
                      int32_t* rdy, cudaStream_t s) {
  if (pp.n > 2 * kT || getenv("TABI_SORT")) return false;
  sort_prep_kernel<<<1, kT, 0, s>>>(P.h, P.w, P.area2, perm, pp, colofs, rowofs, hsorted, tstart,
                                    tix, st, rdy);
  return true;
}

void launch_many_sort_prep(const Proxies& P, const int32_t* abase, int32_t A, int32_t* perm,
                          const PackParams& pp, int32_t* colofs, int32_t* rowofs, int32_t* hsorted,
                          int32_t* tstart, int32_t* tix, Status* sts, cudaStream_t s) {
  many_sort_prep_kernel<<<A, kT, 0, s>>>(P, abase, perm, pp, colofs, rowofs, hsorted, tstart, tix,
                                         sts);
}

void launch_many_reset(Status* sts, AtlasRes* res, int32_t A, const int32_t* order, int32_t E,
                       int32_t* q, int32_t qcap, int32_t* qctl, int32_t inflight, cudaStream_t s) {
  const int64_t work = qcap > A ? qcap : A;
  int blocks = (int)((work + 255) / 256);
  if (blocks > 296) blocks = 296;
  if (blocks < 1) blocks = 1;
  many_reset_kernel<<<blocks, 256, 0, s>>>(sts, res, A, order, E, q, qcap, qctl, inflight);
}

void launch_prep(const Proxies& P, const int32_t* perm, const PackParams& pp, int32_t* colofs,
                 int32_t* rowofs, int32_t* hsorted, int32_t* tstart, int32_t* tix, Status* st,
                 int32_t* rdy, cudaStream_t s, const uint64_t* sorted_keys, PrepSync* ps) {
  const int nb = (pp.n + 4 * kT - 1) / (4 * kT);
  const char* env = getenv("TABI_PREP_MULTI");  // test knob: 0 = one CTA
  if (ps && nb > 1 && nb <= kPrepMaxBlocks && !(env && env[0] == '0')) {
    prep_multi_kernel<<<nb, kT, 0, s>>>(P.h, P.w, P.area2, perm, pp, colofs, rowofs, hsorted,
                                        tstart, tix, st, rdy, sorted_keys, ps);
    return;
  }
  prep_kernel<<<1, kT, 0, s>>>(P.h, P.w, P.area2, perm, pp, colofs, rowofs, hsorted, tstart, tix,
                               st, rdy, sorted_keys);
}

}  // namespace tabi
