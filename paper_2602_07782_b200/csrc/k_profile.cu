// k_profile.cu -- K3: per-(chart, candidate) footprints; K3b: compaction
// offsets and lock flags of adjacent pairs.
//
// K3 evaluates TopEdge/BottomEdge for every texel column and the symmetric
// left/right edges for every texel row of every chart at every candidate
// scale m/M ("We evaluate TopEdge and BottomEdge using both
// proxies and use the result per-texel that provides the tightest bound"),
// rounded outward (D11), then applies the gutter as a Chebyshev dilation by g
// (D13).
//
// Work decomposition (tile kernel): one CTA takes kTC consecutive sorted
// charts of one candidate.  Setup -- the per-(chart, candidate) constants --
// is split into 8 uniform jobs per chart (every division a multiply by a
// reciprocal estimate plus an exact integer correction).  Then all threads
// walk the tile's flattened cells into a shared-memory raw buffer and dilate
// from it into the HBM slots (coalesced).  Charts whose raw cells exceed the
// buffer go to a compacted list processed warp-per-chart (same arithmetic).
// Per cell: the local-AABB bound is the min/max over the 1-2 slices that
// openly overlap it; the OBB bound is an integer compare of the cell index
// with the crossing indices plus one int64 progression (LinDiv) per bound.
// The device code lives in k3_dev.cuh (shared with the fused pack kernel).
//
// K3b computes, per candidate and adjacent sorted pair, the horizontal
// compaction advance (a max-reduction of profile gaps over shared
// rows, D14) and the CannotMoveAbove flags (D15) with warp scans.
// These kernels serve the hybrid tail's re-rasterization (tail mode) and the
// non-fused path (TABI_FUSED=0).
#include "k3_dev.cuh"

namespace tabi {
namespace {

using namespace k3;

constexpr int kTC = 16;      // charts per tile
constexpr int kTT = 128;     // threads per tile CTA (8 per chart during setup)
constexpr int kWarps = 8;    // big-chart / offsets kernels: warps per CTA

__device__ __forceinline__ Scale scale_of(const PackParams& pp, int m) {
  Scale sc{m, (int64_t)pp.M * TABI_UNITS, 0};
  if (pp.tail) {
    sc.num = pp.T.p[m - 1];
    sc.SC = (int64_t)TABI_UNITS << 20;
    sc.r0 = pp.T.r0[m - 1];
  }
  return sc;
}

__global__ void __launch_bounds__(kTT, 4)
profile_tile_kernel(Proxies P, const int32_t* __restrict__ perm, PackParams pp,
                    const int32_t* __restrict__ colofs, const int32_t* __restrict__ rowofs,
                    uint32_t* dcol, uint32_t* drow, int32_t* wd_all, int32_t* hd_all,
                    int32_t* cand_bad, int32_t* big_list, Status* st) {
  __shared__ ChartK3 CH[kTC];
  __shared__ int32_t cells[kTC], cpre[kTC + 1], opre[kTC + 1], big[kTC];
  __shared__ int32_t chunk_end;
  extern __shared__ __align__(16) int32_t dyn[];
  if (st->bad_chart != INT32_MAX || st->capacity) return;
  const int m = wave_m(pp, st->wave, st->pad[2], st->b0, blockIdx.y);
  if (m == 0) return;
  const int s0 = blockIdx.x * kTC;
  const Scale sc = scale_of(pp, m);
  if (pp.tail) {
    if (pp.T.state[m - 1] != TAIL_LAYOUT) return;
    if (s0 + min(kTC, pp.n - s0) <= sc.r0) return;
  }
  int32_t* tabs = dyn;  // [kTC][2 axes][k][2]
  uint32_t* raw = (uint32_t*)(dyn + kTC * 4 * pp.k);
  tile_raster<kTC, kTT, kRaw>(P, perm, pp, colofs, rowofs, dcol, drow, wd_all, hd_all, cand_bad, m - 1,
                              s0, sc, CH, cells, cpre, opre, &chunk_end, big, tabs, raw,
                              min(kTC, pp.n - s0), (int)threadIdx.x, [] { __syncthreads(); });
  if (threadIdx.x == 0) {
    for (int ci = 0; ci < kTC; ci++)
      if (big[ci]) big_list[atomicAdd(&st->pad[1], 1)] = (m - 1) * pp.n + s0 + ci;
  }
}

__global__ void __launch_bounds__(kWarps * 32)
profile_big_kernel(Proxies P, const int32_t* __restrict__ perm, PackParams pp,
                   const int32_t* __restrict__ colofs, const int32_t* __restrict__ rowofs,
                   uint32_t* dcol, uint32_t* drow, const int32_t* __restrict__ big_list,
                   const Status* st) {
  __shared__ ChartK3 CH[kWarps];
  extern __shared__ __align__(16) int32_t dyn[];
  if (st->bad_chart != INT32_MAX || st->capacity) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int32_t* tab = dyn + wib * 4 * pp.k;
  const int nbig = st->pad[1];
  for (int it = blockIdx.x * kWarps + wib; it < nbig; it += gridDim.x * kWarps) {
    const int item = big_list[it];
    const int m = item / pp.n + 1, s = item % pp.n;
    big_chart(P, perm, pp, colofs, rowofs, dcol, drow, m - 1, s, scale_of(pp, m), CH[wib], tab, lane);
  }
}

__global__ void __launch_bounds__(kWarps * 32)
offsets_kernel(PackParams pp, const int32_t* __restrict__ rowofs, const uint32_t* __restrict__ drow,
               const int32_t* __restrict__ wd_all, const int32_t* __restrict__ hd_all,
               int32_t* off_all, uint8_t* lock_all, const int32_t* __restrict__ cand_bad,
               const Status* st) {
  if (st->bad_chart != INT32_MAX || st->capacity) return;
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (item >= (int64_t)pp.n * pp.B) return;
  const int m = wave_m(pp, st->wave, st->pad[2], st->b0, (int)(item / pp.n));
  if (m == 0) return;
  const int s = (int)(item % pp.n);
  if (cand_bad[m - 1]) return;
  if (pp.tail && (pp.T.state[m - 1] != TAIL_LAYOUT || s < pp.T.r0[m - 1])) return;
  pair_offset(pp, rowofs, drow, wd_all, hd_all, off_all, lock_all, m - 1, s, lane);
}

}  // namespace

void launch_profiles(const Proxies& P, const int32_t* perm, const PackParams& pp,
                     const int32_t* colofs, const int32_t* rowofs, int16_t* dcol, int16_t* drow,
                     int32_t* wd, int32_t* hd, int32_t* cand_bad, int32_t* big_list, Status* st,
                     cudaStream_t s) {
  const size_t dyn = sizeof(int32_t) * (size_t)(kTC * 4 * pp.k) + sizeof(uint32_t) * kRaw;
  static std::atomic<unsigned long long> attr{0};
  ensure_dyn_smem((const void*)profile_tile_kernel, (int)(sizeof(int32_t) * (kTC * 4 * TABI_KMAX) + sizeof(uint32_t) * kRaw), attr);
  dim3 grid((pp.n + kTC - 1) / kTC, pp.B);
  profile_tile_kernel<<<grid, kTT, dyn, s>>>(P, perm, pp, colofs, rowofs, (uint32_t*)dcol,
                                             (uint32_t*)drow, wd, hd, cand_bad, big_list, st);
  profile_big_kernel<<<296, kWarps * 32, sizeof(int32_t) * kWarps * 4 * pp.k, s>>>(
      P, perm, pp, colofs, rowofs, (uint32_t*)dcol, (uint32_t*)drow, big_list, st);
}

void launch_offsets(const PackParams& pp, const int32_t* colofs, const int32_t* rowofs,
                    const int16_t* drow, const int32_t* wd, const int32_t* hd, int32_t* off,
                    uint8_t* lockbits, const int32_t* cand_bad, const Status* st,
                    cudaStream_t s) {
  (void)colofs;
  const int64_t items = (int64_t)pp.n * pp.B;
  const int blocks = (int)((items + kWarps - 1) / kWarps);
  offsets_kernel<<<blocks, kWarps * 32, 0, s>>>(pp, rowofs, (const uint32_t*)drow, wd, hd, off,
                                                 lockbits, cand_bad, st);
}

}  // namespace tabi
