// k_floor.cu -- latency floor of the packer's per-row building blocks
// ("measure c with a barrier/reduce microbenchmark and report
// per-row ns x R").  One CTA of 512 threads -- the packer's shape -- times
// dependent chains of each primitive with clock64 and converts cycles to ns
// with %globaltimer over the same loop.  Diagnostic only: not on the pack path.
#include "tabi_internal.cuh"

namespace tabi {
namespace {

constexpr int kFT = 512;

__global__ void __launch_bounds__(kFT, 1) floor_kernel(int iters, int32_t* gbuf, long long* out) {
  __shared__ int32_t buf[kFT];
  __shared__ int32_t red[kFT / 32];
  __shared__ int32_t bcast;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int32_t v = tid;
  buf[tid] = tid;
  __syncthreads();
  long long c[6];
  unsigned long long g0 = 0, g1 = 0;
  // [0] bar.sync alone
  c[0] = clock64();
  if (tid == 0) g0 = gtime();
  for (int i = 0; i < iters; i++) __syncthreads();
  c[1] = clock64();
  if (tid == 0) g1 = gtime();
  // [1] barrier + shared-memory exchange (write own, read a neighbour's)
  for (int i = 0; i < iters; i++) {
    buf[tid] = v;
    __syncthreads();
    v = buf[(tid + 33) & (kFT - 1)] + 1;
    __syncthreads();
  }
  c[2] = clock64();
  // [2] block-wide max: warp reduce, smem, barrier, warp 0 reduce, barrier, broadcast
  for (int i = 0; i < iters; i++) {
    const int32_t m = __reduce_max_sync(0xffffffffu, v);
    if (lane == 0) red[wid] = m;
    __syncthreads();
    if (wid == 0) {
      const int32_t x = __reduce_max_sync(0xffffffffu, lane < kFT / 32 ? red[lane] : INT32_MIN);
      if (lane == 0) bcast = x;
    }
    __syncthreads();
    v = bcast - v + tid;
  }
  c[3] = clock64();
  // [3] shared atomicMax by every thread, then a barrier (the push / commit pattern)
  for (int i = 0; i < iters; i++) {
    atomicMax(&buf[(tid * 7) & (kFT - 1)], v);
    __syncthreads();
    v = buf[tid] & 0xffff;
  }
  c[4] = clock64();
  // [4] thread 0: dependent L2 loads (ld.cg pointer chase) -- a global read in the row chain
  if (tid == 0) {
    int32_t p = 0;
    for (int i = 0; i < iters; i++) p = __ldcg(gbuf + p);
    v += p;
  }
  __syncthreads();
  c[5] = clock64();
  if (tid == 0) {
    for (int i = 0; i < 5; i++) out[i] = c[i + 1] - c[i];
    out[5] = (long long)(g1 - g0);  // ns of the [0] loop
    out[6] = v;                     // keep the chains live
  }
}

}  // namespace

// out8: ns per operation: [0] barrier, [1] barrier + smem exchange (2 barriers),
// [2] block max-reduce (2 barriers), [3] smem atomicMax + barrier,
// [4] dependent L2 load; [5] SM MHz measured; [6], [7] 0.
int latency_floor(int device, double* out8) {
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  const int iters = 4096;
  int32_t* g = nullptr;
  long long* d = nullptr;
  if (cudaMalloc(&g, 4096 * sizeof(int32_t)) != cudaSuccess) return 3;
  if (cudaMalloc(&d, 8 * sizeof(long long)) != cudaSuccess) { cudaFree(g); return 3; }
  int32_t h[4096];
  for (int i = 0; i < 4096; i++) h[i] = (i * 1031 + 17) & 4095;  // a 4096-cycle permutation walk
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  long long r[8] = {0};
  for (int rep = 0; rep < 3; rep++) {  // warm-up, then keep the last
    floor_kernel<<<1, kFT>>>(iters, g, d);
    cudaMemcpy(r, d, 8 * sizeof(long long), cudaMemcpyDeviceToHost);
  }
  cudaFree(g);
  cudaFree(d);
  if (cudaGetLastError() != cudaSuccess) return 3;
  const double mhz = r[5] > 0 ? (double)r[0] / (double)r[5] * 1000.0 : 0.0;
  for (int i = 0; i < 5; i++) out8[i] = mhz > 0 ? (double)r[i] / iters / mhz * 1000.0 : 0.0;
  out8[5] = mhz;
  out8[6] = out8[7] = 0.0;
  return 0;
}

}  // namespace tabi
