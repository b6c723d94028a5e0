// scan.cuh -- device-wide exclusive prefix sums (reduce-then-scan).
//
// Used for every order-preserving offset computation on the update path:
// per-point voxel-win counts -> backlog positions, per-node flags -> dense ids,
// per-node chunk needs -> acquisition indices, and the digit-major tile
// histograms of the stable multisplit (radix.cuh).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lod {

struct U64x2 {  // trivial (no constructors) so it can live in __shared__
  unsigned long long a, b;
};
__host__ __device__ __forceinline__ U64x2 u64x2(unsigned long long a, unsigned long long b) {
  U64x2 r;
  r.a = a;
  r.b = b;
  return r;
}
__host__ __device__ __forceinline__ U64x2 operator+(const U64x2 &x, const U64x2 &y) {
  return u64x2(x.a + y.a, x.b + y.b);
}

__device__ __forceinline__ uint32_t shfl_up_t(uint32_t v, int d) {
  return __shfl_up_sync(0xffffffffu, v, d);
}
__device__ __forceinline__ unsigned long long shfl_up_t(unsigned long long v, int d) {
  return __shfl_up_sync(0xffffffffu, v, d);
}
__device__ __forceinline__ U64x2 shfl_up_t(U64x2 v, int d) {
  return u64x2(__shfl_up_sync(0xffffffffu, v.a, d), __shfl_up_sync(0xffffffffu, v.b, d));
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T u = shfl_up_t(v, d);
    if (lane >= d) v = v + u;
  }
  return v;
}

// Exclusive scan of one value per thread across a BLOCK-thread block; returns
// the thread's exclusive prefix and the block total.  `sh` holds >= BLOCK/32+1
// elements.  Ends with __syncthreads so `sh` can be reused immediately.
template <typename T, int BLOCK>
__device__ __forceinline__ T block_exclusive_scan(T v, T *sh, T &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = BLOCK / 32;
  T inc = warp_inclusive_scan(v);
  T exc = shfl_up_t(inc, 1);
  if (lane == 0) exc = T();
  if (lane == 31) sh[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < NW ? sh[lane] : T();
    T wi = warp_inclusive_scan(w);
    T we = shfl_up_t(wi, 1);
    if (lane == 0) we = T();
    if (lane < NW) sh[lane] = we;  // exclusive warp offsets
    if (lane == NW - 1) sh[NW] = wi;
  }
  __syncthreads();
  T out = sh[warp] + exc;
  total = sh[NW];
  __syncthreads();
  return out;
}

constexpr int kScanBlock = 512;
constexpr int kScanItems = 8;
constexpr long long kScanTile = (long long)kScanBlock * kScanItems;

// Per-tile reduction.
template <typename T>
__global__ void __launch_bounds__(kScanBlock) k_scan_reduce(const T *__restrict__ in, long long n,
                                                            T *__restrict__ partial, const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  __shared__ T sh[kScanBlock / 32 + 1];
  long long base = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  T acc = T();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) acc = acc + in[base + i];
  T total;
  block_exclusive_scan<T, kScanBlock>(acc, sh, total);
  if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

// Scan each tile (thread-contiguous items) with an optional per-tile offset.
template <typename T>
__global__ void __launch_bounds__(kScanBlock) k_scan_tiles(const T *__restrict__ in, long long n,
                                                           T *__restrict__ out,
                                                           const T *__restrict__ tile_off,
                                                           T *__restrict__ total_out, const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  __shared__ T sh[kScanBlock / 32 + 1];
  long long base = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  T v[kScanItems];
  T acc = T();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : T();
    acc = acc + v[i];
  }
  T total;
  T run = block_exclusive_scan<T, kScanBlock>(acc, sh, total);
  if (tile_off) run = run + tile_off[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run = run + v[i];
  }
  if (total_out && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    // the last tile's total plus its offset = grand total
    *total_out = (tile_off ? tile_off[blockIdx.x] : T()) + total;
  }
}

// Scratch needed by exclusive_scan for n elements (in elements of T).
inline long long scan_scratch_elems(long long n) {
  long long need = 0;
  while (n > kScanTile) {
    long long t = (n + kScanTile - 1) / kScanTile;
    need += 2 * t;
    n = t;
  }
  return need + 1;
}

// out[i] = sum(in[0..i)); *total_out (device) = sum(in).  `in` may alias `out`.
// `scratch` must hold scan_scratch_elems(n) elements.  With a guard, every
// kernel returns at once while *guard != 0 (speculative launches).
template <typename T>
void exclusive_scan(const T *in, T *out, long long n, T *total_out, T *scratch, cudaStream_t st,
                    const int *guard = nullptr) {
  if (n <= 0) {
    if (total_out && !guard) cudaMemsetAsync(total_out, 0, sizeof(T), st);
    return;
  }
  if (n <= kScanTile) {
    lod::launch(k_scan_tiles<T>, 1, kScanBlock, 0, st, in, n, out, nullptr, total_out, guard);
    return;
  }
  long long tiles = (n + kScanTile - 1) / kScanTile;
  T *partial = scratch;
  T *partial_scan = scratch + tiles;
  lod::launch(k_scan_reduce<T>, (unsigned)tiles, kScanBlock, 0, st, in, n, partial, guard);
  exclusive_scan<T>(partial, partial_scan, tiles, nullptr, scratch + 2 * tiles, st, guard);
  lod::launch(k_scan_tiles<T>, (unsigned)tiles, kScanBlock, 0, st, in, n, out, partial_scan, total_out, guard);
}

}  // namespace lod
