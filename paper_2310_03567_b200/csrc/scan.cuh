// scan.cuh -- block scans and the device-wide single-pass exclusive scan.
//
// Used for every order-preserving offset computation on the update path:
// per-point voxel-win counts -> backlog positions, per-node flags -> dense ids,
// per-node chunk needs -> acquisition indices; block scans inside the radix
// passes, the split decision, the selection and the delta.
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

__device__ __forceinline__ uint32_t shfl_xor_t(uint32_t v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ unsigned long long shfl_xor_t(unsigned long long v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
__device__ __forceinline__ U64x2 shfl_xor_t(U64x2 v, int m) {
  return u64x2(__shfl_xor_sync(0xffffffffu, v.a, m), __shfl_xor_sync(0xffffffffu, v.b, m));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = v + shfl_xor_t(v, m);
  return v;
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

#ifndef LOD_SCAN_VEC
#define LOD_SCAN_VEC 1
#endif
constexpr int kScanBlock = 512;
constexpr int kScanItems = 8;
constexpr long long kScanTile = (long long)kScanBlock * kScanItems;

// ---- single-pass scan (decoupled look-back) ---------------------------------
//
// One launch instead of reduce + scan-of-partials + scan.  Tiles take tickets in
// launch order (so a tile only ever waits on tiles already running), publish
// their aggregate, look back over predecessors 32 at a time (one warp, one
// status word per lane) until an inclusive prefix, and publish theirs.  Status words carry the call's epoch, so the
// look-back state never needs clearing between calls; the ticket counter keeps
// counting and each call starts at its own base.
struct ScanLB {
  unsigned *status = nullptr;  // per tile: epoch << 2 | 1 (aggregate) / 2 (inclusive prefix)
  void *agg = nullptr;         // per tile: T
  void *incl = nullptr;        // per tile: T
  unsigned long long *ticket = nullptr;
  long long cap_tiles = 0;
  unsigned epoch = 0;              // host: last epoch used
  unsigned long long tickets = 0;  // host: tickets handed out so far
};

__device__ __forceinline__ uint32_t ld_cg(const uint32_t *p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ld_cg(const unsigned long long *p) { return __ldcg(p); }
__device__ __forceinline__ U64x2 ld_cg(const U64x2 *p) {
  const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2 *>(p));
  return u64x2(v.x, v.y);
}

template <typename T>
__global__ void __launch_bounds__(kScanBlock)
    k_scan_lb(const T *__restrict__ in, long long n, T *__restrict__ out, T *__restrict__ total_out,
              unsigned *status, T *agg, T *incl, unsigned long long *ticket, unsigned long long ticket_base,
              unsigned epoch, const int *guard) { lod::pdl_wait();
  __shared__ T sh[kScanBlock / 32 + 1];
  __shared__ long long s_tile;
  __shared__ T s_excl;
  // the ticket is taken even by a stood-down launch: the host counts them
  if (threadIdx.x == 0) s_tile = (long long)(atomicAdd(ticket, 1ull) - ticket_base);
  if (guard && *guard) return;
  __syncthreads();
  const long long tile = s_tile;
  const long long base = tile * kScanTile + (long long)threadIdx.x * kScanItems;
  T v[kScanItems];
  T acc = T();
  // u32 items of a full tile: two 16-byte loads per thread
  constexpr bool kVec = LOD_SCAN_VEC && sizeof(T) == 4 && kScanItems == 8;
  const bool vec = kVec && base + kScanItems <= n;
  if constexpr (kVec) if (vec) {
    const uint4 *p = reinterpret_cast<const uint4 *>(in + base);
    const uint4 a = p[0], b = p[1];
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) v[i] = *reinterpret_cast<const T *>(&w[i]);
  }
  if (!vec) {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) v[i] = base + i < n ? in[base + i] : T();
  }
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) acc = acc + v[i];
  T total;
  T run = block_exclusive_scan<T, kScanBlock>(acc, sh, total);
  if (threadIdx.x < 32) {  // warp 0 publishes and looks back, 32 predecessors per round trip
    const unsigned e = epoch << 2;
    const int lane = threadIdx.x;
    T excl = T();
    if (tile == 0) {
      if (lane == 0) {
        incl[0] = total;
        __threadfence();
        atomicExch(status, e | 2u);
      }
    } else {
      if (lane == 0) {
        agg[tile] = total;
        __threadfence();
        atomicExch(status + tile, e | 1u);
      }
      long long t = tile - 1;
      for (;;) {
        const long long idx = t - lane;
        const unsigned st = idx >= 0 ? *((volatile unsigned *)(status + idx)) : (e | 2u);
        const bool ready = (st & ~3u) == e && (st & 3u) != 0;
        const unsigned incl_mask = __ballot_sync(0xffffffffu, ready && (st & 3u) == 2u);
        const unsigned wait_mask = __ballot_sync(0xffffffffu, !ready);
        const int first_incl = incl_mask ? __ffs(incl_mask) - 1 : 32;
        const int first_wait = wait_mask ? __ffs(wait_mask) - 1 : 32;
        __threadfence();
        // consume the published run of predecessors before the first gap,
        // ending at (and including) the nearest inclusive prefix
        const int take = first_wait < first_incl ? first_wait : first_incl;
        T val = T();
        if (lane < take) val = ld_cg(agg + idx);
        else if (lane == take && take == first_incl && first_incl < 32) val = ld_cg(incl + idx);
        excl = excl + warp_sum(val);
        if (first_incl < 32 && first_incl <= first_wait) break;
        t -= take;
      }
      if (lane == 0) {
        incl[tile] = excl + total;
        __threadfence();
        atomicExch(status + tile, e | 2u);
      }
    }
    if (lane == 0) {
      s_excl = excl;
      if (total_out && (tile + 1) * kScanTile >= n) *total_out = excl + total;
    }
  }
  __syncthreads();
  run = run + s_excl;
  if constexpr (kVec) if (vec) {
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      w[i] = *reinterpret_cast<const uint32_t *>(&run);
      run = run + v[i];
    }
    uint4 *q = reinterpret_cast<uint4 *>(out + base);
    q[0] = make_uint4(w[0], w[1], w[2], w[3]);
    q[1] = make_uint4(w[4], w[5], w[6], w[7]);
    return;
  }
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run = run + v[i];
  }
}

// exclusive_scan in one launch (ScanLB state owned by the caller; tiles <= cap_tiles).
template <typename T>
void exclusive_scan_lb(const T *in, T *out, long long n, T *total_out, ScanLB &lb, cudaStream_t st,
                       const int *guard = nullptr) {
  if (n <= 0) {
    if (total_out && !guard) cudaMemsetAsync(total_out, 0, sizeof(T), st);
    return;
  }
  const long long tiles = (n + kScanTile - 1) / kScanTile;
  lb.epoch = (lb.epoch + 1) & 0x3FFFFFFFu;
  if (lb.epoch == 0) lb.epoch = 1;
  const unsigned long long base = lb.tickets;
  lb.tickets += (unsigned long long)tiles;
  lod::launch(k_scan_lb<T>, (unsigned)tiles, kScanBlock, 0, st, in, n, out, total_out, lb.status,
              reinterpret_cast<T *>(lb.agg), reinterpret_cast<T *>(lb.incl), lb.ticket, base, lb.epoch, guard);
}

}  // namespace lod
