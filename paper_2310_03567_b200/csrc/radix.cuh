// radix.cuh -- stable multisplit of an ordered item list by a small dense key.
//
// The reference appends records to each node in global ingestion order
// (store_points/store_voxels, _kernels.py:155-250: slot = count[node]++ in
// all-array / backlog order).  On the GPU that order is recovered with an LSD
// radix sort over dense node keys: 8-bit digits, one pass per key byte, each
// pass a tile histogram -> digit-major exclusive scan -> stable tile scatter.
// Stability inside a tile comes from warp-ordered rounds: each warp owns a
// contiguous 512-item range, ranks lanes with __match_any_sync, and keeps a
// per-warp digit histogram in shared memory; warps are combined in order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "scan.cuh"

namespace lod {

constexpr int kRadixBits = 8;
constexpr int kRadixDigits = 1 << kRadixBits;
constexpr int kRadixBlock = 256;  // 8 warps
constexpr int kRadixWarps = kRadixBlock / 32;
constexpr int kRadixRounds = 16;  // per warp: 16 rounds x 32 lanes
constexpr long long kRadixTile = (long long)kRadixBlock * kRadixRounds;

__global__ void __launch_bounds__(kRadixBlock)
    k_radix_hist(const uint32_t *__restrict__ keys, long long n, int shift, long long ntiles,
                 uint32_t *__restrict__ hist) {
  __shared__ uint32_t h[kRadixDigits];
  for (int d = threadIdx.x; d < kRadixDigits; d += kRadixBlock) h[d] = 0;
  __syncthreads();
  long long base = (long long)blockIdx.x * kRadixTile;
  for (int i = threadIdx.x; i < kRadixTile; i += kRadixBlock) {
    long long idx = base + i;
    if (idx < n) atomicAdd(&h[(__ldg(keys + idx) >> shift) & (kRadixDigits - 1)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRadixDigits; d += kRadixBlock)
    hist[(long long)d * ntiles + blockIdx.x] = h[d];
}

// vals_in == nullptr means the identity permutation (item index).
__global__ void __launch_bounds__(kRadixBlock)
    k_radix_scatter(const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
                    long long n, int shift, long long ntiles, const uint32_t *__restrict__ gofs,
                    uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out) {
  __shared__ uint32_t wh[kRadixWarps][kRadixDigits];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = lane; d < kRadixDigits; d += 32) wh[warp][d] = 0;
  __syncwarp();
  const long long wbase = (long long)blockIdx.x * kRadixTile + (long long)warp * (32 * kRadixRounds);
  uint32_t key[kRadixRounds], val[kRadixRounds], loc[kRadixRounds];
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    long long idx = wbase + r * 32 + lane;
    bool ok = idx < n;
    key[r] = ok ? __ldg(keys_in + idx) : 0u;
    val[r] = ok ? (vals_in ? __ldg(vals_in + idx) : (uint32_t)idx) : 0u;
    int d = ok ? (int)((key[r] >> shift) & (kRadixDigits - 1)) : kRadixDigits + 1;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    uint32_t b = ok ? wh[warp][d] : 0u;
    loc[r] = b + __popc(peers & lt);
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) wh[warp][d] = b + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRadixDigits; d += kRadixBlock) {
    uint32_t run = gofs[(long long)d * ntiles + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      uint32_t t = wh[w][d];
      wh[w][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    long long idx = wbase + r * 32 + lane;
    if (idx < n) {
      int d = (int)((key[r] >> shift) & (kRadixDigits - 1));
      uint32_t pos = wh[warp][d] + loc[r];
      keys_out[pos] = key[r];
      vals_out[pos] = val[r];
    }
  }
}

struct RadixScratch {
  uint32_t *keys_b = nullptr, *vals_a = nullptr, *vals_b = nullptr;
  uint32_t *hist = nullptr, *scan_tmp = nullptr;
};

inline long long radix_hist_elems(long long n) {
  long long ntiles = (n + kRadixTile - 1) / kRadixTile;
  return ntiles * kRadixDigits;
}

inline int radix_passes(uint32_t max_key) {
  int bits = 0;
  while (bits < 32 && (max_key >> bits) != 0) ++bits;
  int p = (bits + kRadixBits - 1) / kRadixBits;
  return p < 1 ? 1 : p;
}

// Stable sort of (keys, item index) by key.  On return *keys_res / *vals_res
// point at the sorted keys / original item indices (inside keys or scratch).
inline void stable_multisplit(uint32_t *keys, long long n, uint32_t max_key, RadixScratch &s,
                              cudaStream_t st, uint32_t **keys_res, uint32_t **vals_res) {
  int passes = radix_passes(max_key);
  long long ntiles = (n + kRadixTile - 1) / kRadixTile;
  uint32_t *kin = keys, *kout = s.keys_b;
  const uint32_t *vin = nullptr;
  uint32_t *vout = s.vals_a;
  for (int p = 0; p < passes; ++p) {
    int shift = p * kRadixBits;
    if (n > 0) {
      k_radix_hist<<<(unsigned)ntiles, kRadixBlock, 0, st>>>(kin, n, shift, ntiles, s.hist); ++lod::g_launches;
      exclusive_scan<uint32_t>(s.hist, s.hist, ntiles * kRadixDigits, nullptr, s.scan_tmp, st);
      k_radix_scatter<<<(unsigned)ntiles, kRadixBlock, 0, st>>>(kin, vin, n, shift, ntiles, s.hist,
                                                                kout, vout); ++lod::g_launches;
    }
    // ping-pong
    uint32_t *kt = kin;
    kin = kout;
    kout = kt;
    vin = vout;
    vout = (vout == s.vals_a) ? s.vals_b : s.vals_a;
  }
  *keys_res = kin;
  *vals_res = const_cast<uint32_t *>(vin);
}

}  // namespace lod
