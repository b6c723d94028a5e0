// lod_morton.cu -- device Morton order (reference
// lodstream/io.py:419-446, morton_key / morton_sort).
//
// Keys restate io.py bit for bit: per axis q = int64((x - min) * scale) with
// scale = (1 << bits) / size computed by the caller exactly like the reference,
// f64 arithmetic, truncation toward zero (out-of-range / NaN -> INT64_MIN as
// numba/numpy on x86), clip to [0, 2^bits - 1], bits spread 3 apart, x at bit
// 0, y at 1, z at 2.  The sort is the reference's stable argsort: an LSD radix
// sort of the 3*bits-bit keys (onesweep passes of radix.cuh), low word first,
// then the high word carrying the permutation; the records are gathered once.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/lod_b200.h"
#include "lod_common.cuh"
#include "radix.cuh"
#include "scan.cuh"

using namespace lod;

namespace {

__device__ __forceinline__ unsigned long long spread_bits(unsigned long long v) {  // io.py:418-427
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x1F00000000FFFFull;
  v = (v | (v << 16)) & 0x1F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

struct MortonGeo {
  double bmin[3];
  double scale;
  long long top;
};

__global__ void k_morton_keys(const float *__restrict__ xyz, long long n, MortonGeo g, uint32_t *__restrict__ lo,
                              uint32_t *__restrict__ hi, unsigned long long *__restrict__ keys) { lod::pdl_wait();
  for (long long i = gtid(); i < n; i += gstride()) {
    unsigned long long key = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      long long q = f2i64(((double)__ldg(xyz + 3 * i + a) - g.bmin[a]) * g.scale);
      q = q < 0 ? 0 : (q > g.top ? g.top : q);
      key |= spread_bits((unsigned long long)q) << a;
    }
    lo[i] = (uint32_t)key;
    hi[i] = (uint32_t)(key >> 32);
    if (keys) keys[i] = key;
  }
}

__global__ void k_gather_u32(const uint32_t *__restrict__ src, const uint32_t *__restrict__ perm, long long n,
                             uint32_t *__restrict__ dst) { lod::pdl_wait();
  for (long long i = gtid(); i < n; i += gstride()) dst[i] = __ldg(src + perm[i]);
}

__global__ void k_morton_gather(const float *__restrict__ xyz, const uint32_t *__restrict__ rgba,
                                const uint32_t *__restrict__ perm, long long n, float *__restrict__ xyz_out,
                                uint32_t *__restrict__ rgba_out) { lod::pdl_wait();
  for (long long i = gtid(); i < n; i += gstride()) {
    const long long j = perm[i];
    if (xyz_out) {
      xyz_out[3 * i] = __ldg(xyz + 3 * j);
      xyz_out[3 * i + 1] = __ldg(xyz + 3 * j + 1);
      xyz_out[3 * i + 2] = __ldg(xyz + 3 * j + 2);
    }
    if (rgba_out) rgba_out[i] = __ldg(rgba + j);
  }
}

inline unsigned grid_for(long long n, int block = 256) {
  long long b = (n + block - 1) / block;
  if (b < 1) b = 1;
  return (unsigned)std::min<long long>(b, 148LL * 16);
}

int cuda_rc(cudaError_t e) {
  if (e == cudaSuccess) return LOD_OK;
  fprintf(stderr, "[lod_b200] CUDA error: %s\n", cudaGetErrorString(e));
  return LOD_E_CUDA;
}
#define CK(expr)               \
  do {                         \
    int rc__ = cuda_rc(expr);  \
    if (rc__) return rc__;     \
  } while (0)

// Per-device scratch, grown on demand (one Morton sort at a time per device).
struct MortonScratch {
  cudaStream_t st = nullptr;
  long long cap = 0;
  float *xyz = nullptr, *xyz_out = nullptr;
  uint32_t *rgba = nullptr, *rgba_out = nullptr;
  unsigned long long *keys_out = nullptr;
  uint32_t *lo = nullptr, *hi = nullptr, *k0 = nullptr, *kb = nullptr, *v[3] = {nullptr, nullptr, nullptr};
  uint32_t *lb = nullptr, *ghist = nullptr;
};
std::mutex g_mu;
MortonScratch g_ms[64];

int ensure(MortonScratch &s, long long n) {
  if (n <= s.cap) return LOD_OK;
  const long long c = std::max<long long>(n, 2 * s.cap);
  void **bufs[] = {(void **)&s.xyz, (void **)&s.xyz_out, (void **)&s.rgba, (void **)&s.rgba_out,
                   (void **)&s.keys_out, (void **)&s.lo, (void **)&s.hi, (void **)&s.k0, (void **)&s.kb,
                   (void **)&s.v[0], (void **)&s.v[1], (void **)&s.v[2], (void **)&s.lb};
  const size_t sizes[] = {(size_t)c * 12, (size_t)c * 12, (size_t)c * 4, (size_t)c * 4, (size_t)c * 8, (size_t)c * 4,
                          (size_t)c * 4, (size_t)c * 4, (size_t)c * 4, (size_t)c * 4, (size_t)c * 4, (size_t)c * 4,
                          (size_t)(2 * radix_lb_elems(c)) * 4};
  for (size_t k = 0; k < sizeof(sizes) / sizeof(sizes[0]); ++k) {
    if (*bufs[k]) cudaFree(*bufs[k]);
    *bufs[k] = nullptr;
    if (cudaMalloc(bufs[k], sizes[k]) != cudaSuccess) {
      cudaGetLastError();
      s.cap = 0;
      return LOD_E_NOMEM;
    }
  }
  if (!s.ghist) CK(cudaMalloc(&s.ghist, kMaxPasses * kRadixDigits * 4));
  s.cap = c;
  return LOD_OK;
}

// One stable LSD round over `passes` digits of a u32 key word; returns the
// permutation buffer it ends in (never `avoid`).
uint32_t *radix_round(MortonScratch &s, uint32_t *keys, const uint32_t *vals0, long long n, int passes,
                      uint32_t *va, uint32_t *vb, cudaStream_t st) {
  const long long lbw = radix_lb_elems(n);
  cudaMemsetAsync(s.ghist, 0, kMaxPasses * kRadixDigits * 4, st);
  cudaMemsetAsync(s.lb, 0, (size_t)lbw * 4, st);
  lod::launch(k_digit_hist, std::min<unsigned>(grid_for(n), 148 * 4), 256, 0, st, keys, n, 0, passes, s.ghist);
  RadixScratch rs;
  rs.keys_b = s.kb;
  rs.vals_a = va;
  rs.vals_b = vb;
  rs.ghist = s.ghist;
  rs.lb[0] = s.lb;
  rs.lb[1] = s.lb + lbw;
  uint32_t *sk = nullptr, *sv = nullptr;
  stable_multisplit(keys, n, passes, rs, st, &sk, &sv, vals0);
  return sv;
}

}  // namespace

extern "C" {

int lod_morton_sort(int32_t device, const double *bmin, double scale, int32_t bits, const float *xyz,
                    const uint32_t *rgba, int64_t n, float *xyz_out, uint32_t *rgba_out, uint64_t *keys_out,
                    int flags) {
  if (!bmin || bits < 1 || bits > 21 || n < 0 || device < 0 || device >= 64 || (n > 0 && !xyz) ||
      (rgba_out && !rgba) || n >= (1LL << 31))
    return LOD_E_ARG;
  if (n == 0) return LOD_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev) {
    cudaGetLastError();
    return LOD_E_NO_DEVICE;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  cudaSetDevice(device);
  MortonScratch &s = g_ms[device];
  if (!s.st) CK(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
  int rc = ensure(s, n);
  if (rc) return rc;
  cudaStream_t st = s.st;
  const bool dev = (flags & LOD_FLAG_DEVICE_INPUT) != 0;
  const float *dx = xyz;
  const uint32_t *dc = rgba;
  if (!dev) {
    CK(cudaMemcpyAsync(s.xyz, xyz, (size_t)n * 12, cudaMemcpyHostToDevice, st));
    dx = s.xyz;
    if (rgba) {
      CK(cudaMemcpyAsync(s.rgba, rgba, (size_t)n * 4, cudaMemcpyHostToDevice, st));
      dc = s.rgba;
    }
  }
  MortonGeo g;
  memcpy(g.bmin, bmin, sizeof(g.bmin));
  g.scale = scale;
  g.top = (1LL << bits) - 1;
  unsigned long long *ok = dev ? reinterpret_cast<unsigned long long *>(keys_out) : (keys_out ? s.keys_out : nullptr);
  lod::launch(k_morton_keys, grid_for(n), 256, 0, st, dx, (long long)n, g, s.lo, s.hi, ok);
  if (!dev && keys_out) CK(cudaMemcpyAsync(keys_out, s.keys_out, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  if (xyz_out || rgba_out) {
    const int kbits = 3 * bits;
    const int p_lo = (std::min(kbits, 32) + kRadixBits - 1) / kRadixBits;
    const int p_hi = kbits > 32 ? (kbits - 32 + kRadixBits - 1) / kRadixBits : 0;
    // round 1: low words (a copy in k0: the key array is overwritten), identity
    // permutation in, permutation out in v0 or v1
    CK(cudaMemcpyAsync(s.k0, s.lo, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    uint32_t *perm = radix_round(s, s.k0, nullptr, n, p_lo, s.v[0], s.v[1], st);
    if (p_hi) {
      // round 2: high words in round-1 order, carrying round 1's permutation
      uint32_t *spare = perm == s.v[0] ? s.v[1] : s.v[0];
      lod::launch(k_gather_u32, grid_for(n), 256, 0, st, s.hi, perm, (long long)n, s.k0);
      perm = radix_round(s, s.k0, perm, n, p_hi, s.v[2], spare, st);
    }
    float *ox = dev ? xyz_out : (xyz_out ? s.xyz_out : nullptr);
    uint32_t *oc = dev ? rgba_out : (rgba_out ? s.rgba_out : nullptr);
    lod::launch(k_morton_gather, grid_for(n), 256, 0, st, dx, dc, perm, (long long)n, ox, oc);
    if (!dev) {
      if (xyz_out) CK(cudaMemcpyAsync(xyz_out, s.xyz_out, (size_t)n * 12, cudaMemcpyDeviceToHost, st));
      if (rgba_out) CK(cudaMemcpyAsync(rgba_out, s.rgba_out, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    }
  }
  CK(cudaStreamSynchronize(st));
  return LOD_OK;
}

}  // extern "C"
