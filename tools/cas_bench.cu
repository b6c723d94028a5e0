// Microbenchmark (atomic roofline of the claim path): random 128-bit vs 64-bit CAS installs into an open-addressing table.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cas_bench tools/cas_bench.cu && /tmp/cas_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long hmix(unsigned long long k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdULL; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL; k ^= k >> 33; return k;
}
__device__ __forceinline__ ulonglong2 cas128(ulonglong2 *p, ulonglong2 cmp, ulonglong2 val) {
  ulonglong2 old;
  asm volatile("{\n\t.reg .b128 d, b, c;\n\tmov.b128 b, {%2, %3};\n\tmov.b128 c, {%4, %5};\n\t"
               "atom.global.cas.b128 d, [%6], b, c;\n\tmov.b128 {%0, %1}, d;\n\t}"
               : "=l"(old.x), "=l"(old.y) : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(p) : "memory");
  return old;
}
__global__ void k128(ulonglong2 *t, unsigned long long mask, long long n, unsigned long long salt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long key = hmix(i ^ salt);
    unsigned long long s = hmix(key) & mask;
    for (;;) {
      ulonglong2 cur = __ldcg(t + s);
      if (cur.x == ~0ull) {
        cur = cas128(t + s, make_ulonglong2(~0ull, ~0ull), make_ulonglong2(key, i));
        if (cur.x == ~0ull) break;
      }
      if (cur.x == key) break;
      s = (s + 1) & mask;
    }
  }
}
__global__ void k64(unsigned long long *t, unsigned long long mask, long long n, unsigned long long salt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long key = hmix(i ^ salt) | 1;
    unsigned long long s = hmix(key) & mask;
    for (;;) {
      unsigned long long cur = __ldcg(t + s);
      if (cur == ~0ull) {
        cur = atomicCAS(t + s, ~0ull, key);
        if (cur == ~0ull) break;
      }
      if (cur == key) break;
      s = (s + 1) & mask;
    }
  }
}
int main() {
  const long long n = 1500000;
  for (int lg = 21; lg <= 24; ++lg) {
    const unsigned long long H = 1ull << lg;
    ulonglong2 *t16; unsigned long long *t8;
    cudaMalloc(&t16, H * 16); cudaMalloc(&t8, H * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms16 = 0, ms8 = 0;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(t16, 0xFF, H * 16); cudaMemset(t8, 0xFF, H * 8);
      cudaEventRecord(a); k128<<<2368, 256>>>(t16, H - 1, n, rep); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms16, a, b);
      cudaEventRecord(a); k64<<<2368, 256>>>(t8, H - 1, n, rep); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms8, a, b);
    }
    printf("H=2^%d (16B table %4llu MB, 8B %4llu MB): 1.5M installs  cas128 %.1f us  cas64 %.1f us\n", lg,
           H * 16 >> 20, H * 8 >> 20, ms16 * 1e3, ms8 * 1e3);
    cudaFree(t16); cudaFree(t8);
  }
  return 0;
}
