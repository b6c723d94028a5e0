// lod_route.cu -- multi-GPU point routing, local half.
//
// Every rank holds a stripe of each global batch in global order.  Before the
// all-to-all, its points are bucketed by owner rank -- the rank that owns the
// point's depth-L octant prefix, computed with the reference's exact float64
// descent rule (x >= bx + h per axis, _kernels.py:44-56) -- keeping input
// order inside every bucket, and packed into 16-byte records
// (f32 x, y, z | u32 rgba, store.py:14-16) ready to send.  Three launches:
//   k_route_count   owner per point (kept as a byte), per-tile bucket counts;
//   k_route_scan    per-bucket exclusive scans over the tiles + bucket starts;
//   k_route_scatter warp-ordered stable ranks inside each tile, 16-byte writes.
// The bucket sizes stay on the device for the caller (the split sizes of the
// collective); no host round trip happens here.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <chrono>
#include <mutex>

#include "../../include/lod_b200.h"
#include "lod_common.cuh"
#include "scan.cuh"

using namespace lod;

namespace {

constexpr int kRouteBlock = 256;
constexpr int kRouteRounds = 8;  // per warp: 8 x 32 consecutive points
constexpr int kRouteTile = kRouteBlock * kRouteRounds;
constexpr int kRouteMaxWorld = 64;

// A rank's receive window (one cudaMalloc, shared with the other ranks over
// CUDA IPC; NVLink peer memory between GPUs).  Header: two int64 count
// matrices [source rank][owner rank] (one per half), then per half the
// sources' count-ready and data-ready sequence flags (u64 each); then two
// halves of 16-byte records and two halves of uint32 stripe positions.
// Batch k (sequence k + 1) uses half k & 1, so a sender's next batch never
// lands on records or counts the owner may still read.
constexpr size_t kWindowHeader = LOD_WINDOW_HEADER_BYTES;
constexpr size_t kMatBytes = (size_t)kRouteMaxWorld * kRouteMaxWorld * 8;
constexpr size_t kFlagsOff = 2 * kMatBytes;  // u64 cflag[2][64], u64 dflag[2][64], i64 extra[2][64]
static_assert(kWindowHeader == 2 * kMatBytes + 6 * kRouteMaxWorld * 8, "window header");
__device__ __forceinline__ long long *win_matrix(char *w, int half) {
  return reinterpret_cast<long long *>(w + (size_t)half * kMatBytes);
}
__device__ __forceinline__ unsigned long long *win_cflag(char *w, int half, int src) {
  return reinterpret_cast<unsigned long long *>(w + kFlagsOff) + half * kRouteMaxWorld + src;
}
__device__ __forceinline__ unsigned long long *win_dflag(char *w, int half, int src) {
  return reinterpret_cast<unsigned long long *>(w + kFlagsOff) + (2 + half) * kRouteMaxWorld + src;
}
// one int64 per source rank that rides on the count exchange (the facade:
// the source's count of new replicated-top voxels in its previous batch)
__device__ __forceinline__ long long *win_extra(char *w, int half, int src) {
  return reinterpret_cast<long long *>(w + kFlagsOff) + (4 + half) * kRouteMaxWorld + src;
}
// system-scope release / acquire on the sequence flags (peer memory)
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// One warp: wait until every source's count-ready (data = false) or
// data-ready flag of this half reached `seq`.  Gives up after 30 s (a peer
// that died) so a broken run fails instead of hanging the device; returns
// whether every flag arrived.
constexpr unsigned long long kFlagTimeoutNs = 30ull * 1000 * 1000 * 1000;
__device__ __forceinline__ bool wait_flags(char *own, int world, int half, unsigned long long seq, bool data) {
  const unsigned long long t0 = globaltimer();
  bool ok = true;
  for (int s = threadIdx.x & 31; s < world && ok; s += 32) {
    const unsigned long long *f = data ? win_dflag(own, half, s) : win_cflag(own, half, s);
    while (ld_acquire_sys(f) < seq) {
      if (globaltimer() - t0 > kFlagTimeoutNs) {
        ok = false;
        break;
      }
      __nanosleep(200);
    }
  }
  return __all_sync(0xffffffffu, ok);
}
struct PeerWindows {
  char *p[kRouteMaxWorld];  // p[r] = rank r's window as mapped in this process (own window: local)
};

struct RouteGeo {
  double bmin[3];
  double size;
  int depth;
  int world;
};

__device__ __forceinline__ int owner_of(const RouteGeo &g, const int32_t *__restrict__ table, float xf, float yf,
                                        float zf) {
  const double x = xf, y = yf, z = zf;
  double bx = g.bmin[0], by = g.bmin[1], bz = g.bmin[2], s = g.size;
  int key = 0;
  for (int l = 0; l < g.depth; ++l) key = key * 8 + octant_step(x, y, z, bx, by, bz, s);
  return __ldg(table + key);
}

__global__ void __launch_bounds__(kRouteBlock)
    k_route_count(const float *__restrict__ xyz, long long n, RouteGeo g, const int32_t *__restrict__ table,
                  uint8_t *__restrict__ owner, uint32_t *__restrict__ tile_counts) { lod::pdl_wait();
  __shared__ uint32_t cnt[kRouteMaxWorld];
  for (int d = threadIdx.x; d < g.world; d += kRouteBlock) cnt[d] = 0;
  __syncthreads();
  const long long t0 = (long long)blockIdx.x * kRouteTile;
  for (int r = 0; r < kRouteRounds; ++r) {
    const long long i = t0 + r * kRouteBlock + threadIdx.x;
    if (i < n) {
      const int o = owner_of(g, table, __ldg(xyz + 3 * i), __ldg(xyz + 3 * i + 1), __ldg(xyz + 3 * i + 2));
      owner[i] = (uint8_t)o;
      atomicAdd(&cnt[o], 1u);
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < g.world; d += kRouteBlock) tile_counts[(long long)blockIdx.x * g.world + d] = cnt[d];
}

// One CTA: per bucket, the exclusive scan of its tile counts (in place), the
// bucket totals and the bucket starts (exclusive scan of the totals).
__global__ void __launch_bounds__(1024)
    k_route_scan(uint32_t *__restrict__ tile_counts, long long ntiles, int world, long long *__restrict__ counts,
                 long long *__restrict__ starts) { lod::pdl_wait();
  __shared__ uint32_t sh[1024 / 32 + 1];
  __shared__ long long s_tot[kRouteMaxWorld];
  for (int d = 0; d < world; ++d) {
    uint32_t carry = 0;
    for (long long base = 0; base < ntiles; base += 1024) {
      const long long t = base + threadIdx.x;
      const uint32_t v = t < ntiles ? tile_counts[t * world + d] : 0u;
      uint32_t tot;
      const uint32_t ex = block_exclusive_scan<uint32_t, 1024>(v, sh, tot);
      if (t < ntiles) tile_counts[t * world + d] = carry + ex;
      carry += tot;
    }
    if (threadIdx.x == 0) s_tot[d] = carry;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int d = 0; d < world; ++d) {
      starts[d] = run;
      counts[d] = s_tot[d];
      run += s_tot[d];
    }
  }
}

// Where bucket o of this rank's stripe goes: the local packed buffer at
// starts[o] (lod_route_bucket), or -- the fused peer-memory route -- straight
// into owner o's receive window over NVLink, behind the records of the lower
// source ranks (offset = sum over s < rank of the window count matrix's
// column o, identical on every rank after the count exchange).
// Every record also carries its position in the source stripe (a uint32 in
// a parallel array) so the owner can name each point's global index -- the
// order the replicated top nodes' voxels are merged in (lod_merge_voxels).
struct LocalDest {
  static constexpr bool kRemote = false;
  const long long *starts;
  float4 *out;
  uint32_t *pos;  // may be null
  __device__ float4 *base(int o) const { return out + starts[o]; }
  __device__ uint32_t *pos_base(int o) const { return pos ? pos + starts[o] : nullptr; }
};
struct PeerDest {
  static constexpr bool kRemote = true;
  PeerWindows win;
  int rank, world, half;
  long long half_records;
  __device__ long long offset(int o) const {
    const long long *m = win_matrix(win.p[rank], half);  // my copy of this half's matrix
    long long off = 0;
    for (int s = 0; s < rank; ++s) off += m[s * world + o];
    return off;
  }
  __device__ float4 *base(int o) const {
    return reinterpret_cast<float4 *>(win.p[o] + kWindowHeader) + (long long)half * half_records + offset(o);
  }
  // window layout: header | records half 0 | records half 1 | positions half 0 | positions half 1
  __device__ uint32_t *pos_base(int o) const {
    return reinterpret_cast<uint32_t *>(win.p[o] + kWindowHeader + 2 * half_records * 16) +
           (long long)half * half_records + offset(o);
  }
};

template <typename Dest>
__global__ void __launch_bounds__(kRouteBlock)
    k_route_scatter(const float *__restrict__ xyz, const uint32_t *__restrict__ rgba, long long n, int world,
                    const uint8_t *__restrict__ owner, const uint32_t *__restrict__ tile_off, Dest dest) {
  lod::pdl_wait();
  __shared__ uint32_t wtot[kRouteBlock / 32][kRouteMaxWorld];  // per-warp bucket totals -> warp offsets
  __shared__ uint16_t lrank[kRouteTile];
  __shared__ float4 *s_base[kRouteMaxWorld];
  __shared__ uint32_t *s_pos[kRouteMaxWorld];
  for (int d = threadIdx.x; d < world; d += kRouteBlock) {
    s_base[d] = dest.base(d);
    s_pos[d] = dest.pos_base(d);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  const long long t0 = (long long)blockIdx.x * kRouteTile;
  const int wofs = warp * 32 * kRouteRounds;  // each warp ranks a contiguous run of the tile
  // lane d keeps the warp's running count of bucket d (and d + 32)
  uint32_t run0 = 0, run1 = 0;
  for (int r = 0; r < kRouteRounds; ++r) {
    const int li = wofs + r * 32 + lane;
    const long long i = t0 + li;
    const int o = i < n ? owner[i] : kRouteMaxWorld;  // out-of-range lanes form their own group
    const unsigned peers = __match_any_sync(0xffffffffu, o);
    const uint32_t b0 = __shfl_sync(0xffffffffu, run0, o & 31);  // both shuffles in every lane (converged)
    const uint32_t b1 = __shfl_sync(0xffffffffu, run1, o & 31);
    const uint32_t before = o < 32 ? b0 : b1;
    if (i < n) lrank[li] = (uint16_t)(before + __popc(peers & lt));
    for (int d = 0; d < world; ++d) {  // world <= 64 ballots per round
      const unsigned m = __ballot_sync(0xffffffffu, o == d);
      if (lane == (d & 31)) {
        if (d < 32) run0 += __popc(m);
        else run1 += __popc(m);
      }
    }
  }
  if (lane < world) wtot[warp][lane] = run0;
  if (lane + 32 < world) wtot[warp][lane + 32] = run1;
  __syncthreads();
  for (int d = threadIdx.x; d < world; d += kRouteBlock) {
    uint32_t acc = 0;
    for (int w = 0; w < kRouteBlock / 32; ++w) {
      const uint32_t c = wtot[w][d];
      wtot[w][d] = acc;
      acc += c;
    }
  }
  __syncthreads();
  for (int r = 0; r < kRouteRounds; ++r) {
    const int li = wofs + r * 32 + lane;
    const long long i = t0 + li;
    if (i >= n) continue;
    const int o = owner[i];
    const long long pos = tile_off[(long long)blockIdx.x * world + o] + wtot[warp][o] + lrank[li];
    s_base[o][pos] = make_float4(__ldg(xyz + 3 * i), __ldg(xyz + 3 * i + 1), __ldg(xyz + 3 * i + 2),
                           __uint_as_float(__ldg(rgba + i)));
    if (s_pos[o]) s_pos[o][pos] = (uint32_t)i;
  }
  if (Dest::kRemote) __threadfence_system();  // the records are performed before k_route_signal's flags
}

// The count exchange (one CTA): this rank's bucket sizes become row `rank`
// of every peer's count matrix for this half (world x world remote 8-byte
// stores), then each peer's count-ready flag of this rank is released.
// A rank publishes batch k only after its own insert of batch k - 2 (the
// caller's stream is ordered behind it), so a peer that sees every rank's
// flag of batch k knows every window's half k & 1 is free again.
__global__ void __launch_bounds__(1024)
    k_route_publish(const long long *__restrict__ counts, int rank, int world, PeerWindows win, int half,
                    unsigned long long seq, const long long *extra) {
  lod::pdl_wait();
  for (int t = threadIdx.x; t < world * world; t += blockDim.x) {
    const int peer = t / world, o = t % world;
    win_matrix(win.p[peer], half)[rank * world + o] = counts[o];
  }
  if (threadIdx.x < world) *win_extra(win.p[threadIdx.x], half, rank) = extra ? *extra : 0;
  __syncthreads();
  if (threadIdx.x < world) {
    __threadfence_system();
    st_release_sys(win_cflag(win.p[threadIdx.x], half, rank), seq);
  }
}

// Wait (one warp) for every rank's counts of batch `seq`, then hand this
// half's matrix to the host through mapped memory (host_seq last).
__global__ void k_route_wait_counts(char *own, int world, int half, unsigned long long seq, long long *host_mat,
                                    volatile unsigned long long *host_seq) {
  lod::pdl_wait();
  const bool ok = wait_flags(own, world, half, seq, false);
  const long long *m = win_matrix(own, half);
  for (int t = threadIdx.x; t < world * world; t += 32) host_mat[t] = __ldcg(m + t);
  for (int t = threadIdx.x; t < world; t += 32) host_mat[world * world + t] = __ldcg(win_extra(own, half, t));
  __threadfence_system();
  __syncwarp();
  if (threadIdx.x == 0) *host_seq = ok ? seq : ~0ull;
}

// After the scatter: release this rank's data-ready flag in every owner's
// window (the scatter fenced its records at system scope).
__global__ void k_route_signal(PeerWindows win, int rank, int world, int half, unsigned long long seq) {
  lod::pdl_wait();
  if (threadIdx.x < world) st_release_sys(win_dflag(win.p[threadIdx.x], half, rank), seq);
}

// The owner's side: wait (one warp) until every source's records of batch
// `seq` are in; the insert behind it on the stream reads them.
__global__ void k_route_wait_data(char *own, int world, int half, unsigned long long seq) {
  lod::pdl_wait();
  wait_flags(own, world, half, seq, true);
}

// Depth-min composite over peer memory, reduce-scatter and all-gather fused:
// rank r owns pixel slice r; for each of its pixels it reads every rank's
// framebuffer, takes the unsigned 64-bit min (the all-ones sentinel is the
// largest value, so it needs no mapping) and writes the result back into every
// rank's framebuffer.  Slices are disjoint, so the ranks' kernels never touch
// the same word.  Two pixels per thread (16-byte loads/stores).
__global__ void __launch_bounds__(256)
    k_composite_min(PeerWindows fb, int world, long long lo, long long hi) {
  lod::pdl_wait();
  const long long stride = (long long)gridDim.x * blockDim.x * 2;
  for (long long i = lo + ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 2; i < hi; i += stride) {
    if (i + 1 < hi && (i & 1) == 0) {
      ulonglong2 m = make_ulonglong2(~0ull, ~0ull);
      for (int r = 0; r < world; ++r) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(fb.p[r] + i * 8);
        m.x = v.x < m.x ? v.x : m.x;
        m.y = v.y < m.y ? v.y : m.y;
      }
      for (int r = 0; r < world; ++r) *reinterpret_cast<ulonglong2 *>(fb.p[r] + i * 8) = m;
    } else {
      for (long long j = i; j < i + 2 && j < hi; ++j) {
        unsigned long long m = ~0ull;
        for (int r = 0; r < world; ++r) {
          const unsigned long long v = reinterpret_cast<const unsigned long long *>(fb.p[r])[j];
          m = v < m ? v : m;
        }
        for (int r = 0; r < world; ++r) reinterpret_cast<unsigned long long *>(fb.p[r])[j] = m;
      }
    }
  }
  __threadfence_system();
}

inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

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

struct RouteScratch {
  uint8_t *owner = nullptr;
  uint32_t *tiles = nullptr;
  int32_t *table = nullptr;
  long long *counts = nullptr, *starts = nullptr;  // device, for the peer route
  long long *h_mat = nullptr, *h_mat_dev = nullptr;  // mapped: a half's count matrix + its sequence word
  volatile unsigned long long *h_seq = nullptr;
  unsigned long long *h_flags = nullptr;  // pinned: polled flags (host-wait mode)
  cudaStream_t pst = nullptr;             // polling stream (host-wait mode)
  long long cap = 0, tcap = 0, table_cap = 0;
};
std::mutex g_mu;
RouteScratch g_rs[64];

// Owners, per-tile bucket counts and their scans (the first two launches of
// both routes); counts / starts are device arrays of `world` entries.
int route_prepare(RouteScratch &s, const double *bmin, double size, int depth, const int32_t *owner_of_prefix,
                  int world, const float *xyz, long long n, long long *counts, long long *starts, cudaStream_t st) {
  const long long ntiles = std::max<long long>((n + kRouteTile - 1) / kRouteTile, 1);
  if (n > s.cap) {
    if (s.owner) cudaFree(s.owner);
    s.cap = std::max<long long>(n, 2 * s.cap);
    CK(cudaMalloc(&s.owner, (size_t)s.cap));
  }
  if (ntiles * world > s.tcap) {
    if (s.tiles) cudaFree(s.tiles);
    s.tcap = std::max<long long>(ntiles * world, 2 * s.tcap);
    CK(cudaMalloc(&s.tiles, (size_t)s.tcap * 4));
  }
  const long long tsize = 1LL << (3 * depth);
  if (tsize > s.table_cap) {
    if (s.table) cudaFree(s.table);
    s.table_cap = tsize;
    CK(cudaMalloc(&s.table, (size_t)tsize * 4));
  }
  for (long long k = 0; k < tsize; ++k)
    if (owner_of_prefix[k] < 0 || owner_of_prefix[k] >= world) return LOD_E_ARG;
  CK(cudaMemcpyAsync(s.table, owner_of_prefix, (size_t)tsize * 4, cudaMemcpyHostToDevice, st));
  RouteGeo g;
  memcpy(g.bmin, bmin, sizeof(g.bmin));
  g.size = size;
  g.depth = depth;
  g.world = world;
  if (n > 0)
    lod::launch(k_route_count, cdiv(n, kRouteTile), kRouteBlock, 0, st, xyz, n, g, s.table, s.owner, s.tiles);
  else
    CK(cudaMemsetAsync(s.tiles, 0, (size_t)world * 4, st));
  lod::launch(k_route_scan, 1, 1024, 0, st, s.tiles, ntiles, world, counts, starts);
  return LOD_OK;
}

#define RK_(expr)            \
  do {                       \
    int rc__ = (expr);       \
    if (rc__) return rc__;   \
  } while (0)

// Host-wait mode (ranks time-sliced on one device, where a spinning wait
// kernel would hold the device until its time slice ends): poll this half's
// count-ready (data = false) or data-ready flags in the own window with small
// copies on a private stream until every source's reached `seq` (30 s cap).
int host_poll(RouteScratch &s, char *own, int world, int half, unsigned long long seq, bool data) {
  if (!s.pst) {
    CK(cudaStreamCreateWithFlags(&s.pst, cudaStreamNonBlocking));
    CK(cudaHostAlloc(&s.h_flags, kRouteMaxWorld * 8, cudaHostAllocDefault));
  }
  const char *f = own + kFlagsOff + (size_t)((data ? 2 : 0) + half) * kRouteMaxWorld * 8;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    CK(cudaMemcpyAsync(s.h_flags, f, (size_t)world * 8, cudaMemcpyDeviceToHost, s.pst));
    CK(cudaStreamSynchronize(s.pst));
    bool all = true;
    for (int r = 0; r < world; ++r) all &= s.h_flags[r] >= seq;
    if (all) return LOD_OK;
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30)) return LOD_E_CUDA;
  }
}

bool windows_ok(void *const *w, int world) {
  if (!w) return false;
  for (int r = 0; r < world; ++r)
    if (!w[r]) return false;
  return true;
}

PeerWindows pack_windows(void *const *w, int world) {
  PeerWindows pw{};
  for (int r = 0; r < world; ++r) pw.p[r] = static_cast<char *>(w[r]);
  return pw;
}

}  // namespace

extern "C" {

int lod_route_bucket(int32_t device, const double *bmin, double size, int32_t depth, const int32_t *owner_of_prefix,
                     int32_t world, const float *xyz, const uint32_t *rgba, int64_t n, void *out_records,
                     uint32_t *out_positions, int64_t *counts, int64_t *starts, void *stream) {
  if (!bmin || !owner_of_prefix || depth < 0 || depth > 8 || world < 1 || world > kRouteMaxWorld || n < 0 ||
      (n > 0 && (!xyz || !rgba || !out_records)) || !counts || !starts || device < 0 || device >= 64)
    return LOD_E_ARG;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaSetDevice(device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  RouteScratch &s = g_rs[device];
  int rc = route_prepare(s, bmin, size, depth, owner_of_prefix, world, xyz, n, (long long *)counts,
                         (long long *)starts, st);
  if (rc) return rc;
  if (n > 0)
    lod::launch(k_route_scatter<LocalDest>, cdiv(n, kRouteTile), kRouteBlock, 0, st, xyz, rgba, (long long)n,
                (int)world, s.owner, s.tiles,
                LocalDest{(const long long *)starts, reinterpret_cast<float4 *>(out_records), out_positions});
  return cuda_rc(cudaGetLastError());
}

int lod_ipc_alloc(int32_t device, uint64_t bytes, void **ptr, void *handle) {
  if (!ptr || !handle || device < 0) return LOD_E_ARG;
  cudaSetDevice(device);
  if (cudaMalloc(ptr, bytes ? bytes : 1) != cudaSuccess) {
    cudaGetLastError();
    return LOD_E_NOMEM;
  }
  CK(cudaMemset(*ptr, 0, bytes ? bytes : 1));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, *ptr));
  static_assert(sizeof(h) == LOD_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  return cuda_rc(cudaDeviceSynchronize());
}

int lod_ipc_open(int32_t device, const void *handle, void **ptr) {
  if (!ptr || !handle || device < 0) return LOD_E_ARG;
  cudaSetDevice(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cuda_rc(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
}

int lod_ipc_close(void *ptr) { return cuda_rc(cudaIpcCloseMemHandle(ptr)); }

int lod_route_peers_begin(int32_t device, const double *bmin, double size, int32_t depth,
                          const int32_t *owner_of_prefix, int32_t world, int32_t rank, const float *xyz, int64_t n,
                          void *const *windows, int32_t half, uint64_t seq, const int64_t *extra_dev,
                          int64_t *matrix, int64_t *extra, int32_t host_wait, void *stream) {
  if (!bmin || !owner_of_prefix || depth < 0 || depth > 8 || world < 1 || world > kRouteMaxWorld || rank < 0 ||
      rank >= world || n < 0 || (n > 0 && !xyz) || !windows_ok(windows, world) || device < 0 || device >= 64 ||
      half < 0 || half > 1 || seq == 0 || seq == ~0ull || !matrix)
    return LOD_E_ARG;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaSetDevice(device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  RouteScratch &s = g_rs[device];
  if (!s.counts) {
    CK(cudaMalloc(&s.counts, 2 * kRouteMaxWorld * sizeof(long long)));
    s.starts = s.counts + kRouteMaxWorld;
    CK(cudaHostAlloc(&s.h_mat, kMatBytes + kRouteMaxWorld * 8 + 8, cudaHostAllocMapped));
    s.h_seq = reinterpret_cast<volatile unsigned long long *>(reinterpret_cast<char *>(s.h_mat) + kMatBytes +
                                                              kRouteMaxWorld * 8);
    *s.h_seq = 0;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void **>(&s.h_mat_dev), s.h_mat, 0));
  }
  int rc = route_prepare(s, bmin, size, depth, owner_of_prefix, world, xyz, n, s.counts, s.starts, st);
  if (rc) return rc;
  const PeerWindows pw = pack_windows(windows, world);
  *s.h_seq = 0;  // the previous wait kernel is done (its word was seen): no stale match
  lod::launch(k_route_publish, 1, 1024, 0, st, (const long long *)s.counts, (int)rank, (int)world, pw, (int)half,
              (unsigned long long)seq, (const long long *)extra_dev);
  if (host_wait) {
    RK_(host_poll(s, pw.p[rank], world, half, seq, false));
    CK(cudaMemcpyAsync(s.h_mat, pw.p[rank] + (size_t)half * kMatBytes, (size_t)world * world * 8,
                       cudaMemcpyDeviceToHost, s.pst));
    CK(cudaMemcpyAsync(s.h_mat + world * world, pw.p[rank] + kFlagsOff + (size_t)(4 + half) * kRouteMaxWorld * 8,
                       (size_t)world * 8, cudaMemcpyDeviceToHost, s.pst));
    CK(cudaStreamSynchronize(s.pst));
    for (int t = 0; t < world * world; ++t) matrix[t] = s.h_mat[t];
    if (extra)
      for (int t = 0; t < world; ++t) extra[t] = s.h_mat[world * world + t];
    return LOD_OK;
  }
  lod::launch(k_route_wait_counts, 1, 32, 0, st, pw.p[rank], (int)world, (int)half, (unsigned long long)seq,
              s.h_mat_dev, (volatile unsigned long long *)(s.h_mat_dev + kMatBytes / 8 + kRouteMaxWorld));
  CK(cudaGetLastError());
  // the host needs the matrix (window sizes, this rank's record count):
  // poll the mapped sequence word the wait kernel writes last
  for (unsigned spins = 0; *s.h_seq != seq; ++spins) {
    if (*s.h_seq == ~0ull) return LOD_E_CUDA;  // a peer's counts never arrived
    if ((spins & 1023) == 1023) {
      const cudaError_t e = cudaStreamQuery(st);
      if (e != cudaSuccess && e != cudaErrorNotReady) return cuda_rc(e);
      if (e == cudaSuccess && *s.h_seq != seq) return LOD_E_CUDA;  // drained without the write
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  for (int t = 0; t < world * world; ++t) matrix[t] = s.h_mat[t];
  if (extra)
    for (int t = 0; t < world; ++t) extra[t] = s.h_mat[world * world + t];
  return LOD_OK;
}

int lod_route_peers_finish(int32_t device, int32_t world, int32_t rank, const float *xyz, const uint32_t *rgba,
                           int64_t n, void *const *windows, int32_t half, int64_t half_records, uint64_t seq,
                           int32_t host_wait, void *stream) {
  if (world < 1 || world > kRouteMaxWorld || rank < 0 || rank >= world || n < 0 || (n > 0 && (!xyz || !rgba)) ||
      !windows_ok(windows, world) || half < 0 || half > 1 || half_records < 0 || device < 0 || device >= 64 ||
      seq == 0 || seq == ~0ull)
    return LOD_E_ARG;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaSetDevice(device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  RouteScratch &s = g_rs[device];
  if (n > s.cap) return LOD_E_ARG;  // begin() sized the scratch for this stripe
  const PeerWindows pw = pack_windows(windows, world);
  if (n > 0)
    lod::launch(k_route_scatter<PeerDest>, cdiv(n, kRouteTile), kRouteBlock, 0, st, xyz, rgba, (long long)n,
                (int)world, s.owner, s.tiles, PeerDest{pw, (int)rank, (int)world, (int)half, (long long)half_records});
  lod::launch(k_route_signal, 1, 64, 0, st, pw, (int)rank, (int)world, (int)half, (unsigned long long)seq);
  if (host_wait) return host_poll(s, pw.p[rank], world, half, seq, true);
  lod::launch(k_route_wait_data, 1, 32, 0, st, pw.p[rank], (int)world, (int)half, (unsigned long long)seq);
  return cuda_rc(cudaGetLastError());
}

int lod_composite_min_peers(int32_t device, int32_t world, int32_t rank, void *const *fbs, int64_t npix,
                            void *stream) {
  if (world < 1 || world > kRouteMaxWorld || rank < 0 || rank >= world || npix < 0 || !windows_ok(fbs, world) ||
      device < 0)
    return LOD_E_ARG;
  cudaSetDevice(device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // slice boundaries even, so the 16-byte accesses stay aligned
  const long long per = ((npix + world - 1) / world + 1) & ~1LL;
  const long long lo = std::min<long long>(npix, per * rank), hi = std::min<long long>(npix, lo + per);
  if (hi > lo) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const unsigned grid = std::min<long long>(cdiv(hi - lo, 512), 4LL * sms);
    lod::launch(k_composite_min, grid, 256, 0, st, pack_windows(fbs, world), (int)world, lo, hi);
  }
  return cuda_rc(cudaGetLastError());
}

}  // extern "C"
