// lod_raster.cu -- compute rasterizers (render.rasterize / brute_force_render).
//
// Projection, depth and packing restate _kernels.py:290-372 exactly (f64, no
// FMA, IEEE division, float32 depth bits << 32 | rgba, min-combine).  The
// per-node chunk walk of rasterize_nodes becomes a work list over the listed
// nodes' chunks (each node's chunk directory, maintained by the update path),
// cut into pieces of kPiece records, one warp per piece, with an early depth
// test before the 64-bit atomicMin: O(visible samples).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/lod_b200.h"
#include "lod_common.cuh"
#include "scan.cuh"

using namespace lod;

struct LodTree;
cudaStream_t lod_tree_stream(LodTree *t);
int lod_tree_device(LodTree *t);
const uint8_t *lod_tree_arena(LodTree *t);
PoolCols lod_tree_pool(LodTree *t);
long long lod_tree_num_nodes(LodTree *t);
int lod_tree_ensure_woff(LodTree *t, long long n, long long **p);
int lod_tree_ensure_vislist(LodTree *t, long long n, int32_t **p);
int lod_tree_ensure_fb(LodTree *t, long long n, unsigned long long **p);
unsigned long long *lod_tree_counter(LodTree *t);
NodeCols lod_tree_nodes(LodTree *t);
Geo lod_tree_geo(LodTree *t);
int lod_tree_ensure_sel(LodTree *t, long long n, int32_t **a, int32_t **b);

namespace {

struct Cam {
  double c[18];
};

__device__ __forceinline__ void splat(const Cam &cam, long long w, long long h, double x, double y, double z,
                                      uint32_t rgba, unsigned long long *fb) {
  const double *c = cam.c;
  const double dx = x - c[0], dy = y - c[1], dz = z - c[2];
  const double zv = dx * c[9] + dy * c[10] + dz * c[11];
  if (zv <= c[14] || zv >= c[15]) return;
  const double xv = dx * c[3] + dy * c[4] + dz * c[5];
  const double yv = dx * c[6] + dy * c[7] + dz * c[8];
  const double ndc_x = xv / (zv * c[12] * c[13]);
  const double ndc_y = yv / (zv * c[12]);
  const long long px = f2i64(floor((ndc_x + 1.0) * 0.5 * c[16]));
  const long long py = f2i64(floor((1.0 - ndc_y) * 0.5 * c[17]));
  if (px < 0 || px >= w || py < 0 || py >= h) return;
  const double d01 = c[15] * (zv - c[14]) / ((c[15] - c[14]) * zv);
  const unsigned long long packed =
      ((unsigned long long)__float_as_uint(__double2float_rn(d01)) << 32) | (unsigned long long)rgba;
  unsigned long long *cell = fb + (py * w + px);
  if (packed < __ldcg(cell)) atomicMin(cell, packed);
}

__global__ void k_raster_points(const float *__restrict__ xyz, const uint32_t *__restrict__ rgba, long long n,
                                Cam cam, unsigned long long *fb, long long w, long long h) { lod::pdl_wait();
  for (long long i = gtid(); i < n; i += gstride())
    splat(cam, w, h, (double)__ldg(xyz + 3 * i), (double)__ldg(xyz + 3 * i + 1), (double)__ldg(xyz + 3 * i + 2),
          __ldg(rgba + i), fb);
}

// rasterize_nodes (_kernels.py:290-339) over a work list that is O(visible):
// every listed node contributes chunk_count x ppc pieces of at most kPiece
// records (ppc = ceil(C / kPiece)), addressed through the node's chunk
// directory -- so the cost follows the visible samples, not the pool size or
// the chunk capacity (acceptance C9: render time flat across C).  `woff` is
// the exclusive scan of the entries' piece counts (k_select / k_vis_plan),
// plan[0] = samples drawn (every listed occurrence, _kernels.py:307-317),
// plan[2] = pieces.  One warp per piece.
constexpr int kPiece = 256;
__global__ void __launch_bounds__(256)
    k_raster_work(NodeCols nd, PoolCols pool, const uint8_t *__restrict__ arena, const int32_t *__restrict__ list,
                  const long long *__restrict__ woff, const unsigned long long *__restrict__ plan, int ppc, Cam cam,
                  unsigned long long *fb, long long w, long long h) { lod::pdl_wait();
  const long long warp = gtid() >> 5, nwarps = gstride() >> 5;
  const int lane = threadIdx.x & 31;
  const long long n = (long long)plan[1], pieces = (long long)plan[2];
  for (long long p = warp; p < pieces; p += nwarps) {
    long long lo = 0, hi = n - 1;  // last entry whose pieces start at or before p
    while (lo < hi) {
      const long long mid = (lo + hi + 1) >> 1;
      if (woff[mid] <= p) lo = mid;
      else hi = mid - 1;
    }
    const int nid = list[lo];
    const long long k = p - woff[lo], ci = k / ppc, r0 = (k % ppc) * kPiece;
    const int cid = pool.cdir[nd.dir_off[nid] + ci];
    const long long r1 = min((long long)pool.occupied[cid], r0 + kPiece);
    const float4 *rec = reinterpret_cast<const float4 *>(arena + pool.payload_off[cid]);
    for (long long r = r0 + lane; r < r1; r += 32) {
      const float4 v = __ldg(rec + r);
      splat(cam, w, h, (double)v.x, (double)v.y, (double)v.z, __float_as_uint(v.w), fb);
    }
  }
}

// Work-list plan of an explicit node list (lod_rasterize): piece offsets,
// samples, count.  One CTA.
constexpr int kPlanBlock = 1024;
__device__ __forceinline__ void plan_entries(const NodeCols &nd, const int32_t *list, long long n, int ppc,
                                             long long *woff, unsigned long long *plan, U64x2 *sh) {
  U64x2 carry = u64x2(0, 0);
  for (long long base = 0; base < n; base += kPlanBlock) {
    const long long i = base + threadIdx.x;
    U64x2 v = u64x2(0, 0);
    if (i < n) {
      const int nid = list[i];
      v = u64x2((unsigned long long)nd.chunk_count[nid] * (unsigned long long)ppc, (unsigned long long)nd.count[nid]);
    }
    U64x2 tot;
    const U64x2 ex = block_exclusive_scan<U64x2, kPlanBlock>(v, sh, tot);
    if (i < n) woff[i] = (long long)(ex.a + carry.a);
    carry = carry + tot;
  }
  if (threadIdx.x == 0) {
    plan[0] = carry.b;
    plan[1] = (unsigned long long)n;
    plan[2] = carry.a;
  }
}

__global__ void __launch_bounds__(kPlanBlock)
    k_vis_plan(NodeCols nd, const int32_t *__restrict__ list, long long n, int ppc, long long *woff,
               unsigned long long *plan) { lod::pdl_wait();
  __shared__ U64x2 sh[kPlanBlock / 32 + 1];
  plan_entries(nd, list, n, ppc, woff, plan, sh);
}

// ---------------------------------------------------------------- selection

// select_visible (render.py:177-200) on the device.  The reference walks a
// stack depth-first (octant order) and emits every node where the walk stops:
// outside the frustum -> dropped, inner and projecting larger than the pixel
// threshold -> refined into its 8 children, else -> drawn.  Here one CTA keeps
// the whole cut as an ordered list and refines it level by level: every
// pending entry is replaced in place by 0 (culled), 1 (drawn, final) or 8
// (its children, pending) entries, with a block scan placing them.  Replacing
// an entry by its children in octant order keeps the list in depth-first
// order, so the final list is the reference's visit order.  The plane and
// projection arithmetic is the reference's per corner, in f64 without FMA
// (frustum_intersects render.py:151-157, screen_size render.py:160-174).
struct SelParams {
  double planes[24];  // frustum_planes(camera): (normal, d) x 6, host-computed like the reference
  double cam[18];     // Camera.packed()
  double threshold;
};

__device__ __forceinline__ int sel_decide(const NodeCols &nd, const Geo &geo, const SelParams &sp, int nid) {
  const double s = geo.size_by_level[nd.level[nid]];
  const double b0 = nd.bmin[3 * nid], b1 = nd.bmin[3 * nid + 1], b2 = nd.bmin[3 * nid + 2];
  double cx[8], cy[8], cz[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {  // CubeBounds.corners(): corner i at octant offset i
    cx[i] = b0 + ((i & 1) ? s : 0.0);
    cy[i] = b1 + ((i & 2) ? s : 0.0);
    cz[i] = b2 + ((i & 4) ? s : 0.0);
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double *pl = sp.planes + 4 * k;
    bool all_out = true;
#pragma unroll
    for (int i = 0; i < 8; ++i) all_out &= (cx[i] * pl[0] + cy[i] * pl[1] + cz[i] * pl[2] + pl[3] < 0.0);
    if (all_out) return 0;
  }
  if (!nd.inner[nid]) return 1;
  const double *c = sp.cam;
  double sxmin = 0, sxmax = 0, symin = 0, symax = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const double dx = cx[i] - c[0], dy = cy[i] - c[1], dz = cz[i] - c[2];
    const double zv = dx * c[9] + dy * c[10] + dz * c[11];
    if (zv <= c[14]) return ((double)INFINITY > sp.threshold) ? 8 : 1;  // screen_size = inf
    const double sx = ((dx * c[3] + dy * c[4] + dz * c[5]) / (zv * c[12] * c[13]) + 1.0) * 0.5 * c[16];
    const double sy = (1.0 - (dx * c[6] + dy * c[7] + dz * c[8]) / (zv * c[12])) * 0.5 * c[17];
    if (i == 0) {
      sxmin = sxmax = sx;
      symin = symax = sy;
    } else {
      sxmin = fmin(sxmin, sx);
      sxmax = fmax(sxmax, sx);
      symin = fmin(symin, sy);
      symax = fmax(symax, sy);
    }
  }
  const double size = fmax(sxmax - sxmin, symax - symin);
  return size > sp.threshold ? 8 : 1;
}

constexpr int kSelBlock = 1024;
// Entries: nid >= 0 pending, -(nid + 1) final.  Result: the final list of
// node ids in sel_out, and the splat's work list over them (plan_entries).
static_assert(kSelBlock == kPlanBlock, "k_select plans the work list with the plan block size");
__global__ void __launch_bounds__(kSelBlock)
    k_select(NodeCols nd, Geo geo, SelParams sp, int32_t *bufA, int32_t *bufB, int32_t *sel_out,
             unsigned long long *plan, long long *woff, int ppc) { lod::pdl_wait();
  __shared__ uint32_t sh[kSelBlock / 32 + 1];
  __shared__ U64x2 sh64[kSelBlock / 32 + 1];
  int32_t *cur = bufA, *nxt = bufB;
  long long n = 1;
  if (!nd.inner[0] && nd.count[0] == 0) n = 0;  // a tree holding nothing selects nothing
  if (threadIdx.x == 0) cur[0] = 0;
  __syncthreads();
  for (;;) {
    int expanded = 0;  // this thread refined an entry in this round
    long long carry = 0;
    for (long long base = 0; base < n; base += kSelBlock) {
      const long long i = base + threadIdx.x;
      int item = 0, k = 0;
      if (i < n) {
        item = cur[i];
        k = item < 0 ? 1 : sel_decide(nd, geo, sp, item);
      }
      uint32_t tot;
      const uint32_t ex = block_exclusive_scan<uint32_t, kSelBlock>((uint32_t)k, sh, tot);
      const long long o = carry + ex;
      if (k == 1) {
        nxt[o] = item < 0 ? item : -(item + 1);
      } else if (k == 8) {
        expanded = 1;
        const int c0 = nd.desc[item].x;  // children are 8 consecutive ids, octant order
#pragma unroll
        for (int q = 0; q < 8; ++q) nxt[o + q] = c0 + q;
      }
      carry += tot;
    }
    // block-wide OR of the flags doubles as the barrier that publishes `nxt`
    // (a shared flag reset by one thread raced with the other warps' reads)
    const int more = __syncthreads_or(expanded);
    n = carry;
    int32_t *t = cur;
    cur = nxt;
    nxt = t;
    if (!more) break;
  }
  for (long long i = threadIdx.x; i < n; i += kSelBlock) sel_out[i] = -cur[i] - 1;
  __syncthreads();
  // the splat's work list over the selection (O(visible chunks))
  plan_entries(nd, sel_out, n, ppc, woff, plan, reinterpret_cast<U64x2 *>(sh64));
}

__global__ void k_fill_u64(unsigned long long *p, long long n, unsigned long long v) { lod::pdl_wait();
  for (long long i = gtid(); i < n; i += gstride()) p[i] = v;
}

constexpr unsigned kRasterGrid = 148 * 8;  // 8 CTAs x 8 warps per SM, grid-stride over the pieces

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

// Per-device scratch for tree-less brute-force renders.
struct DevScratch {
  cudaStream_t st = nullptr;
  float *xyz = nullptr;
  uint32_t *rgba = nullptr;
  unsigned long long *fb = nullptr;
  long long ncap = 0, fcap = 0;
};
std::mutex g_mu;
DevScratch g_dev[64];

}  // namespace

extern "C" {

int lod_rasterize(LodTree *t, const int32_t *vis, int64_t nvis, const double *cam, uint64_t *fb,
                  int64_t width, int64_t height, int flags, int64_t *samples) {
  if (!t || !cam || !fb || width <= 0 || height <= 0 || nvis < 0 || (nvis > 0 && !vis)) return LOD_E_ARG;
  cudaSetDevice(lod_tree_device(t));
  cudaStream_t st = lod_tree_stream(t);
  const long long nn = lod_tree_num_nodes(t);
  for (int64_t i = 0; i < nvis; ++i)
    if (vis[i] < 0 || vis[i] >= nn) return LOD_E_ARG;
  Cam c;
  memcpy(c.c, cam, sizeof(c.c));
  const long long npx = width * height;
  unsigned long long *dfb = reinterpret_cast<unsigned long long *>(fb);
  if (!(flags & LOD_FLAG_DEVICE_FB)) {
    int rc = lod_tree_ensure_fb(t, npx, &dfb);
    if (rc) return rc;
    if (flags & LOD_FLAG_FB_CLEAR)  // the host target is all sentinel: fill, do not upload
      lod::launch(k_fill_u64, grid_for(npx), 256, 0, st, dfb, npx, ~0ull);
    else
      CK(cudaMemcpyAsync(dfb, fb, npx * 8, cudaMemcpyHostToDevice, st));
  }
  int32_t *dvis = nullptr;
  int rc = lod_tree_ensure_vislist(t, nvis, &dvis);
  if (rc) return rc;
  long long *woff = nullptr;
  if ((rc = lod_tree_ensure_woff(t, nvis, &woff))) return rc;
  if (nvis) CK(cudaMemcpyAsync(dvis, vis, nvis * 4, cudaMemcpyHostToDevice, st));
  unsigned long long *cnt = lod_tree_counter(t);  // [0] samples, [1] entries, [2] pieces
  CK(cudaMemsetAsync(cnt, 0, 24, st));
  const Geo geo = lod_tree_geo(t);
  const int ppc = (int)((geo.C + kPiece - 1) / kPiece);
  if (nvis) {
    const NodeCols nd = lod_tree_nodes(t);
    lod::launch(k_vis_plan, 1, kPlanBlock, 0, st, nd, dvis, (long long)nvis, ppc, woff, cnt);
    lod::launch(k_raster_work, kRasterGrid, 256, 0, st, nd, lod_tree_pool(t), lod_tree_arena(t), dvis,
                (const long long *)woff, (const unsigned long long *)cnt, ppc, c, dfb, width, height);
  }
  unsigned long long drawn = 0;
  CK(cudaMemcpyAsync(&drawn, cnt, 8, cudaMemcpyDeviceToHost, st));
  if (!(flags & LOD_FLAG_DEVICE_FB)) CK(cudaMemcpyAsync(fb, dfb, npx * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (samples) *samples = (int64_t)drawn;
  return LOD_OK;
}

// select_visible on the device (+ optional splat of the selection): one
// selection kernel, one flat chunk pass, one D2H of (count, list, framebuffer).
static int render_impl(LodTree *t, const double *planes, const double *cam, double threshold, uint64_t *fb,
                       int64_t width, int64_t height, int flags, int32_t *selected, int64_t capacity,
                       int64_t *n_selected, int64_t *samples) {
  if (!t || !planes || !cam || (fb && (width <= 0 || height <= 0))) return LOD_E_ARG;
  const long long nn = lod_tree_num_nodes(t);
  if (selected && capacity < nn) return LOD_E_ARG;
  cudaSetDevice(lod_tree_device(t));
  cudaStream_t st = lod_tree_stream(t);
  SelParams sp;
  memcpy(sp.planes, planes, sizeof(sp.planes));
  memcpy(sp.cam, cam, sizeof(sp.cam));
  sp.threshold = threshold;
  int32_t *la = nullptr, *lb = nullptr;
  int rc = lod_tree_ensure_sel(t, nn, &la, &lb);
  if (rc) return rc;
  unsigned long long *cnt = lod_tree_counter(t);  // [0] samples, [1] selected, [2] pieces
  CK(cudaMemsetAsync(cnt, 0, 24, st));
  long long *woff = nullptr;
  if ((rc = lod_tree_ensure_woff(t, nn, &woff))) return rc;
  const Geo geo = lod_tree_geo(t);
  const int ppc = (int)((geo.C + kPiece - 1) / kPiece);
  int32_t *sel = la;  // k_select decodes the final list into la[0, n) (same index as it reads)
  unsigned long long *dfb = reinterpret_cast<unsigned long long *>(fb);
  const long long npx = fb ? width * height : 0;
  if (fb && !(flags & LOD_FLAG_DEVICE_FB)) {
    rc = lod_tree_ensure_fb(t, npx, &dfb);
    if (rc) return rc;
    if (flags & LOD_FLAG_FB_CLEAR)  // the host target is all sentinel: fill, do not upload
      lod::launch(k_fill_u64, grid_for(npx), 256, 0, st, dfb, npx, ~0ull);
    else
      CK(cudaMemcpyAsync(dfb, fb, npx * 8, cudaMemcpyHostToDevice, st));
  }
  const NodeCols nd = lod_tree_nodes(t);
  lod::launch(k_select, 1, kSelBlock, 0, st, nd, geo, sp, la, lb, sel, cnt, woff, ppc);
  if (fb) {
    Cam c;
    memcpy(c.c, cam, sizeof(c.c));
    lod::launch(k_raster_work, kRasterGrid, 256, 0, st, nd, lod_tree_pool(t), lod_tree_arena(t), (const int32_t *)sel,
                (const long long *)woff, (const unsigned long long *)cnt, ppc, c, dfb, width, height);
  }
  unsigned long long h[2] = {0, 0};
  CK(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, st));
  if (fb && !(flags & LOD_FLAG_DEVICE_FB)) CK(cudaMemcpyAsync(fb, dfb, npx * 8, cudaMemcpyDeviceToHost, st));
  if (selected) CK(cudaMemcpyAsync(selected, sel, nn * 4, cudaMemcpyDeviceToHost, st));  // list <= num_nodes
  CK(cudaStreamSynchronize(st));
  if (n_selected) *n_selected = (int64_t)h[1];
  if (samples) *samples = (int64_t)h[0];
  return LOD_OK;
}

int lod_select_visible(LodTree *t, const double *planes, const double *cam, double threshold, int32_t *selected,
                       int64_t capacity, int64_t *n_selected) {
  return render_impl(t, planes, cam, threshold, nullptr, 0, 0, 0, selected, capacity, n_selected, nullptr);
}

int lod_render(LodTree *t, const double *planes, const double *cam, double threshold, uint64_t *fb, int64_t width,
               int64_t height, int flags, int32_t *selected, int64_t capacity, int64_t *n_selected,
               int64_t *samples) {
  if (!fb) return LOD_E_ARG;
  return render_impl(t, planes, cam, threshold, fb, width, height, flags, selected, capacity, n_selected, samples);
}

int lod_raster_points(int32_t device, const float *xyz, const uint32_t *rgba, int64_t n, const double *cam,
                      uint64_t *fb, int64_t width, int64_t height, int flags) {
  if (!cam || !fb || width <= 0 || height <= 0 || n < 0 || (n > 0 && (!xyz || !rgba)) || device < 0 ||
      device >= 64)
    return LOD_E_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev) {
    cudaGetLastError();
    return LOD_E_NO_DEVICE;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  cudaSetDevice(device);
  DevScratch &s = g_dev[device];
  if (!s.st) CK(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
  Cam c;
  memcpy(c.c, cam, sizeof(c.c));
  const long long npx = width * height;
  const float *dx = xyz;
  const uint32_t *dc = rgba;
  if (!(flags & LOD_FLAG_DEVICE_INPUT) && n > 0) {
    if (n > s.ncap) {
      if (s.xyz) cudaFree(s.xyz);
      if (s.rgba) cudaFree(s.rgba);
      long long nc = std::max<long long>(n, 2 * s.ncap);
      CK(cudaMalloc(&s.xyz, nc * 12));
      CK(cudaMalloc(&s.rgba, nc * 4));
      s.ncap = nc;
    }
    CK(cudaMemcpyAsync(s.xyz, xyz, n * 12, cudaMemcpyHostToDevice, s.st));
    CK(cudaMemcpyAsync(s.rgba, rgba, n * 4, cudaMemcpyHostToDevice, s.st));
    dx = s.xyz;
    dc = s.rgba;
  }
  unsigned long long *dfb = reinterpret_cast<unsigned long long *>(fb);
  if (!(flags & LOD_FLAG_DEVICE_FB)) {
    if (npx > s.fcap) {
      if (s.fb) cudaFree(s.fb);
      CK(cudaMalloc(&s.fb, npx * 8));
      s.fcap = npx;
    }
    dfb = s.fb;
    if (flags & LOD_FLAG_FB_CLEAR)
      lod::launch(k_fill_u64, grid_for(npx), 256, 0, s.st, dfb, npx, ~0ull);
    else
      CK(cudaMemcpyAsync(dfb, fb, npx * 8, cudaMemcpyHostToDevice, s.st));
  }
  if (n > 0) lod::launch(k_raster_points, grid_for(n), 256, 0, s.st, dx, dc, n, c, dfb, width, height);
  if (!(flags & LOD_FLAG_DEVICE_FB)) CK(cudaMemcpyAsync(fb, dfb, npx * 8, cudaMemcpyDeviceToHost, s.st));
  CK(cudaStreamSynchronize(s.st));
  return LOD_OK;
}

int lod_device_alloc(int32_t device, uint64_t bytes, void **ptr) {
  if (!ptr) return LOD_E_ARG;
  cudaSetDevice(device);
  if (cudaMalloc(ptr, bytes ? bytes : 1) != cudaSuccess) {
    cudaGetLastError();
    return LOD_E_NOMEM;
  }
  return LOD_OK;
}
int lod_device_free(void *ptr) { return cuda_rc(cudaFree(ptr)); }
int lod_memcpy_h2d(void *dst, const void *src, uint64_t bytes) {
  return cuda_rc(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
}
int lod_memcpy_d2h(void *dst, const void *src, uint64_t bytes) {
  return cuda_rc(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
}
int lod_host_alloc(uint64_t bytes, void **ptr) {
  if (!ptr) return LOD_E_ARG;
  if (cudaMallocHost(ptr, bytes ? bytes : 1) != cudaSuccess) {
    cudaGetLastError();
    return LOD_E_NOMEM;
  }
  return LOD_OK;
}
int lod_host_free(void *ptr) { return cuda_rc(cudaFreeHost(ptr)); }
int lod_fb_fill(int32_t device, uint64_t *fb_dev, int64_t n, uint64_t value) {
  cudaSetDevice(device);
  lod::launch(k_fill_u64, grid_for(n), 256, 0, 0, reinterpret_cast<unsigned long long *>(fb_dev), n, value);
  return cuda_rc(cudaDeviceSynchronize());
}
int lod_l2_flush(int32_t device) {
  static void *buf[64] = {};
  const size_t bytes = 256ull << 20;  // 2x the 126 MB L2
  cudaSetDevice(device);
  if (!buf[device] && cudaMalloc(&buf[device], bytes) != cudaSuccess) return LOD_E_NOMEM;
  CK(cudaMemset(buf[device], device & 0xFF, bytes));
  return cuda_rc(cudaDeviceSynchronize());
}

}  // extern "C"
