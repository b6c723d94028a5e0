// lod_common.cuh -- shared device helpers for the B200 LOD update path.
//
// Arithmetic contract: every float64 formula below is
// evaluated per operation in reference source order.  The library is compiled
// with -fmad=false, so `a * b + c` never contracts into an FMA; float64 `/` is
// IEEE round-to-nearest.  Out-of-range float64 -> int64 conversions emulate the
// x86 cvttsd2si result (INT64_MIN) that numba emits (_kernels.py:107,328).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define LOD_NO_NODE (-1)
#define LOD_NO_CHUNK (-1)

namespace lod {

// kernels launched by this thread (reported per call as LodBatchStats.launches)
inline thread_local long long g_launches = 0;

// Programmatic dependent launch (sm_90+): every update kernel is launched with
// programmatic stream serialization, so the next kernel's launch overlaps the
// tail of the current one; each kernel waits for its predecessor's memory
// before its first dependent access.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launches;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

constexpr int kWarp = 32;

__device__ __forceinline__ long long f2i64(double v) {
  // numba np.int64(float) on x86: cvttsd2si -> INT64_MIN when out of range / NaN.
  if (v >= -9223372036854775808.0 && v < 9223372036854775808.0) return (long long)v;
  return (long long)0x8000000000000000ULL;
}

// direct placement (radix.cuh): items per tile (= per warp) are 1 << tsh,
// tsh from kDirTileShift up to kDirTileShiftMax (large updates: keeps the
// tiles x nodes matrix small; u16 in-tile ranks)
constexpr int kDirTileShift = 11, kDirTileShiftMax = 14;

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-aggregated add of `v` to counter[key]: lanes sharing a key elect one
// leader that issues a single atomic; every lane gets the value the counter had
// before its group's add plus its rank within the group (lower lanes first).
__device__ __forceinline__ unsigned long long warp_agg_add_u64(unsigned long long *counter,
                                                               unsigned long long v_each,
                                                               unsigned active, int key,
                                                               unsigned *rank_out) {
  unsigned peers = __match_any_sync(active, key);
  unsigned leader = __ffs(peers) - 1;
  unsigned rank = __popc(peers & lanemask_lt());
  unsigned long long base = 0;
  if (lane_id() == leader) base = atomicAdd(counter, v_each * (unsigned long long)__popc(peers));
  base = __shfl_sync(peers, base, leader);
  if (rank_out) *rank_out = rank;
  return base;
}

// Read-only load that is not allocated in L1: for random single-use words
// (occupancy grids) that would otherwise evict the L1-resident node table.
__device__ __forceinline__ uint32_t ld_nol1(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// 1D bulk copies global -> shared through the TMA engine, completion tracked
// by an mbarrier (transaction bytes).  Sizes and addresses 16-byte aligned.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LAB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Grid-stride helpers.
__device__ __forceinline__ long long gtid() {
  return (long long)blockIdx.x * blockDim.x + threadIdx.x;
}
__device__ __forceinline__ long long gstride() { return (long long)gridDim.x * blockDim.x; }

// Device view of the tree: the node table (SoA, same column layouts as the
// reference numpy arrays, octree.py:169-182), the chunk pool tables
// (store.py:97-101) and the arena.
struct NodeCols {
  int32_t *parent;
  uint8_t *octant;
  int32_t *level;
  int32_t *children;  // [ncap * 8]
  uint8_t *inner;
  uint8_t *final_;
  long long *count;
  unsigned long long *pending;  // int64 in the reference; non-negative
  int32_t *chunk_head;
  int32_t *chunk_tail;
  int32_t *chunk_count;
  long long *grid_off;
  double *bmin;  // [ncap * 3]
  // device-only descent record: {first child id (children are 8 consecutive
  // ids) or -1 for a leaf, grid offset / 64}; 8 bytes per node, L1-resident
  int2 *desc;
  // device-only chunk directory: the node's chunk ids in list order are
  // PoolCols::cdir[dir_off[n] + i], i < chunk_count[n] (region of dir_cap[n]
  // entries; relocated with doubling when it fills, kept across a split)
  long long *dir_off;
  int32_t *dir_cap;
};

struct PoolCols {
  int32_t *next;
  long long *payload_off;
  int32_t *occupied;
  int32_t *owner;  // node owning the chunk, -1 when free (render work list)
  int32_t *cidx;   // position of the chunk in its owner's list
  int32_t *free_stack;
  int32_t *cdir;   // chunk directory (NodeCols::dir_off / dir_cap): spill gather and render work lists
  unsigned long long cdir_cap;  // entries of cdir: a relocation past it sets Ctrl::dir_overflow instead
};

struct Geo {
  double bmin0[3];
  double size0;
  double size_by_level[64];  // size * 0.5 ** k (octree.py:167); levels <= 62
  double inv_by_level[64];   // 1 / size_by_level[k], exact when pow2
  int pow2;                  // root size is a power of two: x / s == x * (1/s) exactly
  int g;                     // grid_res
  long long grid_bytes;
  long long T;               // leaf_threshold
  int max_depth;
  long long C;               // chunk capacity (records)
  int fresh;                 // arena < 128 GiB: desc .y bit 31 marks a grid still all clear (kFresh)
  uint32_t gmask;            // desc .y bits of the grid offset / 64 (0x7fffffff with `fresh`)
  int f32ok;                 // the count pass may descend in f32 (count_descend<float>; set by the host)
};

// One point source over the reference's all-array [spill || batch]
// (update.py:281-286): spill points are 16-byte records; batch points come
// from the caller's xyz (n,3) f32 + rgba (n,) u32 arrays, or from 16-byte
// records when the batch arrives packed (brec; e.g. routed from other ranks).
struct PointSrc {
  const float4 *spill;
  long long ns;
  const float *bxyz;
  const uint32_t *brgba;
  long long nb;
  const float4 *brec;  // packed batch records, or null
  __device__ __forceinline__ void xyz(long long j, float &x, float &y, float &z) const {
    if (j < ns || brec) {
      const float4 r = j < ns ? __ldg(spill + j) : __ldg(brec + (j - ns));
      x = r.x; y = r.y; z = r.z;
    } else {
      const float *p = bxyz + 3 * (j - ns);
      x = __ldg(p); y = __ldg(p + 1); z = __ldg(p + 2);
    }
  }
  __device__ __forceinline__ float4 record(long long j) const {
    if (j < ns) return __ldg(spill + j);
    if (brec) return __ldg(brec + (j - ns));
    const float *p = bxyz + 3 * (j - ns);
    float4 r;
    r.x = __ldg(p); r.y = __ldg(p + 1); r.z = __ldg(p + 2);
    r.w = __uint_as_float(__ldg(brgba + (j - ns)));
    return r;
  }
  __device__ __forceinline__ uint32_t rgba(long long j) const {
    if (j < ns) return __float_as_uint(__ldg(spill + j).w);
    return brec ? __float_as_uint(__ldg(brec + (j - ns)).w) : __ldg(brgba + (j - ns));
  }
};

// Per-point node cache over the same all-array index space: spilled points'
// entries live in their own array (written by the spill gather), batch points'
// in another, so the batch part never has to move behind the spill.
struct NodeOf {
  int32_t *spill;
  int32_t *batch;
  long long ns;
  __device__ __forceinline__ int32_t &operator[](long long j) const { return j < ns ? spill[j] : batch[j - ns]; }
};

// One descent step (count_points / sample_and_route, _kernels.py:44-56):
// bit set when x >= bx + h, then bx += h; upper children own the split plane.
__device__ __forceinline__ int octant_step(double x, double y, double z, double &bx, double &by,
                                           double &bz, double &s) {
  double h = s * 0.5;
  int o = 0;
  if (x >= bx + h) { o |= 1; bx += h; }
  if (y >= by + h) { o |= 2; by += h; }
  if (z >= bz + h) { o |= 4; bz += h; }
  s = h;
  return o;
}

// Same step also tracking 1/s (exact doubling; only meaningful when pow2).
__device__ __forceinline__ int octant_step(double x, double y, double z, double &bx, double &by, double &bz,
                                           double &s, double &inv_s) {
  inv_s = inv_s * 2.0;
  return octant_step(x, y, z, bx, by, bz, s);
}

// f32 twins of octant_step / cell_of for Geo::f32ok trees: a power-of-two
// root size and grid_res, a root in the non-negative orthant whose corner lies
// on the finest plane grid q = size * 2^-max_depth, with (corner + size) / q <=
// 2^24.  Then every plane bx + h is an f32, every x - bx (x >= bx >= 0) is
// exact in f32, and g * (x - bx) * 2^k only scales by powers of two: the
// compares and floors are the f64 ones bit for bit,
// in half the registers.
__device__ __forceinline__ int octant_step(float x, float y, float z, float &bx, float &by, float &bz, float &s,
                                           float &inv_s) {
  const float h = s * 0.5f;
  int o = 0;
  if (x >= bx + h) { o |= 1; bx += h; }
  if (y >= by + h) { o |= 2; by += h; }
  if (z >= bz + h) { o |= 4; bz += h; }
  s = h;
  inv_s = inv_s * 2.0f;
  return o;
}
__device__ __forceinline__ int clamp_cell(float v, int g) {
  const float f = floorf(v);
  if (!(f < 9223372036854775808.0f)) return 0;  // NaN, +inf, >= 2^63 -> INT64_MIN -> 0
  if (f < 0.0f) return 0;
  if (f > (float)(g - 1)) return g - 1;
  return (int)f;
}

// Clamp of np.int64(np.floor(v)) to [0, g-1] (_kernels.py:107-121) with the
// x86 conversion semantics: NaN and |v| >= 2^63 become INT64_MIN, i.e. cell 0.
__device__ __forceinline__ int clamp_cell(double v, int g) {
  const double f = floor(v);
  if (!(f < 9223372036854775808.0)) return 0;  // NaN, +inf, >= 2^63 -> INT64_MIN -> 0
  if (f < 0.0) return 0;
  if (f > (double)(g - 1)) return g - 1;
  return (int)f;
}

// Occupancy cell (_kernels.py:107-122): floor(g * (x - bx) / s) per axis,
// clamped, cx + g*cy + g*g*cz.  `inv_s` = 1/s is used only when the root size
// is a power of two: then s = 2^-k exactly and (g*(x-bx)) / s == (g*(x-bx)) * 2^k
// bit for bit, saving three IEEE divisions per probe.
__device__ __forceinline__ long long cell_of(const Geo &geo, double x, double y, double z,
                                             double bx, double by, double bz, double s, double inv_s) {
  const double gd = (double)geo.g;
  int cx, cy, cz;
  if (geo.pow2) {
    cx = clamp_cell(gd * (x - bx) * inv_s, geo.g);
    cy = clamp_cell(gd * (y - by) * inv_s, geo.g);
    cz = clamp_cell(gd * (z - bz) * inv_s, geo.g);
  } else {
    cx = clamp_cell(gd * (x - bx) / s, geo.g);
    cy = clamp_cell(gd * (y - by) / s, geo.g);
    cz = clamp_cell(gd * (z - bz) / s, geo.g);
  }
  return (long long)cx + (long long)geo.g * cy + (long long)geo.g * geo.g * cz;
}
__device__ __forceinline__ long long cell_of(const Geo &geo, float x, float y, float z, float bx, float by, float bz,
                                             float s, float inv_s) {
  const float gf = (float)geo.g;
  const int cx = clamp_cell(gf * (x - bx) * inv_s, geo.g);
  const int cy = clamp_cell(gf * (y - by) * inv_s, geo.g);
  const int cz = clamp_cell(gf * (z - bz) * inv_s, geo.g);
  return (long long)cx + (long long)geo.g * cy + (long long)geo.g * geo.g * cz;
}

}  // namespace lod
