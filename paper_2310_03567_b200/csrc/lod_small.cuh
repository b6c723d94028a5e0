// lod_small.cuh -- one whole update cycle of a tiny batch in ONE thread block.
//
// The reference's acceptance gate C1 (pkg/tests/test_acceptance.py:81-101)
// makes 1.52M insert_batch calls of 1 or 7 points; at ~23 launches and a host
// round trip per expansion iteration the multi-kernel pipeline costs ~60 us a
// call.  Here count <-> split, sampling, allocation, store and cleanup of
// update.py:252-393 run in one launch: the order-free passes (count, split
// execution, allocation) use the whole block with __syncthreads() between
// them, the order-defining passes (first-come voxel claims, slot assignment)
// run on one warp in ascending all-array index order, 32 points at a time --
// exactly the reference's sequential rule (_kernels.py:66-250), with lanes
// of a group resolved by __match_any_sync (lowest lane = lowest index).
// The result is identical to the pipeline's; the data structures (node SoA,
// descent records, pool tables, free stack, arena, Ctrl counters) are the
// same, so small and large batches interleave freely on one tree.
//
// The host launches it asynchronously when no error is possible for the
// batch (capacities bounded from the batch size, the leaf threshold and the
// depth), so a stream of tiny calls costs a launch each; otherwise it waits
// for the per-call result the kernel writes into mapped host memory.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lod_common.cuh"
#include "lod_kernels.cuh"
#include "scan.cuh"

namespace lod {

constexpr int kSmallBlock = 512;
constexpr int kSmallMaxBatch = 256;       // batch points per small cycle
constexpr long long kSmallAllMax = 1 << 16;  // bound on [spill || batch] points for the small path

// Per-call result in mapped pinned host memory (seq written last).
struct SmallResult {
  long long n_spill, n_voxels, n_splits, iterations;
  long long num_nodes, splits_total, max_level, allocated_total, free_count, released_total;
  unsigned long long arena_off, dir_top;
  long long device_ns;
  int error;
  unsigned seq;
};

// Running totals of the asynchronous calls since the host last settled
// (device memory; copied out and zeroed by the host when it settles).
struct SmallAccum {
  long long calls, nv_sum, nv_max, ns_max, splits_sum, device_ns;
  int error;
  int pad;
};

struct SmallArgs {
  NodeCols nd;
  PoolCols pool;
  Geo geo;
  uint8_t *arena;
  Ctrl *ctrl;
  const float4 *in;  // the batch as 16-byte records, mapped pinned host memory
  int n;
  float4 *brec;      // batch records (device copy)
  float4 *srec;      // spilled records
  int32_t *node_b, *node_s;  // per-point node; ~nid = re-descend from nid
  int32_t *srank;            // per node: split rank of this iteration, -1 otherwise (shared with the pipeline)
  long long *nnew;           // per node: new voxels this cycle (zero between cycles)
  long long *cur;            // per node: next slot (store)
  long long *wls;            // per node: first write-list entry
  uint4 *backlog;            // new voxels {node, cell, rgba, winner index} in claim order
  int32_t *tl;               // leaves touched in the running iteration
  int32_t *cand;             // split candidates of the running iteration
  int32_t *splits;           // split candidates in ascending id
  int32_t *touched;          // nodes with new samples this cycle (final leaves, inner nodes with voxels)
  long long *pl;             // per touched position: need, acquisition start, write-list start (3 each)
  long long *wl;             // write list: payload offsets
  long long *sp;             // per split rank: stored count, chunk count, spill offset, free offset (4 each)
  long long all_cap, vox_cap, touched_cap, split_cap, wl_cap;
  long long ncap, ccap;
  long long spill_cap, backlog_cap;
  unsigned long long arena_cap;
  SmallResult *res;          // mapped
  volatile unsigned *done;   // mapped
  SmallAccum *acc;           // device
  unsigned seq;
  int async_call;
};

__device__ __forceinline__ long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (long long)t;
}

__device__ __forceinline__ float4 small_record(const SmallArgs &a, long long n_s, long long j) {
  return j < n_s ? a.srec[j] : a.brec[j - n_s];
}

// Block-wide U64x2 exclusive scan over `count` values produced by `val(i)`
// (i in list order), writing `out(i, exclusive)`; returns the total.
template <typename Val, typename Out>
__device__ __forceinline__ U64x2 small_scan(long long count, U64x2 *sh, Val val, Out out) {
  U64x2 carry = u64x2(0, 0);
  for (long long base = 0; base < count; base += kSmallBlock) {
    const long long i = base + threadIdx.x;
    const U64x2 v = i < count ? val(i) : u64x2(0, 0);
    U64x2 tot;
    const U64x2 ex = block_exclusive_scan<U64x2, kSmallBlock>(v, sh, tot);
    if (i < count) out(i, ex + carry, v);
    carry = carry + tot;
  }
  return carry;
}

__global__ void __launch_bounds__(kSmallBlock) k_small_cycle(SmallArgs a) {
  lod::pdl_wait();
  const long long t_start = globaltimer_ns();
  __shared__ long long s_nn, s_stot, s_maxlvl, s_alloc, s_free, s_rel;
  __shared__ unsigned long long s_arena;
  __shared__ long long s_plan_nn0, s_plan_free0, s_spill0;
  __shared__ unsigned long long s_plan_g0;
  __shared__ int s_ntl, s_ncand, s_ntouched, s_err, s_iters;
  __shared__ long long s_err_spill, s_cycle_splits, s_nv, s_F, s_A;
  __shared__ unsigned long long s_base;
  __shared__ U64x2 sh64[kSmallBlock / 32 + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const NodeCols &nd = a.nd;
  const PoolCols &pool = a.pool;
  const Geo &geo = a.geo;
  const long long C = geo.C;
  uint32_t *grid32 = reinterpret_cast<uint32_t *>(a.arena);
  if (tid == 0) {
    Ctrl *c = a.ctrl;
    s_nn = c->num_nodes;
    s_stot = c->splits_total;
    s_maxlvl = c->max_level;
    s_alloc = c->allocated_total;
    s_free = c->free_count;
    s_rel = c->released_total;
    s_arena = c->arena_off;
    s_err = 0;
    s_ntouched = 0;
    s_iters = 0;
    s_cycle_splits = 0;
    s_spill0 = 0;
    s_nv = 0;
  }
  for (int j = tid; j < a.n; j += kSmallBlock) a.brec[j] = a.in[j];  // the batch, over PCIe once
  __syncthreads();

  long long n_s = 0;  // spilled points (all-array prefix)
  // ---------------------------------------------------------------- expansion
  // count_points <-> _split_pass until no leaf splits (update.py:273-296)
  for (int first = 1;; first = 0) {
    if (tid == 0) {
      s_ntl = 0;
      s_ncand = 0;
      s_err_spill = -1;
      ++s_iters;
    }
    __syncthreads();
    const long long nall = first ? a.n : n_s + a.n;
    for (long long j = tid; j < nall; j += kSmallBlock) {
      int32_t *slot = first ? a.node_b + j : (j < n_s ? a.node_s + j : a.node_b + (j - n_s));
      int nid = 0;
      if (!first) {
        nid = *slot;
        if (nid >= 0) continue;  // settled in an earlier iteration
        nid = ~nid;
      }
      const float4 r = first ? a.brec[j] : small_record(a, n_s, j);
      const double x = r.x, y = r.y, z = r.z;
      double bx = nd.bmin[3 * nid], by = nd.bmin[3 * nid + 1], bz = nd.bmin[3 * nid + 2];
      double s = geo.size_by_level[nd.level[nid]];
      int2 d = nd.desc[nid];
      while (d.x >= 0) {  // _kernels.py:38-56
        nid = d.x + octant_step(x, y, z, bx, by, bz, s);
        d = nd.desc[nid];
      }
      *slot = nid;
      if (!nd.final_[nid]) {
        if (atomicAdd(&nd.pending[nid], 1ull) == 0ull) {  // touched on pending 0 -> 1 (_kernels.py:59-61)
          const int k = atomicAdd(&s_ntl, 1);
          if (k < a.all_cap) a.tl[k] = nid;
          else s_err = LOD_E_NOMEM;
        }
      }
    }
    __syncthreads();
    // split iff count + pending > T and level < max depth, else final (update.py:226-249)
    const int ntl = min(s_ntl, (int)a.all_cap);
    for (int i = tid; i < ntl; i += kSmallBlock) {
      const int nid = a.tl[i];
      const long long tot = nd.count[nid] + (long long)nd.pending[nid];
      if (tot > geo.T && nd.level[nid] < geo.max_depth) {
        const int k = atomicAdd(&s_ncand, 1);
        if (k < a.split_cap) a.cand[k] = nid;
        else s_err = LOD_E_NOMEM;
      } else {
        nd.final_[nid] = 1;
        const int k = atomicAdd(&s_ntouched, 1);
        if (k < a.touched_cap) a.touched[k] = nid;
        else s_err = LOD_E_NOMEM;
      }
    }
    __syncthreads();
    const int S = min(s_ncand, (int)a.split_cap);
    if (S == 0 || s_err) break;
    // ascending node id (octree.py:249-261: 8 consecutive child ids per split, in id order)
    for (int i = tid; i < S; i += kSmallBlock) {
      const int me = a.cand[i];
      int r = 0;
      for (int k = 0; k < S; ++k) r += a.cand[k] < me;
      a.splits[r] = me;
      a.srank[me] = r;
      a.sp[4 * r] = nd.count[me];
      a.sp[4 * r + 1] = nd.chunk_count[me];
    }
    __syncthreads();
    const long long spill0 = s_spill0;
    const U64x2 tot = small_scan(
        S, sh64, [&](long long r) { return u64x2((unsigned long long)a.sp[4 * r], (unsigned long long)a.sp[4 * r + 1]); },
        [&](long long r, U64x2 ex, U64x2 v) {
          a.sp[4 * r + 2] = (long long)ex.a;
          a.sp[4 * r + 3] = (long long)ex.b;
          // SpillBuffer.append raises before the node's grid alloc (octree.py:231-244)
          if (v.a > 0 && spill0 + (long long)(ex.a + v.a) > a.spill_cap)
            atomicMin((unsigned long long *)&s_err_spill, (unsigned long long)r);
        });
    if (tid == 0) {
      // grids of the splits in rank order, 64-aligned (store.py:51-69); the
      // first failure in rank order decides the error, spill before arena
      const unsigned long long gb = (unsigned long long)geo.grid_bytes;
      const unsigned long long g0 = (s_arena + 63ull) / 64ull * 64ull;
      const unsigned long long gs = (gb + 63ull) / 64ull * 64ull;
      long long err_ooa = -1;
      if (g0 + gb > a.arena_cap) err_ooa = 0;
      else if (g0 + (unsigned long long)(S - 1) * gs + gb > a.arena_cap) err_ooa = (long long)((a.arena_cap - gb - g0) / gs) + 1;
      const long long es = s_err_spill;
      if (es >= 0 && (err_ooa < 0 || es <= err_ooa)) s_err = LOD_E_SPILL_OVERFLOW;
      else if (err_ooa >= 0) s_err = LOD_E_OUT_OF_ARENA;
      else if (s_nn + 8ll * S > a.ncap || (first && spill0 + (long long)tot.a + a.n > a.all_cap)) s_err = LOD_E_NOMEM;
      else {
        s_plan_nn0 = s_nn;
        s_plan_free0 = s_free;
        s_plan_g0 = g0;
        s_nn += 8ll * S;
        s_stot += S;
        s_free += (long long)tot.b;
        s_rel += (long long)tot.b;
        s_arena = g0 + (unsigned long long)(S - 1) * gs + gb;
        s_spill0 = spill0 + (long long)tot.a;
        s_cycle_splits += S;
      }
    }
    __syncthreads();
    if (s_err) break;
    // Octree.split part 1 (octree.py:231-237, store.py:125-143): every split
    // node's records to its spill segment in walk order, its chunks onto the
    // free stack in walk order.  One warp per split node.
    for (int r = warp; r < S; r += kSmallBlock / 32) {
      const int nid = a.splits[r];
      int cid = nd.chunk_head[nid];
      long long ci = 0;
      const long long sbase = spill0 + a.sp[4 * r + 2];
      const long long fbase = s_plan_free0 + a.sp[4 * r + 3];
      while (cid != LOD_NO_CHUNK) {
        const int occ = pool.occupied[cid];
        const int nxt = pool.next[cid];
        const float4 *src = reinterpret_cast<const float4 *>(a.arena + pool.payload_off[cid]);
        for (int k = lane; k < occ; k += 32) {
          a.srec[sbase + ci * C + k] = src[k];
          a.node_s[sbase + ci * C + k] = ~nid;  // re-descends from the split node
        }
        __syncwarp();
        if (lane == 0) {
          pool.free_stack[fbase + ci] = cid;
          pool.occupied[cid] = 0;
          pool.next[cid] = LOD_NO_CHUNK;
          pool.owner[cid] = -1;
          pool.cidx[cid] = -1;
        }
        cid = nxt;
        ++ci;
      }
    }
    __syncthreads();  // the gather reads the split nodes' chunk lists, which part 2 resets
    // Octree.split part 2 (octree.py:238-264): the node turns inner with a
    // zeroed grid and gets 8 children with bmin = base + half (f64)
    for (long long t = tid; t < 8ll * S; t += kSmallBlock) {
      const long long k = t >> 3;
      const int o = (int)(t & 7);
      const int nid = a.splits[k];
      const int lvl = nd.level[nid];
      const int c = (int)(s_plan_nn0 + 8ll * k + o);
      const double half = geo.size_by_level[lvl] * 0.5;
      nd.parent[c] = nid;
      nd.octant[c] = (uint8_t)o;
      nd.level[c] = lvl + 1;
      for (int q = 0; q < 8; ++q) nd.children[8 * c + q] = LOD_NO_NODE;
      nd.inner[c] = 0;
      nd.final_[c] = 0;
      nd.count[c] = 0;
      nd.pending[c] = 0;
      nd.chunk_head[c] = LOD_NO_CHUNK;
      nd.chunk_tail[c] = LOD_NO_CHUNK;
      nd.chunk_count[c] = 0;
      nd.grid_off[c] = -1;
      nd.desc[c] = make_int2(-1, 0);
      nd.dir_off[c] = 0;
      nd.dir_cap[c] = 0;
      nd.bmin[3 * c + 0] = nd.bmin[3 * nid + 0] + ((o & 1) ? half : 0.0);
      nd.bmin[3 * c + 1] = nd.bmin[3 * nid + 1] + ((o & 2) ? half : 0.0);
      nd.bmin[3 * c + 2] = nd.bmin[3 * nid + 2] + ((o & 4) ? half : 0.0);
      nd.children[8 * nid + o] = c;
      a.srank[c] = -1;
      a.nnew[c] = 0;
      if (o == 0) {
        atomicMax((unsigned long long *)&s_maxlvl, (unsigned long long)(lvl + 1));
        nd.count[nid] = 0;
        nd.pending[nid] = 0;
        nd.inner[nid] = 1;
        nd.chunk_head[nid] = LOD_NO_CHUNK;
        nd.chunk_tail[nid] = LOD_NO_CHUNK;
        nd.chunk_count[nid] = 0;
        const unsigned long long gs = ((unsigned long long)geo.grid_bytes + 63ull) / 64ull * 64ull;
        const unsigned long long goff = s_plan_g0 + (unsigned long long)k * gs;
        nd.grid_off[nid] = (long long)goff;
        nd.desc[nid] = make_int2(c - o, (int)(uint32_t)(goff >> 6));
      }
    }
    __syncthreads();
    // points whose leaf split re-descend from it in the next iteration
    for (long long j = tid; j < nall; j += kSmallBlock) {
      int32_t *slot = first ? a.node_b + j : (j < n_s ? a.node_s + j : a.node_b + (j - n_s));
      const int nid = *slot;
      if (nid >= 0 && a.srank[nid] >= 0) *slot = ~nid;
    }
    __syncthreads();
    for (int r = tid; r < S; r += kSmallBlock) a.srank[a.splits[r]] = -1;
    if (first) n_s = s_spill0;  // only iteration 1 spills (update.py:9-11)
    __syncthreads();
  }
  __syncthreads();  // every warp has left the split loop (it reads s_err) before warp 0 may set it below
  const long long n_all = n_s + a.n;

  // ---------------------------------------------------------------- sampling
  // sample_and_route (_kernels.py:66-152): every point descends from the
  // root in all-array order; at each inner node the first point on a clear
  // cell claims it (bit set, backlog entry, per-node voxel count).  One warp,
  // 32 consecutive points per step, lockstep by level: claims at one node
  // come from one level, and the lowest lane of a matching group is the
  // lowest index, so this is the sequential rule.
  if (warp == 0 && !s_err) {  // (warp first: the other warps never read s_err while warp 0 may set it)
    long long nv = 0;
    for (long long j0 = 0; j0 < n_all; j0 += 32) {
      const long long j = j0 + lane;
      const bool act = j < n_all;
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      if (act) r = small_record(a, n_s, j);
      const double x = r.x, y = r.y, z = r.z;
      const uint32_t rgba = __float_as_uint(r.w);
      double bx = geo.bmin0[0], by = geo.bmin0[1], bz = geo.bmin0[2], s = geo.size0, inv_s = geo.inv_by_level[0];
      int nid = 0;
      int2 d = nd.desc[0];
      for (;;) {
        const bool in = act && d.x >= 0;
        if (!__any_sync(0xffffffffu, in)) break;
        unsigned long long key = ~0ull;
        long long cell = 0;
        bool clear = false;
        if (in) {
          cell = cell_of(geo, x, y, z, bx, by, bz, s, inv_s);
          const uint32_t w = __ldcg(grid32 + ((unsigned long long)((uint32_t)d.y & a.geo.gmask) << 4) + (cell >> 5));
          clear = !(w & (1u << (cell & 31)));
          if (clear) key = ((unsigned long long)(uint32_t)nid << 32) | (unsigned long long)cell;  // warp-local match key
        }
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const bool win = clear && (int)(__ffs(peers) - 1) == lane;
        const unsigned wm = __ballot_sync(0xffffffffu, win);
        if (win) {
          atomicOr(grid32 + ((unsigned long long)((uint32_t)d.y & a.geo.gmask) << 4) + (cell >> 5), 1u << (cell & 31));
          const long long pos = nv + __popc(wm & lanemask_lt());
          if (pos < a.vox_cap) a.backlog[pos] = make_uint4((uint32_t)nid, (uint32_t)cell, rgba, (uint32_t)j);
        }
        const unsigned npeers = __match_any_sync(0xffffffffu, win ? nid : -1);
        if (win && (int)(__ffs(npeers) - 1) == lane) {
          const long long old = a.nnew[nid];
          a.nnew[nid] = old + __popc(npeers);
          if (old == 0) {
            const int k = atomicAdd(&s_ntouched, 1);
            if (k < a.touched_cap) a.touched[k] = nid;
            else s_err = LOD_E_NOMEM;
          }
        }
        nv += __popc(wm);
        if (in) {
          nid = d.x + octant_step(x, y, z, bx, by, bz, s, inv_s);
          d = nd.desc[nid];
        }
        __syncwarp();
      }
    }
    if (lane == 0) {
      s_nv = nv;
      if (nv > a.backlog_cap) s_err = LOD_E_BACKLOG_OVERFLOW;  // update.py:311-312
      else if (nv > a.vox_cap) s_err = LOD_E_NOMEM;
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- allocation
  // collect_allocs + append_chunk + acquire (_kernels.py:253-277,
  // octree.py:328-337, store.py:110-123): per touched node need =
  // ceil((count + new) / C) - chunk_count, LIFO free stack before the arena
  const int K = min(s_ntouched, (int)a.touched_cap);
  if (!s_err) {
    const U64x2 tot = small_scan(
        K, sh64,
        [&](long long d) {
          const int nid = a.touched[d];
          const long long items = nd.inner[nid] ? a.nnew[nid] : (long long)nd.pending[nid];
          const long long cnt = nd.count[nid];
          const long long need = ceil_div(cnt + items, C) - ceil_div(cnt, C);
          return u64x2((unsigned long long)need, (unsigned long long)(need + ((cnt % C) != 0)));
        },
        [&](long long d, U64x2 ex, U64x2 v) {
          a.pl[3 * d] = (long long)v.a;
          a.pl[3 * d + 1] = (long long)ex.a;
          a.pl[3 * d + 2] = (long long)ex.b;
        });
    if (tid == 0) {
      const long long M = (long long)tot.a, F = s_free, A = s_alloc;
      const long long fresh = M > F ? M - F : 0;
      const unsigned long long base = (s_arena + 15ull) / 16ull * 16ull;
      const unsigned long long end = base + (unsigned long long)fresh * (unsigned long long)C * 16ull;
      if (fresh > 0 && end > a.arena_cap) s_err = LOD_E_OUT_OF_ARENA;
      else if (A + fresh > a.ccap || (long long)tot.b > a.wl_cap) s_err = LOD_E_NOMEM;
      else {
        s_F = F;
        s_A = A;
        s_base = base;
        if (fresh > 0) s_arena = end;
        s_free = F - (M < F ? M : F);
        s_alloc = A + fresh;
        s_ncand = (int)M;  // reused: acquisitions
      }
    }
    __syncthreads();
  }
  if (!s_err) {
    const long long F = s_F, A = s_A;
    auto acq = [&](long long q) -> int { return q < F ? pool.free_stack[F - 1 - q] : (int)(A + (q - F)); };
    for (int d = tid; d < K; d += kSmallBlock) {  // per node: tail update and links
      const int nid = a.touched[d];
      const long long items = nd.inner[nid] ? a.nnew[nid] : (long long)nd.pending[nid];
      const long long cnt = nd.count[nid];
      const long long need = a.pl[3 * d], A0 = a.pl[3 * d + 1], W0 = a.pl[3 * d + 2];
      const int tail = nd.chunk_tail[nid];
      a.wls[nid] = W0;
      a.cur[nid] = cnt;
      if (cnt % C) {
        a.wl[W0] = pool.payload_off[tail];
        const long long rem = cnt + items - (cnt / C) * C;
        pool.occupied[tail] = (int)(rem < C ? rem : C);
      }
      if (need > 0) {
        const int f = acq(A0), l = acq(A0 + need - 1);
        if (tail != LOD_NO_CHUNK) pool.next[tail] = f;
        else nd.chunk_head[nid] = f;
        nd.chunk_tail[nid] = l;
        nd.chunk_count[nid] += (int)need;
      }
    }
    const long long M = s_ncand;
    for (long long q = tid; q < M; q += kSmallBlock) {  // per acquisition
      long long lo = 0, hi = K - 1;
      while (lo < hi) {
        const long long mid = (lo + hi + 1) >> 1;
        if (a.pl[3 * mid + 1] <= q) lo = mid;
        else hi = mid - 1;
      }
      const int nid = a.touched[lo];
      const long long need = a.pl[3 * lo], t = q - a.pl[3 * lo + 1];
      const long long items = nd.inner[nid] ? a.nnew[nid] : (long long)nd.pending[nid];
      const long long cnt = nd.count[nid];
      const int cid = acq(q);
      long long poff;
      if (q >= F) {
        poff = (long long)(s_base + (unsigned long long)(q - F) * (unsigned long long)C * 16ull);
        pool.payload_off[cid] = poff;
      } else {
        poff = pool.payload_off[cid];
      }
      pool.next[cid] = (t + 1 < need) ? acq(q + 1) : LOD_NO_CHUNK;
      pool.owner[cid] = nid;
      const long long ci = ceil_div(cnt, C) + t;
      pool.cidx[cid] = (int)ci;
      const long long rem = cnt + items - ci * C;
      pool.occupied[cid] = (int)(rem < C ? rem : C);
      a.wl[a.pl[3 * lo + 2] + ((cnt % C) != 0) + t] = poff;
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- store
  // store_points / store_voxels (_kernels.py:155-250): slot = count + rank in
  // all-array order (points, warp 0) / backlog order (voxels, warp 1)
  if (warp < 2 && !s_err) {
    const long long total = warp == 0 ? n_all : s_nv;
    for (long long i0 = 0; i0 < total; i0 += 32) {
      const long long i = i0 + lane;
      const bool act = i < total;
      int nid = -1;
      float4 rec = make_float4(0.f, 0.f, 0.f, 0.f);
      if (act) {
        if (warp == 0) {
          nid = i < n_s ? a.node_s[i] : a.node_b[i - n_s];
          rec = small_record(a, n_s, i);
        } else {
          const uint4 bl = a.backlog[i];
          nid = (int)bl.x;
          const long long cell = bl.y, g = geo.g;
          const long long cx = cell % g, cy = (cell / g) % g, cz = cell / (g * g);
          const double step = geo.size_by_level[nd.level[nid]] / (double)g;  // _kernels.py:226-245
          const double vx = nd.bmin[3 * nid] + ((double)cx + 0.5) * step;
          const double vy = nd.bmin[3 * nid + 1] + ((double)cy + 0.5) * step;
          const double vz = nd.bmin[3 * nid + 2] + ((double)cz + 0.5) * step;
          rec = make_float4(__double2float_rn(vx), __double2float_rn(vy), __double2float_rn(vz),
                            __uint_as_float(bl.z));
        }
      }
      const unsigned peers = __match_any_sync(0xffffffffu, nid);
      const int leader = __ffs(peers) - 1;
      long long base = 0;
      if (act && lane == leader) {
        base = a.cur[nid];
        a.cur[nid] = base + __popc(peers);
      }
      base = __shfl_sync(0xffffffffu, base, leader);
      if (act) {
        const long long slot = base + __popc(peers & lanemask_lt());
        const long long cnt = nd.count[nid];
        const long long poff = a.wl[a.wls[nid] + slot / C - cnt / C];
        reinterpret_cast<float4 *>(a.arena + poff)[slot % C] = rec;
      }
      __syncwarp();
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- cleanup
  // count += new samples; pending = final = 0 (clear_marks, _kernels.py:280-287);
  // after a fatal error only the marks are cleared (partial state, errors.py:1-5)
  if (s_err) {
    const int ntl = min(s_ntl, (int)a.all_cap);
    for (int i = tid; i < ntl; i += kSmallBlock) {
      nd.pending[a.tl[i]] = 0;
      nd.final_[a.tl[i]] = 0;
    }
    for (int i = tid; i < min(s_ncand, (int)a.split_cap); i += kSmallBlock) a.srank[a.cand[i]] = -1;
  }
  for (int d = tid; d < K; d += kSmallBlock) {
    const int nid = a.touched[d];
    if (!s_err) {
      nd.count[nid] += nd.inner[nid] ? a.nnew[nid] : (long long)nd.pending[nid];
      const long long F = s_F, A = s_A, A0 = a.pl[3 * d + 1];
      dir_append(nd, pool, &a.ctrl->dir_top, nid, a.pl[3 * d], [&](long long t) {
        const long long q = A0 + t;
        return q < F ? pool.free_stack[F - 1 - q] : (int)(A + (q - F));
      });
    }
    nd.pending[nid] = 0;
    nd.final_[nid] = 0;
    a.nnew[nid] = 0;
  }
  __syncthreads();
  if (tid == 0) {
    Ctrl *c = a.ctrl;
    c->num_nodes = s_nn;
    c->splits_total = s_stot;
    c->max_level = s_maxlvl;
    c->allocated_total = s_alloc;
    c->free_count = s_free;
    c->released_total = s_rel;
    c->arena_off = s_arena;
    c->n_used = (unsigned long long)s_nv;
    const long long dt = globaltimer_ns() - t_start;
    SmallResult *r = a.res;
    r->n_spill = n_s;
    r->n_voxels = s_nv;
    r->n_splits = s_cycle_splits;
    r->iterations = s_iters;
    r->num_nodes = s_nn;
    r->splits_total = s_stot;
    r->max_level = s_maxlvl;
    r->allocated_total = s_alloc;
    r->free_count = s_free;
    r->released_total = s_rel;
    r->arena_off = s_arena;
    r->dir_top = c->dir_top;
    r->device_ns = dt;
    r->error = s_err;
    if (a.async_call) {
      SmallAccum *q = a.acc;
      q->calls += 1;
      q->nv_sum += s_nv;
      q->nv_max = max(q->nv_max, s_nv);
      q->ns_max = max(q->ns_max, n_s);
      q->splits_sum += s_cycle_splits;
      q->device_ns += dt;
      if (s_err && !q->error) q->error = s_err;
    }
    __threadfence_system();
    *(volatile unsigned *)&r->seq = a.seq;
    *a.done = a.seq;
  }
}

}  // namespace lod
