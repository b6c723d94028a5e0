// lod_kernels.cuh -- device kernels of one update cycle (insert_batch).
//
// Order of a cycle (reference: update.py:1-27, 252-393):
//   expand   k_count (+ voxel claims, pending counts) -> k_decide -> [sync] -> k_exec_chunks/k_exec_nodes (repeat)
//   resolve  k_resolve (winners set bits, per-point wins) -> k_wcount -> scan -> k_emit
//   sort     k_keys -> stable_multisplit by node id
//   alloc    k_seg_* (touched nodes, ascending id) -> scan(need) -> k_alloc_*
//   store    k_store (points + voxel centres into chunk slots)
//   epilogue k_epilogue (count += len, pending = final = 0)
//
// Voxel claims ride on the count passes.  Every inner node is descended
// through by all of its points exactly once per cycle, in one pass: nodes
// that were inner at cycle start in iteration 1 (batch points only -- spilled
// points' cells at those nodes are already set because they passed them when
// first inserted), nodes split in iteration k in iteration k+1 (their spilled
// and re-routed points).  So min-index claims into one hash per cycle see
// every candidate of a (node, cell) in the same pass, which is the reference's
// sequential first-come rule (sample_and_route, _kernels.py:125-135).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lod_common.cuh"
#include "scan.cuh"

namespace lod {

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// NodeCols::desc .y bit 31 (Geo::fresh, arenas < 128 GiB, where grid
// offsets / 64 stay below 2^31): the node split in the running cycle, its
// grid is still all clear.
constexpr int kFresh = (int)0x80000000u;

// Device-side control block; pinned host mirror is read at each sync point.
struct Ctrl {
  long long num_nodes;
  long long splits_total;
  long long max_level;
  unsigned long long arena_off;
  long long allocated_total;
  long long free_count;
  long long released_total;
  long long spill_total;  // spill points this cycle
  // per expansion iteration
  unsigned int n_touched;
  unsigned int n_splits;
  int error;
  unsigned int iter_max_level;
  long long spill_add;
  // split plan (values before the iteration's splits)
  long long plan_num_nodes0;
  long long plan_free0;
  long long plan_spill0;
  unsigned long long plan_grid0;
  // sampling
  unsigned long long n_used;  // distinct (node, cell) claims = new voxels
  unsigned int hash_overflow;
  unsigned int n_v;           // sum of per-point wins (== n_used when consistent)
  // allocation plan
  unsigned int n_keys;        // touched nodes this cycle (segments)
  unsigned int pad1;
  U64x2 seg_tot;              // (touched nodes, items)
  U64x2 acq_tot;              // (sum need, sum write-list entries)
  U64x2 pack_tot;             // the packed node-plan scan's total (k_radix_ghist layout)
  long long alloc_F;          // free stack size before allocation
  long long alloc_A;          // allocated_total before allocation
  unsigned long long chunk_base;
  long long n_items;
  // BatchDelta capture (LOD_FLAG_DELTA)
  int spec_abort;             // k_decide: a speculatively launched post-expansion pipeline must not run
  unsigned int n_xchunks;     // chunks of the iteration's splitting nodes (k_split_chunk_list)
  unsigned int d_nvg;         // voxel groups (inner nodes with new voxels)
  unsigned int d_npg;         // point groups (leaves with new points)
  long long redescend;        // k_decide: points in the splitting nodes (stored + pending) -- the only
                              // points the next count pass re-descends, each claiming at most one cell
  long long n_wins;           // k_resolve_list: entries of the win list (burst path)
  unsigned long long dir_top;  // chunk directory entries handed out (bump pointer)
  unsigned long long dir_overflow;  // a relocation found no room: directories are stale until the host
                                    // rebuilds them (fix_directory; chains stay authoritative)
  int exec_go;  // k_decide: the iteration splits and its nodes / spill fit the buffers as allocated
                // (k_exec_chunks / k_exec_nodes launched ahead of the host's read run)
  unsigned int mark_done;  // k_decide: blocks done with the split test (the last one decides)
  // device time of a cycle (globaltimer ns): k_cycle_begin stamps the start
  // (and keeps the previous cycle's pair), every k_epilogue block the end
  unsigned long long t_begin, t_end, t_prev_begin, t_prev_end;
};
static_assert(offsetof(Ctrl, dir_overflow) == offsetof(Ctrl, dir_top) + 8, "dir_claim flags dir_top + 1");

// A fresh directory region of `cap` entries, or -1 (and the overflow flag)
// when the bump pointer ran past the allocation: the host sized it from a
// soft bound (small cycles) and rebuilds every directory at its next sync.
__device__ __forceinline__ long long dir_claim(const PoolCols &pool, unsigned long long *dir_top,
                                              long long cap) {
  const unsigned long long noff = atomicAdd(dir_top, (unsigned long long)cap);
  if (noff + (unsigned long long)cap > pool.cdir_cap) {
    atomicExch(dir_top + 1, 1ull);  // Ctrl::dir_overflow follows dir_top
    return -1;
  }
  return (long long)noff;
}

// Chunk directory of node n after `need` chunks were appended to its list
// (chunk_count already includes them): relocate the region with doubling when
// it is full (one thread per node), then record the new chunk ids, `acq(t)`
// for t < need, at list positions chunk_count - need + t.
template <typename Acq>
__device__ __forceinline__ void dir_append(const NodeCols &nd, const PoolCols &pool, unsigned long long *dir_top,
                                           int n, long long need, Acq acq) {
  if (need <= 0) return;
  const long long cc1 = nd.chunk_count[n], cc0 = cc1 - need;
  long long off = nd.dir_off[n];
  if (cc1 > (long long)nd.dir_cap[n]) {
    const long long cap = cc1 * 2 > 4 ? cc1 * 2 : 4;
    const long long noff = dir_claim(pool, dir_top, cap);
    if (noff < 0) return;
    for (long long i = 0; i < cc0; ++i) pool.cdir[noff + i] = pool.cdir[off + i];
    off = noff;
    nd.dir_off[n] = noff;
    nd.dir_cap[n] = (int32_t)cap;
  }
  for (long long t = 0; t < need; ++t) pool.cdir[off + cc0 + t] = acq(t);
}

__device__ __forceinline__ void set_error(Ctrl *c, int code) { atomicCAS(&c->error, 0, code); }

constexpr int kMaxPassesHist = 4 * 256;  // radix digit totals (radix.cuh kMaxPasses * kRadixDigits)

// ---------------------------------------------------------------- claim hash

// Open-addressing table of (node, cell) -> min all-array index, 16-byte slots
// so key and value share one sector.  The value word is (index << 32 | rgba):
// a 64-bit min keeps the lowest claimant together with its colour, so the
// backlog never gathers the winner's colour back from the point arrays.
// Iteration-1 claims (at nodes inner at cycle start) carry batch index | 2^31
// because the spill length is not known yet; all claims at one node live in
// one index space, so min order is exact.
struct HSlot {
  unsigned long long key;
  unsigned long long claim;  // claimant index << 32 | its rgba
};
constexpr unsigned long long kEmptyKey = 0xFFFFFFFFFFFFFFFFULL;
constexpr uint32_t kBatchTag = 0x80000000u;

struct Hash {
  HSlot *slots;
  unsigned long long cap;    // slots (any size: the hash is range-reduced by a multiply-high)
  unsigned long long *used;  // slots inserted this cycle
  unsigned long long limit;  // capacity of `used` (= table capacity)
  unsigned long long tag;    // this cycle's epoch << 56 (0..254)
  int cbits;                 // bits of a cell index (ceil log2 g^3): keys are {epoch:8, node:56-cbits, cell:cbits}
};

// Keys carry the cycle's epoch in their top byte ({epoch:8, node, cell}: the
// node field takes the 56 - cbits bits the cell leaves, 35 at G = 128, so
// node ids reach the reference's int32 range);
// a slot is occupied iff its epoch is the current one.  Slots of earlier
// cycles are simply stale -- nothing clears the table between cycles (the
// clearing writes dirtied ~1.5M random sectors per batch that the next count
// pass had to write back); it is reset with a memset when the epoch wraps.
constexpr int kEpochs = 255;  // epoch 255 = the all-ones memset state, never live
__device__ __forceinline__ bool live(const Hash &h, unsigned long long k) { return (k >> 56) == (h.tag >> 56); }

// New keys are appended to the cycle's used-slot list through a per-warp
// shared-memory stage, so a pass issues one global atomic per warp instead of
// one per new voxel (a single hot counter otherwise serializes in L2), and
// no block-wide barrier is needed to flush it.
constexpr int kStage = 128;  // slots per warp
constexpr int kStageWarps = 8;
struct UsedStage {
  unsigned long long slot[kStageWarps][kStage];
  unsigned int n[kStageWarps];
};

__device__ __forceinline__ unsigned long long hmix(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

// Home slot: the 64-bit mix range-reduced to [0, cap) by a multiply-high (no
// power-of-two table: the sweeps read exactly the slots the load needs).
__device__ __forceinline__ unsigned long long home_slot(const Hash &h, unsigned long long key) {
  return __umul64hi(hmix(key), h.cap);
}
__device__ __forceinline__ unsigned long long next_slot(const Hash &h, unsigned long long s) {
  return s + 1 == h.cap ? 0ull : s + 1;
}

__device__ __forceinline__ unsigned long long claim_key(int nid, long long cell, int cbits) {
  return ((unsigned long long)(uint32_t)nid << cbits) | (unsigned long long)cell;
}
constexpr unsigned long long kKeyLow56 = (1ull << 56) - 1;
__device__ __forceinline__ int key_node(const Hash &h, unsigned long long k) { return (int)((k & kKeyLow56) >> h.cbits); }
__device__ __forceinline__ uint32_t key_cell(const Hash &h, unsigned long long k) {
  return (uint32_t)(k & ((1ull << h.cbits) - 1));
}

__device__ __forceinline__ void used_init(UsedStage &stg) {
  if ((threadIdx.x & 31) == 0) stg.n[threadIdx.x >> 5] = 0;
  __syncwarp();
}

__device__ __forceinline__ void used_append(const Hash &h, UsedStage &stg, unsigned long long slot, Ctrl *ctrl) {
  const int w = threadIdx.x >> 5;
  const unsigned k = atomicAdd(&stg.n[w], 1u);
  if (k < (unsigned)kStage) {
    stg.slot[w][k] = slot;
  } else {  // stage full: direct append
    const unsigned long long u = atomicAdd(&ctrl->n_used, 1ull);
    if (u < h.limit) h.used[u] = slot;
    else ctrl->hash_overflow = 1;
  }
}

// Warp epilogue of a claiming pass (all lanes): flush the warp's staged slots.
__device__ __forceinline__ void used_flush(const Hash &h, UsedStage &stg, Ctrl *ctrl) {
  __syncwarp();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned n = min(stg.n[w], (unsigned)kStage);
  unsigned long long base = 0;
  if (lane == 0 && n) base = atomicAdd(&ctrl->n_used, (unsigned long long)n);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (unsigned i = lane; i < n; i += 32) {
    const unsigned long long u = base + i;
    if (u < h.limit) h.used[u] = stg.slot[w][i];
    else ctrl->hash_overflow = 1;
  }
}

// 16-byte compare-and-swap of a whole slot (ATOMG.CAS.128): a new key is
// installed together with its first claimant's index in one atomic.
__device__ __forceinline__ ulonglong2 cas_slot(HSlot *sl, ulonglong2 cmp, ulonglong2 val) {
  ulonglong2 old;
  asm volatile(
      "{\n\t.reg .b128 d, b, c;\n\t"
      "mov.b128 b, {%2, %3};\n\t"
      "mov.b128 c, {%4, %5};\n\t"
      "atom.global.cas.b128 d, [%6], b, c;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(old.x), "=l"(old.y)
      : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(sl)
      : "memory");
  return old;
}

constexpr unsigned long long kEmptyHi = 0xFFFFFFFFFFFFFFFFULL;  // claim = all ones (index 0xFFFFFFFF)

// Min-combine `v` into the claim of `key`.  Lower indices run earlier, so a
// claimant usually finds a smaller index already there and issues no atomic.
__device__ __forceinline__ void hash_claim(const Hash &h, UsedStage &stg, unsigned long long key, uint32_t v,
                                           uint32_t rgba, Ctrl *ctrl) {
  key |= h.tag;
  unsigned long long slot = home_slot(h, key);
  for (unsigned long long probe = 0; probe < h.cap; ++probe) {
    HSlot *sl = h.slots + slot;
    const unsigned long long mine = ((unsigned long long)v << 32) | rgba;
    ulonglong2 cur = __ldcg(reinterpret_cast<const ulonglong2 *>(sl));
    while (!live(h, cur.x)) {  // empty or stale: install over exactly what was read
      const ulonglong2 old = cas_slot(sl, cur, make_ulonglong2(key, mine));
      if (old.x == cur.x && old.y == cur.y) {
        used_append(h, stg, slot, ctrl);
        return;
      }
      cur = old;
    }
    if (cur.x == key) {
      if ((uint32_t)(cur.y >> 32) > v) atomicMin(&sl->claim, mine);
      return;
    }
    slot = next_slot(h, slot);
  }
  ctrl->hash_overflow = 1;  // table full
}

// Claim at one inner node if the cell's bit is clear (bits never clear and
// nothing sets bits until k_resolve, so "clear" means clear at cycle start).
__device__ __forceinline__ void probe_cell(const NodeCols &nd, const Geo &geo, const uint32_t *grid32,
                                           const Hash &h, UsedStage &stg, Ctrl *ctrl, int nid, double x,
                                           double y, double z, double bx, double by, double bz, double s,
                                           double inv_s, uint32_t v, uint32_t rgba) {
  const long long cell = cell_of(geo, x, y, z, bx, by, bz, s, inv_s);
  const uint32_t w = __ldg(grid32 + (nd.grid_off[nid] >> 2) + (cell >> 5));
  if (!(w & (1u << (cell & 31)))) hash_claim(h, stg, claim_key(nid, cell, h.cbits), v, rgba, ctrl);
}

// Grow the claim table between expansion iterations: re-insert every key
// claimed so far (keys are unique, values carried) into the new table.
__global__ void k_rehash(const HSlot *__restrict__ old_slots, Hash h, const Ctrl *ctrl) { lod::pdl_wait();
  const unsigned long long nu = ctrl->n_used;
  for (long long u = gtid(); u < (long long)nu; u += gstride()) {
    const HSlot o = old_slots[h.used[u]];
    unsigned long long slot = home_slot(h, o.key);
    const ulonglong2 nv = make_ulonglong2(o.key, o.claim);
    for (;;) {  // empty or stale (an earlier cycle's epoch): install over exactly what was read
      HSlot *sl = h.slots + slot;
      ulonglong2 cur = __ldcg(reinterpret_cast<const ulonglong2 *>(sl));
      bool done = false;
      while (!live(h, cur.x)) {
        const ulonglong2 old = cas_slot(sl, cur, nv);
        if (old.x == cur.x && old.y == cur.y) {
          done = true;
          break;
        }
        cur = old;
      }
      if (done) break;
      slot = next_slot(h, slot);
    }
    h.used[u] = slot;
  }
}

// ---------------------------------------------------------------- expansion

// _kernels.count_points (_kernels.py:27-63) fused with the voxel claims of
// sample_and_route (_kernels.py:101-137).  Iteration 1 descends every batch
// point from the root; later iterations re-descend only points whose cached
// node became inner, starting at that node (its stored bmin equals the
// accumulated descent bounds byte for byte, _kernels.py:9-13).
#ifndef LOD_COUNT_MINB
#define LOD_COUNT_MINB 6  // blocks per SM (40 registers; same-box A/B: 6 > 5 > 4, 8)
#endif
#ifndef LOD_COUNT_MINB_F32
#define LOD_COUNT_MINB_F32 6  // 40 registers, no spills (A/B on terrain: 6 > 8; f64 at 6 is 3 % slower)
#endif

// One point's descent from inner node `nid` (descent record d) to its leaf,
// claiming every clear cell it crosses (claimant index v, colour col).
// T = float on Geo::f32ok trees (the f32 twins in lod_common.cuh: identical
// results, half the registers of the f64 state -> more resident warps).
#ifndef LOD_COUNT_PIPE
#define LOD_COUNT_PIPE 1  // f32 descent only (the f64 state spills with it); A/B: count phase 0.139-0.141 vs 0.143 ms
#endif
template <typename T>
__device__ __forceinline__ int count_descend(const NodeCols &nd, const Geo &geo, const uint32_t *__restrict__ grid32,
                                             const Hash &h, UsedStage &stg, Ctrl *ctrl, int nid, int2 d, T x, T y,
                                             T z, uint32_t v, uint32_t col) {
  T bx = (T)nd.bmin[3 * nid], by = (T)nd.bmin[3 * nid + 1], bz = (T)nd.bmin[3 * nid + 2];
  const int lvl0 = nd.level[nid];
  T s = (T)geo.size_by_level[lvl0], inv_s = (T)geo.inv_by_level[lvl0];
  // one dependent load per level, from the compact (L1-resident) descent
  // table; grid words bypass L1 so they do not evict it
  if constexpr (LOD_COUNT_PIPE && sizeof(T) == 4) {
  // the next level's grid word is loaded before this level's claim (claims
  // never set grid bits -- k_resolve does -- so the word is the same either way)
  long long cell = cell_of(geo, x, y, z, bx, by, bz, s, inv_s);
  uint32_t w = (geo.fresh && d.y < 0)
                   ? 0u
                   : ld_nol1(grid32 + ((unsigned long long)((uint32_t)d.y & geo.gmask) << 4) + (cell >> 5));
  do {
    const int cur = nid;
    const long long ccur = cell;
    const uint32_t wcur = w;
    nid = d.x + octant_step(x, y, z, bx, by, bz, s, inv_s);
    d = __ldg(nd.desc + nid);
    if (d.x >= 0) {
      cell = cell_of(geo, x, y, z, bx, by, bz, s, inv_s);
      w = (geo.fresh && d.y < 0)
              ? 0u
              : ld_nol1(grid32 + ((unsigned long long)((uint32_t)d.y & geo.gmask) << 4) + (cell >> 5));
    }
    if (!(wcur & (1u << (ccur & 31)))) {
      const unsigned long long key = claim_key(cur, ccur, h.cbits);
      const unsigned m = __activemask();
      const unsigned lane = lane_id();
      const unsigned long long left = __shfl_up_sync(m, key, 1);
      if (!(lane > 0 && ((m >> (lane - 1)) & 1u) && left == key)) hash_claim(h, stg, key, v, col, ctrl);
    }
  } while (d.x >= 0);
  return nid;
  } else {
  do {
    const long long cell = cell_of(geo, x, y, z, bx, by, bz, s, inv_s);
    // a node split in this cycle has an all-clear grid (fresh arena, bits
    // are set only by k_resolve): its claims need no grid word
    const uint32_t w = (geo.fresh && d.y < 0)
                           ? 0u
                           : ld_nol1(grid32 + ((unsigned long long)((uint32_t)d.y & geo.gmask) << 4) + (cell >> 5));
    const int cur = nid;
    nid = d.x + octant_step(x, y, z, bx, by, bz, s, inv_s);
    d = __ldg(nd.desc + nid);
    if (!(w & (1u << (cell & 31)))) {
      // a lane whose left neighbour (the next lower index: the lanes of a
      // warp are consecutive points) claims the same (node, cell) cannot
      // win: it need not touch the table (locality-ordered input puts runs
      // of lanes on one cell; one shuffle, where a MATCH.ANY + REDUX per
      // claim cost the random-order stream 7 % of the pass)
      const unsigned long long key = claim_key(cur, cell, h.cbits);
      const unsigned m = __activemask();
      const unsigned lane = lane_id();
      const unsigned long long left = __shfl_up_sync(m, key, 1);
      if (!(lane > 0 && ((m >> (lane - 1)) & 1u) && left == key)) hash_claim(h, stg, key, v, col, ctrl);
    }
  } while (d.x >= 0);
  return nid;
  }
}

// The leaf's pending count (fire-and-forget, warp-aggregated): k_decide
// finds the touched leaves by their pending counts.
__device__ __forceinline__ void count_pending(const NodeCols &nd, int leaf) {
  const unsigned act = __ballot_sync(0xffffffffu, leaf >= 0);
  if (leaf >= 0) {
    const unsigned peers = __match_any_sync(act, leaf);
    if ((peers & lanemask_lt()) == 0) atomicAdd(&nd.pending[leaf], (unsigned long long)__popc(peers));
  }
}

template <typename T>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? LOD_COUNT_MINB_F32 : LOD_COUNT_MINB)
    k_count(NodeCols nd, Geo geo, PointSrc src, NodeOf node_of, long long n, int first,
            const uint32_t *__restrict__ grid32, Hash h, Ctrl *ctrl, float4 *__restrict__ copy_out) {
  lod::pdl_wait();
  __shared__ UsedStage stg;
  used_init(stg);
  for (long long j0 = (long long)blockIdx.x * blockDim.x; j0 < n; j0 += gstride()) {
    long long j = j0 + threadIdx.x;
    int leaf = -1;
    if (j < n) {
      int nid = first ? 0 : node_of[j];
      int2 d = __ldg(nd.desc + nid);  // {first child | -1, grid offset / 64}
      // copy_out (iteration 1 of a device batch): the batch as packed records,
      // which every later pass reads, so the caller's arrays are released
      // after this pass instead of after the cycle
      if (copy_out) __stcg(copy_out + j, src.record(j));
      if (d.x >= 0) {
        float xf, yf, zf;
        src.xyz(j, xf, yf, zf);
        const uint32_t v = first ? ((uint32_t)j | kBatchTag) : (uint32_t)j;
        nid = count_descend<T>(nd, geo, grid32, h, stg, ctrl, nid, d, (T)xf, (T)yf, (T)zf, v, src.rgba(j));
        node_of[j] = nid;
        if (!nd.final_[nid]) leaf = nid;
      } else if (first) {
        node_of[j] = nid;
        if (!nd.final_[nid]) leaf = nid;
      }
    }
    count_pending(nd, leaf);
  }
  used_flush(h, stg, ctrl);
}

// Iteration 1 of the count pass (every batch point from the root) with the
// batch staged through shared memory (north_star item 1): each CTA takes one
// kCountTile-point tile, has the TMA engine copy it global -> shared
// (cp.async.bulk: 3 KB of xyz + 1 KB of rgba, or 4 KB of packed records,
// one mbarrier) and descends from shared memory; the CTAs resident on an SM
// overlap one another's copies with their descents, and the hardware block
// scheduler keeps the load balanced (per-point cost varies with the claims).
// Measured against the plain k_count on the terrain stream (same box, A/B,
// count phase median per 1M batch): this kernel 0.183 ms vs 0.177 ms (each
// CTA waits for its whole tile before the first descent step); warp-level
// double-buffered 32-point tiles with a per-warp ticket 0.211 ms (more
// instructions per point), 128-point warp tiles 0.35 ms (coarse work units
// against a per-point cost that varies with the claims), a block-wide
// double-buffered tile with a top-level counting sort 0.205 ms.  The pass is
// bound by the dependent grid-word loads and the claim CAS (ncu: 24 % / 30 %
// of the stall samples), not by the batch reads (8 %), so the plain pass
// stays the default; this one runs with LOD_COUNT_STAGED=1.
// Full tiles only (the ragged tail tile loads directly); 16-byte aligned
// batch base addresses.
constexpr int kCountTile = 256;
template <bool PACKED>
__global__ void __launch_bounds__(kCountTile, LOD_COUNT_MINB)
    k_count_staged(NodeCols nd, Geo geo, PointSrc src, NodeOf node_of, long long n,
                   const uint32_t *__restrict__ grid32, Hash h, Ctrl *ctrl) { lod::pdl_wait();
  __shared__ UsedStage stg;
  __shared__ alignas(128) float4 sbuf[kCountTile];
  __shared__ unsigned long long bar;
  const int tid = threadIdx.x;
  used_init(stg);
  const long long t = blockIdx.x, nfull = n / kCountTile;
  const bool staged = t < nfull;
  if (tid == 0 && staged) {
    mbar_init(&bar, 1);
    mbar_arrive_expect_tx(&bar, kCountTile * 16u);
    if (PACKED) {
      bulk_g2s(sbuf, src.brec + t * kCountTile, kCountTile * 16u, &bar);
    } else {
      bulk_g2s(sbuf, src.bxyz + t * 3 * kCountTile, kCountTile * 12u, &bar);
      bulk_g2s(reinterpret_cast<char *>(sbuf) + kCountTile * 12, src.brgba + t * kCountTile, kCountTile * 4u, &bar);
    }
  }
  const int2 d0 = __ldg(nd.desc);
  const long long j = t * kCountTile + tid;
  float xf = 0.f, yf = 0.f, zf = 0.f;
  uint32_t col = 0;
  if (staged) {
    __syncthreads();  // the barrier is initialised before anyone waits on it
    mbar_wait(&bar, 0);
    if (PACKED) {
      const float4 r = sbuf[tid];
      xf = r.x, yf = r.y, zf = r.z, col = __float_as_uint(r.w);
    } else {
      const float *sx = reinterpret_cast<const float *>(sbuf);
      xf = sx[3 * tid], yf = sx[3 * tid + 1], zf = sx[3 * tid + 2];
      col = reinterpret_cast<const uint32_t *>(reinterpret_cast<const char *>(sbuf) + kCountTile * 12)[tid];
    }
  } else if (j < n) {
    src.xyz(j, xf, yf, zf);
    col = src.rgba(j);
  }
  int leaf = -1;
  if (j < n) {
    int nid = 0;
    if (d0.x >= 0)
      nid = count_descend<double>(nd, geo, grid32, h, stg, ctrl, 0, d0, xf, yf, zf, (uint32_t)j | kBatchTag, col);
    node_of[j] = nid;
    if (!nd.final_[nid]) leaf = nid;
  }
  count_pending(nd, leaf);
  used_flush(h, stg, ctrl);
}

// _split_pass (update.py:226-249): split iff count + pending > T and
// level < max_depth, else mark final.  k_decide's first phase tests every leaf touched
// in this iteration -- a leaf, not final, with pending points (pending 0 -> 1
// is the reference's touched rule, _kernels.py:59-61; every leaf touched in an
// earlier iteration is final or split by now) -- over all nodes grid-wide
// (a large tree touches tens of thousands per batch) and flags the
// splits in a bitmap over node ids; the last of its CTAs to finish ranks them by ascending
// node id (popcount prefix over the bitmap words), so child ids
// num_nodes + 8*rank match the reference's sorted-id split order
// (octree.py:249-261), and plans the spill segments (ascending id, stored
// order), free-stack pushes (walk order) and grid offsets, detecting
// SpillOverflow / OutOfArena in reference order.
constexpr int kDecideBlock = 1024;
__global__ void __launch_bounds__(kDecideBlock)
    k_decide(NodeCols nd, Geo geo, uint32_t *bitmap, int32_t *split_list, int32_t *srank, long long *scnt,
             long long *schk, long long *spill_off, long long *chunk_off, Ctrl *ctrl, long long spill_cap,
             unsigned long long arena_cap, long long backlog_cap, Ctrl *host, volatile unsigned *host_seq,
             unsigned seq, long long spill_buf_cap, long long node_cap, long long num_nodes) { lod::pdl_wait();
  // phase 1, every block: the split test over a
  // grid-stride share of the nodes; the last block to finish then ranks and
  // plans (one launch per decision instead of two)
  for (long long t = gtid(); t < num_nodes; t += gstride()) {
    const int nid = (int)t;
    const unsigned long long pend = nd.pending[nid];
    if (pend == 0 || nd.inner[nid] || nd.final_[nid]) continue;
    const long long tot = nd.count[nid] + (long long)pend;
    if (tot > geo.T && nd.level[nid] < geo.max_depth) atomicOr(&bitmap[nid >> 5], 1u << (nid & 31));
    else nd.final_[nid] = 1;
  }
  if (gridDim.x > 1) {
    __shared__ unsigned s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&ctrl->mark_done, 1u) == gridDim.x - 1 ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) ctrl->mark_done = 0;
  }
  __syncthreads();
  __shared__ uint32_t sh32[kDecideBlock / 32 + 1];
  __shared__ U64x2 sh64[kDecideBlock / 32 + 1];
  __shared__ unsigned int s_maxlvl;
  __shared__ long long s_err_spill;
  __shared__ unsigned long long s_pend;  // pending points of the splitting nodes
  const int tid = threadIdx.x;
  const long long nn = ctrl->num_nodes;
  if (tid == 0) {
    s_maxlvl = 0;
    s_err_spill = -1;
    s_pend = 0;
  }
  // phase 2: popcount prefix over the bitmap words (contiguous word ranges per thread)
  const long long W = (nn + 31) / 32;
  const long long per = (W + kDecideBlock - 1) / kDecideBlock;
  const long long w0 = tid * per, w1 = min(W, w0 + per);
  uint32_t local = 0;
  for (long long w = w0; w < w1; ++w) local += __popc(__ldcg(bitmap + w));
  uint32_t total;
  uint32_t run = block_exclusive_scan<uint32_t, kDecideBlock>(local, sh32, total);
  const unsigned ns = total;
  // phase 3: the splits in id order out of the words (rank = running prefix),
  // their counts; the words are cleared for the next iteration
  for (long long w = w0; w < w1; ++w) {
    uint32_t wv = __ldcg(bitmap + w);
    if (!wv) continue;
    bitmap[w] = 0;
    while (wv) {
      const int b = __ffs(wv) - 1;
      wv &= wv - 1;
      const int nid = (int)(w * 32 + b);
      split_list[run] = nid;
      srank[nid] = (int32_t)run;
      scnt[run] = nd.count[nid];
      schk[run] = nd.chunk_count[nid];
      atomicAdd(&s_pend, (unsigned long long)nd.pending[nid]);
      atomicMax(&s_maxlvl, (unsigned)(nd.level[nid] + 1));
      ++run;
    }
  }
  __syncthreads();
  // phase 4: exclusive scans over ranks (spill offsets, free-stack offsets)
  const long long spill0 = ctrl->spill_total;
  U64x2 carry = u64x2(0, 0);
  for (unsigned base = 0; base < ns; base += kDecideBlock) {
    unsigned r = base + tid;
    U64x2 v = u64x2(0, 0);
    if (r < ns) v = u64x2((unsigned long long)scnt[r], (unsigned long long)schk[r]);
    U64x2 tot;
    U64x2 ex = block_exclusive_scan<U64x2, kDecideBlock>(v, sh64, tot);
    ex = ex + carry;
    if (r < ns) {
      spill_off[r] = (long long)ex.a;
      chunk_off[r] = (long long)ex.b;
      // SpillBuffer.append raises before the node's grid alloc (octree.py:231-244)
      if (v.a > 0 && spill0 + (long long)(ex.a + v.a) > spill_cap)
        atomicMin((unsigned long long *)&s_err_spill, (unsigned long long)r);
    }
    carry = carry + tot;
    __syncthreads();
  }
  // phase 5: errors and counters (thread 0)
  if (tid == 0) {
    unsigned long long off = ctrl->arena_off;
    const unsigned long long gb = (unsigned long long)geo.grid_bytes;
    const unsigned long long g0 = (off + 63ull) / 64ull * 64ull;
    const unsigned long long gstride_b = (gb + 63ull) / 64ull * 64ull;
    long long err_ooa = -1;
    if (ns > 0) {
      // first k with g0 + k*gstride + gb > cap
      if (g0 + gb > arena_cap) err_ooa = 0;
      else if (g0 + (unsigned long long)(ns - 1) * gstride_b + gb > arena_cap)
        err_ooa = (long long)((arena_cap - gb - g0) / gstride_b) + 1;
    }
    long long es = s_err_spill;
    if (es >= 0 && (err_ooa < 0 || es <= err_ooa)) set_error(ctrl, 2 /*LOD_E_SPILL_OVERFLOW*/);
    else if (err_ooa >= 0) set_error(ctrl, 1 /*LOD_E_OUT_OF_ARENA*/);
    ctrl->n_splits = ns;
    ctrl->spill_add = (long long)carry.a;
    ctrl->redescend = (long long)carry.a + (long long)s_pend;
    ctrl->plan_num_nodes0 = nn;
    ctrl->plan_free0 = ctrl->free_count;
    ctrl->plan_spill0 = spill0;
    ctrl->plan_grid0 = g0;
    ctrl->iter_max_level = s_maxlvl;
    // a post-expansion pipeline launched behind this decision runs only if the
    // expansion settled here and the claims fit (else the host takes over)
    ctrl->spec_abort = (ctrl->error != 0 || ns > 0 || ctrl->hash_overflow != 0 ||
                        (long long)ctrl->n_used > backlog_cap) ? 1 : 0;
    ctrl->n_xchunks = 0;
    ctrl->exec_go = (ctrl->error == 0 && ns > 0 && spill0 + (long long)carry.a <= spill_buf_cap &&
                     nn + 8ll * ns <= node_cap) ? 1 : 0;
    if (ctrl->error == 0 && ns > 0) {
      ctrl->num_nodes = nn + 8ll * ns;
      ctrl->splits_total += ns;
      if ((long long)s_maxlvl > ctrl->max_level) ctrl->max_level = s_maxlvl;
      ctrl->free_count += (long long)carry.b;
      ctrl->released_total += (long long)carry.b;
      ctrl->spill_total = spill0 + (long long)carry.a;
      ctrl->arena_off = g0 + (unsigned long long)(ns - 1) * gstride_b + gb;
    }
  }
  if (tid == 0) ctrl->n_touched = 0;  // phase 6: the touched list restarts next iteration
  // phase 7 (host != null): the decision goes straight to the host's mapped
  // copy of the control block (k_publish's job, without its launch)
  if (host) {
    __syncthreads();
    if (tid < 32) {
      constexpr int kWords = (int)(sizeof(Ctrl) / 8);
      const unsigned long long *src = reinterpret_cast<const unsigned long long *>(ctrl);
      volatile unsigned long long *dst = reinterpret_cast<volatile unsigned long long *>(host);
      for (int k = tid; k < kWords; k += 32) dst[k] = __ldcg(src + k);
      __threadfence_system();
      __syncwarp();
      if (tid == 0) *host_seq = seq;
    }
  }
}

// Octree.split, part 1 (octree.py:231-237, store.py:125-143): the chunks of
// the splitting nodes, read from their directories -- the work list is the
// exclusive scan of their chunk counts k_decide already made (chunk_off), so
// a split touches only its own chunks, never the pool.  One warp per chunk:
// copy its records to the node's spill segment (list position = storage
// order) and push the chunk onto the free stack at its walk-order slot.
__global__ void k_exec_chunks(NodeCols nd, PoolCols pool, Geo geo, const uint8_t *__restrict__ arena,
                              const int32_t *__restrict__ split_list, long long ns,
                              const long long *__restrict__ spill_off, const long long *__restrict__ chunk_off,
                              long long nchunks, float4 *spill_buf, int32_t *spill_node_of, const Ctrl *ctrl) {
  lod::pdl_wait();
  if (nchunks < 0) {  // launched ahead of the host's read of the decision (k_exec_nodes)
    if (!ctrl->exec_go) return;
    ns = ctrl->n_splits;
    nchunks = ctrl->free_count - ctrl->plan_free0;
  }
  // one CTA per chunk (a chunk is C records: a warp each left most of the GPU
  // idle on the few hundred chunks a split moves)
  __shared__ long long s_r, s_ci, s_sp;
  __shared__ int s_owner, s_cid, s_occ;
  for (long long q = blockIdx.x; q < nchunks; q += gridDim.x) {
    if (threadIdx.x == 0) {
      long long lo = 0, hi = ns - 1;  // last split rank whose chunks start at or before q
      while (lo < hi) {
        const long long mid = (lo + hi + 1) >> 1;
        if (chunk_off[mid] <= q) lo = mid;
        else hi = mid - 1;
      }
      const long long ci = q - chunk_off[lo];
      const int owner = split_list[lo];
      const int cid = pool.cdir[nd.dir_off[owner] + ci];
      s_r = lo;
      s_ci = ci;
      s_owner = owner;
      s_cid = cid;
      s_occ = pool.occupied[cid];
      s_sp = ctrl->plan_spill0 + spill_off[lo] + ci * geo.C;
    }
    __syncthreads();
    const int owner = s_owner, cid = s_cid, occ = s_occ;
    const long long sp = s_sp;
    const float4 *src = reinterpret_cast<const float4 *>(arena + pool.payload_off[cid]);
    for (int k = threadIdx.x; k < occ; k += blockDim.x) {
      spill_buf[sp + k] = src[k];
      spill_node_of[sp + k] = owner;
    }
    if (threadIdx.x == 0) {
      pool.free_stack[ctrl->plan_free0 + chunk_off[s_r] + s_ci] = (int32_t)cid;
      pool.occupied[cid] = 0;
      pool.next[cid] = LOD_NO_CHUNK;
      pool.owner[cid] = -1;
      pool.cidx[cid] = -1;
    }
    __syncthreads();  // the shared slots are reused by the next chunk
  }
}

// Octree.split, part 2 (octree.py:238-264): the node turns inner with a zeroed
// grid (arena regions are zeroed and never reused) and gets 8 children in
// octant order with bmin = base + half (f64).  One thread per (split, octant).
// ns < 0: launched ahead of the host's read of the decision -- the count is
// the device's, and nothing runs unless k_decide set exec_go.
__global__ void k_exec_nodes(NodeCols nd, Geo geo, const int32_t *__restrict__ split_list, int32_t *srank,
                             long long ns, const Ctrl *ctrl) { lod::pdl_wait();
  if (ns < 0) {
    if (!ctrl->exec_go) return;
    ns = ctrl->n_splits;
  }
  for (long long t = gtid(); t < ns * 8; t += gstride()) {
    const long long k = t >> 3;
    const int o = (int)(t & 7);
    const int nid = split_list[k];
    const int lvl = nd.level[nid];
    const int c = (int)(ctrl->plan_num_nodes0 + 8ll * k + o);
    // node_size(nid) * 0.5 == size * 0.5**level * 0.5 (octree.py:246, 268-269)
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
    srank[c] = -1;
    if (o == 0) {
      nd.count[nid] = 0;
      nd.pending[nid] = 0;
      nd.inner[nid] = 1;
      nd.chunk_head[nid] = LOD_NO_CHUNK;
      nd.chunk_tail[nid] = LOD_NO_CHUNK;
      nd.chunk_count[nid] = 0;
      const unsigned long long gstride_b = ((unsigned long long)geo.grid_bytes + 63ull) / 64ull * 64ull;
      const unsigned long long goff = ctrl->plan_grid0 + (unsigned long long)k * gstride_b;
      nd.grid_off[nid] = (long long)goff;
      // kFresh: the grid is all clear until k_resolve (k_epilogue drops the bit)
      nd.desc[nid] = make_int2((int)(ctrl->plan_num_nodes0 + 8ll * k),
                               (int)((uint32_t)(goff >> 6) | (geo.fresh ? (uint32_t)kFresh : 0u)));
      srank[nid] = -1;
    }
  }
}

// ---------------------------------------------------------------- sampling

// Fallback claim pass (only when the cycle's claim table overflowed): a full
// descent of every point over the final topology with all-array indices.
__global__ void k_claim(NodeCols nd, Geo geo, PointSrc src, const uint32_t *__restrict__ grid32, long long n,
                        Hash h, Ctrl *ctrl) { lod::pdl_wait();
  __shared__ UsedStage stg;
  used_init(stg);
  for (long long j0 = (long long)blockIdx.x * blockDim.x; j0 < n; j0 += gstride()) {
    const long long j = j0 + threadIdx.x;
    if (j >= n) continue;
    float xf, yf, zf;
    src.xyz(j, xf, yf, zf);
    const double x = xf, y = yf, z = zf;
    double bx = geo.bmin0[0], by = geo.bmin0[1], bz = geo.bmin0[2], s = geo.size0, inv_s = geo.inv_by_level[0];
    int nid = 0;
    while (nd.inner[nid]) {
      probe_cell(nd, geo, grid32, h, stg, ctrl, nid, x, y, z, bx, by, bz, s, inv_s, (uint32_t)j, src.rgba(j));
      const int o = octant_step(x, y, z, bx, by, bz, s, inv_s);
      nid = nd.children[8 * nid + o];
    }
  }
  used_flush(h, stg, ctrl);
}

// Every distinct claimed (node, cell): the min index is the winner.  Two
// sequential sweeps of the claim table (every sector read once, coalesced;
// a table larger than L2 costs a streaming read, not a DRAM round trip per
// voxel, and no list or cursor is needed):
//   k_resolve: set the cell's bit and count the win for its winner
//     (fire-and-forget atomics: nothing waits on them);
//   k_scatter (after the exclusive scan wbase of the win counts): take a rank
//     among the winner's wins by counting its count back down (atomicSub --
//     which also leaves the counts zeroed for the next cycle), write the
//     backlog entry at wbase[j] + rank and free the slot.
// The backlog order inside a node is ascending winner index (sample_and_route
// appends per point, _kernels.py:100-151, and a point wins at most one cell
// per node), so a point's own wins -- all at different nodes -- may take any
// order: the stable node sort separates them.
// The same two passes over the cycle's used-slot list instead of the whole
// table (the list holds exactly the installed slots, h.used[0 .. n_used)):
// while the table is L2-resident the random slot reads are cheaper than a
// sweep over every slot (~40 % of which are live).
template <bool LIST>
__device__ __forceinline__ bool claim_slot(const Hash &h, const Ctrl *ctrl, long long i, ulonglong2 &kv,
                                           long long &sidx) {
  if (LIST) {
    if (i >= (long long)min(ctrl->n_used, h.limit)) return false;
    sidx = (long long)h.used[i];
  } else {
    if (i >= (long long)h.cap) return false;
    sidx = i;
  }
  kv = __ldcg(reinterpret_cast<const ulonglong2 *>(h.slots + sidx));
  return live(h, kv.x);
}

__device__ __forceinline__ long long claim_index(uint32_t v, long long n_s) {
  return (v & kBatchTag) ? n_s + (long long)(v & ~kBatchTag) : (long long)v;
}

template <bool LIST>
__global__ void __launch_bounds__(256)
    k_resolve(NodeCols nd, Hash h, uint32_t *grid32, long long n_s, uint32_t *__restrict__ wcount, const Ctrl *ctrl,
              const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  const long long H = LIST ? (long long)h.limit : (long long)h.cap;
  for (long long i = gtid(); i < H; i += gstride()) {
    ulonglong2 kv;
    long long sidx;
    if (!claim_slot<LIST>(h, ctrl, i, kv, sidx)) {
      if (LIST) break;
      continue;
    }
    const int nid = key_node(h, kv.x);
    const uint32_t cell = key_cell(h, kv.x);
    atomicOr(grid32 + (nd.grid_off[nid] >> 2) + (cell >> 5), 1u << (cell & 31));
    atomicAdd(wcount + claim_index((uint32_t)(kv.y >> 32), n_s), 1u);
  }
}

template <bool LIST>
__global__ void __launch_bounds__(256)
    k_scatter(Hash h, long long n_s, const uint32_t *__restrict__ wbase, uint32_t *__restrict__ wcount, PointSrc src,
              uint4 *__restrict__ backlog, const Ctrl *ctrl, const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  const long long H = LIST ? (long long)h.limit : (long long)h.cap;
  for (long long i = gtid(); i < H; i += gstride()) {
    ulonglong2 kv;
    long long sidx;
    if (!claim_slot<LIST>(h, ctrl, i, kv, sidx)) {  // stale slots are left in place
      if (LIST) break;
      continue;
    }
    const long long j = claim_index((uint32_t)(kv.y >> 32), n_s);
    const uint32_t b = __ldg(wbase + j) + atomicSub(wcount + j, 1u) - 1u;
    backlog[b] = make_uint4((uint32_t)key_node(h, kv.x), key_cell(h, kv.x), (uint32_t)kv.y,
                            (uint32_t)j);  // .w: the winner's all-array index (lod_last_voxels)
  }
}

// ---------------------------------------------------------------- sort + alloc

// Touched nodes of the cycle = nodes with new samples (k_radix_prep's per-node
// item counts), in ascending id.  Leaves and inner nodes are disjoint, so the
// stable sort by node id lays every node's new samples out contiguously, in
// reference slot order, starting at the exclusive prefix of the counts (the
// (flag, count) pairs are written by k_radix_ghist).

__device__ __forceinline__ long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

// Segment list + collect_allocs (_kernels.py:253-277): per touched node its
// dense id, segment start and chunk need = ceil((count+pending)/C) -
// chunk_count -- in ascending node id (chunk ids are not observable; the
// acquisition count and the arena growth are the reference's).
// Packed per-node plan (written by k_radix_ghist, scanned once): .a = touched
// flag << 40 | item count, .b = need << 32 | write-list entries (need +
// partial tail).  Exclusive sums stay inside their fields (< 2^24 nodes,
// < 2^40 items, < 2^32 acquisitions per cycle), so one scan yields every
// touched node's dense id, segment start, acquisition start and write-list
// start.
constexpr int kPackShift = 40;
constexpr unsigned long long kPackLow = (1ull << kPackShift) - 1;
__device__ __forceinline__ U64x2 node_plan(const NodeCols &nd, const Geo &geo, long long n, uint32_t len) {
  if (!len) return u64x2(0, 0);
  const long long cnt = nd.count[n];
  const long long need = ceil_div(cnt + len, geo.C) - ceil_div(cnt, geo.C);
  const long long partial = (cnt % geo.C) != 0;
  return u64x2((1ull << kPackShift) | (unsigned long long)len,
               ((unsigned long long)need << 32) | (unsigned long long)(need + partial));
}

struct NodePlanOf {
  NodeCols nd;
  Geo geo;
  __device__ __forceinline__ U64x2 operator()(long long n, uint32_t len) const { return node_plan(nd, geo, n, len); }
};

// k_seg_list's work, per node and for the totals, for a kernel that has the
// node's count and its scanned plan prefix in registers (direct placement:
// the column scan's last row block, radix.cuh k_tile_colscan).
struct SegFinish {
  NodeCols nd;
  Geo geo;
  int32_t *seg_node;
  long long *seg_start;
  int32_t *dense;
  U64x2 *plan;
  U64x2 *plan_ex;
  Ctrl *ctrl;
  __device__ __forceinline__ U64x2 plan_of(long long n, uint32_t len) const { return node_plan(nd, geo, n, len); }
  __device__ __forceinline__ void node(long long i, uint32_t len, const U64x2 &ex, const U64x2 &own) const {
    if (!len) return;
    const long long d = (long long)(ex.a >> kPackShift);
    seg_node[d] = (int32_t)i;
    seg_start[d] = (long long)(ex.a & kPackLow);
    dense[i] = (int32_t)d;
    plan[d] = u64x2(own.b >> 32, own.b & 0xFFFFFFFFull);
    plan_ex[d] = u64x2(ex.b >> 32, ex.b & 0xFFFFFFFFull);
  }
  __device__ __forceinline__ void total(const U64x2 &tot) const {
    ctrl->pack_tot = tot;
    const unsigned long long K = tot.a >> kPackShift;
    ctrl->seg_tot = u64x2(K, tot.a & kPackLow);
    ctrl->acq_tot = u64x2(tot.b >> 32, tot.b & 0xFFFFFFFFull);
    seg_start[K] = (long long)(tot.a & kPackLow);
    ctrl->n_keys = (unsigned)K;
    ctrl->alloc_F = ctrl->free_count;
    ctrl->alloc_A = ctrl->allocated_total;
    ctrl->chunk_base = (ctrl->arena_off + 15ull) / 16ull * 16ull;
  }
};

__global__ void k_seg_list(NodeCols nd, Geo geo, uint32_t *__restrict__ nodecnt, long long num_nodes,
                           const U64x2 *__restrict__ pairs_ex, int32_t *__restrict__ seg_node,
                           long long *__restrict__ seg_start, int32_t *__restrict__ dense, U64x2 *__restrict__ plan,
                           U64x2 *__restrict__ plan_ex, Ctrl *ctrl, const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  // this kernel is the last reader of the node counts: leave them zeroed for
  // the next cycle
  for (long long i = gtid(); i < num_nodes; i += gstride()) {
    const uint32_t len = nodecnt[i];
    if (!len) continue;
    nodecnt[i] = 0;
    const U64x2 ex = pairs_ex[i];
    const long long d = (long long)(ex.a >> kPackShift);
    seg_node[d] = (int32_t)i;
    seg_start[d] = (long long)(ex.a & kPackLow);
    dense[i] = (int32_t)d;
    const U64x2 own = node_plan(nd, geo, i, len);
    plan[d] = u64x2(own.b >> 32, own.b & 0xFFFFFFFFull);
    plan_ex[d] = u64x2(ex.b >> 32, ex.b & 0xFFFFFFFFull);
  }
  if (gtid() == 0) {
    const U64x2 tot = ctrl->pack_tot;
    const unsigned long long K = tot.a >> kPackShift;
    ctrl->seg_tot = u64x2(K, tot.a & kPackLow);
    ctrl->acq_tot = u64x2(tot.b >> 32, tot.b & 0xFFFFFFFFull);
    seg_start[K] = (long long)(tot.a & kPackLow);
    ctrl->n_keys = (unsigned)K;
    // acquisition snapshot (ChunkPool.acquire, store.py:110-123): the free
    // stack pops first, then fresh payloads are cut 16-aligned from the arena
    ctrl->alloc_F = ctrl->free_count;
    ctrl->alloc_A = ctrl->allocated_total;
    ctrl->chunk_base = (ctrl->arena_off + 15ull) / 16ull * 16ull;
  }
}

__device__ __forceinline__ int acq_cid(const PoolCols &pool, const Ctrl *ctrl, long long a) {
  return a < ctrl->alloc_F ? pool.free_stack[ctrl->alloc_F - 1 - a] : (int)(ctrl->alloc_A + (a - ctrl->alloc_F));
}

// What the store needs per touched node, in one 32-byte record indexed by node
// id (written by k_alloc's node pass): its segment start in the sorted order, its
// first write-list entry and its stored count before this cycle.
struct SinkInfo {
  long long seg_start, wl_start, cnt, pad;
};

// Per touched node: link the new run after the old tail (Octree.append_chunk,
// octree.py:328-337) and put the partially filled tail at the head of the
// node's write list.
// The bulk acquisition's bookkeeping (every thread derives the same fresh
// count; OutOfArena at the first fresh payload past capacity, store.py:60-69)
// is done here too: thread 0 advances the arena / free-stack / pool counters.
__device__ __forceinline__ bool alloc_nodes_body(NodeCols nd, PoolCols pool, Geo geo,
                                                 const int32_t *__restrict__ seg_node,
                                                 const long long *__restrict__ seg_start,
                                                 const U64x2 *__restrict__ plan, const U64x2 *__restrict__ plan_ex,
                                                 long long *__restrict__ wlo, SinkInfo *__restrict__ sinfo,
                                                 Ctrl *ctrl, unsigned long long arena_cap) {
  if (ctrl->error) return false;
  {
    const long long M = (long long)ctrl->acq_tot.a;
    const long long F = ctrl->alloc_F, A = ctrl->alloc_A;
    const long long fresh = M > F ? M - F : 0;
    const unsigned long long end = ctrl->chunk_base + (unsigned long long)fresh * (unsigned long long)geo.C * 16ull;
    if (fresh > 0 && end > arena_cap) {
      if (gtid() == 0) set_error(ctrl, 1 /*LOD_E_OUT_OF_ARENA*/);
      return false;
    }
    if (gtid() == 0) {
      if (fresh > 0) ctrl->arena_off = end;
      ctrl->free_count = F - (M < F ? M : F);
      ctrl->allocated_total = A + fresh;
    }
  }
  const long long K = (long long)ctrl->n_keys;
  for (long long d = gtid(); d < K; d += gstride()) {
    const int n = seg_node[d];
    const long long len = seg_start[d + 1] - seg_start[d];
    const long long cnt = nd.count[n];
    const long long need = (long long)plan[d].a;
    const long long A0 = (long long)plan_ex[d].a, W0 = (long long)plan_ex[d].b;
    const int tail = nd.chunk_tail[n];
    sinfo[n] = SinkInfo{seg_start[d], W0, cnt, 0};
    if (cnt % geo.C) {
      wlo[W0] = pool.payload_off[tail];
      const long long ci = cnt / geo.C;  // tail chunk index in the node's list
      const long long rem = cnt + len - ci * geo.C;
      pool.occupied[tail] = (int)(rem < geo.C ? rem : geo.C);
    }
    if (need > 0) {
      const int first = acq_cid(pool, ctrl, A0), last = acq_cid(pool, ctrl, A0 + need - 1);
      if (tail != LOD_NO_CHUNK) pool.next[tail] = first;
      else nd.chunk_head[n] = first;
      nd.chunk_tail[n] = last;
      nd.chunk_count[n] += (int)need;
    }
  }
  return true;
}

// Per acquisition: payload offset for fresh chunks, in-run links, owner,
// position and final occupancy, write-list slot.
__device__ __forceinline__ void alloc_chunks_body(NodeCols nd, PoolCols pool, Geo geo,
                                                  const int32_t *__restrict__ seg_node,
                                                  const long long *__restrict__ seg_start,
                                                  const U64x2 *__restrict__ plan, const U64x2 *__restrict__ plan_ex,
                                                  long long *__restrict__ wlo, const Ctrl *ctrl) {
  const long long M = (long long)ctrl->acq_tot.a;
  const long long K = (long long)ctrl->n_keys;
  for (long long a = gtid(); a < M; a += gstride()) {
    // segment d: last d with plan_ex[d].a <= a
    long long lo = 0, hi = K - 1;
    while (lo < hi) {
      long long mid = (lo + hi + 1) >> 1;
      if ((long long)plan_ex[mid].a <= a) lo = mid;
      else hi = mid - 1;
    }
    const long long d = lo;
    const int n = seg_node[d];
    const long long need = (long long)plan[d].a;
    const long long t = a - (long long)plan_ex[d].a;
    const long long cnt = nd.count[n];
    const long long len = seg_start[d + 1] - seg_start[d];
    const int cid = acq_cid(pool, ctrl, a);
    long long poff;
    if (a >= ctrl->alloc_F) {
      poff = (long long)(ctrl->chunk_base + (unsigned long long)(a - ctrl->alloc_F) * (unsigned long long)geo.C * 16ull);
      pool.payload_off[cid] = poff;
    } else {
      poff = pool.payload_off[cid];
    }
    pool.next[cid] = (t + 1 < need) ? acq_cid(pool, ctrl, a + 1) : LOD_NO_CHUNK;
    pool.owner[cid] = n;
    const long long ci = ceil_div(cnt, geo.C) + t;
    pool.cidx[cid] = (int)ci;
    const long long rem = cnt + len - ci * geo.C;
    pool.occupied[cid] = (int)(rem < geo.C ? rem : geo.C);
    const long long partial = (long long)plan[d].b - need;
    wlo[(long long)plan_ex[d].b + partial + t] = poff;  // the store writes by payload offset
  }
}

// Both allocation passes in one launch: the node pass (links, tails, the
// counters) and the acquisition pass only share read-only snapshots
// (k_seg_list's alloc_F / alloc_A / chunk_base, the plans), and an
// OutOfArena stops every thread before either writes.
__global__ void k_alloc(NodeCols nd, PoolCols pool, Geo geo, const int32_t *__restrict__ seg_node,
                        const long long *__restrict__ seg_start, const U64x2 *__restrict__ plan,
                        const U64x2 *__restrict__ plan_ex, long long *__restrict__ wlo, SinkInfo *__restrict__ sinfo,
                        Ctrl *ctrl, unsigned long long arena_cap, const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  if (!alloc_nodes_body(nd, pool, geo, seg_node, seg_start, plan, plan_ex, wlo, sinfo, ctrl, arena_cap)) return;
  alloc_chunks_body(nd, pool, geo, seg_node, seg_start, plan, plan_ex, wlo, ctrl);
}

// store_points / store_voxels (_kernels.py:155-250): sorted position p of a
// node's segment is its slot count[node] + rank; records are 16-byte
// (f32 x,y,z | u32 rgba, store.py:14-16); voxel centres are
// bmin + (c + 0.5) * (size_by_level[level] / g) in f64, then rounded to f32.
// Used as the sink of the sort's last radix pass (the allocation runs before
// the sort: it needs only the per-node counts), so sorted keys / item ids are
// never written back; k_store is the same body over materialised arrays.
struct StoreSink {
  NodeCols nd;
  PoolCols pool;
  Geo geo;
  uint8_t *arena;
  const SinkInfo *sinfo;
  const long long *wlo;
  long long n_all;
  PointSrc src;
  const uint4 *backlog;  // new voxels in backlog order: {node, cell, rgba, winner index}
  const Ctrl *ctrl;
  // p: the item's position in the node-sorted order (LSD sort)
  __device__ __forceinline__ void operator()(uint32_t p, uint32_t key, uint32_t item) const {
    if (ctrl->error) return;
    store_rank((long long)p - sinfo[(int)key].seg_start, key, item);
  }
  // rank: the item's rank among this cycle's items of its node
  __device__ __forceinline__ void store_rank(long long rank, uint32_t key, uint32_t item) const {
    const int n = (int)key;
    const SinkInfo si = sinfo[n];
    const long long cnt = si.cnt;
    const long long slot = cnt + rank;
    const long long rel = slot / geo.C - cnt / geo.C;
    const long long poff = wlo[si.wl_start + rel];
    const long long off = slot % geo.C;
    const long long i = item;
    float4 rec;
    if (i < n_all) {
      rec = src.record(i);
    } else {
      const long long b = i - n_all;
      const uint4 bl = backlog[b];
      const long long cell = bl.y;
      const long long g = geo.g;
      const long long cx = cell % g, cy = (cell / g) % g, cz = cell / (g * g);
      const double step = geo.size_by_level[nd.level[n]] / (double)g;
      const double x = nd.bmin[3 * n] + ((double)cx + 0.5) * step;
      const double y = nd.bmin[3 * n + 1] + ((double)cy + 0.5) * step;
      const double z = nd.bmin[3 * n + 2] + ((double)cz + 0.5) * step;
      rec = make_float4(__double2float_rn(x), __double2float_rn(y), __double2float_rn(z), __uint_as_float(bl.z));
    }
    float4 *dst = reinterpret_cast<float4 *>(arena + poff) + off;
    *dst = rec;
  }
};

// Direct placement (radix.cuh k_rank_prep / k_tile_colscan): every item in
// input order, rank = its node's items in earlier tiles + its in-tile rank.
// nowait: as k_onesweep's (launched behind k_publish's early release).
__global__ void k_store_direct(StoreSink sink, const uint32_t *__restrict__ keys, const uint16_t *__restrict__ rank,
                               const uint32_t *__restrict__ mat, long long ms, int tsh,
                               const long long *__restrict__ n_items_dev, const int *guard, int nowait) {
  if (!nowait) lod::pdl_wait();
  if (guard && *guard) return;
  if (sink.ctrl->error) return;
  const long long n_items = *n_items_dev;
  for (long long i = gtid(); i < n_items; i += gstride()) {
    const uint32_t key = keys[i];
    const long long t = i >> tsh;
    sink.store_rank((long long)mat[t * ms + key] + rank[i], key, (uint32_t)i);
  }
}

__global__ void k_store(StoreSink sink, const uint32_t *__restrict__ skeys, const uint32_t *__restrict__ svals,
                        const long long *__restrict__ n_items_dev, const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  const long long n_items = *n_items_dev;
  for (long long p = gtid(); p < n_items; p += gstride()) sink((uint32_t)p, skeys[p], svals[p]);
}

// clear_marks (_kernels.py:280-287) + count advance: pending drains into count.
// + the chunk directory of every node that got chunks: one warp per touched
// node, lane 0 relocates a full region (doubling), the warp copies the old
// entries and records the new chunk ids (a large inner node's region holds
// thousands of entries: a thread per node made its copy the pass's tail).
__global__ void k_epilogue(NodeCols nd, PoolCols pool, const int32_t *__restrict__ seg_node,
                           const long long *__restrict__ seg_start, const U64x2 *__restrict__ plan,
                           const U64x2 *__restrict__ plan_ex, Ctrl *ctrl, uint32_t *__restrict__ ghist,
                           const int *guard, int geo_fresh) { lod::pdl_wait();
  if (guard && *guard) return;
  // the sort is the last reader of the digit totals: zeroed for the next cycle
  for (long long i = gtid(); i < kMaxPassesHist; i += gstride()) ghist[i] = 0;
  if (ctrl->error) return;
  const long long K = (long long)ctrl->n_keys;
  const int lane = threadIdx.x & 31;
  for (long long d = gtid() >> 5; d < K; d += gstride() >> 5) {
    const int n = seg_node[d];
    const long long need = (long long)plan[d].a;
    long long off = 0, off_old = 0, cc0 = 0;
    int moved = 0;
    if (lane == 0) {
      nd.count[n] += seg_start[d + 1] - seg_start[d];
      nd.pending[n] = 0;
      nd.final_[n] = 0;
      // a node split this cycle got voxels (every re-descending point claims
      // a cell of its all-clear grid), so it is a segment: its grid is no
      // longer fresh
      if (geo_fresh && nd.desc[n].y < 0) nd.desc[n].y &= ~kFresh;
      if (need > 0) {
        const long long cc1 = nd.chunk_count[n];
        cc0 = cc1 - need;
        off = off_old = nd.dir_off[n];
        if (cc1 > (long long)nd.dir_cap[n]) {
          const long long cap = cc1 * 2 > 4 ? cc1 * 2 : 4;
          off = dir_claim(pool, &ctrl->dir_top, cap);
          if (off >= 0) {
            nd.dir_off[n] = off;
            nd.dir_cap[n] = (int32_t)cap;
            moved = 1;
          } else {
            moved = -1;  // no room: this node's entries are written by the rebuild
          }
        }
      }
    }
    if (!__shfl_sync(0xffffffffu, (int)(need > 0), 0)) continue;
    off = __shfl_sync(0xffffffffu, off, 0);
    off_old = __shfl_sync(0xffffffffu, off_old, 0);
    cc0 = __shfl_sync(0xffffffffu, cc0, 0);
    moved = __shfl_sync(0xffffffffu, moved, 0);
    if (moved < 0) continue;
    if (moved)
      for (long long i = lane; i < cc0; i += 32) pool.cdir[off + i] = pool.cdir[off_old + i];
    const long long A0 = (long long)plan_ex[d].a;
    for (long long t = lane; t < need; t += 32) pool.cdir[off + cc0 + t] = acq_cid(pool, ctrl, A0 + t);
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&ctrl->t_end, gtimer_ns());  // the cycle's device end
}

// ---------------------------------------------------------------- BatchDelta

// collect_delta (update.py:333-355), from the cycle's segment table before the
// epilogue advances the counts: every touched segment is either an inner node
// (its items are new voxels, in claim order) or a leaf (new points).  One CTA
// scans the segments in ascending node id into the voxel-group list (node,
// offset into the delta voxel arrays, count) and the point-group list (node,
// pre-store count, count); vbase[d] is segment d's delta voxel offset.
constexpr int kDeltaBlock = 1024;
__global__ void __launch_bounds__(kDeltaBlock)
    k_delta_segs(NodeCols nd, const int32_t *__restrict__ seg_node, const long long *__restrict__ seg_start,
                 int32_t *__restrict__ vnode, long long *__restrict__ vstart, long long *__restrict__ vcount,
                 int32_t *__restrict__ pnode, long long *__restrict__ pstart, long long *__restrict__ pcount,
                 long long *__restrict__ vbase, Ctrl *ctrl, const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  __shared__ U64x2 sh[kDeltaBlock / 32 + 1];
  if (ctrl->error) return;
  const long long K = (long long)ctrl->n_keys;
  U64x2 carry = u64x2(0, 0);
  for (long long base = 0; base < K; base += kDeltaBlock) {
    const long long d = base + threadIdx.x;
    int n = -1;
    bool inner = false;
    long long len = 0;
    if (d < K) {
      n = seg_node[d];
      inner = nd.inner[n] != 0;
      len = seg_start[d + 1] - seg_start[d];
    }
    // a: group counters (voxel groups low word, point groups high word); b: voxels
    const U64x2 v = u64x2(d < K ? (inner ? 1ull : (1ull << 32)) : 0ull, inner ? (unsigned long long)len : 0ull);
    U64x2 tot;
    U64x2 ex = block_exclusive_scan<U64x2, kDeltaBlock>(v, sh, tot);
    ex = ex + carry;
    if (d < K) {
      if (inner) {
        const long long g = (long long)(ex.a & 0xFFFFFFFFull);
        vnode[g] = n;
        vstart[g] = (long long)ex.b;
        vcount[g] = len;
        vbase[d] = (long long)ex.b;
      } else {
        const long long g = (long long)(ex.a >> 32);
        pnode[g] = n;
        pstart[g] = nd.count[n];
        pcount[g] = len;
      }
    }
    carry = carry + tot;
  }
  if (threadIdx.x == 0) {
    ctrl->d_nvg = (unsigned)(carry.a & 0xFFFFFFFFull);
    ctrl->d_npg = (unsigned)(carry.a >> 32);
  }
}

// Delta voxel payload: every voxel item of the sorted order (node-major,
// ascending claim index inside a node = the reference's stable argsort of the
// backlog by node) copies its (cell, rgba) to its group's slot.
__global__ void k_delta_vox(const uint32_t *__restrict__ skeys, const uint32_t *__restrict__ svals,
                            const int32_t *__restrict__ dense, const long long *__restrict__ seg_start,
                            const long long *__restrict__ vbase, long long n_all,
                            const uint4 *__restrict__ backlog,
                            uint32_t *__restrict__ dcell, uint32_t *__restrict__ drgba, const Ctrl *ctrl,
                            const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  if (ctrl->error) return;
  const long long n_items = ctrl->n_items;
  for (long long p = gtid(); p < n_items; p += gstride()) {
    const long long i = svals[p];
    if (i < n_all) continue;
    const long long d = dense[skeys[p]];
    const long long pos = vbase[d] + (p - seg_start[d]);
    const uint4 bl = backlog[i - n_all];
    dcell[pos] = bl.y;
    drgba[pos] = bl.z;
  }
}

// Safety net after a fatal error: pending/final of every node back to zero.
__global__ void k_clear_marks_all(NodeCols nd, int32_t *srank, long long n, int geo_fresh) { lod::pdl_wait();
  for (long long i = gtid(); i < n; i += gstride()) {
    nd.pending[i] = 0;
    nd.final_[i] = 0;
    srank[i] = -1;
    if (geo_fresh && nd.desc[i].y < 0) nd.desc[i].y &= ~kFresh;
  }
}

}  // namespace lod
