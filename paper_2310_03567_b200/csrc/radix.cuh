// radix.cuh -- stable multisplit of an ordered item list by node id.
//
// The reference appends records to each node in global ingestion order
// (store_points/store_voxels, _kernels.py:155-250: slot = count[node]++ in
// all-array / backlog order).  On the GPU that order is recovered with an LSD
// radix sort over node ids, 8-bit digits, in the onesweep form: one upfront
// pass builds the key array and the per-node item counts (which define the
// node segments and, summed by digit, every pass's digit totals), then ONE
// kernel per digit pass ranks its tile, publishes its per-digit counts and
// resolves its global offsets with a decoupled look-back over earlier tiles.
// Stability inside a tile comes from warp-ordered rounds: each warp owns a
// contiguous 512-item range, ranks lanes with __match_any_sync, and keeps a
// per-warp digit histogram in shared memory; warps are combined in order.
// The tile is then reordered by digit in shared memory so the global writes
// go out as contiguous digit runs.
//
// On trees of up to 24,576 nodes the update does not sort at all: the direct
// placement below (k_rank_prep / k_tile_colscan / k_store_direct) gives every
// item its rank within its node from per-tile node counts, and the LSD passes
// serve the larger trees, the burst resolve's win list and delta emission.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lod_common.cuh"
#include "scan.cuh"

namespace lod {

constexpr int kRadixBits = 8;
constexpr int kRadixDigits = 1 << kRadixBits;
constexpr int kRadixBlock = 256;  // 8 warps
constexpr int kRadixWarps = kRadixBlock / 32;
#ifndef LOD_RADIX_ROUNDS
#define LOD_RADIX_ROUNDS 8  // measured: 8 > 6, 12 > 4 (update bench, same box)
#endif
#ifndef LOD_RADIX_MINB
#define LOD_RADIX_MINB 5  // same-box A/B, driver range: 5 (2385-2392 Mpts/s) > 6 (2376) > 4 (2352-2366) > 3 > 8
#endif
constexpr int kRadixRounds = LOD_RADIX_ROUNDS;  // per warp: 8 rounds x 32 lanes (2048-item tile, ~27 KB smem)
constexpr int kRadixTile = kRadixBlock * kRadixRounds;
constexpr int kMaxPasses = 4;
// Per-CTA node histograms live in dynamic shared memory as 16-bit counters
// (two per word) for trees of up to kNodeHistSmemMax nodes (192 KB); a CTA
// never counts more than 65535 items of one node (checked by the launcher).
constexpr long long kNodeHistSmemMax = 98304;

// look-back words: [31:30] status (0 empty, 1 aggregate, 2 inclusive prefix), [29:0] count
constexpr uint32_t kLbAgg = 1u << 30, kLbPre = 2u << 30, kLbMask = (1u << 30) - 1;

// Items: points j in [0, n_all) keyed by their leaf, then backlog entries keyed
// by their node.  Writes the key array and the per-node item counts (= each
// node's new samples this cycle; per-CTA shared-memory counters when they fit).
// 4 items per thread per round (independent loads in flight), 4 CTAs per SM.
constexpr int kPrepItems = 4;
constexpr int kPrepBlocksPerSM = 4;
#ifndef LOD_PREP_BPS
#define LOD_PREP_BPS 2  // CTAs per SM with shared-memory node histograms (capped by what fits)
#endif
static __global__ void __launch_bounds__(kRadixBlock, kPrepBlocksPerSM)
    k_radix_prep(NodeOf node_of, long long n_all, const uint4 *__restrict__ backlog,
                 long long nc_words, uint32_t *__restrict__ keys, uint32_t *__restrict__ nodecnt,
                 uint32_t *__restrict__ lb0, long long lb_words, const unsigned long long *__restrict__ n_v_dev, long long *__restrict__ n_items_out,
                 const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  extern __shared__ uint32_t nc2[];  // nc_words words: node 2w in the low half, 2w+1 in the high half
  const long long n_v = (long long)*n_v_dev;  // new voxels (device count: launches may precede the host's view)
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_items_out = n_all + n_v;
  for (long long i = gtid(); i < lb_words; i += gstride()) lb0[i] = 0;  // look-back words of pass 0
  const bool smem_nodes = nc_words > 0;
  for (long long w = threadIdx.x; w < nc_words; w += kRadixBlock) nc2[w] = 0;
  __syncthreads();
  const long long n = n_all + n_v;
  constexpr long long kSpan = (long long)kRadixBlock * kPrepItems;
  for (long long i0 = (long long)blockIdx.x * kSpan; i0 < n; i0 += (long long)gridDim.x * kSpan) {
    uint32_t key[kPrepItems];
#pragma unroll
    for (int q = 0; q < kPrepItems; ++q) {
      const long long i = i0 + q * kRadixBlock + threadIdx.x;
      key[q] = 0xFFFFFFFFu;
      if (i < n) key[q] = (uint32_t)(i < n_all ? node_of[i] : __ldg(&backlog[i - n_all].x));
    }
#pragma unroll
    for (int q = 0; q < kPrepItems; ++q) {
      const long long i = i0 + q * kRadixBlock + threadIdx.x;
      const bool ok = i < n;
      if (ok) keys[i] = key[q];
      if (smem_nodes) {  // shared-memory counters: the atomic units resolve same-node lanes
        // (per-warp MATCH.ANY aggregation first was 1.7 % slower end to end);
        // a warp whose 32 items share one node (locality-ordered input: 32
        // serialised atomics on one word) adds them with one
        const uint32_t k0 = __shfl_sync(0xffffffffu, key[q], 0);
        if (__all_sync(0xffffffffu, ok && key[q] == k0)) {
          if (lane_id() == 0) atomicAdd(&nc2[k0 >> 1], 32u << (16 * (k0 & 1)));
        } else if (ok) {
          atomicAdd(&nc2[key[q] >> 1], 1u << (16 * (key[q] & 1)));
        }
        continue;
      }
      const unsigned act = __ballot_sync(0xffffffffu, ok);
      if (ok) {  // global counters: hot nodes are aggregated per warp first
        const unsigned peers = __match_any_sync(act, key[q]);
        if (lane_id() == (unsigned)(__ffs(peers) - 1)) atomicAdd(&nodecnt[key[q]], (uint32_t)__popc(peers));
      }
    }
  }
  __syncthreads();
  for (long long w = threadIdx.x; w < nc_words; w += kRadixBlock) {
    const uint32_t v = nc2[w];
    if (v & 0xFFFFu) atomicAdd(nodecnt + 2 * w, v & 0xFFFFu);
    if (v >> 16) atomicAdd(nodecnt + 2 * w + 1, v >> 16);
  }
}

// ---- direct placement (one pass instead of the LSD passes) -------------------
// The store only needs every item's rank among the earlier items of its node
// (slot order = all-array / backlog order, _kernels.py:155-250).  Cut the item
// list into tiles of 1 << tsh items, one warp per tile: the warp walks its
// tile in order and ranks each item against the tile's earlier items of the
// same node (per-warp u16 counters in shared memory, MATCH.ANY per 32 items),
// then writes the tile's per-node counts as one dense row of a tiles x nodes
// matrix.  A column scan over that matrix (k_tile_colscan) turns each count
// into the node's items in earlier tiles; rank = that + the in-tile rank.
// Chosen when the matrix is small (a few thousand nodes: L2-resident);
// otherwise the LSD multisplit runs.
#ifndef LOD_DIR_ROWBLOCK
#define LOD_DIR_ROWBLOCK 32  // A/B, driver range: 16 / 32 / 64 all 2628-2633 Mpts/s
#endif
constexpr int kDirRowBlock = LOD_DIR_ROWBLOCK;  // tiles per row block of the column scan
constexpr int kDirScanBlock = 256;  // node columns per column-scan CTA
#ifndef LOD_COLSCAN_KEEP
#define LOD_COLSCAN_KEEP 1  // counts kept in registers between the two sweeps (A/B: 2607-2610 vs 2581-2596 re-read)
#endif

// Keys (node ids), in-tile ranks and the tile's node-count row.  Also zeroes
// the column scan's look-back words + ticket (lb_words) and publishes the
// item count like k_radix_prep.  Dynamic smem: W * nn_pad u16 counters.
template <int W>
static __global__ void __launch_bounds__(32 * W)
    k_rank_prep(NodeOf node_of, long long n_all, const uint4 *__restrict__ backlog, long long nn, long long nn_pad,
                uint32_t *__restrict__ keys, uint16_t *__restrict__ rank, uint32_t *__restrict__ mat,
                uint32_t *__restrict__ lb, long long lb_words, const unsigned long long *__restrict__ n_v_dev,
                long long *__restrict__ n_items_out, int tsh, const int *guard) {
  lod::pdl_wait();
  if (guard && *guard) return;
  extern __shared__ __align__(16) uint16_t dcnt[];  // nn_pad (a multiple of 8) per warp
  const long long n_v = (long long)*n_v_dev;
  const long long n = n_all + n_v;
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_items_out = n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < lb_words;
       i += (long long)gridDim.x * blockDim.x)
    lb[i] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long tile = (long long)blockIdx.x * W + warp;
  const long long i0 = tile << tsh;
  if (i0 >= n) return;  // warp-uniform
  uint16_t *cnt = dcnt + (long long)warp * nn_pad;
  for (long long k = lane; k < nn_pad / 8; k += 32) reinterpret_cast<uint4 *>(cnt)[k] = make_uint4(0, 0, 0, 0);
  __syncwarp();
  const unsigned lt = lanemask_lt();
  constexpr int kAhead = 8;  // rounds of keys loaded ahead
  for (int r0 = 0; r0 < (1 << tsh) / 32; r0 += kAhead) {
    if (i0 + (long long)r0 * 32 >= n) break;  // warp-uniform
    uint32_t key[kAhead];
#pragma unroll
    for (int q = 0; q < kAhead; ++q) {
      const long long i = i0 + (long long)(r0 + q) * 32 + lane;
      key[q] = 0xFFFFFFFFu;
      if (i < n) key[q] = (uint32_t)(i < n_all ? node_of[i] : __ldg(&backlog[i - n_all].x));
    }
    // the rounds' lane groups first (independent MATCHes), then the counter
    // chain; a group's leader is its lowest lane (no lanes below it)
    unsigned peers[kAhead];
#pragma unroll
    for (int q = 0; q < kAhead; ++q) peers[q] = __match_any_sync(0xffffffffu, key[q]);
#pragma unroll
    for (int q = 0; q < kAhead; ++q) {
      const long long i = i0 + (long long)(r0 + q) * 32 + lane;
      const bool ok = i < n;
      const uint32_t below = __popc(peers[q] & lt);
      const uint32_t b = ok ? cnt[key[q]] : 0u;
      if (ok) {
        keys[i] = key[q];
        rank[i] = (uint16_t)(b + below);
      }
      __syncwarp();
      if (ok && below == 0) cnt[key[q]] = (uint16_t)(b + __popc(peers[q]));
      __syncwarp();
    }
  }
  // the dense row (stride nn_pad), 8 counters per lane step
  uint4 *row = reinterpret_cast<uint4 *>(mat + tile * nn_pad);
  for (long long k = lane; k < nn_pad / 8; k += 32) {
    const uint4 v = reinterpret_cast<const uint4 *>(cnt)[k];
    row[2 * k] = make_uint4(v.x & 0xFFFFu, v.x >> 16, v.y & 0xFFFFu, v.y >> 16);
    row[2 * k + 1] = make_uint4(v.z & 0xFFFFu, v.z >> 16, v.w & 0xFFFFu, v.w >> 16);
  }
}

// Column scan of the tiles x nodes count matrix (row stride ms), in place: entry (t, k)
// becomes node k's items in tiles < t; the node totals go to nodecnt.  One CTA
// per (row block of kDirRowBlock tiles, kDirScanBlock node columns), taken in
// ticket order; row blocks chain per column with a decoupled look-back
// (status bits as in the onesweep).  lb: rb_cap * nn words + the ticket.
// The last row block also makes each node's plan record (k_radix_ghist's
// other job; the digit totals are not needed here), scans them (the segment
// scan the LSD path runs as its own launch) and unpacks them (Seg: the
// per-node and total work of k_seg_list).
template <class Seg>
static __global__ void __launch_bounds__(kDirScanBlock)
    k_tile_colscan(uint32_t *__restrict__ mat, long long nn, long long ms, long long ncb, long long rb_cap,
                   const long long *__restrict__ n_items_dev, uint32_t *lb, Seg seg, U64x2 *pscan, int tsh,
                   const int *guard) {
  lod::pdl_wait();
  if (guard && *guard) return;
  __shared__ uint32_t s_ticket;
  if (threadIdx.x == 0) s_ticket = atomicAdd(lb + rb_cap * nn, 1u);
  __syncthreads();
  const long long n = *n_items_dev;
  const long long ntiles = (n + (1LL << tsh) - 1) >> tsh;
  const long long nrb = (ntiles + kDirRowBlock - 1) / kDirRowBlock;
  const long long last_rb = nrb > 0 ? nrb - 1 : 0;  // no items: row block 0 writes the zero plans
  const long long rb = s_ticket / ncb, cb = s_ticket % ncb;
  if (rb > last_rb) return;  // CTA-uniform
  const long long k = cb * kDirScanBlock + threadIdx.x;
  const bool live = k < nn;
  uint32_t node_total = 0;
  if (nrb > 0 && live) {
    const long long t0 = rb * kDirRowBlock;
    const int nt = (int)min((long long)kDirRowBlock, ntiles - t0);
#if LOD_COLSCAN_KEEP
    uint32_t c[kDirRowBlock];
#endif
    uint32_t sum = 0;
#pragma unroll
    for (int q = 0; q < kDirRowBlock; ++q) {
      const uint32_t v = q < nt ? mat[(t0 + q) * ms + k] : 0u;
#if LOD_COLSCAN_KEEP
      c[q] = v;
#endif
      sum += v;
    }
    uint32_t *mine = lb + rb * nn + k;
    uint32_t excl = 0;
    if (rb == 0) {
      atomicExch(mine, kLbPre | sum);
    } else {
      atomicExch(mine, kLbAgg | sum);
      // 4 predecessors per round trip; an unpublished one ends the round
      long long p = rb - 1;
      for (bool done = false; !done;) {
        uint32_t v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = p - q >= 0 ? *((volatile uint32_t *)(lb + (p - q) * nn + k)) : (2u << 30);  // kLbPre
        int q = 0;
        for (; q < 4; ++q) {
          if ((v[q] & ~kLbMask) == 0) break;
          excl += v[q] & kLbMask;
          if ((v[q] & ~kLbMask) == kLbPre) {
            done = true;
            break;
          }
        }
        p -= q;
      }
      atomicExch(mine, kLbPre | (excl + sum));
    }
    node_total = excl + sum;
    uint32_t run = excl;
#if LOD_COLSCAN_KEEP
#pragma unroll
    for (int q = 0; q < kDirRowBlock; ++q) {
      if (q < nt) mat[(t0 + q) * ms + k] = run;
      run += c[q];
    }
#else
    for (int q = 0; q < nt; ++q) {  // second read of the block's entries (L1 / L2)
      const uint32_t v = mat[(t0 + q) * ms + k];
      mat[(t0 + q) * ms + k] = run;
      run += v;
    }
#endif
  }
  if (rb != last_rb) return;  // CTA-uniform
  // the last row block: node totals, plan records and their exclusive scan in
  // node order (the segment scan), chained over the column blocks
  // (flags after the ticket word: 1 aggregate, 2 inclusive prefix)
  const U64x2 v = live ? seg.plan_of(k, node_total) : u64x2(0, 0);
  __shared__ U64x2 sh64[kDirScanBlock / 32 + 1];
  __shared__ U64x2 s_excl;
  U64x2 btot;
  const U64x2 ex = block_exclusive_scan<U64x2, kDirScanBlock>(v, sh64, btot);
  if (threadIdx.x == 0) {
    uint32_t *flag = lb + rb_cap * nn + 1;
    U64x2 *agg = pscan, *inc = pscan + ncb;
    U64x2 excl = u64x2(0, 0);
    if (cb > 0) {
      agg[cb] = btot;
      __threadfence();
      atomicExch(flag + cb, 1u);
      for (long long p = cb - 1;;) {
        const uint32_t f = *((volatile uint32_t *)(flag + p));
        if (f == 0) continue;
        __threadfence();
        if (f == 2u) {
          excl = excl + ld_cg(inc + p);
          break;
        }
        excl = excl + ld_cg(agg + p);
        --p;
      }
    }
    inc[cb] = excl + btot;
    __threadfence();
    atomicExch(flag + cb, 2u);
    s_excl = excl;
    if (cb == ncb - 1) seg.total(excl + btot);
  }
  __syncthreads();
  if (live) seg.node(k, node_total, s_excl + ex, v);  // k_seg_list's per-node work
}

// Digit totals of every pass from the per-node counts (keys are node ids).
// Also writes each node's plan record for the segment scan (plan_of(n, count)).
template <class PlanOf>
static __global__ void k_radix_ghist(const uint32_t *__restrict__ nodecnt, long long num_nodes, int passes,
                              uint32_t *__restrict__ ghist, U64x2 *__restrict__ pairs, PlanOf plan_of,
                              const int *guard) { lod::pdl_wait();
  if (guard && *guard) return;
  __shared__ uint32_t h[kMaxPasses * kRadixDigits];
  for (int i = threadIdx.x; i < kMaxPasses * kRadixDigits; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (long long n = gtid(); n < num_nodes; n += gstride()) {
    const uint32_t c = nodecnt[n];
    pairs[n] = plan_of(n, c);
    if (c)
      for (int p = 0; p < passes; ++p) atomicAdd(&h[p * kRadixDigits + ((n >> (p * kRadixBits)) & 0xFF)], c);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadixDigits; i += blockDim.x)
    if (h[i]) atomicAdd(ghist + i, h[i]);
}

// Where a pass writes its sorted items: the next pass's key / value arrays, or
// (the last pass of the update's sort) straight into the consumer (Sink).
struct KVSink {
  uint32_t *keys_out, *vals_out;
  __device__ __forceinline__ void operator()(uint32_t pos, uint32_t key, uint32_t val) const {
    keys_out[pos] = key;
    vals_out[pos] = val;
  }
};

// One LSD pass.  vals_in == nullptr means the identity permutation.
// `lb` holds ntiles * 256 look-back words + 1 tile ticket, zeroed before the pass.
template <class Sink>
static __global__ void __launch_bounds__(kRadixBlock, LOD_RADIX_MINB)
    k_onesweep(const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in, long long n_max,
               const long long *__restrict__ n_dev, int shift, const uint32_t *__restrict__ ghist_pass, uint32_t *lb,
               long long ntiles, Sink sink, uint32_t *lb_next, const int *guard, int nowait) {
  // nowait: launched behind a k_publish that released its dependents after
  // its own wait -- everything this pass reads was complete before that
  if (!nowait) lod::pdl_wait();
  if (guard && *guard) return;
  // item count: n_max, or the device count when launched for an upper bound
  // (tiles past it take their ticket and leave)
  const long long n = n_dev ? *n_dev : n_max;
  // zero the next pass's look-back words (one per thread, + the ticket)
  if (lb_next) {
    lb_next[(long long)blockIdx.x * kRadixDigits + threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) lb_next[ntiles * kRadixDigits] = 0;
  }
  __shared__ uint32_t wh[kRadixWarps][kRadixDigits];  // per-warp digit counts -> warp offsets
  __shared__ uint32_t dstart[kRadixDigits];           // tile-local digit start
  __shared__ uint32_t gbase[kRadixDigits];            // global position of the tile's digit run
  __shared__ alignas(16) uint32_t sk[kRadixTile];
  __shared__ alignas(16) uint32_t sv[kRadixTile];
  __shared__ uint16_t sloc[kRadixTile];
  __shared__ uint32_t sh[kRadixBlock / 32 + 1];
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_bar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_tile = atomicAdd(lb + ntiles * kRadixDigits, 1u);  // launch-order tile ids
    mbar_init(&s_bar, 1);
  }
  for (int d = lane; d < kRadixDigits; d += 32) wh[warp][d] = 0;
  __syncthreads();
  const long long tile = s_tile;
  const long long t0 = tile * kRadixTile;
  if (t0 >= n) return;
  const int wofs = warp * (32 * kRadixRounds);
  const unsigned lt = lanemask_lt();
  const long long valid = min((long long)kRadixTile, n - t0);
  // 0) stage the tile (keys, and item ids unless identity) in shared memory with
  //    TMA bulk copies; the ragged tail (< 4 items) is loaded directly
  const int nbulk = (int)(valid & ~3ll);
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&s_bar, (unsigned)nbulk * 4u * (vals_in ? 2u : 1u));
    if (nbulk) {
      bulk_g2s(sk, keys_in + t0, (unsigned)nbulk * 4u, &s_bar);
      if (vals_in) bulk_g2s(sv, vals_in + t0, (unsigned)nbulk * 4u, &s_bar);
    }
  }
  if (threadIdx.x < valid - nbulk) {
    sk[nbulk + threadIdx.x] = __ldg(keys_in + t0 + nbulk + threadIdx.x);
    if (vals_in) sv[nbulk + threadIdx.x] = __ldg(vals_in + t0 + nbulk + threadIdx.x);
  }
  mbar_wait(&s_bar, 0);
  __syncthreads();
  // 1) warp-ordered ranking over the staged tile (input order)
  unsigned peers[kRadixRounds];  // the rounds' lane groups first (independent MATCHes)
  int dig[kRadixRounds];
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const int li = wofs + r * 32 + lane;
    dig[r] = li < valid ? (int)((sk[li] >> shift) & (kRadixDigits - 1)) : kRadixDigits + 1;
    peers[r] = __match_any_sync(0xffffffffu, dig[r]);
  }
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const int li = wofs + r * 32 + lane;
    const bool ok = li < valid;
    const int d = dig[r];
    const uint32_t below = __popc(peers[r] & lt);
    const uint32_t b = ok ? wh[warp][d] : 0u;
    if (!vals_in) sv[li] = (uint32_t)(t0 + li);
    sloc[li] = (uint16_t)(b + below);
    __syncwarp();
    if (ok && below == 0) wh[warp][d] = b + __popc(peers[r]);
    __syncwarp();
  }
  __syncthreads();
  // 2) per digit: warp offsets, tile-local digit start, decoupled look-back
  {
    const int d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      const uint32_t c = wh[w][d];
      wh[w][d] = run;
      run += c;
    }
    uint32_t tot;
    dstart[d] = block_exclusive_scan<uint32_t, kRadixBlock>(run, sh, tot);
    uint32_t *mine = lb + tile * kRadixDigits + d;
    uint32_t excl = 0;
    if (tile == 0) {
      atomicExch(mine, kLbPre | run);
    } else {
      atomicExch(mine, kLbAgg | run);
      // look back 8 predecessors per round trip (independent loads), consuming
      // aggregates in order until an inclusive prefix; an unpublished tile
      // ends the round and is re-read in the next one
      constexpr int kLook = 8;
      long long t = tile - 1;
      bool done = false;
      while (!done) {
        uint32_t v[kLook];
#pragma unroll
        for (int q = 0; q < kLook; ++q)
          v[q] = t - q >= 0 ? *((volatile uint32_t *)(lb + (t - q) * kRadixDigits + d)) : (2u << 30);  // kLbPre
        int q = 0;
        for (; q < kLook; ++q) {
          if ((v[q] & ~kLbMask) == 0) break;  // predecessor not published yet
          excl += v[q] & kLbMask;
          if ((v[q] & ~kLbMask) == kLbPre) {
            done = true;
            break;
          }
        }
        t -= q;
      }
      atomicExch(mine, kLbPre | (excl + run));
    }
    // digit base of this pass (exclusive scan of the totals) + earlier tiles
    const uint32_t gex = block_exclusive_scan<uint32_t, kRadixBlock>(ghist_pass[d], sh, tot);
    gbase[d] = gex + excl;
  }
  __syncthreads();
  // 3) reorder the tile by digit in shared memory
  uint32_t rk[kRadixRounds], rv[kRadixRounds], rp[kRadixRounds];
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const int li = wofs + r * 32 + lane;
    const uint32_t key = sk[li];
    const int d = (int)((key >> shift) & (kRadixDigits - 1));
    rk[r] = key;
    rv[r] = sv[li];
    rp[r] = dstart[d] + wh[warp][d] + sloc[li];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    if ((long long)(wofs + r * 32 + lane) < valid) {
      sk[rp[r]] = rk[r];
      sv[rp[r]] = rv[r];
    }
  }
  __syncthreads();
  // 4) contiguous digit runs out to global memory
  for (int p = threadIdx.x; p < valid; p += kRadixBlock) {
    const uint32_t key = sk[p];
    const int d = (int)((key >> shift) & (kRadixDigits - 1));
    sink(gbase[d] + (uint32_t)p - dstart[d], key, sv[p]);
  }
}

// Digit histograms of `passes` 8-bit digits starting at bit `shift0` over
// arbitrary u32 keys (the upsweep of a general sort; k_radix_ghist derives
// them from node counts instead).  ghist[p * 256 + d] must be zero on entry.
static __global__ void k_digit_hist(const uint32_t *__restrict__ keys, long long n, int shift0, int passes,
                                   uint32_t *__restrict__ ghist) { lod::pdl_wait();
  __shared__ uint32_t h[kMaxPasses * kRadixDigits];
  for (int i = threadIdx.x; i < kMaxPasses * kRadixDigits; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (long long i = gtid(); i < n; i += gstride()) {
    const uint32_t k = __ldg(keys + i);
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p * kRadixDigits + ((k >> (shift0 + p * kRadixBits)) & 0xFF)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadixDigits; i += blockDim.x)
    if (h[i]) atomicAdd(ghist + i, h[i]);
}

struct RadixScratch {
  uint32_t *keys_b = nullptr, *vals_a = nullptr, *vals_b = nullptr;
  uint32_t *ghist = nullptr;         // kMaxPasses * 256
  uint32_t *lb[2] = {nullptr, nullptr};  // ntiles * 256 + 1 each, alternating per pass
};

inline long long radix_tiles(long long n) { return (n + kRadixTile - 1) / kRadixTile; }
inline long long radix_lb_elems(long long n) { return radix_tiles(n) * kRadixDigits + 1; }

inline int radix_passes(uint32_t max_key) {
  int bits = 0;
  while (bits < 32 && (max_key >> bits) != 0) ++bits;
  int p = (bits + kRadixBits - 1) / kRadixBits;
  return p < 1 ? 1 : p;
}

// Stable sort of (keys, item index) by key (keys/ghist from k_radix_prep +
// k_radix_ghist).  n is the item count, or an upper bound when n_dev holds
// the count on the device.  On return *keys_res / *vals_res point at the sorted keys /
// original item indices -- unless `last` is given: then the last pass hands
// every item's final position to that sink instead of writing the arrays
// (*keys_res / *vals_res are then null).
template <class LastSink = KVSink>
inline void stable_multisplit(uint32_t *keys, long long n, int passes, RadixScratch &s, cudaStream_t st,
                              uint32_t **keys_res, uint32_t **vals_res, const uint32_t *vals0 = nullptr,
                              int shift0 = 0, const LastSink *last = nullptr, const long long *n_dev = nullptr,
                              const int *guard = nullptr, bool first_nowait = false) {
  const long long ntiles = radix_tiles(n);
  uint32_t *kin = keys, *kout = s.keys_b;
  const uint32_t *vin = vals0;
  uint32_t *vout = s.vals_a;
  for (int p = 0; p < passes; ++p) {
    if (n > 0) {
      // look-back buffer p&1 was zeroed by k_radix_prep (p = 0) or by pass p-1
      uint32_t *lbn = p + 1 < passes ? s.lb[(p + 1) & 1] : (uint32_t *)nullptr;
      const int nowait = (first_nowait && p == 0) ? 1 : 0;
      if (last && p + 1 == passes)
        lod::launch(k_onesweep<LastSink>, (unsigned)ntiles, kRadixBlock, 0, st, kin, vin, n, n_dev,
                    shift0 + p * kRadixBits, s.ghist + p * kRadixDigits, s.lb[p & 1], ntiles, *last, lbn, guard,
                    nowait);
      else
        lod::launch(k_onesweep<KVSink>, (unsigned)ntiles, kRadixBlock, 0, st, kin, vin, n, n_dev,
                    shift0 + p * kRadixBits, s.ghist + p * kRadixDigits, s.lb[p & 1], ntiles, KVSink{kout, vout}, lbn,
                    guard, nowait);
    }
    uint32_t *kt = kin;
    kin = kout;
    kout = kt;
    vin = vout;
    vout = (vout == s.vals_a) ? s.vals_b : s.vals_a;
  }
  *keys_res = last ? nullptr : kin;
  *vals_res = last ? nullptr : const_cast<uint32_t *>(vin);
}

}  // namespace lod
