// lod_tree.cu -- host orchestration of the B200 update cycle + the C ABI.
//
// One LodTree owns all device state of one octree (node table, chunk pool,
// arena, per-cycle scratch) and one CUDA stream.  lod_insert_batch replaces
// lodstream.update.insert_batch (update.py:252-393); see lod_kernels.cuh for
// the per-pass kernels and DESIGN.md for the data layout.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <vector>

#include "../../include/lod_b200.h"
#include "lod_common.cuh"
#include "lod_kernels.cuh"
#include "lod_small.cuh"
#include "radix.cuh"
#include "scan.cuh"

using namespace lod;

namespace {

// LOD_DEBUG=1: log buffer growth and slow cycles to stderr
inline bool lod_debug() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LOD_DEBUG");
    v = (e && *e && *e != '0') ? 1 : 0;
  }
  return v == 1;
}

// Bytes of the stream-ordered pool kept backed per device (the warm-up
// reserve); freed scratch beyond it goes back to the driver when a tree is
// destroyed or an allocation fails (cudaMemPoolTrimTo), so the pool never
// hoards memory that plain cudaMalloc (arenas) or another tree needs.
static unsigned long long g_pool_keep[64];
static void trim_pool(int dev, bool all) {
  cudaMemPool_t pool;
  if (dev >= 0 && dev < 64 && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, all ? 0 : (size_t)g_pool_keep[dev]);
  }
  cudaGetLastError();
}

template <typename T>
struct DBuf {
  T *p = nullptr;
  long long cap = 0;
  // Grow to hold n elements; keep the first `keep` elements when growing.
  // 2x the request: a burst (a spill wave) leaves room for the next one, so
  // scratch growth (allocation + copy, host work inside the update) happens
  // a few times per stream instead of at every new high-water mark.  `tight`
  // (the claim tables, memset whole on growth; the chunk directory) and
  // requests past 256 MB: max(n, 2x the old capacity).
  int ensure(long long n, cudaStream_t st, long long keep = 0, bool tight = false) {
    if (n <= cap) return 0;
    const bool exact = tight || (unsigned long long)n * sizeof(T) > (256ull << 20);
    long long nc = std::max<long long>(exact ? n : 2 * n, std::max<long long>(2 * cap, 1024));
    if (lod_debug())
      fprintf(stderr, "[lod] grow buffer %lld -> %lld elems (%.1f MB)\n", cap, nc, nc * sizeof(T) / 1e6);
    T *q = nullptr;
    // stream-ordered: growth never synchronizes the device
    cudaError_t e = cudaMallocAsync(&q, (size_t)nc * sizeof(T), st);
    if (e != cudaSuccess) {  // give the pool's unused memory back and retry once
      cudaGetLastError();
      int dev = 0;
      cudaGetDevice(&dev);
      trim_pool(dev, true);
      if (cudaMallocAsync(&q, (size_t)nc * sizeof(T), st) != cudaSuccess) {
        cudaGetLastError();
        return LOD_E_NOMEM;
      }
    }
    if (p) {
      if (keep > 0) cudaMemcpyAsync(q, p, (size_t)std::min(keep, cap) * sizeof(T), cudaMemcpyDeviceToDevice, st);
      cudaFreeAsync(p, st);
    }
    p = q;
    cap = nc;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

inline unsigned grid_for(long long n, int block = 256) {
  long long b = (n + block - 1) / block;
  if (b < 1) b = 1;
  long long cap = 148LL * 16;
  return (unsigned)std::min(b, cap);
}

// Claim-table sizes: rounded up to a multiple of 64 Ki slots.
inline unsigned long long round_slots(unsigned long long v) { return (v + 65535ull) / 65536ull * 65536ull; }


}  // namespace

__global__ void k_init_root(NodeCols nd, double b0, double b1, double b2) { lod::pdl_wait();
  nd.parent[0] = LOD_NO_NODE;
  nd.octant[0] = 0;
  nd.level[0] = 0;
  for (int q = 0; q < 8; ++q) nd.children[q] = LOD_NO_NODE;
  nd.inner[0] = 0;
  nd.final_[0] = 0;
  nd.count[0] = 0;
  nd.pending[0] = 0;
  nd.chunk_head[0] = LOD_NO_CHUNK;
  nd.chunk_tail[0] = LOD_NO_CHUNK;
  nd.chunk_count[0] = 0;
  nd.grid_off[0] = -1;
  nd.dir_off[0] = 0;
  nd.dir_cap[0] = 0;
  nd.bmin[0] = b0;
  nd.bmin[1] = b1;
  nd.bmin[2] = b2;
  nd.desc[0] = make_int2(-1, 0);
}

__global__ void k_cycle_begin(Ctrl *c) { lod::pdl_wait();
  c->t_prev_begin = c->t_begin;
  c->t_prev_end = c->t_end;
  c->t_begin = gtimer_ns();
  c->t_end = 0;
  c->n_touched = 0;
  c->n_splits = 0;
  c->error = 0;
  c->spill_total = 0;
  c->spill_add = 0;
  c->n_used = 0;
  c->hash_overflow = 0;
  c->n_v = 0;
  c->n_wins = 0;
  c->n_keys = 0;
  c->acq_tot = u64x2(0, 0);
}


// Walk one node's chunk list into a packed record buffer (gather_samples,
// octree.py:298-326).  One CTA per listed node.
__global__ void k_gather_nodes(NodeCols nd, PoolCols pool, Geo geo, const uint8_t *__restrict__ arena,
                               const int32_t *__restrict__ nodes, const long long *__restrict__ starts,
                               const long long *__restrict__ out_off, float4 *__restrict__ out) { lod::pdl_wait();
  __shared__ int s_cid, s_occ;
  __shared__ long long s_poff;
  const int nid = nodes[blockIdx.x];
  const long long start = starts ? starts[blockIdx.x] : 0;
  float4 *dst = out + out_off[blockIdx.x];
  if (threadIdx.x == 0) s_cid = nd.chunk_head[nid];
  __syncthreads();
  long long pos = 0;  // index of the first record of the current chunk
  while (s_cid != LOD_NO_CHUNK) {
    if (threadIdx.x == 0) {
      s_occ = pool.occupied[s_cid];
      s_poff = pool.payload_off[s_cid];
    }
    __syncthreads();
    const int occ = s_occ;
    const float4 *src = reinterpret_cast<const float4 *>(arena + s_poff);
    for (int r = threadIdx.x; r < occ; r += blockDim.x)
      if (pos + r >= start) dst[pos + r - start] = src[r];
    pos += occ;
    __syncthreads();
    if (threadIdx.x == 0) s_cid = pool.next[s_cid];
    __syncthreads();
  }
}

struct LodTree {
  LodParams p{};
  int dev = 0;
  cudaStream_t st = nullptr;
  Geo geo{};
  unsigned long long arena_cap = 0;
  uint8_t *arena = nullptr;
  long long ncap = 0;
  NodeCols nd{};
  long long ccap = 0;
  PoolCols pool{};
  Ctrl *d_ctrl = nullptr;
  Ctrl *h_ctrl = nullptr;       // pinned + mapped: k_publish writes it directly
  Ctrl *h_ctrl_dev = nullptr;   // device alias of h_ctrl
  unsigned *h_seq = nullptr;    // pinned + mapped publication counter
  unsigned *h_seq_dev = nullptr;
  unsigned seq = 0;
  // expansion scratch
  DBuf<int32_t> split_list, node_b, node_all;  // node_b: batch points' node cache; node_all: spilled points'
  DBuf<uint32_t> bitmap;  // split flags over node ids (k_decide: the test phase -> the ranking block)
  DBuf<long long> scnt, schk, spill_off, chunk_off;
  DBuf<float4> spill;
  // sampling scratch
  DBuf<int32_t> srank;  // split rank per node (-1 when not splitting)
  int hepoch = 0;                // claim-key epoch of the running cycle (Hash.tag)
  DBuf<HSlot> hslots, hslots2;  // claim table (`hcap` slots in use) + growth spare
  DBuf<unsigned long long> hused;
  DBuf<uint32_t> wcount, wbase;  // per-point win counts (zero between cycles) / their exclusive scan
  unsigned long long hcap = 0;
  int h2_epoch = -1;  // epoch whose keys the spare claim table (hslots2) may still hold
  long long prev_used = 0;  // claims of the previous cycle (sizes the table)
  int last_iters = 0;       // expansion iterations of the previous cycle (speculation policy)
  long long spec_hits = 0;  // cycles whose pipeline ran speculatively
  DBuf<uint4> backlog;  // the cycle's new voxels in backlog order: {node, cell, rgba, winner index}
  DBuf<uint4> wins;     // burst path: k_resolve_list's win list {winner, node, cell, rgba}
  // sort / alloc scratch
  DBuf<uint32_t> keys, keys_b, vals_a, vals_b, hist, ghist, nodecnt;
  DBuf<uint32_t> dmat, dlb;  // direct placement: tiles x nodes counts -> prefixes; column-scan look-back
  DBuf<uint16_t> drank;      // direct placement: in-tile ranks
  DBuf<U64x2> dpscan;        // direct placement: the plan scan's per-column-block aggregates / prefixes
  DBuf<int32_t> seg_node, dense;
  DBuf<U64x2> pairs;     // packed per-node plans, scanned in place (k_radix_ghist -> k_seg_list)
  DBuf<long long> wlo;   // write list: payload offsets of every touched node's chunks in slot order
  DBuf<SinkInfo> sinfo;  // per node id: segment start, write-list start, count (k_alloc)
  DBuf<long long> seg_start;
  DBuf<U64x2> plan, plan_ex;
  ScanLB lb32, lb64;  // single-pass scan state (u32 win counts; U64x2 segment / need pairs)
  // inputs / outputs
  DBuf<float> in_xyz;
  DBuf<float4> in_rec;  // packed host input (LOD_FLAG_PACKED)
  DBuf<float4> dcopy;   // device batch as packed records (released early, k_count copy_out)
  cudaEvent_t ev_release = nullptr;
  DBuf<uint32_t> in_rgba;
  DBuf<float4> gbuf;
  DBuf<int32_t> gnodes;
  DBuf<long long> goff, gstart;
  DBuf<long long> woff;  // render work list: piece offsets per listed node
  DBuf<int32_t> vislist;
  DBuf<unsigned long long> fb;
  DBuf<unsigned long long> counter;
  // BatchDelta of the last call with LOD_FLAG_DELTA (lod_read_delta)
  DBuf<int32_t> dsplits, dvnode, dpnode;
  DBuf<long long> dvstart, dvcount, dpstart, dpcount, dvbase;
  DBuf<uint32_t> dvcell, dvrgba;
  long long d_nsplits = 0, d_nvg = 0, d_npg = 0, d_nv = 0;
  // ingest feed: batches staged H2D on a copy stream ahead of their insert
  // (lod_prefetch_batch), a ring of kStages slots
  cudaStream_t cst = nullptr;
  struct Stage {
    DBuf<float> xyz;
    DBuf<uint32_t> rgba;
    DBuf<float4> rec;      // packed batches (lod_prefetch_records)
    bool packed = false;   // hx = the packed host records, hc = null
    const void *hx = nullptr, *hc = nullptr;
    long long n = 0;
    bool valid = false;
    bool pending = false;  // copy requested, not yet issued (issued behind the next count pass)
    int parts = 0;         // parts not issued yet: 1 = colours, 2 = positions (packed records: 2)
    unsigned long long order = 0;  // prefetch order (copies are issued oldest first)
    cudaEvent_t ready = nullptr;
  } stage[3];
  unsigned long long stage_order = 0;
  cudaEvent_t ev_counted = nullptr;  // the running cycle's first count pass is done
  cudaEvent_t ev_aux = nullptr;      // lod_last_voxels_count -> caller stream
  cudaEvent_t ev_input = nullptr;    // the caller's input stream (LOD_FLAG_INPUT_STREAM)
  int stage_next = 0;
  cudaEvent_t ev[16] = {};  // 12, 13: per-iteration k_count brackets; 10/11 and 14/15: the two
                            // (inputs resident, settled) pairs, alternating between calls
  int ev_slot = 0;          // pair of the last call
  bool tail_pending = false;  // the last call returned before its sort + store finished
  bool tail_ev = false;       // ... and is timed by its event pair (else by the Ctrl stamps)
  DBuf<int32_t> cdir;  // chunk directory entries (pool.cdir)
  // host copies of counters (authoritative after every call)
  long long num_nodes = 1;
  long long d2h_bytes = 0;  // control-block readbacks since the last reset
  // small-batch path (lod_small.cuh): one launch per cycle
  DBuf<float4> sm_brec, sm_srec;
  DBuf<int32_t> sm_node_b, sm_node_s, sm_tl, sm_cand, sm_splits, sm_touched;
  DBuf<long long> sm_nnew, sm_cur, sm_wls, sm_pl, sm_wl, sm_sp;  // nnew / cur / wls: per node
  DBuf<uint4> sm_backlog;
  float4 *sm_ring = nullptr, *sm_ring_dev = nullptr;  // mapped pinned batch slots
  SmallResult *sm_res = nullptr, *sm_res_dev = nullptr;  // mapped per-call result
  unsigned *sm_done = nullptr, *sm_done_dev = nullptr;    // mapped completion counter
  SmallAccum *sm_acc = nullptr;                           // device: totals of queued cycles
  unsigned sm_seq = 0;
  long long sm_queued = 0;  // asynchronous small cycles since the host copies were exact
  long long sm_unfolded = 0;  // asynchronous small cycles not yet reported by lod_tree_settle
  // upper bounds of the counters while asynchronous small cycles are queued
  // (exact whenever sm_queued == 0)
  long long ub_nodes = 1, ub_alloc = 0, ub_dir = 0;
  long long ncap_hint = 0, ccap_hint = 0;  // node / chunk rows at the first large batch
  bool sized_large = false;
  bool fixing_dir = false;  // fix_directory running (its own sync must not recurse)
  long long dir_rebuilds = 0;
  unsigned long long ub_arena = 0;
  long long ingested = 0;  // points inserted so far (bounds the spill of a cycle)
  // the last cycle's backlog (lod_last_voxels): which buffer, entries, spill length
  const uint4 *last_backlog = nullptr;
  long long last_nv = 0, last_ns = 0;
};

static constexpr int kSmallRing = 512;  // batch slots of kSmallMaxBatch records each

// ---------------------------------------------------------------- burst resolve
// A split wave re-descends tens of millions of spilled points in one cycle
// (density-skew stream: 20-43M), and as many new voxels are claimed.  The
// regular resolve then does two random atomics per voxel on per-point win
// counters far larger than L2 (plus a random backlog write); instead the
// burst path lists every occupied slot once, {winner, node, cell, rgba},
// with the winner as a sort key, and orders the list by winner with the
// stable LSD radix passes -- ascending winner index is exactly the backlog
// order (a point's wins lie at different nodes, so their mutual order is
// irrelevant after the node sort).  The last pass writes the backlog.
constexpr int kResolveItems = 8;  // slots per thread per round: one list reservation per 2048 slots
__global__ void __launch_bounds__(256)
    k_resolve_list(NodeCols nd, Hash h, uint32_t *grid32, long long n_s, uint4 *__restrict__ wins,
                   uint32_t *__restrict__ wkey, int passes, uint32_t *__restrict__ ghist, Ctrl *ctrl,
                   const int *guard) { lod::pdl_wait();
  __shared__ uint32_t sh[256 / 32 + 1];
  __shared__ unsigned long long s_base;
  __shared__ uint32_t hist[kMaxPasses * kRadixDigits];
  if (guard && *guard) return;
  for (int i = threadIdx.x; i < kMaxPasses * kRadixDigits; i += blockDim.x) hist[i] = 0;
  const long long H = (long long)h.cap;
  constexpr long long kRound = 256LL * kResolveItems;
  for (long long r0 = (long long)blockIdx.x * kRound; r0 < H; r0 += (long long)gridDim.x * kRound) {
    ulonglong2 kv[kResolveItems];
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kResolveItems; ++k) {
      const long long sidx = r0 + k * 256 + threadIdx.x;
      kv[k] = make_ulonglong2(kEmptyKey, kEmptyHi);
      if (sidx < H) kv[k] = __ldcg(reinterpret_cast<const ulonglong2 *>(h.slots + sidx));
      cnt += live(h, kv[k].x);
    }
    uint32_t tot;
    const uint32_t off = block_exclusive_scan<uint32_t, 256>(cnt, sh, tot);
    if (tot == 0) continue;  // block-uniform
    if (threadIdx.x == 0) s_base = atomicAdd(reinterpret_cast<unsigned long long *>(&ctrl->n_wins),
                                             (unsigned long long)tot);
    __syncthreads();
    unsigned long long pos = s_base + off;
    __syncthreads();  // s_base is rewritten next round
#pragma unroll
    for (int k = 0; k < kResolveItems; ++k) {
      if (!live(h, kv[k].x)) continue;  // stale from the next cycle on: no clearing write
      const int nid = key_node(h, kv[k].x);
      const uint32_t cell = key_cell(h, kv[k].x);
      const uint32_t j = (uint32_t)claim_index((uint32_t)(kv[k].y >> 32), n_s);
      atomicOr(grid32 + (nd.grid_off[nid] >> 2) + (cell >> 5), 1u << (cell & 31));
      wins[pos] = make_uint4(j, (uint32_t)nid, cell, (uint32_t)kv[k].y);
      wkey[pos] = j;
      ++pos;
      for (int p = 0; p < passes; ++p) atomicAdd(&hist[p * kRadixDigits + ((j >> (p * kRadixBits)) & 0xFF)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadixDigits; i += blockDim.x)
    if (hist[i]) atomicAdd(ghist + i, hist[i]);
}

// The win sort's last pass: the entry at sorted position `pos` becomes
// backlog entry `pos` {node, cell, rgba}.
struct WinSink {
  const uint4 *wins;
  uint4 *backlog;
  __device__ __forceinline__ void operator()(uint32_t pos, uint32_t, uint32_t val) const {
    const uint4 e = wins[val];
    backlog[pos] = make_uint4(e.y, e.z, e.w, e.x);
  }
};

// ---------------------------------------------------------------- helpers

static int cuda_rc(cudaError_t e) {
  if (e == cudaSuccess) return LOD_OK;
  fprintf(stderr, "[lod_b200] CUDA error: %s\n", cudaGetErrorString(e));
  return LOD_E_CUDA;
}

#define CK(expr)                             \
  do {                                       \
    int rc__ = cuda_rc(expr);                \
    if (rc__) return rc__;                   \
  } while (0)
#define RK(expr)                             \
  do {                                       \
    int rc__ = (expr);                       \
    if (rc__) return rc__;                   \
  } while (0)

// Host view of the control block after all work queued so far: one warp
// copies it into mapped pinned memory and then bumps a publication counter,
// which the host polls -- no copy-engine round trip and no stream-sync wake-up
// on the critical path of the expansion loop.  A stream error while polling
// (or LOD_SYNC_MEMCPY=1) falls back to copy + synchronize.
// release != 0: the next kernel may start as soon as this one has waited (it
// must then skip its own wait: k_onesweep's nowait) -- the system-scope fence
// below takes 4-5 us, and ~20 us while the copy engines stream a batch in
// over PCIe, which would otherwise stall the stream behind the publication.
__global__ void k_publish(const Ctrl *__restrict__ d, Ctrl *h, volatile unsigned *seq_out, unsigned seq,
                          int release) {
  lod::pdl_wait();
  if (release) lod::pdl_trigger();
  constexpr int kWords = (int)(sizeof(Ctrl) / 8);
  static_assert(sizeof(Ctrl) % 8 == 0, "Ctrl is copied in 8-byte words");
  const unsigned long long *src = reinterpret_cast<const unsigned long long *>(d);
  volatile unsigned long long *dst = reinterpret_cast<volatile unsigned long long *>(h);
  for (int k = threadIdx.x; k < kWords; k += 32) dst[k] = src[k];
  __threadfence_system();
  __syncwarp();
  if (threadIdx.x == 0) *seq_out = seq;
}

static unsigned publish_ctrl(LodTree *t, bool release = false);
static int wait_ctrl(LodTree *t, unsigned want);

// Control-block reads through mapped pinned memory (k_publish), unless
// LOD_SYNC_MEMCPY asks for a copy + stream sync.
static bool mapped_sync(const LodTree *t) {
  static const bool memcpy_sync = getenv("LOD_SYNC_MEMCPY") != nullptr;
  return !memcpy_sync && t->h_seq_dev;
}

// then_issue: the queued batches' H2D copies are issued behind the
// publication (a copy streaming over PCIe slows the publication's
// system-scope write from ~5 to ~20 us).
static int issue_pending(LodTree *t, const LodTree::Stage *upto = nullptr, int mask = 3);
static int sync_ctrl(LodTree *t, bool then_issue = false) {
  if (!mapped_sync(t)) {
    if (then_issue) RK(issue_pending(t));
    t->d2h_bytes += (long long)sizeof(Ctrl);
    CK(cudaMemcpyAsync(t->h_ctrl, t->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, t->st));
    CK(cudaStreamSynchronize(t->st));
  } else {
    const unsigned want = publish_ctrl(t);
    if (then_issue) RK(issue_pending(t));
    RK(wait_ctrl(t, want));
  }
  // published behind everything queued: the directory's bump pointer is exact
  t->ub_dir = (long long)t->h_ctrl->dir_top;
  return LOD_OK;
}

// Queue a publication of the control block on the tree stream (no wait).
static unsigned publish_ctrl(LodTree *t, bool release) {
  const unsigned want = ++t->seq;
  t->d2h_bytes += (long long)sizeof(Ctrl);
  lod::launch(k_publish, 1, 32, 0, t->st, t->d_ctrl, t->h_ctrl_dev, t->h_seq_dev, want, release ? 1 : 0);
  return want;
}

// Wait until publication `want` reached the host (the stream work queued
// before it is done; work queued after it may still run).
static int wait_ctrl(LodTree *t, unsigned want) {
  volatile unsigned *flag = t->h_seq;
  for (unsigned spins = 0; *flag != want; ++spins) {
    if ((spins & 1023) == 1023) {
      const cudaError_t e = cudaStreamQuery(t->st);
      if (e != cudaSuccess && e != cudaErrorNotReady) return cuda_rc(e);
      if (e == cudaSuccess && *flag != want) {  // stream drained without the flag: should not happen
        CK(cudaMemcpyAsync(t->h_ctrl, t->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, t->st));
        CK(cudaStreamSynchronize(t->st));
        return LOD_OK;
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return LOD_OK;
}

// The counters as the host last saw them become exact again (after queued
// asynchronous small cycles: one publication behind everything queued).
static int fix_directory(LodTree *t);

static int exact_bounds(LodTree *t) {
  const Ctrl &c = *t->h_ctrl;
  t->num_nodes = c.num_nodes;
  t->ub_nodes = c.num_nodes;
  t->ub_alloc = c.allocated_total;
  t->ub_arena = c.arena_off;
  t->sm_queued = 0;
  return c.dir_overflow ? fix_directory(t) : LOD_OK;
}

static int refresh(LodTree *t) {
  if (t->sm_queued == 0) return LOD_OK;
  RK(sync_ctrl(t));
  return exact_bounds(t);
}

template <typename T>
static int grow_col(T *&ptr, long long old_cap, long long new_cap, long long keep, cudaStream_t st) {
  T *q = nullptr;
  if (cudaMallocAsync(&q, (size_t)new_cap * sizeof(T), st) != cudaSuccess) {
    cudaGetLastError();
    return LOD_E_NOMEM;
  }
  if (ptr && keep > 0) CK(cudaMemcpyAsync(q, ptr, (size_t)keep * sizeof(T), cudaMemcpyDeviceToDevice, st));
  if (ptr) CK(cudaFreeAsync(ptr, st));
  ptr = q;
  (void)old_cap;
  return LOD_OK;
}

// Bits of a cell index (g^3 cells) and the node ids a claim key can hold
// (int32 ids, like the reference's, capped by the key's 56 - cbits bits).
static int cell_bits(long long g) {
  const unsigned long long cells = (unsigned long long)g * g * g;
  int b = 1;
  while ((1ull << b) < cells) ++b;
  return b;
}
static long long max_nodes(const LodTree *t) {
  const int nb = 56 - cell_bits(t->geo.g);
  return nb >= 31 ? (1LL << 31) - 1 : (1LL << nb);
}

// Node table capacity (Octree._grow doubling, octree.py:192-209).
static int ensure_nodes(LodTree *t, long long want, long long live) {
  if (want <= t->ncap) return LOD_OK;
  if (want > max_nodes(t)) return LOD_E_NOMEM;  // claim keys hold 56 - cbits bits of node id
  long long nc = std::max<long long>(t->ncap, 1024);
  while (nc < want) nc *= 2;
  if (lod_debug()) fprintf(stderr, "[lod] grow node table %lld -> %lld\n", t->ncap, nc);
  cudaStream_t st = t->st;
  RK(grow_col(t->nd.parent, t->ncap, nc, live, st));
  RK(grow_col(t->nd.octant, t->ncap, nc, live, st));
  RK(grow_col(t->nd.level, t->ncap, nc, live, st));
  RK(grow_col(t->nd.children, t->ncap * 8, nc * 8, live * 8, st));
  RK(grow_col(t->nd.inner, t->ncap, nc, live, st));
  RK(grow_col(t->nd.final_, t->ncap, nc, live, st));
  RK(grow_col(t->nd.count, t->ncap, nc, live, st));
  RK(grow_col(t->nd.pending, t->ncap, nc, live, st));
  RK(grow_col(t->nd.chunk_head, t->ncap, nc, live, st));
  RK(grow_col(t->nd.chunk_tail, t->ncap, nc, live, st));
  RK(grow_col(t->nd.chunk_count, t->ncap, nc, live, st));
  RK(grow_col(t->nd.grid_off, t->ncap, nc, live, st));
  RK(grow_col(t->nd.bmin, t->ncap * 3, nc * 3, live * 3, st));
  RK(grow_col(t->nd.desc, t->ncap, nc, live, st));
  RK(grow_col(t->nd.dir_off, t->ncap, nc, live, st));
  RK(grow_col(t->nd.dir_cap, t->ncap, nc, live, st));
  // node-indexed scratch
  long long words = (nc + 31) / 32 + 1;
  long long oldw = t->bitmap.cap;
  RK(t->bitmap.ensure(words, st, oldw));
  if (t->bitmap.cap > oldw) CK(cudaMemsetAsync(t->bitmap.p + oldw, 0, (size_t)(t->bitmap.cap - oldw) * 4, st));
  // the split plan of the running iteration survives the growth (k_execute reads it)
  RK(t->split_list.ensure(nc, st, t->split_list.cap));
  RK(t->scnt.ensure(nc, st));
  RK(t->schk.ensure(nc, st));
  RK(t->spill_off.ensure(nc, st, t->spill_off.cap));
  RK(t->chunk_off.ensure(nc, st, t->chunk_off.cap));
  long long olds = t->srank.cap;
  RK(t->srank.ensure(nc, st, olds));
  if (t->srank.cap > olds) CK(cudaMemsetAsync(t->srank.p + olds, 0xFF, (size_t)(t->srank.cap - olds) * 4, st));
  long long oldnn = t->sm_nnew.cap;  // zero between cycles
  RK(t->sm_nnew.ensure(nc, st, oldnn));
  if (t->sm_nnew.cap > oldnn) CK(cudaMemsetAsync(t->sm_nnew.p + oldnn, 0, (size_t)(t->sm_nnew.cap - oldnn) * 8, st));
  RK(t->sm_cur.ensure(nc, st));
  RK(t->sm_wls.ensure(nc, st));
  t->ncap = nc;
  return LOD_OK;
}

// Chunk pool row capacity (ChunkPool._grow, store.py:104-108).
static int ensure_chunks(LodTree *t, long long want, long long live) {
  if (want <= t->ccap) return LOD_OK;
  long long nc = std::max<long long>(t->ccap, 1024);
  while (nc < want) nc *= 2;
  if (lod_debug()) fprintf(stderr, "[lod] grow chunk table %lld -> %lld\n", t->ccap, nc);
  cudaStream_t st = t->st;
  RK(grow_col(t->pool.next, t->ccap, nc, live, st));
  RK(grow_col(t->pool.payload_off, t->ccap, nc, live, st));
  RK(grow_col(t->pool.occupied, t->ccap, nc, live, st));
  RK(grow_col(t->pool.owner, t->ccap, nc, live, st));
  RK(grow_col(t->pool.cidx, t->ccap, nc, live, st));
  RK(grow_col(t->pool.free_stack, t->ccap, nc, live, st));
  t->ccap = nc;
  return LOD_OK;
}

// Chunk-directory capacity for a cycle that may append `acq` chunks to up to
// `touched` nodes: every region relocation takes max(4, 2 x the node's new
// chunk count), so a cycle hands out at most 2 (chunks after it) + 4 touched
// entries past the current bump pointer (h_ctrl->dir_top, exact between calls).
// t->ub_dir bounds dir_top after everything launched so far: exact after every
// sync_ctrl (published behind all queued work), plus the reserve of every
// cycle launched since.
static int grow_dir(LodTree *t, long long want) {
  if (want <= t->cdir.cap) return LOD_OK;
  // the whole old allocation travels: a soft-bounded small cycle may have
  // handed out entries past t->ub_dir
  RK(t->cdir.ensure(want, t->st, t->cdir.cap, true));
  t->pool.cdir = t->cdir.p;
  t->pool.cdir_cap = (unsigned long long)t->cdir.cap;
  return LOD_OK;
}

static int ensure_dir(LodTree *t, long long chunks_after, long long touched) {
  t->ub_dir += 2 * chunks_after + 4 * touched + 1024;
  return grow_dir(t, t->ub_dir);
}

// Look-back state of the single-pass scan for up to `tiles` tiles of T.
template <typename T>
static int ensure_scan_lb(ScanLB &lb, long long n, cudaStream_t st) {
  const long long tiles = std::max<long long>((n + kScanTile - 1) / kScanTile, 1);
  if (tiles <= lb.cap_tiles) return LOD_OK;
  const long long c = std::max<long long>(2 * tiles, 2 * lb.cap_tiles);
  // stream-ordered: the old arrays go back to the pool behind the launches
  // that still use them (a device-wide sync here stalled the update ~0.2 ms)
  if (lb.status) CK(cudaFreeAsync(lb.status, st));
  if (lb.agg) CK(cudaFreeAsync(lb.agg, st));
  if (lb.incl) CK(cudaFreeAsync(lb.incl, st));
  if (!lb.ticket) {
    CK(cudaMallocAsync(reinterpret_cast<void **>(&lb.ticket), 8, st));
    CK(cudaMemsetAsync(lb.ticket, 0, 8, st));
    lb.tickets = 0;
  }
  CK(cudaMallocAsync(reinterpret_cast<void **>(&lb.status), (size_t)c * 4, st));
  CK(cudaMemsetAsync(lb.status, 0, (size_t)c * 4, st));
  CK(cudaMallocAsync(&lb.agg, (size_t)c * sizeof(T), st));
  CK(cudaMallocAsync(&lb.incl, (size_t)c * sizeof(T), st));
  lb.epoch = 0;
  lb.cap_tiles = c;
  return LOD_OK;
}

static void release_scan_lb(ScanLB &lb) {
  if (lb.status) cudaFree(lb.status);
  if (lb.agg) cudaFree(lb.agg);
  if (lb.incl) cudaFree(lb.incl);
  if (lb.ticket) cudaFree(lb.ticket);
  lb = ScanLB{};
}

static int issue_stage(LodTree *t, LodTree::Stage &sg, int mask);
constexpr int kPartSmall = 1, kPartBig = 2, kPartsAll = 3;

// Issue the oldest queued batch's deferred H2D copy behind the work queued so
// far (through `upto`, when given: every copy up to that slot).  One copy
// per cycle keeps pace with the inserts and leaves the copy engines idle for
// part of each cycle -- where the split iteration's publication lands (a
// copy streaming over PCIe slows that system-scope write from ~5 to ~20 us).
// `mask` = the parts to issue: the colours (1/4 of the bytes) go at the
// start of a cycle, the positions behind the split decision -- so the copy of
// the next batch is done by the end of this cycle without a DMA under the
// decision's publication.
static int issue_pending(LodTree *t, const LodTree::Stage *upto, int mask) {
  if (!t->cst) return LOD_OK;
  bool recorded = false;
  for (;;) {
    LodTree::Stage *old = nullptr;
    for (auto &sg : t->stage)
      if (sg.valid && sg.pending && (sg.parts & mask) && (!old || sg.order < old->order)) old = &sg;
    if (!old) return LOD_OK;
    if (!recorded) {
      CK(cudaEventRecord(t->ev_counted, t->st));
      CK(cudaStreamWaitEvent(t->cst, t->ev_counted, 0));
      recorded = true;
    }
    RK(issue_stage(t, *old, upto ? kPartsAll : mask));
    if (!upto || old == upto || !upto->pending) return LOD_OK;
  }
}

static float stamp_ms(unsigned long long b, unsigned long long e) {
  return e > b ? (float)((double)(e - b) * 1e-6) : -1.f;
}

static void fill_stats(LodTree *t, LodBatchStats *s) {
  const Ctrl &c = *t->h_ctrl;
  s->num_nodes = c.num_nodes;
  s->splits_total = c.splits_total;
  s->max_level = c.max_level;
  s->allocated_total = c.allocated_total;
  s->free_count = c.free_count;
  s->released_total = c.released_total;
  s->arena_offset = c.arena_off;
}

// After a fatal error: drop per-cycle marks and the claim table so the
// structure stays walkable (the reference leaves partial state, errors.py:1-5).
static int abort_cycle(LodTree *t, int code) {
  lod::launch(k_clear_marks_all, grid_for(t->num_nodes), 256, 0, t->st, t->nd, t->srank.p, t->num_nodes,
              t->geo.fresh);
  if (t->hslots.p) {
    cudaMemsetAsync(t->hslots.p, 0xFF, (size_t)t->hslots.cap * sizeof(HSlot), t->st);
    if (t->wcount.p) cudaMemsetAsync(t->wcount.p, 0, (size_t)t->wcount.cap * 4, t->st);
  }
  long long words = (t->ncap + 31) / 32 + 1;
  cudaMemsetAsync(t->bitmap.p, 0, (size_t)words * 4, t->st);
  if (t->ghist.p) cudaMemsetAsync(t->ghist.p, 0, (size_t)t->ghist.cap * 4, t->st);
  if (t->nodecnt.p) cudaMemsetAsync(t->nodecnt.p, 0, (size_t)t->nodecnt.cap * 4, t->st);
  cudaStreamSynchronize(t->st);
  // counters: the device ctrl keeps whatever was applied before the failure
  sync_ctrl(t);
  (void)exact_bounds(t);
  return code;
}

// ---------------------------------------------------------------- small batches

// Spin until a mapped counter reaches `want` (a stream error ends the wait).
static int wait_mapped(LodTree *t, volatile unsigned *flag, unsigned want) {
  for (unsigned spins = 0; (int)(*flag - want) < 0; ++spins) {
    if ((spins & 1023) == 1023) {
      const cudaError_t e = cudaStreamQuery(t->st);
      if (e != cudaSuccess && e != cudaErrorNotReady) return cuda_rc(e);
      if (e == cudaSuccess && (int)(*flag - want) < 0) return LOD_E_CUDA;  // drained without the write
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return LOD_OK;
}

// One update cycle of a tiny host batch in one launch (k_small_cycle).  The
// worst case of the cycle is bounded from n alone: a leaf below max depth
// holds <= T points, so the spill is <= n*T, a path crosses <= max_depth
// inner nodes, every split needs > T points.  When that worst case cannot
// overflow the backlog, the spill buffer or the arena, the call returns as
// soon as the kernel is queued (its counters are folded in by
// lod_tree_settle; host copies are refreshed by the next reader); otherwise
// it waits for the kernel's result and reports errors like the pipeline.
// *handled = false: not eligible, the caller runs the pipeline.
static int small_insert(LodTree *t, const float *xyz, const uint32_t *rgba, long long n, long long backlog_cap,
                        long long spill_cap, LodBatchStats &S, bool *handled) {
  *handled = false;
  const Geo &g = t->geo;
  const long long T = std::max<long long>(g.T, 0), D = std::max<long long>(g.max_depth, 1), C = g.C;
  if (n * T > kSmallAllMax && t->ingested > kSmallAllMax) return LOD_OK;
  const long long spill_max = std::min<long long>(n * T, t->ingested);
  const long long all_max = n + spill_max;
  if (all_max > kSmallAllMax) return LOD_OK;
  const long long s_max = n + D * (all_max / (T + 1));
  const long long nv_max = all_max * D;
  const long long touched_max = std::min<long long>(all_max + nv_max, (n + 8 * s_max) + (n * D + s_max));
  const long long chunks_max = (all_max + nv_max) / C + touched_max + 1;
  const unsigned long long gs = ((unsigned long long)g.grid_bytes + 63ull) / 64ull * 64ull;
  const unsigned long long arena_max =
      (unsigned long long)s_max * gs + 80ull + (unsigned long long)chunks_max * (unsigned long long)C * 16ull;
  *handled = true;
  cudaStream_t st = t->st;
  // capacities for the worst case (stream-ordered growth; exact counters first)
  // Node and chunk rows are bounded rigorously; growth leaves headroom for
  // many more worst cases so that the exact counters are re-read (a sync)
  // only every few dozen calls at least, not whenever the bound grazes the
  // capacity.  The directory is sized softly: a relocation takes 2 x the
  // node's chunk count, which the host does not track; a cycle that finds no
  // room flags it and the host rebuilds every directory from the chains at
  // its next sync (fix_directory).
  const long long Rn = 8 * s_max + 1, Rc = chunks_max + 1, Rd = 4 * touched_max + 2 * chunks_max + 1024;
  if (t->sm_queued && (t->ub_nodes + Rn > t->ncap || t->ub_alloc + Rc > t->ccap ||
                       t->ub_arena + arena_max > t->arena_cap || t->sm_queued >= 4096))
    RK(refresh(t));
  RK(ensure_nodes(t, t->ub_nodes + Rn + std::min(63 * Rn, t->ub_nodes + 4096), t->ub_nodes));
  RK(ensure_chunks(t, t->ub_alloc + Rc + std::min(63 * Rc, t->ub_alloc + 4096), t->ub_alloc));
  if (t->sm_queued == 0) RK(grow_dir(t, 2 * t->ub_dir + 64 * Rd));  // ub_dir is an upper bound here
  t->ub_dir += Rd;
  const bool async_call = nv_max <= backlog_cap && spill_max <= spill_cap && t->ub_arena + arena_max <= t->arena_cap;
  RK(t->sm_brec.ensure(kSmallMaxBatch, st));
  RK(t->sm_node_b.ensure(kSmallMaxBatch, st));
  RK(t->sm_srec.ensure(spill_max + 1, st));
  RK(t->sm_node_s.ensure(spill_max + 1, st));
  RK(t->sm_tl.ensure(all_max, st));
  RK(t->sm_cand.ensure(all_max, st));
  RK(t->sm_splits.ensure(all_max, st));
  RK(t->sm_sp.ensure(4 * all_max, st));
  RK(t->sm_touched.ensure(touched_max, st));
  RK(t->sm_pl.ensure(3 * touched_max, st));
  RK(t->sm_wl.ensure(chunks_max + touched_max, st));
  RK(t->sm_backlog.ensure(nv_max, st));
  if (!t->sm_ring) {
    CK(cudaHostAlloc(&t->sm_ring, (size_t)kSmallRing * kSmallMaxBatch * sizeof(float4), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&t->sm_ring_dev, t->sm_ring, 0));
    CK(cudaHostAlloc(&t->sm_res, sizeof(SmallResult), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&t->sm_res_dev, t->sm_res, 0));
    CK(cudaHostAlloc(&t->sm_done, sizeof(unsigned), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&t->sm_done_dev, t->sm_done, 0));
    memset(t->sm_res, 0, sizeof(SmallResult));
    *t->sm_done = t->sm_seq;
    CK(cudaMalloc(&t->sm_acc, sizeof(SmallAccum)));
    CK(cudaMemsetAsync(t->sm_acc, 0, sizeof(SmallAccum), st));
  }
  const unsigned seq = t->sm_seq + 1;
  // the slot was last used kSmallRing cycles ago: that cycle must be done
  RK(wait_mapped(t, t->sm_done, seq - kSmallRing));
  const size_t off = (size_t)(seq % kSmallRing) * kSmallMaxBatch;
  float4 *slot = t->sm_ring + off;
  for (long long i = 0; i < n; ++i) {
    float4 r;
    r.x = xyz[3 * i];
    r.y = xyz[3 * i + 1];
    r.z = xyz[3 * i + 2];
    uint32_t c = rgba[i];
    memcpy(&r.w, &c, 4);
    slot[i] = r;
  }
  SmallArgs a;
  a.nd = t->nd;
  a.pool = t->pool;
  a.geo = t->geo;
  a.arena = t->arena;
  a.ctrl = t->d_ctrl;
  a.in = t->sm_ring_dev + off;
  a.n = (int)n;
  a.brec = t->sm_brec.p;
  a.srec = t->sm_srec.p;
  a.node_b = t->sm_node_b.p;
  a.node_s = t->sm_node_s.p;
  a.srank = t->srank.p;
  a.nnew = t->sm_nnew.p;
  a.cur = t->sm_cur.p;
  a.wls = t->sm_wls.p;
  a.backlog = t->sm_backlog.p;
  a.tl = t->sm_tl.p;
  a.cand = t->sm_cand.p;
  a.splits = t->sm_splits.p;
  a.touched = t->sm_touched.p;
  a.pl = t->sm_pl.p;
  a.wl = t->sm_wl.p;
  a.sp = t->sm_sp.p;
  a.all_cap = std::min<long long>({t->sm_tl.cap, t->sm_cand.cap, t->sm_splits.cap, t->sm_sp.cap / 4,
                                   t->sm_srec.cap + n, t->sm_node_s.cap + n});
  a.vox_cap = t->sm_backlog.cap;
  a.touched_cap = std::min<long long>(t->sm_touched.cap, t->sm_pl.cap / 3);
  a.split_cap = std::min<long long>(t->sm_cand.cap, t->sm_splits.cap);
  a.wl_cap = t->sm_wl.cap;
  a.ncap = t->ncap;
  a.ccap = t->ccap;
  a.spill_cap = spill_cap;
  a.backlog_cap = backlog_cap;
  a.arena_cap = t->arena_cap;
  a.res = t->sm_res_dev;
  a.done = t->sm_done_dev;
  a.acc = t->sm_acc;
  a.seq = seq;
  a.async_call = async_call ? 1 : 0;
  static const bool force_overflow = getenv("LOD_DIR_FORCE_OVERFLOW") != nullptr;  // test switch
  if (force_overflow) a.pool.cdir_cap = 0;  // every relocation of this cycle finds no room
  t->sm_seq = seq;
  CK(lod::launch(k_small_cycle, 1, kSmallBlock, 0, st, a));
  t->ingested += n;
  S.launches = 1;
  S.h2d_bytes = 16 * n;  // read by the kernel from mapped host memory
  if (async_call) {  // no error is possible: return now
    t->ub_nodes += 8 * s_max;
    t->ub_alloc += chunks_max;
    t->ub_arena += arena_max;
    ++t->sm_queued;
    ++t->sm_unfolded;
    t->last_backlog = nullptr;  // counts unknown until settled: lod_last_voxels runs the cycle synchronously
    S.iterations = -1;  // queued: lod_tree_settle reports the counts
    S.device_ms = -1.f;
    S.device_ms_prev = -1.f;
    S.n_spill = S.n_voxels = S.n_splits = -1;
    S.num_nodes = t->ub_nodes;  // upper bounds
    S.allocated_total = t->ub_alloc;
    S.arena_offset = t->ub_arena;
    return LOD_OK;
  }
  volatile SmallResult *r = t->sm_res;
  RK(wait_mapped(t, &r->seq, seq));
  S.n_spill = r->n_spill;
  S.n_voxels = r->n_voxels;
  S.n_splits = r->n_splits;
  S.iterations = r->iterations;
  S.num_nodes = r->num_nodes;
  S.splits_total = r->splits_total;
  S.max_level = r->max_level;
  S.allocated_total = r->allocated_total;
  S.free_count = r->free_count;
  S.released_total = r->released_total;
  S.arena_offset = r->arena_off;
  S.device_ms = (float)(r->device_ns * 1e-6);
  S.device_ms_prev = -1.f;
  t->num_nodes = r->num_nodes;
  t->ub_nodes = r->num_nodes;
  t->ub_alloc = r->allocated_total;
  t->ub_arena = r->arena_off;
  t->ub_dir = (long long)r->dir_top;
  t->sm_queued = 0;
  t->prev_used = r->n_voxels;
  t->last_backlog = t->sm_backlog.p;
  t->last_nv = r->n_voxels;
  t->last_ns = r->n_spill;
  const int err = r->error;
  if (r->dir_top > (unsigned long long)t->cdir.cap) {  // a relocation found no room
    RK(sync_ctrl(t));
    RK(exact_bounds(t));
  }
  return err;
}

// ---------------------------------------------------------------- C ABI

extern "C" {

const char *lod_strerror(int code) {
  switch (code) {
    case LOD_OK: return "ok";
    case LOD_E_OUT_OF_ARENA: return "arena exhausted";
    case LOD_E_SPILL_OVERFLOW: return "spill buffer past capacity";
    case LOD_E_BACKLOG_OVERFLOW: return "voxel backlog past capacity";
    case LOD_E_CUDA: return "CUDA error";
    case LOD_E_ARG: return "bad argument";
    case LOD_E_NOMEM: return "device out of memory";
    case LOD_E_NO_DEVICE: return "no CUDA device";
    default: return "unknown";
  }
}

int lod_device_count(int *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *count = n;
  return n > 0 ? LOD_OK : LOD_E_NO_DEVICE;
}

int lod_tree_create(const LodParams *params, LodTree **out) {
  if (!params || !out) return LOD_E_ARG;
  const LodParams &p = *params;
  if (p.grid_res < 2 || (p.grid_res & 1) || p.chunk_capacity <= 0 || p.arena_bytes == 0 ||
      p.max_depth < 0 || p.max_depth > 60 || p.grid_res > 1024)
    return LOD_E_ARG;
  int ndev = 0;
  if (lod_device_count(&ndev) != LOD_OK || p.device >= ndev) return LOD_E_NO_DEVICE;
  LodTree *t = new LodTree();
  t->p = p;
  t->dev = p.device;
  cudaSetDevice(t->dev);
  CK(cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking));
  {
    // keep freed scratch cached in the stream-ordered pool (growth without syncs)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, t->dev) == cudaSuccess) {
      unsigned long long thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      // Back the pool with physical memory once per device (LOD_POOL_RESERVE_MIB,
      // default 16 GiB, at most 1/8 of free HBM): scratch growth during a split
      // burst is then a pool sub-allocation instead of a page-table mapping
      // inside the update (measured: 20-27 ms first-touch stalls on 5.8M-point
      // spills; the skew stream's 20-43M-point split waves need ~10 GiB of
      // scratch: 6 -> 16 GiB took its bench from 1202 to 1362 M points/s).
      static bool warmed[64] = {};
      if (t->dev < 64 && !warmed[t->dev]) {
        warmed[t->dev] = true;
        const char *e = getenv("LOD_POOL_RESERVE_MIB");
        unsigned long long want = (e ? strtoull(e, nullptr, 10) : 16384ull) << 20;
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) want = std::min<unsigned long long>(want, fr / 8);
        void *q = nullptr;
        const auto w0 = std::chrono::steady_clock::now();
        if (want && cudaMallocAsync(&q, want, t->st) == cudaSuccess) {
          cudaFreeAsync(q, t->st);
          cudaStreamSynchronize(t->st);
          g_pool_keep[t->dev] = want;
        }
        if (lod_debug())
          fprintf(stderr, "[lod] pool reserve %.1f GiB in %.1f ms\n", want / 1073741824.0,
                  std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count());
        cudaGetLastError();
      }
    }
  }
  for (auto &e : t->ev) CK(cudaEventCreate(&e));
  Geo &g = t->geo;
  for (int k = 0; k < 3; ++k) g.bmin0[k] = p.bmin[k];
  g.size0 = p.size;
  for (int k = 0; k < 64; ++k) g.size_by_level[k] = p.size * std::pow(0.5, (double)k);
  {
    // a power-of-two root size makes every node size a power of two: then the
    // cell formula's division is an exact multiplication by 1/s
    int e = 0;
    const double m = std::frexp(p.size, &e);
    g.pow2 = (m == 0.5 && p.size >= 0x1p-900 && p.size <= 0x1p900) ? 1 : 0;
    for (int k = 0; k < 64; ++k) g.inv_by_level[k] = g.pow2 ? 1.0 / g.size_by_level[k] : 0.0;
  }
  g.g = (int)p.grid_res;
  g.grid_bytes = p.grid_res * p.grid_res * p.grid_res / 8;
  g.T = p.leaf_threshold;
  g.max_depth = (int)p.max_depth;
  g.C = p.chunk_capacity;
  g.fresh = p.arena_bytes < (1ull << 37) ? 1 : 0;  // grid offsets / 64 below 2^31 leave bit 31 free
  {
    // the count pass may descend in f32 (lod_common.cuh, the f32 twins)
    static const bool no_f32 = getenv("LOD_COUNT_F64") != nullptr;  // A/B switch
    bool ok = g.pow2 && p.grid_res >= 2 && (p.grid_res & (p.grid_res - 1)) == 0 && p.max_depth >= 0 &&
              p.max_depth <= 23 && !no_f32;
    const double q = p.size * std::ldexp(1.0, -(int)p.max_depth);
    for (int k = 0; k < 3 && ok; ++k) {
      const double r = p.bmin[k] / q, top = (p.bmin[k] + p.size) / q;
      ok = p.bmin[k] >= 0.0 && r == std::floor(r) && top <= 16777216.0 && (double)(float)p.bmin[k] == p.bmin[k];
    }
    g.f32ok = ok ? 1 : 0;
  }
  g.gmask = g.fresh ? 0x7fffffffu : 0xffffffffu;
  t->arena_cap = (p.arena_bytes + 15ull) / 16ull * 16ull;  // store.py:41-42
  if (cudaMalloc(&t->arena, t->arena_cap) != cudaSuccess) {
    cudaGetLastError();
    trim_pool(t->dev, true);
    if (cudaMalloc(&t->arena, t->arena_cap) != cudaSuccess) {
      cudaGetLastError();
      delete t;
      return LOD_E_NOMEM;
    }
  }
  CK(cudaMemsetAsync(t->arena, 0, t->arena_cap, t->st));
  RK(ensure_nodes(t, 1024, 0));
  RK(ensure_chunks(t, 1024, 0));
  {
    // Node / chunk rows a tree fed large batches gets at its first one: what
    // the arena can hold (an inner node owns a grid, a chunk C records),
    // capped at a few tens of MB.  Growth copies every column inside the
    // update that needs it (~140 us of host time per doubling of the node
    // table, measured), so a tree sized like the bench's never grows its node
    // table mid-stream; trees fed tiny batches stay small.
    const long long gsz = std::max<long long>(((long long)g.grid_bytes + 63) / 64 * 64, 64);
    t->ncap_hint = std::min<long long>(std::min<long long>(8 * ((long long)t->arena_cap / gsz) + 1, 1 << 17),
                                       max_nodes(t));
    t->ccap_hint = std::min<long long>((long long)t->arena_cap / std::max<long long>(16 * (long long)g.C, 16), 1 << 18);
  }
  CK(cudaMalloc(&t->d_ctrl, sizeof(Ctrl)));
  CK(cudaHostAlloc(&t->h_ctrl, sizeof(Ctrl), cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(&t->h_ctrl_dev, t->h_ctrl, 0));
  CK(cudaHostAlloc(&t->h_seq, sizeof(unsigned), cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(&t->h_seq_dev, t->h_seq, 0));
  *t->h_seq = 0;
  CK(cudaMemsetAsync(t->d_ctrl, 0, sizeof(Ctrl), t->st));
  memset(t->h_ctrl, 0, sizeof(Ctrl));
  lod::launch(k_init_root, 1, 1, 0, t->st, t->nd, p.bmin[0], p.bmin[1], p.bmin[2]);
  Ctrl c0{};
  c0.num_nodes = 1;
  CK(cudaMemcpyAsync(t->d_ctrl, &c0, sizeof(Ctrl), cudaMemcpyHostToDevice, t->st));
  RK(t->counter.ensure(4, t->st));
  RK(sync_ctrl(t));
  t->num_nodes = 1;
  *out = t;
  return LOD_OK;
}

int lod_tree_destroy(LodTree *t) {
  if (!t) return LOD_OK;
  cudaSetDevice(t->dev);
  cudaStreamSynchronize(t->st);
  auto f = [](void *q) { if (q) cudaFree(q); };
  f(t->arena);
  f(t->nd.parent); f(t->nd.octant); f(t->nd.level); f(t->nd.children); f(t->nd.inner);
  f(t->nd.final_); f(t->nd.count); f(t->nd.pending); f(t->nd.chunk_head); f(t->nd.chunk_tail);
  f(t->nd.chunk_count); f(t->nd.grid_off); f(t->nd.bmin); f(t->nd.desc); f(t->nd.dir_off); f(t->nd.dir_cap);
  t->cdir.release();
  f(t->pool.next); f(t->pool.payload_off); f(t->pool.occupied); f(t->pool.owner); f(t->pool.cidx);
  f(t->pool.free_stack);
  f(t->d_ctrl);
  if (t->h_ctrl) cudaFreeHost(t->h_ctrl);
  if (t->sm_ring) cudaFreeHost(t->sm_ring);
  if (t->sm_res) cudaFreeHost(t->sm_res);
  if (t->sm_done) cudaFreeHost(t->sm_done);
  f(t->sm_acc);
  t->sm_brec.release(); t->sm_srec.release(); t->sm_node_b.release(); t->sm_node_s.release();
  t->sm_tl.release(); t->sm_cand.release(); t->sm_splits.release(); t->sm_touched.release();
  t->sm_nnew.release(); t->sm_cur.release(); t->sm_wls.release(); t->sm_pl.release(); t->sm_wl.release();
  t->sm_sp.release(); t->sm_backlog.release();
  if (t->h_seq) cudaFreeHost(t->h_seq);
  t->split_list.release(); t->node_b.release(); t->node_all.release();
  t->bitmap.release(); t->scnt.release(); t->schk.release();
  t->spill_off.release(); t->chunk_off.release(); t->spill.release(); t->hslots.release(); t->hslots2.release();
  t->hused.release(); t->srank.release(); t->wcount.release(); t->wbase.release();
  t->backlog.release(); t->wins.release(); t->keys.release(); t->keys_b.release();
  t->vals_a.release(); t->vals_b.release(); t->hist.release(); t->ghist.release(); t->nodecnt.release();
  t->dmat.release(); t->dlb.release(); t->drank.release(); t->dpscan.release();
  t->dense.release();
  t->seg_node.release(); t->pairs.release(); t->wlo.release(); t->sinfo.release(); t->seg_start.release();
  t->plan.release(); t->plan_ex.release(); t->in_xyz.release();
  t->in_rgba.release(); t->in_rec.release(); t->dcopy.release(); t->gbuf.release(); t->gnodes.release(); t->goff.release(); t->gstart.release();
  t->woff.release(); t->vislist.release(); t->fb.release(); t->counter.release();
  release_scan_lb(t->lb32);
  release_scan_lb(t->lb64);
  t->dsplits.release(); t->dvnode.release(); t->dpnode.release(); t->dvstart.release(); t->dvcount.release();
  t->dpstart.release(); t->dpcount.release(); t->dvbase.release(); t->dvcell.release(); t->dvrgba.release();
  if (t->cst) cudaStreamSynchronize(t->cst);
  if (t->ev_counted) cudaEventDestroy(t->ev_counted);
  if (t->ev_aux) cudaEventDestroy(t->ev_aux);
  if (t->ev_release) cudaEventDestroy(t->ev_release);
  if (t->ev_input) cudaEventDestroy(t->ev_input);
  for (auto &sg : t->stage) {
    sg.xyz.release();
    sg.rgba.release();
    sg.rec.release();
    if (sg.ready) cudaEventDestroy(sg.ready);
  }
  if (t->cst) cudaStreamDestroy(t->cst);
  for (auto &e : t->ev) if (e) cudaEventDestroy(e);
  cudaStreamDestroy(t->st);
  const int dev = t->dev;
  delete t;
  trim_pool(dev, false);
  return LOD_OK;
}

int lod_tree_info(LodTree *t, LodTreeInfo *info) {
  if (!t || !info) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(sync_ctrl(t));
  RK(exact_bounds(t));  // between calls the published counters are exact
  const Ctrl &c = *t->h_ctrl;
  info->num_nodes = c.num_nodes;
  info->node_capacity = t->ncap;
  info->splits_total = c.splits_total;
  info->max_level = c.max_level;
  info->allocated_total = c.allocated_total;
  info->free_count = c.free_count;
  info->released_total = c.released_total;
  info->chunk_capacity_rows = t->ccap;
  info->arena_offset = c.arena_off;
  info->arena_capacity = t->arena_cap;
  info->grid_bytes = t->geo.grid_bytes;
  info->chunk_capacity = t->geo.C;
  return LOD_OK;
}

int lod_insert_batch(LodTree *t, const float *xyz, const uint32_t *rgba, int64_t n,
                     const LodLimits *limits, int flags, LodBatchStats *stats) {
  const bool packed = (flags & LOD_FLAG_PACKED) != 0;
  if (!t || n < 0 || (n > 0 && (!xyz || (!rgba && !packed)))) return LOD_E_ARG;
  LodBatchStats local{};
  LodBatchStats &S = stats ? *stats : local;
  memset(&S, 0, sizeof(S));
  S.n_batch = n;
  cudaSetDevice(t->dev);
  cudaStream_t st = t->st;
  const bool prof = (flags & LOD_FLAG_PROFILE) != 0;
  const bool delta = (flags & LOD_FLAG_DELTA) != 0;
  t->d_nsplits = t->d_nvg = t->d_npg = t->d_nv = 0;
  const long long backlog_cap = limits ? limits->backlog_capacity : 10000000LL;
  const long long spill_cap = limits ? limits->spill_capacity : 100000000LL;
  if (n == 0) {  // update.py:266-268
    fill_stats(t, &S);
    return LOD_OK;
  }
  if (n >= (1LL << 31)) return LOD_E_ARG;
  static const bool no_small = getenv("LOD_NO_SMALL") != nullptr;  // A/B switch: pipeline for every batch
  if (!no_small && n <= kSmallMaxBatch &&
      !(flags & (LOD_FLAG_DEVICE_INPUT | LOD_FLAG_PACKED | LOD_FLAG_DELTA | LOD_FLAG_PROFILE))) {
    bool handled = false;
    const int rc = small_insert(t, xyz, rgba, n, backlog_cap, spill_cap, S, &handled);
    if (handled) {
      if (rc) {  // the structure stays walkable (partial state, errors.py:1-5)
        RK(sync_ctrl(t));
        RK(exact_bounds(t));
      }
      return rc;
    }
  }
  RK(refresh(t));  // the pipeline sizes its launches from exact host copies
  if (n >= (1 << 16) && !t->sized_large) {  // first large batch
    t->sized_large = true;
    RK(ensure_nodes(t, std::max<long long>(t->ncap_hint, t->ncap), t->num_nodes));
    RK(ensure_chunks(t, std::max<long long>(t->ccap_hint, t->ccap), t->h_ctrl->allocated_total));
    // both claim tables for 16 x the batch: the re-descent after a split burst
    // (spill of several batches) then rehashes into a table that is already
    // there, instead of allocating and clearing one inside that update
    const long long H = std::min<long long>(16 * n, 1LL << 27);
    for (DBuf<HSlot> *tb : {&t->hslots, &t->hslots2}) {
      const long long old = tb->cap;
      RK(tb->ensure(H, st, 0, true));
      if (tb->cap != old) CK(cudaMemsetAsync(tb->p, 0xFF, (size_t)tb->cap * sizeof(HSlot), st));
    }
    t->h2_epoch = -1;
  }
  // device-time events: this call's pair, the previous call's kept for its
  // report when that call returned before its tail ran
  const bool prev_pending = t->tail_pending, prev_ev = t->tail_ev;
  const int prev_slot = t->ev_slot, es = t->ev_slot ^ 1;
  t->ev_slot = es;
  t->tail_pending = false;
  cudaEvent_t EB = es ? t->ev[14] : t->ev[11], EE = es ? t->ev[15] : t->ev[10];
  // Early return: once allocation has run, nothing later in the cycle can fail
  // or change what the call reports, so the host returns after the control
  // block published behind k_alloc while the sort + store + cleanup
  // still run on the tree stream (every later call and reader is ordered
  // behind them on that stream; device inputs are released to the caller's
  // stream by an event).  Not with a delta or phase profile (both read the
  // tail's results), nor for device inputs without a stream to order.
  static const bool no_early = getenv("LOD_NO_EARLY") != nullptr;  // A/B switch
  const bool early = !no_early && !prof && !delta && mapped_sync(t) &&
                     (!(flags & LOD_FLAG_DEVICE_INPUT) || ((flags & LOD_FLAG_INPUT_STREAM) && limits));
  unsigned mid_seq = 0;
  const long long C = t->geo.C;
  const long long launches0 = lod::g_launches;
  t->d2h_bytes = 0;
  S.h2d_bytes = (flags & LOD_FLAG_DEVICE_INPUT) ? 0 : 16 * n;
  float count_ms = 0.f;
  auto mark = [&](int phase) {
    if (prof) cudaEventRecord(t->ev[1 + phase], st);
  };
  // LOD_DEBUG=2: host timeline of the call (microseconds since entry)
  const bool tl = getenv("LOD_DEBUG") && atoi(getenv("LOD_DEBUG")) >= 2;
  const auto t_entry = std::chrono::steady_clock::now();
  char tlbuf[2048];
  int tlpos = 0;
  auto tp = [&](const char *what) {
    if (!tl || tlpos > 1900) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_entry).count();
    tlpos += snprintf(tlbuf + tlpos, sizeof(tlbuf) - tlpos, " %s=%.0f", what, us);
  };
  if ((flags & LOD_FLAG_INPUT_STREAM) && limits) {  // device inputs produced on the caller's stream
    // an idle caller stream has nothing to wait for (a cross-stream wait costs
    // the device ~5 us between calls even when it is already satisfied)
    const cudaStream_t in = reinterpret_cast<cudaStream_t>(limits->input_stream);
    const cudaError_t q = cudaStreamQuery(in);
    if (q != cudaSuccess) {
      if (q != cudaErrorNotReady) return cuda_rc(q);
      cudaGetLastError();
      if (!t->ev_input) CK(cudaEventCreateWithFlags(&t->ev_input, cudaEventDisableTiming));
      CK(cudaEventRecord(t->ev_input, in));
      CK(cudaStreamWaitEvent(st, t->ev_input, 0));
    }
  }
  if (prof) CK(cudaEventRecord(t->ev[0], st));
  // ---- inputs
  const float *bx = xyz;
  const uint32_t *bc = rgba;
  const float4 *brec = nullptr;  // packed 16-byte input records
  LodTree::Stage *staged = nullptr;
  if (!(flags & LOD_FLAG_DEVICE_INPUT)) {
    for (auto &sg : t->stage)
      if (sg.valid && sg.packed == packed && sg.hx == (const void *)xyz && (packed || sg.hc == rgba) && sg.n == n)
        staged = &sg;
  }
  if (staged) {  // prefetched on the copy stream: wait for it, no copy here
    // a copy not issued yet goes behind the work queued so far on the tree
    // stream: an earlier early-returning insert's tail may still read this slot
    if (staged->pending) RK(issue_pending(t, staged));
    // a copy that has already landed needs no cross-stream wait (which would
    // also break the programmatic launch into this cycle)
    const cudaError_t q = cudaEventQuery(staged->ready);
    if (q != cudaSuccess) {
      if (q != cudaErrorNotReady) return cuda_rc(q);
      cudaGetLastError();
      CK(cudaStreamWaitEvent(st, staged->ready, 0));
    }
    staged->valid = false;
    if (packed) {
      brec = staged->rec.p;
    } else {
      bx = staged->xyz.p;
      bc = staged->rgba.p;
    }
  } else if (packed) {
    if (flags & LOD_FLAG_DEVICE_INPUT) {
      brec = reinterpret_cast<const float4 *>(xyz);
    } else {
      RK(t->in_rec.ensure(n, st));
      CK(cudaMemcpyAsync(t->in_rec.p, xyz, (size_t)n * 16, cudaMemcpyHostToDevice, st));
      brec = t->in_rec.p;
    }
  } else if (!(flags & LOD_FLAG_DEVICE_INPUT)) {
    RK(t->in_xyz.ensure(3 * n, st));
    RK(t->in_rgba.ensure(n, st));
    CK(cudaMemcpyAsync(t->in_xyz.p, xyz, (size_t)n * 12, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(t->in_rgba.p, rgba, (size_t)n * 4, cudaMemcpyHostToDevice, st));
    bx = t->in_xyz.p;
    bc = t->in_rgba.p;
  }
  // a device batch (xyz + rgba arrays) with an input stream to release: the
  // first count pass copies it into packed records (staged count: off)
  static const int staged_cfg = getenv("LOD_COUNT_STAGED") ? atoi(getenv("LOD_COUNT_STAGED")) : 0;
  const bool release_early = early && (flags & LOD_FLAG_DEVICE_INPUT) && !brec && !staged_cfg;
  // events around the cycle only for the phase profile and for handing a
  // device batch back to its stream at the end (each event between two
  // kernels breaks the programmatic launch: ~6 us per call); the cycle's
  // device time comes from the Ctrl stamps otherwise
  const bool use_ev = prof || (early && (flags & LOD_FLAG_DEVICE_INPUT) && !release_early);
  if (use_ev) CK(cudaEventRecord(EB, st));  // inputs resident
  RK(issue_pending(t, nullptr, kPartSmall));  // the next batch's colours overlap the first count pass
  lod::launch(k_cycle_begin, 1, 1, 0, st, t->d_ctrl);
  // ---- expansion (update.py:273-296) with the voxel claims folded in
  RK(t->node_b.ensure(n, st));
  if (release_early) RK(t->dcopy.ensure(n, st));
  PointSrc src{nullptr, 0, bx, bc, n, brec};
  NodeOf node_of{nullptr, t->node_b.p, 0};
  long long n_all = n, n_s = 0;
  int first = 1, iters = 0;
  long long splits_cycle = 0;
  // claim table: sized from the batch and the previous cycle's claims, grown
  // (rehashed) between iterations when the next pass could overfill it; a
  // table that still fills up falls back to a separate claim pass
  {
#ifndef LOD_HASH_FACTOR_X4
#define LOD_HASH_FACTOR_X4 6  // table slots ~ 1.5 x (previous cycle's claims + batch), next power of two (A/B: 5 within 0.2 %, 8 -1.3 %)
#endif
    const long long want = std::max<long long>(LOD_HASH_FACTOR_X4 * (t->prev_used + n) / 4, 1 << 20);
    const unsigned long long H = round_slots((unsigned long long)want);
    if ((long long)H > t->hslots.cap) {
      RK(t->hslots.ensure((long long)H, st, 0, true));
      CK(cudaMemsetAsync(t->hslots.p, 0xFF, (size_t)t->hslots.cap * sizeof(HSlot), st));
    }
    t->hcap = H;
    RK(t->hused.ensure((long long)H, st));
  }
  // this cycle's epoch; the table is reset when the epochs wrap
  t->hepoch = (t->hepoch + 1) % kEpochs;
  if (t->hepoch == 0) {  // epochs wrap: both tables back to the all-ones state
    if (t->hslots.p) CK(cudaMemsetAsync(t->hslots.p, 0xFF, (size_t)t->hslots.cap * sizeof(HSlot), st));
    if (t->hslots2.p) CK(cudaMemsetAsync(t->hslots2.p, 0xFF, (size_t)t->hslots2.cap * sizeof(HSlot), st));
    t->h2_epoch = -1;
  }
  const unsigned long long htag = (unsigned long long)t->hepoch << 56;
  const int cbits = cell_bits(t->geo.g);
  Hash hs{t->hslots.p, t->hcap, t->hused.p, t->hcap, htag, cbits};
  uint32_t *grid32 = reinterpret_cast<uint32_t *>(t->arena);
  // ---- post-expansion pipeline: resolve -> backlog -> alloc -> sort+store ->
  // [delta] -> epilogue.  Launched either after the expansion settled (guard
  // null, nv = the claim count), or speculatively behind an expansion
  // iteration's k_decide (guard = Ctrl.spec_abort, nv = an upper bound): every
  // kernel then returns at once unless that decide settled the expansion, and
  // counts that only the device knows yet (new voxels) are read on the device.
  bool pipeline_launched = false;
  auto pipeline = [&](const int *guard, long long nv) -> int {
    const long long num_nodes = t->num_nodes;
    // sort scratch first: the burst resolve sorts its win list with it
    const long long n_items = n_all + nv;  // exact, or an upper bound (the device count is Ctrl.n_items)
    // the packed node plans count touched nodes in 24 bits (kPackShift)
    if (num_nodes >= (1LL << 24) && n_items >= (1LL << 24)) return LOD_E_ARG;
    const int passes = radix_passes((uint32_t)(num_nodes - 1));
    RK(t->keys.ensure(n_items, st));
    RK(t->keys_b.ensure(n_items, st));
    RK(t->vals_a.ensure(n_items, st));
    RK(t->vals_b.ensure(n_items, st));
    RK(t->hist.ensure(2 * radix_lb_elems(n_items), st));
    {
      long long oldg = t->ghist.cap, oldn = t->nodecnt.cap;
      RK(t->ghist.ensure(kMaxPasses * kRadixDigits, st));
      RK(t->nodecnt.ensure(std::max<long long>(num_nodes, t->ncap), st, oldn));
      // zero once when (re)allocated; afterwards k_seg_list / k_epilogue leave them zeroed
      if (t->ghist.cap > oldg) CK(cudaMemsetAsync(t->ghist.p, 0, (size_t)t->ghist.cap * 4, st));
      if (t->nodecnt.cap > oldn) CK(cudaMemsetAsync(t->nodecnt.p + oldn, 0, (size_t)(t->nodecnt.cap - oldn) * 4, st));
    }
    RK(t->backlog.ensure(std::max<long long>(nv, 1), st));
    static const long long winsort_min = getenv("LOD_WINSORT_MIN") ? atoll(getenv("LOD_WINSORT_MIN")) : (4LL << 20);
    if (nv > 0 && nv >= winsort_min) {  // ---- burst resolve: win list sorted by winner
      RK(t->wins.ensure(nv, st));
      const int wpasses = radix_passes((uint32_t)std::max<long long>(n_all - 1, 1));
      const long long lbw_w = radix_lb_elems(nv);
      CK(cudaMemsetAsync(t->hist.p, 0, (size_t)lbw_w * 4, st));  // pass 0's look-back words
      lod::launch(k_resolve_list, grid_for((long long)t->hcap), 256, 0, st, t->nd, hs, grid32, n_s, t->wins.p,
                  t->keys.p, wpasses, t->ghist.p, t->d_ctrl, guard);
      mark(1);
      tp("resolve_launched");
      RadixScratch rw;
      rw.keys_b = t->keys_b.p;
      rw.vals_a = t->vals_a.p;
      rw.vals_b = t->vals_b.p;
      rw.ghist = t->ghist.p;
      rw.lb[0] = t->hist.p;
      rw.lb[1] = t->hist.p + lbw_w;
      const WinSink ws{t->wins.p, t->backlog.p};
      uint32_t *wk = nullptr, *wv = nullptr;
      stable_multisplit(t->keys.p, nv, wpasses, rw, st, &wk, &wv, nullptr, 0, &ws, &t->d_ctrl->n_wins, guard);
      CK(cudaMemsetAsync(t->ghist.p, 0, (size_t)kMaxPasses * kRadixDigits * 4, st));  // the node sort's totals
    } else {
      {
        long long oldw = t->wcount.cap;  // zero when (re)allocated; k_scatter counts every entry back to zero
        RK(t->wcount.ensure(n_all, st));
        if (t->wcount.cap > oldw) CK(cudaMemsetAsync(t->wcount.p, 0, (size_t)t->wcount.cap * 4, st));
      }
      RK(t->wbase.ensure(n_all, st));
      RK(ensure_scan_lb<uint32_t>(t->lb32, n_all, st));
      // the used-slot list while the table fits L2 comfortably, else a sweep
      static const long long list_max = getenv("LOD_RESOLVE_LIST_MAX_MB")
                                            ? atoll(getenv("LOD_RESOLVE_LIST_MAX_MB")) << 20
                                            : (64LL << 20);
      const bool use_list = (long long)t->hcap * (long long)sizeof(HSlot) <= list_max;
      const unsigned rgrid = use_list ? grid_for(nv) : grid_for((long long)t->hcap);
      if (nv > 0) {
        if (use_list)
          lod::launch(k_resolve<true>, rgrid, 256, 0, st, t->nd, hs, grid32, n_s, t->wcount.p,
                      (const Ctrl *)t->d_ctrl, guard);
        else
          lod::launch(k_resolve<false>, rgrid, 256, 0, st, t->nd, hs, grid32, n_s, t->wcount.p,
                      (const Ctrl *)t->d_ctrl, guard);
      }
      mark(1);
      tp("resolve_launched");
      if (nv > 0) {
        exclusive_scan_lb<uint32_t>(t->wcount.p, t->wbase.p, n_all, &t->d_ctrl->n_v, t->lb32, st, guard);
        if (use_list)
          lod::launch(k_scatter<true>, rgrid, 256, 0, st, hs, n_s, t->wbase.p, t->wcount.p, src, t->backlog.p,
                      (const Ctrl *)t->d_ctrl, guard);
        else
          lod::launch(k_scatter<false>, rgrid, 256, 0, st, hs, n_s, t->wbase.p, t->wcount.p, src, t->backlog.p,
                      (const Ctrl *)t->d_ctrl, guard);
      }
    }
    mark(2);
    // ---- sort: every new sample by node id, stable (slot order)
    // allocation scratch (segments, chunk needs, write lists, pool rows)
    const long long Kb = num_nodes + 1;  // bound on touched nodes
    // per-node scratch follows the node table's capacity (grows with it, not
    // with every new node-count high-water mark inside an update)
    const long long Kc = std::max<long long>(Kb, t->ncap + 1);
    RK(t->seg_node.ensure(Kc, st));
    RK(t->seg_start.ensure(Kc + 1, st));
    RK(t->dense.ensure(Kc, st));
    RK(t->plan.ensure(Kc, st));
    RK(t->plan_ex.ensure(Kc, st));
    RK(ensure_scan_lb<U64x2>(t->lb64, Kc, st));
    const long long acq_bound = n_items / C + Kb + 1;
    RK(t->wlo.ensure(acq_bound + Kb + 1, st));
    RK(t->sinfo.ensure(Kc, st));
    const long long alloc0 = t->h_ctrl->allocated_total;
    RK(ensure_chunks(t, alloc0 + acq_bound + 1, alloc0));
    RK(ensure_dir(t, alloc0 + acq_bound + 1, Kb));
    const long long lbw = radix_lb_elems(n_items);
    long long *n_items_dev = &t->d_ctrl->n_items;
    // direct placement (radix.cuh) instead of the LSD multisplit when its
    // tiles x nodes matrix stays small; LOD_STORE_LSD=1 keeps the LSD sort
    static const bool store_lsd = getenv("LOD_STORE_LSD") != nullptr;
    static const long long dir_max = getenv("LOD_DIRECT_MAX_ENTRIES") ? atoll(getenv("LOD_DIRECT_MAX_ENTRIES"))
                                                                      : (8LL << 20);
    // the smallest tile (2048 items and up) whose matrix fits the cap
    int tsh = kDirTileShift;
    auto tiles_of = [&](int sh) { return (n_items + (1LL << sh) - 1) >> sh; };
    while (tsh < kDirTileShiftMax && num_nodes * tiles_of(tsh) > dir_max) ++tsh;
    const long long dtiles = tiles_of(tsh);
    const long long nn_pad = (num_nodes + 7) & ~7LL;  // matrix row stride, per-warp counters
    const bool direct = !delta && !store_lsd && nn_pad * 2 <= 49152 && num_nodes * dtiles <= dir_max &&
                        n_items < (1LL << 30);
    const long long drb = (dtiles + kDirRowBlock - 1) / kDirRowBlock;
    const long long dcb = (num_nodes + kDirScanBlock - 1) / kDirScanBlock;
    if (direct) {
      RK(t->dmat.ensure(nn_pad * dtiles, st));
      RK(t->dlb.ensure(drb * num_nodes + 1 + dcb, st));  // look-back words, ticket, plan-scan flags
      RK(t->drank.ensure(n_items, st));
      // warps per CTA: as many per-warp counter arrays as fit 48 KB
      // (LOD_DIR_W; default one warp per CTA: same-box A/B, driver range,
      // 1 warp 2596-2603 Mpts/s > 2: 2590-2593 > 4: 2560-2564 > 8: 2534)
      static const long long wenv = getenv("LOD_DIR_W") ? atoll(getenv("LOD_DIR_W")) : 1;
      const long long wfit = std::min<long long>(49152 / (nn_pad * 2), std::max<long long>(wenv, 1));
      const int W = wfit >= 8 ? 8 : wfit >= 4 ? 4 : wfit >= 2 ? 2 : 1;
      const unsigned grid = (unsigned)std::max<long long>((dtiles + W - 1) / W, 1);
      const size_t sm = (size_t)W * nn_pad * 2;
      const long long lbwd = drb * num_nodes + 1 + dcb;
      auto go = [&](auto kern) {
        lod::launch(kern, grid, 32 * W, sm, st, node_of, n_all, (const uint4 *)t->backlog.p, num_nodes, nn_pad,
                    t->keys.p, t->drank.p, t->dmat.p, t->dlb.p, lbwd, (const unsigned long long *)&t->d_ctrl->n_used,
                    n_items_dev, tsh, guard);
      };
      if (W == 8) go(k_rank_prep<8>);
      else if (W == 4) go(k_rank_prep<4>);
      else if (W == 2) go(k_rank_prep<2>);
      else go(k_rank_prep<1>);
      RK(t->dpscan.ensure(2 * dcb, st));
      const SegFinish seg{t->nd, t->geo, t->seg_node.p, t->seg_start.p, t->dense.p, t->plan.p, t->plan_ex.p, t->d_ctrl};
      lod::launch(k_tile_colscan<SegFinish>, (unsigned)std::max<long long>(drb * dcb, dcb), kDirScanBlock, 0, st,
                  t->dmat.p, num_nodes, nn_pad, dcb, drb, (const long long *)n_items_dev, t->dlb.p, seg, t->dpscan.p,
                  tsh, guard);
    } else {
      // node counts in per-CTA shared memory (16-bit counters) up to
      // kNodeHistSmemMax nodes, as long as no CTA can see 65535 items
      // kNodeHistSmemMax nodes, as long as no CTA can see 65535 items; one
      // wave: as many CTAs per SM as their histograms fit (228 KB per SM)
      long long nc_words = (num_nodes + 1) / 2;
      int bps = LOD_PREP_BPS;
      if (num_nodes <= kNodeHistSmemMax)
        bps = (int)std::max<long long>(1, std::min<long long>(LOD_PREP_BPS, 233472 / (nc_words * 4 + 1024)));
      unsigned grid = std::min<unsigned>(grid_for(n_items, kRadixBlock * kPrepItems), 148 * bps);
      if (num_nodes > kNodeHistSmemMax || n_items > (long long)grid * 65535) {
        nc_words = 0;
        grid = std::min<unsigned>(grid_for(n_items, kRadixBlock * kPrepItems), 148 * kPrepBlocksPerSM);
      }
      static bool smem_attr[64] = {};  // per device
      if (t->dev < 64 && !smem_attr[t->dev]) {
        CK(cudaFuncSetAttribute(k_radix_prep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(kNodeHistSmemMax / 2 * 4)));
        smem_attr[t->dev] = true;
      }
      lod::launch(k_radix_prep, grid, kRadixBlock, (size_t)nc_words * 4, st, node_of, n_all, t->backlog.p, nc_words,
                  t->keys.p, t->nodecnt.p, t->hist.p, lbw, &t->d_ctrl->n_used, n_items_dev, guard);
    }  // direct / LSD prep
    RK(t->pairs.ensure(Kc, st));
    if (!direct)  // (direct: the column scan wrote the plans)
      lod::launch(k_radix_ghist<NodePlanOf>, std::min<unsigned>(grid_for(num_nodes), 64), 256, 0, st, t->nodecnt.p,
                num_nodes, passes, t->ghist.p, t->pairs.p, NodePlanOf{t->nd, t->geo}, guard);
    // ---- allocation (update.py:317-331): touched nodes = nodes with new samples, ascending id.
    // It needs only the per-node counts, so it runs before the sort, whose last
    // pass then writes every record straight into its chunk slot.
    // one scan of the packed node plans: dense ids, segment starts, acquisition
    // and write-list starts (k_seg_list unpacks them per touched node)
    if (!direct)  // (direct: the column scan scanned and unpacked the plans)
      exclusive_scan_lb<U64x2>(t->pairs.p, t->pairs.p, num_nodes, &t->d_ctrl->pack_tot, t->lb64, st, guard);
    if (!direct)
      lod::launch(k_seg_list, grid_for(num_nodes), 256, 0, st, t->nd, t->geo, t->nodecnt.p, num_nodes, t->pairs.p,
                t->seg_node.p, t->seg_start.p, t->dense.p, t->plan.p, t->plan_ex.p, t->d_ctrl, guard);
    lod::launch(k_alloc, std::max(grid_for(Kb), grid_for(acq_bound)), 256, 0, st, t->nd, t->pool, t->geo,
                t->seg_node.p, t->seg_start.p, t->plan.p, t->plan_ex.p, t->wlo.p, t->sinfo.p, t->d_ctrl,
                t->arena_cap, guard);
    // the early return's publication: the sort's first pass starts without
    // waiting for its host write (publish_ctrl release + first_nowait)
    const bool release = early && !prof;
    if (early) mid_seq = publish_ctrl(t, release);
    mark(3);
    tp("alloc_launched");
    // ---- sort + store (update.py:357-373): stable by node id = slot order
    RadixScratch rs;
    rs.keys_b = t->keys_b.p;
    rs.vals_a = t->vals_a.p;
    rs.vals_b = t->vals_b.p;
    rs.ghist = t->ghist.p;
    rs.lb[0] = t->hist.p;
    rs.lb[1] = t->hist.p + lbw;
    const StoreSink sink{t->nd, t->pool, t->geo, t->arena, t->sinfo.p, t->wlo.p, n_all, src, t->backlog.p, t->d_ctrl};
    uint32_t *skeys = nullptr, *svals = nullptr;
    if (direct) {
      lod::launch(k_store_direct, grid_for(n_items), 256, 0, st, sink, (const uint32_t *)t->keys.p,
                  (const uint16_t *)t->drank.p, (const uint32_t *)t->dmat.p, nn_pad, tsh, (const long long *)n_items_dev,
                  guard, release ? 1 : 0);
    } else if (delta) {  // the delta reads the sorted order: materialise it, then store
      stable_multisplit(t->keys.p, n_items, passes, rs, st, &skeys, &svals, nullptr, 0, (const KVSink *)nullptr,
                        n_items_dev, guard);
      lod::launch(k_store, grid_for(n_items), 256, 0, st, sink, skeys, svals, (const long long *)n_items_dev, guard);
    } else {
      stable_multisplit(t->keys.p, n_items, passes, rs, st, &skeys, &svals, nullptr, 0, &sink, n_items_dev, guard,
                        release);
    }
    mark(4);
    tp("sort_launched");
    if (delta) {  // ---- BatchDelta (update.py:333-355), before the counts advance
      RK(t->dvnode.ensure(Kb, st));
      RK(t->dvstart.ensure(Kb, st));
      RK(t->dvcount.ensure(Kb, st));
      RK(t->dpnode.ensure(Kb, st));
      RK(t->dpstart.ensure(Kb, st));
      RK(t->dpcount.ensure(Kb, st));
      RK(t->dvbase.ensure(Kb, st));
      RK(t->dvcell.ensure(std::max<long long>(nv, 1), st));
      RK(t->dvrgba.ensure(std::max<long long>(nv, 1), st));
      lod::launch(k_delta_segs, 1, kDeltaBlock, 0, st, t->nd, t->seg_node.p, t->seg_start.p, t->dvnode.p,
                  t->dvstart.p, t->dvcount.p, t->dpnode.p, t->dpstart.p, t->dpcount.p, t->dvbase.p, t->d_ctrl, guard);
      if (nv > 0)
        lod::launch(k_delta_vox, grid_for(n_items), 256, 0, st, skeys, svals, t->dense.p, t->seg_start.p,
                    t->dvbase.p, n_all, t->backlog.p, t->dvcell.p, t->dvrgba.p, t->d_ctrl, guard);
    }
    mark(5);
    // ---- cleanup (update.py:375-380)
    lod::launch(k_epilogue, grid_for(Kb * 32), 256, 0, st, t->nd, t->pool, t->seg_node.p, t->seg_start.p, t->plan.p,
                t->plan_ex.p, t->d_ctrl, t->ghist.p, guard, t->geo.fresh);
    return LOD_OK;
  };
  // speculate on "this iteration settles the expansion" from the second
  // iteration on (the first usually splits), or from the first when the last
  // cycle needed a single one; never while profiling (phase events)
  static const bool no_spec = getenv("LOD_NO_SPEC") != nullptr;
  long long spec_used = 0;    // claims after the last synced iteration
  long long spec_redesc = 0;  // points the next count pass re-descends (each claims at most one cell)
  const bool may_speculate = !prof && !no_spec;
  for (;;) {
    ++iters;
    if (prof) cudaEventRecord(t->ev[12], st);
    // iteration 1 (batch points from the root): the TMA-staged count pass on
    // request (LOD_COUNT_STAGED=1; batch 16-byte aligned, >= one full tile).
    // Off by default: same-box A/B on the terrain stream, count phase 0.183 ms
    // staged vs 0.177 ms with direct loads (k_count_staged's comment)
    static const int staged_mode = getenv("LOD_COUNT_STAGED") ? atoi(getenv("LOD_COUNT_STAGED")) : 0;
    const bool aligned = brec ? ((uintptr_t)brec % 16 == 0)
                              : ((uintptr_t)bx % 16 == 0 && (uintptr_t)bc % 16 == 0);
    if (first && staged_mode && aligned && n_all >= kCountTile) {
      const unsigned g = (unsigned)((n_all + kCountTile - 1) / kCountTile);  // one tile per CTA
      if (brec)
        lod::launch(k_count_staged<true>, g, kCountTile, 0, st, t->nd, t->geo, src, node_of, n_all, grid32, hs,
                    t->d_ctrl);
      else
        lod::launch(k_count_staged<false>, g, kCountTile, 0, st, t->nd, t->geo, src, node_of, n_all, grid32, hs,
                    t->d_ctrl);
    } else {
      if (t->geo.f32ok)
        lod::launch(k_count<float>, grid_for(n_all), 256, 0, st, t->nd, t->geo, src, node_of, n_all, first, grid32,
                    hs, t->d_ctrl, (first && release_early) ? t->dcopy.p : (float4 *)nullptr);
      else
        lod::launch(k_count<double>, grid_for(n_all), 256, 0, st, t->nd, t->geo, src, node_of, n_all, first, grid32,
                    hs, t->d_ctrl, (first && release_early) ? t->dcopy.p : (float4 *)nullptr);
    }
    if (first && release_early) {
      // the caller's xyz / rgba are no longer read: its stream may go on
      // (the next call's input handshake then finds it long satisfied)
      if (!t->ev_release) CK(cudaEventCreateWithFlags(&t->ev_release, cudaEventDisableTiming));
      CK(cudaEventRecord(t->ev_release, st));
      CK(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(limits->input_stream), t->ev_release, 0));
      src.bxyz = nullptr;
      src.brgba = nullptr;
      src.brec = t->dcopy.p;
    }
    if (prof) cudaEventRecord(t->ev[13], st);
    // a speculative pipeline's host-side sizes: nodes as of now (no further
    // split if it runs); new voxels at most the claims so far + one per
    // re-descending point (known after an iteration), else the claim table's
    // capacity -- k_decide stands the pipeline down past that bound (or past
    // backlog_capacity; the host path then decides)
    const bool speculate = may_speculate && (iters >= 2 || t->last_iters == 1);
    const long long nv_bound = iters >= 2 ? std::min<long long>((long long)t->hcap, spec_used + spec_redesc)
                                          : (long long)t->hcap;
    // without a speculative pipeline behind it the host reads this decision
    // next: k_decide publishes it itself (no k_publish launch on the path)
    const bool fused_pub = !speculate && mapped_sync(t);
    const unsigned dec_seq = fused_pub ? ++t->seq : 0u;
    if (fused_pub) t->d2h_bytes += (long long)sizeof(Ctrl);
    // ... and the split's execution is launched behind it before the host
    // has read it: it runs iff the decision splits and its children and spill
    // fit the buffers as allocated (Ctrl.exec_go; else the host launches it)
    const bool spec_exec = fused_pub && !prof;
    const long long spill_buf = spec_exec ? std::min<long long>(t->spill.cap, t->node_all.cap) : -1;
    lod::launch(k_decide, (unsigned)std::min<long long>(std::max<long long>((t->num_nodes + kDecideBlock - 1) / kDecideBlock, 1), 148LL * 2),
                kDecideBlock, 0, st, t->nd, t->geo, t->bitmap.p, t->split_list.p, t->srank.p,
                t->scnt.p, t->schk.p, t->spill_off.p, t->chunk_off.p, t->d_ctrl, spill_cap, t->arena_cap,
                std::min<long long>(backlog_cap, nv_bound), fused_pub ? t->h_ctrl_dev : (Ctrl *)nullptr,
                fused_pub ? (volatile unsigned *)t->h_seq_dev : (volatile unsigned *)nullptr, dec_seq, spill_buf,
                spec_exec ? t->ncap : -1LL, (long long)t->num_nodes);
    if (spec_exec) {
      lod::launch(k_exec_chunks, 148u * 8u, 256, 0, st, t->nd, t->pool, t->geo, t->arena, t->split_list.p, -1LL,
                  t->spill_off.p, t->chunk_off.p, -1LL, t->spill.p, t->node_all.p, t->d_ctrl);
      lod::launch(k_exec_nodes, 148u * 2u, 256, 0, st, t->nd, t->geo, t->split_list.p, t->srank.p, -1LL,
                  t->d_ctrl);
    }
    if (speculate) {
      if (first) RK(issue_pending(t));  // queued batches' copies overlap the speculative pipeline
      RK(pipeline(&t->d_ctrl->spec_abort, nv_bound));
      if (use_ev) CK(cudaEventRecord(EE, st));
      pipeline_launched = true;
    }
    tp("pre_sync");
    if (pipeline_launched && early) {
      RK(wait_ctrl(t, mid_seq));
    } else if (fused_pub) {
      if (first) RK(issue_pending(t));  // queued batches' copies start behind the publication
      RK(wait_ctrl(t, dec_seq));
      t->ub_dir = (long long)t->h_ctrl->dir_top;  // as sync_ctrl: published behind all queued work
    } else {
      RK(sync_ctrl(t, first && !speculate));  // queued batches' copies start behind the publication
    }
    tp("sync");
    if (prof) {
      float x = 0.f;
      cudaEventElapsedTime(&x, t->ev[12], t->ev[13]);
      count_ms += x;
    }
    const Ctrl &h = *t->h_ctrl;
    spec_used = (long long)h.n_used;
    spec_redesc = h.redescend;
    if (h.error) return abort_cycle(t, h.error);
    const long long ns = h.n_splits;
    if (ns == 0) break;  // settled (a speculative pipeline ran iff spec_abort == 0)
    pipeline_launched = false;  // the speculative pipeline (if any) stood down
    splits_cycle += ns;
    if (delta) {  // events.append(("split", nid)) in split order (update.py:240-245)
      RK(t->dsplits.ensure(t->d_nsplits + ns, st, t->d_nsplits));
      CK(cudaMemcpyAsync(t->dsplits.p + t->d_nsplits, t->split_list.p, (size_t)ns * 4, cudaMemcpyDeviceToDevice, st));
      t->d_nsplits += ns;
    }
    const bool exec_ran = spec_exec && h.exec_go;  // (then no buffer below grows)
    // capacity for the new children and the spill segment
    RK(ensure_nodes(t, h.num_nodes, h.plan_num_nodes0));
    tp("nodes_ok");
    if (h.spill_add > 0) {
      if (!first) return abort_cycle(t, LOD_E_ARG);  // only iteration 1 can spill (update.py:9-11)
      RK(t->spill.ensure(h.spill_total, st));
      RK(t->node_all.ensure(h.spill_total, st));
      tp("spill_ok");
      const long long xchunks = h.free_count - h.plan_free0;  // chunks of the splitting nodes
      if (!exec_ran)
        lod::launch(k_exec_chunks, (unsigned)std::min<long long>(std::max<long long>(xchunks, 1), 148LL * 16), 256, 0,
                    st, t->nd, t->pool, t->geo, t->arena,
                    t->split_list.p, ns, t->spill_off.p, t->chunk_off.p, xchunks, t->spill.p, t->node_all.p,
                    t->d_ctrl);
    }
    if (!exec_ran)
      lod::launch(k_exec_nodes, grid_for(8 * ns), 256, 0, st, t->nd, t->geo, t->split_list.p, t->srank.p, ns,
                  t->d_ctrl);
    t->num_nodes = h.num_nodes;
    tp("exec_launched");
    if (first) {
      n_s = h.spill_total;
      if (n_s > 0) {
        node_of.spill = t->node_all.p;
        node_of.ns = n_s;
        src.spill = t->spill.p;
        src.ns = n_s;
      }
      n_all = n_s + n;
      first = 0;
    }
    // the next pass claims at most one cell per re-descending point (the
    // points of the nodes that just split)
    if ((long long)h.n_used + h.redescend > (long long)(3 * t->hcap / 4)) {
      const unsigned long long H = round_slots((unsigned long long)(2 * ((long long)h.n_used + h.redescend)));
      if (lod_debug()) fprintf(stderr, "[lod] claim table grow %llu -> %llu (rehash %llu)\n", t->hcap, H, h.n_used);
      // the spare table needs no clearing: k_rehash installs over stale
      // slots like the claims do -- unless it is fresh memory, or still holds
      // this cycle's keys (a second rehash in one cycle)
      const long long old2 = t->hslots2.cap;
      RK(t->hslots2.ensure((long long)H, st, 0, true));
      if (t->hslots2.cap != old2 || t->h2_epoch == (int)t->hepoch)
        CK(cudaMemsetAsync(t->hslots2.p, 0xFF, (size_t)t->hslots2.cap * sizeof(HSlot), st));
      RK(t->hused.ensure((long long)H, st, (long long)h.n_used));
      Hash nh{t->hslots2.p, H, t->hused.p, H, htag, cbits};
      lod::launch(k_rehash, grid_for(std::max<long long>((long long)h.n_used, 1)), 256, 0, st, t->hslots.p, nh, t->d_ctrl);
      // the old table keeps this cycle's keys: stale from the next cycle on
      t->h2_epoch = (int)t->hepoch;
      std::swap(t->hslots, t->hslots2);
      t->hcap = H;
      hs = nh;
      tp("rehashed");
    }
  }
  mark(0);
  tp("expand_done");
  Ctrl h1 = *t->h_ctrl;
  t->num_nodes = h1.num_nodes;
  // a pipeline launched behind the settling decide has already run (the sync
  // waited for it) unless the claims overflowed, which the host handles here
  if (pipeline_launched && h1.spec_abort) pipeline_launched = false;
  t->spec_hits += pipeline_launched ? 1 : 0;
  if (!pipeline_launched) {
    // ---- resolve the claims (update.py:298-315)
    const int D = (int)std::max<long long>(h1.max_level, 1);
    if (h1.hash_overflow) {
      if (lod_debug())
        fprintf(stderr, "[lod] claim table overflow (H=%llu, used>=%llu): fallback pass\n", t->hcap, h1.n_used);
      // fallback: clean table sized by the reference's backlog bound, full claim pass
      const long long bound = std::min<long long>(n_all * D, backlog_cap + 1);
      const unsigned long long H = round_slots((unsigned long long)std::max<long long>(2 * bound, 1 << 20));
      if ((long long)H > t->hslots.cap) RK(t->hslots.ensure((long long)H, st, 0, true));
      CK(cudaMemsetAsync(t->hslots.p, 0xFF, (size_t)t->hslots.cap * sizeof(HSlot), st));
      t->hcap = H;
      RK(t->hused.ensure(bound + 1, st));
      hs = Hash{t->hslots.p, t->hcap, t->hused.p, (unsigned long long)bound + 1, htag, cbits};
      CK(cudaMemsetAsync(&t->d_ctrl->n_used, 0, 8, st));
      CK(cudaMemsetAsync(&t->d_ctrl->hash_overflow, 0, 4, st));
      lod::launch(k_claim, grid_for(n_all), 256, 0, st, t->nd, t->geo, src, grid32, n_all, hs, t->d_ctrl);
      RK(sync_ctrl(t));
      h1 = *t->h_ctrl;
    }
    if ((long long)h1.n_used > backlog_cap) return abort_cycle(t, LOD_E_BACKLOG_OVERFLOW);  // update.py:311-312
    if (h1.hash_overflow) return abort_cycle(t, LOD_E_NOMEM);
    RK(pipeline(nullptr, (long long)h1.n_used));
    mark(6);
    if (use_ev) CK(cudaEventRecord(EE, st));
    tp("all_launched");
    if (early) RK(wait_ctrl(t, mid_seq));
    else RK(sync_ctrl(t));
    tp("final_sync");
  }
  if (tl) fprintf(stderr, "[lod] timeline%s\n", tlbuf);
  t->last_iters = iters;
  const Ctrl &h3 = *t->h_ctrl;
  if (h3.error) return abort_cycle(t, h3.error);
  const long long n_v = (long long)h3.n_used;
  t->prev_used = n_v;
  if (delta) {
    t->d_nvg = h3.d_nvg;
    t->d_npg = h3.d_npg;
    t->d_nv = n_v;
  }
  S.n_spill = n_s;
  S.launches = lod::g_launches - launches0;
  S.d2h_bytes = t->d2h_bytes;
  S.n_voxels = n_v;
  S.n_splits = splits_cycle;
  S.iterations = iters;
  fill_stats(t, &S);
  RK(exact_bounds(t));  // the counters published behind k_alloc are final
  t->ingested += n;
  t->last_backlog = t->backlog.p;
  t->last_nv = n_v;
  t->last_ns = n_s;
  float ms = -1.f;
  if (early) {  // the tail is still running: its time is reported by the next call / lod_tree_wait
    t->tail_pending = true;
    t->tail_ev = use_ev;
    // the store re-reads the batch: the caller's stream waits for the tail.
    // (Releasing it by an event recorded right after the store instead broke
    // the programmatic dependent launch into the epilogue, +5 us, and the
    // call-to-call gap stayed ~10 us: measured with tools/kineto_gaps.py.)
    if ((flags & LOD_FLAG_DEVICE_INPUT) && !release_early)
      CK(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(limits->input_stream), EE, 0));
  } else if (use_ev) {
    cudaEventElapsedTime(&ms, EB, EE);
  } else {  // settled: the final publication carries this cycle's stamps
    ms = stamp_ms(h3.t_begin, h3.t_end);
  }
  S.device_ms = ms;
  S.device_ms_prev = -1.f;
  if (prev_pending) {  // queued before this call's last publication: complete by now
    if (prev_ev) {
      cudaEvent_t pb = prev_slot ? t->ev[14] : t->ev[11], pe = prev_slot ? t->ev[15] : t->ev[10];
      if (cudaEventQuery(pe) == cudaSuccess) cudaEventElapsedTime(&S.device_ms_prev, pb, pe);
      else cudaGetLastError();
    } else {  // this cycle's k_cycle_begin kept the previous cycle's stamps
      S.device_ms_prev = stamp_ms(h3.t_prev_begin, h3.t_prev_end);
    }
  }
  if (lod_debug())
    fprintf(stderr, "[lod] batch n=%lld n_s=%lld n_v=%lld iters=%d splits=%lld nodes=%lld %.3f ms\n", (long long)n,
            n_s, n_v, iters, splits_cycle, (long long)S.num_nodes, ms);
  if (prof) {
    // phases: count, split, resolve, backlog, alloc, sort (+ store), delta, epilogue, h2d, total
    float h2d = 0.f;
    cudaEventElapsedTime(&h2d, t->ev[0], EB);
    cudaEvent_t prev = EB;
    float seg[7];
    for (int k = 0; k < 7; ++k) {
      seg[k] = 0.f;
      cudaEventElapsedTime(&seg[k], prev, t->ev[1 + k]);
      prev = t->ev[1 + k];
    }
    S.phase_ms[0] = count_ms;
    S.phase_ms[1] = seg[0] - count_ms;
    for (int k = 1; k < 7; ++k) S.phase_ms[1 + k] = seg[k];
    S.phase_ms[8] = h2d;
    S.phase_ms[9] = ms;
  }
  return LOD_OK;
}

// Device time of an early-returned cycle whose tail has finished (the stream
// is idle): its event pair, or the Ctrl stamps (one publication).
static int tail_ms(LodTree *t, float *ms) {
  if (t->tail_ev) {
    cudaEventElapsedTime(ms, t->ev_slot ? t->ev[14] : t->ev[11], t->ev_slot ? t->ev[15] : t->ev[10]);
    return LOD_OK;
  }
  RK(sync_ctrl(t));
  *ms = stamp_ms(t->h_ctrl->t_begin, t->h_ctrl->t_end);
  return LOD_OK;
}

int lod_tree_settle(LodTree *t, LodSettleStats *out) {
  if (!t || !out) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  memset(out, 0, sizeof(*out));
  CK(cudaStreamSynchronize(t->st));
  float ms = 0.f;
  if (t->tail_pending) {
    float x = 0.f;
    RK(tail_ms(t, &x));
    if (x > 0.f) ms += x;  // (-1: an aborted cycle left no end stamp)
    t->tail_pending = false;
  }
  if (t->sm_acc && t->sm_unfolded) {
    SmallAccum acc;
    CK(cudaMemcpy(&acc, t->sm_acc, sizeof(acc), cudaMemcpyDeviceToHost));
    CK(cudaMemset(t->sm_acc, 0, sizeof(acc)));
    out->calls = acc.calls;
    out->n_voxels = acc.nv_sum;
    out->n_voxels_max = acc.nv_max;
    out->n_spill_max = acc.ns_max;
    out->n_splits = acc.splits_sum;
    out->error = acc.error;
    ms += (float)(acc.device_ns * 1e-6);
  }
  t->sm_unfolded = 0;
  RK(sync_ctrl(t));
  RK(exact_bounds(t));
  out->num_nodes = t->h_ctrl->num_nodes;
  out->splits_total = t->h_ctrl->splits_total;
  out->max_level = t->h_ctrl->max_level;
  out->device_ms = ms;
  return out->error;
}

int lod_tree_wait(LodTree *t, float *last_device_ms) {
  if (!t) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  CK(cudaStreamSynchronize(t->st));
  RK(refresh(t));
  float ms = -1.f;
  if (t->tail_pending) {
    RK(tail_ms(t, &ms));
    t->tail_pending = false;
  }
  if (last_device_ms) *last_device_ms = ms;
  return LOD_OK;
}

int lod_read_nodes(LodTree *t, int64_t n, int32_t *parent, uint8_t *octant, int32_t *level,
                   int32_t *children, uint8_t *inner, uint8_t *final_, int64_t *count, int64_t *pending,
                   int32_t *chunk_head, int32_t *chunk_tail, int32_t *chunk_count, int64_t *grid_off,
                   double *bmin) {
  if (!t || n < 0 || n > t->ncap) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  cudaStream_t st = t->st;
  auto cp = [&](void *dst, const void *src, size_t bytes) -> int {
    if (dst && bytes) return cuda_rc(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    return LOD_OK;
  };
  RK(cp(parent, t->nd.parent, n * 4));
  RK(cp(octant, t->nd.octant, n));
  RK(cp(level, t->nd.level, n * 4));
  RK(cp(children, t->nd.children, n * 32));
  RK(cp(inner, t->nd.inner, n));
  RK(cp(final_, t->nd.final_, n));
  RK(cp(count, t->nd.count, n * 8));
  RK(cp(pending, t->nd.pending, n * 8));
  RK(cp(chunk_head, t->nd.chunk_head, n * 4));
  RK(cp(chunk_tail, t->nd.chunk_tail, n * 4));
  RK(cp(chunk_count, t->nd.chunk_count, n * 4));
  RK(cp(grid_off, t->nd.grid_off, n * 8));
  RK(cp(bmin, t->nd.bmin, n * 24));
  CK(cudaStreamSynchronize(st));
  return LOD_OK;
}

int lod_read_pool(LodTree *t, int64_t n, int32_t *next, int64_t *payload_off, int32_t *occupied,
                  int32_t *free_list, int64_t n_free) {
  if (!t || n < 0 || n > t->ccap || n_free < 0 || n_free > t->ccap) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  cudaStream_t st = t->st;
  if (next && n) CK(cudaMemcpyAsync(next, t->pool.next, n * 4, cudaMemcpyDeviceToHost, st));
  if (payload_off && n) CK(cudaMemcpyAsync(payload_off, t->pool.payload_off, n * 8, cudaMemcpyDeviceToHost, st));
  if (occupied && n) CK(cudaMemcpyAsync(occupied, t->pool.occupied, n * 4, cudaMemcpyDeviceToHost, st));
  if (free_list && n_free)
    CK(cudaMemcpyAsync(free_list, t->pool.free_stack, n_free * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return LOD_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- replicated top nodes

// The last cycle's new voxels at nodes above `max_level`, with their winner's
// batch position (all-array index - spill length): compacted, unordered.
__global__ void k_last_voxels(NodeCols nd, const uint4 *__restrict__ backlog, long long nv, int max_level,
                              long long n_s, long long cap, int32_t *node, uint32_t *cell, uint32_t *rgba,
                              long long *winner, unsigned long long *count) {
  lod::pdl_wait();
  for (long long i = gtid(); i < nv; i += gstride()) {
    const uint4 e = backlog[i];
    if (nd.level[e.x] >= max_level) continue;
    const unsigned long long k = atomicAdd(count, 1ull);
    if ((long long)k >= cap) continue;
    node[k] = (int32_t)e.x;
    cell[k] = e.y;
    rgba[k] = e.z;
    winner[k] = (long long)e.w - n_s;
  }
}

// lod_last_voxels_log: append the last cycle's voxels at nodes of level <
// max_level to a device log (node, cell, rgba, order key = key_base + the
// winner's batch position mapped through `gidx`, when given).
__global__ void k_last_voxels_log(NodeCols nd, const uint4 *__restrict__ backlog, long long nv, int max_level,
                                  long long n_s, const long long *__restrict__ gidx, long long key_base,
                                  int32_t *node, uint32_t *cell, uint32_t *rgba, long long *key, long long cap,
                                  unsigned long long *count) {
  lod::pdl_wait();
  for (long long i = gtid(); i < nv; i += gstride()) {
    const uint4 e = backlog[i];
    if (nd.level[e.x] >= max_level) continue;
    const unsigned long long k = atomicAdd(count, 1ull);
    if ((long long)k >= cap) continue;
    const long long w = (long long)e.w - n_s;
    node[k] = (int32_t)e.x;
    cell[k] = e.y;
    rgba[k] = e.z;
    key[k] = key_base + (gidx ? gidx[w] : w);
  }
}

// Rewrite / extend the voxel sequences of listed nodes (lod_merge_voxels):
// one warp per group; lane 0 links the chunks the longer sequence needs
// (acquisitions numbered by an atomic counter: LIFO free stack first, then
// arena cuts, k_merge_finish settles the counters), the warp writes the
// records and sets the cells' grid bits.
__global__ void k_merge_groups(NodeCols nd, PoolCols pool, Geo geo, uint8_t *arena, long long n_groups,
                               const int32_t *__restrict__ gnode, const long long *__restrict__ gstart,
                               const long long *__restrict__ goff, const uint32_t *__restrict__ cell,
                               const uint32_t *__restrict__ rgba, Ctrl *c, unsigned long long *acq,
                               unsigned long long arena_cap) {
  lod::pdl_wait();
  const long long warp = gtid() >> 5, nw = gstride() >> 5;
  const int lane = threadIdx.x & 31;
  const long long F = c->free_count, A = c->allocated_total, C = geo.C;
  const unsigned long long base = (c->arena_off + 15ull) / 16ull * 16ull;
  uint32_t *grid32 = reinterpret_cast<uint32_t *>(arena);
  for (long long g = warp; g < n_groups; g += nw) {
    const int nid = gnode[g];
    const long long start = gstart[g], len = goff[g + 1] - goff[g], cnt1 = start + len;
    if (lane == 0) {
      const long long cc = nd.chunk_count[nid], need = ceil_div(cnt1, C) - cc;
      if (need > 0) {
        const long long a0 = (long long)atomicAdd(acq, (unsigned long long)need);
        auto cid_of = [&](long long a) { return a < F ? pool.free_stack[F - 1 - a] : (int)(A + (a - F)); };
        int tail = nd.chunk_tail[nid];
        for (long long q = 0; q < need; ++q) {
          const long long a = a0 + q;
          const int cid = cid_of(a);
          if (a >= F) {
            const unsigned long long off = base + (unsigned long long)(a - F) * (unsigned long long)C * 16ull;
            if (off + (unsigned long long)C * 16ull > arena_cap) c->error = 1;  // LOD_E_OUT_OF_ARENA
            pool.payload_off[cid] = (long long)off;
          }
          pool.next[cid] = LOD_NO_CHUNK;
          pool.owner[cid] = nid;
          pool.cidx[cid] = (int)(cc + q);
          if (tail != LOD_NO_CHUNK) pool.next[tail] = cid;
          else nd.chunk_head[nid] = cid;
          tail = cid;
        }
        nd.chunk_tail[nid] = tail;
        nd.chunk_count[nid] = (int)(cc + need);
        dir_append(nd, pool, &c->dir_top, nid, need, [&](long long q) { return cid_of(a0 + q); });
      }
    }
    __syncwarp();
    const long long off0 = nd.dir_off[nid];
    const double step = geo.size_by_level[nd.level[nid]] / (double)geo.g;
    const double b0 = nd.bmin[3 * nid], b1 = nd.bmin[3 * nid + 1], b2 = nd.bmin[3 * nid + 2];
    const long long gg = geo.g;
    for (long long i = lane; i < len; i += 32) {
      const long long slot = start + i, cl = cell[goff[g] + i];
      const long long cx = cl % gg, cy = (cl / gg) % gg, cz = cl / (gg * gg);
      const float4 rec = make_float4(__double2float_rn(b0 + ((double)cx + 0.5) * step),
                                     __double2float_rn(b1 + ((double)cy + 0.5) * step),
                                     __double2float_rn(b2 + ((double)cz + 0.5) * step),
                                     __uint_as_float(rgba[goff[g] + i]));
      const int cid = pool.cdir[off0 + slot / C];
      reinterpret_cast<float4 *>(arena + pool.payload_off[cid])[slot % C] = rec;
      atomicOr(grid32 + (nd.grid_off[nid] >> 2) + (cl >> 5), 1u << (cl & 31));
    }
    __syncwarp();
    if (lane == 0) {
      for (long long pos = start / C; pos * C < cnt1; ++pos)  // occupancy of the rewritten chunks
        pool.occupied[pool.cdir[off0 + pos]] = (int)min(C, cnt1 - pos * C);
      nd.count[nid] = cnt1;
    }
  }
}

__global__ void k_merge_finish(Ctrl *c, const unsigned long long *acq, unsigned long long arena_cap, Geo geo) {
  lod::pdl_wait();
  const long long M = (long long)*acq, F = c->free_count;
  const long long fresh = M > F ? M - F : 0;
  if (fresh > 0) {
    const unsigned long long end =
        (c->arena_off + 15ull) / 16ull * 16ull + (unsigned long long)fresh * (unsigned long long)geo.C * 16ull;
    if (end > arena_cap) c->error = 1;
    else c->arena_off = end;
  }
  c->free_count = F - (M < F ? M : F);
  c->allocated_total += fresh;
}

extern "C" {

int lod_last_voxels(LodTree *t, int32_t max_level, int64_t capacity, int32_t *node, uint32_t *cell, uint32_t *rgba,
                    int64_t *winner, int64_t *n) {
  if (!t || !n || capacity < 0 || (capacity > 0 && (!node || !cell || !rgba || !winner))) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  if (!t->last_backlog && t->last_nv) return LOD_E_ARG;
  cudaStream_t st = t->st;
  const long long nv = t->last_backlog ? t->last_nv : 0;
  RK(t->counter.ensure(4, st));
  RK(t->gnodes.ensure(std::max<long long>(capacity, 1), st));
  RK(t->goff.ensure(std::max<long long>(capacity, 1), st));
  RK(t->dvcell.ensure(std::max<long long>(2 * capacity, 1), st));
  unsigned long long *cnt = t->counter.p + 2;
  CK(cudaMemsetAsync(cnt, 0, 8, st));
  if (nv)
    lod::launch(k_last_voxels, grid_for(nv), 256, 0, st, t->nd, t->last_backlog, nv, (int)max_level, t->last_ns,
                (long long)capacity, t->gnodes.p, t->dvcell.p, t->dvcell.p + std::max<long long>(capacity, 1),
                t->goff.p, cnt);
  unsigned long long k = 0;
  CK(cudaMemcpyAsync(&k, cnt, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *n = (int64_t)k;
  if ((long long)k > capacity) return capacity == 0 ? LOD_OK : LOD_E_ARG;  // query: *n is the size
  if (k) {
    CK(cudaMemcpyAsync(node, t->gnodes.p, k * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(cell, t->dvcell.p, k * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rgba, t->dvcell.p + std::max<long long>(capacity, 1), k * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(winner, t->goff.p, k * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return LOD_OK;
}

int lod_last_voxels_count(LodTree *t, int32_t max_level, int64_t *dev_count, void *stream) {
  if (!t || !dev_count) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  cudaStream_t st = t->st;
  if (!t->last_backlog && t->last_nv) {  // a queued small cycle: unknown
    CK(cudaMemsetAsync(dev_count, 0xFF, 8, st));
  } else {
    CK(cudaMemsetAsync(dev_count, 0, 8, st));
    const long long nv = t->last_backlog ? t->last_nv : 0;
    if (nv)  // counting only (capacity 0: nothing is written)
      lod::launch(k_last_voxels, grid_for(nv), 256, 0, st, t->nd, t->last_backlog, nv, (int)max_level, t->last_ns,
                  0LL, (int32_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr, (long long *)nullptr,
                  reinterpret_cast<unsigned long long *>(dev_count));
  }
  if (!t->ev_aux) CK(cudaEventCreateWithFlags(&t->ev_aux, cudaEventDisableTiming));
  CK(cudaEventRecord(t->ev_aux, st));
  CK(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), t->ev_aux, 0));
  return LOD_OK;
}

int lod_last_voxels_log(LodTree *t, int32_t max_level, const int64_t *gidx, int64_t key_base, int32_t *node,
                        uint32_t *cell, uint32_t *rgba, int64_t *key, int64_t capacity, int64_t *dev_count,
                        void *stream) {
  if (!t || !dev_count || capacity < 0 || (capacity > 0 && (!node || !cell || !rgba || !key))) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  if (!t->last_backlog && t->last_nv) return LOD_E_ARG;  // a queued small cycle: unknown
  cudaStream_t st = t->st;
  // the log and the index map were written on the caller's stream (NULL: the
  // legacy default stream, which the tree's non-blocking stream does not
  // follow implicitly)
  if (!t->ev_aux) CK(cudaEventCreateWithFlags(&t->ev_aux, cudaEventDisableTiming));
  CK(cudaEventRecord(t->ev_aux, reinterpret_cast<cudaStream_t>(stream)));
  CK(cudaStreamWaitEvent(st, t->ev_aux, 0));
  const long long nv = t->last_backlog ? t->last_nv : 0;
  if (nv)
    lod::launch(k_last_voxels_log, grid_for(nv), 256, 0, st, t->nd, t->last_backlog, nv, (int)max_level, t->last_ns,
                (const long long *)gidx, (long long)key_base, node, cell, rgba, (long long *)key, (long long)capacity,
                reinterpret_cast<unsigned long long *>(dev_count));
  CK(cudaEventRecord(t->ev_aux, st));
  CK(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), t->ev_aux, 0));
  return LOD_OK;
}

int lod_merge_voxels(LodTree *t, int64_t n_groups, const int32_t *gnode, const int64_t *gstart, const int64_t *goff,
                     const uint32_t *cell, const uint32_t *rgba) {
  if (!t || n_groups < 0 || (n_groups > 0 && (!gnode || !gstart || !goff))) return LOD_E_ARG;
  if (n_groups == 0) return LOD_OK;
  cudaSetDevice(t->dev);
  RK(refresh(t));
  cudaStream_t st = t->st;
  const long long items = goff[n_groups];
  if (items > 0 && (!cell || !rgba)) return LOD_E_ARG;
  for (long long g = 0; g < n_groups; ++g)
    if (gnode[g] < 0 || gnode[g] >= t->num_nodes || gstart[g] < 0 || goff[g + 1] < goff[g]) return LOD_E_ARG;
  const long long acq_bound = items / t->geo.C + n_groups + 1;
  const long long alloc = t->h_ctrl->allocated_total;
  RK(ensure_chunks(t, alloc + acq_bound + 1, alloc));
  RK(ensure_dir(t, alloc + acq_bound + 1, n_groups));
  RK(t->gnodes.ensure(n_groups, st));
  RK(t->gstart.ensure(n_groups, st));
  RK(t->goff.ensure(n_groups + 1, st));
  RK(t->dvcell.ensure(std::max<long long>(items, 1), st));
  RK(t->dvrgba.ensure(std::max<long long>(items, 1), st));
  RK(t->counter.ensure(4, st));
  CK(cudaMemcpyAsync(t->gnodes.p, gnode, n_groups * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(t->gstart.p, gstart, n_groups * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(t->goff.p, goff, (n_groups + 1) * 8, cudaMemcpyHostToDevice, st));
  if (items) {
    CK(cudaMemcpyAsync(t->dvcell.p, cell, items * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(t->dvrgba.p, rgba, items * 4, cudaMemcpyHostToDevice, st));
  }
  unsigned long long *acq = t->counter.p + 3;
  CK(cudaMemsetAsync(acq, 0, 8, st));
  lod::launch(k_merge_groups, grid_for(n_groups * 32), 256, 0, st, t->nd, t->pool, t->geo, t->arena, (long long)n_groups,
              t->gnodes.p, t->gstart.p, t->goff.p, t->dvcell.p, t->dvrgba.p, t->d_ctrl, acq, t->arena_cap);
  lod::launch(k_merge_finish, 1, 1, 0, st, t->d_ctrl, (const unsigned long long *)acq, t->arena_cap, t->geo);
  RK(sync_ctrl(t));
  RK(exact_bounds(t));
  if (t->h_ctrl->error) {
    const int e = t->h_ctrl->error;
    CK(cudaMemsetAsync(&t->d_ctrl->error, 0, 4, st));
    return e;
  }
  return LOD_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- structural edits

// Octree.split of one leaf (octree.py:222-264); one thread.
__global__ void k_split_one(NodeCols nd, PoolCols pool, Geo geo, Ctrl *c, int nid, unsigned long long arena_cap,
                            int *status) {
  lod::pdl_wait();
  if (nd.inner[nid] || nd.level[nid] >= geo.max_depth) {
    *status = -LOD_E_ARG;
    return;
  }
  // release the chain onto the free stack in walk order (store.py:125-143)
  for (int cid = nd.chunk_head[nid]; cid != LOD_NO_CHUNK;) {
    const int nxt = pool.next[cid];
    pool.free_stack[c->free_count++] = cid;
    ++c->released_total;
    pool.occupied[cid] = 0;
    pool.next[cid] = LOD_NO_CHUNK;
    pool.owner[cid] = -1;
    pool.cidx[cid] = -1;
    cid = nxt;
  }
  nd.chunk_head[nid] = LOD_NO_CHUNK;
  nd.chunk_tail[nid] = LOD_NO_CHUNK;
  nd.chunk_count[nid] = 0;
  nd.count[nid] = 0;
  nd.pending[nid] = 0;
  const unsigned long long gb = (unsigned long long)geo.grid_bytes;
  const unsigned long long g0 = (c->arena_off + 63ull) / 64ull * 64ull;  // Arena.alloc(grid_bytes, 64)
  if (g0 + gb > arena_cap) {
    *status = -LOD_E_OUT_OF_ARENA;
    return;
  }
  c->arena_off = g0 + gb;
  const long long first = c->num_nodes;
  const int lvl = nd.level[nid];
  const double half = geo.size_by_level[lvl] * 0.5;
  for (int o = 0; o < 8; ++o) {
    const int k = (int)first + o;
    nd.parent[k] = nid;
    nd.octant[k] = (uint8_t)o;
    nd.level[k] = lvl + 1;
    for (int q = 0; q < 8; ++q) nd.children[8 * k + q] = LOD_NO_NODE;
    nd.inner[k] = 0;
    nd.final_[k] = 0;
    nd.count[k] = 0;
    nd.pending[k] = 0;
    nd.chunk_head[k] = LOD_NO_CHUNK;
    nd.chunk_tail[k] = LOD_NO_CHUNK;
    nd.chunk_count[k] = 0;
    nd.grid_off[k] = -1;
    nd.desc[k] = make_int2(-1, 0);
    nd.dir_off[k] = 0;
    nd.dir_cap[k] = 0;
    nd.bmin[3 * k + 0] = nd.bmin[3 * nid + 0] + ((o & 1) ? half : 0.0);
    nd.bmin[3 * k + 1] = nd.bmin[3 * nid + 1] + ((o & 2) ? half : 0.0);
    nd.bmin[3 * k + 2] = nd.bmin[3 * nid + 2] + ((o & 4) ? half : 0.0);
    nd.children[8 * nid + o] = k;
  }
  nd.inner[nid] = 1;
  nd.grid_off[nid] = (long long)g0;
  nd.desc[nid] = make_int2((int)first, (int)(uint32_t)(g0 >> 6));
  c->num_nodes = first + 8;
  c->splits_total += 1;
  if (lvl + 1 > c->max_level) c->max_level = lvl + 1;
  *status = (int)first;  // >= 1: the first child
}

// Octree.append_chunk + ChunkPool.acquire (octree.py:328-337, store.py:110-123); one thread.
__global__ void k_append_one(NodeCols nd, PoolCols pool, Geo geo, Ctrl *c, int nid, unsigned long long arena_cap,
                             int *status) {
  lod::pdl_wait();
  int cid;
  if (c->free_count > 0) {
    cid = pool.free_stack[--c->free_count];
  } else {
    const unsigned long long off = (c->arena_off + 15ull) / 16ull * 16ull;  // alloc(payload, RECORD_BYTES)
    const unsigned long long end = off + (unsigned long long)geo.C * 16ull;
    if (end > arena_cap) {
      *status = -LOD_E_OUT_OF_ARENA;
      return;
    }
    cid = (int)c->allocated_total++;
    pool.payload_off[cid] = (long long)off;
    c->arena_off = end;
  }
  pool.next[cid] = LOD_NO_CHUNK;
  pool.occupied[cid] = 0;
  const int tail = nd.chunk_tail[nid];
  if (tail != LOD_NO_CHUNK) pool.next[tail] = cid;
  else nd.chunk_head[nid] = cid;
  nd.chunk_tail[nid] = cid;
  pool.owner[cid] = nid;
  pool.cidx[cid] = nd.chunk_count[nid];
  nd.chunk_count[nid] += 1;
  dir_append(nd, pool, &c->dir_top, nid, 1, [&](long long) { return cid; });
  *status = cid;
}

__global__ void k_grid_tas(NodeCols nd, uint8_t *arena, int nid, long long cell, int *status) {
  lod::pdl_wait();
  uint32_t *w = reinterpret_cast<uint32_t *>(arena + nd.grid_off[nid]) + (cell >> 5);
  const uint32_t bit = 1u << (cell & 31);
  *status = (atomicOr(w, bit) & bit) ? 0 : 1;
}

// The device-only indexes after host edits of the node / pool columns:
// descent records from inner / children / grid_off, and per chunk list (walk
// order) the owners, positions and a fresh directory region.  One thread per node.
__global__ void k_rebuild_indexes(NodeCols nd, PoolCols pool, long long n, Ctrl *c) {
  lod::pdl_wait();
  for (long long i = gtid(); i < n; i += gstride()) {
    const int nid = (int)i;
    nd.desc[nid] = nd.inner[nid] ? make_int2(nd.children[8 * nid], (int)(uint32_t)(nd.grid_off[nid] >> 6))
                                 : make_int2(-1, 0);
    const long long cc = nd.chunk_count[nid];
    long long off = nd.dir_off[nid];
    if (cc > nd.dir_cap[nid]) {
      const long long cap = cc * 2 > 4 ? cc * 2 : 4;
      off = dir_claim(pool, &c->dir_top, cap);
      if (off >= 0) {
        nd.dir_off[nid] = off;
        nd.dir_cap[nid] = (int32_t)cap;
      }
    }
    long long ci = 0;
    for (int cid = nd.chunk_head[nid]; cid != LOD_NO_CHUNK && ci < cc; cid = pool.next[cid], ++ci) {
      pool.owner[cid] = nid;
      pool.cidx[cid] = (int)ci;
      if (off >= 0) pool.cdir[off + ci] = cid;
    }
  }
}

__global__ void k_dir_reset(NodeCols nd, long long n, Ctrl *c) {
  lod::pdl_wait();
  for (long long i = gtid(); i < n; i += gstride()) {
    nd.dir_off[i] = 0;
    nd.dir_cap[i] = 0;
  }
  if (gtid() == 0) {
    c->dir_top = 0;
    c->dir_overflow = 0;
  }
}

// Every node's directory handed out again from the chains (which stay
// authoritative) after a soft-sized small cycle ran out of room: at most
// 4 + 2 x chunk_count entries per node.  Only between cycles (exact_bounds),
// with every node row initialised.
static int fix_directory(LodTree *t) {
  if (t->fixing_dir) return LOD_OK;
  t->fixing_dir = true;
  const long long nn = t->h_ctrl->num_nodes, alloc = t->h_ctrl->allocated_total;
  if (lod_debug()) fprintf(stderr, "[lod] chunk directory overflow: rebuilding (%lld nodes)\n", nn);
  int rc = grow_dir(t, 2 * alloc + 4 * nn + 1024);
  if (rc == LOD_OK) {
    lod::launch(k_dir_reset, grid_for(nn), 256, 0, t->st, t->nd, nn, t->d_ctrl);
    lod::launch(k_rebuild_indexes, grid_for(nn), 256, 0, t->st, t->nd, t->pool, nn, t->d_ctrl);
    ++t->dir_rebuilds;
    rc = sync_ctrl(t);
  }
  t->fixing_dir = false;
  return rc;
}

static int one_shot(LodTree *t, int *status_host, const std::function<void(int *)> &launch_fn) {
  RK(refresh(t));
  RK(t->counter.ensure(4, t->st));
  int *d_status = reinterpret_cast<int *>(t->counter.p + 3);
  CK(cudaMemsetAsync(d_status, 0, 4, t->st));
  launch_fn(d_status);
  CK(cudaMemcpyAsync(status_host, d_status, 4, cudaMemcpyDeviceToHost, t->st));
  RK(sync_ctrl(t));  // also waits for the copy
  RK(exact_bounds(t));
  return LOD_OK;
}

extern "C" {

int lod_split_node(LodTree *t, int64_t nid, int32_t *first_child) {
  if (!t || nid < 0) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(refresh(t));
  if (nid >= t->num_nodes) return LOD_E_ARG;
  RK(ensure_nodes(t, t->num_nodes + 8, t->num_nodes));
  int status = 0;
  RK(one_shot(t, &status, [&](int *d) {
    lod::launch(k_split_one, 1, 1, 0, t->st, t->nd, t->pool, t->geo, t->d_ctrl, (int)nid, t->arena_cap, d);
  }));
  if (status <= 0) return status == 0 ? LOD_E_CUDA : -status;  // errors come back negated
  if (first_child) *first_child = status;
  return LOD_OK;
}

int lod_append_chunk(LodTree *t, int64_t nid, int32_t *cid) {
  if (!t || nid < 0) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(refresh(t));
  if (nid >= t->num_nodes) return LOD_E_ARG;
  RK(ensure_chunks(t, t->h_ctrl->allocated_total + 1, t->h_ctrl->allocated_total));
  RK(ensure_dir(t, t->h_ctrl->allocated_total + 1, 1));
  int status = 0;
  RK(one_shot(t, &status, [&](int *d) {
    lod::launch(k_append_one, 1, 1, 0, t->st, t->nd, t->pool, t->geo, t->d_ctrl, (int)nid, t->arena_cap, d);
  }));
  if (status < 0) return -status;
  if (cid) *cid = status;
  return LOD_OK;
}

int lod_grid_test_and_set(LodTree *t, int64_t nid, int64_t cell, int32_t *was_clear) {
  if (!t || nid < 0 || cell < 0 || cell >= t->geo.g * t->geo.g * t->geo.g || !was_clear) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(refresh(t));
  if (nid >= t->num_nodes) return LOD_E_ARG;
  long long goff = -1;
  CK(cudaMemcpyAsync(&goff, t->nd.grid_off + nid, 8, cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  if (goff < 0) return LOD_E_ARG;  // leaves have no grid
  int status = 0;
  RK(one_shot(t, &status, [&](int *d) {
    lod::launch(k_grid_tas, 1, 1, 0, t->st, t->nd, t->arena, (int)nid, (long long)cell, d);
  }));
  *was_clear = status;
  return LOD_OK;
}

int lod_write_nodes(LodTree *t, int64_t n, const int32_t *parent, const uint8_t *octant, const int32_t *level,
                    const int32_t *children, const uint8_t *inner, const uint8_t *final_, const int64_t *count,
                    const int64_t *pending, const int32_t *chunk_head, const int32_t *chunk_tail,
                    const int32_t *chunk_count, const int64_t *grid_off, const double *bmin) {
  if (!t || n < 0) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(refresh(t));
  if (n > t->num_nodes) return LOD_E_ARG;
  cudaStream_t st = t->st;
  auto cp = [&](void *dst, const void *src, size_t bytes) -> int {
    if (src && bytes) return cuda_rc(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return LOD_OK;
  };
  RK(cp(t->nd.parent, parent, n * 4));
  RK(cp(t->nd.octant, octant, n));
  RK(cp(t->nd.level, level, n * 4));
  RK(cp(t->nd.children, children, n * 32));
  RK(cp(t->nd.inner, inner, n));
  RK(cp(t->nd.final_, final_, n));
  RK(cp(t->nd.count, count, n * 8));
  RK(cp(t->nd.pending, pending, n * 8));
  RK(cp(t->nd.chunk_head, chunk_head, n * 4));
  RK(cp(t->nd.chunk_tail, chunk_tail, n * 4));
  RK(cp(t->nd.chunk_count, chunk_count, n * 4));
  RK(cp(t->nd.grid_off, grid_off, n * 8));
  RK(cp(t->nd.bmin, bmin, n * 24));
  const long long alloc = t->h_ctrl->allocated_total;
  RK(ensure_dir(t, alloc, n));
  lod::launch(k_rebuild_indexes, grid_for(n), 256, 0, st, t->nd, t->pool, (long long)n, t->d_ctrl);
  RK(sync_ctrl(t));
  RK(exact_bounds(t));
  return LOD_OK;
}

int lod_write_pool(LodTree *t, int64_t n, const int32_t *next, const int64_t *payload_off, const int32_t *occupied) {
  if (!t || n < 0) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(refresh(t));
  if (n > t->h_ctrl->allocated_total) return LOD_E_ARG;
  cudaStream_t st = t->st;
  if (next && n) CK(cudaMemcpyAsync(t->pool.next, next, n * 4, cudaMemcpyHostToDevice, st));
  if (payload_off && n) CK(cudaMemcpyAsync(t->pool.payload_off, payload_off, n * 8, cudaMemcpyHostToDevice, st));
  if (occupied && n) CK(cudaMemcpyAsync(t->pool.occupied, occupied, n * 4, cudaMemcpyHostToDevice, st));
  if (next) {  // the chain links define the owners and the directory
    const long long nn = t->num_nodes;
    RK(ensure_dir(t, t->h_ctrl->allocated_total, nn));
    lod::launch(k_rebuild_indexes, grid_for(nn), 256, 0, st, t->nd, t->pool, nn, t->d_ctrl);
  }
  RK(sync_ctrl(t));
  RK(exact_bounds(t));
  return LOD_OK;
}

int lod_write_arena(LodTree *t, uint64_t off, uint64_t size, const void *src) {
  if (!t || (size && !src) || off + size > t->arena_cap) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(refresh(t));
  if (size) CK(cudaMemcpyAsync(t->arena + off, src, size, cudaMemcpyHostToDevice, t->st));
  CK(cudaStreamSynchronize(t->st));
  return LOD_OK;
}

int lod_read_directory(LodTree *t, int64_t n, int64_t *dir_off, int32_t *dir_cap, int32_t *cdir, int64_t cdir_len,
                       uint64_t *dir_top) {
  if (!t || n < 0 || n > t->ncap || !dir_top) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(sync_ctrl(t));
  RK(exact_bounds(t));
  *dir_top = t->h_ctrl->dir_top;
  if (n && dir_off) CK(cudaMemcpyAsync(dir_off, t->nd.dir_off, n * 8, cudaMemcpyDeviceToHost, t->st));
  if (n && dir_cap) CK(cudaMemcpyAsync(dir_cap, t->nd.dir_cap, n * 4, cudaMemcpyDeviceToHost, t->st));
  if (cdir) {
    if (cdir_len < (int64_t)*dir_top) return LOD_E_ARG;
    if (*dir_top) CK(cudaMemcpyAsync(cdir, t->pool.cdir, *dir_top * 4, cudaMemcpyDeviceToHost, t->st));
  }
  CK(cudaStreamSynchronize(t->st));
  return LOD_OK;
}

static int gather_impl(LodTree *t, const std::vector<int32_t> &nodes, const std::vector<long long> &starts,
                       const std::vector<long long> &offs, long long total, float4 *host_out) {
  cudaStream_t st = t->st;
  const long long m = (long long)nodes.size();
  if (m == 0 || total == 0) return LOD_OK;
  RK(t->gnodes.ensure(m, st));
  RK(t->gstart.ensure(m, st));
  RK(t->goff.ensure(m, st));
  RK(t->gbuf.ensure(total, st));
  CK(cudaMemcpyAsync(t->gnodes.p, nodes.data(), m * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(t->gstart.p, starts.data(), m * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(t->goff.p, offs.data(), m * 8, cudaMemcpyHostToDevice, st));
  for (long long b = 0; b < m; b += 65535) {
    long long cnt = std::min<long long>(65535, m - b);
    lod::launch(k_gather_nodes, (unsigned)cnt, 256, 0, st, t->nd, t->pool, t->geo, t->arena, t->gnodes.p + b,
                                                  t->gstart.p + b, t->goff.p + b, t->gbuf.p);
  }
  CK(cudaMemcpyAsync(host_out, t->gbuf.p, total * 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return LOD_OK;
}

int lod_gather(LodTree *t, int64_t nid, int64_t start, float *xyz, uint32_t *rgba) {
  if (t) RK(refresh(t));
  if (!t || nid < 0 || nid >= t->num_nodes || start < 0) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  long long cnt = 0;
  CK(cudaMemcpyAsync(&cnt, t->nd.count + nid, 8, cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  long long k = cnt - start;
  if (k <= 0) return LOD_OK;
  std::vector<float4> buf((size_t)k);
  RK(gather_impl(t, {(int32_t)nid}, {start}, {0}, k, buf.data()));
  for (long long i = 0; i < k; ++i) {
    xyz[3 * i] = buf[i].x;
    xyz[3 * i + 1] = buf[i].y;
    xyz[3 * i + 2] = buf[i].z;
    uint32_t c;
    memcpy(&c, &buf[i].w, 4);
    rgba[i] = c;
  }
  return LOD_OK;
}

int lod_dump_records(LodTree *t, int64_t num_nodes, int64_t *offsets, void *records) {
  if (t) RK(refresh(t));
  if (!t || num_nodes < 0 || num_nodes > t->num_nodes || !offsets) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  std::vector<long long> cnt((size_t)num_nodes);
  if (num_nodes) CK(cudaMemcpyAsync(cnt.data(), t->nd.count, num_nodes * 8, cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  std::vector<int32_t> nodes;
  std::vector<long long> starts, offs;
  long long total = 0;
  offsets[0] = 0;
  for (long long i = 0; i < num_nodes; ++i) {
    if (cnt[i] > 0) {
      nodes.push_back((int32_t)i);
      starts.push_back(0);
      offs.push_back(total);
    }
    total += cnt[i];
    offsets[i + 1] = total;
  }
  if (!records) return LOD_OK;
  return gather_impl(t, nodes, starts, offs, total, reinterpret_cast<float4 *>(records));
}

int lod_read_arena(LodTree *t, uint64_t off, uint64_t size, void *dst) {
  if (!t || !dst || off + size > t->arena_cap) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  CK(cudaMemcpyAsync(dst, t->arena + off, size, cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  return LOD_OK;
}

}  // extern "C"

static int prefetch_impl(LodTree *t, const void *xyz, const uint32_t *rgba, int64_t n, bool packed);

int lod_prefetch_batch(LodTree *t, const float *xyz, const uint32_t *rgba, int64_t n) {
  if (!t || n < 0 || (n > 0 && (!xyz || !rgba))) return LOD_E_ARG;
  return prefetch_impl(t, xyz, rgba, n, false);
}

int lod_prefetch_records(LodTree *t, const void *records, int64_t n) {
  if (!t || n < 0 || (n > 0 && !records)) return LOD_E_ARG;
  return prefetch_impl(t, records, nullptr, n, true);
}

static int prefetch_impl(LodTree *t, const void *xyz, const uint32_t *rgba, int64_t n, bool packed) {
  if (n == 0) return LOD_OK;
  // only page-locked host memory can be copied asynchronously; anything else
  // is left to lod_insert_batch's own copy
  cudaPointerAttributes ax{}, ac{};
  if (cudaPointerGetAttributes(&ax, xyz) != cudaSuccess ||
      (!packed && cudaPointerGetAttributes(&ac, rgba) != cudaSuccess)) {
    cudaGetLastError();
    return LOD_OK;
  }
  if (ax.type != cudaMemoryTypeHost || (!packed && ac.type != cudaMemoryTypeHost)) return LOD_OK;
  cudaSetDevice(t->dev);
  if (!t->cst) {
    CK(cudaStreamCreateWithFlags(&t->cst, cudaStreamNonBlocking));
    for (auto &sg : t->stage) CK(cudaEventCreateWithFlags(&sg.ready, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&t->ev_counted, cudaEventDisableTiming));
  }
  for (auto &sg : t->stage)
    if (sg.valid && sg.packed == packed && sg.hx == xyz && sg.hc == rgba && sg.n == n) return LOD_OK;  // staged
  LodTree::Stage &sg = t->stage[t->stage_next];
  t->stage_next = (t->stage_next + 1) % 3;
  // the slot's previous batch was consumed by an earlier insert (or is
  // superseded); that insert's tail may still read it on the tree stream, so
  // a growing slot frees its old buffers only behind the tree stream
  const bool grow = packed ? n > sg.rec.cap : (3 * n > sg.xyz.cap || n > sg.rgba.cap);
  if (grow) {
    CK(cudaEventRecord(t->ev_counted, t->st));
    CK(cudaStreamWaitEvent(t->cst, t->ev_counted, 0));
  }
  if (packed) {
    RK(sg.rec.ensure(n, t->cst));
  } else {
    RK(sg.xyz.ensure(3 * n, t->cst));
    RK(sg.rgba.ensure(n, t->cst));
  }
  sg.packed = packed;
  // The copy itself is issued by the next lod_insert_batch behind its first
  // count pass: a 16 MB DMA into HBM running alongside the claim-heavy count
  // slows it by ~50 % (L2 pressure), while the rest of the cycle hides it.
  sg.hx = xyz;
  sg.hc = rgba;
  sg.n = n;
  sg.valid = true;
  sg.pending = true;
  sg.parts = packed ? kPartBig : kPartsAll;
  sg.order = ++t->stage_order;
  return LOD_OK;
}

static int issue_stage(LodTree *t, LodTree::Stage &sg, int mask) {
  const int go = sg.parts & mask;
  if (sg.packed) {
    if (go & kPartBig) CK(cudaMemcpyAsync(sg.rec.p, sg.hx, (size_t)sg.n * 16, cudaMemcpyHostToDevice, t->cst));
  } else {
    if (go & kPartSmall) CK(cudaMemcpyAsync(sg.rgba.p, sg.hc, (size_t)sg.n * 4, cudaMemcpyHostToDevice, t->cst));
    if (go & kPartBig) CK(cudaMemcpyAsync(sg.xyz.p, sg.hx, (size_t)sg.n * 12, cudaMemcpyHostToDevice, t->cst));
  }
  sg.parts &= ~go;
  if (sg.parts == 0) {  // the last part: the slot is ready once it lands
    CK(cudaEventRecord(sg.ready, t->cst));
    sg.pending = false;
  }
  return LOD_OK;
}

int lod_prefetch_drain(LodTree *t) {
  if (!t) return LOD_E_ARG;
  if (!t->cst) return LOD_OK;
  cudaSetDevice(t->dev);
  CK(cudaStreamSynchronize(t->cst));
  for (auto &sg : t->stage) sg.valid = sg.pending = false;
  return LOD_OK;
}

int lod_delta_info(LodTree *t, LodDeltaInfo *info) {
  if (!t || !info) return LOD_E_ARG;
  info->n_splits = t->d_nsplits;
  info->n_voxel_groups = t->d_nvg;
  info->n_voxels = t->d_nv;
  info->n_point_groups = t->d_npg;
  return LOD_OK;
}

int lod_read_delta(LodTree *t, int32_t *splits, int32_t *vnode, int64_t *vstart, int64_t *vcount, uint32_t *vcells,
                   uint32_t *vrgba, int32_t *pnode, int64_t *pstart, int64_t *pcount) {
  if (!t) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  cudaStream_t st = t->st;
  auto cp = [&](void *dst, const void *src, long long bytes) -> int {
    if (bytes <= 0 || !dst) return LOD_OK;
    if (!src) return LOD_E_ARG;
    t->d2h_bytes += bytes;
    CK(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, st));
    return LOD_OK;
  };
  RK(cp(splits, t->dsplits.p, t->d_nsplits * 4));
  RK(cp(vnode, t->dvnode.p, t->d_nvg * 4));
  RK(cp(vstart, t->dvstart.p, t->d_nvg * 8));
  RK(cp(vcount, t->dvcount.p, t->d_nvg * 8));
  RK(cp(vcells, t->dvcell.p, t->d_nv * 4));
  RK(cp(vrgba, t->dvrgba.p, t->d_nv * 4));
  RK(cp(pnode, t->dpnode.p, t->d_npg * 4));
  RK(cp(pstart, t->dpstart.p, t->d_npg * 8));
  RK(cp(pcount, t->dpcount.p, t->d_npg * 8));
  CK(cudaStreamSynchronize(st));
  return LOD_OK;
}

// accessors for lod_raster.cu
cudaStream_t lod_tree_stream(LodTree *t) { return t->st; }
int lod_tree_device(LodTree *t) { return t->dev; }
const uint8_t *lod_tree_arena(LodTree *t) { return t->arena; }
PoolCols lod_tree_pool(LodTree *t) { return t->pool; }
long long lod_tree_num_nodes(LodTree *t) {
  refresh(t);
  return t->num_nodes;
}
int lod_tree_ensure_woff(LodTree *t, long long n, long long **p) {
  RK(t->woff.ensure(std::max<long long>(n, 1), t->st));
  *p = t->woff.p;
  return LOD_OK;
}
int lod_tree_ensure_vislist(LodTree *t, long long n, int32_t **p) {
  int rc = t->vislist.ensure(std::max<long long>(n, 1), t->st);
  *p = t->vislist.p;
  return rc;
}
int lod_tree_ensure_fb(LodTree *t, long long n, unsigned long long **p) {
  int rc = t->fb.ensure(std::max<long long>(n, 1), t->st);
  *p = t->fb.p;
  return rc;
}
unsigned long long *lod_tree_counter(LodTree *t) { return t->counter.p; }
NodeCols lod_tree_nodes(LodTree *t) { return t->nd; }
Geo lod_tree_geo(LodTree *t) { return t->geo; }
// two ping-pong selection lists of num_nodes entries each (the cut never
// holds a node twice, so num_nodes bounds every list)
int lod_tree_ensure_sel(LodTree *t, long long n, int32_t **a, int32_t **b) {
  int rc = t->vislist.ensure(std::max<long long>(2 * n, 2), t->st);
  *a = t->vislist.p;
  *b = t->vislist.p + std::max<long long>(n, 1);
  return rc;
}

// ---------------------------------------------------------------- replication

namespace {
struct PackHeader {
  unsigned long long magic;
  long long num_nodes, allocated_total, free_count;
  unsigned long long arena_off;
  // the source tree's geometry: a pack unpacks only into an identically
  // configured tree (node ids, grid offsets and chunk payloads depend on it)
  double bmin[3], size;
  long long grid_res, leaf_threshold, max_depth, chunk_capacity;
  Ctrl ctrl;
};

bool same_geometry(const PackHeader &h, const LodParams &p) {
  return h.bmin[0] == p.bmin[0] && h.bmin[1] == p.bmin[1] && h.bmin[2] == p.bmin[2] && h.size == p.size &&
         h.grid_res == p.grid_res && h.leaf_threshold == p.leaf_threshold && h.max_depth == p.max_depth &&
         h.chunk_capacity == p.chunk_capacity;
}
constexpr unsigned long long kPackMagic = 0x4C4F4442323030ULL;  // "LODB200"

struct PackLayout {
  size_t off[32];
  size_t total;
};

// Byte layout of a packed tree: header, 14 node columns [0, n), 6 pool columns
// [0, allocated_total), the free stack [0, free_count), arena [0, arena_off).
PackLayout pack_layout(const Ctrl &c) {
  PackLayout L{};
  const size_t n = (size_t)c.num_nodes, a = (size_t)c.allocated_total, f = (size_t)c.free_count;
  const size_t sizes[] = {sizeof(PackHeader),
                          n * 4, n * 1, n * 4, n * 32, n * 1, n * 1, n * 8, n * 8, n * 4, n * 4, n * 4, n * 8,
                          n * 24, n * 8, n * 8, n * 4,
                          a * 4, a * 8, a * 4, a * 4, a * 4,
                          f * 4, (size_t)c.dir_top * 4,
                          (size_t)c.arena_off};
  size_t o = 0;
  int k = 0;
  for (size_t s : sizes) {
    L.off[k++] = o;
    o += (s + 255) / 256 * 256;
  }
  L.off[k] = o;
  L.total = o;
  return L;
}
}  // namespace

extern "C" {

int lod_tree_pack_size(LodTree *t, uint64_t *bytes) {
  if (!t || !bytes) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(sync_ctrl(t));
  RK(exact_bounds(t));  // a pending directory rebuild first
  *bytes = pack_layout(*t->h_ctrl).total;
  return LOD_OK;
}

int lod_tree_pack(LodTree *t, void *dev_buf, uint64_t bytes) {
  if (!t || !dev_buf) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(sync_ctrl(t));
  RK(exact_bounds(t));
  const Ctrl c = *t->h_ctrl;
  const PackLayout L = pack_layout(c);
  if (bytes < L.total) return LOD_E_ARG;
  uint8_t *b = static_cast<uint8_t *>(dev_buf);
  PackHeader hd{};
  hd.magic = kPackMagic;
  hd.num_nodes = c.num_nodes;
  hd.allocated_total = c.allocated_total;
  hd.free_count = c.free_count;
  hd.arena_off = c.arena_off;
  for (int k = 0; k < 3; ++k) hd.bmin[k] = t->p.bmin[k];
  hd.size = t->p.size;
  hd.grid_res = t->p.grid_res;
  hd.leaf_threshold = t->p.leaf_threshold;
  hd.max_depth = t->p.max_depth;
  hd.chunk_capacity = t->p.chunk_capacity;
  hd.ctrl = c;
  cudaStream_t st = t->st;
  CK(cudaMemcpyAsync(b + L.off[0], &hd, sizeof(hd), cudaMemcpyHostToDevice, st));
  const size_t n = (size_t)c.num_nodes, a = (size_t)c.allocated_total, f = (size_t)c.free_count;
  const void *src[] = {t->nd.parent, t->nd.octant, t->nd.level, t->nd.children, t->nd.inner, t->nd.final_,
                       t->nd.count, t->nd.pending, t->nd.chunk_head, t->nd.chunk_tail, t->nd.chunk_count,
                       t->nd.grid_off, t->nd.bmin, t->nd.desc, t->nd.dir_off, t->nd.dir_cap, t->pool.next,
                       t->pool.payload_off, t->pool.occupied, t->pool.owner, t->pool.cidx, t->pool.free_stack,
                       t->pool.cdir, t->arena};
  const size_t sz[] = {n * 4, n, n * 4, n * 32, n, n, n * 8, n * 8, n * 4, n * 4, n * 4, n * 8, n * 24, n * 8,
                       n * 8, n * 4, a * 4, a * 8, a * 4, a * 4, a * 4, f * 4, (size_t)c.dir_top * 4,
                       (size_t)c.arena_off};
  for (int k = 0; k < 24; ++k)
    if (sz[k]) CK(cudaMemcpyAsync(b + L.off[k + 1], src[k], sz[k], cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  return LOD_OK;
}

int lod_tree_unpack(LodTree *t, const void *dev_buf, uint64_t bytes) {
  if (!t || !dev_buf || bytes < sizeof(PackHeader)) return LOD_E_ARG;
  cudaSetDevice(t->dev);
  RK(refresh(t));
  cudaStream_t st = t->st;
  const uint8_t *b = static_cast<const uint8_t *>(dev_buf);
  PackHeader hd;
  CK(cudaMemcpy(&hd, b, sizeof(hd), cudaMemcpyDeviceToHost));
  if (hd.magic != kPackMagic || !same_geometry(hd, t->p)) return LOD_E_ARG;
  const Ctrl c = hd.ctrl;
  const PackLayout L = pack_layout(c);
  if (bytes < L.total || c.arena_off > t->arena_cap) return LOD_E_ARG;
  RK(ensure_nodes(t, std::max<long long>(c.num_nodes, 1), 0));
  RK(ensure_chunks(t, std::max<long long>(c.allocated_total + 1, 1), 0));
  t->ub_dir = 0;
  RK(ensure_dir(t, (long long)c.dir_top, 0));
  const size_t n = (size_t)c.num_nodes, a = (size_t)c.allocated_total, f = (size_t)c.free_count;
  void *dst[] = {t->nd.parent, t->nd.octant, t->nd.level, t->nd.children, t->nd.inner, t->nd.final_,
                 t->nd.count, t->nd.pending, t->nd.chunk_head, t->nd.chunk_tail, t->nd.chunk_count,
                 t->nd.grid_off, t->nd.bmin, t->nd.desc, t->nd.dir_off, t->nd.dir_cap, t->pool.next,
                 t->pool.payload_off, t->pool.occupied, t->pool.owner, t->pool.cidx, t->pool.free_stack,
                 t->pool.cdir, t->arena};
  const size_t sz[] = {n * 4, n, n * 4, n * 32, n, n, n * 8, n * 8, n * 4, n * 4, n * 4, n * 8, n * 24, n * 8,
                       n * 8, n * 4, a * 4, a * 8, a * 4, a * 4, a * 4, f * 4, (size_t)c.dir_top * 4,
                       (size_t)c.arena_off};
  for (int k = 0; k < 24; ++k)
    if (sz[k]) CK(cudaMemcpyAsync(dst[k], b + L.off[k + 1], sz[k], cudaMemcpyDeviceToDevice, st));
  // the rest of the arena must stay zeroed (regions are handed out zeroed)
  if (t->arena_cap > c.arena_off) CK(cudaMemsetAsync(t->arena + c.arena_off, 0, t->arena_cap - c.arena_off, st));
  Ctrl nc{};
  nc.num_nodes = c.num_nodes;
  nc.splits_total = c.splits_total;
  nc.max_level = c.max_level;
  nc.arena_off = c.arena_off;
  nc.allocated_total = c.allocated_total;
  nc.free_count = c.free_count;
  nc.released_total = c.released_total;
  nc.dir_top = c.dir_top;
  CK(cudaMemcpyAsync(t->d_ctrl, &nc, sizeof(Ctrl), cudaMemcpyHostToDevice, st));
  RK(sync_ctrl(t));
  RK(exact_bounds(t));
  t->ingested = 1LL << 40;  // unknown: the spill of a cycle is then bounded by n * T alone
  return LOD_OK;
}

}  // extern "C"
