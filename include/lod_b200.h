/*
 * lod_b200.h -- C ABI of the B200-native incremental LOD update path.
 *
 * Drop-in boundary for the reference package `lodstream` (arXiv 2310.03567,
 * /root/reference/pkg/src/lodstream).  The reference's operator layer is eight
 * numba kernels over flat arrays (_kernels.py:27-372) driven by Python
 * orchestration (update.py:252-417, render.py:213-239); this library replaces
 * that whole layer at the insert_batch / rasterize level, because the B200
 * design fuses the passes and keeps the tree resident in HBM.
 *
 * Conventions: plain C types only; every function returns LOD_OK (0) or one
 * of the LOD_E_* codes.  Pointers are HOST pointers unless the flag
 * LOD_FLAG_DEVICE_INPUT / LOD_FLAG_DEVICE_FB says they are device pointers.
 * Every call is ordered on the tree's own CUDA stream and returns only after
 * the results it reports are final (one event sync per call).  One writer per
 * tree (update.py:16-17 of the reference's single-writer model).
 */
#ifndef LOD_B200_H
#define LOD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The first three map 1:1 onto the reference's fatal
 * exceptions (errors.py:10-19): OutOfArena(MemoryError), SpillOverflow,
 * BacklogOverflow.  Partial tree state is permitted after them (errors.py:1-5). */
enum {
    LOD_OK = 0,
    LOD_E_OUT_OF_ARENA = 1,
    LOD_E_SPILL_OVERFLOW = 2,
    LOD_E_BACKLOG_OVERFLOW = 3,
    LOD_E_CUDA = 4,
    LOD_E_ARG = 5,
    LOD_E_NOMEM = 6,
    LOD_E_NO_DEVICE = 7
};

enum {
    LOD_FLAG_DEVICE_INPUT = 1, /* xyz / rgba are device pointers (resident in HBM)          */
    LOD_FLAG_DEVICE_FB = 2,    /* framebuffer pointer is a device pointer                   */
    LOD_FLAG_PROFILE = 4,      /* record per-phase CUDA-event times into LodBatchStats      */
    LOD_FLAG_DELTA = 8,        /* capture the cycle's BatchDelta (collect_delta=True)       */
    LOD_FLAG_PACKED = 16       /* xyz points at n 16-byte records (f32 x,y,z | u32 rgba);
                                  rgba is ignored (may be NULL)                              */
    , LOD_FLAG_INPUT_STREAM = 32 /* order the device inputs after LodLimits.input_stream      */
    , LOD_FLAG_FB_CLEAR = 64   /* host framebuffer is all sentinel (a fresh Framebuffer): the
                                  device target is filled instead of uploaded             */
};

typedef struct LodTree LodTree;

/* Octree(bounds, Arena(arena_bytes), ChunkPool(arena, chunk_capacity),
 *        grid_res=, leaf_threshold=, max_depth=)   -- octree.py:148-167,
 * store.py:39-46, store.py:89-100.  grid_res must be even (octree.py:158). */
typedef struct {
    double bmin[3];
    double size;
    int64_t grid_res;
    int64_t leaf_threshold;
    int64_t max_depth;
    int64_t chunk_capacity;
    uint64_t arena_bytes;
    int32_t device; /* CUDA ordinal */
    int32_t reserved;
} LodParams;

/* UpdateConfig capacities (update.py:59-64), passed per call because the
 * reference keeps them in the per-tree UpdateState, not in the Octree. */
typedef struct {
    int64_t backlog_capacity;
    int64_t spill_capacity;
    /* With LOD_FLAG_INPUT_STREAM: the CUDA stream (cudaStream_t; 0 = the legacy
     * default stream) that produces the device inputs.  The tree's own stream
     * waits for the work queued on it so far (an event, no host sync), so a
     * batch written by a copy, kernel or collective on the caller's stream is
     * read only once it is complete. */
    void *input_stream;
} LodLimits;

enum { LOD_NPHASE = 10 };

/* Per-call result: what insert_batch changed (UpdateStats fields, update.py:382-392)
 * plus the counts B_alg needs. */
typedef struct {
    int64_t n_batch, n_spill, n_voxels, n_splits, iterations;
    int64_t num_nodes, splits_total, max_level;
    int64_t allocated_total, free_count, released_total;
    uint64_t arena_offset;
    int64_t launches;              /* kernels this call launched                              */
    int64_t h2d_bytes, d2h_bytes;  /* host<->device traffic of this call                      */
    float device_ms;               /* CUDA-event time of the whole update on the tree stream,
                                      -1 when the call returned before its tail (sort + store +
                                      cleanup) ran: reported by the next call or lod_tree_wait */
    float device_ms_prev;          /* the previous call's device_ms if it was -1, else -1     */
    float phase_ms[LOD_NPHASE];    /* with LOD_FLAG_PROFILE: count (k_count only), split,
                                      resolve, backlog, alloc, sort (+ store), delta,
                                      epilogue, h2d, total                                    */
} LodBatchStats;

/* Counters of the live tree (Octree / ChunkPool / Arena scalar attributes). */
typedef struct {
    int64_t num_nodes, node_capacity, splits_total, max_level;
    int64_t allocated_total, free_count, released_total, chunk_capacity_rows;
    uint64_t arena_offset, arena_capacity;
    int64_t grid_bytes, chunk_capacity;
} LodTreeInfo;

const char *lod_strerror(int code);
int lod_device_count(int *count);

/* replaces Octree.__init__ + Arena/ChunkPool construction (octree.py:148-188) */
int lod_tree_create(const LodParams *params, LodTree **out);
int lod_tree_destroy(LodTree *tree);
int lod_tree_info(LodTree *tree, LodTreeInfo *info);

/* replaces update.insert_batch (update.py:252-393) and with it
 * _kernels.count_points / sample_and_route / collect_allocs / store_points /
 * store_voxels / clear_marks (_kernels.py:27-287), Octree.split
 * (octree.py:222-264), Octree.append_chunk (octree.py:328-337) and
 * ChunkPool.acquire/release (store.py:110-143). */
int lod_insert_batch(LodTree *tree, const float *xyz, const uint32_t *rgba, int64_t n,
                     const LodLimits *limits, int flags, LodBatchStats *stats);

/* Counts of the cycles whose insert returned before the device ran them:
 * batches of at most 256 host points run as ONE kernel per cycle, and when no
 * error is possible for the batch (its worst case bounded from n, the leaf
 * threshold and the depth cannot overflow the backlog, the spill buffer or
 * the arena) lod_insert_batch returns once the kernel is queued, reporting
 * iterations = -1 and n_voxels = n_spill = n_splits = -1.  lod_tree_settle
 * waits for the tree's stream (those cycles and an early-returning insert's
 * tail included) and reports what the queued cycles did since the last
 * settle; every other entry point that reads the tree is ordered behind them. */
typedef struct {
    int64_t calls;                          /* queued cycles folded by this call          */
    int64_t n_voxels, n_voxels_max;         /* their new voxels: sum, largest cycle        */
    int64_t n_spill_max, n_splits;          /* largest spill, sum of splits                */
    int64_t num_nodes, splits_total, max_level;  /* the tree after them                    */
    float device_ms;                        /* device time of those cycles + the last tail */
    int32_t error;                          /* LOD_OK (a queued cycle cannot fail)         */
} LodSettleStats;
int lod_tree_settle(LodTree *tree, LodSettleStats *out);

/* Wait until the tree's stream is idle (the last insert's tail included);
 * `last_device_ms` (may be NULL) receives that insert's device_ms when the
 * call returned early (else -1).  Every other entry point that reads the
 * tree is already ordered behind the tail. */
int lod_tree_wait(LodTree *tree, float *last_device_ms);

/* Ingest feed (the reference's BatchSource queue feeding
 * run_frame_updates, io.py:340-413, update.py:396-417): start the H2D copy of
 * a batch in PAGE-LOCKED host memory on the tree's copy stream (a ring of 3
 * staging slots: up to two batches in flight ahead of the one updating), so
 * it overlaps the updates running ahead of it.  A later
 * lod_insert_batch with the same (xyz, rgba, n) consumes the staged copy
 * instead of copying.  Pageable memory is ignored (the insert copies it).
 * The caller keeps the host arrays unchanged until that insert, or until
 * lod_prefetch_drain (waits for outstanding copies, drops unused stages). */
int lod_prefetch_batch(LodTree *tree, const float *xyz, const uint32_t *rgba, int64_t n);
int lod_prefetch_drain(LodTree *tree);

/* lod_prefetch_batch for a batch of n packed 16-byte records (the SIM file
 * layout, io.py:38-40; page-locked), consumed by a later lod_insert_batch with
 * LOD_FLAG_PACKED and the same pointer and n. */
int lod_prefetch_records(LodTree *tree, const void *records, int64_t n);

/* Disk feed (io.py:218-290 _DirectReader + io.py:340-413 BatchSource): a
 * reader thread reads a SIM file (16-byte records, io.py:60-92) batch after
 * batch with O_DIRECT (buffered when the filesystem refuses) into a ring of
 * `slots` page-locked buffers; lod_sim_next hands out the next batch in file
 * order (blocking; *n = 0 at end of file), valid until lod_sim_release.
 * batch_records * 16 must be a multiple of 4096.  LOD_E_ARG for an empty or
 * truncated file (io.py: EmptyFile / Truncated).  No GPU is needed. */
typedef struct LodSim LodSim;
typedef struct {
    uint64_t file_bytes, bytes_read;
    double read_seconds;   /* time the reader thread spent in read calls */
    int32_t direct;        /* 1: O_DIRECT (page cache bypassed)         */
    int32_t pinned;        /* 1: slots are page-locked (a CUDA device)  */
} LodSimInfo;
int lod_sim_open(const char *path, int64_t batch_records, int32_t slots, LodSim **out);
int lod_sim_next(LodSim *sim, const void **records, int64_t *n);
int lod_sim_release(LodSim *sim, const void *records);
int lod_sim_info(LodSim *sim, LodSimInfo *info);
int lod_sim_close(LodSim *sim);

/* D2H mirror of the node table columns (octree.py:169-182), rows [0, n).
 * Any pointer may be NULL to skip that column. children is (n,8), bmin (n,3). */
int lod_read_nodes(LodTree *tree, int64_t n, int32_t *parent, uint8_t *octant, int32_t *level,
                   int32_t *children, uint8_t *inner, uint8_t *final_, int64_t *count,
                   int64_t *pending, int32_t *chunk_head, int32_t *chunk_tail,
                   int32_t *chunk_count, int64_t *grid_off, double *bmin);

/* D2H mirror of the chunk pool tables (store.py:97-101), rows [0, n), and
 * the LIFO free list bottom-to-top (store.py:102). */
int lod_read_pool(LodTree *tree, int64_t n, int32_t *next, int64_t *payload_off,
                  int32_t *occupied, int32_t *free_list, int64_t n_free);

/* Structural edits outside an update cycle (the reference's Octree / ChunkPool
 * mutators, used by its unit tests and by callers that build trees by hand):
 *   lod_split_node        Octree.split (octree.py:222-264) after the caller
 *                         gathered the leaf's samples (lod_gather) into its
 *                         spill buffer: the chunk chain goes onto the free
 *                         stack in walk order, the node turns inner with a
 *                         zeroed 64-aligned grid (LOD_E_OUT_OF_ARENA past
 *                         capacity) and gets 8 children, ids *first_child + o
 *                         in octant order; LOD_E_ARG unless nid is a leaf
 *                         below max depth;
 *   lod_append_chunk      Octree.append_chunk + ChunkPool.acquire
 *                         (octree.py:328-337, store.py:110-123): LIFO free
 *                         stack first, else a 16-aligned arena cut;
 *   lod_grid_test_and_set Octree.grid_test_and_set (octree.py:281-288).
 * Host edits of the mirrored columns are written back with lod_write_nodes /
 * lod_write_pool / lod_write_arena (same layouts as the readers; NULL skips a
 * column); the device-only indexes (descent records, chunk directory, chunk
 * owners) are rebuilt from the written columns. */
int lod_split_node(LodTree *tree, int64_t nid, int32_t *first_child);
int lod_append_chunk(LodTree *tree, int64_t nid, int32_t *cid);
int lod_grid_test_and_set(LodTree *tree, int64_t nid, int64_t cell, int32_t *was_clear);
int lod_write_nodes(LodTree *tree, int64_t n, const int32_t *parent, const uint8_t *octant, const int32_t *level,
                    const int32_t *children, const uint8_t *inner, const uint8_t *final_, const int64_t *count,
                    const int64_t *pending, const int32_t *chunk_head, const int32_t *chunk_tail,
                    const int32_t *chunk_count, const int64_t *grid_off, const double *bmin);
int lod_write_pool(LodTree *tree, int64_t n, const int32_t *next, const int64_t *payload_off, const int32_t *occupied);
int lod_write_arena(LodTree *tree, uint64_t off, uint64_t size, const void *src);

/* Replicated top nodes of an octant-prefix partitioned tree (multigpu.py,
 * SURVEY 8(e) "all-gathered and merged by global index"):
 *   lod_last_voxels   the voxels the last lod_insert_batch created at nodes
 *                     of level < max_level: node, cell, rgba and the winner's
 *                     batch position (all-array index - spill length), in no
 *                     particular order; capacity 0 queries *n.  Call before
 *                     the next insert (it reads that cycle's backlog);
 *   lod_last_voxels_count  how many there are, written to the device word
 *                     *dev_count (-1 when the last insert's counts are
 *                     unknown: a queued small cycle) without a host wait;
 *                     `stream` is ordered behind the write;
 *   lod_last_voxels_log  append them to a device log instead (no host
 *                     wait): node, cell, rgba and an order key = key_base +
 *                     gidx[winner's batch position] (gidx: a device int64
 *                     array, NULL = the position itself); *dev_count (device
 *                     int64) is advanced by every voxel, entries past
 *                     `capacity` are dropped (the caller sizes the log from
 *                     the batch's n_voxels); ordered after `stream`'s work
 *                     and `stream` after it (NULL = the legacy stream);
 *   lod_merge_voxels  rewrite each listed node's voxel sequence from gstart[g]
 *                     on with the items goff[g] .. goff[g+1]-1 (cells and
 *                     colours in their final order; the node's own voxels of
 *                     the last cycle are among them), extending its chunk
 *                     list and setting the cells' grid bits -- so every rank's
 *                     copy of a top node holds the single-tree sequence. */
int lod_last_voxels(LodTree *tree, int32_t max_level, int64_t capacity, int32_t *node, uint32_t *cell,
                    uint32_t *rgba, int64_t *winner, int64_t *n);
int lod_last_voxels_count(LodTree *tree, int32_t max_level, int64_t *dev_count, void *stream);
int lod_last_voxels_log(LodTree *tree, int32_t max_level, const int64_t *gidx, int64_t key_base, int32_t *node,
                        uint32_t *cell, uint32_t *rgba, int64_t *key, int64_t capacity, int64_t *dev_count,
                        void *stream);
int lod_merge_voxels(LodTree *tree, int64_t n_groups, const int32_t *gnode, const int64_t *gstart,
                     const int64_t *goff, const uint32_t *cell, const uint32_t *rgba);

/* The device-only chunk directory (inspection / tests): per node its region
 * offset and capacity, the entries [0, *dir_top) (node n's chunk ids in list
 * order are cdir[dir_off[n] + i], i < chunk_count[n]).  cdir may be NULL to
 * read *dir_top only; cdir_len is its capacity in entries. */
int lod_read_directory(LodTree *tree, int64_t n, int64_t *dir_off, int32_t *dir_cap, int32_t *cdir,
                       int64_t cdir_len, uint64_t *dir_top);

/* Octree.gather_samples (octree.py:298-326): samples [start, count) of node nid
 * in storage order.  xyz is (k,3) f32, rgba (k,) u32, k = count - start. */
int lod_gather(LodTree *tree, int64_t nid, int64_t start, float *xyz, uint32_t *rgba);

/* Every node's samples, packed in node-id order: offsets (num_nodes+1) are the
 * prefix sums of count; records are 16-byte (x,y,z,rgba). */
int lod_dump_records(LodTree *tree, int64_t num_nodes, int64_t *offsets, void *records);

/* BatchDelta of the last lod_insert_batch made with LOD_FLAG_DELTA -- replaces
 * insert_batch(collect_delta=True) (update.py:183-194, 333-355), the producer
 * of the streaming service (service.py:228-243, 299):
 *   splits        split nodes in split order (each split's 8 "create" events
 *                 are its children, ids children[8*nid+o], octant o);
 *   voxel groups  ascending node id: node, [vstart, vstart+vcount) into
 *                 vcells / vrgba (claim order inside a node);
 *   point groups  ascending node id: leaf, pre-store count (gather start), new points.
 * lod_delta_info gives the sizes; lod_read_delta copies to host (NULL skips). */
typedef struct {
    int64_t n_splits, n_voxel_groups, n_voxels, n_point_groups;
} LodDeltaInfo;
int lod_delta_info(LodTree *tree, LodDeltaInfo *info);
int lod_read_delta(LodTree *tree, int32_t *splits, int32_t *vnode, int64_t *vstart, int64_t *vcount,
                   uint32_t *vcells, uint32_t *vrgba, int32_t *pnode, int64_t *pstart, int64_t *pcount);

/* Raw arena bytes [off, off+size) (Octree.grid, octree.py:275-279). */
int lod_read_arena(LodTree *tree, uint64_t off, uint64_t size, void *dst);

/* Whole-tree state as one contiguous DEVICE byte buffer (node table, chunk
 * pool, free stack, used arena bytes, counters), for replicating a tree to
 * other ranks (e.g. an NCCL broadcast before octant-prefix partitioning).
 * lod_tree_pack_size -> bytes; lod_tree_pack writes them to `dev_buf`;
 * lod_tree_unpack replaces `tree`'s state (same params, arena large enough). */
int lod_tree_pack_size(LodTree *tree, uint64_t *bytes);
int lod_tree_pack(LodTree *tree, void *dev_buf, uint64_t bytes);
int lod_tree_unpack(LodTree *tree, const void *dev_buf, uint64_t bytes);

/* _kernels.rasterize_nodes via render.rasterize (_kernels.py:290-339,
 * render.py:213-225): splat every sample of the listed nodes into the packed
 * u64 framebuffer (float32 depth bits << 32 | rgba, atomicMin).  cam is the
 * 18-double Camera.packed() block (render.py:68-82).  *samples = samples walked. */
int lod_rasterize(LodTree *tree, const int32_t *vis, int64_t nvis, const double *cam,
                  uint64_t *fb, int64_t width, int64_t height, int flags, int64_t *samples);

/* render.select_visible (render.py:177-200) on the device: the depth-first,
 * octant-ordered cut of nodes to draw.  planes = frustum_planes(camera)
 * (6 x (normal, d), render.py:127-148, computed by the caller like the
 * reference), cam = Camera.packed().  `selected` (host, capacity >= num_nodes)
 * receives the node ids in the reference's visit order; *n_selected their count. */
int lod_select_visible(LodTree *tree, const double *planes, const double *cam, double threshold,
                       int32_t *selected, int64_t capacity, int64_t *n_selected);

/* render.rasterize (render.py:213-225) in one call: device selection as in
 * lod_select_visible, then the chunk splat of lod_rasterize into fb (host
 * pointer, or device with LOD_FLAG_DEVICE_FB).  `selected` may be NULL. */
int lod_render(LodTree *tree, const double *planes, const double *cam, double threshold, uint64_t *fb,
               int64_t width, int64_t height, int flags, int32_t *selected, int64_t capacity,
               int64_t *n_selected, int64_t *samples);

/* _kernels.rasterize_points via render.brute_force_render (_kernels.py:342-372,
 * render.py:228-239).  device selects the GPU when no tree is involved. */
int lod_raster_points(int32_t device, const float *xyz, const uint32_t *rgba, int64_t n,
                      const double *cam, uint64_t *fb, int64_t width, int64_t height, int flags);

/* io.morton_key / io.morton_sort (io.py:419-446) on the device: keys_out gets
 * the 64-bit Morton keys in INPUT order (`bits` 1..21 per axis, x at bit 0,
 * then y, z; scale = (1 << bits) / size computed by the caller like the
 * reference); xyz_out / rgba_out get the stable reorder of the points by key.
 * Any output may be NULL (no sort runs when both record outputs are NULL);
 * rgba may be NULL when rgba_out is.  Host pointers, or device pointers with
 * LOD_FLAG_DEVICE_INPUT. */
int lod_morton_sort(int32_t device, const double *bmin, double scale, int32_t bits, const float *xyz,
                    const uint32_t *rgba, int64_t n, float *xyz_out, uint32_t *rgba_out, uint64_t *keys_out,
                    int flags);

/* Multi-GPU routing, local half: bucket a stripe of points by
 * owner rank -- owner_of_prefix[octant path over `depth` levels], the path
 * computed with the reference's float64 descent rule -- keeping input order
 * inside each bucket, as packed 16-byte records in out_records (bucket r at
 * starts[r], counts[r] records), and (out_positions, may be NULL) each
 * record's position in the stripe.  xyz / rgba / out_records / counts / starts
 * are DEVICE pointers; owner_of_prefix is a host array of 8^depth ranks;
 * `stream` is the cudaStream_t to order the work on (NULL = legacy default).
 * Asynchronous: counts / starts are valid once the stream reaches them. */
int lod_route_bucket(int32_t device, const double *bmin, double size, int32_t depth, const int32_t *owner_of_prefix,
                     int32_t world, const float *xyz, const uint32_t *rgba, int64_t n, void *out_records,
                     uint32_t *out_positions, int64_t *counts, int64_t *starts, void *stream);

/* Multi-GPU routing and composite over peer memory (the fused
 * replacement for the all-to-all and the all-reduce): each rank owns one
 * receive window -- an IPC-shareable device allocation (NVLink peer memory
 * between GPUs) -- and maps every peer's window (`windows[r]` = rank r's
 * window as seen by this process, its own included).  Window layout: the
 * header (LOD_WINDOW_HEADER_BYTES: two int64 count matrices [source][owner],
 * one per half, then per half every source's count-ready and data-ready
 * sequence flags and its extra word), two halves of `half_records` 16-byte records, two halves
 * of `half_records` uint32 stripe positions (each record's index in its
 * source stripe).  Batch k of a stream uses half k & 1 and sequence k + 1;
 * the ranks synchronise through the flags alone (no host barrier):
 *   lod_route_peers_begin   owners + bucket sizes of this rank's stripe,
 *                           stored as row `rank` of every peer's matrix with
 *                           a system-scope release of the count flag; then
 *                           waits (device warp + mapped host word) until
 *                           every rank's counts are in and copies the full
 *                           world x world matrix to `matrix` (host); one
 *                           int64 per rank rides along (`extra_dev`: a device
 *                           word of this rank, NULL = 0; `extra`: every
 *                           rank's, host, may be NULL);
 *   lod_route_peers_finish  the stable bucket scatter, each record written
 *                           straight into its owner's window half behind the
 *                           lower source ranks' records, then the data flags;
 *                           the stream then waits on the device until every
 *                           source's records are in (work queued behind it
 *                           -- the insert -- reads the half in global order).
 * A rank must not begin batch k before its own use of batch k - 2's half is
 * ordered on `stream` (the facade inserts on a stream ordered behind it).
 * host_wait != 0 (ranks time-sliced on ONE device, where a spinning wait
 * kernel holds the device for its whole time slice): both waits poll the
 * flags from the host with small copies instead, and finish returns once
 * every source's records are in.
 * lod_composite_min_peers: the depth-min of all ranks' framebuffers (`fbs`,
 * mapped windows of npix u64 each) over this rank's pixel slice, written back
 * into every framebuffer; after all ranks ran it (stream sync + barrier)
 * every framebuffer holds the composite.  Handles are
 * LOD_IPC_HANDLE_BYTES-byte cudaIpcMemHandle_t blobs. */
#define LOD_IPC_HANDLE_BYTES 64
#define LOD_WINDOW_HEADER_BYTES (2 * 64 * 64 * 8 + 6 * 64 * 8)
int lod_ipc_alloc(int32_t device, uint64_t bytes, void **ptr, void *handle); /* zeroed; free: lod_device_free */
int lod_ipc_open(int32_t device, const void *handle, void **ptr);
int lod_ipc_close(void *ptr);
int lod_route_peers_begin(int32_t device, const double *bmin, double size, int32_t depth,
                          const int32_t *owner_of_prefix, int32_t world, int32_t rank, const float *xyz, int64_t n,
                          void *const *windows, int32_t half, uint64_t seq, const int64_t *extra_dev,
                          int64_t *matrix, int64_t *extra, int32_t host_wait, void *stream);
int lod_route_peers_finish(int32_t device, int32_t world, int32_t rank, const float *xyz, const uint32_t *rgba,
                           int64_t n, void *const *windows, int32_t half, int64_t half_records, uint64_t seq,
                           int32_t host_wait, void *stream);
int lod_composite_min_peers(int32_t device, int32_t world, int32_t rank, void *const *fbs, int64_t npix,
                            void *stream);

/* Device-side helpers for benchmarking the resident path (inputs in HBM). */
int lod_device_alloc(int32_t device, uint64_t bytes, void **ptr);
int lod_device_free(void *ptr);
int lod_memcpy_h2d(void *dst, const void *src, uint64_t bytes);
int lod_memcpy_d2h(void *dst, const void *src, uint64_t bytes);
int lod_host_alloc(uint64_t bytes, void **ptr); /* pinned */
int lod_host_free(void *ptr);
int lod_fb_fill(int32_t device, uint64_t *fb_dev, int64_t n, uint64_t value);
int lod_l2_flush(int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* LOD_B200_H */
