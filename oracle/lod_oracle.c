/*
 * lod_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A sequential CPU restatement of the reference `lodstream` incremental LOD
 * update path and its two rasterizers, written in plain C so that it finishes
 * the 1M-point configs in about the time the numba reference does.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/pkg/src/lodstream/).  The restatement keeps the reference's
 * sequential semantics exactly, including its chunk-id assignment (touched-list
 * order in collect_allocs, LIFO free list), so its whole observable state is
 * bit-identical to the reference's; tests/test_oracle_golden.py pins that
 * against fixtures produced by the reference itself (tests/golden/make_golden.py).
 *
 * Float contract: compiled with -ffp-contract=off -fno-fast-math, so every
 * float64 expression rounds per operation in source order, like numba's LLVM
 * codegen (no FMA contraction).  Out-of-range float64 -> int64 conversions
 * follow x86 cvttsd2si (INT64_MIN), which is what numba emits.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NO_NODE (-1)
#define NO_CHUNK (-1)

enum { ORC_OK = 0, ORC_OUT_OF_ARENA = 1, ORC_SPILL_OVERFLOW = 2, ORC_BACKLOG_OVERFLOW = 3,
       ORC_NOMEM = 4, ORC_BAD_ARG = 5 };

typedef struct {
    double bmin[3];
    double size;
    int64_t grid_res;
    int64_t leaf_threshold;
    int64_t max_depth;
    int64_t chunk_capacity;
    uint64_t arena_bytes;
    int64_t backlog_capacity;
    int64_t spill_capacity;
} OrcParams;

typedef struct {
    int64_t n_batch, n_spill, n_voxels, n_splits, iterations;
} OrcBatchStats;

typedef struct {
    OrcParams p;
    /* node table, octree.py:169-182 */
    int64_t ncap, num_nodes, splits_total, max_level;
    int32_t *parent, *level, *children, *chunk_head, *chunk_tail, *chunk_count;
    uint8_t *octant, *inner, *final_;
    int64_t *count, *pending, *grid_off;
    double *bmin;
    double *size_by_level; /* octree.py:167 */
    int64_t grid_bytes;
    /* arena, store.py:34-78 */
    uint8_t *arena;
    uint64_t arena_cap, arena_off;
    /* chunk pool, store.py:81-166 */
    int64_t ccap, allocated_total, released_total;
    int32_t *next, *occupied;
    int64_t *payload_off;
    int32_t *free_;
    int64_t free_n, free_cap;
    /* spill buffer (update.py:106-140): records in 16-byte layout */
    float *spill_xyz;
    uint32_t *spill_rgba;
    int64_t spill_n, spill_cap_alloc, spill_high_water;
    /* voxel backlog (update.py:143-171) */
    int32_t *bnode, *bcell;
    uint32_t *brgba;
    int64_t blen_arr, backlog_high_water;
    /* scratch (update.py:206-213) */
    int32_t *touched, *vtouched, *leaf_ids, *alloc_node, *alloc_need, *cursor;
    int64_t *stamp;
    int64_t touched_cap, vtouched_cap, leaf_cap, alloc_cap, scratch_nodes;
    int64_t pass_no;
    /* BatchDelta capture (update.py:183-194, 333-355), on when collect_delta */
    int delta_on;
    int32_t *d_splits;            /* split nodes in split order */
    int64_t d_nsplits, d_splits_cap;
    int32_t *d_vnode;             /* per voxel group: node, start, count (ascending node) */
    int64_t *d_vstart, *d_vcount;
    int32_t *d_vcell;             /* voxel cells / colours, stable by node (claim order) */
    uint32_t *d_vrgba;
    int64_t d_nvgroups, d_nvox;
    int32_t *d_pnode;             /* per touched leaf: node, pre-store count, new points */
    int64_t *d_pstart, *d_pcount;
    int64_t d_npts;
} OrcTree;

/* x86 cvttsd2si: out-of-range / NaN -> INT64_MIN (numba np.int64(float)). */
static inline int64_t f2i64(double v) {
    if (v >= -9223372036854775808.0 && v < 9223372036854775808.0) return (int64_t)v;
    return INT64_MIN;
}

static void *xrealloc(void *p, size_t n) { return realloc(p, n ? n : 1); }

/* Octree._grow, octree.py:192-209 (doubling with the same fill values). */
static int grow_nodes(OrcTree *t, int64_t want) {
    if (want <= t->ncap) return 0;
    int64_t nc = t->ncap ? t->ncap : 1024;
    while (nc < want) nc *= 2;
    int64_t o = t->ncap;
#define GROW(field, type, per, fillexpr)                                                   \
    do {                                                                                   \
        type *np_ = (type *)xrealloc(t->field, sizeof(type) * (size_t)(nc * (per)));       \
        if (!np_) return ORC_NOMEM;                                                        \
        t->field = np_;                                                                    \
        for (int64_t i_ = o * (per); i_ < nc * (per); ++i_) np_[i_] = (fillexpr);          \
    } while (0)
    GROW(parent, int32_t, 1, NO_NODE);
    GROW(octant, uint8_t, 1, 0);
    GROW(level, int32_t, 1, 0);
    GROW(children, int32_t, 8, NO_NODE);
    GROW(inner, uint8_t, 1, 0);
    GROW(final_, uint8_t, 1, 0);
    GROW(count, int64_t, 1, 0);
    GROW(pending, int64_t, 1, 0);
    GROW(chunk_head, int32_t, 1, NO_CHUNK);
    GROW(chunk_tail, int32_t, 1, NO_CHUNK);
    GROW(chunk_count, int32_t, 1, 0);
    GROW(grid_off, int64_t, 1, -1);
    GROW(bmin, double, 3, 0.0);
#undef GROW
    t->ncap = nc;
    return 0;
}

/* Octree._new_node, octree.py:211-220 */
static int new_node(OrcTree *t, int32_t parent, int octant, const double bmin[3], int32_t level,
                    int64_t *out) {
    int64_t nid = t->num_nodes;
    if (nid >= t->ncap) {
        int rc = grow_nodes(t, nid + 1);
        if (rc) return rc;
    }
    t->parent[nid] = parent;
    t->octant[nid] = (uint8_t)octant;
    t->level[nid] = level;
    t->bmin[nid * 3 + 0] = bmin[0];
    t->bmin[nid * 3 + 1] = bmin[1];
    t->bmin[nid * 3 + 2] = bmin[2];
    t->num_nodes += 1;
    *out = nid;
    return 0;
}

/* Arena.alloc, store.py:51-69 (offset = -offset % align + offset). */
static int arena_alloc(OrcTree *t, uint64_t size, uint64_t align, uint64_t *off_out) {
    uint64_t off = t->arena_off;
    uint64_t rem = off % align;
    if (rem) off += align - rem;
    uint64_t end = off + size;
    if (end > t->arena_cap) return ORC_OUT_OF_ARENA;
    t->arena_off = end;
    *off_out = off;
    return 0;
}

/* ChunkPool.acquire, store.py:110-123 */
static int pool_acquire(OrcTree *t, int32_t *cid_out) {
    int32_t cid;
    if (t->free_n > 0) {
        cid = t->free_[--t->free_n];
    } else {
        cid = (int32_t)t->allocated_total;
        if (cid >= t->ccap) { /* ChunkPool._grow, store.py:104-108 */
            int64_t nc = t->ccap * 2;
            int32_t *nn = (int32_t *)xrealloc(t->next, sizeof(int32_t) * nc);
            if (!nn) return ORC_NOMEM;
            t->next = nn;
            int64_t *np_ = (int64_t *)xrealloc(t->payload_off, sizeof(int64_t) * nc);
            if (!np_) return ORC_NOMEM;
            t->payload_off = np_;
            int32_t *no = (int32_t *)xrealloc(t->occupied, sizeof(int32_t) * nc);
            if (!no) return ORC_NOMEM;
            t->occupied = no;
            for (int64_t i = t->ccap; i < nc; ++i) { nn[i] = NO_CHUNK; np_[i] = 0; no[i] = 0; }
            t->ccap = nc;
        }
        uint64_t off;
        int rc = arena_alloc(t, (uint64_t)t->p.chunk_capacity * 16u, 16u, &off);
        if (rc) return rc;
        t->payload_off[cid] = (int64_t)off;
        t->allocated_total += 1;
    }
    t->next[cid] = NO_CHUNK;
    t->occupied[cid] = 0;
    *cid_out = cid;
    return 0;
}

/* ChunkPool.release, store.py:125-143: push the chain in walk order. */
static int64_t pool_release(OrcTree *t, int32_t head) {
    int64_t n = 0;
    int32_t cid = head;
    while (cid != NO_CHUNK) {
        int32_t nxt = t->next[cid];
        t->occupied[cid] = 0;
        t->next[cid] = NO_CHUNK;
        if (t->free_n >= t->free_cap) {
            int64_t nc = t->free_cap ? t->free_cap * 2 : 1024;
            t->free_ = (int32_t *)xrealloc(t->free_, sizeof(int32_t) * nc);
            t->free_cap = nc;
        }
        t->free_[t->free_n++] = cid;
        t->released_total += 1;
        n += 1;
        cid = nxt;
    }
    return n;
}

OrcTree *orc_tree_create(const OrcParams *p) {
    if (!p || p->grid_res < 2 || (p->grid_res & 1) || p->chunk_capacity <= 0 || p->arena_bytes == 0)
        return NULL;
    OrcTree *t = (OrcTree *)calloc(1, sizeof(OrcTree));
    if (!t) return NULL;
    t->p = *p;
    t->arena_cap = (p->arena_bytes + 15u) / 16u * 16u; /* store.py:41-42 */
    t->arena = (uint8_t *)calloc(t->arena_cap, 1);
    if (!t->arena) { free(t); return NULL; }
    t->grid_bytes = p->grid_res * p->grid_res * p->grid_res / 8;
    t->size_by_level = (double *)malloc(sizeof(double) * (size_t)(p->max_depth + 2));
    for (int64_t k = 0; k < p->max_depth + 2; ++k) /* size * 0.5 ** arange(max_depth + 2) */
        t->size_by_level[k] = p->size * pow(0.5, (double)k);
    grow_nodes(t, 1024);
    t->ccap = 1024;
    t->next = (int32_t *)malloc(sizeof(int32_t) * 1024);
    t->payload_off = (int64_t *)calloc(1024, sizeof(int64_t));
    t->occupied = (int32_t *)calloc(1024, sizeof(int32_t));
    for (int i = 0; i < 1024; ++i) t->next[i] = NO_CHUNK;
    int64_t n0 = p->backlog_capacity < 4096 ? p->backlog_capacity : 4096; /* update.py:154 */
    t->blen_arr = n0;
    t->bnode = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n0 > 0 ? n0 : 1));
    t->bcell = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n0 > 0 ? n0 : 1));
    t->brgba = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n0 > 0 ? n0 : 1));
    int64_t root;
    new_node(t, NO_NODE, 0, p->bmin, 0, &root);
    return t;
}

void orc_tree_destroy(OrcTree *t) {
    if (!t) return;
    free(t->parent); free(t->octant); free(t->level); free(t->children); free(t->inner);
    free(t->final_); free(t->count); free(t->pending); free(t->chunk_head); free(t->chunk_tail);
    free(t->chunk_count); free(t->grid_off); free(t->bmin); free(t->size_by_level);
    free(t->arena); free(t->next); free(t->occupied); free(t->payload_off); free(t->free_);
    free(t->spill_xyz); free(t->spill_rgba); free(t->bnode); free(t->bcell); free(t->brgba);
    free(t->touched); free(t->vtouched); free(t->leaf_ids); free(t->alloc_node);
    free(t->alloc_need); free(t->cursor); free(t->stamp);
    free(t->d_splits); free(t->d_vnode); free(t->d_vstart); free(t->d_vcount); free(t->d_vcell);
    free(t->d_vrgba); free(t->d_pnode); free(t->d_pstart); free(t->d_pcount);
    free(t);
}

/* Octree.gather_samples, octree.py:298-326 */
int64_t orc_gather(const OrcTree *t, int64_t nid, int64_t start, float *xyz, uint32_t *rgba) {
    int64_t total = t->count[nid];
    int64_t k = total - start;
    if (k <= 0) return 0;
    int64_t cap = t->p.chunk_capacity;
    int32_t cid = t->chunk_head[nid];
    for (int64_t s = 0; s < start / cap; ++s) cid = t->next[cid];
    int64_t pos = start, out = 0;
    while (out < k) {
        const uint8_t *base = t->arena + t->payload_off[cid];
        int64_t lo = pos % cap;
        int64_t take = cap - lo < total - pos ? cap - lo : total - pos;
        for (int64_t r = 0; r < take; ++r) {
            const uint8_t *rec = base + 16 * (lo + r);
            memcpy(xyz + 3 * (out + r), rec, 12);
            memcpy(rgba + out + r, rec + 12, 4);
        }
        out += take;
        pos += take;
        cid = t->next[cid];
    }
    return k;
}

static int spill_append_node(OrcTree *t, int64_t nid) {
    int64_t n = t->count[nid];
    if (t->spill_n + n > t->p.spill_capacity) return ORC_SPILL_OVERFLOW; /* update.py:122-123 */
    if (t->spill_n + n > t->spill_cap_alloc) {
        int64_t nc = t->spill_cap_alloc ? t->spill_cap_alloc : 1024;
        while (nc < t->spill_n + n) nc *= 2;
        t->spill_xyz = (float *)xrealloc(t->spill_xyz, sizeof(float) * 3 * nc);
        t->spill_rgba = (uint32_t *)xrealloc(t->spill_rgba, sizeof(uint32_t) * nc);
        t->spill_cap_alloc = nc;
    }
    orc_gather(t, nid, 0, t->spill_xyz + 3 * t->spill_n, t->spill_rgba + t->spill_n);
    t->spill_n += n;
    if (t->spill_n > t->spill_high_water) t->spill_high_water = t->spill_n;
    return 0;
}

/* Octree.split, octree.py:222-264 */
static int split_node(OrcTree *t, int64_t nid) {
    int rc;
    if (t->count[nid]) {
        rc = spill_append_node(t, nid);
        if (rc) return rc;
    }
    if (t->chunk_head[nid] != NO_CHUNK) pool_release(t, t->chunk_head[nid]);
    t->chunk_head[nid] = NO_CHUNK;
    t->chunk_tail[nid] = NO_CHUNK;
    t->chunk_count[nid] = 0;
    t->count[nid] = 0;
    t->pending[nid] = 0;
    t->inner[nid] = 1;
    uint64_t goff;
    rc = arena_alloc(t, (uint64_t)t->grid_bytes, 64u, &goff);
    if (rc) return rc;
    t->grid_off[nid] = (int64_t)goff;
    /* node_size(nid) * 0.5; node_size = bounds.size * (0.5 ** level) (octree.py:268-269) */
    double half = t->p.size * pow(0.5, (double)t->level[nid]) * 0.5;
    double base[3] = {t->bmin[nid * 3], t->bmin[nid * 3 + 1], t->bmin[nid * 3 + 2]};
    int32_t lvl = t->level[nid] + 1;
    for (int o = 0; o < 8; ++o) {
        double cb[3] = {base[0] + ((o & 1) ? half : 0.0), base[1] + ((o & 2) ? half : 0.0),
                        base[2] + ((o & 4) ? half : 0.0)};
        int64_t kid;
        rc = new_node(t, (int32_t)nid, o, cb, lvl, &kid);
        if (rc) return rc;
        t->children[nid * 8 + o] = (int32_t)kid;
    }
    t->splits_total += 1;
    if (lvl > t->max_level) t->max_level = lvl;
    return 0;
}

/* Octree.append_chunk, octree.py:328-337 */
static int append_chunk(OrcTree *t, int64_t nid) {
    int32_t cid;
    int rc = pool_acquire(t, &cid);
    if (rc) return rc;
    if (t->chunk_head[nid] == NO_CHUNK) t->chunk_head[nid] = cid;
    else t->next[t->chunk_tail[nid]] = cid;
    t->chunk_tail[nid] = cid;
    t->chunk_count[nid] += 1;
    return 0;
}

/* point accessor over [spill || batch] */
typedef struct {
    const float *sx; const uint32_t *sc; int64_t ns;
    const float *bx; const uint32_t *bc; int64_t nb;
} Src;
static inline void src_get(const Src *s, int64_t i, double *x, double *y, double *z) {
    const float *p = i < s->ns ? s->sx + 3 * i : s->bx + 3 * (i - s->ns);
    *x = (double)p[0]; *y = (double)p[1]; *z = (double)p[2];
}
static inline const float *src_xyz(const Src *s, int64_t i) {
    return i < s->ns ? s->sx + 3 * i : s->bx + 3 * (i - s->ns);
}
static inline uint32_t src_rgba(const Src *s, int64_t i) {
    return i < s->ns ? s->sc[i] : s->bc[i - s->ns];
}

static void ensure_i32(int32_t **a, int64_t *cap, int64_t n) {
    if (*cap >= n) return;
    int64_t nc = *cap ? *cap : 1024;
    if (nc < n) nc = n > 2 * nc ? n : 2 * nc;
    *a = (int32_t *)xrealloc(*a, sizeof(int32_t) * nc);
    *cap = nc;
}

/* _kernels.count_points, _kernels.py:27-63 */
static int64_t count_points(OrcTree *t, const Src *s, int64_t nt) {
    const double bx0 = t->p.bmin[0], by0 = t->p.bmin[1], bz0 = t->p.bmin[2], size0 = t->p.size;
    int64_t n = s->ns + s->nb;
    for (int64_t i = 0; i < n; ++i) {
        double x, y, z;
        src_get(s, i, &x, &y, &z);
        int64_t nid = 0;
        double bx = bx0, by = by0, bz = bz0, sz = size0;
        while (t->inner[nid]) {
            double h = sz * 0.5;
            int o = 0;
            if (x >= bx + h) { o |= 1; bx += h; }
            if (y >= by + h) { o |= 2; by += h; }
            if (z >= bz + h) { o |= 4; bz += h; }
            sz = h;
            nid = t->children[nid * 8 + o];
        }
        if (t->final_[nid]) continue;
        if (t->pending[nid] == 0) t->touched[nt++] = (int32_t)nid;
        t->pending[nid] += 1;
    }
    return nt;
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* update._split_pass, update.py:226-249 */
static int split_pass(OrcTree *t, int32_t *ids, int64_t n, int64_t *n_splits) {
    *n_splits = 0;
    if (n == 0) return 0;
    /* np.sort returns a sorted copy: the touched list keeps first-touch order */
    int32_t *sorted = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    memcpy(sorted, ids, sizeof(int32_t) * (size_t)n);
    if (n > 1) qsort(sorted, (size_t)n, sizeof(int32_t), cmp_i32);
    int rc = 0;
    for (int64_t k = 0; k < n && !rc; ++k) {
        int64_t nid = sorted[k];
        if (t->count[nid] + t->pending[nid] > t->p.leaf_threshold && t->level[nid] < t->p.max_depth) {
            rc = split_node(t, nid);
            if (!rc) *n_splits += 1;
            if (!rc && t->delta_on) { /* events.append(("split", nid)), update.py:240-245 */
                if (t->d_nsplits == t->d_splits_cap) {
                    t->d_splits_cap = t->d_splits_cap ? 2 * t->d_splits_cap : 64;
                    t->d_splits = (int32_t *)xrealloc(t->d_splits, sizeof(int32_t) * t->d_splits_cap);
                }
                t->d_splits[t->d_nsplits++] = (int32_t)nid;
            }
        } else {
            t->final_[nid] = 1;
        }
    }
    free(sorted);
    return rc;
}

/* VoxelBacklog.ensure, update.py:159-168 (tracks the array length only). */
static void backlog_ensure(OrcTree *t, int64_t length, int64_t extra) {
    int64_t cap = t->p.backlog_capacity;
    int64_t want = length + extra < cap ? length + extra : cap;
    if (want > t->blen_arr) {
        int64_t size = want > 2 * t->blen_arr ? want : 2 * t->blen_arr;
        if (size > cap) size = cap;
        t->bnode = (int32_t *)xrealloc(t->bnode, sizeof(int32_t) * size);
        t->bcell = (int32_t *)xrealloc(t->bcell, sizeof(int32_t) * size);
        t->brgba = (uint32_t *)xrealloc(t->brgba, sizeof(uint32_t) * size);
        t->blen_arr = size;
    }
}

/* _kernels.sample_and_route, _kernels.py:66-152 */
static int sample_and_route(OrcTree *t, const Src *s, int64_t *blen_io, int64_t *vnt_io) {
    const double bx0 = t->p.bmin[0], by0 = t->p.bmin[1], bz0 = t->p.bmin[2], size0 = t->p.size;
    const int64_t g = t->p.grid_res;
    const double gd = (double)g;
    int64_t blen = *blen_io, nt = *vnt_io, cap = t->blen_arr;
    int overflow = 0;
    int64_t n = s->ns + s->nb;
    for (int64_t i = 0; i < n; ++i) {
        double x, y, z;
        src_get(s, i, &x, &y, &z);
        int64_t nid = 0;
        double bx = bx0, by = by0, bz = bz0, sz = size0;
        while (t->inner[nid]) {
            int64_t cx = f2i64(floor(gd * (x - bx) / sz));
            int64_t cy = f2i64(floor(gd * (y - by) / sz));
            int64_t cz = f2i64(floor(gd * (z - bz) / sz));
            if (cx < 0) cx = 0; else if (cx > g - 1) cx = g - 1;
            if (cy < 0) cy = 0; else if (cy > g - 1) cy = g - 1;
            if (cz < 0) cz = 0; else if (cz > g - 1) cz = g - 1;
            int64_t cell = cx + g * cy + g * g * cz;
            int64_t byte = t->grid_off[nid] + (cell >> 3);
            uint8_t mask = (uint8_t)(1u << (cell & 7));
            if ((t->arena[byte] & mask) == 0) {
                t->arena[byte] |= mask;
                if (blen < cap) {
                    t->bnode[blen] = (int32_t)nid;
                    t->bcell[blen] = (int32_t)cell;
                    t->brgba[blen] = src_rgba(s, i);
                    blen += 1;
                    if (t->pending[nid] == 0) t->vtouched[nt++] = (int32_t)nid;
                    t->pending[nid] += 1;
                } else {
                    overflow = 1;
                }
            }
            double h = sz * 0.5;
            int o = 0;
            if (x >= bx + h) { o |= 1; bx += h; }
            if (y >= by + h) { o |= 2; by += h; }
            if (z >= bz + h) { o |= 4; bz += h; }
            sz = h;
            nid = t->children[nid * 8 + o];
        }
        t->leaf_ids[i] = (int32_t)nid;
    }
    *blen_io = blen;
    *vnt_io = nt;
    return overflow;
}

static inline void write_record(OrcTree *t, int32_t cid, int64_t rel, float x, float y, float z,
                                uint32_t c) {
    uint8_t *rec = t->arena + t->payload_off[cid] + 16 * rel;
    memcpy(rec, &x, 4);
    memcpy(rec + 4, &y, 4);
    memcpy(rec + 8, &z, 4);
    memcpy(rec + 12, &c, 4);
}

/* cursor walk shared by store_points / store_voxels (_kernels.py:178-197, 233-250) */
static inline int32_t cursor_for(OrcTree *t, int64_t nid) {
    int64_t c = t->count[nid];
    if (t->stamp[nid] != t->pass_no) {
        t->stamp[nid] = t->pass_no;
        int32_t cid = t->chunk_head[nid];
        for (int64_t k = 0; k < c / t->p.chunk_capacity; ++k) cid = t->next[cid];
        t->cursor[nid] = cid;
    }
    return t->cursor[nid];
}

/* _kernels.store_points, _kernels.py:155-197 */
static void store_points(OrcTree *t, const Src *s) {
    int64_t n = s->ns + s->nb, cap = t->p.chunk_capacity;
    for (int64_t i = 0; i < n; ++i) {
        int64_t nid = t->leaf_ids[i];
        int64_t c = t->count[nid];
        int32_t cid = cursor_for(t, nid);
        int64_t rel = c % cap;
        const float *p = src_xyz(s, i);
        write_record(t, cid, rel, p[0], p[1], p[2], src_rgba(s, i));
        t->occupied[cid] += 1;
        t->count[nid] = c + 1;
        if (rel + 1 == cap) t->cursor[nid] = t->next[cid];
    }
}

/* _kernels.store_voxels, _kernels.py:200-250 */
static void store_voxels(OrcTree *t, int64_t n) {
    const int64_t g = t->p.grid_res, cap = t->p.chunk_capacity;
    const double gd = (double)g;
    for (int64_t i = 0; i < n; ++i) {
        int64_t nid = t->bnode[i];
        int64_t cell = t->bcell[i];
        int64_t cx = cell % g, cy = (cell / g) % g, cz = cell / (g * g);
        double step = t->size_by_level[t->level[nid]] / gd;
        double x = t->bmin[nid * 3 + 0] + ((double)cx + 0.5) * step;
        double y = t->bmin[nid * 3 + 1] + ((double)cy + 0.5) * step;
        double z = t->bmin[nid * 3 + 2] + ((double)cz + 0.5) * step;
        int64_t c = t->count[nid];
        int32_t cid = cursor_for(t, nid);
        int64_t rel = c % cap;
        write_record(t, cid, rel, (float)x, (float)y, (float)z, t->brgba[i]);
        t->occupied[cid] += 1;
        t->count[nid] = c + 1;
        if (rel + 1 == cap) t->cursor[nid] = t->next[cid];
    }
}

static void node_scratch(OrcTree *t) { /* UpdateState._node_scratch, update.py:215-223 */
    if (t->scratch_nodes >= t->num_nodes) return;
    int64_t n = t->scratch_nodes ? t->scratch_nodes : 1024;
    if (n < t->num_nodes) n = t->num_nodes > 2 * n ? t->num_nodes : 2 * n;
    t->stamp = (int64_t *)xrealloc(t->stamp, sizeof(int64_t) * n);
    t->cursor = (int32_t *)xrealloc(t->cursor, sizeof(int32_t) * n);
    for (int64_t i = t->scratch_nodes; i < n; ++i) { t->stamp[i] = -1; t->cursor[i] = -1; }
    t->scratch_nodes = n;
}

/* BatchDelta voxels / points (update.py:333-355), captured before the store
 * passes advance the counts: voxels grouped by node with a stable sort of the
 * backlog (claim order inside a node), points as (leaf, count, pending) over
 * the sorted touched leaves that are still leaves and received points. */
static void build_delta(OrcTree *t, int64_t blen, int64_t leaf_touch_end) {
    int64_t nn = t->num_nodes;
    int64_t *cnt = (int64_t *)calloc((size_t)nn + 1, sizeof(int64_t));
    for (int64_t i = 0; i < blen; ++i) cnt[t->bnode[i] + 1] += 1;
    t->d_nvgroups = 0;
    for (int64_t k = 0; k < nn; ++k) t->d_nvgroups += cnt[k + 1] > 0;
    t->d_vnode = (int32_t *)xrealloc(t->d_vnode, sizeof(int32_t) * (size_t)t->d_nvgroups);
    t->d_vstart = (int64_t *)xrealloc(t->d_vstart, sizeof(int64_t) * (size_t)t->d_nvgroups);
    t->d_vcount = (int64_t *)xrealloc(t->d_vcount, sizeof(int64_t) * (size_t)t->d_nvgroups);
    int64_t g = 0;
    for (int64_t k = 0; k < nn; ++k) {
        if (cnt[k + 1]) { t->d_vnode[g] = (int32_t)k; t->d_vcount[g] = cnt[k + 1]; g++; }
        cnt[k + 1] += cnt[k];
    }
    for (int64_t q = 0; q < g; ++q) t->d_vstart[q] = cnt[t->d_vnode[q]];
    t->d_vcell = (int32_t *)xrealloc(t->d_vcell, sizeof(int32_t) * (size_t)blen);
    t->d_vrgba = (uint32_t *)xrealloc(t->d_vrgba, sizeof(uint32_t) * (size_t)blen);
    for (int64_t i = 0; i < blen; ++i) {
        int64_t pos = cnt[t->bnode[i]]++;
        t->d_vcell[pos] = t->bcell[i];
        t->d_vrgba[pos] = t->brgba[i];
    }
    t->d_nvox = blen;
    free(cnt);
    int32_t *ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(leaf_touch_end ? leaf_touch_end : 1));
    memcpy(ids, t->touched, sizeof(int32_t) * (size_t)leaf_touch_end);
    qsort(ids, (size_t)leaf_touch_end, sizeof(int32_t), cmp_i32);
    t->d_pnode = (int32_t *)xrealloc(t->d_pnode, sizeof(int32_t) * (size_t)leaf_touch_end);
    t->d_pstart = (int64_t *)xrealloc(t->d_pstart, sizeof(int64_t) * (size_t)leaf_touch_end);
    t->d_pcount = (int64_t *)xrealloc(t->d_pcount, sizeof(int64_t) * (size_t)leaf_touch_end);
    t->d_npts = 0;
    for (int64_t k = 0; k < leaf_touch_end; ++k) {
        int32_t nid = ids[k];
        if (!t->inner[nid] && t->pending[nid] > 0) {
            t->d_pnode[t->d_npts] = nid;
            t->d_pstart[t->d_npts] = t->count[nid];
            t->d_pcount[t->d_npts] = t->pending[nid];
            t->d_npts++;
        }
    }
    free(ids);
}

/* update.insert_batch, update.py:252-393; with t->delta_on the BatchDelta of
 * the cycle is captured (update.py:333-355) and read with orc_delta_view. */
int orc_insert_batch(OrcTree *t, const float *xyz, const uint32_t *rgba, int64_t n_batch,
                     OrcBatchStats *st) {
    memset(st, 0, sizeof(*st));
    st->n_batch = n_batch;
    t->d_nsplits = t->d_nvgroups = t->d_nvox = t->d_npts = 0;
    if (n_batch == 0) return 0; /* update.py:266-268 */
    int rc;
    Src s = {NULL, NULL, 0, xyz, rgba, n_batch};
    /* expansion, update.py:274-296 */
    ensure_i32(&t->touched, &t->touched_cap, n_batch + 8);
    int64_t nt = count_points(t, &s, 0);
    int64_t leaf_touch_end = nt, n_splits, iters = 1;
    rc = split_pass(t, t->touched, nt, &n_splits);
    st->n_splits += n_splits;
    if (rc) return rc;
    if (t->spill_n) { s.sx = t->spill_xyz; s.sc = t->spill_rgba; s.ns = t->spill_n; }
    int64_t n_all = s.ns + s.nb;
    st->n_spill = s.ns;
    while (n_splits) {
        ensure_i32(&t->touched, &t->touched_cap, leaf_touch_end + n_all + 8);
        nt = count_points(t, &s, leaf_touch_end);
        int32_t *fresh = t->touched + leaf_touch_end;
        int64_t nf = nt - leaf_touch_end;
        leaf_touch_end = nt;
        iters += 1;
        rc = split_pass(t, fresh, nf, &n_splits);
        st->n_splits += n_splits;
        if (rc) return rc;
    }
    st->iterations = iters;
    /* sampling, update.py:299-315 */
    node_scratch(t);
    ensure_i32(&t->vtouched, &t->vtouched_cap, t->num_nodes + 8);
    ensure_i32(&t->leaf_ids, &t->leaf_cap, n_all);
    int64_t ml = t->max_level > 1 ? t->max_level : 1;
    backlog_ensure(t, 0, n_all * ml);
    int64_t blen = 0, vnt = 0;
    int overflow = sample_and_route(t, &s, &blen, &vnt);
    if (overflow) return ORC_BACKLOG_OVERFLOW;
    st->n_voxels = blen;
    if (blen > t->backlog_high_water) t->backlog_high_water = blen;
    /* allocation, update.py:318-331 (collect_allocs, _kernels.py:253-277) */
    t->pass_no += 1;
    ensure_i32(&t->alloc_node, &t->alloc_cap, leaf_touch_end + vnt);
    {
        int64_t cap = t->p.chunk_capacity;
        for (int src = 0; src < 2; ++src) {
            int32_t *lst = src == 0 ? t->touched : t->vtouched;
            int64_t nl = src == 0 ? leaf_touch_end : vnt;
            for (int64_t i = 0; i < nl; ++i) {
                int64_t nid = lst[i];
                if (t->stamp[nid] == t->pass_no) continue;
                t->stamp[nid] = t->pass_no;
                int64_t need = (t->count[nid] + t->pending[nid] + cap - 1) / cap - t->chunk_count[nid];
                for (int64_t k = 0; k < need; ++k) {
                    rc = append_chunk(t, nid);
                    if (rc) return rc;
                }
            }
        }
    }
    if (t->delta_on) build_delta(t, blen, leaf_touch_end);
    /* store, update.py:358-373 */
    t->pass_no += 1;
    store_points(t, &s);
    if (blen) {
        t->pass_no += 1;
        store_voxels(t, blen);
    }
    /* cleanup, update.py:376-380 (clear_marks, _kernels.py:280-287) */
    for (int64_t i = 0; i < leaf_touch_end; ++i) {
        t->pending[t->touched[i]] = 0;
        t->final_[t->touched[i]] = 0;
    }
    for (int64_t i = 0; i < vnt; ++i) t->pending[t->vtouched[i]] = 0;
    t->spill_n = 0;
    return 0;
}

/* ---- rasterizers, _kernels.py:290-372 ---------------------------------- */

static inline void splat(const double *cam, int64_t w, int64_t h, double x, double y, double z,
                         uint32_t rgba, uint64_t *fb) {
    double dx = x - cam[0], dy = y - cam[1], dz = z - cam[2];
    double zv = dx * cam[9] + dy * cam[10] + dz * cam[11];
    if (zv <= cam[14] || zv >= cam[15]) return;
    double xv = dx * cam[3] + dy * cam[4] + dz * cam[5];
    double yv = dx * cam[6] + dy * cam[7] + dz * cam[8];
    double ndc_x = xv / (zv * cam[12] * cam[13]);
    double ndc_y = yv / (zv * cam[12]);
    int64_t px = f2i64(floor((ndc_x + 1.0) * 0.5 * cam[16]));
    int64_t py = f2i64(floor((1.0 - ndc_y) * 0.5 * cam[17]));
    if (px < 0 || px >= w || py < 0 || py >= h) return;
    double d01 = cam[15] * (zv - cam[14]) / ((cam[15] - cam[14]) * zv);
    float df = (float)d01;
    uint32_t bits;
    memcpy(&bits, &df, 4);
    uint64_t packed = ((uint64_t)bits << 32) | (uint64_t)rgba;
    int64_t idx = py * w + px;
    if (packed < fb[idx]) fb[idx] = packed;
}

/* _kernels.rasterize_nodes, _kernels.py:290-339 */
int64_t orc_rasterize_nodes(const OrcTree *t, const int32_t *vis, int64_t nvis, const double *cam,
                            uint64_t *fb) {
    int64_t w = f2i64(cam[16]), h = f2i64(cam[17]), touched = 0;
    for (int64_t k = 0; k < nvis; ++k) {
        int32_t cid = t->chunk_head[vis[k]];
        while (cid != NO_CHUNK) {
            const uint8_t *base = t->arena + t->payload_off[cid];
            int32_t occ = t->occupied[cid];
            for (int32_t s = 0; s < occ; ++s) {
                float p[3];
                uint32_t c;
                memcpy(p, base + 16 * s, 12);
                memcpy(&c, base + 16 * s + 12, 4);
                touched += 1;
                splat(cam, w, h, (double)p[0], (double)p[1], (double)p[2], c, fb);
            }
            cid = t->next[cid];
        }
    }
    return touched;
}

/* _kernels.rasterize_points, _kernels.py:342-372 */
void orc_rasterize_points(const float *xyz, const uint32_t *rgba, int64_t n, const double *cam,
                          uint64_t *fb) {
    int64_t w = f2i64(cam[16]), h = f2i64(cam[17]);
    for (int64_t i = 0; i < n; ++i)
        splat(cam, w, h, (double)xyz[3 * i], (double)xyz[3 * i + 1], (double)xyz[3 * i + 2], rgba[i], fb);
}

/* ---- state export for the Python wrapper -------------------------------- */

typedef struct {
    int64_t num_nodes, splits_total, max_level, ncap;
    int64_t allocated_total, released_total, free_count, ccap;
    uint64_t arena_offset, arena_capacity;
    int64_t spill_high_water, backlog_high_water;
    int32_t *parent, *level, *children, *chunk_head, *chunk_tail, *chunk_count;
    uint8_t *octant, *inner, *final_;
    int64_t *count, *pending, *grid_off;
    double *bmin;
    int32_t *next, *occupied, *free_list;
    int64_t *payload_off;
    uint8_t *arena;
} OrcView;

void orc_view(const OrcTree *t, OrcView *v) {
    v->num_nodes = t->num_nodes; v->splits_total = t->splits_total; v->max_level = t->max_level;
    v->ncap = t->ncap; v->allocated_total = t->allocated_total; v->released_total = t->released_total;
    v->free_count = t->free_n; v->ccap = t->ccap; v->arena_offset = t->arena_off;
    v->arena_capacity = t->arena_cap; v->spill_high_water = t->spill_high_water;
    v->backlog_high_water = t->backlog_high_water;
    v->parent = t->parent; v->level = t->level; v->children = t->children;
    v->chunk_head = t->chunk_head; v->chunk_tail = t->chunk_tail; v->chunk_count = t->chunk_count;
    v->octant = t->octant; v->inner = t->inner; v->final_ = t->final_; v->count = t->count;
    v->pending = t->pending; v->grid_off = t->grid_off; v->bmin = t->bmin; v->next = t->next;
    v->occupied = t->occupied; v->free_list = t->free_; v->payload_off = t->payload_off;
    v->arena = t->arena;
}

/* ---- BatchDelta export (collect_delta=True) ------------------------------ */

typedef struct {
    int64_t n_splits, n_voxel_groups, n_voxels, n_point_groups;
    int32_t *splits, *vnode, *vcell, *pnode;
    int64_t *vstart, *vcount, *pstart, *pcount;
    uint32_t *vrgba;
} OrcDeltaView;

void orc_set_delta(OrcTree *t, int on) { t->delta_on = on; }

void orc_delta_view(const OrcTree *t, OrcDeltaView *v) {
    v->n_splits = t->d_nsplits; v->n_voxel_groups = t->d_nvgroups; v->n_voxels = t->d_nvox;
    v->n_point_groups = t->d_npts;
    v->splits = t->d_splits; v->vnode = t->d_vnode; v->vcell = t->d_vcell; v->pnode = t->d_pnode;
    v->vstart = t->d_vstart; v->vcount = t->d_vcount; v->pstart = t->d_pstart; v->pcount = t->d_pcount;
    v->vrgba = t->d_vrgba;
}
