/*
 * bkt_oracle.c -- CPU restatement of the reference bufferknn query path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the
 * "port" CPU baseline timed by bench.py's cpu_baseline / --impl reference
 * legs).  Only tests/, __graft_entry__.smoke() and bench.py may load it.
 * The product (paper_1512_02831_b200) never links or calls it.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/bufferknn
 * in the build container and stores its outputs); see tests/test_oracle.py.
 *
 * Everything here restates reference semantics, each function citing the
 * reference file:line it follows.  Compile with -ffp-contract=off: the
 * reference distance has two roundings per dimension (no FMA).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define OR_INDEX_SENTINEL 0xFFFFFFFFu               /* core.py:39 */
#define OR_EMPTY_KEY 0x7F800000FFFFFFFFull          /* core.py:41-45: (inf bits << 32) | sentinel */

/* core.py:108-122 (sq_euclidean) / core.py:138-146 (sq_distances_block):
 * acc = 0; for j: diff = q[j] - p[j]; acc = acc + diff*diff, all float32. */
static float or_sq_dist(const float *q, const float *p, int d) {
    float acc = 0.0f;
    for (int j = 0; j < d; ++j) {
        float diff = q[j] - p[j];
        float sq = diff * diff;
        acc = acc + sq;
    }
    return acc;
}

/* core.py:152-160 (pack_keys): (float32 bits << 32) | index. */
static uint64_t or_pack(float dist, uint32_t idx) {
    uint32_t bits;
    memcpy(&bits, &dist, 4);
    return ((uint64_t)bits << 32) | (uint64_t)idx;
}

static float or_key_dist(uint64_t key) {
    uint32_t bits = (uint32_t)(key >> 32);
    float f;
    memcpy(&f, &bits, 4);
    return f;
}

/* kdtree.py:46-52 (_float_order_bits): order-preserving map float32 -> uint32. */
static uint32_t or_order_bits(float v) {
    uint32_t b;
    memcpy(&b, &v, 4);
    return (b & 0x80000000u) ? ~b : (b ^ 0x80000000u);
}

/* Top-k insertion.  core.py:251-262 (NeighborBatch.update_rows) keeps the k
 * smallest keys of (existing U candidates) ascending; candidate keys are
 * unique per query (each reference row is scanned at most once), so a
 * strict-less insertion into an ascending array is the same selection. */
static void or_topk_insert(uint64_t *keys, int k, uint64_t c) {
    if (!(c < keys[k - 1])) return;
    int i = k - 1;
    while (i > 0 && keys[i - 1] > c) {
        keys[i] = keys[i - 1];
        --i;
    }
    keys[i] = c;
}

/* ---------------------------------------------------------------- build */

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/*
 * buffer_tree.py:149-197 (build_buffer_tree) + kdtree.py:55-70 (median_split).
 * Level by level, each subset is ordered by key = order_bits(coord[dim]) << 32 | idx
 * with dim = depth % d; the split value is the coordinate at position s//2;
 * left = positions [0, s//2), right = [s//2, s).  Split values are stored in
 * level order (node j's children 2j+1, 2j+2).  Within-leaf order is not part
 * of the contract (the reference leaves numpy's introselect order); here each
 * subset is fully sorted by key, which yields the same sets.
 * Returns 0, or -1 on bad arguments.
 */
int or_build_tree(const float *refs, int64_t n, int d, int h,
                  float *split_out, int64_t *order_out, int64_t *leaf_starts_out) {
    if (h < 1 || d < 1 || n < ((int64_t)1 << h)) return -1;
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * n);
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * n);
    int64_t nsub_max = (int64_t)1 << h;
    int64_t *starts = (int64_t *)malloc(sizeof(int64_t) * (nsub_max + 1));
    int64_t *nstarts = (int64_t *)malloc(sizeof(int64_t) * (nsub_max + 1));
    if (!cur || !keys || !starts || !nstarts) { free(cur); free(keys); free(starts); free(nstarts); return -2; }
    for (int64_t i = 0; i < n; ++i) cur[i] = i;
    starts[0] = 0; starts[1] = n;
    int64_t nsub = 1, node = 0;
    for (int depth = 0; depth < h; ++depth) {
        int dim = depth % d;
        for (int64_t s = 0; s < nsub; ++s) {
            int64_t lo = starts[s], hi = starts[s + 1], sz = hi - lo, mid = sz / 2;
            for (int64_t t = lo; t < hi; ++t)
                keys[t] = ((uint64_t)or_order_bits(refs[cur[t] * d + dim]) << 32) | (uint64_t)cur[t];
            qsort(keys + lo, (size_t)sz, sizeof(uint64_t), cmp_u64);
            for (int64_t t = lo; t < hi; ++t) cur[t] = (int64_t)(keys[t] & 0xFFFFFFFFull);
            split_out[node++] = refs[cur[lo + mid] * d + dim];
            nstarts[2 * s] = lo;
            nstarts[2 * s + 1] = lo + mid;
        }
        nstarts[2 * nsub] = n;
        nsub *= 2;
        memcpy(starts, nstarts, sizeof(int64_t) * (nsub + 1));
    }
    memcpy(order_out, cur, sizeof(int64_t) * n);
    memcpy(leaf_starts_out, starts, sizeof(int64_t) * (nsub + 1));
    free(cur); free(keys); free(starts); free(nstarts);
    return 0;
}

/* -------------------------------------------------------------- search */

typedef struct {
    int h, d, k;
    int64_t n;
    const float *split;       /* 2^h - 1, level order */
    const float *points;      /* n x d, leaf-sorted */
    const int64_t *orig;      /* n */
    const int64_t *leaf_starts; /* 2^h + 1 */
    const float *queries;     /* m x d */
    int64_t m;
    uint64_t *keys_out;       /* m x k ascending */
    int32_t *visited_out;     /* m, may be NULL */
    int32_t *seq_out;         /* m x max_seq, may be NULL; unused entries -1 */
    int max_seq;
    int64_t *pairs_out;       /* per worker pair count, may be NULL */
    int64_t q_lo, q_hi;
    int worker;
} or_job;

/*
 * One query, classic traversal order: kdtree.py:157-204 (query_kdtree), which
 * the reference proves equal to lazy_search's per-query leaf sequence
 * (tests/test_acceptance.py:206-231).  Descent: go left iff q[sd] < split
 * (strict, buffer_tree.py:370); after the near subtree returns, the far one
 * is visited unless (q[sd]-split)^2 > kth in float32 (buffer_tree.py:346-347),
 * kth = current k-th key's distance (+inf until k candidates, core.py:269-271).
 * Implemented with an explicit stack of (node, pending-far) frames.
 */
static void or_query_one(const or_job *J, int64_t qi, uint64_t *keys, int64_t *pairs) {
    const int h = J->h, d = J->d, k = J->k;
    const float *q = J->queries + qi * d;
    const int64_t n_internal = ((int64_t)1 << h) - 1;
    for (int t = 0; t < k; ++t) keys[t] = OR_EMPTY_KEY;
    int32_t nvis = 0;
    /* stack of far children still to consider (node ids), with parent info */
    int64_t stack[64];
    int sp = 0;
    int64_t node = 0;
    for (;;) {
        /* descend from `node` to a leaf, pushing far children */
        while (node < n_internal) {
            int sd = (int)(/*levels[node]*/ 0) ;
            /* depth of node in level order: floor(log2(node+1)) */
            int depth = 63 - __builtin_clzll((uint64_t)(node + 1));
            sd = depth % d;
            float sv = J->split[node];
            int64_t left = 2 * node + 1, right = 2 * node + 2;
            if (q[sd] < sv) { stack[sp++] = right; node = left; }
            else            { stack[sp++] = left;  node = right; }
        }
        int64_t leaf = node - n_internal;
        int64_t lo = J->leaf_starts[leaf], hi = J->leaf_starts[leaf + 1];
        for (int64_t r = lo; r < hi; ++r) {
            float dist = or_sq_dist(q, J->points + r * d, d);
            or_topk_insert(keys, k, or_pack(dist, (uint32_t)J->orig[r]));
        }
        *pairs += hi - lo;
        if (J->seq_out && nvis < J->max_seq) J->seq_out[qi * J->max_seq + nvis] = (int32_t)leaf;
        ++nvis;
        /* pop until a far child survives the slab test */
        node = -1;
        while (sp > 0) {
            int64_t far = stack[--sp];
            int64_t parent = (far - 1) >> 1;
            int depth = 63 - __builtin_clzll((uint64_t)(parent + 1));
            int sd = depth % d;
            float hp = q[sd] - J->split[parent];
            float hp2 = hp * hp;
            float kth = or_key_dist(keys[k - 1]);
            if (!(hp2 > kth)) { node = far; break; }
        }
        if (node < 0) break;
    }
    if (J->visited_out) J->visited_out[qi] = nvis;
}

static void *or_worker(void *arg) {
    or_job *J = (or_job *)arg;
    int64_t pairs = 0;
    for (int64_t qi = J->q_lo; qi < J->q_hi; ++qi)
        or_query_one(J, qi, J->keys_out + qi * J->k, &pairs);
    if (J->pairs_out) J->pairs_out[J->worker] = pairs;
    return NULL;
}

/*
 * k-NN of m queries over a built buffer tree, results in the reference's
 * NeighborBatch.keys layout ((m, k) uint64 ascending, core.py:230-262).
 * visited_out: per-query visited-leaf count (SearchStats.visited_per_query,
 * buffer_tree.py:447, 643-644).  seq_out: per-query leaf sequence
 * (SearchStats.leaf_sequences), truncated to max_seq.  Returns total pairs.
 */
int64_t or_knn_tree(int h, int d, int64_t n, const float *split, const float *points,
                    const int64_t *orig, const int64_t *leaf_starts,
                    const float *queries, int64_t m, int k,
                    uint64_t *keys_out, int32_t *visited_out,
                    int32_t *seq_out, int max_seq, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (h > 60 || k < 1) return -1;
    if (seq_out) for (int64_t i = 0; i < m * (int64_t)max_seq; ++i) seq_out[i] = -1;
    or_job *jobs = (or_job *)calloc((size_t)nthreads, sizeof(or_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    int64_t *pairs = (int64_t *)calloc((size_t)nthreads, sizeof(int64_t));
    for (int w = 0; w < nthreads; ++w) {
        or_job *J = &jobs[w];
        J->h = h; J->d = d; J->k = k; J->n = n; J->split = split; J->points = points;
        J->orig = orig; J->leaf_starts = leaf_starts; J->queries = queries; J->m = m;
        J->keys_out = keys_out; J->visited_out = visited_out; J->seq_out = seq_out;
        J->max_seq = max_seq; J->pairs_out = pairs; J->worker = w;
        J->q_lo = m * w / nthreads; J->q_hi = m * (w + 1) / nthreads;
    }
    for (int w = 1; w < nthreads; ++w) pthread_create(&th[w], NULL, or_worker, &jobs[w]);
    or_worker(&jobs[0]);
    for (int w = 1; w < nthreads; ++w) pthread_join(th[w], NULL);
    int64_t total = 0;
    for (int w = 0; w < nthreads; ++w) total += pairs[w];
    free(jobs); free(th); free(pairs);
    return total;
}

/* ---------------------------------------------------------------- brute */

typedef struct {
    const float *refs; int64_t n; int d;
    const float *queries; int k;
    uint64_t *keys_out;
    int64_t q_lo, q_hi;
} or_bjob;

static void *or_bworker(void *arg) {
    or_bjob *J = (or_bjob *)arg;
    for (int64_t qi = J->q_lo; qi < J->q_hi; ++qi) {
        uint64_t *keys = J->keys_out + qi * J->k;
        for (int t = 0; t < J->k; ++t) keys[t] = OR_EMPTY_KEY;
        const float *q = J->queries + qi * J->d;
        for (int64_t r = 0; r < J->n; ++r)
            or_topk_insert(keys, J->k, or_pack(or_sq_dist(q, J->refs + r * J->d, J->d), (uint32_t)r));
    }
    return NULL;
}

/* brute.py:41-80 (brute_knn): exhaustive scan, same keys as the tree engines. */
int or_brute(const float *refs, int64_t n, int d, const float *queries, int64_t m,
             int k, uint64_t *keys_out, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (k < 1) return -1;
    or_bjob *jobs = (or_bjob *)calloc((size_t)nthreads, sizeof(or_bjob));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int w = 0; w < nthreads; ++w) {
        or_bjob *J = &jobs[w];
        J->refs = refs; J->n = n; J->d = d; J->queries = queries; J->k = k; J->keys_out = keys_out;
        J->q_lo = m * w / nthreads; J->q_hi = m * (w + 1) / nthreads;
    }
    for (int w = 1; w < nthreads; ++w) pthread_create(&th[w], NULL, or_bworker, &jobs[w]);
    or_bworker(&jobs[0]);
    for (int w = 1; w < nthreads; ++w) pthread_join(th[w], NULL);
    free(jobs); free(th);
    return 0;
}
