/*
 * skip_sim.c -- design experiment (not product, not oracle): how many of a
 * leaf visit's 128-point chunks could a tile skip if it tested every query's
 * box lower bound against its k-th distance at the start of the visit?
 *
 * Input (raw little-endian files written by tools/skip_sim.py):
 *   tree: h, d, n, split[2^h-1], points[n*d] leaf-sorted, orig[n] i64, starts[2^h+1] i64
 *   queries: m, q[m*d]
 * Per leaf the points are re-ordered into 64-point blocks by widest-dimension
 * median splits (as engine.cu build_leaf_blocks), chunk = 2 adjacent blocks.
 * The traversal is the classic per-query order (= the reference's), f32 two
 * roundings, so kth at each visit start is the reference's.
 *
 * Output: per visit a record {round, leaf, qid, entry chunk, mask of chunks
 * that CANNOT be skipped}; then tiles = groups of T consecutive records of
 * one (round, leaf) in a chosen order, and the fraction of chunks a whole
 * tile could skip.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct { int32_t round, leaf, qid, entry; uint64_t need; float kth; } rec_t;

static int h, d, nl;
static int64_t n, m;
static float *split, *pts, *qs, *boxlo, *boxhi;
static int64_t *orig, *starts, *cbase; /* cbase: first chunk id of each leaf */
static int K = 10;

static float sqd(const float *q, const float *p) {
  float acc = 0.f;
  for (int j = 0; j < d; ++j) { float df = q[j] - p[j]; float s = df * df; acc = acc + s; }
  return acc;
}
static float lbox(const float *q, int64_t c) {
  double acc = 0;
  for (int j = 0; j < d; ++j) {
    float lo = boxlo[c * d + j], hi = boxhi[c * d + j];
    double e = q[j] < lo ? (double)lo - q[j] : (q[j] > hi ? (double)q[j] - hi : 0.0);
    acc += e * e;
  }
  return (float)acc;
}

/* widest-dim median recursion over idx[lo,hi) into nb blocks of 64 */
static float *gp; static int gdim;
static int cmpf(const void *a, const void *b) {
  float x = gp[(*(const int64_t *)a) * d + gdim], y = gp[(*(const int64_t *)b) * d + gdim];
  return x < y ? -1 : (x > y ? 1 : 0);
}
static void rec_blocks(int64_t *idx, int64_t lo, int64_t hi, int nb) {
  if (nb == 1) return;
  int64_t left = 64LL * ((nb + 1) / 2);
  int dim = 0; float best = -1;
  for (int j = 0; j < d; ++j) {
    float mn = pts[idx[lo] * d + j], mx = mn;
    for (int64_t i = lo + 1; i < hi; ++i) { float v = pts[idx[i] * d + j]; if (v < mn) mn = v; if (v > mx) mx = v; }
    if (mx - mn > best) { best = mx - mn; dim = j; }
  }
  gp = pts; gdim = dim;
  qsort(idx + lo, hi - lo, sizeof(int64_t), cmpf);
  rec_blocks(idx, lo, lo + left, (nb + 1) / 2);
  rec_blocks(idx, lo + left, hi, nb - (nb + 1) / 2);
}

static void insert(uint64_t *keys, uint64_t c) {
  if (!(c < keys[K - 1])) return;
  int i = K - 1;
  while (i > 0 && keys[i - 1] > c) { keys[i] = keys[i - 1]; --i; }
  keys[i] = c;
}
static uint64_t pack(float f, uint32_t i) { uint32_t b; memcpy(&b, &f, 4); return ((uint64_t)b << 32) | i; }
static float kdist(uint64_t k) { uint32_t b = (uint32_t)(k >> 32); float f; memcpy(&f, &b, 4); return f; }

static rec_t *recs; static int64_t *qoff; /* per query record offset (max visits cap) */
static int maxv;
static int32_t *nvis;

static void query(int64_t qi) {
  const float *q = qs + qi * d;
  uint64_t keys[64];
  for (int t = 0; t < K; ++t) keys[t] = 0x7F800000FFFFFFFFull;
  int64_t st[64]; int sp = 0; int64_t node = 0; const int64_t ni = ((int64_t)1 << h) - 1;
  int v = 0;
  for (;;) {
    while (node < ni) {
      int depth = 63 - __builtin_clzll((uint64_t)(node + 1));
      float sv = split[node];
      if (q[depth % d] < sv) { st[sp++] = 2 * node + 2; node = 2 * node + 1; }
      else { st[sp++] = 2 * node + 1; node = 2 * node + 2; }
    }
    int64_t leaf = node - ni;
    float kth = kdist(keys[K - 1]);
    int64_t c0 = cbase[leaf], c1 = cbase[leaf + 1];
    uint64_t need = 0; int entry = 0; float best = INFINITY;
    for (int64_t c = c0; c < c1 && c - c0 < 64; ++c) {
      float lb = lbox(q, c);
      if (lb < best) { best = lb; entry = (int)(c - c0); }
      if (!(lb * (1.0f - 1e-5f) > kth)) need |= 1ull << (c - c0);
    }
    if (v < maxv) {
      rec_t *r = &recs[qi * maxv + v];
      r->round = v; r->leaf = (int32_t)leaf; r->qid = (int32_t)qi; r->entry = entry; r->need = need; r->kth = kth;
    }
    ++v;
    for (int64_t r = starts[leaf]; r < starts[leaf + 1]; ++r) insert(keys, pack(sqd(q, pts + r * d), (uint32_t)orig[r]));
    node = -1;
    while (sp > 0) {
      int64_t far = st[--sp], par = (far - 1) >> 1;
      int depth = 63 - __builtin_clzll((uint64_t)(par + 1));
      float hp = q[depth % d] - split[par];
      float hp2 = hp * hp;
      if (!(hp2 > kdist(keys[K - 1]))) { node = far; break; }
    }
    if (node < 0) break;
  }
  nvis[qi] = v;
}

static int64_t next_q = 0; static pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
static void *worker(void *arg) {
  (void)arg;
  for (;;) {
    pthread_mutex_lock(&mu); int64_t a = next_q; next_q += 256; pthread_mutex_unlock(&mu);
    if (a >= m) break;
    int64_t b = a + 256 < m ? a + 256 : m;
    for (int64_t i = a; i < b; ++i) query(i);
  }
  return NULL;
}

static int order_mode;
static int cmprec(const void *A, const void *B) {
  const rec_t *a = A, *b = B;
  if (a->round != b->round) return a->round - b->round;
  if (a->leaf != b->leaf) return a->leaf - b->leaf;
  if (order_mode == 1 && a->entry != b->entry) return a->entry - b->entry;
  return a->qid - b->qid;
}

int main(int argc, char **argv) {
  if (argc < 4) { fprintf(stderr, "usage: skip_sim tree.bin queries.bin maxvisits [threads] [k]\n"); return 1; }
  FILE *f = fopen(argv[1], "rb");
  int32_t hd[2]; fread(hd, 4, 2, f); h = hd[0]; d = hd[1]; fread(&n, 8, 1, f);
  nl = 1 << h;
  split = malloc(4 * (nl - 1)); pts = malloc(4 * n * d); orig = malloc(8 * n); starts = malloc(8 * (nl + 1));
  fread(split, 4, nl - 1, f); fread(pts, 4, n * d, f); fread(orig, 8, n, f); fread(starts, 8, nl + 1, f); fclose(f);
  f = fopen(argv[2], "rb"); fread(&m, 8, 1, f); qs = malloc(4 * m * d); fread(qs, 4, m * d, f); fclose(f);
  maxv = atoi(argv[3]);
  int nth = argc > 4 ? atoi(argv[4]) : 8;
  if (argc > 5) K = atoi(argv[5]);
  /* re-order each leaf into blocks, chunk boxes */
  cbase = malloc(8 * (nl + 1)); cbase[0] = 0;
  for (int l = 0; l < nl; ++l) cbase[l + 1] = cbase[l] + (starts[l + 1] - starts[l] + 127) / 128;
  boxlo = malloc(4 * cbase[nl] * d); boxhi = malloc(4 * cbase[nl] * d);
  float *np_ = malloc(4 * n * d); int64_t *no = malloc(8 * n);
  for (int l = 0; l < nl; ++l) {
    int64_t s = starts[l], L = starts[l + 1] - s;
    int64_t *idx = malloc(8 * L);
    for (int64_t i = 0; i < L; ++i) idx[i] = s + i;
    rec_blocks(idx, 0, L, (int)((L + 63) / 64));
    for (int64_t i = 0; i < L; ++i) { memcpy(np_ + (s + i) * d, pts + idx[i] * d, 4 * d); no[s + i] = orig[idx[i]]; }
    free(idx);
  }
  memcpy(pts, np_, 4 * n * d); memcpy(orig, no, 8 * n); free(np_); free(no);
  for (int l = 0; l < nl; ++l)
    for (int64_t c = cbase[l]; c < cbase[l + 1]; ++c) {
      int64_t r0 = starts[l] + (c - cbase[l]) * 128, r1 = r0 + 128 < starts[l + 1] ? r0 + 128 : starts[l + 1];
      for (int j = 0; j < d; ++j) {
        float lo = INFINITY, hi = -INFINITY;
        for (int64_t r = r0; r < r1; ++r) { float v = pts[r * d + j]; if (v < lo) lo = v; if (v > hi) hi = v; }
        boxlo[c * d + j] = lo; boxhi[c * d + j] = hi;
      }
    }
  recs = calloc((size_t)m * maxv, sizeof(rec_t)); nvis = malloc(4 * m);
  pthread_t th[64];
  for (int t = 0; t < nth; ++t) pthread_create(&th[t], NULL, worker, NULL);
  for (int t = 0; t < nth; ++t) pthread_join(th[t], NULL);
  /* compact */
  int64_t nr = 0; double vis = 0; int trunc = 0;
  for (int64_t qi = 0; qi < m; ++qi) {
    int v = nvis[qi] < maxv ? nvis[qi] : maxv; if (nvis[qi] > maxv) trunc++;
    vis += nvis[qi];
    for (int j = 0; j < v; ++j) recs[nr++] = recs[qi * maxv + j];
  }
  printf("m=%lld mean visits %.2f truncated %d\n", (long long)m, vis / m, trunc);
  /* per-query skip fraction (non-home visits, home visits) */
  double tot[2] = {0, 0}, needc[2] = {0, 0};
  for (int64_t i = 0; i < nr; ++i) {
    int nc = (int)(cbase[recs[i].leaf + 1] - cbase[recs[i].leaf]); if (nc > 64) nc = 64;
    int hm = recs[i].round == 0;
    tot[hm] += nc; needc[hm] += __builtin_popcountll(recs[i].need);
  }
  printf("per-query needed chunk fraction: later visits %.4f, home visits %.4f\n", needc[0] / tot[0], needc[1] / tot[1]);
  int tiles[] = {1, 13, 26, 52, 128, 256};
  for (order_mode = 0; order_mode < 2; ++order_mode) {
    qsort(recs, nr, sizeof(rec_t), cmprec);
    for (int ti = 0; ti < 6; ++ti) {
      int T = tiles[ti];
      double tc = 0, tn = 0;
      int64_t i = 0;
      while (i < nr) {
        int64_t j = i;
        while (j < nr && recs[j].round == recs[i].round && recs[j].leaf == recs[i].leaf) ++j;
        if (recs[i].round > 0) {
          int nc = (int)(cbase[recs[i].leaf + 1] - cbase[recs[i].leaf]); if (nc > 64) nc = 64;
          for (int64_t a = i; a < j; a += T) {
            uint64_t u = 0;
            for (int64_t b = a; b < j && b < a + T; ++b) u |= recs[b].need;
            tc += nc; tn += __builtin_popcountll(u);
          }
        }
        i = j;
      }
      printf("order=%s tile=%d: later-visit needed chunk fraction %.4f\n", order_mode ? "entry" : "qid", T, tn / tc);
    }
  }
  return 0;
}
