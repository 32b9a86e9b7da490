// engine.cu -- context, tree residency, the device-resident LazySearch round
// loop and the C ABI of libbkt.so (include/bkt.h).
//
// Reference mapping:
//   bkt_open / bkt_close   <- device.py:361-364 device_init, SimulatedDevice.close (351-358)
//   bkt_load_tree          <- ChunkPipeline staging of the leaf structure (device.py:380-420)
//   bkt_search             <- lazy_search (buffer_tree.py:523-646), Alg. 1 of PAPER.md
//   bkt_scan_groups        <- SimulatedDevice.enqueue_brute_kernel (device.py:283-337)
//
// Device data layout (HBM):
//   split      f32[2^h-1]                       top tree, level order
//   quad_base  i64[2^h+1]                       first quad of each leaf; leaves padded to 4 points
//   leaf_size  i32[2^h]                         real points per leaf
//   pts        f32[total_quads * 4 * D]         quad g, dim j, point t at g*4D + 4j + t
//   pidx       u32[total_quads * 4]             original row of each point (padding: 0xFFFFFFFF)
//   per batch of m queries: q f32[m*D], keys u64[m*k], state u32[m], next i32[m],
//   visits u32[m], bucket slot per work-list position int2[m], two work lists i32[m]; per leaf: counts, leaf_off, tile_off.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bkt.h"
#include "dims.h"
#include "leafscan_tc.cuh"
#include "round_kernels.cuh"
#include "split_launch.cuh"
#include "wide_search.cuh"
#include "seam.h"

using namespace bkt;

namespace bkt {
cudaError_t launch_leafscan_tc(int kt, int kb, bool fma, int grid, cudaStream_t s, const TcArgs& a, int* occ,
                               int nr, int cps);
}

namespace {
thread_local std::string g_thread_err;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct LaunchCfg {
  int grid = 0;
};
}  // namespace

struct bkt_ctx {
  int device = 0;
  int sm_count = 0;
  int sm_clock_khz = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;
  std::string err;

  // ---- tree
  bool has_tree = false;
  int h = 0, d = 0, D = 0, nl = 0;
  long long n = 0, total_quads = 0;
  float* split = nullptr;
  long long* quad_base = nullptr;
  int* leaf_size = nullptr;
  float* pts = nullptr;
  uint32_t* pidx = nullptr;
  // general-domain trees (h > 16 or d > 32): only the wide path (wide_search.cuh)
  bool wide_only = false;
  const float* wide_pts = nullptr;      // quad layout the wide kernel reads (HBM, or mapped host memory)
  const uint32_t* wide_pidx = nullptr;
  uint64_t* wide_scratch = nullptr;     // per-CTA top-k rows when 2k keys exceed shared memory
  long long wide_scratch_elems = 0;
  // host-resident (out-of-core) leaf structure
  int residency = 0;
  float* h_pts = nullptr;
  uint32_t* h_pidx = nullptr;
  std::vector<long long> h_quad_base;
  std::vector<int> h_leaf_size;
  int num_chunks = 1;
  std::vector<long long> chunk_q;      // chunk j = quads [chunk_q[j], chunk_q[j+1])
  std::vector<int> chunk_leaf_lo, chunk_leaf_hi;  // leaves overlapping chunk j: [lo, hi]
  float* slot_pts[2] = {nullptr, nullptr};
  uint32_t* slot_idx[2] = {nullptr, nullptr};
  int slot_chunk[2] = {-1, -1};
  cudaEvent_t slot_free[2] = {nullptr, nullptr};
  cudaEvent_t slot_ready[2] = {nullptr, nullptr};
  long long slot_quads = 0;
  // out-of-core drain: leaf-aligned streaming units (each leaf goes to the
  // chunk holding its first row), unit u = leaves [unit_leaf_lo[u], unit_leaf_hi[u]]
  // = quads [unit_q[u], unit_q[u + 1]); slot_unit[s] = unit resident in slot s
  std::vector<int> unit_leaf_lo, unit_leaf_hi;
  std::vector<long long> unit_q;
  int slot_unit[2] = {-1, -1};
  int* park[2] = {nullptr, nullptr};  // park lists (queries waiting for a later unit)
  long long park_cap = 0;
  // host-resident tensor-core layout (rows [unit_r[u], unit_r[u + 1]) per unit) and its slots
  float* h_tcB = nullptr;
  uint32_t* h_tcidx = nullptr;
  float* h_tcrows = nullptr;
  std::vector<long long> h_row_base, unit_r;
  float* slot_tcB[2] = {nullptr, nullptr};
  uint32_t* slot_tcidx[2] = {nullptr, nullptr};
  float* slot_tcrows[2] = {nullptr, nullptr};
  // file-backed host structure (bkt_set_spill_dir): mappings of unlinked files
  std::string spill_dir;
  std::vector<std::pair<void*, size_t>> spill_maps;
  // tensor-core filter layout (resident trees with d <= 31)
  bool has_tc = false;
  int KT = 0;
  long long tc_rows = 0;
  float* tc_B = nullptr;
  uint32_t* tc_idx = nullptr;
  float* tc_rowsxyz = nullptr;
  long long* tc_row_base = nullptr;
  float* tc_centroid = nullptr;
  float* tc_pnmax = nullptr;
  int* tc_cbase = nullptr;     // nl + 1: first 128-row chunk of each leaf (TC layout)
  float* tc_box = nullptr;     // per 128-row chunk: lo[d], hi[d] bounding box of its points
  unsigned long long* tc_need = nullptr;  // BKT_TC_SKIPDIAG: per-tile mask of chunks some query needs
  unsigned long long* tc_ctr = nullptr;  // BKT_TC_COUNTERS diagnostics (8 counters)
  // leaf-internal blocks: each leaf of the tensor-core layout is ordered as
  // kBlockRows-point blocks along a small k-d split tree.  Queries are
  // bucketed per (leaf, block) so that a warp's queries are neighbours, and
  // the leaf scan skips blocks no query of a warp can reach.  Without the TC
  // layout every leaf is one block.
  int nkeys = 0;              // total blocks
  int sub_w = 1;              // bucket keys per leaf (power of two): key = leaf * sub_w + sub
  int nbuckets = 0;           // nl * sub_w
  int* blk_base = nullptr;    // nl + 1: first block of each leaf
  int4* nodes = nullptr;      // {split value bits, dim, left, right}; child < 0: ~local block
  // split rounds (split_scan.cuh): each leaf's chunks grouped into windows
  // of split_W consecutive 128-row chunks; key = leaf * split_NW + window
  int split_W = 0, split_NW = 0;  // split_NW == 0: split rounds unavailable
  int min_leaf = 0;                // smallest leaf (split rounds need kth finite after the home visit)
  int* win_base = nullptr;         // nl + 1
  float* win_box = nullptr;        // per window, per dimension: {lo, -hi}

  // ---- per-batch work buffers
  long long cap_m = 0;
  int cap_k = 0;
  float* q = nullptr;
  float* q_raw = nullptr;   // unpadded staging (d != D)
  uint64_t* keys = nullptr;
  uint32_t* state = nullptr;
  int* next = nullptr;
  uint32_t* visits = nullptr;
  float* kthv = nullptr;    // per query k-th distance (TC kernel's lazy top-k)
  int* work[2] = {nullptr, nullptr};
  int cap_nl = 0;
  int cap_keys = 0;
  int* counts = nullptr;    // per bucket key
  int* counts_alt = nullptr;  // fused plan+scatter rounds: odd rounds' counts (plan_scatter_kernel)
  int* key_off = nullptr;   // nkeys + 1: first work-list slot of each key
  int* qkey = nullptr;      // per query: bucket key of its next leaf visit
  int2* pos = nullptr;      // per work-list position: {next leaf or -1, slot in its next bucket}
  int* leaf_off = nullptr;
  int* tile_off = nullptr;
  int4* tiles = nullptr;    // per-tile records (capacity tiles_cap)
  long long tiles_cap = 0;
  RoundCtl* ctl = nullptr;
  unsigned long long* pairs = nullptr;
  unsigned long long* seq_pos = nullptr;
  int* hist = nullptr;  // active queries per round (BKT_TRACE_ROUNDS diagnostics)
  int* seq_dev = nullptr;
  long long seq_dev_cap = 0;
  // pinned host mirrors
  RoundCtl* h_ctl = nullptr;  // ring of kMirror slots (mapped page-locked memory)
  RoundCtl* d_ctl_mirror = nullptr;  // device address of h_ctl (plan_kernel writes its slot)
  int* h_tile_off = nullptr;
  int h_tile_off_cap = 0;
  uint64_t* h_stage = nullptr;  // pinned staging for D2H / H2D
  size_t h_stage_bytes = 0;
  // pinned staging for host <-> device streaming: set 0 carries queries in, set 1
  // results out, each on its own stream so both overlap the search
  struct StageSet {
    char* slot[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t stream = nullptr;
  } io[2];
  // second query / result buffers for the overlapped host I/O pipeline
  float* q_alt = nullptr;
  float* q_raw_alt = nullptr;
  uint64_t* keys_alt = nullptr;
  long long cap_alt = 0;
  int cap_alt_k = 0;
  // query renumbering (capacity perm_cap queries)
  long long perm_cap = 0;
  int perm_k = 0;
  int* perm = nullptr;          // search id -> caller's id
  float* q_perm = nullptr;      // m x D rows in search order
  uint64_t* keys_tmp = nullptr; // m x k
  uint32_t* visits_tmp = nullptr;
  // split-round per-query buffers (capacity split_cap queries)
  long long split_cap = 0;
  long long last_per_query = 0;  // per-query bytes the work buffers were last sized for
  int split_capw = 0;          // candidate slice size of the current search (split_capw(NW, k))
  int split_capw_alloc = 0;    // slice size the cand buffer was allocated for
  float* arow = nullptr;                 // m x kSplitKT
  uint8_t* ccnt = nullptr;               // m x split_NW
  uint32_t* cand = nullptr;              // m x split_NW x capw survivor rows
  int* ovflag = nullptr;                 // m
  int* ovf = nullptr;                    // m
  unsigned long long* qmask = nullptr;   // m
  int4* qs = nullptr;                    // m: split_state records {kth, state, visits, next}
  int* cbase = nullptr;                  // route tiles x split_NW
  int* items = nullptr;                  // m x split_NW
  int* stoff = nullptr;                  // nl * split_NW + 1
  int4* stiles = nullptr;
  long long stiles_cap = 0;

  bkt_internal::SeamSlot seam[bkt_internal::kSeamSlots];  // fine seam chunk slots (misc.cu)
  std::vector<cudaEvent_t> ev_pool;   // leafscan timing events
  cudaEvent_t ring_ev[4] = {};        // round-check ring (kRing)
  cudaEvent_t group_ev[2] = {};       // graph mode: end of the last two round groups
  cudaEvent_t t_ev[3] = {};           // whole-search timing + early-drain marker
  // leafscan grid per (D, KB, mode)
  std::vector<std::pair<long long, int>> grid_cache;
};

namespace {
constexpr int kRing = 4;
constexpr int kGraphRounds = 4;            // split rounds per captured graph
constexpr int kMirror = 2 * kGraphRounds;  // mapped control-block slots (>= kRing)
constexpr int kHistCap = 1 << 17;

int set_err(bkt_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  g_thread_err = msg;
  return code;
}

#define CU(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return set_err(ctx, BKT_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " \
                                         + __FILE__ + ":" + std::to_string(__LINE__) + " (" #call ")"); \
  } while (0)

template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}
template <typename T>
void hfree(T*& p) {
  if (p) cudaFreeHost(p);
  p = nullptr;
}

int kernel_dim(int d) {
  int best = -1;
#define BKT_PICK(D) \
  if (best < 0 && D >= d) best = D;
  BKT_DIM_LIST(BKT_PICK)
#undef BKT_PICK
  return best;
}
int kb_bucket(int k) {
  int best = -1;
#define BKT_PICK(KB) \
  if (best < 0 && KB >= k) best = KB;
  BKT_KB_LIST(BKT_PICK)
#undef BKT_PICK
  return best;
}

cudaError_t launch_leafscan(int D, int kb, bool fma, int grid, cudaStream_t s, const ScanArgs& a, int* occ) {
  switch (D) {
#define BKT_CASE(DD) \
  case DD:           \
    return launch_leafscan_d##DD(kb, fma, grid, s, a, occ);
    BKT_DIM_LIST(BKT_CASE)
#undef BKT_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

int leafscan_grid(bkt_ctx* ctx, int D, int kb, bool fma, int* grid) {
  long long key = ((long long)D << 16) | ((long long)kb << 1) | (fma ? 1 : 0);
  for (auto& e : ctx->grid_cache)
    if (e.first == key) { *grid = e.second; return BKT_OK; }
  int occ = 0;
  ScanArgs dummy{};
  CU(launch_leafscan(D, kb, fma, 0, nullptr, dummy, &occ));
  if (occ < 1) occ = 1;
  *grid = occ * ctx->sm_count;
  ctx->grid_cache.push_back({key, *grid});
  return BKT_OK;
}

// Host memory of a host-resident structure: page-locked, or -- with a spill
// directory -- a shared mapping of an unlinked file there, so the kernel can
// write clean pages back and the structure may exceed host RAM (PAPER.md
// sec. 3.2: disk -> host -> device; the drain streams each unit once per pass).
int host_alloc(bkt_ctx* ctx, void** out, size_t bytes, const char* tag) {
  bkt_ctx* c = ctx;
  *out = nullptr;
  if (c->spill_dir.empty()) {
    CU(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable));
    return BKT_OK;
  }
  std::string path = c->spill_dir + "/bkt_" + std::to_string((long long)getpid()) + "_" +
                     std::to_string(reinterpret_cast<uintptr_t>(c)) + "_" + tag + ".bin";
  const int fd = open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0600);
  if (fd < 0) return set_err(c, BKT_EINVAL, "spill directory: cannot create " + path);
  const size_t len = std::max<size_t>(bytes, 1);
  if (ftruncate(fd, (off_t)len) != 0) {
    close(fd);
    unlink(path.c_str());
    return set_err(c, BKT_ECONFIG, "spill directory: cannot size " + path);
  }
  void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  unlink(path.c_str());  // the mapping keeps the file; its blocks go when it is unmapped
  if (p == MAP_FAILED) return set_err(c, BKT_ECONFIG, "spill directory: cannot map " + path);
  c->spill_maps.emplace_back(p, len);
  *out = p;
  return BKT_OK;
}

void free_spill(bkt_ctx* c) {
  for (auto& m : c->spill_maps) {
    if (c->h_pts == m.first) c->h_pts = nullptr;
    if (c->h_pidx == m.first) c->h_pidx = nullptr;
    if (c->h_tcB == m.first) c->h_tcB = nullptr;
    if (c->h_tcidx == m.first) c->h_tcidx = nullptr;
    if (c->h_tcrows == m.first) c->h_tcrows = nullptr;
    munmap(m.first, m.second);
  }
  c->spill_maps.clear();
}

void free_tree(bkt_ctx* c) {
  dfree(c->tc_B); dfree(c->tc_idx); dfree(c->tc_rowsxyz); dfree(c->tc_row_base); dfree(c->tc_centroid); dfree(c->tc_pnmax); dfree(c->tc_cbase); dfree(c->tc_box);
  c->has_tc = false;
  dfree(c->blk_base); dfree(c->nodes);
  dfree(c->win_base); dfree(c->win_box);
  c->split_W = 0; c->split_NW = 0;
  c->nkeys = 0;
  dfree(c->split); dfree(c->quad_base); dfree(c->leaf_size); dfree(c->pts); dfree(c->pidx);
  free_spill(c);
  hfree(c->h_pts); hfree(c->h_pidx);
  for (int s = 0; s < 2; ++s) {
    dfree(c->slot_pts[s]); dfree(c->slot_idx[s]);
    c->slot_chunk[s] = -1;
    c->slot_unit[s] = -1;
    dfree(c->slot_tcB[s]); dfree(c->slot_tcidx[s]); dfree(c->slot_tcrows[s]);
  }
  c->unit_leaf_lo.clear(); c->unit_leaf_hi.clear(); c->unit_q.clear(); c->unit_r.clear(); c->h_row_base.clear();
  hfree(c->h_tcB); hfree(c->h_tcidx); hfree(c->h_tcrows);
  c->has_tree = false;
  c->wide_only = false;
  c->wide_pts = nullptr;
  c->wide_pidx = nullptr;
}

void free_work(bkt_ctx* c) {
  dfree(c->tiles);
  c->tiles_cap = 0;
  dfree(c->kthv);
  dfree(c->qkey);
  dfree(c->pos);
  dfree(c->q); dfree(c->q_raw); dfree(c->keys); dfree(c->state); dfree(c->next); dfree(c->visits);
  dfree(c->work[0]); dfree(c->work[1]);
  dfree(c->park[0]); dfree(c->park[1]);
  c->park_cap = 0;
  c->cap_m = 0; c->cap_k = 0;
  dfree(c->q_alt); dfree(c->q_raw_alt); dfree(c->keys_alt);
  c->cap_alt = 0; c->cap_alt_k = 0;
  dfree(c->arow); dfree(c->ccnt); dfree(c->cand); dfree(c->ovflag); dfree(c->ovf); dfree(c->qmask); dfree(c->cbase);
  dfree(c->qs);
  dfree(c->items); dfree(c->stoff); dfree(c->stiles);
  c->split_cap = 0; c->stiles_cap = 0;
  dfree(c->perm); dfree(c->q_perm); dfree(c->keys_tmp); dfree(c->visits_tmp);
  c->perm_cap = 0; c->perm_k = 0;
}

int ensure_perm(bkt_ctx* ctx, long long m, int k) {
  if (ctx->perm_cap >= m && ctx->perm_k >= k) return BKT_OK;
  dfree(ctx->perm); dfree(ctx->q_perm); dfree(ctx->keys_tmp); dfree(ctx->visits_tmp);
  const long long M = std::max<long long>(m, 1);
  CU(cudaMalloc(&ctx->perm, sizeof(int) * M));
  CU(cudaMalloc(&ctx->q_perm, sizeof(float) * M * ctx->D));
  CU(cudaMalloc(&ctx->keys_tmp, sizeof(uint64_t) * M * k));
  CU(cudaMalloc(&ctx->visits_tmp, sizeof(uint32_t) * M));
  ctx->perm_cap = M;
  ctx->perm_k = k;
  return BKT_OK;
}

// per-query bytes of the split-round buffers
long long split_bytes_per_query(const bkt_ctx* c) {
  return 4ll * kSplitKT + (1ll + 4ll * c->split_capw) * c->split_NW + 4 + 4 + 8 + 16 + 4ll * c->split_NW +
         16ll * c->split_NW / kNT + 16;
}

int ensure_split(bkt_ctx* ctx, long long m) {
  if (ctx->split_cap >= m && ctx->split_capw_alloc == ctx->split_capw) return BKT_OK;
  dfree(ctx->arow); dfree(ctx->ccnt); dfree(ctx->cand); dfree(ctx->ovflag); dfree(ctx->ovf); dfree(ctx->qmask); dfree(ctx->cbase);
  dfree(ctx->qs);
  dfree(ctx->items); dfree(ctx->stoff); dfree(ctx->stiles);
  const long long M = std::max<long long>(m, 1);
  const long long NW = ctx->split_NW;
  CU(cudaMalloc(&ctx->arow, sizeof(float) * M * kSplitKT));
  CU(cudaMalloc(&ctx->ccnt, M * NW));
  CU(cudaMemset(ctx->ccnt, 0, M * NW));
  CU(cudaMalloc(&ctx->cand, sizeof(uint32_t) * M * NW * ctx->split_capw));
  CU(cudaMalloc(&ctx->ovflag, sizeof(int) * M));
  CU(cudaMemset(ctx->ovflag, 0, sizeof(int) * M));
  CU(cudaMalloc(&ctx->ovf, sizeof(int) * M));
  CU(cudaMalloc(&ctx->qmask, sizeof(unsigned long long) * M));
  CU(cudaMalloc(&ctx->qs, sizeof(int4) * M));
  CU(cudaMalloc(&ctx->cbase, sizeof(int) * (M / kRouteQ + ctx->nl + 1) * NW));
  CU(cudaMalloc(&ctx->items, sizeof(int) * M * NW));
  CU(cudaMalloc(&ctx->stoff, sizeof(int) * ((long long)ctx->nl * NW + 1)));
  ctx->stiles_cap = M * NW / kNT + (long long)ctx->nl * NW + 1;
  CU(cudaMalloc(&ctx->stiles, sizeof(int4) * ctx->stiles_cap));
  ctx->split_cap = M;
  ctx->split_capw_alloc = ctx->split_capw;
  return BKT_OK;
}

int ensure_alt(bkt_ctx* ctx, long long m, int k) {
  if (ctx->cap_alt >= m && ctx->cap_alt_k >= k) return BKT_OK;
  dfree(ctx->q_alt); dfree(ctx->q_raw_alt); dfree(ctx->keys_alt);
  CU(cudaMalloc(&ctx->q_alt, sizeof(float) * m * ctx->D));
  if (ctx->D != ctx->d) CU(cudaMalloc(&ctx->q_raw_alt, sizeof(float) * m * ctx->d));
  CU(cudaMalloc(&ctx->keys_alt, sizeof(uint64_t) * m * k));
  ctx->cap_alt = m;
  ctx->cap_alt_k = k;
  return BKT_OK;
}

void free_leafbufs(bkt_ctx* c) {
  dfree(c->counts); dfree(c->counts_alt); dfree(c->key_off); dfree(c->leaf_off); dfree(c->tile_off);
  hfree(c->h_tile_off);
  c->cap_nl = 0;
  c->cap_keys = 0;
  c->h_tile_off_cap = 0;
}

int ensure_leafbufs(bkt_ctx* ctx, int nl, int nkeys) {
  if (ctx->cap_nl >= nl && ctx->cap_keys >= nkeys) return BKT_OK;
  free_leafbufs(ctx);
  CU(cudaMalloc(&ctx->counts, sizeof(int) * nkeys));
  CU(cudaMalloc(&ctx->key_off, sizeof(int) * (nkeys + 1)));
  CU(cudaMemset(ctx->counts, 0, sizeof(int) * nkeys));
  CU(cudaMalloc(&ctx->counts_alt, sizeof(int) * nkeys));
  CU(cudaMemset(ctx->counts_alt, 0, sizeof(int) * nkeys));
  CU(cudaMalloc(&ctx->leaf_off, sizeof(int) * (nl + 1)));
  CU(cudaMalloc(&ctx->tile_off, sizeof(int) * (nl + 1)));
  CU(cudaHostAlloc(&ctx->h_tile_off, sizeof(int) * (nl + 1), cudaHostAllocDefault));
  ctx->cap_nl = nl;
  ctx->cap_keys = nkeys;
  ctx->h_tile_off_cap = nl + 1;
  return BKT_OK;
}

int ensure_work(bkt_ctx* ctx, long long m, int k) {
  if (ctx->cap_m >= m && ctx->cap_k >= k && (ctx->D == ctx->d || ctx->q_raw)) return BKT_OK;
  free_work(ctx);
  long long M = std::max<long long>(m, 1);
  CU(cudaMalloc(&ctx->q, sizeof(float) * M * ctx->D));
  if (ctx->D != ctx->d) CU(cudaMalloc(&ctx->q_raw, sizeof(float) * M * ctx->d));
  CU(cudaMalloc(&ctx->keys, sizeof(uint64_t) * M * k));
  CU(cudaMalloc(&ctx->state, sizeof(uint32_t) * M));
  CU(cudaMalloc(&ctx->next, sizeof(int) * M));
  CU(cudaMalloc(&ctx->visits, sizeof(uint32_t) * M));
  CU(cudaMalloc(&ctx->kthv, sizeof(float) * M));
  CU(cudaMalloc(&ctx->qkey, sizeof(int) * M));
  CU(cudaMalloc(&ctx->pos, sizeof(int2) * M));
  CU(cudaMalloc(&ctx->work[0], sizeof(int) * M));
  CU(cudaMalloc(&ctx->work[1], sizeof(int) * M));
  ctx->tiles_cap = ctx->wide_only ? 1 : M / kNT + (1ll << ctx->h) + 1;
  CU(cudaMalloc(&ctx->tiles, sizeof(int4) * ctx->tiles_cap));
  ctx->cap_m = M;
  ctx->cap_k = k;
  return BKT_OK;
}

int ensure_stage(bkt_ctx* ctx, size_t bytes) {
  if (ctx->h_stage_bytes >= bytes) return BKT_OK;
  hfree(ctx->h_stage);
  ctx->h_stage_bytes = 0;
  CU(cudaHostAlloc(&ctx->h_stage, bytes, cudaHostAllocDefault));
  ctx->h_stage_bytes = bytes;
  return BKT_OK;
}

cudaEvent_t get_event(bkt_ctx* c, size_t i) {
  while (c->ev_pool.size() <= i) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[i];
}

constexpr size_t kStageSlot = 32ull << 20;

// memcpy with a few host threads (host <-> pinned staging is the e2e bottleneck)
void par_memcpy(void* dst, const void* src, size_t n) {
  const int nt = (int)std::min<size_t>(8, std::max<size_t>(1, n >> 22));
  if (nt <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    size_t a = t * per, b = std::min(n, a + per);
    if (a >= b) break;
    th.emplace_back([=]() { std::memcpy((char*)dst + a, (const char*)src + a, b - a); });
  }
  for (auto& x : th) x.join();
}

int ensure_stageset(bkt_ctx* ctx, bkt_ctx::StageSet& S) {
  for (int i = 0; i < 2; ++i) {
    if (!S.slot[i]) CU(cudaHostAlloc(&S.slot[i], kStageSlot, cudaHostAllocDefault));
    if (!S.ev[i]) CU(cudaEventCreateWithFlags(&S.ev[i], cudaEventDisableTiming));
  }
  if (!S.stream) CU(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
  return BKT_OK;
}

void free_stageset(bkt_ctx::StageSet& S) {
  for (int i = 0; i < 2; ++i) {
    hfree(S.slot[i]);
    if (S.ev[i]) cudaEventDestroy(S.ev[i]);
    S.ev[i] = nullptr;
  }
  if (S.stream) cudaStreamDestroy(S.stream);
  S.stream = nullptr;
}

// pageable host -> device: host threads fill one pinned slot while the other DMAs
int h2d_staged(bkt_ctx* ctx, bkt_ctx::StageSet& S, void* dst, const void* src, size_t bytes) {
  int rc = ensure_stageset(ctx, S);
  if (rc != BKT_OK) return rc;
  {
    // page-locked source (e.g. bkt_host_alloc): one direct DMA, no staging copy
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();  // pageable memory reports an error on some drivers: clear it
    if (pinned) {
      CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S.stream));
      CU(cudaStreamSynchronize(S.stream));
      return BKT_OK;
    }
  }
  size_t off = 0;
  for (int i = 0; off < bytes; ++i) {
    const int s = i & 1;
    const size_t n = std::min(kStageSlot, bytes - off);
    CU(cudaEventSynchronize(S.ev[s]));  // slot's previous DMA done (never-recorded events return at once)
    par_memcpy(S.slot[s], (const char*)src + off, n);
    CU(cudaMemcpyAsync((char*)dst + off, S.slot[s], n, cudaMemcpyHostToDevice, S.stream));
    CU(cudaEventRecord(S.ev[s], S.stream));
    off += n;
  }
  CU(cudaStreamSynchronize(S.stream));
  return BKT_OK;
}

// device -> pageable host: one slot DMAs while host threads drain the other
int d2h_staged(bkt_ctx* ctx, bkt_ctx::StageSet& S, void* dst, const void* src, size_t bytes) {
  int rc = ensure_stageset(ctx, S);
  if (rc != BKT_OK) return rc;
  const size_t nchunks = (bytes + kStageSlot - 1) / kStageSlot;
  auto issue = [&](size_t i) -> int {
    const int s = (int)(i & 1);
    const size_t off = i * kStageSlot, n = std::min(kStageSlot, bytes - off);
    CU(cudaMemcpyAsync(S.slot[s], (const char*)src + off, n, cudaMemcpyDeviceToHost, S.stream));
    CU(cudaEventRecord(S.ev[s], S.stream));
    return BKT_OK;
  };
  if (nchunks == 0) return BKT_OK;
  if ((rc = issue(0)) != BKT_OK) return rc;
  for (size_t i = 0; i < nchunks; ++i) {
    const int s = (int)(i & 1);
    CU(cudaEventSynchronize(S.ev[s]));
    if (i + 1 < nchunks && (rc = issue(i + 1)) != BKT_OK) return rc;
    const size_t off = i * kStageSlot, n = std::min(kStageSlot, bytes - off);
    par_memcpy((char*)dst + off, S.slot[s], n);
  }
  return BKT_OK;
}

// host quad-interleaved layout of the leaf structure
void build_quad_layout(const float* leaf_points, const int64_t* orig, const int64_t* starts, int nl, int d, int D,
                       const std::vector<long long>& qb, float* out_pts, uint32_t* out_idx) {
  auto work = [&](int l0, int l1) {
    for (int l = l0; l < l1; ++l) {
      long long s = starts[l], e = starts[l + 1];
      long long L = e - s, nq = qb[l + 1] - qb[l];
      for (long long qd = 0; qd < nq; ++qd) {
        float* dst = out_pts + (qb[l] + qd) * 4 * D;
        uint32_t* di = out_idx + (qb[l] + qd) * 4;
        for (int t = 0; t < 4; ++t) {
          long long r = qd * 4 + t;
          bool real = r < L;
          di[t] = real ? (uint32_t)orig[s + r] : kIndexSentinel;
          for (int j = 0; j < D; ++j) {
            float v;
            if (!real) v = __builtin_inff();
            else v = (j < d) ? leaf_points[(s + r) * d + j] : 0.0f;
            dst[4 * j + t] = v;
          }
        }
      }
    }
  };
  int nt = std::max(1, std::min<int>(16, (int)std::thread::hardware_concurrency()));
  if (nl < 64) nt = 1;
  std::vector<std::thread> th;
  for (int w = 0; w < nt; ++w) th.emplace_back(work, (int)((long long)nl * w / nt), (int)((long long)nl * (w + 1) / nt));
  for (auto& t : th) t.join();
}

// Leaf-internal blocks.  Each leaf's points are ordered so that consecutive
// runs of kBlockRows form blocks of a small k-d split tree (split on the
// widest dimension; the left side takes ceil(nb/2) full blocks).  The split
// nodes route a home-leaf visit to its block, so the home bucket is ordered by
// position and the scan of a first visit starts next to its queries (its k-th
// distance bound is tight from the first chunk).  The order inside a leaf
// never changes a result: keys are (distance, original index) and the leaf's
// point set is the reference's.
struct LeafBlocks {
  std::vector<int> blk_base;     // nl + 1
  std::vector<int4> nodes;       // nkeys - nl split nodes; leaf l's start at blk_base[l] - l
  std::vector<uint32_t> perm;    // n: local row order of every leaf (offset by leaf start)
};

void build_leaf_blocks(const float* pts, const int64_t* starts, int nl, int d, int bs, LeafBlocks& out) {
  out.blk_base.assign(nl + 1, 0);
  for (int l = 0; l < nl; ++l) {
    long long L = starts[l + 1] - starts[l];
    out.blk_base[l + 1] = out.blk_base[l] + (int)((L + bs - 1) / bs);
  }
  const int nkeys = out.blk_base[nl];
  out.nodes.assign(std::max(0, nkeys - nl), int4{0, 0, 0, 0});
  out.perm.resize((size_t)starts[nl]);
  auto work = [&](int l0, int l1) {
    std::vector<uint32_t> idx;
    for (int l = l0; l < l1; ++l) {
      const long long s = starts[l], L = starts[l + 1] - s;
      idx.resize(L);
      for (long long i = 0; i < L; ++i) idx[i] = (uint32_t)i;
      const int nb_leaf = out.blk_base[l + 1] - out.blk_base[l];
      int4* nodes = out.nodes.data() + (out.blk_base[l] - l);
      int next_node = 0, next_block = 0;
      auto coord = [&](uint32_t i, int j) { return pts[(s + i) * d + j]; };
      // returns the child code of [lo, hi) holding nb blocks
      std::function<int(long long, long long, int)> rec = [&](long long lo, long long hi, int nb) -> int {
        if (nb == 1) return ~(next_block++);
        const long long left = (long long)bs * ((nb + 1) / 2);
        int dim = 0;
        float best = -1.0f;
        for (int j = 0; j < d; ++j) {
          float mn = coord(idx[lo], j), mx = mn;
          for (long long i = lo + 1; i < hi; ++i) {
            float v = coord(idx[i], j);
            mn = std::min(mn, v);
            mx = std::max(mx, v);
          }
          if (mx - mn > best) { best = mx - mn; dim = j; }
        }
        std::nth_element(idx.begin() + lo, idx.begin() + lo + left, idx.begin() + hi, [&](uint32_t a, uint32_t b) {
          float va = coord(a, dim), vb = coord(b, dim);
          return va < vb || (va == vb && a < b);
        });
        const float val = coord(idx[lo + left], dim);
        const int me = next_node++;
        const int lc = rec(lo, lo + left, (nb + 1) / 2);
        const int rc = rec(lo + left, hi, nb - (nb + 1) / 2);
        int vb;
        std::memcpy(&vb, &val, 4);
        nodes[me] = int4{vb, dim, lc, rc};
        return me;
      };
      rec(0, L, nb_leaf);
      for (long long i = 0; i < L; ++i) out.perm[s + i] = idx[i];
    }
  };
  int nt = std::max(1, std::min<int>(16, (int)std::thread::hardware_concurrency()));
  if (nl < 64) nt = 1;
  std::vector<std::thread> th;
  for (int w = 0; w < nt; ++w) th.emplace_back(work, (int)((long long)nl * w / nt), (int)((long long)nl * (w + 1) / nt));
  for (auto& t : th) t.join();
}

// round-to-nearest (ties away) float32 -> tf32, matching cvt.rna.tf32.f32
inline float tf32_rna_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return x;  // inf / nan unchanged
  u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// Tensor-core filter layout (see leafscan_tc.cuh): every leaf padded to a
// multiple of 32 rows; per padded row R the K-major canonical UMMA layout
// B[(R/8)*8*KT + (k/4)*32 + (R%8)*4 + k%4] holds tf32(-2 p'_k) for k < d,
// tf32((1 - C) |p'|^2) in column d, zeros after; padding rows carry +inf in
// column d so they never pass the filter.
void build_tc_layout(const float* leaf_points, const int64_t* orig, const int64_t* starts, int nl, int d, int KT,
                     const std::vector<long long>& rb, const std::vector<uint32_t>& perm, float* B, uint32_t* ridx,
                     float* rows, float* centroid, float* pnmax) {
  auto work = [&](int l0, int l1) {
    std::vector<double> acc(d);
    for (int l = l0; l < l1; ++l) {
      long long s = starts[l], e = starts[l + 1];
      std::fill(acc.begin(), acc.end(), 0.0);
      for (long long r = s; r < e; ++r)
        for (int j = 0; j < d; ++j) acc[j] += leaf_points[r * d + j];
      float* cen = centroid + (long long)l * KT;
      for (int j = 0; j < KT; ++j) cen[j] = j < d ? (float)(acc[j] / (double)(e - s)) : 0.0f;
      float pmax = 0.0f;
      for (long long R = rb[l]; R < rb[l + 1]; ++R) {
        const long long loc = R - rb[l];
        const bool real = s + loc < e;
        const long long r = real ? s + (long long)perm[s + loc] : e;
        float* bg = B + (R / 8) * 8 * KT + (R % 8) * 4;
        float pn = 0.0f;
        for (int k = 0; k < KT; ++k) {
          float v = 0.0f;
          if (k < d && real) {
            float pc = leaf_points[r * d + k] - cen[k];
            pn = std::fma(pc, pc, pn);
            v = tf32_rna_host(-2.0f * pc);
          }
          bg[(k / 4) * 32 + (k % 4)] = v;
        }
        bg[(d / 4) * 32 + (d % 4)] = real ? tf32_rna_host((1.0f - kTcMargin) * pn) : __builtin_inff();
        if (real) pmax = std::max(pmax, pn);
        ridx[R] = real ? (uint32_t)orig[r] : kIndexSentinel;
        for (int j = 0; j < d; ++j) rows[R * d + j] = real ? leaf_points[r * d + j] : __builtin_inff();
      }
      pnmax[l] = pmax * 1.0001f;
    }
  };
  int nt = std::max(1, std::min<int>(16, (int)std::thread::hardware_concurrency()));
  if (nl < 64) nt = 1;
  std::vector<std::thread> th;
  for (int w = 0; w < nt; ++w) th.emplace_back(work, (int)((long long)nl * w / nt), (int)((long long)nl * (w + 1) / nt));
  for (auto& t : th) t.join();
}
}  // namespace

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

const char* bkt_last_error(const bkt_ctx* ctx) {
  if (ctx) return ctx->err.c_str();
  return g_thread_err.c_str();
}

int bkt_open(int cuda_device, bkt_ctx** out) {
  bkt_ctx* ctx = nullptr;
  if (!out) return set_err(nullptr, BKT_EINVAL, "out is NULL");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return set_err(nullptr, BKT_ECUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
  if (cuda_device < 0 || cuda_device >= ndev)
    return set_err(nullptr, BKT_EINVAL, "cuda_device " + std::to_string(cuda_device) + " out of range [0, " +
                                            std::to_string(ndev) + ")");
  ctx = new bkt_ctx();
  ctx->device = cuda_device;
  CU(cudaSetDevice(cuda_device));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, cuda_device));
  if (prop.major < 10) {
    std::string msg = std::string("device ") + prop.name + " is sm_" + std::to_string(prop.major) +
                      std::to_string(prop.minor) + "; this engine is built for sm_100a (B200)";
    delete ctx;
    return set_err(nullptr, BKT_ECUDA, msg);
  }
  ctx->sm_count = prop.multiProcessorCount;
  cudaDeviceGetAttribute(&ctx->sm_clock_khz, cudaDevAttrClockRate, cuda_device);
  CU(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  CU(cudaMalloc(&ctx->ctl, sizeof(RoundCtl)));
  CU(cudaMalloc(&ctx->pairs, sizeof(unsigned long long)));
  CU(cudaMalloc(&ctx->seq_pos, sizeof(unsigned long long)));
  CU(cudaMalloc(&ctx->hist, sizeof(int) * kHistCap));
  CU(cudaHostAlloc(&ctx->h_ctl, sizeof(RoundCtl) * kMirror, cudaHostAllocMapped));
  CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->d_ctl_mirror), ctx->h_ctl, 0));
  for (int i = 0; i < kRing; ++i) CU(cudaEventCreateWithFlags(&ctx->ring_ev[i], cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) CU(cudaEventCreateWithFlags(&ctx->group_ev[i], cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) CU(cudaEventCreate(&ctx->t_ev[i]));
  CU(cudaEventCreateWithFlags(&ctx->t_ev[2], cudaEventDisableTiming));
  for (int s = 0; s < 2; ++s) {
    CU(cudaEventCreateWithFlags(&ctx->slot_free[s], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ctx->slot_ready[s], cudaEventDisableTiming));
  }
  *out = ctx;
  return BKT_OK;
}

void bkt_close(bkt_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
  free_tree(ctx);
  free_work(ctx);
  free_leafbufs(ctx);
  dfree(ctx->ctl); dfree(ctx->pairs); dfree(ctx->seq_pos); dfree(ctx->seq_dev); dfree(ctx->hist); dfree(ctx->tc_ctr);
  hfree(ctx->h_ctl); hfree(ctx->h_stage);
  for (int i = 0; i < 2; ++i) free_stageset(ctx->io[i]);
  dfree(ctx->q_alt); dfree(ctx->q_raw_alt); dfree(ctx->keys_alt);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto& sl : ctx->seam) {
    dfree(sl.pts); dfree(sl.ids);
    if (sl.ready) cudaEventDestroy(sl.ready);
  }
  for (int i = 0; i < kRing; ++i)
    if (ctx->ring_ev[i]) cudaEventDestroy(ctx->ring_ev[i]);
  for (int i = 0; i < 2; ++i)
    if (ctx->group_ev[i]) cudaEventDestroy(ctx->group_ev[i]);
  for (int i = 0; i < 3; ++i)
    if (ctx->t_ev[i]) cudaEventDestroy(ctx->t_ev[i]);
  for (int s = 0; s < 2; ++s) {
    if (ctx->slot_free[s]) cudaEventDestroy(ctx->slot_free[s]);
    if (ctx->slot_ready[s]) cudaEventDestroy(ctx->slot_ready[s]);
  }
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  delete ctx;
}

int bkt_set_spill_dir(bkt_ctx* ctx, const char* dir) {
  if (!ctx) return set_err(nullptr, BKT_EINVAL, "ctx is NULL");
  ctx->spill_dir = dir ? dir : "";
  while (ctx->spill_dir.size() > 1 && ctx->spill_dir.back() == '/') ctx->spill_dir.pop_back();
  return BKT_OK;
}

int bkt_device_info(bkt_ctx* ctx, int32_t* sm_count, int32_t* sm_clock_khz, int64_t* free_bytes,
                    int64_t* total_bytes) {
  if (!ctx) return set_err(nullptr, BKT_EINVAL, "ctx is NULL");
  CU(cudaSetDevice(ctx->device));
  size_t fr = 0, to = 0;
  CU(cudaMemGetInfo(&fr, &to));
  if (sm_count) *sm_count = ctx->sm_count;
  if (sm_clock_khz) *sm_clock_khz = ctx->sm_clock_khz;
  if (free_bytes) *free_bytes = (int64_t)fr;
  if (total_bytes) *total_bytes = (int64_t)to;
  return BKT_OK;
}

int bkt_load_tree(bkt_ctx* ctx, int32_t h, int32_t d, int64_t n, const float* split_values,
                  const float* leaf_points, const int64_t* original_index, const int64_t* leaf_starts,
                  int32_t residency, int32_t num_chunks, const int64_t* chunk_bounds) {
  if (!ctx) return set_err(nullptr, BKT_EINVAL, "ctx is NULL");
  if (h < 1 || h > kMaxWideHeight)
    return set_err(ctx, BKT_EINVAL, "height " + std::to_string(h) + " outside the supported range [1, 30]");
  if (d < 1) return set_err(ctx, BKT_EINVAL, "dimensionality must be >= 1");
  if (n < (1ll << h)) return set_err(ctx, BKT_EINVAL, "height needs at least 2^h points");
  if (n >= (long long)kIndexSentinel) return set_err(ctx, BKT_EINVAL, "point count exceeds the supported maximum");
  if (residency != 0 && residency != 1) return set_err(ctx, BKT_EINVAL, "residency must be 0 or 1");
  if (num_chunks < 1 || num_chunks > n) return set_err(ctx, BKT_EINVAL, "num_chunks must be in [1, n]");
  CU(cudaSetDevice(ctx->device));
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaStreamSynchronize(ctx->copy_stream));
  free_tree(ctx);
  ctx->grid_cache.clear();
  const int nl = 1 << h;
  // h > 16 or d > 32: outside the round engine's packed state / compiled
  // dimensionalities; the tree is searched by the wide path only (quad layout
  // of width d)
  const bool wide_only = h > kMaxHeight || d > kMaxKernelDim;
  const int D = wide_only && d > kMaxKernelDim ? d : kernel_dim(d);
  ctx->h = h; ctx->d = d; ctx->D = D; ctx->nl = nl; ctx->n = n;
  ctx->wide_only = wide_only;
  // quad bases: each leaf padded to a multiple of 4 points
  ctx->h_quad_base.assign(nl + 1, 0);
  ctx->h_leaf_size.assign(nl, 0);
  for (int l = 0; l < nl; ++l) {
    long long L = leaf_starts[l + 1] - leaf_starts[l];
    if (L < 1) return set_err(ctx, BKT_EINVAL, "leaf ranges do not partition the point set");
    ctx->h_leaf_size[l] = (int)L;
    ctx->h_quad_base[l + 1] = ctx->h_quad_base[l] + (L + 3) / 4;
  }
  if (leaf_starts[0] != 0 || leaf_starts[nl] != n)
    return set_err(ctx, BKT_EINVAL, "leaf ranges do not partition the point set");
  const long long TQ = ctx->h_quad_base[nl];
  ctx->total_quads = TQ;
  free_work(ctx);  // per-query buffers depend on D; reallocated by the next search

  CU(cudaMalloc(&ctx->split, sizeof(float) * (nl - 1)));
  CU(cudaMalloc(&ctx->quad_base, sizeof(long long) * (nl + 1)));
  CU(cudaMalloc(&ctx->leaf_size, sizeof(int) * nl));
  CU(cudaMemcpy(ctx->split, split_values, sizeof(float) * (nl - 1), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->quad_base, ctx->h_quad_base.data(), sizeof(long long) * (nl + 1), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->leaf_size, ctx->h_leaf_size.data(), sizeof(int) * nl, cudaMemcpyHostToDevice));

  const size_t pts_bytes = sizeof(float) * (size_t)TQ * 4 * D;
  const size_t idx_bytes = sizeof(uint32_t) * (size_t)TQ * 4;
  // mapped: the wide path reads a host-resident structure in place; a
  // host-resident structure with a spill directory lives in file-backed pages
  const bool spill = residency == 1 && !ctx->spill_dir.empty();
  if (spill) {
    if (int rc = host_alloc(ctx, reinterpret_cast<void**>(&ctx->h_pts), pts_bytes, "pts")) return rc;
    if (int rc = host_alloc(ctx, reinterpret_cast<void**>(&ctx->h_pidx), idx_bytes, "pidx")) return rc;
  } else {
    CU(cudaHostAlloc(&ctx->h_pts, pts_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    CU(cudaHostAlloc(&ctx->h_pidx, idx_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  }
  build_quad_layout(leaf_points, original_index, leaf_starts, nl, d, D, ctx->h_quad_base, ctx->h_pts, ctx->h_pidx);

  // tensor-core filter layout (d + 1 <= 32); host_big: its row arrays stay in
  // page-locked host memory (host-resident structure)
  auto build_tc = [&](bool host_big) -> int {
    if (d + 1 <= 32 && !wide_only) {
      const int KT = (d + 1 <= 16) ? 16 : 32;
      std::vector<long long> rb(nl + 1, 0);
      for (int l = 0; l < nl; ++l) rb[l + 1] = rb[l] + ((long long)ctx->h_leaf_size[l] + 31) / 32 * 32;
      const long long R = rb[nl];
      std::vector<float> hBv, hrowsv, hcen((size_t)nl * KT), hpn((size_t)nl);
      std::vector<uint32_t> hidxv;
      float *hB = nullptr, *hrows = nullptr;
      uint32_t* hidx = nullptr;
      if (host_big) {
        // host-resident structure: the filter rows are built in place in
        // page-locked memory (or file-backed pages, bkt_set_spill_dir) and
        // stream into the drain's slots per unit (ooc_drain)
        if (int rc = host_alloc(ctx, reinterpret_cast<void**>(&ctx->h_tcB), sizeof(float) * R * KT, "tcB")) return rc;
        if (int rc = host_alloc(ctx, reinterpret_cast<void**>(&ctx->h_tcidx), sizeof(uint32_t) * R, "tcidx")) return rc;
        if (int rc = host_alloc(ctx, reinterpret_cast<void**>(&ctx->h_tcrows), sizeof(float) * R * d, "tcrows")) return rc;
        hB = ctx->h_tcB;
        hidx = ctx->h_tcidx;
        hrows = ctx->h_tcrows;
      } else {
        hBv.resize((size_t)R * KT);
        hrowsv.resize((size_t)R * d);
        hidxv.resize((size_t)R);
        hB = hBv.data();
        hidx = hidxv.data();
        hrows = hrowsv.data();
      }
      LeafBlocks lb;
      build_leaf_blocks(leaf_points, leaf_starts, nl, d, kBlockRows, lb);
      if (std::getenv("BKT_NO_PERM"))
        for (int l = 0; l < nl; ++l)
          for (long long i = leaf_starts[l]; i < leaf_starts[l + 1]; ++i) lb.perm[i] = (uint32_t)(i - leaf_starts[l]);
      build_tc_layout(leaf_points, original_index, leaf_starts, nl, d, KT, rb, lb.perm, hB, hidx,
                      hrows, hcen.data(), hpn.data());
      ctx->nkeys = lb.blk_base[nl];
      CU(cudaMalloc(&ctx->blk_base, sizeof(int) * (nl + 1)));
      CU(cudaMemcpy(ctx->blk_base, lb.blk_base.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice));
      if (!lb.nodes.empty()) {
        CU(cudaMalloc(&ctx->nodes, sizeof(int4) * lb.nodes.size()));
        CU(cudaMemcpy(ctx->nodes, lb.nodes.data(), sizeof(int4) * lb.nodes.size(), cudaMemcpyHostToDevice));
      }
      CU(cudaMalloc(&ctx->tc_pnmax, sizeof(float) * nl));
      CU(cudaMemcpy(ctx->tc_pnmax, hpn.data(), sizeof(float) * nl, cudaMemcpyHostToDevice));
      CU(cudaMalloc(&ctx->tc_row_base, sizeof(long long) * (nl + 1)));
      CU(cudaMalloc(&ctx->tc_centroid, sizeof(float) * nl * KT));
      if (!host_big) {
        CU(cudaMalloc(&ctx->tc_B, sizeof(float) * R * KT));
        CU(cudaMalloc(&ctx->tc_idx, sizeof(uint32_t) * R));
        CU(cudaMalloc(&ctx->tc_rowsxyz, sizeof(float) * R * d));
        CU(cudaMemcpy(ctx->tc_B, hB, sizeof(float) * R * KT, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(ctx->tc_idx, hidx, sizeof(uint32_t) * R, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(ctx->tc_rowsxyz, hrows, sizeof(float) * R * d, cudaMemcpyHostToDevice));
      }
      ctx->h_row_base = rb;
      CU(cudaMemcpy(ctx->tc_row_base, rb.data(), sizeof(long long) * (nl + 1), cudaMemcpyHostToDevice));
      CU(cudaMemcpy(ctx->tc_centroid, hcen.data(), sizeof(float) * nl * KT, cudaMemcpyHostToDevice));
      {
        // bounding box of every 128-row chunk (the scan's chunk) of the TC layout
        std::vector<int> cb(nl + 1, 0);
        for (int l = 0; l < nl; ++l) cb[l + 1] = cb[l] + (int)((rb[l + 1] - rb[l] + 127) / 128);
        std::vector<float> box((size_t)cb[nl] * 2 * d);
        for (int l = 0; l < nl; ++l)
          for (int c = 0; c < cb[l + 1] - cb[l]; ++c) {
            float* bx = box.data() + (size_t)(cb[l] + c) * 2 * d;
            for (int j = 0; j < d; ++j) { bx[j] = __builtin_inff(); bx[d + j] = -__builtin_inff(); }
            const long long r0 = rb[l] + 128ll * c, r1 = std::min(rb[l + 1], r0 + 128);
            for (long long r = r0; r < r1; ++r) {
              if (hidx[r] == kIndexSentinel) continue;
              for (int j = 0; j < d; ++j) {
                bx[j] = std::min(bx[j], hrows[r * d + j]);
                bx[d + j] = std::max(bx[d + j], hrows[r * d + j]);
              }
            }
          }
        CU(cudaMalloc(&ctx->tc_cbase, sizeof(int) * (nl + 1)));
        CU(cudaMemcpy(ctx->tc_cbase, cb.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice));
        CU(cudaMalloc(&ctx->tc_box, sizeof(float) * box.size()));
        CU(cudaMemcpy(ctx->tc_box, box.data(), sizeof(float) * box.size(), cudaMemcpyHostToDevice));
        if (KT == kSplitKT && d <= kSplitMaxD) {
          // split rounds: windows of W consecutive chunks (<= 64 per leaf), box = union of its chunks
          int W = 4;  // config 2: W = 1 / 2 / 4 -> 22.1 / 27.7 / 29.9 M q/s (before renumbering)
          if (const char* e = std::getenv("BKT_SPLIT_W")) W = std::max(1, std::atoi(e));
          int maxch = 1;
          for (int l = 0; l < nl; ++l) maxch = std::max(maxch, cb[l + 1] - cb[l]);
          while ((maxch + W - 1) / W > 64) W *= 2;
          std::vector<int> wb(nl + 1, 0);
          for (int l = 0; l < nl; ++l) wb[l + 1] = wb[l] + (cb[l + 1] - cb[l] + W - 1) / W;
          std::vector<float> wbox((size_t)wb[nl] * 2 * d);
          int NW = 1;
          for (int l = 0; l < nl; ++l) {
            const int nch = cb[l + 1] - cb[l];
            NW = std::max(NW, wb[l + 1] - wb[l]);
            for (int w = 0; w < wb[l + 1] - wb[l]; ++w) {
              float* bx = wbox.data() + (size_t)(wb[l] + w) * 2 * d;  // {lo, -hi} per dimension
              for (int j = 0; j < d; ++j) { bx[2 * j] = __builtin_inff(); bx[2 * j + 1] = __builtin_inff(); }
              for (int c = w * W; c < std::min(nch, (w + 1) * W); ++c) {
                const float* cx = box.data() + (size_t)(cb[l] + c) * 2 * d;
                for (int j = 0; j < d; ++j) {
                  bx[2 * j] = std::min(bx[2 * j], cx[j]);
                  bx[2 * j + 1] = std::min(bx[2 * j + 1], -cx[d + j]);
                }
              }
            }
          }
          CU(cudaMalloc(&ctx->win_base, sizeof(int) * (nl + 1)));
          CU(cudaMemcpy(ctx->win_base, wb.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice));
          CU(cudaMalloc(&ctx->win_box, sizeof(float) * wbox.size()));
          CU(cudaMemcpy(ctx->win_box, wbox.data(), sizeof(float) * wbox.size(), cudaMemcpyHostToDevice));
          ctx->split_W = W;
          ctx->split_NW = NW;
        }
      }
      ctx->KT = KT;
      ctx->tc_rows = R;
      // The filter's error bound is relative to |q'|^2 + |p'|^2 and assumes
      // no overflow and no flushed products (leafscan_tc.cuh header): a leaf
      // whose centred norms overflow or are tiny-but-nonzero keeps the tree
      // on the CUDA-core scan (same results, no filter).
      bool tc_safe = true;
      for (int l = 0; l < nl; ++l) {
        const float pm = hpn[l];
        if (!(pm <= 1e30f) || (pm > 0.0f && pm < 1e-30f)) tc_safe = false;
      }
      ctx->has_tc = tc_safe;
    }
    return BKT_OK;
  };
  ctx->residency = residency;
  if (residency == 0) {
    CU(cudaMalloc(&ctx->pts, pts_bytes));
    CU(cudaMalloc(&ctx->pidx, idx_bytes));
    CU(cudaMemcpy(ctx->pts, ctx->h_pts, pts_bytes, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->pidx, ctx->h_pidx, idx_bytes, cudaMemcpyHostToDevice));
    hfree(ctx->h_pts);
    hfree(ctx->h_pidx);
    ctx->num_chunks = 1;
    ctx->wide_pts = ctx->pts;
    ctx->wide_pidx = ctx->pidx;
    if (int rc = build_tc(false)) return rc;
  } else {
    // chunk bounds: the reference row bounds (ChunkPlan.bounds) mapped to the
    // containing quad of the padded layout; results do not depend on where a
    // chunk boundary falls (reference scheduler.py:1-10, acceptance crit. 2).
    ctx->num_chunks = num_chunks;
    if (!spill) {
      float* dp = nullptr;
      uint32_t* di = nullptr;
      CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), ctx->h_pts, 0));
      CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&di), ctx->h_pidx, 0));
      ctx->wide_pts = dp;
      ctx->wide_pidx = di;
    }
    ctx->chunk_q.assign(num_chunks + 1, 0);
    for (int j = 0; j <= num_chunks; ++j) {
      long long row = chunk_bounds ? chunk_bounds[j] : (long long)(((__int128)j * n + num_chunks - 1) / num_chunks);
      if (row <= 0) { ctx->chunk_q[j] = 0; continue; }
      if (row >= n) { ctx->chunk_q[j] = TQ; continue; }
      int l = (int)(std::upper_bound(leaf_starts, leaf_starts + nl + 1, (int64_t)row) - leaf_starts) - 1;
      long long off = row - leaf_starts[l];
      ctx->chunk_q[j] = ctx->h_quad_base[l] + (off + 3) / 4;
    }
    for (int j = 0; j < num_chunks; ++j)
      if (ctx->chunk_q[j + 1] < ctx->chunk_q[j]) return set_err(ctx, BKT_EINVAL, "chunk bounds must be non-decreasing");
    ctx->chunk_leaf_lo.assign(num_chunks, 0);
    ctx->chunk_leaf_hi.assign(num_chunks, -1);
    long long maxq = 0;
    for (int j = 0; j < num_chunks; ++j) {
      long long a = ctx->chunk_q[j], b = ctx->chunk_q[j + 1];
      maxq = std::max(maxq, b - a);
      if (b <= a) continue;
      int lo = (int)(std::upper_bound(ctx->h_quad_base.begin(), ctx->h_quad_base.end(), a) - ctx->h_quad_base.begin()) - 1;
      int hi = (int)(std::lower_bound(ctx->h_quad_base.begin(), ctx->h_quad_base.end(), b) - ctx->h_quad_base.begin()) - 1;
      ctx->chunk_leaf_lo[j] = lo;
      ctx->chunk_leaf_hi[j] = hi;
    }
    // leaf-aligned streaming units of the drain schedule (ooc_drain)
    ctx->unit_leaf_lo.clear();
    ctx->unit_leaf_hi.clear();
    ctx->unit_q.assign(1, 0);
    for (int l = 0, u = -1; l < nl; ++l) {
      const long long q0 = ctx->h_quad_base[l];
      int j = (int)(std::upper_bound(ctx->chunk_q.begin(), ctx->chunk_q.end(), q0) - ctx->chunk_q.begin()) - 1;
      j = std::max(0, std::min(j, num_chunks - 1));
      if (j != u) {
        if (!ctx->unit_leaf_lo.empty()) ctx->unit_q.push_back(q0);
        ctx->unit_leaf_lo.push_back(l);
        ctx->unit_leaf_hi.push_back(l);
        u = j;
      } else {
        ctx->unit_leaf_hi.back() = l;
      }
    }
    ctx->unit_q.push_back(ctx->h_quad_base[nl]);
    for (size_t u = 0; u + 1 < ctx->unit_q.size(); ++u) maxq = std::max(maxq, ctx->unit_q[u + 1] - ctx->unit_q[u]);
    ctx->slot_quads = std::max<long long>(maxq, 1);
    // tensor-core drain: the filter layout stays on the host, streamed per unit
    if (int rc = build_tc(true)) return rc;
    if (ctx->has_tc) {
      long long maxr = 1;
      ctx->unit_r.clear();
      for (size_t u = 0; u < ctx->unit_leaf_lo.size(); ++u) {
        ctx->unit_r.push_back(ctx->h_row_base[ctx->unit_leaf_lo[u]]);
        maxr = std::max(maxr, ctx->h_row_base[ctx->unit_leaf_hi[u] + 1] - ctx->h_row_base[ctx->unit_leaf_lo[u]]);
      }
      ctx->unit_r.push_back(ctx->h_row_base[nl]);
      for (int s = 0; s < 2; ++s) {
        CU(cudaMalloc(&ctx->slot_tcB[s], sizeof(float) * maxr * ctx->KT));
        CU(cudaMalloc(&ctx->slot_tcidx[s], sizeof(uint32_t) * maxr));
        CU(cudaMalloc(&ctx->slot_tcrows[s], sizeof(float) * maxr * d));
      }
    }
    for (int s = 0; s < 2; ++s) {
      CU(cudaMalloc(&ctx->slot_pts[s], sizeof(float) * ctx->slot_quads * 4 * D));
      CU(cudaMalloc(&ctx->slot_idx[s], sizeof(uint32_t) * ctx->slot_quads * 4));
      ctx->slot_chunk[s] = -1;
      ctx->slot_unit[s] = -1;
    }
  }
  if (wide_only) {
    ctx->min_leaf = *std::min_element(ctx->h_leaf_size.begin(), ctx->h_leaf_size.end());
    ctx->has_tree = true;
    return BKT_OK;
  }
  if (ctx->nkeys == 0) {
    // one block per leaf (no leaf-internal order)
    ctx->nkeys = nl;
    std::vector<int> ident(nl + 1);
    for (int l = 0; l <= nl; ++l) ident[l] = l;
    CU(cudaMalloc(&ctx->blk_base, sizeof(int) * (nl + 1)));
    CU(cudaMemcpy(ctx->blk_base, ident.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice));
  }
  // sub-buckets per leaf: one per block of the largest leaf (power of two)
  ctx->sub_w = 1;
  {
    int maxnb = 1;
    for (int l = 0; l < nl; ++l) maxnb = std::max(maxnb, (int)((ctx->h_leaf_size[l] + kBlockRows - 1) / kBlockRows));
    if (ctx->nkeys > nl)
      while (ctx->sub_w < maxnb && ctx->sub_w < 64) ctx->sub_w <<= 1;
  }
  if (const char* e = std::getenv("BKT_SUB_W")) {
    int w = std::atoi(e);
    if (w >= 1 && (w & (w - 1)) == 0) ctx->sub_w = w;
  }
  ctx->nbuckets = nl * std::max(ctx->sub_w, ctx->split_NW);
  ctx->min_leaf = *std::min_element(ctx->h_leaf_size.begin(), ctx->h_leaf_size.end());
  if (ensure_leafbufs(ctx, nl, ctx->nbuckets) != BKT_OK) return BKT_ECUDA;
  ctx->has_tree = true;
  return BKT_OK;
}

}  // extern "C"

// =============================================================================
// search
// =============================================================================
namespace {

struct SearchRun {
  long long m = 0;
  int k = 0;
  int kb = 0;
  bool fma = false;
  bool tc = false;
  bool unfused = false;
  int tc_rows = 128;  // TC chunk width (BKT_TC_N): 64 or 128 columns
  int tc_cps = 2;     // TC CTAs per SM (BKT_TC_CPS=3: 64-column chunks, one control warp)
  int grid_scan = 0;
  int grid_small = 0;
  bool timing = false;
  long long launches = 0;
  long long leafscan_launches = 0;
  double leafscan_ms = 0;
  size_t ev_next = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> scan_events;
  long long rounds = 0;
  long long scans = 0;
  bool seq = false;
  long long seq_cap = 0;
  bool counters = false;
  unsigned long long* ctr_rounds = nullptr;  // BKT_TRACE_ROUNDS + counters: a 16-counter snapshot per leafscan launch
  int ctr_rounds_cap = 0;
  // early result drain (single batch, host results): when at most drain_at
  // queries remain active, snapshot them and start copying every row to the
  // host while the tail rounds run; drain_start() launches the copy
  long long drain_at = -1;
  long long finish_at = -1;  // tail finisher: one launch once at most this many queries remain (-1: off)
  bool finish_cta = false;   // finisher with one CTA per query (else one warp per query)
  bool split = false;        // later rounds as (leaf, window) items (split_scan.cuh)
  const float* unit_B = nullptr;       // drain: the resident unit's filter rows (row-indexed, origin applied)
  const uint32_t* unit_idx = nullptr;
  const float* unit_rows = nullptr;
  bool pdl = true;           // fused leaf-level rounds: programmatic dependent launches (BKT_PDL=0: off)
  bool scan_pdl = false;     // the next leaf-scan launch uses PDL
  bool drain = true;         // out-of-core: drain schedule (ooc_drain); BKT_OOC_ROUNDS=1: one round per leaf visit
  bool graph = false;        // split rounds replayed from a captured CUDA graph (launch-bound searches)
  long long stream_bytes = 0;   // out-of-core chunk streaming (bkt_stats.stream_bytes)
  long long stream_copies = 0;
  bool wide = false;         // general-domain path (wide_search.cuh)
  bool wide_rows_smem = true;
  size_t wide_smem = 0;
  bool renumber = false;     // search in home-bucket order (gather_rows_kernel)
  bool verbose = false;      // BKT_VERBOSE: split-round totals on stderr
  int split_from = 1;        // first split round (earlier rounds: leaf-level tiles)
  bool drain_fired = false;
  std::function<void()> drain_start;
};

ScanArgs make_scan_args(bkt_ctx* ctx, SearchRun& R, int cur) {
  ScanArgs a{};
  a.q = ctx->q;
  a.keys = ctx->keys;
  a.state = ctx->state;
  a.next = ctx->next;
  a.visits = ctx->visits;
  a.work = ctx->work[cur];
  a.leaf_off = ctx->leaf_off;
  a.tile_off = ctx->tile_off;
  a.num_tiles = &ctx->ctl->num_tiles;
  a.tile_lo = 0;
  a.tile_hi = -1;
  a.tiles = ctx->tiles;
  a.counts = ctx->counts;
  a.pos = ctx->pos;
  // dynamic tile order for the CUDA-core scan when leaves are long (config 4
  // d = 5: +10%); with leaves of a few chunks (config 1: 2 chunks per tile)
  // the producer's shorter lookahead costs more than the balance gains (-14%)
  a.tile_next = ctx->n >= 1024ll * ctx->nl ? &ctx->ctl->tile_next : nullptr;
  a.pts = ctx->pts;
  a.pidx = ctx->pidx;
  a.quad_origin = 0;
  a.clip_lo = 0;
  a.clip_hi = ctx->total_quads;
  a.quad_base = ctx->quad_base;
  a.leaf_size = ctx->leaf_size;
  a.top = TopTreeView{ctx->split, ctx->h, ctx->d};
  a.k = R.k;
  a.fused = 1;
  a.zero = 0ull;
  a.pairs = ctx->pairs;
  a.seq_log = R.seq ? ctx->seq_dev : nullptr;
  a.seq_pos = ctx->seq_pos;
  a.seq_cap = R.seq_cap;
  return a;
}

int launch_scan(bkt_ctx* ctx, SearchRun& R, const ScanArgs& a) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (R.timing) {
    e0 = get_event(ctx, R.ev_next++);
    e1 = get_event(ctx, R.ev_next++);
    CU(cudaEventRecord(e0, ctx->stream));
  }
  if (R.tc) {
    TcArgs t{};
    t.s = a;
    t.B = R.unit_B ? R.unit_B : ctx->tc_B;
    t.ridx = R.unit_idx ? R.unit_idx : ctx->tc_idx;
    t.rows = R.unit_rows ? R.unit_rows : ctx->tc_rowsxyz;
    t.row_base = ctx->tc_row_base;
    t.centroid = ctx->tc_centroid;
    t.pnmax = ctx->tc_pnmax;
    t.cbase = ctx->tc_cbase;
    t.box = ctx->tc_box;
    t.kth = ctx->kthv;
    t.d = ctx->d;
    t.qstride = ctx->D;
    t.spin = 0;  // measured: suspending waits beat spinning by 2.6% on config 2 (BKT_TC_SPIN: 1 MMA, 2 epilogue)
    t.ctr = R.counters ? ctx->tc_ctr : nullptr;
    t.sub_w = ctx->sub_w;
    t.tile_next = &ctx->ctl->tile_next;
    t.pdl = R.scan_pdl && !R.timing ? 1 : 0;  // (timed launches keep their events adjacent)
    if (const char* e = std::getenv("BKT_TC_SPIN")) t.spin = std::atoi(e);
    const char* dbg_env = std::getenv("BKT_TC_DEBUG");
    if (dbg_env && R.leafscan_launches == (*dbg_env ? std::atoi(dbg_env) : 5)) {
      // per-chunk timestamps of CTA 0 in one leafscan launch (BKT_TC_DEBUG=<launch>: 0 is the home
      // round; empty: the 6th)
      static long long* dbg = nullptr;
      const int cap = 4096;
      const int extra = 2048;  // per-CTA start / end stamps
      if (!dbg) cudaMalloc(&dbg, sizeof(long long) * (16 * cap + extra));
      cudaMemsetAsync(dbg, 0, sizeof(long long) * (16 * cap + extra), ctx->stream);
      t.dbg = dbg;
      t.dbg_cap = cap;
      CU(launch_leafscan_tc(ctx->KT, R.kb, R.fma, R.grid_scan, ctx->stream, t, nullptr, R.tc_rows, R.tc_cps));
      std::vector<long long> h(16 * cap + extra);
      CU(cudaMemcpyAsync(h.data(), dbg, sizeof(long long) * (16 * cap + extra), cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      {
        // load balance: per-CTA end of the epilogue's tile loop, from the earliest CTA start
        long long s0 = LLONG_MAX, e_min = LLONG_MAX, e_max = 0;
        double e_sum = 0;
        const int nct = std::min(R.grid_scan, 1024);
        for (int c = 0; c < nct; ++c) s0 = std::min(s0, h[16 * cap + c]);
        for (int c = 0; c < nct; ++c) {
          const long long e = h[16 * cap + 1024 + c] - s0;
          e_min = std::min(e_min, e);
          e_max = std::max(e_max, e);
          e_sum += e;
        }
        std::fprintf(stderr, "cta balance: %d CTAs, end min %.1f us mean %.1f us max %.1f us (max/mean %.3f)\n", nct,
                     e_min / 1e3, e_sum / nct / 1e3, e_max / 1e3, e_max / (e_sum / nct));
      }
      long long base = h[0];
      auto rel = [&](long long v) { return v ? v - base : -1; };
      for (int g = 0; g < cap && h[16 * g + 5]; ++g)
        std::fprintf(stderr, "chunk %d tile %lld prod_wait %lld prod_issue %lld mma_ready %lld epi_start %lld epi_ready %lld "
                     "epi_done %lld ld0 %lld g0 %lld g1 %lld g2 %lld g3 %lld trips %lld anyg %lld\n",
                     g, h[16 * g + 6], rel(h[16 * g]), rel(h[16 * g + 1]), rel(h[16 * g + 2]), rel(h[16 * g + 3]),
                     rel(h[16 * g + 4]), rel(h[16 * g + 5]), rel(h[16 * g + 7]), rel(h[16 * g + 8]), rel(h[16 * g + 9]),
                     rel(h[16 * g + 10]), rel(h[16 * g + 11]), h[16 * g + 12], h[16 * g + 13]);
      R.launches++;
      R.leafscan_launches++;
      return BKT_OK;
    }
    const bool skipdiag = R.counters && std::getenv("BKT_TC_SKIPDIAG");
    if (skipdiag) {
      // how many (tile, chunk) pairs some query of the tile needs (box lower
      // bound <= its k-th distance at the tile start), per round
      constexpr int kNeedCap = 1 << 21;
      if (!ctx->tc_need) CU(cudaMalloc(&ctx->tc_need, sizeof(unsigned long long) * kNeedCap));
      CU(cudaMemsetAsync(ctx->tc_need, 0, sizeof(unsigned long long) * kNeedCap, ctx->stream));
      t.need_dbg = ctx->tc_need;
    }
    CU(launch_leafscan_tc(ctx->KT, R.kb, R.fma, R.grid_scan, ctx->stream, t, nullptr, R.tc_rows, R.tc_cps));
    if (skipdiag) {
      int nt = 0;
      CU(cudaMemcpyAsync(&nt, &ctx->ctl->num_tiles, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      nt = std::min(nt, 1 << 21);
      std::vector<int4> tiles(nt);
      std::vector<unsigned long long> need(nt);
      std::vector<long long> rbh(ctx->nl + 1);
      CU(cudaMemcpy(tiles.data(), ctx->tiles, sizeof(int4) * nt, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(need.data(), ctx->tc_need, sizeof(unsigned long long) * nt, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(rbh.data(), ctx->tc_row_base, sizeof(long long) * (ctx->nl + 1), cudaMemcpyDeviceToHost));
      long long tot = 0, nd = 0;
      for (int i = 0; i < nt; ++i) {
        const long long nc = std::min(64ll, (rbh[tiles[i].x + 1] - rbh[tiles[i].x] + 127) / 128);
        tot += nc;
        nd += __builtin_popcountll(need[i]);
      }
      std::fprintf(stderr, "skipdiag launch %d tiles %d cta_chunks %lld cta_needed %lld (%.3f)\n", R.leafscan_launches, nt,
                   tot, nd, tot ? (double)nd / tot : 0.0);
    }
    if (R.ctr_rounds && R.leafscan_launches < R.ctr_rounds_cap)
      CU(cudaMemcpyAsync(R.ctr_rounds + 16 * R.leafscan_launches, ctx->tc_ctr, sizeof(unsigned long long) * 16,
                         cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    CU(launch_leafscan(ctx->D, R.kb, R.fma, R.grid_scan, ctx->stream, a, nullptr));
  }
  if (R.timing) {
    CU(cudaEventRecord(e1, ctx->stream));
    R.scan_events.push_back({e0, e1});
  }
  R.launches++;
  R.leafscan_launches++;
  return BKT_OK;
}

// Out-of-core round: stream the chunks that hold buffered work through the two
// device slots (sec. 3.2 Brute/Copy/Wait; reference ChunkPipeline.run_round,
// device.py:422-446).  Chunks without work are skipped and chunks still resident
// from the previous round are not copied again.
int ooc_round(bkt_ctx* ctx, SearchRun& R, int cur) {
  // tile offsets of this round to the host (needed to pick chunks with work)
  CU(cudaMemcpyAsync(ctx->h_tile_off, ctx->tile_off, sizeof(int) * (ctx->nl + 1), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  std::vector<int> need;
  for (int j = 0; j < ctx->num_chunks; ++j) {
    if (ctx->chunk_leaf_hi[j] < ctx->chunk_leaf_lo[j]) continue;
    int t0 = ctx->h_tile_off[ctx->chunk_leaf_lo[j]], t1 = ctx->h_tile_off[ctx->chunk_leaf_hi[j] + 1];
    if (t1 > t0) need.push_back(j);
  }
  // Chunks still resident from the previous round go first, so a round copies
  // only (chunks with work - 2) chunks and leaves its last two resident for the
  // next round (the reference re-streams every chunk every round,
  // device.py:432-446; results do not depend on the order).
  std::stable_partition(need.begin(), need.end(),
                        [&](int j) { return ctx->slot_chunk[0] == j || ctx->slot_chunk[1] == j; });
  const int D = ctx->D;
  auto ensure_resident = [&](int j, int avoid_slot) -> int {
    for (int s = 0; s < 2; ++s)
      if (ctx->slot_chunk[s] == j) return s;
    int s = (avoid_slot == 0) ? 1 : 0;
    if (avoid_slot < 0) s = (ctx->slot_chunk[0] < 0) ? 0 : ((ctx->slot_chunk[1] < 0) ? 1 : 0);
    long long a = ctx->chunk_q[j], b = ctx->chunk_q[j + 1];
    cudaStreamWaitEvent(ctx->copy_stream, ctx->slot_free[s], 0);
    cudaMemcpyAsync(ctx->slot_pts[s], ctx->h_pts + a * 4 * D, sizeof(float) * (b - a) * 4 * D,
                    cudaMemcpyHostToDevice, ctx->copy_stream);
    cudaMemcpyAsync(ctx->slot_idx[s], ctx->h_pidx + a * 4, sizeof(uint32_t) * (b - a) * 4, cudaMemcpyHostToDevice,
                    ctx->copy_stream);
    cudaEventRecord(ctx->slot_ready[s], ctx->copy_stream);
    ctx->slot_chunk[s] = j;
    ctx->slot_unit[s] = -1;
    R.stream_bytes += (sizeof(float) * 4 * D + sizeof(uint32_t) * 4) * (b - a);
    R.stream_copies += 1;
    return s;
  };
  std::vector<int> slot_of(need.size(), -1);
  if (!need.empty()) slot_of[0] = ensure_resident(need[0], -1);
  for (size_t i = 0; i < need.size(); ++i) {
    int j = need[i];
    int s = slot_of[i];
    // prefetch the next chunk into the other slot while this one computes
    if (i + 1 < need.size()) slot_of[i + 1] = ensure_resident(need[i + 1], s);
    CU(cudaStreamWaitEvent(ctx->stream, ctx->slot_ready[s], 0));
    ScanArgs a = make_scan_args(ctx, R, cur);
    a.fused = 0;
    a.pts = ctx->slot_pts[s];
    a.pidx = ctx->slot_idx[s];
    a.quad_origin = ctx->chunk_q[j];
    a.clip_lo = ctx->chunk_q[j];
    a.clip_hi = ctx->chunk_q[j + 1];
    a.tile_lo = ctx->h_tile_off[ctx->chunk_leaf_lo[j]];
    a.tile_hi = ctx->h_tile_off[ctx->chunk_leaf_hi[j] + 1];
    int rc = launch_scan(ctx, R, a);
    if (rc != BKT_OK) return rc;
    CU(cudaEventRecord(ctx->slot_free[s], ctx->stream));
  }
  // FindLeaf after every chunk of the round has been scanned
  findleaf_kernel<<<R.grid_small, 256, start_tree_smem(ctx->h) * 4, ctx->stream>>>(
      ctx->work[cur], ctx->ctl, ctx->q, ctx->D, R.k, TopTreeView{ctx->split, ctx->h, ctx->d}, ctx->keys, ctx->state,
      ctx->next, ctx->visits, ctx->counts, ctx->pos, R.seq ? ctx->seq_dev : nullptr, ctx->seq_pos, R.seq_cap);
  CU(cudaGetLastError());
  R.launches++;
  return BKT_OK;
}

// One batch: queries already in ctx->q (m x D).  Runs rounds until no query is active.
// one launch of the tail finisher over `list` (ctl->active entries)
int launch_finisher(bkt_ctx* ctx, SearchRun& R, const int* list, const FinishUnit& fu = FinishUnit{},
                    const float* unit_pts = nullptr, const uint32_t* unit_pidx = nullptr) {
  const float* pts = unit_pts ? unit_pts : ctx->pts;
  const uint32_t* pidx = unit_pidx ? unit_pidx : ctx->pidx;
  const int blocks = (int)std::max<long long>(1, (R.finish_at + kFinishWarps - 1) / kFinishWarps);
  const TopTreeView top{ctx->split, ctx->h, ctx->d};
  int* seq = R.seq ? ctx->seq_dev : nullptr;
  const int cta_blocks = (int)std::max<long long>(1, std::min<long long>(R.finish_at, ctx->sm_count * 8ll));
  if (R.finish_cta && R.fma)
    finish_cta_kernel<true><<<cta_blocks, kFinishT, 0, ctx->stream>>>(
        list, ctx->ctl, ctx->q, ctx->D, R.k, top, ctx->keys, ctx->state, ctx->next, ctx->visits,
        pts, pidx, ctx->quad_base, ctx->leaf_size, ctx->pairs, seq, ctx->seq_pos, R.seq_cap, fu);
  else if (R.finish_cta)
    finish_cta_kernel<false><<<cta_blocks, kFinishT, 0, ctx->stream>>>(
        list, ctx->ctl, ctx->q, ctx->D, R.k, top, ctx->keys, ctx->state, ctx->next, ctx->visits,
        pts, pidx, ctx->quad_base, ctx->leaf_size, ctx->pairs, seq, ctx->seq_pos, R.seq_cap, fu);
  else if (R.fma)
    finish_kernel<true><<<blocks, kFinishWarps * 32, 0, ctx->stream>>>(
        list, ctx->ctl, ctx->q, ctx->D, R.k, top, ctx->keys, ctx->state, ctx->next, ctx->visits,
        pts, pidx, ctx->quad_base, ctx->leaf_size, ctx->pairs, seq, ctx->seq_pos, R.seq_cap, fu);
  else
    finish_kernel<false><<<blocks, kFinishWarps * 32, 0, ctx->stream>>>(
        list, ctx->ctl, ctx->q, ctx->D, R.k, top, ctx->keys, ctx->state, ctx->next, ctx->visits,
        pts, pidx, ctx->quad_base, ctx->leaf_size, ctx->pairs, seq, ctx->seq_pos, R.seq_cap, fu);
  CU(cudaGetLastError());
  R.launches++;
  return BKT_OK;
}

// advance over `list` (ctl->active entries): merge, FindLeaf, next-leaf bucket slot, A row
int launch_advance_round(bkt_ctx* ctx, SearchRun& R, const int* list) {
  AdvanceArgs a{};
  a.list = list;
  a.ctl = ctx->ctl;
  a.pos = ctx->pos;
  a.counts = ctx->counts;
  a.q = ctx->q;
  a.D = ctx->D;
  a.k = R.k;
  a.top = TopTreeView{ctx->split, ctx->h, ctx->d};
  a.keys = ctx->keys;
  a.qs = ctx->qs;
  a.ccnt = ctx->ccnt;
  a.cand = ctx->cand;
  a.rows = ctx->tc_rowsxyz;
  a.ridx = ctx->tc_idx;
  a.fma = R.fma ? 1 : 0;
  a.NW = ctx->split_NW;
  a.capw = ctx->split_capw;
  a.centroid = ctx->tc_centroid;
  a.arow = ctx->arow;
  a.seq_log = R.seq ? ctx->seq_dev : nullptr;
  a.seq_pos = ctx->seq_pos;
  a.seq_cap = R.seq_cap;
  CU(launch_advance(R.kb, R.grid_small, ctx->stream, a));
  R.launches++;
  return BKT_OK;
}

// Out-of-core drain (residency 1, the default schedule): the streaming units
// are taken in order and each resident unit is drained -- its queries are
// scanned, advanced and re-bucketed round after round until none of them has
// a next leaf inside the unit -- before the next unit is used.  A query whose
// next leaf lies in another unit is parked; a pass over the units classifies
// the park list.  Every query's visits happen in its own traversal order with
// the same per-visit merge, so keys, visited counts and leaf sequences equal
// the round-synchronous schedule's (reference buffer_tree.py:523-646; results
// do not depend on the processing schedule, reference tests 263-284); what
// changes is the number of times a unit crosses PCIe: a depth-first traversal
// leaves a leaf-aligned unit (a subtree when chunks are equal) once, so a
// query needs about one pass per unit it touches instead of one round per
// leaf (sec. 3.2 processes a chunk's buffers the same way: all
// queries buffered for its leaves, repeatedly, while it is resident).
// Sub-rounds are launched kRing - 1 ahead of the host's check of their
// active count; rounds after the unit empties have no work.
int ooc_drain(bkt_ctx* ctx, SearchRun& R) {
  const long long m = R.m;
  if (ctx->park_cap < m) {
    dfree(ctx->park[0]); dfree(ctx->park[1]);
    ctx->park_cap = 0;
    CU(cudaMalloc(&ctx->park[0], sizeof(int) * std::max<long long>(m, 1)));
    CU(cudaMalloc(&ctx->park[1], sizeof(int) * std::max<long long>(m, 1)));
    ctx->park_cap = m;
  }
  // the start kernel's home-round buckets are not used: the drain buckets by leaf
  CU(cudaMemsetAsync(ctx->counts, 0, sizeof(int) * ctx->nbuckets, ctx->stream));
  ooc_init_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(ctx->park[0], m, ctx->ctl);
  CU(cudaGetLastError());
  R.launches++;
  for (int s = 0; s < 2; ++s) ctx->slot_chunk[s] = -1;  // the round schedule's slot tags
  const int U = (int)ctx->unit_leaf_lo.size();
  const int D = ctx->D;
  cudaEvent_t* ring = ctx->ring_ev;
  int plans = 0;
  // control block of the plan launched as number `seq` in mirror slot `slot`
  auto mirror = [&](int slot, int seq, RoundCtl& c) -> int {
    CU(cudaEventSynchronize(ring[slot]));
    volatile RoundCtl* v = ctx->h_ctl + slot;
    // the event orders the plan before this read; the mapped write can trail it briefly
    for (long long spin = 0; v->plan_seq != seq; ++spin)
      if (spin > (1ll << 32)) return set_err(ctx, BKT_ECUDA, "out-of-core drain: control block never arrived");
    std::memcpy(&c, const_cast<RoundCtl*>(v), sizeof(RoundCtl));
    return BKT_OK;
  };
  auto plan = [&](long long slot) -> int {
    plan_kernel<<<1, kPlanThreads, 0, ctx->stream>>>(ctx->counts, ctx->key_off, 1, ctx->nl, ctx->leaf_off,
                                                     ctx->tile_off, ctx->ctl, ctx->nl, kNT, ctx->hist, kHistCap,
                                                     ctx->d_ctl_mirror + slot);
    CU(cudaGetLastError());
    CU(cudaEventRecord(ring[slot], ctx->stream));
    R.launches++;
    return ++plans;
  };
  auto scatter = [&](const int* prev, int* out) -> int {
    scatter_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(prev, 0, ctx->pos, ctx->qkey, ctx->key_off, out, ctx->ctl,
                                                           ctx->leaf_off, ctx->tile_off, ctx->nl, 1, kNT, ctx->tiles,
                                                           (int)std::min<long long>(ctx->tiles_cap, INT32_MAX));
    CU(cudaGetLastError());
    R.launches++;
    return BKT_OK;
  };
  auto ensure_resident = [&](int u, int avoid_slot) -> int {
    for (int s = 0; s < 2; ++s)
      if (ctx->slot_unit[s] == u) return s;
    int s = avoid_slot >= 0 ? (avoid_slot ^ 1) : (ctx->slot_unit[0] < 0 ? 0 : (ctx->slot_unit[1] < 0 ? 1 : 0));
    const long long a = ctx->unit_q[u], b = ctx->unit_q[u + 1];
    cudaStreamWaitEvent(ctx->copy_stream, ctx->slot_free[s], 0);
    cudaMemcpyAsync(ctx->slot_pts[s], ctx->h_pts + a * 4 * D, sizeof(float) * (b - a) * 4 * D,
                    cudaMemcpyHostToDevice, ctx->copy_stream);
    cudaMemcpyAsync(ctx->slot_idx[s], ctx->h_pidx + a * 4, sizeof(uint32_t) * (b - a) * 4, cudaMemcpyHostToDevice,
                    ctx->copy_stream);
    R.stream_bytes += (sizeof(float) * 4 * D + sizeof(uint32_t) * 4) * (b - a);
    if (R.tc) {
      const long long r0 = ctx->unit_r[u], r1 = ctx->unit_r[u + 1], KT = ctx->KT, dd = ctx->d;
      cudaMemcpyAsync(ctx->slot_tcB[s], ctx->h_tcB + r0 * KT, sizeof(float) * (r1 - r0) * KT, cudaMemcpyHostToDevice,
                      ctx->copy_stream);
      cudaMemcpyAsync(ctx->slot_tcidx[s], ctx->h_tcidx + r0, sizeof(uint32_t) * (r1 - r0), cudaMemcpyHostToDevice,
                      ctx->copy_stream);
      cudaMemcpyAsync(ctx->slot_tcrows[s], ctx->h_tcrows + r0 * dd, sizeof(float) * (r1 - r0) * dd,
                      cudaMemcpyHostToDevice, ctx->copy_stream);
      R.stream_bytes += (sizeof(float) * (KT + dd) + sizeof(uint32_t)) * (r1 - r0);
    }
    cudaEventRecord(ctx->slot_ready[s], ctx->copy_stream);
    ctx->slot_unit[s] = u;
    R.stream_copies += 1;
    return s;
  };
  int a = 0;  // park[a]: the list the next classify reads
  int cur = 0;
  long long slot_ctr = 0;
  // start with a unit already resident (a previous batch's last)
  int u0 = 0;
  for (int s = 0; s < 2; ++s)
    if (ctx->slot_unit[s] >= 0) u0 = ctx->slot_unit[s];
  bool done = false;
  int idle = 0;  // consecutive units without work (a full pass of them: nothing left)
  for (int step = 0; !done; ++step) {
    const int u = (u0 + step) % U;
    const int lo = ctx->unit_leaf_lo[u], hi = ctx->unit_leaf_hi[u];
    ooc_switch_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctl);
    ooc_classify_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(ctx->park[a], ctx->ctl, ctx->next, lo, hi, ctx->counts,
                                                               ctx->pos, ctx->park[a ^ 1]);
    CU(cudaGetLastError());
    R.launches += 2;
    const int slot0 = (int)(slot_ctr++ % kRing);
    const int seq0 = plan(slot0);
    if (seq0 < 0) return seq0;
    RoundCtl c0;
    if (int rc = mirror(slot0, seq0, c0)) return rc;
    const int list = a;
    a ^= 1;
    if (c0.active == 0) {
      if (c0.park_n == 0) done = true;
      else if (++idle > U) return set_err(ctx, BKT_ECUDA, "out-of-core drain: parked queries match no unit");
      continue;
    }
    idle = 0;
    const int s = ensure_resident(u, -1);
    // the next unit streams into the other slot while this one drains
    if (U > 1) ensure_resident((u + 1) % U, s);
    scatter(ctx->park[list], ctx->work[cur]);
    CU(cudaStreamWaitEvent(ctx->stream, ctx->slot_ready[s], 0));
    std::vector<int> seqs(kRing, 0);
    long long sub = 0;
    int parked = 0;
    for (;;) {
      ScanArgs sa = make_scan_args(ctx, R, cur);
      if (R.tc) {
        // row-indexed views of the slot (the kernel adds the leaf's global row)
        const long long r0 = ctx->unit_r[u];
        R.unit_B = ctx->slot_tcB[s] - r0 * ctx->KT;
        R.unit_idx = ctx->slot_tcidx[s] - r0;
        R.unit_rows = ctx->slot_tcrows[s] - r0 * ctx->d;
      }
      sa.fused = 0;
      sa.pts = ctx->slot_pts[s];
      sa.pidx = ctx->slot_idx[s];
      sa.quad_origin = ctx->unit_q[u];
      sa.clip_lo = ctx->unit_q[u];
      sa.clip_hi = ctx->unit_q[u + 1];
      int rc = launch_scan(ctx, R, sa);
      if (rc != BKT_OK) return rc;
      findleaf_kernel<<<R.grid_small, 256, start_tree_smem(ctx->h) * 4, ctx->stream>>>(
          ctx->work[cur], ctx->ctl, ctx->q, D, R.k, TopTreeView{ctx->split, ctx->h, ctx->d}, ctx->keys, ctx->state,
          ctx->next, ctx->visits, ctx->counts, ctx->pos, R.seq ? ctx->seq_dev : nullptr, ctx->seq_pos, R.seq_cap, lo,
          hi, ctx->park[a], &ctx->ctl->park_n);
      CU(cudaGetLastError());
      R.launches++;
      const int sl = (int)(slot_ctr++ % kRing);
      seqs[sl] = plan(sl);
      if (seqs[sl] < 0) return seqs[sl];
      scatter(ctx->work[cur], ctx->work[cur ^ 1]);
      cur ^= 1;
      ++sub;
      if (sub >= kRing - 1) {
        const int chk = (int)((slot_ctr - (kRing - 1)) % kRing);
        RoundCtl c;
        if (int rc = mirror(chk, seqs[chk], c)) return rc;
        if (c.active == 0) {
          parked = c.park_n;
          break;
        }
        if (R.finish_at >= 0 && c.active <= R.finish_at) {
          // the unit's last queries walk the rest of their stretch inside it
          // in one launch (work[cur]: the list the last launched round built)
          FinishUnit fu;
          fu.origin = ctx->unit_q[u];
          fu.leaf_lo = lo;
          fu.leaf_hi = hi;
          fu.park = ctx->park[a];
          fu.park_n = &ctx->ctl->park_n;
          fu.kth = ctx->kthv;
          rc = launch_finisher(ctx, R, ctx->work[cur], fu, ctx->slot_pts[s], ctx->slot_idx[s]);
          if (rc != BKT_OK) return rc;
          const int sf = (int)(slot_ctr++ % kRing);
          const int seqf = plan(sf);  // no counts left: active 0, the park count mirrored
          if (seqf < 0) return seqf;
          RoundCtl cf;
          if (int rf = mirror(sf, seqf, cf)) return rf;
          parked = cf.park_n;
          break;
        }
      }
    }
    CU(cudaEventRecord(ctx->slot_free[s], ctx->stream));
    if (parked == 0) done = true;
  }
  R.unit_B = nullptr;
  R.unit_idx = nullptr;
  R.unit_rows = nullptr;
  return BKT_OK;
}

// rounds >= 1 as (leaf, window) items until no query is active.  On entry
// work[cur ^ 1] holds the queries just advanced (pos = their next leaf and
// bucket slot, counts per leaf).
// Enqueues one split round on ctx->stream (no host synchronisation, so it
// can be captured into a CUDA graph).  The round's control block goes to
// mirror slot `slot`; `ring_ev` (or null) is recorded after the plan.
int enqueue_split_round(bkt_ctx* ctx, SearchRun& R, int cur, int slot, cudaEvent_t ring_ev, bool capturing) {
  const int nkeys = ctx->nl * ctx->split_NW;
  {
    // the round's queries bucketed by leaf, in route tiles of kRouteQ
    plan_kernel<<<1, kPlanThreads, 0, ctx->stream>>>(ctx->counts, ctx->key_off, 1, ctx->nl, ctx->leaf_off,
                                                     ctx->tile_off, ctx->ctl, ctx->nl, kRouteQ, ctx->hist, kHistCap,
                                                     ctx->d_ctl_mirror + slot);
    CU(cudaGetLastError());
    R.launches++;
    if (ring_ev) CU(cudaEventRecord(ring_ev, ctx->stream));
    scatter_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(ctx->work[cur ^ 1], 0, ctx->pos, ctx->qkey, ctx->key_off,
                                                           ctx->work[cur], ctx->ctl, ctx->leaf_off, ctx->tile_off,
                                                           ctx->nl, 1, kRouteQ, ctx->tiles,
                                                           (int)std::min<long long>(ctx->tiles_cap, INT32_MAX));
    CU(cudaGetLastError());
    R.launches++;
    RouteArgs ra{};
    ra.work = ctx->work[cur];
    ra.rtiles = ctx->tiles;
    ra.ctl = ctx->ctl;
    ra.qs = ctx->qs;
    ra.q = ctx->q;
    ra.D = ctx->D;
    ra.d = ctx->d;
    ra.NW = ctx->split_NW;
    ra.win_base = ctx->win_base;
    ra.win_box = ctx->win_box;
    ra.leaf_size = ctx->leaf_size;
    ra.qmask = ctx->qmask;
    ra.counts = ctx->counts;
    ra.cbase = ctx->cbase;
    ra.key_off = ctx->key_off;
    ra.stoff = ctx->stoff;
    ra.nkeys = nkeys;
    ra.items = ctx->items;
    ra.stiles = ctx->stiles;
    ra.stiles_cap = (int)std::min<long long>(ctx->stiles_cap, INT32_MAX);
    ra.pairs = ctx->pairs;
    CU(launch_route(R.grid_small, ctx->stream, ra));
    R.launches++;
    CU(launch_plan_split(ctx->stream, ctx->counts, ctx->key_off, nkeys, ctx->stoff, ctx->ctl));
    R.launches++;
    CU(launch_place(R.grid_small, ctx->stream, ra));
    R.launches++;
    SplitScanArgs sa{};
    sa.arow = ctx->arow;
    sa.ccnt = ctx->ccnt;
    sa.cand = ctx->cand;
    sa.ovflag = ctx->ovflag;
    sa.NW = ctx->split_NW;
    sa.capw = ctx->split_capw;
    sa.ovf = ctx->ovf;
    sa.novf = &ctx->ctl->novf;
    sa.items = ctx->items;
    sa.tiles = ctx->stiles;
    sa.num_tiles = &ctx->ctl->stiles;
    sa.tile_next = &ctx->ctl->tile_next;
    sa.B = ctx->tc_B;
    sa.row_base = ctx->tc_row_base;
    sa.W = ctx->split_W;
    sa.stats = R.verbose ? &ctx->ctl->sc_tiles : nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (R.timing && !capturing) {
      e0 = get_event(ctx, R.ev_next++);
      e1 = get_event(ctx, R.ev_next++);
      CU(cudaEventRecord(e0, ctx->stream));
    }
    static long long* sdbg = nullptr;
    const char* sdbg_env = std::getenv("BKT_SPLIT_DEBUG");
    const bool sdbg_now = !capturing && sdbg_env && R.leafscan_launches == std::atoi(sdbg_env);
    constexpr int kDbgCap = 4096;
    if (sdbg_now) {
      if (!sdbg) CU(cudaMalloc(&sdbg, sizeof(long long) * 16 * kDbgCap));
      CU(cudaMemsetAsync(sdbg, 0, sizeof(long long) * 16 * kDbgCap, ctx->stream));
      sa.dbg = sdbg;
      sa.dbg_cap = kDbgCap;
    }
    CU(launch_splitscan(R.fma, kSplitCtas * ctx->sm_count, ctx->stream, sa));
    if (sdbg_now) {
      // per tile: published (producer), afull wait start/ready (epilogue), afull ready (MMA);
      // per chunk: MMA issued, epilogue tfull wait start/ready, released, TMA issued, full ready (MMA)
      std::vector<long long> h(16 * kDbgCap);
      CU(cudaMemcpyAsync(h.data(), sdbg, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      const long long b0 = h[5];
      for (int j = 0; j < kDbgCap && h[8 * j + 5]; ++j)
        std::fprintf(stderr, "stile %d pub %lld ewait %lld eready %lld mready %lld esetup %lld eq %lld\n", j,
                     h[8 * j] - b0, h[8 * j + 5] - b0, h[8 * j + 6] ? h[8 * j + 6] - b0 : -1,
                     h[8 * j + 7] ? h[8 * j + 7] - b0 : -1, h[8 * j + 1] ? h[8 * j + 1] - b0 : -1,
                     h[8 * j + 2] ? h[8 * j + 2] - b0 : -1);
      const long long* hc = h.data() + 8 * kDbgCap;
      for (int g = 0; g < kDbgCap && hc[8 * g + 4]; ++g)
        std::fprintf(stderr, "schunk %d tma %lld full %lld mma %lld ewait %lld eready %lld edone %lld\n", g,
                     hc[8 * g + 5] - b0, hc[8 * g + 6] - b0, hc[8 * g + 1] - b0, hc[8 * g + 2] - b0,
                     hc[8 * g + 3] - b0, hc[8 * g + 4] - b0);
    }
    if (R.timing && !capturing) {
      CU(cudaEventRecord(e1, ctx->stream));
      R.scan_events.emplace_back(e0, e1);
    }
    R.launches++;
    R.leafscan_launches++;
    CU(launch_rescan(R.fma, ctx->sm_count * 4, ctx->stream, ctx->ovf, ctx->ctl, ctx->q, ctx->D, R.k, ctx->d,
                     ctx->keys, ctx->qs, ctx->pts, ctx->pidx, ctx->quad_base, ctx->ccnt,
                     ctx->split_NW, ctx->ovflag));
    R.launches++;
    return launch_advance_round(ctx, R, ctx->work[cur]);
  }
}

// Rounds >= 1 as (leaf, window) items until no query is active.  On entry
// work[cur ^ 1] holds the queries just advanced (pos = their next leaf and
// bucket slot, counts per leaf).
//
// Eager mode: rounds are launched ahead of the host check; the active count
// of round r is read back through mapped memory kRing-1 rounds later.
// Graph mode (launch-bound searches, R.graph): kGraphRounds rounds are
// captured once into a CUDA graph and replayed, one graph launch per group
// instead of eight kernel launches per round; the host checks the last
// round of the previous group (mirror slots: 2 x kGraphRounds).
int split_rounds_loop(bkt_ctx* ctx, SearchRun& R, int cur, long long round, const int** fin) {
  cudaEvent_t* ring = ctx->ring_ev;
  if (!R.graph) {
    for (;;) {
      int rc = enqueue_split_round(ctx, R, cur, (int)(round % kRing), ring[round % kRing], false);
      if (rc != BKT_OK) return rc;
      cur ^= 1;
      ++round;
      if (round >= kRing - 1) {
        const int chk = (int)((round - (kRing - 1)) % kRing);
        CU(cudaEventSynchronize(ring[chk]));
        if (ctx->h_ctl[chk].active == 0) break;
        if (R.finish_at >= 0 && ctx->h_ctl[chk].active <= R.finish_at) {
          // the list just advanced (work[cur ^ 1], ctl->active entries) holds every
          // query still active, each with its next leaf set: finish in one launch
          *fin = ctx->work[cur ^ 1];
          break;
        }
      }
    }
    return BKT_OK;
  }
  static_assert(kGraphRounds % 2 == 0, "a group must return the work lists to their parity");
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  const long long launches0 = R.launches;
  CU(configure_split_kernels(R.fma, R.kb, ctx->h, ctx->d));
  CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  int rc = BKT_OK;
  for (int g = 0; g < kGraphRounds && rc == BKT_OK; ++g)
    rc = enqueue_split_round(ctx, R, cur ^ (g & 1), (int)((round + g) % kMirror), nullptr, true);
  cudaError_t ec = cudaStreamEndCapture(ctx->stream, &graph);
  if (rc != BKT_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  CU(ec);
  const long long per_group = R.launches - launches0;
  R.launches = launches0;
  ec = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  CU(ec);
  struct ExecGuard {
    cudaGraphExec_t e;
    ~ExecGuard() { if (e) cudaGraphExecDestroy(e); }
  } guard{exec};
  cudaEvent_t* gev = ctx->group_ev;
  for (long long j = 0;; ++j) {
    CU(cudaGraphLaunch(exec, ctx->stream));
    CU(cudaEventRecord(gev[j & 1], ctx->stream));
    R.launches += per_group;
    R.leafscan_launches += kGraphRounds;
    round += kGraphRounds;
    if (j == 0) continue;
    // group j-1 done (group j in flight): its last round's control block
    CU(cudaEventSynchronize(gev[(j - 1) & 1]));
    const RoundCtl& c = ctx->h_ctl[(round - kGraphRounds - 1) % kMirror];
    if (c.active == 0) break;
    if (R.finish_at >= 0 && c.active <= R.finish_at) {
      *fin = ctx->work[cur ^ 1];
      break;
    }
  }
  return BKT_OK;
}

// The split rounds on the packed per-query records, then (when the tail is
// handed over) the finisher on the unpacked arrays.  On entry work[cur]
// holds the queries the home round scanned.
int split_rounds(bkt_ctx* ctx, SearchRun& R, int cur, long long round) {
  split_state_pack<<<R.grid_small, 256, 0, ctx->stream>>>(R.m, ctx->kthv, ctx->state, ctx->visits, ctx->next, ctx->qs);
  CU(cudaGetLastError());
  R.launches++;
  int rc = launch_advance_round(ctx, R, ctx->work[cur]);
  if (rc != BKT_OK) return rc;
  const int* fin = nullptr;
  rc = split_rounds_loop(ctx, R, cur ^ 1, round, &fin);
  if (rc != BKT_OK) return rc;
  split_state_unpack<<<R.grid_small, 256, 0, ctx->stream>>>(R.m, ctx->qs, ctx->kthv, ctx->state, ctx->visits,
                                                            ctx->next);
  CU(cudaGetLastError());
  R.launches++;
  return fin ? launch_finisher(ctx, R, fin) : BKT_OK;
}

int search_batch_impl(bkt_ctx* ctx, SearchRun& R);

// The batch in home-bucket order: a first start/plan/scatter pass orders the
// queries by (home leaf, home block); the search runs on the reordered rows
// and its per-query outputs (keys, visit counts, visit log) are mapped back.
// The general-domain path: every query's whole traversal in one launch.
int wide_batch(bkt_ctx* ctx, SearchRun& R) {
  RoundCtl init{};
  init.active = (int)R.m;
  CU(cudaMemcpyAsync(ctx->ctl, &init, sizeof(RoundCtl), cudaMemcpyHostToDevice, ctx->stream));
  WideArgs a{};
  a.q = ctx->q;
  a.D = ctx->D;
  a.m = (int)R.m;
  a.k = R.k;
  a.top = TopTreeView{ctx->split, ctx->h, ctx->d};
  a.keys = ctx->keys;
  a.visits = ctx->visits;
  a.pts = ctx->wide_pts;
  a.pidx = ctx->wide_pidx;
  a.quad_base = ctx->quad_base;
  a.leaf_size = ctx->leaf_size;
  a.pairs = ctx->pairs;
  a.ctl = ctx->ctl;
  a.seq_log = R.seq ? ctx->seq_dev : nullptr;
  a.seq_pos = ctx->seq_pos;
  a.seq_cap = R.seq_cap;
  a.scratch = R.wide_rows_smem ? nullptr : ctx->wide_scratch;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (R.timing) {
    e0 = get_event(ctx, R.ev_next++);
    e1 = get_event(ctx, R.ev_next++);
    CU(cudaEventRecord(e0, ctx->stream));
  }
  CU(launch_wide(R.fma, (int)std::min<long long>(R.grid_scan, std::max<long long>(R.m, 1)), ctx->stream, a,
                 R.wide_smem, nullptr));
  if (R.timing) {
    CU(cudaEventRecord(e1, ctx->stream));
    R.scan_events.emplace_back(e0, e1);
  }
  R.launches++;
  R.leafscan_launches++;
  CU(cudaStreamSynchronize(ctx->stream));
  RoundCtl fin;
  CU(cudaMemcpy(&fin, ctx->ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost));
  R.rounds += fin.rounds;
  R.scans += fin.scans;
  return BKT_OK;
}

int search_batch(bkt_ctx* ctx, SearchRun& R) {
  if (R.wide) return wide_batch(ctx, R);
  if (!R.renumber || R.m < (1 << 16)) return search_batch_impl(ctx, R);
  const long long m = R.m;
  TopTreeView top{ctx->split, ctx->h, ctx->d};
  RoundCtl init{};
  init.active = (int)m;
  CU(cudaMemcpyAsync(ctx->ctl, &init, sizeof(RoundCtl), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemsetAsync(ctx->counts, 0, sizeof(int) * ctx->nbuckets, ctx->stream));
  start_kernel<<<R.grid_small, kStartQ, start_smem_bytes(ctx->h, ctx->D), ctx->stream>>>(
      ctx->q, ctx->D, m, R.k, top, ctx->keys, ctx->state, ctx->next, ctx->visits, nullptr, ctx->seq_pos, 0,
      ctx->kthv, ctx->blk_base, ctx->nodes, ctx->sub_w, ctx->qkey, ctx->counts, ctx->pos);
  CU(cudaGetLastError());
  plan_kernel<<<1, kPlanThreads, 0, ctx->stream>>>(ctx->counts, ctx->key_off, ctx->sub_w, ctx->nl * ctx->sub_w,
                                                   ctx->leaf_off, ctx->tile_off, ctx->ctl, ctx->nl, kNT, nullptr, 0,
                                                   nullptr);
  CU(cudaGetLastError());
  scatter_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(nullptr, 1, ctx->pos, ctx->qkey, ctx->key_off, ctx->perm,
                                                         ctx->ctl, ctx->leaf_off, ctx->tile_off, ctx->nl, ctx->sub_w,
                                                         kNT, ctx->tiles, 0);
  CU(cudaGetLastError());
  gather_rows_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(ctx->q, ctx->perm, ctx->D, m, ctx->q_perm);
  CU(cudaGetLastError());
  R.launches += 4;
  float* q_caller = ctx->q;
  ctx->q = ctx->q_perm;
  int rc = search_batch_impl(ctx, R);
  ctx->q = q_caller;
  if (rc != BKT_OK) return rc;
  unpermute_keys_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(ctx->keys, ctx->perm, R.k, m, ctx->keys_tmp);
  unpermute_u32_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(ctx->visits, ctx->perm, m, ctx->visits_tmp);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(ctx->keys, ctx->keys_tmp, sizeof(uint64_t) * m * R.k, cudaMemcpyDeviceToDevice, ctx->stream));
  CU(cudaMemcpyAsync(ctx->visits, ctx->visits_tmp, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, ctx->stream));
  R.launches += 2;
  if (R.seq) {
    remap_seq_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(ctx->seq_dev, ctx->seq_pos, R.seq_cap, ctx->perm);
    CU(cudaGetLastError());
    R.launches++;
  }
  CU(cudaStreamSynchronize(ctx->stream));  // callers read the results from other streams
  return BKT_OK;
}

int search_batch_impl(bkt_ctx* ctx, SearchRun& R) {
  const long long m = R.m;
  TopTreeView top{ctx->split, ctx->h, ctx->d};
  RoundCtl init{};
  init.active = (int)m;
  CU(cudaMemcpyAsync(ctx->ctl, &init, sizeof(RoundCtl), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemsetAsync(ctx->counts, 0, sizeof(int) * ctx->nbuckets, ctx->stream));
  if (R.split) {
    CU(cudaMemsetAsync(ctx->ccnt, 0, (size_t)m * ctx->split_NW, ctx->stream));
    CU(cudaMemsetAsync(ctx->ovflag, 0, sizeof(int) * m, ctx->stream));
  }
  start_kernel<<<R.grid_small, kStartQ, start_smem_bytes(ctx->h, ctx->D), ctx->stream>>>(
      ctx->q, ctx->D, m, R.k, top, ctx->keys, ctx->state, ctx->next,
                                                       ctx->visits, R.seq ? ctx->seq_dev : nullptr, ctx->seq_pos,
                                                       R.seq_cap, ctx->kthv, ctx->blk_base, ctx->nodes, ctx->sub_w,
                                                       ctx->qkey, ctx->counts, ctx->pos);
  CU(cudaGetLastError());
  R.launches++;

  int cur = 0;
  long long round = 0;
  // rounds are launched ahead of the host check; the active count of round r
  // is read back asynchronously and checked kRing-1 rounds later
  cudaEvent_t* ring = ctx->ring_ev;
  const bool ooc = ctx->residency == 1;
  // leaf-level rounds over a small bucket table: plan and scatter fused
  // (plan_scatter_kernel; BKT_FUSED_PS=0 keeps two launches)
  bool fused_ps = !ooc && !R.split && (long long)ctx->nl * ctx->sub_w <= kPsMaxKeys;
  if (const char* e = std::getenv("BKT_FUSED_PS")) fused_ps = fused_ps && std::atoi(e) != 0;
  int* counts_buf[2] = {ctx->counts, ctx->counts_alt};
  const int ps_grid = ctx->sm_count * 2;
  if (fused_ps) CU(cudaMemsetAsync(ctx->counts_alt, 0, sizeof(int) * ctx->nbuckets, ctx->stream));
  if (ooc && R.drain) {
    int rc = ooc_drain(ctx, R);
    if (rc != BKT_OK) return rc;
  }
  for (; !(ooc && R.drain);) {
    // queries with a next leaf -> bucket keys (leaf, block) + counts
    // home visits (round 0) are sub-bucketed per block; later rounds key by leaf only
    const int sw = round == 0 ? ctx->sub_w : 1;
    int* const cnt_now = fused_ps ? counts_buf[round & 1] : ctx->counts;
    if (fused_ps) {
      // plan + scatter in one launch (small bucket tables, leaf-level rounds);
      // with PDL its launch overlaps the previous scan's tail
      int* const cnt_next = counts_buf[(round + 1) & 1];
      const int nkeys_r = ctx->nl * sw;
      RoundCtl* const mir = ctx->d_ctl_mirror + round % kRing;
      const int* const prevw = ctx->work[cur ^ 1];
      const int ident = round == 0 ? 1 : 0;
      int* const outw = ctx->work[cur];
      const int tcap = (int)std::min<long long>(ctx->tiles_cap, INT32_MAX);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(ps_grid);
      cfg.blockDim = dim3(kPsThreads);
      cfg.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = R.pdl ? 1 : 0;
      CU(cudaLaunchKernelEx(&cfg, plan_scatter_kernel, (const int*)cnt_now, cnt_next, ctx->key_off, sw, nkeys_r,
                            ctx->leaf_off, ctx->tile_off, ctx->ctl, ctx->nl, (int)kNT, ctx->hist, (int)kHistCap, mir,
                            prevw, ident, (const int2*)ctx->pos, (const int*)ctx->qkey, outw, ctx->tiles, tcap));
    } else {
      plan_kernel<<<1, kPlanThreads, 0, ctx->stream>>>(ctx->counts, ctx->key_off, sw, ctx->nl * sw,
                                                       ctx->leaf_off, ctx->tile_off, ctx->ctl, ctx->nl, kNT,
                                                       ctx->hist, kHistCap, ctx->d_ctl_mirror + round % kRing);
    }
    CU(cudaGetLastError());
    R.launches++;
    const int slot = (int)(round % kRing);
    if (!(fused_ps && R.pdl)) CU(cudaEventRecord(ring[slot], ctx->stream));
    if (ooc) {
      // out-of-core needs the plan on the host anyway; check synchronously
      CU(cudaEventSynchronize(ring[slot]));
      if (ctx->h_ctl[slot].active == 0) break;
    }
    if (!fused_ps) {
      scatter_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(ctx->work[cur ^ 1], round == 0 ? 1 : 0, ctx->pos,
                                                             ctx->qkey, ctx->key_off, ctx->work[cur],
                                                             ctx->ctl, ctx->leaf_off, ctx->tile_off, ctx->nl, sw, kNT,
                                                             ctx->tiles,
                                                             (int)std::min<long long>(ctx->tiles_cap, INT32_MAX));
      CU(cudaGetLastError());
      R.launches++;
    }
    if (ooc) {
      int rc = ooc_round(ctx, R, cur);
      if (rc != BKT_OK) return rc;
    } else {
      ScanArgs a = make_scan_args(ctx, R, cur);
      if (fused_ps) a.counts = counts_buf[(round + 1) & 1];  // next round's buckets
      R.scan_pdl = fused_ps && R.pdl;
      const bool unfused = R.tc && R.unfused;
      const bool to_split = R.split && round == R.split_from - 1;
      if (unfused || to_split) a.fused = 0;
      int rc = launch_scan(ctx, R, a);
      R.scan_pdl = false;
      if (rc != BKT_OK) return rc;
      if (fused_ps && R.pdl) CU(cudaEventRecord(ring[slot], ctx->stream));  // the plan's mirror is older still
      if (to_split) {
        // this round's rows and kth are final: the split rounds start with
        // its queries' advance (FindLeaf, next-leaf buckets, A rows)
        rc = split_rounds(ctx, R, cur, round + 1);
        if (rc != BKT_OK) return rc;
        break;
      }
      if (unfused) {
        // FindLeaf as its own high-occupancy pass: its dependent top-tree loads
        // then overlap across many warps instead of stalling the scan's epilogue
        findleaf_kernel<<<R.grid_small, 256, start_tree_smem(ctx->h) * 4, ctx->stream>>>(
            ctx->work[cur], ctx->ctl, ctx->q, ctx->D, R.k, TopTreeView{ctx->split, ctx->h, ctx->d}, ctx->keys,
            ctx->state, ctx->next, ctx->visits, fused_ps ? counts_buf[(round + 1) & 1] : ctx->counts, ctx->pos, R.seq ? ctx->seq_dev : nullptr, ctx->seq_pos,
            R.seq_cap);
        CU(cudaGetLastError());
        R.launches++;
      }
    }
    cur ^= 1;
    ++round;
    if (!ooc && round >= kRing - 1) {
      // check the round launched kRing-1 iterations ago
      const int chk = (int)((round - (kRing - 1)) % kRing);
      CU(cudaEventSynchronize(ring[chk]));
      if (ctx->h_ctl[chk].active == 0) break;
      if (R.finish_at >= 0 && ctx->h_ctl[chk].active <= R.finish_at) {
        // the list just scanned (work[cur ^ 1], ctl->active entries) holds
        // every query that is still active; finish them in one launch
        int rc = launch_finisher(ctx, R, ctx->work[cur ^ 1]);
        if (rc != BKT_OK) return rc;
        break;
      }
      if (R.drain_at >= 0 && !R.drain_fired && ctx->h_ctl[chk].active <= R.drain_at) {
        // the list just scanned holds every query that can still change
        snapshot_active<<<R.grid_small, 256, 0, ctx->stream>>>(ctx->work[cur ^ 1], ctx->ctl, ctx->qkey);
        CU(cudaGetLastError());
        R.launches++;
        R.drain_fired = true;
        R.drain_start();
      }
    }
  }
  CU(cudaStreamSynchronize(ctx->stream));
  RoundCtl fin;
  CU(cudaMemcpy(&fin, ctx->ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost));
  R.rounds += fin.rounds;
  R.scans += fin.scans;
  if (R.verbose && R.split)
    std::fprintf(stderr, "split rounds: W %d NW %d tiles %llu chunks %llu items %llu candidates %llu writers %llu "
                 "survivors %llu trips %llu (m %lld)\n",
                 ctx->split_W, ctx->split_NW, fin.sc_tiles, fin.sc_chunks, fin.sc_items, fin.sc_cands, fin.sc_flushes,
                 fin.sc_surv, fin.sc_trips, R.m);
  return BKT_OK;
}

}  // namespace

extern "C" int bkt_search(bkt_ctx* ctx, const float* queries, int64_t m, int32_t k, const bkt_search_opts* opts,
                          uint64_t* out_keys, bkt_stats* stats) {
  if (!ctx) return set_err(nullptr, BKT_EINVAL, "ctx is NULL");
  if (!ctx->has_tree) return set_err(ctx, BKT_ESTATE, "no tree loaded (call bkt_load_tree first)");
  if (m < 0) return set_err(ctx, BKT_EINVAL, "m must be >= 0");
  if (k < 1) return set_err(ctx, BKT_EINVAL, "k must be >= 1, got " + std::to_string(k));
  if (k > ctx->n)
    return set_err(ctx, BKT_EINVAL, "k=" + std::to_string(k) + " exceeds the number of reference points (" +
                                        std::to_string(ctx->n) + ")");
  bkt_search_opts o{};
  o.exact = 1;
  if (opts) o = *opts;
  bkt_stats st{};
  CU(cudaSetDevice(ctx->device));
  if (m == 0) {
    if (stats) *stats = st;
    return BKT_OK;
  }
  SearchRun R;
  R.k = k;
  R.kb = kb_bucket(k);
  R.fma = o.exact == 0;
  R.timing = o.record_timing != 0;
  R.seq = o.seq_log != nullptr && o.seq_cap > 0;
  R.seq_cap = R.seq ? o.seq_cap : 0;
  // auto: the tensor-core filter from d >= 8 (below that the CUDA-core scan is
  // as fast: few pairs per query and a mostly empty K=16 MMA; tools/configs.py cfg4)
  // k > 64 or a general-domain tree: the wide path (one CTA per query, wide_search.cuh)
  R.wide = ctx->wide_only || k > kMaxK;
  if (R.wide && ctx->residency == 1 && !ctx->wide_pts)
    return set_err(ctx, BKT_EINVAL, "the general-domain path (k > 64, d > 32 or h > 16) needs a page-locked "
                                    "structure; this one is spilled to files (bkt_set_spill_dir)");
  if (const char* e = std::getenv("BKT_OOC_ROUNDS")) R.drain = std::atoi(e) == 0;
  // host-resident trees run the tensor-core filter on the drain's resident units
  R.tc = !R.wide && ctx->has_tc && (ctx->residency == 0 || R.drain) && (o.kernel == 2 || (o.kernel == 0 && ctx->d >= 8));
  R.unfused = false;
  if (const char* e = std::getenv("BKT_TC_N")) R.tc_rows = std::atoi(e) == 64 ? 64 : (std::atoi(e) == 256 ? 256 : 128);
  if (const char* e = std::getenv("BKT_TC_CPS")) R.tc_cps = std::atoi(e) == 3 ? 3 : 2;
  if (R.tc_cps == 3 && !std::getenv("BKT_TC_N")) R.tc_rows = 64;
  if (const char* e = std::getenv("BKT_TC_UNFUSED")) R.unfused = std::atoi(e) != 0;
  if (o.kernel == 2 && !R.tc) return set_err(ctx, BKT_EINVAL, "tensor-core kernel requested but unavailable (needs a resident tree and d <= 31)");
  // split rounds (split_scan.cuh): tensor-core path with the 16-column layout
  // (d <= 13), k <= 64 (the rescan's row) and leaves of >= k points (a finite
  // k-th distance after the home visit); BKT_SPLIT=0 keeps the leaf-level rounds
  // Leaves of one window (NW = 1: < 5 chunks of 128 points) gain nothing
  // from routing: config 1 (256-point leaves) runs 6.15 M q/s on leaf-level
  // rounds against 4.06 M with split rounds.
  // One-window leaves (NW = 1) gain only on large batches, where the
  // leaf-level rounds' per-thread top-k and fused FindLeaf cost more than the
  // split rounds' extra kernels: config 5 h = 14 (m = 10M) k = 10 5.5 -> 7.4
  // M q/s, k = 50 1.4 -> 3.3 M; config 1 (m = 65K) 6.2 -> 4.1 M the other way.
  const bool nw_ok = ctx->split_NW > 1 || (ctx->split_NW == 1 && m >= (1 << 20)) ||
                     (std::getenv("BKT_SPLIT_NW1") && ctx->split_NW == 1);
  R.split = R.tc && ctx->residency == 0 && !R.unfused && nw_ok && k <= 64 && ctx->min_leaf >= k && R.tc_rows == 128 && R.tc_cps == 2;
  if (const char* e = std::getenv("BKT_SPLIT")) R.split = R.split && std::atoi(e) != 0;
  // Leaf-level tensor-core rounds over short leaves (no split rounds, KT = 16,
  // <= 1,024 points per leaf): three CTAs per SM with one 128-column
  // accumulator each -- a tile is a few chunks, so more CTAs in flight beat a
  // second accumulator (config 1, 256-point leaves: 6.5 -> 7.2 M q/s; config
  // 4 d = 15, 3,906-point leaves, measured 18.7 -> 16.4 M the other way, and
  // the home-round scan under split rounds 52.5 -> 51.7 M: kept at two;
  // profiles/r2h/cps3_ab.txt)
  if (R.tc && !R.split && ctx->KT == 16 && ctx->n <= 1024ll * ctx->nl && !std::getenv("BKT_TC_CPS") &&
      !std::getenv("BKT_TC_N"))
    R.tc_cps = 3;
  if (const char* e = std::getenv("BKT_SPLIT_FROM")) R.split_from = std::max(1, std::atoi(e));
  // graph mode (opt-in, BKT_GRAPH=1): measured slower than eager launches on
  // config 1 (3.9 vs 5.0 M q/s: its rounds are bound by the kernels' own
  // fixed costs, not by host launch overhead); per-launch leaf-scan timing is
  // not recorded in this mode
  R.graph = R.split && std::getenv("BKT_GRAPH") && std::atoi(std::getenv("BKT_GRAPH")) != 0 &&
            !std::getenv("BKT_SPLIT_DEBUG");
  R.renumber = ctx->residency == 0 && !R.wide && !std::getenv("BKT_EARLY_DRAIN");
  R.verbose = std::getenv("BKT_VERBOSE") != nullptr;
  if (const char* e = std::getenv("BKT_PDL")) R.pdl = std::atoi(e) != 0;
  if (const char* e = std::getenv("BKT_RENUMBER")) R.renumber = R.renumber && std::atoi(e) != 0;
  int rc = BKT_OK;
  if (R.wide) {
    // rows of 2k keys in shared memory while they fit (up to ~190 KB per CTA)
    R.wide_rows_smem = wide_smem_bytes(k, ctx->d, true) <= 190u * 1024u;
    R.wide_smem = wide_smem_bytes(k, ctx->d, R.wide_rows_smem);
    int occ = 0;
    WideArgs dummy{};
    CU(launch_wide(R.fma, 0, nullptr, dummy, R.wide_smem, &occ));
    if (occ < 1) return set_err(ctx, BKT_ECUDA, "wide search kernel cannot be resident");
    R.grid_scan = occ * ctx->sm_count;
    if (!R.wide_rows_smem) {
      const long long need = 2ll * k * R.grid_scan;
      if (ctx->wide_scratch_elems < need) {
        dfree(ctx->wide_scratch);
        ctx->wide_scratch_elems = 0;
        CU(cudaMalloc(&ctx->wide_scratch, sizeof(uint64_t) * need));
        ctx->wide_scratch_elems = need;
      }
    }
  } else if (R.tc) {
    // two CTAs per SM (2 x 256 TMEM columns); the attributes are set by the query
    int occ = 0;
    TcArgs dummy{};
    CU(launch_leafscan_tc(ctx->KT, R.kb, R.fma, 0, nullptr, dummy, &occ, R.tc_rows, R.tc_cps));
    // two CTAs per SM: the variants are sized for it (2 x 256 TMEM columns,
    // shared memory and registers); the occupancy query is only a sanity check
    int per_sm = (ctx->KT == 16) ? R.tc_cps : 2;
    if (R.kb >= 32) {
      // register-heavy top-k variants (leafscan_tc.cuh launch bounds); BKT_TC_BIGK_CTAS
      // for builds with BKT_TC_BIGK_MINB = 2 (experiment)
      per_sm = 1;
      if (const char* e = std::getenv("BKT_TC_BIGK_CTAS")) per_sm = std::max(1, std::min(2, std::atoi(e)));
    }
    if (occ < 1) return set_err(ctx, BKT_ECUDA, "tensor-core leaf kernel cannot be resident");
    if (const char* e = std::getenv("BKT_TC_CTAS")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    if (std::getenv("BKT_VERBOSE")) std::fprintf(stderr, "tc kernel: occupancy %d CTAs/SM, grid %d\n", occ, per_sm * ctx->sm_count);
    R.grid_scan = per_sm * ctx->sm_count;
  } else {
    rc = leafscan_grid(ctx, ctx->D, R.kb, R.fma, &R.grid_scan);
    if (rc != BKT_OK) return rc;
  }
  R.grid_small = ctx->sm_count * 8;
  // Tail finisher (resident structure, d <= 32, k <= 64): the last queries
  // walk the rest of their traversals in one launch instead of one round per
  // leaf (tools/finish_sweep.py, profiles/r1d/finish_sweep*.txt):
  //  * leaves of >= 512 points: one CTA per query once <= 48 per SM remain
  //    (config 2 27.8 -> 28.3 M q/s; config 5 h = 11 +8%; uniform h = 11 +3%);
  //  * deeper trees of short leaves (h >= 12): one warp per query once
  //    <= min(512 per SM, m / 8) remain (config 5 h = 14: 1.27 -> 2.0 M q/s);
  //  * otherwise off (config 1, 256-point leaves: no gain).
  if ((ctx->residency == 0 || R.drain) && ctx->d <= 32 && k <= 64 && !R.wide) {
    if (ctx->n >= 512ll * ctx->nl) {
      R.finish_at = (long long)ctx->sm_count * 48;
      R.finish_cta = true;
    } else if (ctx->h >= 12) {
      R.finish_at = std::min<long long>((long long)ctx->sm_count * 512, m / 8);
    }
  }
  if (const char* e = std::getenv("BKT_FINISH_AT")) R.finish_at = std::atoll(e);
  if (const char* e = std::getenv("BKT_FINISH_CTA")) R.finish_cta = std::atoi(e) != 0;

  if (R.split) ctx->split_capw = split_capw(ctx->split_NW, k);
  // batch size: whatever fits comfortably in free memory (or the caller's choice)
  const long long per_query = 4ll * ctx->D + 4ll * ctx->d + 8ll * k + 4 * 5 + (R.split ? split_bytes_per_query(ctx) : 0) +
                              (R.renumber ? 4ll * ctx->D + 8ll * k + 8 : 0);
  long long batch = o.batch_queries;
  if (batch <= 0) {
    // buffers sized for another per-query footprint (another k or path) are
    // released first, so the estimate below sees them as free
    if (ctx->last_per_query != per_query) {
      CU(cudaStreamSynchronize(ctx->stream));
      free_work(ctx);
    }
    size_t fr = 0, to = 0;
    CU(cudaMemGetInfo(&fr, &to));
    long long usable = (long long)(fr * 0.6) + (long long)ctx->cap_m * per_query;
    batch = std::max<long long>(1 << 16, usable / per_query);
    batch = std::min<long long>(batch, 1ll << 30);
  }
  batch = std::min<long long>(batch, m);
  if (o.batch_queries <= 0 && (!o.queries_on_device || !o.keys_on_device) && !(o.seq_log && o.seq_cap > 0)) {
    // host I/O: split large searches so transfers overlap the search (bkt_search pipeline)
    // measured on B200 (config 2): one batch is best at 10M queries, the extra
    // per-batch tail rounds cost more than the transfers the overlap hides
    long long nio = 1;
    if (const char* e = std::getenv("BKT_IO_BATCHES")) nio = std::max(1, std::atoi(e));
    if (m >= (2ll << 20) && nio > 1) batch = std::min(batch, (m + nio - 1) / nio);
  }
  batch = std::min<long long>(batch, (long long)INT32_MAX / 2);
  ctx->last_per_query = per_query;
  rc = ensure_work(ctx, batch, k);
  if (rc != BKT_OK) return rc;
  if (R.split) {
    rc = ensure_split(ctx, batch);
    if (rc != BKT_OK) return rc;
  }
  if (R.renumber) {
    rc = ensure_perm(ctx, batch, k);
    if (rc != BKT_OK) return rc;
  }
  if (R.seq) {
    if (ctx->seq_dev_cap < R.seq_cap) {
      dfree(ctx->seq_dev);
      CU(cudaMalloc(&ctx->seq_dev, sizeof(int) * 3 * R.seq_cap));
      ctx->seq_dev_cap = R.seq_cap;
    }
    if (m > batch) return set_err(ctx, BKT_EINVAL, "sequence recording requires a single batch");
  }
  CU(cudaMemsetAsync(ctx->pairs, 0, sizeof(unsigned long long), ctx->stream));
  CU(cudaMemsetAsync(ctx->seq_pos, 0, sizeof(unsigned long long), ctx->stream));
  const bool counters = R.tc && std::getenv("BKT_TC_COUNTERS") != nullptr;
  if (counters) {
    if (!ctx->tc_ctr) CU(cudaMalloc(&ctx->tc_ctr, sizeof(unsigned long long) * 16));
    CU(cudaMemsetAsync(ctx->tc_ctr, 0, sizeof(unsigned long long) * 16, ctx->stream));
  }
  R.counters = counters;
  if (counters && std::getenv("BKT_TRACE_ROUNDS")) {
    R.ctr_rounds_cap = kHistCap;
    CU(cudaMalloc(&R.ctr_rounds, sizeof(unsigned long long) * 16 * R.ctr_rounds_cap));
  }

  // Host I/O pipeline: with host-resident queries or results and at least two
  // batches, batch b+1's queries stream in (io set 0, its own host thread and
  // stream) and batch b-1's results stream out (io set 1) while batch b is
  // searched; the two batches alternate between two query/result buffers.
  const bool host_io = !o.queries_on_device || !o.keys_on_device;
  const long long nbatch = (m + batch - 1) / batch;
  const bool overlap = host_io && nbatch >= 2;
  if (overlap) {
    rc = ensure_alt(ctx, batch, k);
    if (rc != BKT_OK) return rc;
  }
  float* qbuf[2] = {ctx->q, ctx->q_alt};
  float* rawbuf[2] = {ctx->q_raw, ctx->q_raw_alt};
  uint64_t* kbuf[2] = {ctx->keys, ctx->keys_alt};
  std::mutex st_mu;
  // queries of batch b -> buffer set `slot` (device queries: an async copy on the engine stream)
  auto load_in = [&](long long b, int slot) -> int {
    const long long b0 = b * batch, bm = std::min(batch, m - b0);
    const float* src = queries + b0 * ctx->d;
    const size_t qbytes = sizeof(float) * bm * ctx->d;
    if (o.queries_on_device) return BKT_OK;  // handled on the engine stream
    CU(cudaSetDevice(ctx->device));
    float* raw = (ctx->D == ctx->d) ? qbuf[slot] : rawbuf[slot];
    auto c0 = std::chrono::steady_clock::now();
    int r = h2d_staged(ctx, ctx->io[0], raw, src, qbytes);
    if (r != BKT_OK) return r;
    std::lock_guard<std::mutex> lk(st_mu);
    st.h2d_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count();
    st.h2d_bytes += qbytes;
    return BKT_OK;
  };
  // page-locked results (bkt_host_alloc) are copied straight from the device
  bool out_pinned = false;
  if (!o.keys_on_device) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, out_keys) == cudaSuccess && pa.type == cudaMemoryTypeHost) out_pinned = true;
    cudaGetLastError();  // pageable memory reports an error on some drivers: clear it
  }
  // results of batch b from buffer set `slot` (device results: async copy on the engine stream)
  auto store_out = [&](long long b, int slot) -> int {
    const long long b0 = b * batch, bm = std::min(batch, m - b0);
    const size_t kbytes = sizeof(uint64_t) * bm * k;
    if (o.keys_on_device) return BKT_OK;
    CU(cudaSetDevice(ctx->device));
    auto c0 = std::chrono::steady_clock::now();
    int r = BKT_OK;
    if (out_pinned) {
      if ((r = ensure_stageset(ctx, ctx->io[1])) != BKT_OK) return r;
      CU(cudaMemcpyAsync(out_keys + b0 * k, kbuf[slot], kbytes, cudaMemcpyDeviceToHost, ctx->io[1].stream));
      CU(cudaStreamSynchronize(ctx->io[1].stream));
    } else {
      r = d2h_staged(ctx, ctx->io[1], out_keys + b0 * k, kbuf[slot], kbytes);
    }
    if (r != BKT_OK) return r;
    std::lock_guard<std::mutex> lk(st_mu);
    st.d2h_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count();
    st.d2h_bytes += kbytes;
    return BKT_OK;
  };

  cudaEvent_t t_all0 = ctx->t_ev[0], t_all1 = ctx->t_ev[1];
  CU(cudaEventRecord(t_all0, ctx->stream));
  if (!o.queries_on_device && (rc = load_in(0, 0)) != BKT_OK) return rc;
  std::thread t_in, t_out;
  int rc_in = BKT_OK, rc_out = BKT_OK;
  auto join_all = [&]() {
    if (t_in.joinable()) t_in.join();
    if (t_out.joinable()) t_out.join();
    ctx->q = qbuf[0];
    ctx->q_raw = rawbuf[0];
    ctx->keys = kbuf[0];
  };
  for (long long b = 0; b < nbatch; ++b) {
    const int slot = overlap ? (int)(b & 1) : 0;
    const long long b0 = b * batch, bm = std::min(batch, m - b0);
    R.m = bm;
    if (overlap && b + 1 < nbatch && !o.queries_on_device)
      t_in = std::thread([&, b, slot]() { rc_in = load_in(b + 1, slot ^ 1); });
    else if (!overlap && b > 0 && !o.queries_on_device && (rc = load_in(b, slot)) != BKT_OK) {
      join_all();
      return rc;
    }
    ctx->q = qbuf[slot];
    ctx->q_raw = rawbuf[slot];
    ctx->keys = kbuf[slot];
    float* raw = (ctx->D == ctx->d) ? ctx->q : ctx->q_raw;
    if (o.queries_on_device) {
      const float* src = queries + b0 * ctx->d;
      if (ctx->D == ctx->d)
        rc = cudaMemcpyAsync(ctx->q, src, sizeof(float) * bm * ctx->d, cudaMemcpyDeviceToDevice, ctx->stream) ==
                     cudaSuccess ? BKT_OK : set_err(ctx, BKT_ECUDA, "query copy failed");
      else raw = const_cast<float*>(src);
      if (rc != BKT_OK) { join_all(); return rc; }
    }
    if (ctx->D != ctx->d) {
      pad_rows_kernel<<<R.grid_small, 256, 0, ctx->stream>>>(raw, ctx->d, ctx->q, ctx->D, bm);
      R.launches++;
    }
    // Early result drain for a single host-result batch: rows of finished
    // queries leave the GPU while the tail rounds run; the rows of queries
    // still active at that point are fixed up afterwards.
    std::thread t_drain;
    int rc_drain = BKT_OK;
    // (opt-in: measured 2% slower end to end on config 2 -- the copy competes with the tail rounds)
    const bool drain = !o.keys_on_device && nbatch == 1 && bm >= (1 << 20) && std::getenv("BKT_EARLY_DRAIN");
    cudaEvent_t drain_ev = ctx->t_ev[2];
    if (drain) {
      R.drain_at = std::max<long long>(1024, bm / 128);
      R.drain_fired = false;
      R.drain_start = [&, slot]() {
        cudaEventRecord(drain_ev, ctx->stream);
        t_drain = std::thread([&, slot]() {
          cudaSetDevice(ctx->device);
          if (cudaEventSynchronize(drain_ev) != cudaSuccess) {
            rc_drain = BKT_ECUDA;
            return;
          }
          rc_drain = store_out(0, slot);
        });
      };
    } else {
      R.drain_at = -1;
    }
    rc = search_batch(ctx, R);
    if (drain) {
      if (t_drain.joinable()) t_drain.join();
      if (rc == BKT_OK) rc = rc_drain;
      if (rc == BKT_OK && R.drain_fired) {
        // fix up the rows that were still active when the drain started
        gather_late<<<R.grid_small, 256, 0, ctx->stream>>>(ctx->keys, k, ctx->qkey, ctx->ctl,
                                                          reinterpret_cast<uint64_t*>(ctx->kthv));
        RoundCtl fin;
        std::vector<int> ids;
        std::vector<uint64_t> rows;
        if (cudaMemcpyAsync(&fin, ctx->ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
            cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
          rc = set_err(ctx, BKT_ECUDA, "early drain fix-up failed");
        } else {
          ids.resize(fin.late_n);
          rows.resize((size_t)fin.late_n * k);
          if ((fin.late_n > 0 &&
               (cudaMemcpyAsync(ids.data(), ctx->qkey, sizeof(int) * fin.late_n, cudaMemcpyDeviceToHost,
                                ctx->stream) != cudaSuccess ||
                cudaMemcpyAsync(rows.data(), ctx->kthv, sizeof(uint64_t) * rows.size(), cudaMemcpyDeviceToHost,
                                ctx->stream) != cudaSuccess)) ||
              cudaStreamSynchronize(ctx->stream) != cudaSuccess)
            rc = set_err(ctx, BKT_ECUDA, "early drain fix-up failed");
          for (int i = 0; i < fin.late_n && rc == BKT_OK; ++i)
            std::memcpy(out_keys + (b0 + ids[i]) * k, rows.data() + (size_t)i * k, sizeof(uint64_t) * k);
        }
      }
      R.drain_at = -1;
      R.drain_start = nullptr;
    }
    if (rc == BKT_OK && o.keys_on_device &&
        cudaMemcpyAsync(out_keys + b0 * k, ctx->keys, sizeof(uint64_t) * bm * k, cudaMemcpyDeviceToDevice,
                        ctx->stream) != cudaSuccess)
      rc = set_err(ctx, BKT_ECUDA, "result copy failed");
    // optional per-query visit counts (the total is counted on the device)
    if (rc == BKT_OK && o.visited_out) {
      static_assert(sizeof(uint32_t) == sizeof(int32_t), "visit counters are 32-bit");
      if (cudaMemcpyAsync(o.visited_out + b0, ctx->visits, sizeof(uint32_t) * bm, cudaMemcpyDeviceToHost,
                          ctx->stream) != cudaSuccess || cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        rc = set_err(ctx, BKT_ECUDA, "visit count copy failed");
    }
    if (t_out.joinable()) t_out.join();  // the previous batch's results are out
    if (rc == BKT_OK) rc = rc_out;
    if (rc != BKT_OK) { join_all(); return rc; }
    if (!o.keys_on_device && !(drain && R.drain_fired)) {
      if (overlap) {
        t_out = std::thread([&, b, slot]() { rc_out = store_out(b, slot); });
      } else if ((rc = store_out(b, slot)) != BKT_OK) {
        join_all();
        return rc;
      }
    }
    if (t_in.joinable()) t_in.join();  // the next batch's queries are in
    if (rc_in != BKT_OK) { join_all(); return rc_in; }
  }
  join_all();
  if (rc_out != BKT_OK) return rc_out;
  CU(cudaEventRecord(t_all1, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, t_all0, t_all1));
  unsigned long long pairs = 0;
  CU(cudaMemcpy(&pairs, ctx->pairs, sizeof(pairs), cudaMemcpyDeviceToHost));
  if (R.seq) {
    unsigned long long cnt = 0;
    CU(cudaMemcpy(&cnt, ctx->seq_pos, sizeof(cnt), cudaMemcpyDeviceToHost));
    long long ncopy = std::min<long long>((long long)cnt, R.seq_cap);
    if (ncopy > 0) CU(cudaMemcpy(o.seq_log, ctx->seq_dev, sizeof(int) * 3 * ncopy, cudaMemcpyDeviceToHost));
    if (o.seq_count_out) *o.seq_count_out = (int64_t)cnt;
  }
  std::vector<float> per_launch;
  for (auto& pr : R.scan_events) {
    float t = 0;
    CU(cudaEventElapsedTime(&t, pr.first, pr.second));
    R.leafscan_ms += t;
    per_launch.push_back(t);
  }
  if (counters) {
    unsigned long long c[16];
    CU(cudaMemcpy(c, ctx->tc_ctr, sizeof(c), cudaMemcpyDeviceToHost));
    std::fprintf(stderr,
                 "tc counters: groups %llu any %llu survivors %llu loop_trips %llu merges %llu tiles %llu "
                 "queries %llu first_visit_survivors %llu pairs %llu inserted %llu warp_chunks %llu warp_needed %llu\n",
                 c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7], pairs, c[8], c[9], c[10]);
  }
  if (std::getenv("BKT_TRACE_ROUNDS") && !per_launch.empty()) {
    // per-round diagnostics of the last batch: active queries and leafscan ms
    std::vector<int> hist(std::min<long long>(kHistCap, per_launch.size()));
    CU(cudaMemcpy(hist.data(), ctx->hist, sizeof(int) * hist.size(), cudaMemcpyDeviceToHost));
    size_t off = per_launch.size() - hist.size();
    std::vector<unsigned long long> cr;
    if (R.ctr_rounds) {
      cr.resize(16 * (size_t)std::min<long long>(R.ctr_rounds_cap, R.leafscan_launches));
      CU(cudaMemcpy(cr.data(), R.ctr_rounds, sizeof(unsigned long long) * cr.size(), cudaMemcpyDeviceToHost));
    }
    for (size_t r = 0; r < hist.size(); ++r) {
      std::fprintf(stderr, "round %zu active %d leafscan_ms %.4f", r, hist[r], per_launch[off + r]);
      if (off == 0 && 16 * (r + 1) <= cr.size()) {
        // counter deltas of this round's launch (same fields as "tc counters")
        const unsigned long long* c1 = &cr[16 * r];
        unsigned long long c0[16] = {};
        if (r > 0) std::copy(&cr[16 * (r - 1)], &cr[16 * r], c0);
        std::fprintf(stderr, " groups %llu any %llu survivors %llu trips %llu merges %llu tiles %llu queries %llu first %llu inserted %llu",
                     c1[0] - c0[0], c1[1] - c0[1], c1[2] - c0[2], c1[3] - c0[3], c1[4] - c0[4], c1[5] - c0[5],
                     c1[6] - c0[6], c1[7] - c0[7], c1[8] - c0[8]);
      }
      std::fprintf(stderr, "\n");
    }
  }
  if (R.ctr_rounds) cudaFree(R.ctr_rounds);
  st.rounds = R.rounds;
  st.leaf_visits = R.scans;
  st.pairs = (int64_t)pairs;
  st.kernel_launches = R.launches;
  st.leafscan_launches = R.leafscan_launches;
  st.leafscan_ms = R.leafscan_ms;
  st.search_ms = ms;
  st.stream_bytes = R.stream_bytes;
  st.stream_copies = R.stream_copies;
  if (stats) *stats = st;
  return BKT_OK;
}

// accessors for the other translation units (misc.cu)
namespace bkt_internal {
int ctx_device(bkt_ctx* c) { return c->device; }
cudaStream_t ctx_stream(bkt_ctx* c) { return c->stream; }
int ctx_fail(bkt_ctx* c, int code, const std::string& msg) { return set_err(c, code, msg); }
SeamSlot* ctx_seam_slot(bkt_ctx* c, int slot) { return slot >= 0 && slot < kSeamSlots ? &c->seam[slot] : nullptr; }
cudaStream_t ctx_copy_stream(bkt_ctx* c) { return c->copy_stream; }
}  // namespace bkt_internal
