// leafscan_tc.cuh -- ProcessAllBuffers' leaf stage on the 5th-gen tensor cores:
// a TF32 tcgen05 GEMM as a conservative distance filter, exact re-evaluation of
// the survivors on the CUDA cores.  Results are bit-identical to leafscan.cuh
// (and to the reference) in exact mode.
//
// Math.  Tile = (leaf, <=128 queries).  Both sides are centred on the leaf
// centroid c: q' = fl(q - c), p' = fl(p - c), qn = |q'|^2, pn = |p'|^2.  The
// GEMM computes, per (query, point),
//      T = pnc - 2 q'.p'      with pnc = (1 - C) pn folded into B as column d
// (A carries 1.0 in that column), FP32 accumulation.  Error bound: operands
// are pre-rounded to TF32 with round-to-nearest (cvt.rna; unrounded FP32
// operands would be truncated by the tensor core), u = 2^-11 each, so the
// products err by <= 2u sum|a_k b_k| <= 2^-10 (qn + pn) (2|q'||p'| <= qn+pn);
// the pnc column adds u pn; the tensor core's accumulation adds
// <= 2^-21.7 sum|a_k b_k| (measured with pre-rounded operands of mixed
// magnitude, tools/tc_probe.cu, profiles/r1b/tc_accumulation_probe.txt); the
// centring and the reference's own rounding < 2^-18 (qn + pn).  In all
// |T - (pnc - 2 q'.p')| <= 2^-9.4 (qn + pn) < C (qn + pn) for C = 2^-9, hence
//      D_ref(q, p) <= kth   ==>   T <= kth - (1 - C) qn
// so every point that can enter the top-k passes the test, and each
// survivor's distance is recomputed with the reference arithmetic
// (core.py:108-122) before it may enter the top-k.  Since the set of
// inserted candidates is unchanged, kth, pruning and the traversal are the
// reference's exactly.  (C = 2^-7 and 2^-8 were used before; 2^-9 cuts the
// survivors that fail the exact test and gives +11% on config 2.)
//
// Pipeline per CTA (warp-specialised, no CTA barriers in the main loop):
//   warp 4   TMA producer: leaf chunks (128 points x KT tf32 + ids) -> smem ring
//   warp 5   MMA issuer (one thread): tcgen05.mma M=128 N=128 K=KT into one of
//            two TMEM accumulators, tcgen05.commit -> mbarriers
//   warps 0-3 epilogue, one thread per query: writes its A row, reads its TMEM
//            lane (tcgen05.ld 32x32b.x32), filters, re-evaluates survivors,
//            keeps the top-k in registers, runs FindLeaf at the end of the tile.
#pragma once
#include "leafscan.cuh"

namespace bkt {

// Launch shape.  CPS CTAs share an SM (3 for KT = 16, 2 for KT = 32, limited
// by shared memory); each owns 512 / CPS TMEM columns (rounded down to a
// power of two) split into accumulator buffers of NR columns.  A CTA = 4
// epilogue warps (one thread per query row) + a TMA producer warp + an MMA warp.
constexpr int kTcEpiWarps = 4;
constexpr int kTcThreads = (kTcEpiWarps + 2) * 32;
// CPS >= 3: one control warp whose lane 0 runs the TMA producer and the MMA
// issuer as one non-blocking loop (5 warps per CTA, 15 per SM: 4 per
// sub-partition at most, so 128 registers per thread without setmaxnreg)
__host__ __device__ constexpr int tc_ctl_warps(int cps) { return cps >= 3 ? 1 : 2; }
__host__ __device__ constexpr int tc_threads(int cps) { return (kTcEpiWarps + tc_ctl_warps(cps)) * 32; }
#ifndef BKT_TC_MARGIN_LOG2
#define BKT_TC_MARGIN_LOG2 9
#endif
constexpr float kTcMargin = 1.0f / (float)(1 << BKT_TC_MARGIN_LOG2);  // C
constexpr int kBlockRows = 64;               // leaf-internal block (home-visit bucket key), engine.cu
#ifndef BKT_TC_DIAG
#define BKT_TC_DIAG 0  // 1: per-chunk timelines (BKT_TC_DEBUG) and filter counters (BKT_TC_COUNTERS)
#endif
constexpr bool kTcDiag = BKT_TC_DIAG != 0;
#ifndef BKT_TC_EAGER
#define BKT_TC_EAGER 0
#endif
constexpr bool kTcEagerMerge = BKT_TC_EAGER != 0;  // merge queued candidates at the end of every chunk

__host__ __device__ constexpr int tc_tmem_cols(int cps) { return cps >= 3 ? 128 : (cps == 2 ? 256 : 512); }
// shared memory one CTA may use when CPS share an SM (228 KB - 1 KB reserved per CTA)
__host__ __device__ constexpr int tc_smem_per_cta(int cps) { return (228 - cps) * 1024 / cps; }
// registers: CPS x 192 threads share 64K; with setmaxnreg the two control warps
// give theirs to the four epilogue warps
// Registers.  A warp lives in one of the 4 SM sub-partitions (16K registers
// each), so the launch allows 16384 / (32 * ceil(6 CPS / 4)) per thread: 168
// for CPS = 2, 96 for CPS = 3.  With CPS = 3 the two control warps drop to 40
// (setmaxnreg.dec) and the epilogue warps rise to 112 (setmaxnreg.inc): the
// CTA pool (96 x 192) covers 4 x 32 x 112 + 2 x 32 x 40, and a sub-partition
// holding one epilogue warp of each of the 3 CTAs plus up to two control
// warps needs 3 x 112 + 2 x 40 <= 512 registers per lane (a CTA's four
// epilogue warps sit in four different sub-partitions); even four epilogue
// warps and one control warp fit (4 x 112 + 40 <= 512).
constexpr int kTcCtlRegs = 40;
__host__ __device__ constexpr int tc_launch_regs(int cps) {
  return (16384 / (32 * ((cps * (tc_threads(cps) / 32) + 3) / 4))) & ~7;
}
static_assert(tc_launch_regs(3) == 128 && tc_launch_regs(2) == 168, "register budget");

struct TcArgs {
  ScanArgs s;                  // queries, keys, schedule, top tree, stats (quad fields unused)
  const float* B;              // canonical K-major tf32 blocks of every leaf (see engine.cu)
  const uint32_t* ridx;        // original index per padded row (0xFFFFFFFF padding)
  const float* rows;           // padded row-major original coordinates, stride d (padding rows +inf)
  const long long* row_base;   // nl + 1, first padded row of each leaf (multiples of 32)
  const float* centroid;       // nl x KT
  const float* pnmax;          // nl: max over the leaf of |p - c|^2 (upper-bound helper)
  const int* cbase;            // nl + 1: first 128-row chunk of each leaf
  const float* box;            // per 128-row chunk: lo[d], hi[d]
  unsigned long long* need_dbg;  // diagnostics (BKT_TC_SKIPDIAG): per tile, chunks some query needs
  float* kth;                  // per query: current k-th distance (== key_dist(keys[k-1]))
  int d;                       // real dimensionality
  int qstride;                 // row stride of the query block (kernel D of the direct path)
  int spin;                    // bit 0: the MMA warp, bit 1: the epilogue spins on mbarriers instead of suspending
  int tree_smem;               // 1: the top tree's split values are copied to shared memory
  int sub_w;                   // home-round sub-buckets per leaf (tile records carry the sub-bucket)
  int* tile_next;              // round's tile counter (dynamic tile scheduling, CPS < 3), zeroed by plan_kernel
  long long* dbg;              // diagnostics (BKT_TC_DEBUG): per-chunk timestamps of CTA 0
  int dbg_cap;
  unsigned long long* ctr;     // diagnostics (BKT_TC_COUNTERS): filter/survivor counters, see engine.cu
  int pdl;                     // host: launch with programmatic stream serialization (prologue overlaps the previous kernel)
};

// Chunk order of a tile: starting at the chunk of the block its first query
// was routed to (a first visit then bounds its k-th distance from nearby
// points first), wrapping around.
__device__ __forceinline__ int tc_chunk_at(int i, int c0, int nchunks) {
  int c = c0 + i;
  return c >= nchunks ? c - nchunks : c;
}


template <int KT, int NR, int CPS>
struct TcSmem {
  static constexpr int kRows = NR;
  static constexpr int kBufs = tc_tmem_cols(CPS) / NR;
#ifdef BKT_TC_STAGES
  static constexpr int kStages = BKT_TC_STAGES;  // experiments
#else
  static constexpr int kStages = CPS >= 3 ? (NR == 128 ? 2 : 3) : ((KT <= 16 ? 512 : 128) / NR < 2 ? 2 : (KT <= 16 ? 512 : 128) / NR);
#endif
  static constexpr int kStageB = NR * KT * 4;
  static constexpr int kStageIdx = NR * 4;
  static constexpr int kStageRows = NR * (KT - 1) * 4;  // original coordinates (d <= KT - 1)
  static constexpr int kA = 128 * KT * 4;
  static constexpr int kQs = 128 * (KT - 1) * 4;        // one query-coordinate buffer: [j][128]
  static constexpr int kOffIdx = kStages * kStageB;
  static constexpr int kOffRows = kOffIdx + kStages * kStageIdx;
  static constexpr int kOffA = kOffRows + kStages * kStageRows;
  static constexpr int kOffQs = kOffA + 2 * kA;
  static constexpr int kOffCen = kOffQs + 2 * kQs;       // [warp][buf][KT] leaf centroid copies
  static constexpr int kOffQ = kOffCen + kTcEpiWarps * 2 * KT * 4;
  static constexpr int kOffBar = kOffQ + kQueue * 128 * 8;
  static constexpr int kNumBars = 2 * kStages + 2 * kBufs + 6;
  static constexpr int kOffTree = (kOffBar + kNumBars * 8 + 16 + 15) & ~15;
  static constexpr int kBytes = kOffTree + 1024;  // + alignment slack; the top tree (runtime size) follows
  static_assert(kBufs >= 1, "need a TMEM accumulator");
  static_assert(kBytes <= tc_smem_per_cta(CPS), "shared memory exceeds the per-CTA share");
};

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// SWIZZLE_NONE K-major UMMA shared-memory descriptor: core matrix = 8 rows x 16 B,
// rows 16 B apart, K-chunks LBO apart, 8-row groups SBO apart (sm100: version 1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// kind::tf32, D f32, A/B tf32 K-major, M = 128, N = n
__device__ __forceinline__ uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

// tcgen05.ld of 32 consecutive columns of this warp's 32 TMEM lanes (asynchronous:
// the registers are valid after tmem_wait()).
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
// tcgen05.wait::ld with the loaded registers as operands, so the compiler cannot
// hoist a use of v above the wait.
__device__ __forceinline__ void tmem_wait(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                 "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),
                 "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]),
                 "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}

// orders later uses of v after a preceding tmem_wait() (which waits for every
// outstanding tcgen05.ld of the thread)
__device__ __forceinline__ void tmem_touch(uint32_t (&v)[32]) {
  asm volatile(""
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                 "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),
                 "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]),
                 "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}

__device__ __forceinline__ long long dmin_ll(long long x, long long y) { return x < y ? x : y; }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// first chunk of a tile's chunk order: the chunk holding the first block of
// the tile's home sub-bucket (0 when the leaf was not sub-bucketed)
template <int kTcRows>
__device__ __forceinline__ int tc_first_chunk(int sub, long long rows, int nchunks, int sub_w) {
  const int nb = (int)((rows + kBlockRows - 1) / kBlockRows);
  const int blk = sub << home_block_shift(nb, sub_w);
  return (blk / (kTcRows / kBlockRows)) % nchunks;
}

struct TcTile {
  int leaf, qbeg, qcnt, c0;  // c0: first chunk of the tile's chunk order
  long long r0, r1;          // padded rows of the leaf
  int nchunks;
};

template <int kTcRows>
__device__ __forceinline__ TcTile tc_tile_info(const TcArgs& A, int t) {
  const int4 rec = __ldg(A.s.tiles + t);
  TcTile T;
  T.leaf = rec.x;
  T.qbeg = rec.y;
  T.qcnt = rec.z;
  T.r0 = __ldg(A.row_base + rec.x);
  T.r1 = __ldg(A.row_base + rec.x + 1);
  T.nchunks = (int)((T.r1 - T.r0 + kTcRows - 1) / kTcRows);
  T.c0 = tc_first_chunk<kTcRows>(rec.w, T.r1 - T.r0, T.nchunks, A.sub_w);
  return T;
}

// Per-thread inputs of one tile, fetched a tile ahead (see the epilogue).
struct TcTileIn {
  int leaf, qbeg, qcnt, c0blk;
  long long r0, r1;
  int qi;
  bool valid;
  float kth, pnmax;
  uint32_t st, vis;
};

#ifndef BKT_TC_PIPE
#define BKT_TC_PIPE 1
#endif

// 3-input-min tree over 32 TMEM values (depth 4 instead of a 31-long chain)
__device__ __forceinline__ float min32(const uint32_t (&v)[32]) {
  float m1[11];
#pragma unroll
  for (int i = 0; i < 10; ++i)
    m1[i] = fminf(fminf(__uint_as_float(v[3 * i]), __uint_as_float(v[3 * i + 1])), __uint_as_float(v[3 * i + 2]));
  m1[10] = fminf(__uint_as_float(v[30]), __uint_as_float(v[31]));
  const float m2a = fminf(fminf(m1[0], m1[1]), m1[2]), m2b = fminf(fminf(m1[3], m1[4]), m1[5]);
  const float m2c = fminf(fminf(m1[6], m1[7]), m1[8]), m2d = fminf(m1[9], m1[10]);
  return fminf(fminf(m2a, m2b), fminf(m2c, m2d));
}

template <int KT, int KB, bool FMA, int NR, int CPS>
#ifndef BKT_TC_MINB
#define BKT_TC_MINB CPS
#endif
#ifndef BKT_TC_BIGK_MINB
#define BKT_TC_BIGK_MINB 1  // experiments: 2 = two CTAs per SM for KB >= 32 (registers capped, spills)
#endif
// KB >= 32 (k > 16): the register top-k alone needs 64-128 registers, so
// these variants run one CTA per SM with the full register file instead of
// spilling at two (engine.cu launches them one per SM)
__global__ void __launch_bounds__(tc_threads(CPS), (KB >= 32 ? BKT_TC_BIGK_MINB : BKT_TC_MINB)) leafscan_tc_kernel(const TcArgs A) {
  using S = TcSmem<KT, NR, CPS>;
  constexpr int kTcRows = NR;
  constexpr int kTcBufs = S::kBufs;
  constexpr int kTcStages = S::kStages;
  constexpr int kTmemCols = tc_tmem_cols(CPS);
  const ScanArgs& a = A.s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 1 KB alignment for the operand tiles; pointer arithmetic on the shared
  // symbol (not an integer round trip) keeps every access below an LDS/STS
  unsigned char* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  float* sB = reinterpret_cast<float*>(smem);
  uint32_t* sIdx = reinterpret_cast<uint32_t*>(smem + S::kOffIdx);
  float* sRows = reinterpret_cast<float*>(smem + S::kOffRows);
  float* sA = reinterpret_cast<float*>(smem + S::kOffA);
  float* sQ = reinterpret_cast<float*>(smem + S::kOffQs);    // [buf][j][128] original query coordinates
  float* sCen = reinterpret_cast<float*>(smem + S::kOffCen);  // [warp][buf][KT]
  uint64_t* s_queue = reinterpret_cast<uint64_t*>(smem + S::kOffQ);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* full = bars;                      // [kTcStages] TMA -> MMA/epilogue
  uint64_t* empty = bars + kTcStages;         // [kTcStages] epilogue -> TMA
  uint64_t* tfull = bars + 2 * kTcStages;     // [kTcBufs] MMA -> epilogue
  uint64_t* tempty = tfull + kTcBufs;         // [kTcBufs] epilogue -> MMA
  uint64_t* afull = tempty + kTcBufs;         // [2] epilogue (A written) -> MMA
  uint64_t* aempty = afull + 2;               // [2] MMA (tile done) -> epilogue
  uint64_t* tready = aempty + 2;              // [2] epilogue (next tile index published) -> all warps
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + S::kNumBars);
  volatile int* s_tile = reinterpret_cast<volatile int*>(s_tmem + 1);  // [2] published tile indices
  float* sSplit = reinterpret_cast<float*>(smem + S::kOffTree);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nsplit = (1 << a.top.h) - 1;
  auto gtimer = []() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return (long long)v;
  };
  if constexpr (kTcDiag) {
    // load balance of the launch (BKT_TC_DEBUG): per-CTA start / end of the epilogue's tile loop
    if (A.dbg && tid == 0 && blockIdx.x < 1024) A.dbg[16 * A.dbg_cap + blockIdx.x] = gtimer();
  }
  if (A.tree_smem)
    for (int i = tid; i < nsplit; i += tc_threads(CPS)) sSplit[i] = __ldg(a.top.split + i);
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTcEpiWarps);
    }
    for (int b = 0; b < kTcBufs; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kTcEpiWarps);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], kTcEpiWarps);
      mbar_init(&aempty[b], 1);
      mbar_init(&tready[b], 1);
    }
    fence_mbar_init();
  }
  constexpr int kAllocWarp = kTcEpiWarps + tc_ctl_warps(CPS) - 1;
  if (warp == kAllocWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Programmatic dependent launch: everything above (barriers, TMEM, the
  // static top tree) may overlap the previous kernel; every read of its
  // results comes after this wait (a no-op for a normal launch).  The next
  // kernel may be scheduled as soon as this grid's CTAs leave the SMs.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const uint32_t tmem = *s_tmem;
  const int tiles_end = a.tile_hi >= 0 ? a.tile_hi : *a.num_tiles;
  // Tile order.  CPS < 3: dynamic -- the epilogue's thread 0 takes tiles from
  // the round's counter (one atomic a tile ahead, so its latency is hidden)
  // and publishes the j-th tile of this CTA in s_tile[j & 1] (tready[j & 1]);
  // every warp follows the published sequence.  A CTA whose tiles carried
  // little survivor work takes more tiles instead of idling at the end of the
  // launch (static striding measured max/mean CTA time 1.04-1.06).
  // CPS >= 3 (non-blocking control loop): static striding.
  constexpr bool kDynTiles = CPS < 3;
  auto seq_tile = [&](uint32_t j) -> int {
    if constexpr (kDynTiles) {
      mbar_wait(&tready[j & 1u], (j >> 1) & 1u);
      return s_tile[j & 1u];
    } else {
      return a.tile_lo + (int)blockIdx.x + (int)j * (int)gridDim.x;
    }
  };

  // MMA issue of chunk c of tile T into TMEM buffer b from smem stage s (A buffer ab)
  auto issue_mma = [&](const TcTile& T, int c, int s, uint32_t b, uint32_t ab) {
    const uint32_t a_base = smem_addr(sA), b_base = smem_addr(sB);
    const int nr = (int)dmin_ll(kTcRows, T.r1 - (T.r0 + (long long)c * kTcRows));
    const uint32_t idesc = idesc_tf32(nr);
#pragma unroll
    for (int h = 0; h < KT / 8; ++h) {
      const uint64_t da = umma_desc(a_base + ab * S::kA + h * 256, 128, KT * 32);
      const uint64_t db = umma_desc(b_base + s * S::kStageB + h * 256, 128, KT * 32);
      const uint32_t acc = h > 0 ? 1u : 0u;
      asm volatile(
          "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(
              tmem + b * kTcRows),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_addr(&tfull[b]))
                 : "memory");
  };
  // TMA load of chunk c of tile T into stage s
  auto issue_tma = [&](const TcTile& T, int c, int s) {
    const long long row = T.r0 + (long long)c * kTcRows;
    const int nr = (int)dmin_ll(kTcRows, T.r1 - row);
    mbar_arrive_expect_tx(&full[s], nr * (KT * 4 + 4 + A.d * 4));
    bulk_g2s(sB + s * (S::kStageB / 4), A.B + row * KT, nr * KT * 4, &full[s]);
    bulk_g2s(sIdx + s * kTcRows, A.ridx + row, nr * 4, &full[s]);
    bulk_g2s(sRows + s * (S::kStageRows / 4), A.rows + row * A.d, nr * A.d * 4, &full[s]);
  };

  if (tc_ctl_warps(CPS) == 1 && warp == kTcEpiWarps) {
    // ===== one control thread: TMA producer and MMA issuer, never blocking =====
    if (lane == 0) {
      const int t0 = a.tile_lo + (int)blockIdx.x;
      int tp = t0, tm = t0, ip = 0, im = 0;
      uint32_t gp = 0, gm = 0, ttm = 0;
      bool p_done = tp >= tiles_end, m_done = tm >= tiles_end, m_has_a = false;
      TcTile Tp{}, Tm{};
      if (!p_done) Tp = tc_tile_info<kTcRows>(A, tp);
      if (!m_done) Tm = tc_tile_info<kTcRows>(A, tm);
      unsigned idle = 0;
      while (!p_done || !m_done) {
        bool progress = false;
        if (!p_done) {
          const int s = gp % kTcStages;
          const uint32_t use = gp / kTcStages;
          if (use == 0 || mbar_test(&empty[s], (use - 1) & 1u)) {
            issue_tma(Tp, tc_chunk_at(ip, Tp.c0, Tp.nchunks), s);
            ++gp;
            if (++ip == Tp.nchunks) {
              ip = 0;
              tp += gridDim.x;
              if (tp >= tiles_end) p_done = true;
              else Tp = tc_tile_info<kTcRows>(A, tp);
            }
            progress = true;
          }
        }
        if (!m_done) {
          const uint32_t ab = ttm & 1u;
          if (!m_has_a && mbar_test(&afull[ab], (ttm >> 1) & 1u)) {
            tc_fence_after();
            m_has_a = true;
          }
          if (m_has_a) {
            const int s = gm % kTcStages;
            const uint32_t b = gm % kTcBufs, use = gm / kTcBufs;
            if (gm < gp && mbar_test(&full[s], (gm / kTcStages) & 1u) &&
                (use == 0 || mbar_test(&tempty[b], (use - 1) & 1u))) {
              tc_fence_after();
              issue_mma(Tm, tc_chunk_at(im, Tm.c0, Tm.nchunks), s, b, ab);
              ++gm;
              if (++im == Tm.nchunks) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_addr(&aempty[ab]))
                             : "memory");
                im = 0;
                ++ttm;
                m_has_a = false;
                tm += gridDim.x;
                if (tm >= tiles_end) m_done = true;
                else Tm = tc_tile_info<kTcRows>(A, tm);
              }
              progress = true;
            }
          }
        }
        if (progress) idle = 0;
        else if (++idle > 8) __nanosleep(64);
      }
    }
  } else if (warp == kTcEpiWarps) {
    // ===== TMA producer =====
    if (lane == 0) {
      uint32_t g = 0;
      for (uint32_t j = 0;; ++j) {
        const int t = seq_tile(j);
        if (t >= tiles_end) break;
        const TcTile T = tc_tile_info<kTcRows>(A, t);
        for (int i = 0; i < T.nchunks; ++i) {
          const int c = tc_chunk_at(i, T.c0, T.nchunks);
          const int s = g % kTcStages;
          const uint32_t use = g / kTcStages;
          const long long tp0 = kTcDiag ? clock64() : 0;
          if (use > 0) mbar_wait(&empty[s], (use - 1) & 1u);
          if constexpr (kTcDiag) {
            if (A.dbg && blockIdx.x == 0 && (int)g < A.dbg_cap) {
              A.dbg[16 * g + 0] = tp0;
              A.dbg[16 * g + 1] = clock64();
            }
          }
          const long long row = T.r0 + (long long)c * kTcRows;
          const int nr = (int)dmin_ll(kTcRows, T.r1 - row);
          mbar_arrive_expect_tx(&full[s], nr * (KT * 4 + 4 + A.d * 4));
          bulk_g2s(sB + s * (S::kStageB / 4), A.B + row * KT, nr * KT * 4, &full[s]);
          bulk_g2s(sIdx + s * kTcRows, A.ridx + row, nr * 4, &full[s]);
          bulk_g2s(sRows + s * (S::kStageRows / 4), A.rows + row * A.d, nr * A.d * 4, &full[s]);
          ++g;
        }
      }
    }
  } else if (warp == kTcEpiWarps + 1) {
    // ===== MMA issuer =====
    if (lane == 0) {
      uint32_t g = 0, tt = 0;
      const uint32_t a_base = smem_addr(sA), b_base = smem_addr(sB);
      for (;; ++tt) {
        const int t = seq_tile(tt);
        if (t >= tiles_end) break;
        const TcTile T = tc_tile_info<kTcRows>(A, t);
        const uint32_t ab = tt & 1u;
        if (A.spin & 1) mbar_wait_spin(&afull[ab], (tt >> 1) & 1u); else mbar_wait(&afull[ab], (tt >> 1) & 1u);
        tc_fence_after();
        for (int i = 0; i < T.nchunks; ++i) {
          const int c = tc_chunk_at(i, T.c0, T.nchunks);
          const int s = g % kTcStages;
          const uint32_t b = g % kTcBufs, use = g / kTcBufs;
          if (A.spin & 1) {
            mbar_wait_spin(&full[s], (g / kTcStages) & 1u);
            if (use > 0) mbar_wait_spin(&tempty[b], (use - 1) & 1u);
          } else {
            mbar_wait(&full[s], (g / kTcStages) & 1u);
            if (use > 0) mbar_wait(&tempty[b], (use - 1) & 1u);
          }
          tc_fence_after();
          if constexpr (kTcDiag) {
            if (A.dbg && blockIdx.x == 0 && (int)g < A.dbg_cap) A.dbg[16 * g + 2] = clock64();
          }
          const int nr = (int)dmin_ll(kTcRows, T.r1 - (T.r0 + (long long)c * kTcRows));
          const uint32_t idesc = idesc_tf32(nr);
#pragma unroll
          for (int h = 0; h < KT / 8; ++h) {
            // K-chunk pair h: 2 x 16 B chunks of 8 tf32 (LBO 128 B, SBO = 8 rows x KT x 4 B)
            const uint64_t da = umma_desc(a_base + ab * S::kA + h * 256, 128, KT * 32);
            const uint64_t db = umma_desc(b_base + s * S::kStageB + h * 256, 128, KT * 32);
            const uint32_t acc = h > 0 ? 1u : 0u;
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(
                    tmem + b * kTcRows),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_addr(&tfull[b]))
                       : "memory");
          ++g;
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_addr(&aempty[ab]))
                     : "memory");
      }
    }
  } else {
    // ===== epilogue: one thread per query =====
    //
    // A tile's inputs (tile record, query id, coordinates, k-th distance,
    // traversal state) are fetched while the previous tile is being scanned,
    // in four stages spread over its first chunks, and its A operand is
    // written as soon as they arrive; the MMA warp therefore runs from one
    // tile into the next without waiting for this tile's FindLeaf.  The top-k
    // list itself stays in global memory (NeighborBatch.keys layout) and is
    // read-modified-written only when queued candidates are merged.
    uint64_t* qslot = s_queue + tid;
    const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
    const int d = A.d;
    const bool tree_smem = A.tree_smem != 0;
    const int th = a.top.h;
    [[maybe_unused]] unsigned long long c_grp = 0, c_any = 0, c_surv = 0, c_iter = 0, c_merge = 0, c_tile = 0,
                                        c_q = 0, c_first = 0, c_ins = 0;

    TcTileIn nx{};  // the next tile's inputs
    // stage 0: tile record
    auto stage0 = [&](int tn) {
      const int4 rec = __ldg(a.tiles + tn);
      nx.leaf = rec.x;
      nx.qbeg = rec.y;
      nx.qcnt = rec.z;
      nx.c0blk = rec.w;
    };
    // stage 1: leaf rows, query id, leaf radius helper
    auto stage1 = [&]() {
      nx.r0 = __ldg(A.row_base + nx.leaf);
      nx.r1 = __ldg(A.row_base + nx.leaf + 1);
      nx.valid = tid < nx.qcnt;
      nx.qi = nx.valid ? __ldg(a.work + nx.qbeg + tid) : 0;
      nx.pnmax = __ldg(A.pnmax + nx.leaf);
    };
    // stage 2: coordinates -> sQ[nb] (cp.async), centroid -> this warp's sCen[nb], per-query scalars
    auto stage2 = [&](uint32_t nb) {
      float* q_dst = sQ + nb * (S::kQs / 4) + tid;
      if (nx.valid) {
        const float* qp = a.q + (long long)nx.qi * A.qstride;
        for (int j = 0; j < d; ++j) cp_async4(q_dst + j * 128, qp + j);
        nx.kth = __ldg(A.kth + nx.qi);
        nx.st = a.state[nx.qi];
        nx.vis = a.visits[nx.qi];
      } else {
        nx.kth = -__int_as_float(0x7f800000);  // invalid rows never take candidates
        nx.st = 0;
        nx.vis = 0;
      }
      if (lane < KT) cp_async4(sCen + (warp * 2 + nb) * KT + lane, A.centroid + (long long)nx.leaf * KT + lane);
    };
    // stage 3: A row of the next tile: tf32(q - c) in dims < d, 1.0 in column d, zeros after
    auto stage3 = [&](uint32_t nb, uint32_t tn_idx) -> float {
      cp_async_wait_all();
      __syncwarp();
      if (tn_idx >= 2) mbar_wait(&aempty[nb], ((tn_idx >> 1) - 1) & 1u);
      const float* cen = sCen + (warp * 2 + nb) * KT;
      const float* qs = sQ + nb * (S::kQs / 4) + tid;
      float* base = sA + nb * (S::kA / 4) + (tid >> 3) * (KT * 8) + (tid & 7) * 4;
      float qn = 0.0f;
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        float v = 0.0f;
        if (j < d) {
          float qc = nx.valid ? __fsub_rn(qs[j * 128], cen[j]) : 0.0f;
          qn = __fmaf_rn(qc, qc, qn);
          v = __uint_as_float(tf32_rna(qc));
        } else if (j == d) {
          v = 1.0f;
        }
        base[(j >> 2) * 32 + (j & 3)] = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[nb]);
      return qn;
    };

    // The loop starts at a placeholder tile (-1) without chunks whose only job
    // is the first real tile's prefetch, so the prefetch code has one call site.
    int t = a.tile_lo + (int)blockIdx.x - (int)gridDim.x;
    uint32_t g = 0, tt = 0xFFFFFFFFu;
    float nx_qn = 0.0f;
    // dynamic order: the tile after next, taken by thread 0 one tile ahead
    int grabbed = 0;
    if (kDynTiles && tid == 0) grabbed = a.tile_lo + atomicAdd(A.tile_next, 1);
    int tn_next = 0;
    for (; tt == 0xFFFFFFFFu || t < tiles_end; t = tn_next, ++tt) {
      const bool placeholder = tt == 0xFFFFFFFFu;
      // current tile <- prefetched inputs
      const TcTileIn cu = nx;
      const float qn = nx_qn;
      const uint32_t ab = tt & 1u;
      const int nchunks = placeholder ? 0 : (int)((cu.r1 - cu.r0 + kTcRows - 1) / kTcRows);
      const int c0 = placeholder ? 0 : tc_first_chunk<kTcRows>(cu.c0blk, cu.r1 - cu.r0, nchunks, A.sub_w);
      int tn;
      if constexpr (kDynTiles) {
        // publish the next tile (sequence index tt + 1) and take the one after
        const uint32_t jn = tt + 1u;
        if (tid == 0) {
          s_tile[jn & 1u] = grabbed;
          mbar_arrive(&tready[jn & 1u]);
          if (grabbed < tiles_end) grabbed = a.tile_lo + atomicAdd(A.tile_next, 1);
        }
        tn = seq_tile(jn);
      } else {
        tn = t + (int)gridDim.x;
      }
      tn_next = tn;
      const bool has_next = tn < tiles_end;
      int pf = has_next ? 0 : 4;  // next-tile prefetch stage
      auto prefetch_step = [&]() {
        if (pf == 0) stage0(tn);
        else if (pf == 1) stage1();
        else if (pf == 2) stage2(ab ^ 1u);
        else nx_qn = stage3(ab ^ 1u, tt + 1);
        ++pf;
      };

      const bool valid = cu.valid;
      const int qi = cu.qi;
      const float* sq = sQ + ab * (S::kQs / 4) + tid;  // this query's coordinates, stride 128
      float kth = cu.kth;
      const float kth_in = kth;
      const bool first_visit = valid && kth == __int_as_float(0x7f800000);
      if constexpr (kTcDiag) {
        if (A.ctr) { c_tile += 1; c_q += valid ? 1 : 0; }
      }
      const float qnc = (1.0f - kTcMargin) * qn;
      // The error bound needs |q'|^2 in [1e-30, 1e30] (no overflow, no flushed
      // products; the load-time check covers the points).  Rows outside it
      // pass every point to the exact re-evaluation (comparisons below are
      // written !(v > thr) so that NaN from an overflowed dot product passes).
      const bool force = valid && !(qn >= 1e-30f && qn <= 1e30f);
      auto threshold = [&](float kk) {
        if (force) return __int_as_float(0x7f800000);
        // kth - (1 - C) qn, rounded up by a hair so the fp32 subtraction cannot cut a candidate
        float t0 = __fsub_ru(kk, qnc);
        return t0 + 1e-6f * (fabsf(kk) + qnc);
      };
      // kflt: the radius the filter and the queue test against = min(kth, kub)
      // where kub is a proven upper bound of the k-th distance (below)
      float kflt = kth;
      float thr = valid ? threshold(kflt) : kth;
      int cn = 0;

      // insert this lane's queued candidates into its top-k list; the list is
      // read from global memory at the first merge of the tile and kept in
      // registers until the tile ends (CPS >= 3: read-modify-written per merge,
      // the register budget has no room for it)
      constexpr bool kRegTopK = CPS < 3;
      uint64_t arr[kRegTopK ? KB : 1];
#pragma unroll
      for (int j = 0; j < (kRegTopK ? KB : 1); ++j) arr[j] = 0;
      bool have_list = false;
      auto merge = [&]() {
        if (cn > 0) {
          if constexpr (kRegTopK) {
            if (!have_list) {
              const uint64_t* kp = a.keys + (long long)qi * a.k;
#pragma unroll
              for (int j = 0; j < KB; ++j) arr[j] = (j < a.k) ? kp[a.k - 1 - j] : 0ull;
              have_list = true;
            }
            merge_queue<KB>(arr, qslot, cn, kth);
          } else {
            uint64_t* kp = a.keys + (long long)qi * a.k;
            uint64_t tmp[KB];
#pragma unroll
            for (int j = 0; j < KB; ++j) tmp[j] = (j < a.k) ? kp[a.k - 1 - j] : 0ull;
            merge_queue<KB>(tmp, qslot, cn, kth);
#pragma unroll
            for (int j = 0; j < KB; ++j)
              if (j < a.k) kp[a.k - 1 - j] = tmp[j];
          }
        }
      };

      // this query's coordinates for survivor re-evaluation: loaded once per
      // chunk that has survivors (pass 2), not once per survivor
      float qv[KT - 1];
      auto load_qv = [&]() {
#pragma unroll
        for (int jj = 0; jj < KT - 1; ++jj) qv[jj] = jj < d ? sq[jj * 128] : 0.0f;
      };
      // survivors of one 32-column group of TMEM values (the caller has seen a
      // lane's group minimum pass the filter): bitmask, exact re-evaluation
      auto process = [&](const uint32_t (&v)[32], int gcol, int s) {
        if constexpr (kTcDiag) c_grp += 1;
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) mask |= (!(__uint_as_float(v[j]) > thr) ? 1u : 0u) << j;
        if constexpr (kTcDiag) {
          c_any += 1;
          c_surv += __popc(mask);
          if (first_visit) c_first += __popc(mask);
        }
        const uint32_t* ids = sIdx + s * kTcRows + gcol;
        const float* prow = sRows + s * (S::kStageRows / 4) + gcol * d;
        while (__any_sync(0xffffffffu, mask != 0)) {
          if constexpr (kTcDiag) c_iter += 1;
          if (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            const float* pp = prow + j * d;
            // unrolled to KT - 1 >= d with predication: every shared load issues
            // up front, only the (ordered) accumulation chain stays serial
            float pv[KT - 1];
#pragma unroll
            for (int jj = 0; jj < KT - 1; ++jj) pv[jj] = jj < d ? pp[jj] : 0.0f;
            float acc = 0.0f;
#pragma unroll
            for (int jj = 0; jj < KT - 1; ++jj) {
              if (jj < d) {
                float df = __fsub_rn(qv[jj], pv[jj]);
                if constexpr (FMA) acc = __fmaf_rn(df, df, acc);
                else acc = __fadd_rn(acc, __fmul_rn(df, df));
              }
            }
            if (acc <= kflt && ids[j] != kIndexSentinel) {  // padding rows pass only forced rows
              qslot[(cn++) * kNT] = pack_key(acc, ids[j]);
              if constexpr (kTcDiag) c_ins += 1;
            }
          }
          if (__any_sync(0xffffffffu, cn == kQueue)) {
            if constexpr (kTcDiag) c_merge += 1;
            merge();
            kflt = fminf(kflt, kth);
            if (valid) thr = threshold(kflt);
          }
        }
      };

      bool first_chunk = true;
      for (int i = 0; i < nchunks || pf < 4; ++i) {
        if (i >= nchunks) {  // tiles shorter than the prefetch pipeline
          prefetch_step();
          continue;
        }
        const int c = tc_chunk_at(i, c0, nchunks);
        const int s = g % kTcStages;
        const uint32_t b = g % kTcBufs;
        const long long te0 = kTcDiag ? clock64() : 0;
        if constexpr (kTcDiag) {
          if (A.need_dbg) {
            // could this warp / this tile skip the chunk?  box lower bound vs
            // the k-th distance at the tile start (later visits only)
            const float* bx = A.box + (long long)(__ldg(A.cbase + cu.leaf) + c) * 2 * d;
            float lb = 0.0f;
            for (int j = 0; j < d; ++j) {
              const float qj = sq[j * 128];
              const float e = fmaxf(fmaxf(__ldg(bx + j) - qj, qj - __ldg(bx + d + j)), 0.0f);
              lb = __fmaf_rn(e, e, lb);
            }
            const bool need = valid && !(lb * 0.99999f > kth_in);
            const unsigned bal = __ballot_sync(0xffffffffu, need), anyv = __ballot_sync(0xffffffffu, valid);
            if (lane == 0 && anyv && !first_visit) {
              atomicAdd(A.ctr + 9, 1ull);
              if (bal) {
                atomicAdd(A.ctr + 10, 1ull);
                if (c < 64) atomicOr(A.need_dbg + t, 1ull << c);
              }
            }
          }
        }
        // Only the accumulator is waited for here.  The stage's ids and
        // coordinates (TMA -> full[s]) are read by survivor re-evaluation
        // alone, which waits for full[s] itself; most chunks have none.
        // Skipping a phase is safe: the producer cannot refill stage s
        // before this warp's empty[s] arrival below.
        if (A.spin & 2) mbar_wait_spin(&tfull[b], (g / kTcBufs) & 1u);
        else mbar_wait(&tfull[b], (g / kTcBufs) & 1u);
        tc_fence_after();
        const long long te1 = kTcDiag ? clock64() : 0;
        const long long row0 = cu.r0 + (long long)c * kTcRows;
        const int ngrp = (int)dmin_ll(kTcRows, cu.r1 - row0) / 32;
        const uint32_t tbase = tmem + lane_base + b * kTcRows;
        uint32_t va[32], vb[32];
        if constexpr (KB <= 16) {
          if (first_chunk && __any_sync(0xffffffffu, first_visit)) {
            // No k-th neighbour yet (first leaf): bound it from this chunk.  With
            // U_j = T_j + qn + 2C (qn + pnmax_leaf) >= D_ref(q, p_j) (the filter's
            // error analysis), each of the KB >= k disjoint column classes
            // contains a point with D_ref <= min_{j in class} U_j, so the k-th
            // distance is <= max_i min_{j in class i} U_j.  Filtering against it
            // drops only points that cannot enter the top-k.
            float gm[KB];
#pragma unroll
            for (int i = 0; i < KB; ++i) gm[i] = __int_as_float(0x7f800000);
            // classes: column index within its 32-column group, mod KB (a partition
            // of the chunk's columns into KB non-empty classes)
#pragma unroll 1
            for (int gi = 0; gi < ngrp; ++gi) {
              tmem_ld32_async(tbase + 32 * gi, va);
              tmem_wait(va);
#pragma unroll
              for (int j = 0; j < 32; ++j) gm[j % KB] = fminf(gm[j % KB], __uint_as_float(va[j]));
            }
            float gmax = -__int_as_float(0x7f800000);
#pragma unroll
            for (int i = 0; i < KB; ++i) gmax = fmaxf(gmax, gm[i]);
            const float kub = __fadd_ru(__fadd_ru(gmax, qn), 2.0f * kTcMargin * (qn + cu.pnmax) * 1.0001f);
            if (first_visit && !force && kub < kflt) {
              kflt = kub;
              thr = threshold(kflt);
            }
          }
        }
        // Pass 1: the minimum over the whole chunk (two 32-column groups in
        // flight per wait, independent min trees) and ONE vote.  Most chunks end
        // here; a chunk with a candidate is re-read group by group (pass 2).
        first_chunk = false;
        const bool dbg_on = kTcDiag && A.dbg && blockIdx.x == 0 && tid == 0 && (int)g < A.dbg_cap;
        // per-group minima stay in registers: pass 2 re-reads only the groups
        // in which some lane has a candidate (thr only decreases meanwhile)
        constexpr int kGrp = NR / 32;
        float gmn[kGrp];
        const float kInf = __int_as_float(0x7f800000);
#if BKT_TC_PIPE
        // every group loaded unconditionally (columns past a short chunk hold
        // an earlier chunk's values and are masked below), each load issued
        // while the previous group's minimum is computed
        tmem_ld32_async(tbase, va);
        tmem_ld32_async(tbase + 32, vb);
        tmem_wait(va);
        tmem_touch(vb);
        if (dbg_on) A.dbg[16 * g + 7] = clock64();
        gmn[0] = min32(va);
#pragma unroll
        for (int gp = 2; gp < kGrp; gp += 2) {
          tmem_ld32_async(tbase + 32 * gp, va);
          gmn[gp - 1] = min32(vb);
          tmem_ld32_async(tbase + 32 * (gp + 1), vb);
          tmem_wait(va);
          tmem_touch(vb);
          gmn[gp] = min32(va);
        }
        gmn[kGrp - 1] = min32(vb);
#pragma unroll
        for (int gi = 1; gi < kGrp; ++gi)
          if (gi >= ngrp) gmn[gi] = kInf;
#else
        tmem_ld32_async(tbase, va);
        if (ngrp > 1) tmem_ld32_async(tbase + 32, vb);
        tmem_wait(va);
        tmem_touch(vb);
        if (dbg_on) A.dbg[16 * g + 7] = clock64();
        gmn[0] = min32(va);
        gmn[1] = ngrp > 1 ? min32(vb) : kInf;
#pragma unroll
        for (int gp = 2; gp < kGrp; gp += 2) {
          if (gp < ngrp) {
            tmem_ld32_async(tbase + 32 * gp, va);
            if (gp + 1 < ngrp) tmem_ld32_async(tbase + 32 * (gp + 1), vb);
            tmem_wait(va);
            tmem_touch(vb);
            gmn[gp] = min32(va);
            gmn[gp + 1] = gp + 1 < ngrp ? min32(vb) : kInf;
          } else {
            gmn[gp] = kInf;
            gmn[gp + 1] = kInf;
          }
        }
#endif
        float mchunk = gmn[0];
#pragma unroll
        for (int gi = 1; gi < kGrp; ++gi) mchunk = fminf(mchunk, gmn[gi]);
        if (dbg_on) A.dbg[16 * g + 8] = clock64();
        if (__any_sync(0xffffffffu, !(mchunk > thr))) {
          mbar_wait(&full[s], (g / kTcStages) & 1u);
          load_qv();
          if (NR == 64) {
            // both groups are still in registers.  Group 1 only when the chunk
            // has it: with thr = +inf (no k-th distance yet, no bound) the
            // masked minimum (+inf) would pass and its stale columns would be
            // re-evaluated against stale stage rows (fuzz seed 11 case 68)
            if (__any_sync(0xffffffffu, !(gmn[0] > thr))) process(va, 0, s);
            if (ngrp > 1 && __any_sync(0xffffffffu, !(gmn[1] > thr))) process(vb, 32, s);
          } else {
#pragma unroll 1
            for (int gi = 0; gi < ngrp; ++gi) {
              // static-index select (no local-memory array), one process() call site
              float gv = gmn[0];
#pragma unroll
              for (int j = 1; j < kGrp; ++j) gv = gi == j ? gmn[j] : gv;
              if (!__any_sync(0xffffffffu, !(gv > thr))) continue;
              tmem_ld32_async(tbase + 32 * gi, va);
              tmem_wait(va);
              process(va, 32 * gi, s);
            }
          }
          if (kTcEagerMerge && __any_sync(0xffffffffu, cn > 0)) {
            // fold this chunk's candidates in now: a tighter k-th distance for the
            // rest of the leaf means fewer survivors (the queue would otherwise
            // wait until some lane's queue is full)
            merge();
            kflt = fminf(kflt, kth);
            if (valid) thr = threshold(kflt);
          }
          if (dbg_on) A.dbg[16 * g + 9] = clock64();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&tempty[b]);
          mbar_arrive(&empty[s]);
        }
        if constexpr (kTcDiag) {
          if (dbg_on) {
            A.dbg[16 * g + 3] = te0;
            A.dbg[16 * g + 4] = te1;
            A.dbg[16 * g + 5] = clock64();
            A.dbg[16 * g + 6] = tt;
            A.dbg[16 * g + 12] = (long long)c_iter;
            A.dbg[16 * g + 13] = (long long)c_any;
          }
        }
        ++g;
        if (pf < 4) prefetch_step();
      }
      if (placeholder) continue;
      if (__any_sync(0xffffffffu, cn > 0)) merge();

      if (tid == 0 && a.pairs) atomicAdd(a.pairs, (unsigned long long)(__ldg(a.leaf_size + cu.leaf)) * cu.qcnt);

      if (valid) {
        if (kRegTopK && have_list) {
          uint64_t* kp = a.keys + (long long)qi * a.k;
#pragma unroll
          for (int j = 0; j < KB; ++j)
            if (j < a.k) kp[a.k - 1 - j] = arr[j];
        }
        if (kth != kth_in) A.kth[qi] = kth;
        if (a.fused) {
          auto qget = [sq](int j) { return sq[j * 128]; };
          uint32_t lf = cu.st & 0xFFFFu, pend = cu.st >> 16;
          // one FindLeaf body (instruction-cache footprint): the split values are
          // read through a generic pointer, shared memory when the tree fits
          const float* sp = tree_smem ? sSplit : a.top.split;
          const int nxt = find_next_leaf_with(th, d, [sp](uint32_t node) { return sp[node]; }, qget, kth, lf, pend);
          a.state[qi] = (pend << 16) | lf;
          a.next[qi] = nxt;
          int rk = 0;
          if (nxt >= 0) {
            const uint32_t vv = cu.vis + 1;
            a.visits[qi] = vv;
            log_visit(a, qi, vv, nxt);
            rk = warp_reserve(a.counts, nxt);  // next round's bucket (key = leaf) and slot
          }
          a.pos[cu.qbeg + tid] = make_int2(nxt, rk);  // coalesced: read back by position in scatter
        }
      }
    }
    if constexpr (kTcDiag) {
      if (A.dbg && tid == 0 && blockIdx.x < 1024) A.dbg[16 * A.dbg_cap + 1024 + blockIdx.x] = gtimer();
    }
    if constexpr (kTcDiag) {
      if (A.ctr) {
        // per-thread sums reduced over the warp; warp-level counts taken from lane 0
        unsigned long long ts = c_surv, tf = c_first, tq = c_q, ti = c_ins;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ti += __shfl_xor_sync(0xffffffffu, ti, o);
          ts += __shfl_xor_sync(0xffffffffu, ts, o);
          tf += __shfl_xor_sync(0xffffffffu, tf, o);
          tq += __shfl_xor_sync(0xffffffffu, tq, o);
        }
        if (lane == 0) {
          atomicAdd(A.ctr + 0, c_grp);
          atomicAdd(A.ctr + 1, c_any);
          atomicAdd(A.ctr + 2, ts);
          atomicAdd(A.ctr + 3, c_iter);
          atomicAdd(A.ctr + 4, c_merge);
          if (warp == 0) atomicAdd(A.ctr + 5, c_tile);
          atomicAdd(A.ctr + 6, tq);
          atomicAdd(A.ctr + 7, tf);
          atomicAdd(A.ctr + 8, ti);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kAllocWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

}  // namespace bkt
