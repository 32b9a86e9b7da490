// leafscan_tc.cuh -- ProcessAllBuffers' leaf stage on the 5th-gen tensor cores:
// a TF32 tcgen05 GEMM as a conservative distance filter, exact re-evaluation of
// the survivors on the CUDA cores.  Results are bit-identical to leafscan.cuh
// (and to the reference) in exact mode.
//
// Math.  Tile = (leaf, <=128 queries).  Both sides are centred on the leaf
// centroid c: q' = fl(q - c), p' = fl(p - c), qn = |q'|^2, pn = |p'|^2.  The
// GEMM computes, per (query, point),
//      T = pnc - 2 q'.p'      with pnc = (1 - C) pn folded into B as column d
// (A carries 1.0 in that column), operands pre-rounded to TF32, FP32
// accumulation.  With TF32 rounding (2^-11 relative per operand) and FP32
// accumulation, |T - (pnc - 2 q'.p')| <= 2^-9.4 (qn + pn); the centring and
// the reference's own rounding add < 2^-18 (qn + pn).  Hence
//      D_ref(q, p) <= kth   ==>   T <= kth - (1 - C) qn        (C = 2^-7)
// so every point that can enter the top-k passes the test, and each
// survivor's distance is recomputed with the reference arithmetic
// (core.py:108-122) before it may enter the top-k.  Since the set of
// inserted candidates is unchanged, kth, pruning and the traversal are the
// reference's exactly.
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

// chunk width NR (MMA N) is a template parameter: NR = 64 with 4 TMEM
// accumulators or NR = 128 with 2; both use 256 TMEM columns (two CTAs/SM)
constexpr int kTcEpiWarps = 4;
constexpr int kTcThreads = (kTcEpiWarps + 2) * 32;
constexpr int kTcTmemCols = 256;
constexpr float kTcMargin = 1.0f / 128.0f;    // C

struct TcArgs {
  ScanArgs s;                  // queries, keys, schedule, top tree, stats (quad fields unused)
  const float* B;              // canonical K-major tf32 blocks of every leaf (see engine.cu)
  const uint32_t* ridx;        // original index per padded row (0xFFFFFFFF padding)
  const float* rows;           // padded row-major original coordinates, stride d (padding rows +inf)
  const long long* row_base;   // nl + 1, first padded row of each leaf (multiples of 32)
  const float* centroid;       // nl x KT
  const float* pnmax;          // nl: max over the leaf of |p - c|^2 (upper-bound helper)
  float* kth;                  // per query: current k-th distance (== key_dist(keys[k-1]))
  int d;                       // real dimensionality
  int qstride;                 // row stride of the query block (kernel D of the direct path)
  int spin;                    // 1: MMA/epilogue warps spin on mbarriers instead of suspending
  long long* dbg;              // diagnostics (BKT_TC_DEBUG): per-chunk timestamps of CTA 0
  int dbg_cap;
};

template <int KT, int NR>
struct TcSmem {
  static constexpr int kRows = NR;
  static constexpr int kBufs = kTcTmemCols / NR;
  static constexpr int kStages = (KT <= 16 ? 8 : 4) * 64 / NR;
  static constexpr int kStageB = NR * KT * 4;
  static constexpr int kStageIdx = NR * 4;
  static constexpr int kStageRows = NR * (KT - 1) * 4;  // original coordinates (d <= KT - 1)
  static constexpr int kA = 128 * KT * 4;
  static constexpr int kOffIdx = kStages * kStageB;
  static constexpr int kOffRows = kOffIdx + kStages * kStageIdx;
  static constexpr int kOffA = kOffRows + kStages * kStageRows;
  static constexpr int kOffQs = kOffA + 2 * kA;
  static constexpr int kOffQ = kOffQs + 128 * KT * 4;
  static constexpr int kOffBar = kOffQ + kQueue * 128 * 8;
  static constexpr int kNumBars = 2 * kStages + 2 * kBufs + 4;
  static constexpr int kBytes = kOffBar + kNumBars * 8 + 16 + 1024;  // + alignment slack
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

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

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
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ long long dmin_ll(long long x, long long y) { return x < y ? x : y; }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

struct TcTile {
  int leaf, qbeg, qcnt;
  long long r0, r1;  // padded rows of the leaf
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
  return T;
}

// Exact re-evaluation of one candidate with the reference arithmetic.
template <bool FMA>
__device__ __forceinline__ float exact_dist(const float* __restrict__ qp, const float* __restrict__ pp, int d) {
  float acc = 0.0f;
  for (int j = 0; j < d; ++j) {
    float df = __fsub_rn(__ldg(qp + j), __ldg(pp + j));
    if constexpr (FMA) acc = __fmaf_rn(df, df, acc);
    else acc = __fadd_rn(acc, __fmul_rn(df, df));
  }
  return acc;
}

template <int KT, int KB, bool FMA, int NR>
__global__ void __launch_bounds__(kTcThreads, 2) leafscan_tc_kernel(const TcArgs A) {
  using S = TcSmem<KT, NR>;
  constexpr int kTcRows = NR;
  constexpr int kTcBufs = S::kBufs;
  const ScanArgs& a = A.s;
  extern __shared__ unsigned char smem_raw[];
  // 1 KB alignment for the operand tiles
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  constexpr int kTcStages = S::kStages;
  float* sB = reinterpret_cast<float*>(smem);
  uint32_t* sIdx = reinterpret_cast<uint32_t*>(smem + S::kOffIdx);
  float* sRows = reinterpret_cast<float*>(smem + S::kOffRows);
  float* sA = reinterpret_cast<float*>(smem + S::kOffA);
  float* sQ = reinterpret_cast<float*>(smem + S::kOffQs);  // [j][128] original query coordinates
  uint64_t* s_queue = reinterpret_cast<uint64_t*>(smem + S::kOffQ);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* full = bars;                      // [kTcStages] TMA -> MMA/epilogue
  uint64_t* empty = bars + kTcStages;         // [kTcStages] epilogue -> TMA
  uint64_t* tfull = bars + 2 * kTcStages;     // [kTcBufs] MMA -> epilogue
  uint64_t* tempty = tfull + kTcBufs;         // [kTcBufs] epilogue -> MMA
  uint64_t* afull = tempty + kTcBufs;         // [2] epilogue (A written) -> MMA
  uint64_t* aempty = afull + 2;               // [2] MMA (tile done) -> epilogue
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + S::kNumBars);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
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
    }
    fence_mbar_init();
  }
  if (warp == kTcEpiWarps + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(s_tmem)),
                 "r"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const int tiles_end = a.tile_hi >= 0 ? a.tile_hi : *a.num_tiles;

  if (warp == kTcEpiWarps) {
    // ===== TMA producer =====
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = a.tile_lo + blockIdx.x; t < tiles_end; t += gridDim.x) {
        const TcTile T = tc_tile_info<kTcRows>(A, t);
        for (int c = 0; c < T.nchunks; ++c, ++g) {
          const int s = g % kTcStages;
          const uint32_t use = g / kTcStages;
          const long long tp0 = clock64();
          if (use > 0) mbar_wait(&empty[s], (use - 1) & 1u);
          if (A.dbg && blockIdx.x == 0 && (int)g < A.dbg_cap) {
            A.dbg[8 * g + 0] = tp0;
            A.dbg[8 * g + 1] = clock64();
          }
          const long long row = T.r0 + (long long)c * kTcRows;
          const int nr = (int)dmin_ll(kTcRows, T.r1 - row);
          mbar_arrive_expect_tx(&full[s], nr * (KT * 4 + 4 + A.d * 4));
          bulk_g2s(sB + s * (S::kStageB / 4), A.B + row * KT, nr * KT * 4, &full[s]);
          bulk_g2s(sIdx + s * kTcRows, A.ridx + row, nr * 4, &full[s]);
          bulk_g2s(sRows + s * (S::kStageRows / 4), A.rows + row * A.d, nr * A.d * 4, &full[s]);
        }
      }
    }
  } else if (warp == kTcEpiWarps + 1) {
    // ===== MMA issuer =====
    if (lane == 0) {
      uint32_t g = 0, tt = 0;
      const uint32_t a_base = smem_addr(sA), b_base = smem_addr(sB);
      for (int t = a.tile_lo + blockIdx.x; t < tiles_end; t += gridDim.x, ++tt) {
        const TcTile T = tc_tile_info<kTcRows>(A, t);
        const uint32_t ab = tt & 1u;
        if (A.spin) mbar_wait_spin(&afull[ab], (tt >> 1) & 1u); else mbar_wait(&afull[ab], (tt >> 1) & 1u);
        tc_fence_after();
        for (int c = 0; c < T.nchunks; ++c, ++g) {
          const int s = g % kTcStages;
          const uint32_t b = g % kTcBufs, use = g / kTcBufs;
          if (A.spin) {
            mbar_wait_spin(&full[s], (g / kTcStages) & 1u);
            if (use > 0) mbar_wait_spin(&tempty[b], (use - 1) & 1u);
          } else {
            mbar_wait(&full[s], (g / kTcStages) & 1u);
            if (use > 0) mbar_wait(&tempty[b], (use - 1) & 1u);
          }
          tc_fence_after();
          if (A.dbg && blockIdx.x == 0 && (int)g < A.dbg_cap) A.dbg[8 * g + 2] = clock64();
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
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_addr(&aempty[ab]))
                     : "memory");
      }
    }
  } else {
    // ===== epilogue: one thread per query =====
    uint64_t* qslot = s_queue + tid;
    const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
    const int d = A.d;
    uint32_t g = 0, tt = 0;
    for (int t = a.tile_lo + blockIdx.x; t < tiles_end; t += gridDim.x, ++tt) {
      const TcTile T = tc_tile_info<kTcRows>(A, t);
      const uint32_t ab = tt & 1u;
      const bool valid = tid < T.qcnt;
      const int qi = valid ? __ldg(a.work + T.qbeg + tid) : 0;
      const float* qp = a.q + (long long)qi * A.qstride;
      // The full top-k list is only needed when a candidate enters it; a tile
      // starts from the query's k-th distance alone (kth array) and loads the
      // list lazily at the first merge.
      uint64_t arr[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) arr[j] = 0;
      bool have_list = false;
      float kth = valid ? __ldg(A.kth + qi) : -__int_as_float(0x7f800000);  // invalid rows never take candidates
      // A row: tf32(q - c) in dims < d, 1.0 in column d, zeros after
      if (tt >= 2) mbar_wait(&aempty[ab], ((tt >> 1) - 1) & 1u);
      const float* cen = A.centroid + (long long)T.leaf * KT;
      float qn = 0.0f;
      {
        float* arow = sA + ab * (S::kA / 4);
        // canonical layout: row r -> group r/8 (KT*32 B), chunk k/4 (128 B), row r%8 (16 B)
        float* base = arow + (tid >> 3) * (KT * 8) + (tid & 7) * 4;
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          float v = 0.0f;
          if (j < d) {
            const float qv = valid ? __ldg(qp + j) : 0.0f;
            sQ[j * 128 + tid] = qv;
            float qc = valid ? __fsub_rn(qv, __ldg(cen + j)) : 0.0f;
            qn = __fmaf_rn(qc, qc, qn);
            v = __uint_as_float(tf32_rna(qc));
          } else if (j == d) {
            v = 1.0f;
          }
          base[(j >> 2) * 32 + (j & 3)] = v;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ab]);
      const float qnc = (1.0f - kTcMargin) * qn;
      auto threshold = [&](float kk) {
        // kth - (1 - C) qn, rounded up by a hair so the fp32 subtraction cannot cut a candidate
        float t0 = __fsub_ru(kk, qnc);
        return t0 + 1e-6f * (fabsf(kk) + qnc);
      };
      // kflt: the radius the filter and the queue test against = min(kth, kub)
      // where kub is a proven upper bound of the k-th distance (below)
      float kflt = kth;
      float thr = valid ? threshold(kflt) : kth;
      int cn = 0;
      const float leaf_pnmax = __ldg(A.pnmax + T.leaf);

      // insert this lane's queued candidates; the list is fetched on first use
      auto merge = [&]() {
        if (cn > 0) {
          if (!have_list) {
            const uint64_t* kp = a.keys + (long long)qi * a.k;
#pragma unroll
            for (int j = 0; j < KB; ++j) arr[j] = (j < a.k) ? kp[a.k - 1 - j] : 0ull;
            have_list = true;
          }
          merge_queue<KB>(arr, qslot, cn, kth);
        }
      };

      // filter one 32-column group of TMEM values, then re-evaluate survivors
      auto process = [&](const uint32_t (&v)[32], int gcol, int s, long long row0) {
        // depth-4 tree of 3-input minima (FMNMX3) instead of a 31-long dependent chain
        float m1[11];
#pragma unroll
        for (int i = 0; i < 10; ++i)
          m1[i] = fminf(fminf(__uint_as_float(v[3 * i]), __uint_as_float(v[3 * i + 1])), __uint_as_float(v[3 * i + 2]));
        m1[10] = fminf(__uint_as_float(v[30]), __uint_as_float(v[31]));
        const float m2a = fminf(fminf(m1[0], m1[1]), m1[2]), m2b = fminf(fminf(m1[3], m1[4]), m1[5]);
        const float m2c = fminf(fminf(m1[6], m1[7]), m1[8]), m2d = fminf(m1[9], m1[10]);
        const float mn = fminf(fminf(m2a, m2b), fminf(m2c, m2d));
        if (!__any_sync(0xffffffffu, mn <= thr)) return;
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) mask |= (__uint_as_float(v[j]) <= thr ? 1u : 0u) << j;
        const uint32_t* ids = sIdx + s * kTcRows + gcol;
        const float* prow = sRows + s * (S::kStageRows / 4) + gcol * d;
        while (__any_sync(0xffffffffu, mask != 0)) {
          if (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            const float* pp = prow + j * d;
            float acc = 0.0f;
            for (int jj = 0; jj < d; ++jj) {
              float df = __fsub_rn(sQ[jj * 128 + tid], pp[jj]);
              if constexpr (FMA) acc = __fmaf_rn(df, df, acc);
              else acc = __fadd_rn(acc, __fmul_rn(df, df));
            }
            if (acc <= kflt) qslot[(cn++) * kNT] = pack_key(acc, ids[j]);
          }
          if (__any_sync(0xffffffffu, cn == kQueue)) {
            merge();
            kflt = fminf(kflt, kth);
            if (valid) thr = threshold(kflt);
          }
        }
      };

      for (int c = 0; c < T.nchunks; ++c, ++g) {
        const int s = g % kTcStages;
        const uint32_t b = g % kTcBufs;
        const long long te0 = clock64();
        if (A.spin) {
          mbar_wait_spin(&tfull[b], (g / kTcBufs) & 1u);
          mbar_wait_spin(&full[s], (g / kTcStages) & 1u);
        } else {
          mbar_wait(&tfull[b], (g / kTcBufs) & 1u);
          mbar_wait(&full[s], (g / kTcStages) & 1u);
        }
        tc_fence_after();
        const long long te1 = clock64();
        const long long row0 = T.r0 + (long long)c * kTcRows;
        const int ngrp = (int)dmin_ll(kTcRows, T.r1 - row0) / 32;
        const uint32_t tbase = tmem + lane_base + b * kTcRows;
        // two 32-column groups in flight, one wait (NR = 128: second pair below)
        uint32_t va[32], vb[32];
        tmem_ld32_async(tbase, va);
        if (ngrp > 1) tmem_ld32_async(tbase + 32, vb);
        tmem_wait_ld();
        if constexpr (KB <= 32) {
          if (c == 0 && valid && kth == __int_as_float(0x7f800000)) {
            // No k-th neighbour yet (first leaf): bound it from this chunk's first
            // 32 points.  With U_j = T_j + qn + 2C (qn + pnmax_leaf) >= D_ref(q, p_j)
            // (the filter's error analysis), the KB >= k disjoint column groups
            // j = g (mod KB) each contain a point with D_ref <= min_g U, so the
            // k-th distance is <= max_g min_{j in g} U_j.  Filtering against it
            // drops only points that cannot enter the top-k.
            float gmax = -__int_as_float(0x7f800000);
#pragma unroll
            for (int gi = 0; gi < KB; ++gi) {
              float gm = __uint_as_float(va[gi]);
#pragma unroll
              for (int j = gi + KB; j < 32; j += KB) gm = fminf(gm, __uint_as_float(va[j]));
              gmax = fmaxf(gmax, gm);
            }
            const float kub = __fadd_ru(__fadd_ru(gmax, qn), 2.0f * kTcMargin * (qn + leaf_pnmax) * 1.0001f);
            if (kub < kflt) {
              kflt = kub;
              thr = threshold(kflt);
            }
          }
        }
        process(va, 0, s, row0);
        if (ngrp > 1) process(vb, 32, s, row0);
        if constexpr (NR > 64) {
          if (ngrp > 2) {
            tmem_ld32_async(tbase + 64, va);
            if (ngrp > 3) tmem_ld32_async(tbase + 96, vb);
            tmem_wait_ld();
            process(va, 64, s, row0);
            if (ngrp > 3) process(vb, 96, s, row0);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&tempty[b]);
          mbar_arrive(&empty[s]);
        }
        if (A.dbg && blockIdx.x == 0 && tid == 0 && (int)g < A.dbg_cap) {
          A.dbg[8 * g + 3] = te0;
          A.dbg[8 * g + 4] = te1;
          A.dbg[8 * g + 5] = clock64();
          A.dbg[8 * g + 6] = tt;
        }
      }
      if (__any_sync(0xffffffffu, cn > 0)) merge();

      if (tid == 0 && a.pairs) atomicAdd(a.pairs, (unsigned long long)(__ldg(a.leaf_size + T.leaf)) * T.qcnt);

      if (valid) {
        if (have_list) {
          uint64_t* kp = a.keys + (long long)qi * a.k;
#pragma unroll
          for (int j = 0; j < KB; ++j)
            if (j < a.k) kp[a.k - 1 - j] = arr[j];
          A.kth[qi] = kth;
        }
        if (a.fused) {
          auto qget = [qp](int j) { return __ldg(qp + j); };
          uint32_t st = a.state[qi];
          uint32_t lf = st & 0xFFFFu, pend = st >> 16;
          int nxt = find_next_leaf(a.top, qget, kth, lf, pend);
          a.state[qi] = (pend << 16) | lf;
          a.next[qi] = nxt;
          if (nxt >= 0) {
            uint32_t vv = a.visits[qi] + 1;
            a.visits[qi] = vv;
            log_visit(a, qi, vv, nxt);
            warp_count(a.counts, nxt);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kTcEpiWarps + 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcTmemCols));
  }
}

}  // namespace bkt
