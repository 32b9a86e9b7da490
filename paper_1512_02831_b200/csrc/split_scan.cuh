// split_scan.cuh -- ProcessAllBuffers' leaf stage for rounds >= 1, split into
// (leaf, window) work items.
//
// Why.  A query that visits a leaf a second time or later (every round after
// the home round) carries a finite k-th distance kth, and only the part of the
// leaf inside its kth-ball can change its top-k.  A leaf of the tensor-core
// layout is ordered as 64-point blocks along a small k-d split tree
// (engine.cu build_leaf_blocks), so consecutive 128-row chunks are compact
// boxes; on config 2 a later visit needs only 26% of a leaf's chunks (box
// lower bound <= kth, tools/skip_sim.c).  A 128-query tile of the leaf-level
// scan needs the union over its queries -- 94-98% of the chunks, measured on
// the B200 (BKT_TC_SKIPDIAG) -- so the skip has to happen per query: every
// query is routed to the windows (W consecutive chunks) it needs, and a tile
// is (leaf, window, <= 128 queries).
//
// Per round (engine.cu split_rounds):
//   plan, scatter : the queries of the round bucketed by leaf (plan_kernel and
//              scatter_kernel of round_kernels.cuh, 1024-query route tiles).
//   route    : per route tile, the leaf's window boxes in shared memory; each
//              query's needed windows (box lower bound <= kth) -> mask, per
//              window counts (shared, then one global atomic per tile and
//              window: the tile's base slot in that key).
//   plan_split : key offsets and 128-item tiles per key (key = leaf * NW + window).
//   place    : items into their key's slice (route tile base + shared rank),
//              and the (leaf, window) tile records.
//   scan     : splitscan_tc_kernel -- the tensor-core filter of leafscan_tc.cuh
//              on each tile's window against each query's kth; the rows of
//              the points that survive go to the (query, window)'s slice of
//              the survivor list (the scan reads only TMEM: its TMA stages
//              carry the B operand alone).
//   rescan   : a query whose survivors exceed a window's slice in one round gets its
//              whole leaf rescanned by one warp (exact), instead of merging.
//   advance  : per query -- re-evaluate its survivors in the reference
//              arithmetic (row-major coordinates of the tensor-core layout)
//              and merge those below the k-th key into the top-k row (the
//              reference's update_rows, core.py:251-262; any order: the result
//              is the best k of the row and the leaf), FindLeaf
//              (buffer_tree.py:330-349) with the new kth, count the next leaf
//              (bucket slot), write the A row of the next visit
//              (tf32(q - c_leaf), 1, .., kth, |q - c|^2).
// A visit none of whose windows can hold a point within kth is a visit with
// no items: the query still goes through advance the next round.
//
// Exactness.  A point can enter the top-k during a visit only if its key is
// below the k-th key at the visit's start, so its reference distance is
// <= kth; such a point lies in a window whose box lower bound (computed in
// f32, relaxed by 1e-5) is <= kth, survives the filter (leafscan_tc.cuh
// header) and is re-evaluated exactly.  The top-k after the visit = best k of
// (row, survivors) = best k of (row, leaf): identical to the reference.
#pragma once
#include "leafscan_tc.cuh"
#include "round_kernels.cuh"

namespace bkt {


#ifndef BKT_ADV_Q2
#define BKT_ADV_Q2 1  // advance_kernel loads query rows as float pairs (even strides; 52.55 -> 52.69 M q/s, r4w)
#endif
#ifndef BKT_SPLIT_MMA_SPIN
#define BKT_SPLIT_MMA_SPIN 0  // experiments: the MMA warp spins on its barriers instead of suspending
#endif
#ifndef BKT_SPLIT_EPI_SPIN
#define BKT_SPLIT_EPI_SPIN 0  // experiments: the epilogue spins on the accumulator-full barrier
#endif
#ifndef BKT_SPLIT_ONEPASS
#define BKT_SPLIT_ONEPASS 1
#endif

constexpr int kSplitKT = 16;     // A row: d coordinates, 1.0 at column d, zeros, kth at KT-2, |q'|^2 at KT-1 (d <= 13)
constexpr int kSplitMaxD = kSplitKT - 3;
#ifndef BKT_SPLIT_CTAS
#define BKT_SPLIT_CTAS 3
#endif
constexpr int kSplitNA = BKT_SPLIT_CTAS >= 4 ? 3 : 4;  // A operand buffers: the producer gathers kAhead = 2 tiles ahead
// CTAs per SM: 2 (two 128-column TMEM accumulators each, 8 TMA stages), 3
// (one accumulator each, 4 stages) or 4 (one accumulator, 3 stages, 3 A
// buffers): with one accumulator a CTA's MMA and epilogue alternate and the
// CTAs interleave on the SM's tensor core (config 2: 2 -> 3 CTAs 48.7 ->
// 52.5 M q/s)
constexpr int kSplitCtas = BKT_SPLIT_CTAS;
constexpr int kSplitAcc = kSplitCtas >= 3 ? 1 : 2;  // TMEM accumulators per CTA
#ifndef BKT_SPLIT_STAGES
#define BKT_SPLIT_STAGES (BKT_SPLIT_CTAS >= 4 ? 3 : (BKT_SPLIT_CTAS == 3 ? 4 : 8))
#endif
constexpr int kSplitStages = BKT_SPLIT_STAGES;  // TMA ring stages (128-row chunks)
constexpr int kSplitThreads = 192;
// Survivor entries (u32 rows of the tensor-core layout) per (query, window)
// slice: 32 for leaves of <= 8 windows, at least 16 for leaves of more (the
// survivors of a visit concentrate in the few windows near the query), and
// about 2k for k > 16 (a larger kth-ball); a query whose survivors overflow a
// slice has its leaf rescanned exactly.  A multiple of 4, so every slice
// starts 16-byte aligned.
__host__ __device__ inline int split_capw(int NW, int k) {
  const int base = NW <= 8 ? 32 : max(16, (256 / NW) & ~3);
  // (k > 16: at most ~8 KB of slices per query)
  return k > 16 ? max(base, min(min(128, (2 * k + 3) & ~3), max(base, (2048 / NW) & ~3))) : base;
}

struct SplitScanArgs {
  const float* arow;         // m x kSplitKT A rows (advance_kernel)
  uint8_t* ccnt;             // m x NW: survivors of each (query, window) this round
  uint32_t* cand;            // m x NW x capw survivor rows (tensor-core layout rows)
  int* ovflag;               // m: the query's survivors overflowed (rescan)
  int* ovf;                  // queries to rescan
  int* novf;
  int NW, capw;
  const int* items;          // this round's items (query ids), grouped by key
  const int4* tiles;         // {leaf, first item, item count, window}
  const int* num_tiles;
  int* tile_next;            // dynamic tile counter (zeroed by plan_split_kernel)
  const float* B;            // tensor-core layout (engine.cu build_tc_layout)
  const long long* row_base;
  int W;                     // chunks per window
  unsigned long long* stats; // diagnostics: tiles, chunks, survivors, writers, items, -, trips (or null)
  long long* dbg;            // BKT_SPLIT_DEBUG: per-event clock64 stamps of CTA 0 (or null)
  int dbg_cap;
};

struct SplitWin {
  long long r0, r1;  // padded rows of the leaf
  int cb, ce;        // the window's chunks [cb, ce)
};

struct SplitSmem {
  static constexpr int KT = kSplitKT;
  static constexpr int kStageB = 128 * KT * 4;
  static constexpr int kA = 128 * KT * 4;
  static constexpr int kOffA = kSplitStages * kStageB;
  static constexpr int kOffQi = kOffA + kSplitNA * kA;
  static constexpr int kOffRec = kOffQi + kSplitNA * 128 * 4;
  static constexpr int kOffWin = kOffRec + kSplitNA * 16;
  static constexpr int kOffBar = kOffWin + kSplitNA * 32;
  static constexpr int kNumBars = 2 * kSplitStages + 4 + 2 * kSplitNA;
  static constexpr int kBytes = kOffBar + kNumBars * 8 + 16 + 1024;  // + tmem slot + alignment slack
  static_assert(sizeof(SplitWin) <= 32, "window record");
  static_assert(kBytes <= tc_smem_per_cta(kSplitCtas), "split scan shared memory exceeds the SM's share");
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}

// element (r, k) of a 128 x KT K-major canonical (SWIZZLE_NONE) operand, in floats
__host__ __device__ __forceinline__ int canon_off(int r, int k, int KT) {
  return (r >> 3) * (KT * 8) + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}

__global__ void __launch_bounds__(kSplitThreads, kSplitCtas) splitscan_tc_kernel(const SplitScanArgs A) {
  using S = SplitSmem;
  constexpr int KT = kSplitKT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  float* sB = reinterpret_cast<float*>(smem);
  float* sA = reinterpret_cast<float*>(smem + S::kOffA);
  int* sQi = reinterpret_cast<int*>(smem + S::kOffQi);
  int4* s_rec = reinterpret_cast<int4*>(smem + S::kOffRec);
  SplitWin* s_win = reinterpret_cast<SplitWin*>(smem + S::kOffWin);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* full = bars;                       // [stages] TMA -> MMA
  uint64_t* empty = bars + kSplitStages;       // [stages] MMA completion (tcgen05.commit) -> TMA
  uint64_t* tfull = bars + 2 * kSplitStages;   // [2] MMA -> epilogue
  uint64_t* tempty = tfull + 2;                // [kSplitAcc] epilogue -> MMA
  uint64_t* afull = tempty + 2;                // [NA] producer (A rows, ids, tile record) -> MMA, epilogue
  uint64_t* aempty = afull + kSplitNA;         // [NA] MMA (tile issued) + 4 epilogue warps -> producer
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + S::kNumBars);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kSplitStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < kSplitAcc; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kTcEpiWarps);
    }
    for (int b = 0; b < kSplitNA; ++b) {
      mbar_init(&afull[b], 32);
      mbar_init(&aempty[b], 1 + kTcEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(s_tmem)),
                 "r"(128 * kSplitAcc));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const int tiles_end = *A.num_tiles;

  if (warp == 4) {
    // ===== producer: tile records, A-row gather (all lanes, cp.async, kAhead
    // tiles in flight), TMA of the window's B chunks (lane 0).  The dependent
    // loads of a tile (its index from the counter, its record, its query ids
    // and leaf rows) are spread over three consecutive issues, so each one's
    // latency overlaps a tile of work. =====
    constexpr int kAhead = 2;
    uint32_t g = 0;
    int t_a = 0;                     // stage a: tile index grabbed
    int4 rec_b;                      // stage b: its record
    int4 rec_c;                      // stage c: record, query ids, window of the tile to issue next
    int qi_c[4];
    long long r0_c = 0, r1_c = 0;
    auto grab = [&]() {
      int t = 0;
      if (lane == 0) t = atomicAdd(A.tile_next, 1);
      return __shfl_sync(0xffffffffu, t, 0);
    };
    auto load_rec = [&](int t) { return t < tiles_end ? __ldg(A.tiles + t) : make_int4(0, 0, -1, 0); };
    auto shift = [&]() {
      rec_c = rec_b;
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const int r = lane + 32 * rr;
        qi_c[rr] = r < rec_c.z ? __ldg(A.items + rec_c.y + r) : -1;
      }
      if (rec_c.z >= 0) {
        r0_c = __ldg(A.row_base + rec_c.x);
        r1_c = __ldg(A.row_base + rec_c.x + 1);
      }
      rec_b = load_rec(t_a);
      t_a = grab();
    };
    bool done_issue = false;
    uint32_t issued = 0;
    auto issue = [&]() {
      if (!done_issue) {
        const uint32_t ab = issued % kSplitNA;
        if (issued >= kSplitNA) mbar_wait(&aempty[ab], ((issued / kSplitNA) - 1) & 1u);
        if (lane == 0) {
          s_rec[ab] = rec_c;
          SplitWin w;
          w.r0 = r0_c;
          w.r1 = r1_c;
          const int nch = (int)((r1_c - r0_c + 127) / 128);
          w.cb = rec_c.w * A.W;
          w.ce = min(nch, w.cb + A.W);
          s_win[ab] = w;
        }
        float* abuf = sA + ab * (S::kA / 4);
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const int r = lane + 32 * rr;
          const int qi = qi_c[rr];
          sQi[ab * 128 + r] = qi;
          if (qi >= 0) {
            const float* src = A.arow + (long long)qi * KT;
            float* dst = abuf + canon_off(r, 0, KT);
#pragma unroll
            for (int kc = 0; kc < KT / 4; ++kc) cp_async16(dst + kc * 32, src + 4 * kc);
          }
        }
        ++issued;
        if (rec_c.z < 0) done_issue = true;
        else shift();
      }
      asm volatile("cp.async.commit_group;" ::: "memory");  // (empty once every tile is issued)
    };
    t_a = grab();
    rec_b = load_rec(t_a);
    t_a = grab();
    shift();
    for (int a0 = 0; a0 < kAhead; ++a0) issue();
    for (uint32_t j = 0;; ++j) {
      issue();  // tile j + kAhead
      asm volatile("cp.async.wait_group %0;" ::"n"(kAhead) : "memory");  // tile j's rows landed
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      const uint32_t ab = j % kSplitNA;
      const int4 rec = s_rec[ab];
      const SplitWin win = s_win[ab];
      mbar_arrive(&afull[ab]);
      if (A.dbg && blockIdx.x == 0 && lane == 0 && (int)j < A.dbg_cap) A.dbg[8 * j + 0] = clock64();
      if (rec.z < 0) break;
      if (lane == 0) {
        if (A.stats) {
          atomicAdd(A.stats + 0, 1ull);
          atomicAdd(A.stats + 1, (unsigned long long)(win.ce - win.cb));
          atomicAdd(A.stats + 4, (unsigned long long)rec.z);
        }
        for (int c = win.cb; c < win.ce; ++c, ++g) {
          const int s = g % kSplitStages;
          const uint32_t use = g / kSplitStages;
          if (use > 0) mbar_wait(&empty[s], (use - 1) & 1u);
          const long long row = win.r0 + (long long)c * 128;
          const int nr = (int)dmin_ll(128, win.r1 - row);
          if (A.dbg && blockIdx.x == 0 && (int)g < A.dbg_cap) A.dbg[8 * A.dbg_cap + 8 * g + 5] = clock64();
          mbar_arrive_expect_tx(&full[s], nr * KT * 4);
          bulk_g2s(sB + s * (S::kStageB / 4), A.B + row * KT, nr * KT * 4, &full[s]);
        }
      }
      __syncwarp();
    }
  } else if (warp == 5) {
    // ===== MMA issuer: per chunk two tf32 MMAs (K = 16) into one of two TMEM
    // accumulators; the commit frees the smem stage (the epilogue reads only
    // TMEM) and then signals the epilogue =====
    if (lane == 0) {
      uint32_t g = 0;
      const uint32_t a_base = smem_addr(sA), b_base = smem_addr(sB);
      for (uint32_t j = 0;; ++j) {
        const uint32_t ab = j % kSplitNA;
        mbar_wait(&afull[ab], (j / kSplitNA) & 1u);
        if (A.dbg && blockIdx.x == 0 && (int)j < A.dbg_cap) A.dbg[8 * j + 7] = clock64();
        const int4 rec = s_rec[ab];
        if (rec.z < 0) break;
        const SplitWin win = s_win[ab];
        tc_fence_after();
        for (int c = win.cb; c < win.ce; ++c, ++g) {
          const int s = g % kSplitStages;
          const uint32_t b = g % kSplitAcc, use = g / kSplitAcc;
#if BKT_SPLIT_MMA_SPIN
          mbar_wait_spin(&full[s], (g / kSplitStages) & 1u);
#else
          mbar_wait(&full[s], (g / kSplitStages) & 1u);
#endif
          if (A.dbg && blockIdx.x == 0 && (int)g < A.dbg_cap) A.dbg[8 * A.dbg_cap + 8 * g + 6] = clock64();
#if BKT_SPLIT_MMA_SPIN
          if (use > 0) mbar_wait_spin(&tempty[b], (use - 1) & 1u);
#else
          if (use > 0) mbar_wait(&tempty[b], (use - 1) & 1u);
#endif
          tc_fence_after();
          const int nr = (int)dmin_ll(128, win.r1 - (win.r0 + (long long)c * 128));
          const uint32_t idesc = idesc_tf32(nr);
#pragma unroll
          for (int h = 0; h < KT / 8; ++h) {
            const uint64_t da = umma_desc(a_base + ab * S::kA + h * 256, 128, KT * 32);
            const uint64_t db = umma_desc(b_base + s * S::kStageB + h * 256, 128, KT * 32);
            const uint32_t acc = h > 0 ? 1u : 0u;
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(
                    tmem + b * 128),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_addr(&empty[s]))
                       : "memory");
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_addr(&tfull[b]))
                       : "memory");
          if (A.dbg && blockIdx.x == 0 && (int)g < A.dbg_cap) A.dbg[8 * A.dbg_cap + 8 * g + 1] = clock64();
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_addr(&aempty[ab]))
                     : "memory");
      }
    }
  } else {
    // ===== epilogue: one thread per item (query) of the tile.  Per chunk the
    // filter's minimum over 128 columns and one vote; the rows of the points
    // that survive are appended to the item's slice (their exact evaluation
    // runs in advance_kernel) =====
    const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
    const int capw = A.capw;
    uint32_t g = 0;
    const bool dbg_on = A.dbg && blockIdx.x == 0 && tid == 0;
    for (uint32_t j = 0;; ++j) {
      const uint32_t ab = j % kSplitNA;
      if (dbg_on && (int)j < A.dbg_cap) A.dbg[8 * j + 5] = clock64();
      mbar_wait(&afull[ab], (j / kSplitNA) & 1u);
      if (dbg_on && (int)j < A.dbg_cap) A.dbg[8 * j + 6] = clock64();
      const int4 rec = s_rec[ab];
      if (rec.z < 0) break;
      const SplitWin win = s_win[ab];
      const bool valid = tid < rec.z;
      const int qi = valid ? sQi[ab * 128 + tid] : 0;
      const float* arow_s = sA + ab * (S::kA / 4);
      const float kth = valid ? arow_s[canon_off(tid, KT - 2, KT)] : -__int_as_float(0x7f800000);
      const float qn = valid ? arow_s[canon_off(tid, KT - 1, KT)] : 0.0f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&aempty[ab]);

      const float qnc = (1.0f - kTcMargin) * qn;
      const bool force = valid && !(qn >= 1e-30f && qn <= 1e30f);
      // kth - (1 - C) qn, rounded up by a hair (leafscan_tc.cuh); forced rows pass everything
      float thr = -__int_as_float(0x7f800000);
      if (valid) thr = force ? __int_as_float(0x7f800000) : __fsub_ru(kth, qnc) + 1e-6f * (fabsf(kth) + qnc);
      int cn = 0;
      // this (query, window)'s survivors go straight to its slice of the list
      uint32_t* cdst = A.cand + ((long long)qi * A.NW + rec.w) * capw;

      for (int c = win.cb; c < win.ce; ++c, ++g) {
        const uint32_t b = g % kSplitAcc;
        const bool dbg_c = dbg_on && (int)g < A.dbg_cap;
        if (dbg_c) A.dbg[8 * A.dbg_cap + 8 * g + 2] = clock64();
#if BKT_SPLIT_EPI_SPIN
        mbar_wait_spin(&tfull[b], (g / kSplitAcc) & 1u);
#else
        mbar_wait(&tfull[b], (g / kSplitAcc) & 1u);
#endif
        if (dbg_c) A.dbg[8 * A.dbg_cap + 8 * g + 3] = clock64();
        tc_fence_after();
        const long long row0 = win.r0 + (long long)c * 128;
        const int ngrp = (int)dmin_ll(128, win.r1 - row0) / 32;
        const uint32_t tbase = tmem + lane_base + b * 128;
        uint32_t va[32], vb[32];
        float gmn[4];
        const float kInf = __int_as_float(0x7f800000);
#if BKT_SPLIT_ONEPASS
        // One pass over the four 32-column groups, each load issued while the
        // previous group's minimum is computed; a group whose minimum passes
        // in some lane has its survivor bitmask built from the registers it
        // is already in, so the accumulator is released before the survivor
        // rows are written and nothing is read from TMEM twice.  Columns past
        // a short chunk (groups >= ngrp) hold an earlier chunk's values and
        // are never tested.
        auto gmask = [&](const uint32_t(&v)[32]) {
          uint32_t mk = 0;
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) mk |= (!(__uint_as_float(v[jj]) > thr) ? 1u : 0u) << jj;
          return valid ? mk : 0u;
        };
        auto passes = [&](float m) { return __any_sync(0xffffffffu, valid && !(m > thr)); };
        uint32_t mk0 = 0, mk1 = 0, mk2 = 0, mk3 = 0;
        tmem_ld32_async(tbase, va);
        tmem_ld32_async(tbase + 32, vb);
        tmem_wait(va);
        tmem_touch(vb);
        if (passes(min32(va))) mk0 = gmask(va);
        tmem_ld32_async(tbase + 64, va);
        if (ngrp > 1 && passes(min32(vb))) mk1 = gmask(vb);
        tmem_ld32_async(tbase + 96, vb);
        tmem_wait(va);
        tmem_touch(vb);
        if (ngrp > 2 && passes(min32(va))) mk2 = gmask(va);
        if (ngrp > 3 && passes(min32(vb))) mk3 = gmask(vb);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
        if (A.stats) {
          unsigned long long sv = __popc(mk0) + __popc(mk1) + __popc(mk2) + __popc(mk3);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
          if (lane == 0) atomicAdd(A.stats + 5, sv);
        }
        const uint32_t rbase = (uint32_t)row0;
        auto emit = [&](uint32_t mk, uint32_t base) {
          for (; mk; mk &= mk - 1) {
            if (cn < capw) cdst[cn] = base + (uint32_t)(__ffs(mk) - 1);
            ++cn;
          }
        };
        emit(mk0, rbase);
        emit(mk1, rbase + 32);
        emit(mk2, rbase + 64);
        emit(mk3, rbase + 96);
        (void)gmn;
#else
        // all four groups unconditionally (columns past a short chunk hold an
        // earlier chunk's values and are masked below), each load issued
        // while the previous group's minimum is computed
        tmem_ld32_async(tbase, va);
        tmem_ld32_async(tbase + 32, vb);
        tmem_wait(va);
        tmem_touch(vb);
        gmn[0] = min32(va);
        tmem_ld32_async(tbase + 64, va);
        gmn[1] = min32(vb);
        tmem_ld32_async(tbase + 96, vb);
        tmem_wait(va);
        tmem_touch(vb);
        gmn[2] = min32(va);
        gmn[3] = min32(vb);
        if (ngrp < 4) {
          gmn[3] = kInf;
          if (ngrp < 3) gmn[2] = kInf;
          if (ngrp < 2) gmn[1] = kInf;
        }
        const float mchunk = fminf(fminf(gmn[0], gmn[1]), fminf(gmn[2], gmn[3]));
        if (__any_sync(0xffffffffu, valid && !(mchunk > thr))) {
          // groups in the order 2, 3, 0, 1: groups 2 and 3 are still in va / vb
#pragma unroll 1
          for (int it = 0; it < 4; ++it) {
            const int gi = it ^ 2;
            if (gi >= ngrp) continue;
            float gv = gmn[0];
#pragma unroll
            for (int jj = 1; jj < 4; ++jj) gv = gi == jj ? gmn[jj] : gv;
            if (!__any_sync(0xffffffffu, valid && !(gv > thr))) continue;
            if (gi < 2) {
              tmem_ld32_async(tbase + 32 * gi, va);
              tmem_wait(va);
            }
            const uint32_t(&v)[32] = gi == 3 ? vb : va;
            uint32_t mask = 0;
            if (valid) {
#pragma unroll
              for (int jj = 0; jj < 32; ++jj) mask |= (!(__uint_as_float(v[jj]) > thr) ? 1u : 0u) << jj;
            }
            if (A.stats) {
              unsigned long long sv = __popc(mask);
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
              if (lane == 0) atomicAdd(A.stats + 5, sv);
            }
            const uint32_t rbase = (uint32_t)(row0 + 32 * gi);
            for (; mask; mask &= mask - 1) {
              if (cn < capw) cdst[cn] = rbase + (uint32_t)(__ffs(mask) - 1);
              ++cn;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
#endif
        if (dbg_c) A.dbg[8 * A.dbg_cap + 8 * g + 4] = clock64();
      }
      if (cn > 0) {
        A.ccnt[(long long)qi * A.NW + rec.w] = (uint8_t)min(cn, 255);
        if (cn > capw && atomicOr(A.ovflag + qi, 1) == 0) A.ovf[atomicAdd(A.novf, 1)] = qi;
        if (A.stats) {
          atomicAdd(A.stats + 2, (unsigned long long)cn);
          atomicAdd(A.stats + 3, 1ull);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128 * kSplitAcc));
  }
}

// ---------------------------------------------------------------------------
// per-query records of the split rounds: the traversal state the round
// kernels read and write per query in one 16-byte record (one sector)
// instead of four scattered arrays; packed when the split rounds start and
// unpacked when they end (the home round, finishers and the result path use
// the arrays)
// ---------------------------------------------------------------------------
__global__ void split_state_pack(long long m, const float* __restrict__ kthv, const uint32_t* __restrict__ state,
                                 const uint32_t* __restrict__ visits, const int* __restrict__ next,
                                 int4* __restrict__ qs) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
    qs[i] = make_int4(__float_as_int(kthv[i]), (int)state[i], (int)visits[i], next[i]);
}
__global__ void split_state_unpack(long long m, const int4* __restrict__ qs, float* __restrict__ kthv,
                                   uint32_t* __restrict__ state, uint32_t* __restrict__ visits,
                                   int* __restrict__ next) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    const int4 r = qs[i];
    kthv[i] = __int_as_float(r.x);
    state[i] = (uint32_t)r.y;
    visits[i] = (uint32_t)r.z;
    next[i] = r.w;
  }
}

// ---------------------------------------------------------------------------
// advance: merge -> FindLeaf -> route (one thread per query of the list)
// ---------------------------------------------------------------------------
struct AdvanceArgs {
  const int* list;           // queries of the round just scanned (length ctl->active)
  RoundCtl* ctl;
  int2* pos;                 // per list position: {next leaf or -1, slot in that leaf's bucket}
  int* counts;               // per leaf: next round's bucket sizes
  const float* q;
  int D;
  int k;
  TopTreeView top;
  uint64_t* keys;
  int4* qs;                  // per query {kth bits, traversal state, visits, next leaf} (split_state)
  uint8_t* ccnt;             // m x NW survivors of the round per window (all zero after the home round)
  const uint32_t* cand;      // m x NW x capw survivor rows of the tensor-core layout
  int NW, capw;
  const float* rows;         // tensor-core layout: row-major original coordinates (exact re-evaluation)
  const uint32_t* ridx;      // tensor-core layout: original index per row (padding: kIndexSentinel)
  int fma;                   // 1: FMA accumulation (exact = 0: the reference's two roundings)
  const float* centroid;     // nl x kSplitKT
  float* arow;               // m x kSplitKT
  int* seq_log;
  unsigned long long* seq_pos;
  long long seq_cap;
};

constexpr int kAdvThreads = 256;
__host__ __device__ inline int advance_smem_bytes(int h, int d) { return (start_tree_smem(h) + d * kAdvThreads) * 4; }

// The packed key of survivor `row` for query coordinates qv, in the
// reference arithmetic (core.py:138-146): acc = sum over j of (q_j - p_j)^2,
// left to right, two roundings per term (exact) or one (FMA).  ~0 for a
// padding row.
__device__ __forceinline__ uint64_t survivor_key(const float (&qv)[kSplitMaxD], int d, const float* __restrict__ rows,
                                                 const uint32_t* __restrict__ ridx, uint32_t row, int fma) {
  const uint32_t id = __ldg(ridx + row);
  const float* pp = rows + (long long)row * d;
  float pv[kSplitMaxD];
#pragma unroll
  for (int j = 0; j < kSplitMaxD; ++j) pv[j] = j < d ? __ldg(pp + j) : 0.0f;
  float acc = 0.0f;
  if (fma) {
#pragma unroll
    for (int j = 0; j < kSplitMaxD; ++j)
      if (j < d) {
        const float df = __fsub_rn(qv[j], pv[j]);
        acc = __fmaf_rn(df, df, acc);
      }
  } else {
#pragma unroll
    for (int j = 0; j < kSplitMaxD; ++j)
      if (j < d) {
        const float df = __fsub_rn(qv[j], pv[j]);
        acc = __fadd_rn(acc, __fmul_rn(df, df));
      }
  }
  return id == kIndexSentinel ? ~0ull : pack_key(acc, id);
}

// survivor_key with the query's coordinates at qp[j * qs] (shared memory)
__device__ __forceinline__ uint64_t survivor_key_s(const float* qp, int qs, int d, const float* __restrict__ rows,
                                                   const uint32_t* __restrict__ ridx, uint32_t row, int fma) {
  float qv[kSplitMaxD];
#pragma unroll
  for (int j = 0; j < kSplitMaxD; ++j) qv[j] = j < d ? qp[j * qs] : 0.0f;
  return survivor_key(qv, d, rows, ridx, row, fma);
}

// A top-k row of k <= 64 keys across a warp (lane j: row[j] in r0, row[32 + j]
// in r1, ascending, ~0 past k).  Inserts cv (below the k-th key) at its rank
// by a one-lane shift; returns the new k-th key.
__device__ __forceinline__ uint64_t warp_row_insert(uint64_t& r0, uint64_t& r1, uint64_t cv, int k, int lane) {
  const uint32_t full = 0xffffffffu;
  const int p = __popc(__ballot_sync(full, r0 < cv)) + __popc(__ballot_sync(full, r1 < cv));
  const uint64_t up0 = __shfl_up_sync(full, r0, 1), up1 = __shfl_up_sync(full, r1, 1);
  const uint64_t last0 = __shfl_sync(full, r0, 31);
  const uint64_t n1v = lane + 32 > p ? (lane == 0 ? last0 : up1) : (lane + 32 == p ? cv : r1);
  r0 = lane > p ? up0 : (lane == p ? cv : r0);
  r1 = n1v;
  return k <= 32 ? __shfl_sync(full, r0, k - 1) : __shfl_sync(full, r1, k - 33);
}

// Warp-cooperative merge of one query's candidate lists into its top-k row
// (k <= 64: lane j holds row[j] and row[32 + j]), used for k > 10 where a
// per-thread register top-k (KB >= 16) spills.  Each candidate below the current k-th
// key is inserted at its rank (two ballots) by a one-lane shift of the row;
// the result is the best k of (row, candidates) -- the reference's
// update_rows (core.py:251-262) in any insertion order.  Returns the new
// k-th key; the counts are zeroed.
__device__ __forceinline__ uint64_t warp_merge_query(uint64_t* __restrict__ row, int k, uint8_t* cc, int NW,
                                                     const uint32_t* __restrict__ cand, int capw, int lane,
                                                     const float (&qv)[kSplitMaxD], int d,
                                                     const float* __restrict__ rows,
                                                     const uint32_t* __restrict__ ridx, int fma) {
  const uint32_t full = 0xffffffffu;
  uint64_t r0 = lane < k ? row[lane] : ~0ull;
  uint64_t r1 = lane + 32 < k ? row[lane + 32] : ~0ull;
  const int n0 = lane < NW ? cc[lane] : 0;
  const int n1 = lane + 32 < NW ? cc[lane + 32] : 0;
  uint64_t kk = k <= 32 ? __shfl_sync(full, r0, k - 1) : __shfl_sync(full, r1, k - 33);
  for (int half = 0; half < 2; ++half) {
    unsigned wm = __ballot_sync(full, (half ? n1 : n0) > 0);
    while (wm) {
      const int src = __ffs(wm) - 1;
      wm &= wm - 1;
      const int w = src + 32 * half;
      const int nc = min(__shfl_sync(full, half ? n1 : n0, src), capw);
      for (int e0 = 0; e0 < nc; e0 += 32) {  // the slice in batches of 32, one survivor per lane
        const uint64_t c =
            e0 + lane < nc ? survivor_key(qv, d, rows, ridx, cand[(long long)w * capw + e0 + lane], fma) : ~0ull;
        unsigned todo = __ballot_sync(full, c < kk);
        while (todo) {
          const int e = __ffs(todo) - 1;
          todo &= todo - 1;
          const uint64_t cv = __shfl_sync(full, c, e);
          if (cv < kk) kk = warp_row_insert(r0, r1, cv, k, lane);  // (kk may have fallen meanwhile)
        }
      }
    }
  }
  if (lane < k) row[lane] = r0;
  if (lane + 32 < k) row[lane + 32] = r1;
  if (lane < NW) cc[lane] = 0;
  if (lane + 32 < NW) cc[lane + 32] = 0;
  return kk;
}

template <int KB>
__global__ void __launch_bounds__(kAdvThreads, 4) advance_kernel(const AdvanceArgs a) {
  extern __shared__ float s_adv[];
  __shared__ uint64_t s_keys[kAdvThreads];  // survivor keys of each warp's evaluation pass
  const int ntree = start_tree_smem(a.top.h);
  float* s_split = s_adv;
  float* myq = s_adv + ntree + threadIdx.x;  // [j][thread]: the thread's query coordinates
  for (int i = threadIdx.x; i < ntree; i += blockDim.x) s_split[i] = __ldg(a.top.split + i);
  __syncthreads();
  const int n = a.ctl->active;
  const int d = a.top.d;
  const int k = a.k;
  const int NW = a.NW;
  const int lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  // whole warps per iteration (the k > 10 merge is cooperative); lane i of
  // the warp owns list position base + i
  for (int base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < n; base += nwarps * 32) {
    const int i = base + lane;
    const bool valid = i < n;
    const int qi = valid ? __ldg(a.list + i) : 0;
    // every per-query input is loaded before the first store (the stores could
    // alias them), so the loads' latencies overlap instead of chaining
    uint8_t* cc = a.ccnt + (long long)qi * NW;
    auto counts8 = [&](int w0) {
      // eight windows' counts per load when the rows are 8-byte aligned
      uint64_t word = 0;
      if ((NW & 7) == 0) {
        word = *reinterpret_cast<const uint64_t*>(cc + w0);
      } else {
        for (int w = w0; w < min(NW, w0 + 8); ++w) word |= (uint64_t)cc[w] << (8 * (w - w0));
      }
      return word;
    };
    const int4 rec = valid ? a.qs[qi] : make_int4(0, 0, 0, 0);  // one 16-byte record: kth, state, visits
    float kth = __int_as_float(rec.x);
    const uint32_t st = (uint32_t)rec.y;
    const uint32_t vis0 = (uint32_t)rec.z;
    const uint64_t word0 = valid ? counts8(0) : 0ull;
    float qv[kSplitMaxD];
    const float* qp = a.q + (long long)qi * a.D;
#if BKT_ADV_Q2
    if ((a.D & 1) == 0) {
      // even row stride: the row in 8-byte pairs (half the load instructions)
      const float2* qp2 = reinterpret_cast<const float2*>(qp);
#pragma unroll
      for (int j = 0; j < (kSplitMaxD + 1) / 2; ++j) {
        float2 v = make_float2(0.0f, 0.0f);
        if (valid && 2 * j < d) v = __ldg(qp2 + j);
        qv[2 * j] = v.x;
        if (2 * j + 1 < kSplitMaxD) qv[2 * j + 1] = (2 * j + 1 < d) ? v.y : 0.0f;
      }
    } else
#endif
    {
#pragma unroll
      for (int j = 0; j < kSplitMaxD; ++j) qv[j] = (valid && j < d) ? __ldg(qp + j) : 0.0f;
    }
#pragma unroll
    for (int j = 0; j < kSplitMaxD; ++j)
      if (j < d) myq[j * kAdvThreads] = qv[j];  // (FindLeaf and the survivor evaluation read it)
    __syncwarp();
    // 1. merge this visit's candidates (one list per window) into the top-k row
    //    (a query the rescan handled has its counts zeroed: its row and kth are final)
    if constexpr (KB >= 16) {
      bool any = word0 != 0ull;
      for (int w0 = 8; w0 < NW && valid && !any; w0 += 8) any = counts8(w0) != 0ull;
      unsigned mq = __ballot_sync(0xffffffffu, any);
      while (mq) {
        const int src = __ffs(mq) - 1;
        mq &= mq - 1;
        const int q = __shfl_sync(0xffffffffu, qi, src);
        float qq[kSplitMaxD];
#pragma unroll
        for (int j = 0; j < kSplitMaxD; ++j) qq[j] = __shfl_sync(0xffffffffu, qv[j], src);
        const uint64_t kk = warp_merge_query(a.keys + (long long)q * k, k, a.ccnt + (long long)q * NW, NW,
                                             a.cand + (long long)q * NW * a.capw, a.capw, lane, qq, d, a.rows,
                                             a.ridx, a.fma);
        if (lane == src) kth = key_dist(kk);
      }
    } else {
      // (k <= 10) The warp's survivors, 32 per pass, one per lane: each lane evaluates
      // one (owner query, row) pair exactly (the owner's coordinates by
      // shuffle), the keys go through shared memory, and every owner inserts
      // its own keys into its register top-k (descending, sentinel-padded:
      // leafscan.cuh merge_queue).
      const uint32_t full = 0xffffffffu;
      int S = 0;
      bool any = false;
      for (int w0 = 0; w0 < NW && valid; w0 += 8) {
        const uint64_t word = w0 == 0 ? word0 : counts8(w0);
        any |= word != 0ull;
#pragma unroll
        for (int b = 0; b < 8; ++b) S += min((int)((word >> (8 * b)) & 0xFF), a.capw);
      }
      int incl = S;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += t;
      }
      const int off = incl - S;
      const int T = __shfl_sync(full, incl, 31);
      if (T > 0) {
        uint64_t arr[KB];
        bool loaded = false;
        uint64_t* row = a.keys + (long long)qi * k;
        uint64_t* s_k = s_keys + (threadIdx.x & ~31);
        for (int e0 = 0; e0 < T; e0 += 32) {
          const int e = e0 + lane;
          // owner: the last lane whose first entry is <= e (offsets are non-decreasing)
          int own = 0;
#pragma unroll
          for (int stp = 16; stp > 0; stp >>= 1)
            if (__shfl_sync(full, off, own + stp) <= e) own += stp;
          int idx = e - __shfl_sync(full, off, own);
          const int oq = __shfl_sync(full, qi, own);
          // the owner's window holding its entry idx (walk its counts)
          int wsel = 0;
          if (e < T) {
            const uint8_t* occ = a.ccnt + (long long)oq * NW;
            for (;; ++wsel) {
              const int c = min((int)occ[wsel], a.capw);
              if (idx < c) break;
              idx -= c;
            }
          }
          // the owner's coordinates: its column of myq
          s_k[lane] = e < T ? survivor_key_s(myq - lane + own, kAdvThreads, d, a.rows, a.ridx,
                                             __ldg(a.cand + ((long long)oq * NW + wsel) * a.capw + idx), a.fma)
                            : ~0ull;
          __syncwarp();
          const int b0 = max(off, e0) - e0, b1 = min(off + S, e0 + 32) - e0;
          if (b0 < b1) {
            if (!loaded) {
#pragma unroll
              for (int j = 0; j < KB; ++j) arr[j] = j < k ? row[k - 1 - j] : 0ull;
              loaded = true;
            }
            for (int x = b0; x < b1; ++x) {
              const uint64_t c = s_k[x];
              if (c < arr[0]) topk_insert<KB>(arr, c);
            }
          }
          __syncwarp();
        }
        if (loaded) {
#pragma unroll
          for (int j = 0; j < KB; ++j)
            if (j < k) row[k - 1 - j] = arr[j];
          kth = key_dist(arr[0]);
        }
        if (any) {  // the counts were read by the evaluating lanes: cleared last
          if ((NW & 7) == 0) {
            for (int w0 = 0; w0 < NW; w0 += 8) *reinterpret_cast<uint64_t*>(cc + w0) = 0ull;
          } else {
            for (int w = 0; w < NW; ++w) cc[w] = 0;
          }
        }
      }
    }
    if (!valid) continue;
    // 2. FindLeaf with the new k-th distance
    auto qget = [myq](int j) { return myq[j * kAdvThreads]; };
    uint32_t lf = st & 0xFFFFu, pend = st >> 16;
    int nxt;
    if (ntree)
      nxt = find_next_leaf_with(a.top.h, d, [s_split](uint32_t node) { return s_split[node]; }, qget, kth, lf, pend);
    else
      nxt = find_next_leaf(a.top, qget, kth, lf, pend);
    int rk = 0;
    const uint32_t vis = nxt >= 0 ? vis0 + 1 : vis0;
    a.qs[qi] = make_int4(__float_as_int(kth), (int)((pend << 16) | lf), (int)vis, nxt);
    if (nxt >= 0) {
      if (a.seq_log) {
        const unsigned long long p = atomicAdd(a.seq_pos, 1ull);
        if ((long long)p < a.seq_cap) {
          a.seq_log[3 * p] = qi; a.seq_log[3 * p + 1] = (int)vis; a.seq_log[3 * p + 2] = nxt;
        }
      }
      rk = warp_reserve(a.counts, nxt);  // next round's bucket (key = leaf) and slot
      // A row of the next visit: tf32(q - c) | 1 | 0.. | kth | |q - c|^2
      const float4* cen4 = reinterpret_cast<const float4*>(a.centroid + (long long)nxt * kSplitKT);
      float cen[kSplitKT];
#pragma unroll
      for (int j = 0; j < kSplitKT / 4; ++j) {
        const float4 c4 = __ldg(cen4 + j);
        cen[4 * j] = c4.x; cen[4 * j + 1] = c4.y; cen[4 * j + 2] = c4.z; cen[4 * j + 3] = c4.w;
      }
      float r[kSplitKT];
      float qn = 0.0f;
#pragma unroll
      for (int j = 0; j < kSplitKT; ++j) {
        float v = 0.0f;
        if (j < d) {
          const float qc = __fsub_rn(myq[j * kAdvThreads], cen[j]);
          qn = __fmaf_rn(qc, qc, qn);
          v = __uint_as_float(tf32_rna(qc));
        } else if (j == d) {
          v = 1.0f;
        }
        r[j] = v;
      }
      r[kSplitKT - 2] = kth;
      r[kSplitKT - 1] = qn;
      float4* dst = reinterpret_cast<float4*>(a.arow + (long long)qi * kSplitKT);
#pragma unroll
      for (int j = 0; j < kSplitKT / 4; ++j) dst[j] = make_float4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
    }
    a.pos[i] = make_int2(nxt, rk);
  }
}

// ---------------------------------------------------------------------------
// route: windows per query, one route tile = (leaf, <= kRouteQ queries of its bucket)
// ---------------------------------------------------------------------------
constexpr int kRouteQ = 1024;
constexpr int kRouteThreads = 256;
constexpr int kMaxWin = 64;

struct RouteArgs {
  const int* work;           // this round's queries, bucketed by leaf
  const int4* rtiles;        // route tiles {leaf, first, count, -}
  const RoundCtl* ctl;       // num_tiles = route tiles
  const int4* qs;            // split_state records (kth in .x)
  const float* q;
  int D;
  int d;
  int NW;
  const int* win_base;
  const float* win_box;
  const int* leaf_size;
  unsigned long long* qmask; // per work-list position
  int* counts;               // per key
  int* cbase;                // per route tile x NW: the tile's first slot in each key
  const int* key_off;        // (place) per key
  const int* stoff;          // (place) split tiles per key
  int nkeys;
  int* items;
  int4* stiles;
  int stiles_cap;
  unsigned long long* pairs;
};

// pass 1: masks, per-key counts, each route tile's base slot per window; pairs
__global__ void __launch_bounds__(kRouteThreads) route_kernel(const RouteArgs a) {
  __shared__ __align__(16) uint64_t s_box[kMaxWin * kSplitMaxD];  // per window, per dimension f32x2 {lo, -hi}
  __shared__ int s_cnt[kMaxWin];
  const int nt = a.ctl->num_tiles;
  const int d = a.d;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const int4 rt = __ldg(a.rtiles + t);
    const int leaf = rt.x;
    const int w0 = __ldg(a.win_base + leaf), nw = __ldg(a.win_base + leaf + 1) - w0;
    __syncthreads();  // previous tile's shared state consumed
    const uint64_t* gbox = reinterpret_cast<const uint64_t*>(a.win_box) + (long long)w0 * d;
    for (int e = threadIdx.x; e < nw * d; e += blockDim.x) s_box[e] = __ldg(gbox + e);
    for (int e = threadIdx.x; e < kMaxWin; e += blockDim.x) s_cnt[e] = 0;
    __syncthreads();
    // per-window counts of this lane's windows (lane w: windows w and w + 32),
    // summed over the warp's iterations, then one shared atomic per warp and window
    int cnt0 = 0, cnt1 = 0;
    const int lane = threadIdx.x & 31;
    const bool pairs2 = (d & 1) == 0 && (a.D & 1) == 0;  // 16-byte box pairs, 8-byte query pairs
    // whole warps per iteration (the per-window counts below are kept by lane w)
    for (int r0 = threadIdx.x & ~31; r0 < rt.z; r0 += blockDim.x) {
      const int r = r0 + lane;
      const bool valid = r < rt.z;
      const int p = rt.y + (valid ? r : 0);
      const int qi = __ldg(a.work + p);
      const float kth = valid ? __int_as_float(__ldg(reinterpret_cast<const int*>(a.qs + qi))) : -1.0f;
      // {q_j, -q_j}: one packed subtraction per dimension gives {lo - q, q - hi}
      uint64_t qq[kSplitMaxD];
      const float* qp = a.q + (long long)qi * a.D;
      if (pairs2) {
#pragma unroll
        for (int j = 0; j < kSplitMaxD / 2; ++j) {
          const float2 v = 2 * j < d ? __ldg(reinterpret_cast<const float2*>(qp) + j) : make_float2(0.0f, 0.0f);
          qq[2 * j] = ((uint64_t)__float_as_uint(-v.x) << 32) | __float_as_uint(v.x);
          qq[2 * j + 1] = ((uint64_t)__float_as_uint(-v.y) << 32) | __float_as_uint(v.y);
        }
        qq[kSplitMaxD - 1] = 0;
      } else {
#pragma unroll
        for (int j = 0; j < kSplitMaxD; ++j) {
          const float v = j < d ? __ldg(qp + j) : 0.0f;
          qq[j] = ((uint64_t)__float_as_uint(-v) << 32) | __float_as_uint(v);
        }
      }
      unsigned long long mask = 0;
      for (int w = 0; w < nw; ++w) {
        // box lower bound in f32, relaxed by 1e-5: never above the reference distance
        const uint64_t* bx = s_box + w * d;
        float lb = 0.0f;
        if (pairs2) {
#pragma unroll
          for (int j = 0; j < kSplitMaxD / 2; ++j) {
            if (2 * j < d) {
              const ulonglong2 b2 = reinterpret_cast<const ulonglong2*>(bx)[j];
              const uint64_t df0 = f2_sub(b2.x, qq[2 * j]), df1 = f2_sub(b2.y, qq[2 * j + 1]);
              const float e0 = fmaxf(fmaxf(f2_lo(df0), f2_hi(df0)), 0.0f);
              const float e1 = fmaxf(fmaxf(f2_lo(df1), f2_hi(df1)), 0.0f);
              lb = __fmaf_rn(e0, e0, lb);
              lb = __fmaf_rn(e1, e1, lb);
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < kSplitMaxD; ++j) {
            if (j < d) {
              const uint64_t df = f2_sub(bx[j], qq[j]);
              const float e = fmaxf(fmaxf(f2_lo(df), f2_hi(df)), 0.0f);
              lb = __fmaf_rn(e, e, lb);
            }
          }
        }
        if (!(lb * 0.99999f > kth)) mask |= 1ull << w;
      }
      if (valid) a.qmask[p] = mask;
      for (int w = 0; w < nw; ++w) {
        const int c = __popc(__ballot_sync(0xffffffffu, (mask >> w) & 1ull));
        if (lane == (w & 31)) {
          if (w < 32) cnt0 += c; else cnt1 += c;
        }
      }
    }
    if (lane < nw && cnt0) atomicAdd(&s_cnt[lane], cnt0);
    if (lane + 32 < nw && cnt1) atomicAdd(&s_cnt[lane + 32], cnt1);
    __syncthreads();
    for (int w = threadIdx.x; w < nw; w += blockDim.x) {
      const int c = s_cnt[w];
      a.cbase[(long long)t * a.NW + w] = c ? atomicAdd(a.counts + leaf * a.NW + w, c) : 0;
    }
    if (threadIdx.x == 0 && a.pairs) atomicAdd(a.pairs, (unsigned long long)__ldg(a.leaf_size + leaf) * rt.z);
  }
}

// pass 2 (after plan_split): items into their key's slice; split tile records
__global__ void __launch_bounds__(kRouteThreads) place_kernel(const RouteArgs a) {
  __shared__ int s_cnt[kMaxWin];
  __shared__ int s_base[kMaxWin];
  const int nt = a.ctl->num_tiles;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const int4 rt = __ldg(a.rtiles + t);
    const int leaf = rt.x;
    const int nw = __ldg(a.win_base + leaf + 1) - __ldg(a.win_base + leaf);
    __syncthreads();
    for (int w = threadIdx.x; w < nw; w += blockDim.x) {
      s_cnt[w] = 0;
      s_base[w] = __ldg(a.key_off + leaf * a.NW + w) + __ldg(a.cbase + (long long)t * a.NW + w);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < rt.z; r += blockDim.x) {
      const int p = rt.y + r;
      const int qi = __ldg(a.work + p);
      unsigned long long m = __ldg(a.qmask + p);
      while (m) {
        const int w = __ffsll((long long)m) - 1;
        m &= m - 1;
        a.items[s_base[w] + atomicAdd(&s_cnt[w], 1)] = qi;
      }
    }
  }
  // (leaf, window) tile records {leaf, first item, count, window}
  const int ns = min(a.ctl->stiles, a.stiles_cap);
  const int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ns; t += stride) {
    int lo = 0, hi = a.nkeys;  // last key with stoff[key] <= t (the key holding tile t)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(a.stoff + mid) <= t) lo = mid; else hi = mid;
    }
    const int p = __ldg(a.key_off + lo) + (t - __ldg(a.stoff + lo)) * kNT;
    a.stiles[t] = make_int4(lo / a.NW, p, min(kNT, __ldg(a.key_off + lo + 1) - p), lo % a.NW);
  }
}

// counts -> key offsets and 128-item tiles per key (one CTA)
__global__ void __launch_bounds__(kPlanThreads) plan_split_kernel(int* __restrict__ counts, int* __restrict__ key_off,
                                                                  int nkeys, int* __restrict__ toff, RoundCtl* ctl,
                                                                  int tile_q) {
  const int per = (nkeys + kPlanThreads - 1) / kPlanThreads;
  const int lo = min(nkeys, (int)threadIdx.x * per), hi = min(nkeys, lo + per);
  long long sc = 0, st = 0;
  for (int e = lo; e < hi; ++e) {
    const int c = counts[e];
    sc += c;
    st += (c + tile_q - 1) / tile_q;
  }
  long long ec = sc, et = st, tot_c, tot_t;
  block_scan2(ec, et, tot_c, tot_t);
  for (int e = lo; e < hi; ++e) {
    const int c = counts[e];
    key_off[e] = (int)ec;
    toff[e] = (int)et;
    ec += c;
    et += (c + tile_q - 1) / tile_q;
    counts[e] = 0;
  }
  if (threadIdx.x == 0) {
    key_off[nkeys] = (int)tot_c;
    toff[nkeys] = (int)tot_t;
    ctl->novf = 0;
    ctl->stiles = (int)tot_t;
    ctl->tile_next = 0;
    ctl->items = (int)tot_c;
  }
}

// A query whose candidates overflowed its list: one warp rescans the whole
// leaf of this round's visit (reference arithmetic over the quad layout, as
// finish_kernel) and merges every point below the k-th key.
template <bool FMA>
__global__ void __launch_bounds__(kFinishWarps * 32) rescan_kernel(
    const int* __restrict__ ovf, const RoundCtl* ctl, const float* __restrict__ q, int D, int k, int d,
    uint64_t* __restrict__ keys, int4* __restrict__ qs,
    const float* __restrict__ pts, const uint32_t* __restrict__ pidx, const long long* __restrict__ quad_base,
    uint8_t* __restrict__ ccnt, int NW, int* __restrict__ ovflag) {
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int n = ctl->novf;
  for (int i = blockIdx.x * kFinishWarps + wl; i < n; i += gridDim.x * kFinishWarps) {
    const int qi = __ldg(ovf + i);
    const int leaf = qs[qi].w;
    // the row and kth become final here: advance_kernel merges nothing for this visit
    for (int w = lane; w < NW; w += 32) ccnt[(long long)qi * NW + w] = 0;
    if (lane == 0) ovflag[qi] = 0;
    uint64_t* kp = keys + (long long)qi * k;
    // the row across the warp (warp_row_insert)
    uint64_t r0 = lane < k ? kp[lane] : ~0ull;
    uint64_t r1 = lane + 32 < k ? kp[lane + 32] : ~0ull;
    uint64_t kkey = k <= 32 ? __shfl_sync(0xffffffffu, r0, k - 1) : __shfl_sync(0xffffffffu, r1, k - 33);
    float qv[kSplitMaxD];
#pragma unroll
    for (int j = 0; j < kSplitMaxD; ++j) qv[j] = j < d ? __ldg(q + (long long)qi * D + j) : 0.0f;
    const long long g0 = __ldg(quad_base + leaf), g1 = __ldg(quad_base + leaf + 1);
    for (long long gb = g0; gb < g1; gb += 32) {
      const long long g = gb + lane;
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      const bool has = g < g1;
      if (has) {
        const float4* pq = reinterpret_cast<const float4*>(pts + g * 4 * D);
#pragma unroll
        for (int j = 0; j < kSplitMaxD; ++j) {
          if (j < d) {
            const float4 p = __ldg(pq + j);
            const float e[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float df = __fsub_rn(qv[j], e[t]);
              if constexpr (FMA) acc[t] = __fmaf_rn(df, df, acc[t]);
              else acc[t] = __fadd_rn(acc[t], __fmul_rn(df, df));
            }
          }
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint64_t key = has ? pack_key(acc[t], __ldg(pidx + g * 4 + t)) : ~0ull;
        unsigned bal = __ballot_sync(0xffffffffu, key < kkey);
        while (bal) {
          const int src = __ffs(bal) - 1;
          bal &= bal - 1;
          const uint64_t c = __shfl_sync(0xffffffffu, key, src);
          if (c < kkey) kkey = warp_row_insert(r0, r1, c, k, lane);
        }
      }
    }
    if (lane < k) kp[lane] = r0;
    if (lane + 32 < k) kp[lane + 32] = r1;
    if (lane == 0) reinterpret_cast<int*>(qs + qi)[0] = __float_as_int(key_dist(kkey));
  }
}

}  // namespace bkt
