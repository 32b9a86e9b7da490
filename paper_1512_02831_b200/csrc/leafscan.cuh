// leafscan.cuh -- ProcessAllBuffers' brute-force leaf stage on sm_100a, with the
// next FindLeaf step fused into its epilogue.
//
// Replaces (reference):
//   device.py:283-337  SimulatedDevice.enqueue_brute_kernel / scan (316-321)
//   core.py:138-146    sq_distances_block
//   core.py:152-160    pack_keys
//   core.py:251-262    NeighborBatch.update_rows (top-k merge)
//   buffer_tree.py:292-378 find_leaf_batch (fused epilogue, resumed queries)
//
// Work unit ("tile"): up to kNT queries that all sit in the same leaf's
// buffer this round.  One thread owns one query: its coordinates live in
// registers (splatted to f32x2 pairs), its top-k list lives in registers
// (descending, arr[0] = pruning radius).  The leaf's points stream through
// shared memory in quad-interleaved form (4 points x D dims per 16*D bytes),
// staged by 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx) in a
// kStages-deep ring.  Every lane reads the same quad (shared-memory broadcast),
// so one LDS.128 feeds two FADD2/FFMA2 chains (points 0,1 and 2,3).
//
// The grid is persistent (a multiple of the SM count); CTAs stride over the
// round's tile list, whose length lives in device memory, so a round needs no
// host round trip.
#pragma once
#include "bkt_device.cuh"

namespace bkt {

constexpr int kNT = 128;         // consumer threads (= queries) per tile
constexpr int kStages = 4;       // TMA ring depth
constexpr int kChunkQuads = 32;  // quads (4 points) per ring stage

struct ScanArgs {
  // per-query state, indexed by batch-local query id
  const float* q;        // m x D (kernel dimensionality, zero padded past d)
  uint64_t* keys;        // m x k, ascending (NeighborBatch.keys layout)
  uint32_t* state;       // m, packed path + pending mask
  int* next;             // m, next leaf or -1
  uint32_t* visits;      // m, leaves visited so far
  // this round's schedule
  const int* work;       // active query ids grouped by leaf
  const int* leaf_off;   // nl + 1: start of each leaf's group in `work`
  const int* tile_off;   // nl + 1: first tile of each leaf
  const int* num_tiles;  // device scalar: tiles this round
  int tile_lo, tile_hi;  // chunk mode: tile sub-range; tile_hi < 0 = [0, *num_tiles)
  const int4* tiles;     // per-tile {leaf, qbeg, qcnt} written by plan_kernel
  int* counts;           // nl: next-round histogram (fused epilogue)
  int2* pos;             // m: per work-list position {next leaf or -1, slot in that leaf's next-round bucket}
  int* tile_next;        // round's tile counter for dynamic tile scheduling (zeroed by plan_kernel), or null
  // leaf structure, quad-interleaved: quad g, dim j, point t at pts[(g - quad_origin)*4D + 4j + t]
  const float* pts;
  const uint32_t* pidx;  // original index of point (g - quad_origin)*4 + t (padding: 0xFFFFFFFF)
  long long quad_origin;
  long long clip_lo, clip_hi;   // quad range present in `pts` (chunk mode); whole structure otherwise
  const long long* quad_base;   // nl + 1: first quad of each leaf
  const int* leaf_size;         // nl: real points per leaf
  TopTreeView top;
  int k;
  int fused;
  uint64_t zero;                // runtime +0.0f pair (see dist_step)
  unsigned long long* pairs;    // algorithmic (query, real point) pairs scanned
  int* seq_log;                 // optional: (query, visit number, leaf) triples
  unsigned long long* seq_pos;
  long long seq_cap;
};

constexpr int kConsumerWarps = kNT / 32;
constexpr int kThreads = kNT + 32;  // + one TMA producer warp
#ifndef BKT_QUEUE
#define BKT_QUEUE 8
#endif
constexpr int kQueue = BKT_QUEUE;   // per-thread candidate queue (shared memory)

template <int D>
struct ScanSmem {
  static constexpr int kQuadBytes = 16 * D;
  static constexpr int kStagePts = kChunkQuads * kQuadBytes;
  static constexpr int kStageIdx = kChunkQuads * 16;
  static constexpr int kQueueBytes = kQueue * kNT * 8;
  // + full/empty barriers, 8 tile-publication barriers and 8 tile slots
  static constexpr int kBytes = kStages * (kStagePts + kStageIdx) + kQueueBytes + 2 * kStages * 8 + 8 * 8 + 8 * 4 + 64;
};

__device__ __forceinline__ void log_visit(const ScanArgs& a, int qi, uint32_t visit, int leaf) {
  if (a.seq_log) {
    unsigned long long p = atomicAdd(a.seq_pos, 1ull);
    if ((long long)p < a.seq_cap) {
      a.seq_log[3 * p + 0] = qi;
      a.seq_log[3 * p + 1] = (int)visit;
      a.seq_log[3 * p + 2] = leaf;
    }
  }
}

// Resident CTAs per SM the register budget allows: query (2D) + top-k (2KB)
// registers plus ~48 of working set, within 64K registers per SM.
template <int D, int KB>
struct ScanOcc {
  static constexpr int kRegs = 2 * D + 2 * KB + 48;
  static constexpr int kMinBlocks = kRegs <= 96 ? 4 : (kRegs <= 128 ? 3 : 2);
};

struct TileInfo {
  int leaf, qbeg, qcnt;
  long long g0, g1, lq0;  // clipped quad range and the leaf's first quad
  int nchunks;
};

__device__ __forceinline__ TileInfo tile_info(const ScanArgs& a, int t) {
  const int4 rec = __ldg(a.tiles + t);
  TileInfo T;
  T.leaf = rec.x;
  T.qbeg = rec.y;
  T.qcnt = rec.z;
  T.lq0 = __ldg(a.quad_base + rec.x);
  T.g0 = max(T.lq0, a.clip_lo);
  T.g1 = min(__ldg(a.quad_base + rec.x + 1), a.clip_hi);
  const int nq = (int)max(0ll, T.g1 - T.g0);
  T.nchunks = (nq + kChunkQuads - 1) / kChunkQuads;
  return T;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Insert every queued candidate of this lane into its register top-k.  All
// lanes of the warp run this together (warp-convergent), so a burst of
// candidates costs one pass instead of one divergent pass per candidate.
template <int KB>
__device__ __forceinline__ void merge_queue(uint64_t (&arr)[KB], const uint64_t* qslot, int& cn, float& kth) {
#pragma unroll 1
  for (int j = 0; j < cn; ++j) {
    uint64_t c = qslot[j * kNT];
    if (c < arr[0]) topk_insert<KB>(arr, c);
  }
  cn = 0;
  kth = key_dist(arr[0]);
}

template <int D, int KB, bool FMA>
__global__ void __launch_bounds__(kThreads, (ScanOcc<D, KB>::kMinBlocks)) leafscan_kernel(const ScanArgs a) {
  using S = ScanSmem<D>;
  extern __shared__ __align__(128) unsigned char smem[];
  float* s_pts = reinterpret_cast<float*>(smem);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(smem + kStages * S::kStagePts);
  uint64_t* s_queue = reinterpret_cast<uint64_t*>(smem + kStages * (S::kStagePts + S::kStageIdx));
  uint64_t* s_full = reinterpret_cast<uint64_t*>(smem + kStages * (S::kStagePts + S::kStageIdx) + S::kQueueBytes);
  uint64_t* s_empty = s_full + kStages;
  uint64_t* s_tready = s_empty + kStages;                                // [8]
  volatile int* s_tile = reinterpret_cast<volatile int*>(s_tready + 8);  // [8]

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], kConsumerWarps);
    }
    for (int s = 0; s < 8; ++s) mbar_init(&s_tready[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int tiles_end = a.tile_hi >= 0 ? a.tile_hi : *a.num_tiles;
  // Tile order (see leafscan_tc.cuh): dynamic from the round's counter when
  // the launch covers the whole round -- consumer thread 0 publishes the j-th
  // tile of this CTA two tiles ahead in s_tile[j & 7] (the consumer warps
  // drift apart by at most kStages chunks, so eight slots never collide) --
  // static striding for a chunk's tile sub-range (out-of-core rounds).
  const bool dyn = a.tile_next != nullptr && a.tile_hi < 0;
  auto seq_tile = [&](uint32_t j) -> int {
    if (dyn) {
      mbar_wait(&s_tready[j & 7u], (j >> 3) & 1u);
      return s_tile[j & 7u];
    }
    return a.tile_lo + (int)blockIdx.x + (int)j * (int)gridDim.x;
  };

  if (warp == kConsumerWarps) {
    // ===== TMA producer: streams every tile's leaf chunks through the ring,
    // running ahead across tile boundaries =====
    if (lane == 0) {
      uint32_t g = 0;
      for (uint32_t j = 0;; ++j) {
        const int t = seq_tile(j);
        if (t >= tiles_end) break;
        const TileInfo T = tile_info(a, t);
        const int nquads = (int)(T.g1 - T.g0);
        for (int c = 0; c < T.nchunks; ++c, ++g) {
          const int s = g % kStages;
          const uint32_t use = g / kStages;
          if (use > 0) mbar_wait(&s_empty[s], (use - 1) & 1u);
          const int nq = min(kChunkQuads, nquads - c * kChunkQuads);
          const long long gq = T.g0 + (long long)c * kChunkQuads - a.quad_origin;
          mbar_arrive_expect_tx(&s_full[s], nq * (S::kQuadBytes + 16));
          bulk_g2s(s_pts + s * (S::kStagePts / 4), a.pts + gq * 4 * D, nq * S::kQuadBytes, &s_full[s]);
          bulk_g2s(s_idx + s * (S::kStageIdx / 4), a.pidx + gq * 4, nq * 16, &s_full[s]);
        }
      }
    }
    return;
  }

  // ===== consumers: one thread per query =====
  uint64_t* qslot = s_queue + tid;  // this thread's queue: qslot[j * kNT]
  const uint64_t zero = a.zero;
  uint32_t g = 0;
  int grabbed = 0;
  auto publish = [&](uint32_t j) {  // consumer thread 0
    s_tile[j & 7u] = grabbed;
    mbar_arrive(&s_tready[j & 7u]);
    if (grabbed < tiles_end) grabbed = a.tile_lo + atomicAdd(a.tile_next, 1);
  };
  if (dyn && tid == 0) {
    grabbed = a.tile_lo + atomicAdd(a.tile_next, 1);
    publish(0);
    publish(1);
  }
  for (uint32_t j = 0;; ++j) {
    if (dyn && tid == 0) publish(j + 2);
    const int t = seq_tile(j);
    if (t >= tiles_end) break;
    const TileInfo T = tile_info(a, t);
    const int nquads = (int)(T.g1 - T.g0);
    const bool valid = tid < T.qcnt;
    const bool warp_active = warp * 32 < T.qcnt;
    int qi = 0;
    uint64_t qq[D];
    uint64_t arr[KB];
    float kth = -__int_as_float(0x7f800000);  // -inf: invalid lanes never take candidates
    if (valid) {
      qi = __ldg(a.work + T.qbeg + tid);
      const float* qp = a.q + (long long)qi * D;
#pragma unroll
      for (int j = 0; j < D; ++j) qq[j] = f2_splat(__ldg(qp + j));
      const uint64_t* kp = a.keys + (long long)qi * a.k;
#pragma unroll
      for (int j = 0; j < KB; ++j) arr[j] = (j < a.k) ? kp[a.k - 1 - j] : 0ull;
      kth = key_dist(arr[0]);
    } else {
#pragma unroll
      for (int j = 0; j < D; ++j) qq[j] = 0;
#pragma unroll
      for (int j = 0; j < KB; ++j) arr[j] = 0;
    }
    int cn = 0;  // queued candidates

    for (int c = 0; c < T.nchunks; ++c, ++g) {
      const int s = g % kStages;
      mbar_wait(&s_full[s], (g / kStages) & 1u);
      if (warp_active) {
        const int nq = min(kChunkQuads, nquads - c * kChunkQuads);
        // quad u, dim j: 16 bytes = (p0, p1) | (p2, p3) as two f32x2 lanes
        const ulonglong2* sp = reinterpret_cast<const ulonglong2*>(s_pts + s * (S::kStagePts / 4));
        const uint4* si = reinterpret_cast<const uint4*>(s_idx + s * (S::kStageIdx / 4));
#pragma unroll 1
        for (int u = 0; u < nq; u += 2) {
          const bool two = u + 1 < nq;
          const int u1 = two ? u + 1 : u;  // odd tail: recompute quad u (its candidates are deduplicated below)
          // j = 0: acc = RN(diff^2) == RN(+0 + diff^2), the reference's first step
          ulonglong2 va = sp[u * D], vb = sp[u1 * D];
          uint64_t da0 = f2_sub(qq[0], va.x), da1 = f2_sub(qq[0], va.y);
          uint64_t db0 = f2_sub(qq[0], vb.x), db1 = f2_sub(qq[0], vb.y);
          uint64_t a0 = f2_fma(da0, da0, zero), a1 = f2_fma(da1, da1, zero);
          uint64_t b0 = f2_fma(db0, db0, zero), b1 = f2_fma(db1, db1, zero);
#pragma unroll
          for (int j = 1; j < D; ++j) {
            ulonglong2 wa = sp[u * D + j], wb = sp[u1 * D + j];
            a0 = dist_step<FMA>(a0, qq[j], wa.x, zero);
            a1 = dist_step<FMA>(a1, qq[j], wa.y, zero);
            b0 = dist_step<FMA>(b0, qq[j], wb.x, zero);
            b1 = dist_step<FMA>(b1, qq[j], wb.y, zero);
          }
          float dd[8] = {f2_lo(a0), f2_hi(a0), f2_lo(a1), f2_hi(a1), f2_lo(b0), f2_hi(b0), f2_lo(b1), f2_hi(b1)};
          float mn = fminf(fminf(fminf(dd[0], dd[1]), fminf(dd[2], dd[3])),
                           fminf(fminf(dd[4], dd[5]), fminf(dd[6], dd[7])));
          if (__any_sync(0xffffffffu, mn <= kth)) {
            // rare (except in a query's first leaves): queue the candidates
            const uint4 ia = si[u], ib = si[u1];
            const uint32_t ii[8] = {ia.x, ia.y, ia.z, ia.w, ib.x, ib.y, ib.z, ib.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              if (e == 4 && (!two || __any_sync(0xffffffffu, cn > kQueue - 4))) {
                merge_queue<KB>(arr, qslot, cn, kth);
                if (!two) break;
              }
              if (dd[e] <= kth) qslot[(cn++) * kNT] = pack_key(dd[e], ii[e]);
            }
            if (__any_sync(0xffffffffu, cn > kQueue - 4)) merge_queue<KB>(arr, qslot, cn, kth);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[s]);
    }
    if (warp_active && __any_sync(0xffffffffu, cn > 0)) merge_queue<KB>(arr, qslot, cn, kth);

    if (tid == 0 && a.pairs) {
      // real points of this leaf inside the clipped quad range
      long long L = __ldg(a.leaf_size + T.leaf);
      long long p0 = (T.g0 - T.lq0) * 4, p1 = (T.g1 - T.lq0) * 4;
      long long real = max(0ll, min(L, p1) - p0);
      atomicAdd(a.pairs, (unsigned long long)(real * T.qcnt));
    }

    if (valid) {
      uint64_t* kp = a.keys + (long long)qi * a.k;
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < a.k) kp[a.k - 1 - j] = arr[j];
      if (a.fused) {
        const float* qp = a.q + (long long)qi * D;
        auto qget = [qp](int j) { return __ldg(qp + j); };
        uint32_t st = a.state[qi];
        uint32_t lf = st & 0xFFFFu, pend = st >> 16;
        int nxt = find_next_leaf(a.top, qget, key_dist(arr[0]), lf, pend);
        a.state[qi] = (pend << 16) | lf;
        a.next[qi] = nxt;
        int rk = 0;
        if (nxt >= 0) {
          uint32_t v = a.visits[qi] + 1;
          a.visits[qi] = v;
          log_visit(a, qi, v, nxt);
          rk = warp_reserve(a.counts, nxt);  // next round's bucket (key = leaf) and slot
        }
        a.pos[T.qbeg + tid] = make_int2(nxt, rk);  // coalesced: read back by position in scatter
      }
    }
  }
}

}  // namespace bkt
