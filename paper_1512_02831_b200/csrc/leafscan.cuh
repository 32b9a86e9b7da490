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

constexpr int kNT = 128;         // threads (= queries) per tile
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
  int* counts;           // nl: next-round histogram (fused epilogue)
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

template <int D>
struct ScanSmem {
  static constexpr int kQuadBytes = 16 * D;
  static constexpr int kStagePts = kChunkQuads * kQuadBytes;
  static constexpr int kStageIdx = kChunkQuads * 16;
  static constexpr int kBytes = kStages * (kStagePts + kStageIdx) + kStages * 8 + 64;
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
// registers plus ~40 of working set, within 64K registers per SM.
template <int D, int KB>
struct ScanOcc {
  static constexpr int kRegs = 2 * D + 2 * KB + 40;
  static constexpr int kMinBlocks = kRegs <= 128 ? 4 : (kRegs <= 168 ? 3 : 2);
};

template <int D, int KB, bool FMA>
__global__ void __launch_bounds__(kNT, (ScanOcc<D, KB>::kMinBlocks)) leafscan_kernel(const ScanArgs a) {
  using S = ScanSmem<D>;
  extern __shared__ __align__(128) unsigned char smem[];
  float* s_pts = reinterpret_cast<float*>(smem);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(smem + kStages * S::kStagePts);
  uint64_t* s_full = reinterpret_cast<uint64_t*>(smem + kStages * (S::kStagePts + S::kStageIdx));
  int* s_tile = reinterpret_cast<int*>(s_full + kStages);  // leaf, q-begin, q-count

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&s_full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int tiles_end = a.tile_hi >= 0 ? a.tile_hi : *a.num_tiles;
  const int nl = 1 << a.top.h;
  uint32_t gchunk = 0;  // chunks consumed by this CTA so far (ring position / phase)

  for (int t = a.tile_lo + blockIdx.x; t < tiles_end; t += gridDim.x) {
    if (tid == 0) {
      // last leaf with tile_off[leaf] <= t (empty leaves repeat the offset)
      int lo = 0, hi = nl - 1;
      while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(a.tile_off + mid) <= t) lo = mid; else hi = mid - 1;
      }
      int leaf = lo;
      int j = t - __ldg(a.tile_off + leaf);
      int beg = __ldg(a.leaf_off + leaf) + j * kNT;
      int cnt = min(kNT, __ldg(a.leaf_off + leaf + 1) - beg);
      s_tile[0] = leaf; s_tile[1] = beg; s_tile[2] = cnt;
    }
    __syncthreads();
    const int leaf = s_tile[0];
    const int qbeg = s_tile[1];
    const int qcnt = s_tile[2];

    long long g0 = __ldg(a.quad_base + leaf);
    long long g1 = __ldg(a.quad_base + leaf + 1);
    const long long lq0 = g0;
    g0 = max(g0, a.clip_lo);
    g1 = min(g1, a.clip_hi);
    const int nquads = (int)max(0ll, g1 - g0);
    const int nchunks = (nquads + kChunkQuads - 1) / kChunkQuads;

    // producer prologue: fill the ring
    if (tid == 0) {
      for (int c = 0; c < min(kStages, nchunks); ++c) {
        int s = (gchunk + c) % kStages;
        int nq = min(kChunkQuads, nquads - c * kChunkQuads);
        long long gq = g0 + (long long)c * kChunkQuads - a.quad_origin;
        mbar_arrive_expect_tx(&s_full[s], nq * (S::kQuadBytes + 16));
        bulk_g2s(s_pts + s * (S::kStagePts / 4), a.pts + gq * 4 * D, nq * S::kQuadBytes, &s_full[s]);
        bulk_g2s(s_idx + s * (S::kStageIdx / 4), a.pidx + gq * 4, nq * 16, &s_full[s]);
      }
    }

    // this thread's query
    const bool valid = tid < qcnt;
    int qi = 0;
    uint64_t qq[D];
    uint64_t arr[KB];
    if (valid) {
      qi = __ldg(a.work + qbeg + tid);
      const float* qp = a.q + (long long)qi * D;
#pragma unroll
      for (int j = 0; j < D; ++j) qq[j] = f2_splat(__ldg(qp + j));
      const uint64_t* kp = a.keys + (long long)qi * a.k;
#pragma unroll
      for (int j = 0; j < KB; ++j) arr[j] = (j < a.k) ? kp[a.k - 1 - j] : 0ull;
    } else {
#pragma unroll
      for (int j = 0; j < D; ++j) qq[j] = 0;
#pragma unroll
      for (int j = 0; j < KB; ++j) arr[j] = 0;
    }
    float kth = key_dist(arr[0]);
    const uint64_t zero = a.zero;

    for (int c = 0; c < nchunks; ++c) {
      const int s = (gchunk + c) % kStages;
      const uint32_t ph = ((gchunk + c) / kStages) & 1u;
      const int nq = min(kChunkQuads, nquads - c * kChunkQuads);
      mbar_wait(&s_full[s], ph);
      if (valid) {
        // quad u, dim j: 16 bytes = (p0, p1) | (p2, p3) as two f32x2 lanes
        const ulonglong2* sp = reinterpret_cast<const ulonglong2*>(s_pts + s * (S::kStagePts / 4));
        const uint32_t* si = s_idx + s * (S::kStageIdx / 4);
#pragma unroll 1
        for (int u = 0; u < nq; ++u) {
          // j = 0: acc = RN(diff^2) (== RN(0 + diff^2), the reference's first step)
          ulonglong2 v0 = sp[u * D];
          uint64_t df0 = f2_sub(qq[0], v0.x), df1 = f2_sub(qq[0], v0.y);
          uint64_t acc0 = f2_fma(df0, df0, zero), acc1 = f2_fma(df1, df1, zero);
#pragma unroll
          for (int j = 1; j < D; ++j) {
            ulonglong2 v = sp[u * D + j];
            acc0 = dist_step<FMA>(acc0, qq[j], v.x, zero);
            acc1 = dist_step<FMA>(acc1, qq[j], v.y, zero);
          }
          float d0 = f2_lo(acc0), d1 = f2_hi(acc0), d2 = f2_lo(acc1), d3 = f2_hi(acc1);
          float mn = fminf(fminf(d0, d1), fminf(d2, d3));
          if (mn <= kth) {
            // rare: at least one of the four may enter the top-k
            uint4 ids = *reinterpret_cast<const uint4*>(si + 4 * u);
            uint64_t c0 = pack_key(d0, ids.x), c1 = pack_key(d1, ids.y);
            uint64_t c2 = pack_key(d2, ids.z), c3 = pack_key(d3, ids.w);
            if (c0 < arr[0]) topk_insert<KB>(arr, c0);
            if (c1 < arr[0]) topk_insert<KB>(arr, c1);
            if (c2 < arr[0]) topk_insert<KB>(arr, c2);
            if (c3 < arr[0]) topk_insert<KB>(arr, c3);
            kth = key_dist(arr[0]);
          }
        }
      }
      __syncthreads();  // stage s fully consumed
      if (tid == 0 && c + kStages < nchunks) {
        int cc = c + kStages;
        int nq2 = min(kChunkQuads, nquads - cc * kChunkQuads);
        long long gq = g0 + (long long)cc * kChunkQuads - a.quad_origin;
        mbar_arrive_expect_tx(&s_full[s], nq2 * (S::kQuadBytes + 16));
        bulk_g2s(s_pts + s * (S::kStagePts / 4), a.pts + gq * 4 * D, nq2 * S::kQuadBytes, &s_full[s]);
        bulk_g2s(s_idx + s * (S::kStageIdx / 4), a.pidx + gq * 4, nq2 * 16, &s_full[s]);
      }
    }
    gchunk += nchunks;

    if (tid == 0 && a.pairs) {
      // real points of this leaf inside the clipped quad range
      long long L = __ldg(a.leaf_size + leaf);
      long long p0 = (g0 - lq0) * 4, p1 = (g1 - lq0) * 4;
      long long real = max(0ll, min(L, p1) - p0);
      atomicAdd(a.pairs, (unsigned long long)(real * qcnt));
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
        if (nxt >= 0) {
          uint32_t v = a.visits[qi] + 1;
          a.visits[qi] = v;
          log_visit(a, qi, v, nxt);
          warp_count(a.counts, nxt);
        }
      }
    }
    __syncthreads();  // s_tile reuse
  }
}

}  // namespace bkt
