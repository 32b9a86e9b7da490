// wide_search.cuh -- the general-domain search path: any k <= n, any d, any
// height 2^h <= n (h <= 30), on resident or host-resident (mapped) leaf
// structures.
//
// The round engine (leafscan*.cuh, split_scan.cuh) keeps a query's top-k in
// registers (k <= 64), its traversal state in 4 bytes (h <= 16) and compiles
// the distance loop per dimensionality (d <= 32).  The reference has none of
// these limits (core.py:92-102 accepts any k <= n, buffer_tree.py:159-163 any
// h with 2^h <= n, and any d), so queries outside them run here: one CTA per
// query (queries taken from a global counter), the whole per-query traversal
// in one launch -- the reference's per-query leaf order, which equals
// lazy_search's (acceptance criterion 4; buffer_tree.py:292-378 FindLeaf,
// 523-646 lazy_search) -- with
//   * the query's coordinates in shared memory,
//   * each leaf scanned by all threads (thread per 4-point quad, reference
//     arithmetic: d sub + d mul + d add left to right, core.py:108-146),
//   * points whose packed key beats the current k-th key appended to a
//     shared candidate list, which is merged into the sorted top-k row by a
//     bitonic sort + merge-path step (the best k of row and candidates, the
//     reference's NeighborBatch.update_rows, core.py:251-262),
//   * FindLeaf by thread 0 with the k-th distance after the leaf
//     (buffer_tree.py:330-349), traversal state (path, pending far-child
//     depths) in two 32-bit registers.
// The k-th key read while a leaf is scanned can only be stale-high (it only
// decreases), so a candidate is never lost; the row after a leaf is the best k
// of (row, leaf), so kth, pruning and the visit order are the reference's.
#pragma once
#include "bkt_device.cuh"
#include "round_kernels.cuh"

namespace bkt {

constexpr int kWideT = 256;        // threads per CTA
constexpr int kWideC = 2048;       // candidate list capacity (a slice adds <= 4 * kWideT)
constexpr int kWideQSmem = 8192;   // query coordinates kept in shared memory up to this d

struct WideArgs {
  const float* q;                  // m x D query rows
  int D;                           // row stride of q and quad layout width
  int m;
  int k;
  TopTreeView top;
  uint64_t* keys;                  // m x k result rows (ascending)
  uint32_t* visits;
  const float* pts;                // quad layout (engine.cu): quad g, dim j, point t at g*4D + 4j + t
  const uint32_t* pidx;
  const long long* quad_base;
  const int* leaf_size;
  unsigned long long* pairs;
  RoundCtl* ctl;                   // scans (+=), rounds (max visits), tile_next (query counter)
  int* seq_log;
  unsigned long long* seq_pos;
  long long seq_cap;
  uint64_t* scratch;               // 2k keys per CTA when the rows do not fit in shared memory (else null)
};

__host__ __device__ inline size_t wide_smem_bytes(int k, int d, bool rows_in_smem) {
  return sizeof(uint64_t) * (kWideC + (rows_in_smem ? 2ll * k : 0)) + (d <= kWideQSmem ? sizeof(float) * d : 0) + 64;
}

// number of entries of a (ascending) that are < x, a[0..n)
__device__ __forceinline__ int count_less(const uint64_t* a, int n, uint64_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <bool FMA>
__global__ void __launch_bounds__(kWideT) wide_search_kernel(const WideArgs a) {
  extern __shared__ __align__(16) unsigned char s_wide[];
  uint64_t* s_cand = reinterpret_cast<uint64_t*>(s_wide);
  const bool rows_smem = a.scratch == nullptr;
  uint64_t* rowbuf[2];
  float* s_qv;
  if (rows_smem) {
    rowbuf[0] = s_cand + kWideC;
    rowbuf[1] = rowbuf[0] + a.k;
    s_qv = reinterpret_cast<float*>(rowbuf[1] + a.k);
  } else {
    rowbuf[0] = a.scratch + 2ll * a.k * blockIdx.x;
    rowbuf[1] = rowbuf[0] + a.k;
    s_qv = reinterpret_cast<float*>(s_cand + kWideC);
  }
  __shared__ int s_nc, s_leaf, s_qi;
  const int tid = threadIdx.x;
  const int d = a.top.d, D = a.D, k = a.k;
  unsigned long long pairs_acc = 0, scans_acc = 0;
  uint32_t max_vis = 0;
  for (;;) {
    __syncthreads();  // the previous query's shared state is consumed
    if (tid == 0) s_qi = atomicAdd(&a.ctl->tile_next, 1);
    __syncthreads();
    const int qi = s_qi;
    if (qi >= a.m) break;
    const float* qrow = a.q + (long long)qi * D;
    const float* qv = d <= kWideQSmem ? s_qv : qrow;
    if (d <= kWideQSmem)
      for (int j = tid; j < d; j += kWideT) s_qv[j] = __ldg(qrow + j);
    int cur = 0;
    for (int j = tid; j < k; j += kWideT) rowbuf[0][j] = kEmptyKey;
    if (tid == 0) s_nc = 0;
    __syncthreads();
    // root -> home leaf (buffer_tree.py:365-376), by thread 0
    uint32_t lf = 0, pend = 0, vis = 0;
    const float* sp = a.top.split;
    auto sget = [sp](uint32_t node) { return __ldg(sp + node); };
    auto qget = [qv](int j) { return qv[j]; };
    if (tid == 0) {
      descend_with(a.top.h, d, sget, qget, lf, pend, 0);
      vis = 1;
      s_leaf = (int)lf;
      if (a.seq_log) {
        const unsigned long long p = atomicAdd(a.seq_pos, 1ull);
        if ((long long)p < a.seq_cap) {
          a.seq_log[3 * p] = qi; a.seq_log[3 * p + 1] = 1; a.seq_log[3 * p + 2] = (int)lf;
        }
      }
    }
    __syncthreads();
    int leaf = s_leaf;
    while (leaf >= 0) {
      const long long g0 = __ldg(a.quad_base + leaf), g1 = __ldg(a.quad_base + leaf + 1);
      for (long long gb = g0; gb < g1; gb += kWideT) {
        const uint64_t kkey = rowbuf[cur][k - 1];
        const long long g = gb + tid;
        if (g < g1) {
          float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
          const float4* pq = reinterpret_cast<const float4*>(a.pts + g * 4 * D);
#pragma unroll 4
          for (int j = 0; j < d; ++j) {
            const float4 p = pq[j];
            const float qj = qv[j];
            const float e[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float df = __fsub_rn(qj, e[t]);
              if constexpr (FMA) acc[t] = __fmaf_rn(df, df, acc[t]);
              else acc[t] = __fadd_rn(acc[t], __fmul_rn(df, df));
            }
          }
          const uint4 id4 = reinterpret_cast<const uint4*>(a.pidx)[g];
          const uint32_t ids[4] = {id4.x, id4.y, id4.z, id4.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint64_t key = pack_key(acc[t], ids[t]);
            if (ids[t] != kIndexSentinel && key < kkey) s_cand[atomicAdd(&s_nc, 1)] = key;
          }
        }
        __syncthreads();
        const int nc = s_nc;
        __syncthreads();  // every thread has read nc before the next slice appends
        // merge when the list could overflow with the next slice, or at the leaf's end
        if (nc > 0 && (nc > kWideC - 4 * kWideT || gb + kWideT >= g1)) {
          // bitonic sort of the candidates (padded to a power of two with ~0)
          int n2 = 2;
          while (n2 < nc) n2 <<= 1;
          for (int i = nc + tid; i < n2; i += kWideT) s_cand[i] = ~0ull;
          __syncthreads();
          for (int size = 2; size <= n2; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
              for (int t = tid; t < (n2 >> 1); t += kWideT) {
                const int lo = 2 * stride * (t / stride) + (t % stride), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t x = s_cand[lo], y = s_cand[hi];
                if ((x > y) == up) { s_cand[lo] = y; s_cand[hi] = x; }
              }
              __syncthreads();
            }
          }
          // merge path: every element's rank in the union; the first k survive
          const uint64_t* src = rowbuf[cur];
          uint64_t* dst = rowbuf[cur ^ 1];
          for (int i = tid; i < k; i += kWideT) {
            const uint64_t x = src[i];
            const int r = i + count_less(s_cand, nc, x);
            if (r < k) dst[r] = x;
          }
          for (int i = tid; i < nc; i += kWideT) {
            const uint64_t x = s_cand[i];
            const int r = i + count_less(src, k, x);
            if (r < k) dst[r] = x;
          }
          cur ^= 1;
          __syncthreads();
          if (tid == 0) s_nc = 0;
          __syncthreads();
        }
      }
      if (tid == 0) {
        pairs_acc += (unsigned long long)__ldg(a.leaf_size + leaf);
        scans_acc += 1;
        const float kth = key_dist(rowbuf[cur][k - 1]);
        const int nxt = find_next_leaf_with(a.top.h, d, sget, qget, kth, lf, pend);
        if (nxt >= 0) {
          ++vis;
          if (a.seq_log) {
            const unsigned long long p = atomicAdd(a.seq_pos, 1ull);
            if ((long long)p < a.seq_cap) {
              a.seq_log[3 * p] = qi; a.seq_log[3 * p + 1] = (int)vis; a.seq_log[3 * p + 2] = nxt;
            }
          }
        }
        s_leaf = nxt;
      }
      __syncthreads();
      leaf = s_leaf;
    }
    uint64_t* kp = a.keys + (long long)qi * k;
    for (int j = tid; j < k; j += kWideT) kp[j] = rowbuf[cur][j];
    if (tid == 0) {
      a.visits[qi] = vis;
      max_vis = max(max_vis, vis);
    }
  }
  if (tid == 0 && scans_acc) {
    if (a.pairs) atomicAdd(a.pairs, pairs_acc);
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.ctl->scans), scans_acc);
    atomicMax(&a.ctl->rounds, (int)max_vis);
  }
}

// Launch: one CTA per query at a time, persistent over the batch.  grid = 0
// only reports the resident CTAs per SM for this shared-memory size.
template <bool FMA>
inline cudaError_t launch_wide_one(int grid, cudaStream_t s, const WideArgs& a, size_t smem, int* occ) {
  auto fn = wide_search_kernel<FMA>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, kWideT, smem);
  fn<<<grid, kWideT, smem, s>>>(a);
  return cudaGetLastError();
}

inline cudaError_t launch_wide(bool fma, int grid, cudaStream_t s, const WideArgs& a, size_t smem, int* occ) {
  return fma ? launch_wide_one<true>(grid, s, a, smem, occ) : launch_wide_one<false>(grid, s, a, smem, occ);
}

}  // namespace bkt
