// round_kernels.cuh -- the per-round scheduling kernels of the device-resident
// LazySearch loop (Alg. 1; reference buffer_tree.py:523-646).
//
// One round = plan -> scatter -> leafscan(+fused FindLeaf and bucket count):
//   start   : every fresh query descends to its home leaf (find_leaf_batch for
//             fresh queries, buffer_tree.py:318-321, 351-376), is routed down
//             that leaf's block split tree and counted into bucket (leaf, block).
//   later rounds count each query's next leaf in the scan epilogue.
//   plan    : exclusive scans of the per-key counts -> each key's and each
//             leaf's slice of the work list and the leaf's tile range (the
//             "buffers" of QueryBuffers.drain_all, buffer_tree.py:420-430, in
//             leaf order; inside a leaf, ordered by block).
//   scatter : counting-sort placement of the still-active queries into their
//             key's slice at the slot taken when counted (the reference's
//             stable argsort + insert_many, buffer_tree.py:603-619).  DONE
//             queries drop out (buffer_tree.py:482-485).
//   findleaf: unfused FindLeaf for the out-of-core path (leafscan fuses it
//             when the whole leaf structure is resident).
//   finish  : the tail -- once few queries remain, one warp per query runs
//             the rest of its traversal (leaf scan, top-k, FindLeaf) in a
//             single launch instead of one round per remaining leaf.
#pragma once
#include "bkt_device.cuh"

namespace bkt {

struct RoundCtl {
  int active;       // queries with a leaf to scan this round
  int prev_active;  // length of the previous round's work list
  int num_tiles;    // tiles this round
  int rounds;       // rounds with active > 0
  long long scans;  // (query, leaf) scans so far (SearchStats.leaf_scan_events)
  int late_n;       // early result drain: queries still active when it started
  int tile_next;    // dynamic tile counter of the round's leaf scan (reset by plan_kernel)
  // split rounds (split_scan.cuh)
  int stiles;       // (leaf, window) tiles this round
  int novf;         // queries whose candidate list overflowed this round
  int items;        // (query, window) work items this round
  // split-round totals of the batch (diagnostics, BKT_VERBOSE)
  unsigned long long sc_tiles, sc_chunks, sc_cands, sc_flushes, sc_items, sc_surv, sc_trips;
  // out-of-core drain (engine.cu ooc_drain)
  int park_n;       // queries parked for a later streaming unit
  int plan_seq;     // plan_kernel launches so far (the host matches it against its mirror slot)
  unsigned ps_done; // plan_scatter_kernel: CTAs finished this launch (the last one publishes the round)
};

// Out-of-core drain: append `qi` to the park list for the lanes with `pred`
// (one atomic per warp).
__device__ __forceinline__ void park_append(bool pred, int qi, int* __restrict__ park, int* park_n) {
  const unsigned mask = __activemask();
  const unsigned b = __ballot_sync(mask, pred);
  if (!b) return;
  const int lane = threadIdx.x & 31, leader = __ffs(b) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(park_n, __popc(b));
  base = __shfl_sync(mask, base, leader);
  if (pred) park[base + __popc(b & ((1u << lane) - 1u))] = qi;
}

// The park list becomes the list to classify: active = its length, a fresh
// (empty) park count for the next list.
__global__ void ooc_switch_kernel(RoundCtl* ctl) {
  ctl->active = ctl->park_n;
  ctl->park_n = 0;
}

// First park list of a batch: every query (start_kernel set its home leaf).
__global__ void ooc_init_kernel(int* __restrict__ park, long long m, RoundCtl* ctl) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
    park[i] = (int)i;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->park_n = (int)m;
}

// Queries of `list` (ctl->active entries) whose next leaf lies in the
// resident unit [leaf_lo, leaf_hi] take a bucket slot for it; the others are
// parked again (pos.x = -1: scatter_kernel skips them).
__global__ void ooc_classify_kernel(const int* __restrict__ list, RoundCtl* ctl, const int* __restrict__ next,
                                    int leaf_lo, int leaf_hi, int* __restrict__ counts, int2* __restrict__ pos,
                                    int* __restrict__ park) {
  const int n = ctl->active;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int qi = __ldg(list + i);
    const int nx = __ldg(next + qi);
    const bool in = nx >= leaf_lo && nx <= leaf_hi;
    int rk = 0;
    if (in) rk = warp_reserve(counts, nx);
    park_append(!in && nx >= 0, qi, park, &ctl->park_n);
    pos[i] = make_int2(in ? nx : -1, rk);
  }
}

// Early result drain: remember the queries of the round just scanned (every
// query still active later is among them; the active set only shrinks).
__global__ void snapshot_active(const int* __restrict__ work, RoundCtl* ctl, int* __restrict__ late_ids) {
  const int n = ctl->active;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) late_ids[i] = work[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->late_n = n;
}

// ... and at the end gather their final top-k rows for the host fix-up.
__global__ void gather_late(const uint64_t* __restrict__ keys, int k, const int* __restrict__ late_ids,
                            const RoundCtl* ctl, uint64_t* __restrict__ out) {
  const long long total = (long long)ctl->late_n * k;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / k;
    out[t] = keys[(long long)late_ids[i] * k + (t - i * k)];
  }
}

constexpr int kPlanThreads = 1024;

// FindLeafBatch for fresh queries (buffer_tree.py:318-321, 351-376): EMPTY
// top-k, descend from the root, route to the home block, count.  Each CTA
// takes 256 consecutive queries at a time: their rows (one contiguous block)
// arrive with coalesced 16-byte loads into shared memory, their top-k rows
// are initialised with coalesced stores, and the top tree's split values sit
// in shared memory when they fit (start_smem_bytes).
constexpr int kStartQ = 256;
// split values kept in shared memory: up to 16 KB (h <= 12) beside ...
__host__ __device__ inline int start_tree_smem(int h) { return ((1 << h) - 1) * 4 <= 16384 ? ((1 << h) - 1) : 0; }
// ... and for start_kernel only while tree + rows stay within the 48 KB default
__host__ __device__ inline int start_tree_n(int h, int D) {
  const int t = start_tree_smem(h);
  return t * 4 + kStartQ * (D + 1) * 4 <= 48 * 1024 ? t : 0;
}
__host__ __device__ inline int start_smem_bytes(int h, int D) { return start_tree_n(h, D) * 4 + kStartQ * (D + 1) * 4; }

__global__ void __launch_bounds__(kStartQ) start_kernel(const float* __restrict__ q, int D, long long m, int k,
                                                        TopTreeView top, uint64_t* __restrict__ keys,
                                                        uint32_t* __restrict__ state, int* __restrict__ next,
                                                        uint32_t* __restrict__ visits, int* seq_log,
                                                        unsigned long long* seq_pos, long long seq_cap,
                                                        float* __restrict__ kth, const int* __restrict__ blk_base,
                                                        const int4* __restrict__ nodes, int sub_w,
                                                        int* __restrict__ qkey, int* __restrict__ counts,
                                                        int2* __restrict__ pos) {
  extern __shared__ float s_start[];
  const int ntree = start_tree_n(top.h, D);
  float* s_split = s_start;
  float* s_rows = s_start + ntree;  // [kStartQ][D + 1] (odd stride: conflict-free row reads)
  for (int i = threadIdx.x; i < ntree; i += blockDim.x) s_split[i] = __ldg(top.split + i);
  const int stride = D + 1;
  for (long long c0 = (long long)blockIdx.x * kStartQ; c0 < m; c0 += (long long)gridDim.x * kStartQ) {
    const int nq = (int)min((long long)kStartQ, m - c0);
    __syncthreads();  // previous chunk's rows consumed (and the tree staged)
    const float* src = q + c0 * D;
    const int nf = nq * D;
    if (((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (nf & 3) == 0) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      for (int t = threadIdx.x; t < nf / 4; t += blockDim.x) {
        const float4 v = __ldg(s4 + t);
        const int e = 4 * t;
        s_rows[(e / D) * stride + e % D] = v.x;
        s_rows[((e + 1) / D) * stride + (e + 1) % D] = v.y;
        s_rows[((e + 2) / D) * stride + (e + 2) % D] = v.z;
        s_rows[((e + 3) / D) * stride + (e + 3) % D] = v.w;
      }
    } else {
      for (int t = threadIdx.x; t < nf; t += blockDim.x) s_rows[(t / D) * stride + t % D] = __ldg(src + t);
    }
    // EMPTY top-k rows of the chunk: one contiguous block of nq * k keys
    uint64_t* kp = keys + c0 * k;
    for (int t = threadIdx.x; t < nq * k; t += blockDim.x) kp[t] = kEmptyKey;
    __syncthreads();
    if (threadIdx.x >= nq) continue;
    const long long i = c0 + threadIdx.x;
    const float* row = s_rows + threadIdx.x * stride;
    auto qget = [row](int j) { return row[j]; };
    uint32_t leaf = 0, pend = 0;
    if (ntree) descend_with(top.h, top.d, [s_split](uint32_t node) { return s_split[node]; }, qget, leaf, pend, 0);
    else descend(top, qget, leaf, pend, 0);
    kth[i] = __int_as_float(0x7f800000);
    state[i] = (pend << 16) | leaf;
    next[i] = (int)leaf;
    visits[i] = 1;
    if (seq_log) {
      unsigned long long p = atomicAdd(seq_pos, 1ull);
      if ((long long)p < seq_cap) {
        seq_log[3 * p] = (int)i; seq_log[3 * p + 1] = 1; seq_log[3 * p + 2] = (int)leaf;
      }
    }
    // home bucket: (leaf, block of the leaf the query falls in) -- the home
    // bucket is ordered by position and each tile's scan starts at its block
    int sub = 0;
    if (sub_w > 1) {
      const int b0 = __ldg(blk_base + leaf), nb = __ldg(blk_base + leaf + 1) - b0;
      if (nb > 1) {
        const int4* nd = nodes + (b0 - (int)leaf);
        int c = 0;
        for (;;) {
          const int4 v = __ldg(nd + c);
          c = (row[v.y] >= __int_as_float(v.x)) ? v.w : v.z;
          if (c < 0) break;
        }
        sub = (~c) >> home_block_shift(nb, sub_w);
      }
    }
    const int key = (int)leaf * sub_w + sub;
    qkey[i] = key;
    pos[i] = make_int2((int)leaf, warp_reserve(counts, key));  // position i = query i in the home round
  }
}

// Block-wide exclusive scan of (a, b) over kPlanThreads threads.
__device__ __forceinline__ void block_scan2(long long& a, long long& b, long long& tot_a, long long& tot_b) {
  __shared__ long long wa[32], wb[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long ta = __shfl_up_sync(0xffffffffu, ia, o);
    long long tb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) { ia += ta; ib += tb; }
  }
  if (lane == 31) { wa[w] = ia; wb[w] = ib; }
  __syncthreads();
  if (w == 0) {
    long long xa = (lane < (int)(blockDim.x >> 5)) ? wa[lane] : 0;
    long long xb = (lane < (int)(blockDim.x >> 5)) ? wb[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long ta = __shfl_up_sync(0xffffffffu, xa, o);
      long long tb = __shfl_up_sync(0xffffffffu, xb, o);
      if (lane >= o) { xa += ta; xb += tb; }
    }
    wa[lane] = xa; wb[lane] = xb;
  }
  __syncthreads();
  long long pa = (w > 0) ? wa[w - 1] : 0, pb = (w > 0) ? wb[w - 1] : 0;
  tot_a = wa[31]; tot_b = wb[31];
  a = pa + ia - a;  // exclusive
  b = pb + ib - b;
  __syncthreads();
}

// counts -> key_off, leaf_off, tile_off; resets counts; updates ctl.  One CTA
// of kPlanThreads threads; each thread owns a contiguous run of keys (phase 1)
// and of leaves (phase 2).  The per-tile records are written by scatter_kernel.
__global__ void __launch_bounds__(kPlanThreads) plan_kernel(int* __restrict__ counts, int* __restrict__ key_off,
                                                            int sub_w, int nkeys,
                                                            int* __restrict__ leaf_off, int* __restrict__ tile_off,
                                                            RoundCtl* ctl, int nl, int tile_q, int* hist,
                                                            int hist_cap, RoundCtl* mirror) {
  long long tot_c, tot_t;
  {
    const int per = (nkeys + kPlanThreads - 1) / kPlanThreads;
    const int lo = min(nkeys, (int)threadIdx.x * per), hi = min(nkeys, lo + per);
    long long sc = 0, dummy = 0, tot_dummy;
    for (int e = lo; e < hi; ++e) sc += counts[e];
    long long ec = sc;
    block_scan2(ec, dummy, tot_c, tot_dummy);
    for (int e = lo; e < hi; ++e) {
      key_off[e] = (int)ec;
      ec += counts[e];
      counts[e] = 0;
    }
    if (threadIdx.x == 0) key_off[nkeys] = (int)tot_c;
  }
  __syncthreads();
  const int per = (nl + kPlanThreads - 1) / kPlanThreads;
  const int lo = min(nl, (int)threadIdx.x * per), hi = min(nl, lo + per);
  long long st = 0;
  for (int l = lo; l < hi; ++l) {
    int c = key_off[(l + 1) * sub_w] - key_off[l * sub_w];
    st += (c + tile_q - 1) / tile_q;
  }
  long long et = st, dummy = 0, tot_dummy;
  block_scan2(et, dummy, tot_t, tot_dummy);
  for (int l = lo; l < hi; ++l) {
    const int ec = key_off[l * sub_w];
    const int c = key_off[(l + 1) * sub_w] - ec;
    leaf_off[l] = ec;
    tile_off[l] = (int)et;
    et += (c + tile_q - 1) / tile_q;
  }
  if (threadIdx.x == 0) {
    leaf_off[nl] = (int)tot_c;
    tile_off[nl] = (int)tot_t;
    ctl->prev_active = ctl->active;
    ctl->active = (int)tot_c;
    ctl->num_tiles = (int)tot_t;
    ctl->tile_next = 0;
    ctl->plan_seq += 1;
    if (tot_c > 0) {
      if (hist && ctl->rounds < hist_cap) hist[ctl->rounds] = (int)tot_c;
      ctl->rounds += 1;
      ctl->scans += tot_c;
    }
    // the host's copy of this round's control block, written straight into
    // mapped page-locked memory (no copy-engine operation between the round's
    // kernels); the host reads it after the round's event completes, which
    // orders the kernel's writes before the read (no system-scope fence: a
    // stale slot could only hold an older, larger active count, which delays
    // a decision by one check and never ends a search early)
    if (mirror) *mirror = *ctl;
  }
}

// Place every still-active query of the previous work list into its key's
// slice of the new list, at the slot it took when it was counted, and
// write the round's per-tile records {leaf, first work-list slot, query
// count, sub-bucket of the first query (its block for a home-leaf visit)}.
// identity: previous list is 0..prev_active-1.  No atomics.
__global__ void scatter_kernel(const int* __restrict__ prev, int identity, const int2* __restrict__ pos,
                               const int* __restrict__ qkey, const int* __restrict__ key_off,
                               int* __restrict__ work, const RoundCtl* ctl,
                               const int* __restrict__ leaf_off, const int* __restrict__ tile_off, int nl, int sub_w,
                               int tile_q, int4* __restrict__ tiles, int tiles_cap) {
  const int n = ctl->prev_active;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    // position i of the list just scanned: its next leaf and bucket slot were
    // written by position (coalesced), only the store into the new list scatters
    const int2 pr = __ldg(pos + i);
    if (pr.x >= 0) {
      const int qi = identity ? i : __ldg(prev + i);
      const int key = identity ? __ldg(qkey + i) : pr.x;  // home round: (leaf, block) keys
      work[__ldg(key_off + key) + pr.y] = qi;
    }
  }
  const int nt = min(ctl->num_tiles, tiles_cap);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += stride) {
    // leaf: last l with tile_off[l] <= t (binary search over nl + 1 offsets)
    int lo = 0, hi = nl;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(tile_off + mid) <= t) lo = mid; else hi = mid;
    }
    const int l = lo, j = t - __ldg(tile_off + l);
    const int ec = __ldg(leaf_off + l), c = __ldg(leaf_off + l + 1) - ec;
    const int p = ec + j * tile_q;
    // sub-bucket of slot p: last e in [l sub_w, (l + 1) sub_w) with key_off[e] <= p
    int e0 = l * sub_w, e1 = e0 + sub_w;
    while (e1 - e0 > 1) {
      const int mid = (e0 + e1) >> 1;
      if (__ldg(key_off + mid) <= p) e0 = mid; else e1 = mid;
    }
    tiles[t] = make_int4(l, p, min(tile_q, c - j * tile_q), e0 - l * sub_w);
  }
}

// plan_kernel + scatter_kernel in one launch for small bucket tables
// (nkeys <= kPsMaxKeys: config 1's 256 leaves): every CTA scans the whole
// count table in shared memory, places its share of the previous list and
// writes its share of the tile records; the last CTA to finish publishes the
// round's control block.  Counts are double-buffered by round parity: this
// round reads `counts` and zeroes `counts_next`, which the round's scan then
// fills (it was last read by the previous round's launch).
constexpr int kPsMaxKeys = 4096;
constexpr int kPsThreads = 512;
__global__ void __launch_bounds__(kPsThreads) plan_scatter_kernel(
    const int* __restrict__ counts, int* __restrict__ counts_next, int* __restrict__ key_off_g, int sub_w, int nkeys,
    int* __restrict__ leaf_off_g, int* __restrict__ tile_off_g, RoundCtl* ctl, int nl, int tile_q, int* hist,
    int hist_cap, RoundCtl* mirror, const int* __restrict__ prev, int identity, const int2* __restrict__ pos,
    const int* __restrict__ qkey, int* __restrict__ work, int4* __restrict__ tiles, int tiles_cap) {
  __shared__ int s_key_off[kPsMaxKeys + 1];
  __shared__ int s_tile_off[kPsMaxKeys + 1];
  __shared__ int s_tot[2];
  __shared__ bool s_last;
  // programmatic dependent launch (engine.cu fused rounds): the previous
  // scan's results are read only after this wait (a no-op for a normal launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int n_prev = ctl->active;  // read before this launch's last CTA rewrites it
  // exclusive scans of the counts (per key) and of the tiles (per leaf)
  {
    const int per = (nkeys + kPsThreads - 1) / kPsThreads;
    const int lo = min(nkeys, (int)threadIdx.x * per), hi = min(nkeys, lo + per);
    long long sc = 0, dummy = 0, tot_c, tot_dummy;
    for (int e = lo; e < hi; ++e) sc += __ldg(counts + e);
    long long ec = sc;
    block_scan2(ec, dummy, tot_c, tot_dummy);
    for (int e = lo; e < hi; ++e) {
      s_key_off[e] = (int)ec;
      ec += __ldg(counts + e);
    }
    if (threadIdx.x == 0) {
      s_key_off[nkeys] = (int)tot_c;
      s_tot[0] = (int)tot_c;
    }
  }
  __syncthreads();
  {
    const int per = (nl + kPsThreads - 1) / kPsThreads;
    const int lo = min(nl, (int)threadIdx.x * per), hi = min(nl, lo + per);
    long long st = 0;
    for (int l = lo; l < hi; ++l) st += (s_key_off[(l + 1) * sub_w] - s_key_off[l * sub_w] + tile_q - 1) / tile_q;
    long long et = st, dummy = 0, tot_t, tot_dummy;
    block_scan2(et, dummy, tot_t, tot_dummy);
    for (int l = lo; l < hi; ++l) {
      s_tile_off[l] = (int)et;
      et += (s_key_off[(l + 1) * sub_w] - s_key_off[l * sub_w] + tile_q - 1) / tile_q;
    }
    if (threadIdx.x == 0) {
      s_tile_off[nl] = (int)tot_t;
      s_tot[1] = (int)tot_t;
    }
  }
  __syncthreads();
  const int stride = gridDim.x * blockDim.x;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e <= nkeys; e += blockDim.x) key_off_g[e] = s_key_off[e];
    for (int l = threadIdx.x; l <= nl; l += blockDim.x) {
      tile_off_g[l] = s_tile_off[l];
      leaf_off_g[l] = s_key_off[l * sub_w];
    }
  }
  for (int e = gtid; e < nkeys; e += stride) counts_next[e] = 0;
  for (int i = gtid; i < n_prev; i += stride) {
    const int2 pr = __ldg(pos + i);
    if (pr.x >= 0) {
      const int qi = identity ? i : __ldg(prev + i);
      const int key = identity ? __ldg(qkey + i) : pr.x;
      work[s_key_off[key] + pr.y] = qi;
    }
  }
  const int nt = min(s_tot[1], tiles_cap);
  for (int t = gtid; t < nt; t += stride) {
    int lo = 0, hi = nl;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_tile_off[mid] <= t) lo = mid; else hi = mid;
    }
    const int l = lo, j = t - s_tile_off[l];
    const int ec = s_key_off[l * sub_w], c = s_key_off[(l + 1) * sub_w] - ec;
    const int p = ec + j * tile_q;
    int e0 = l * sub_w, e1 = e0 + sub_w;
    while (e1 - e0 > 1) {
      const int mid = (e0 + e1) >> 1;
      if (s_key_off[mid] <= p) e0 = mid; else e1 = mid;
    }
    tiles[t] = make_int4(l, p, min(tile_q, c - j * tile_q), e0 - l * sub_w);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&ctl->ps_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    const int tot_c = s_tot[0], tot_t = s_tot[1];
    ctl->ps_done = 0;
    ctl->prev_active = n_prev;
    ctl->active = tot_c;
    ctl->num_tiles = tot_t;
    ctl->tile_next = 0;
    ctl->plan_seq += 1;
    if (tot_c > 0) {
      if (hist && ctl->rounds < hist_cap) hist[ctl->rounds] = tot_c;
      ctl->rounds += 1;
      ctl->scans += tot_c;
    }
    __threadfence();
    if (mirror) *mirror = *ctl;
  }
}

// Unfused FindLeaf over this round's work list (out-of-core rounds, where a
// leaf may be split across chunk passes).  buffer_tree.py:292-378.
__global__ void findleaf_kernel(const int* __restrict__ work, const RoundCtl* ctl, const float* __restrict__ q,
                                int D, int k, TopTreeView top, const uint64_t* __restrict__ keys,
                                uint32_t* __restrict__ state, int* __restrict__ next, uint32_t* __restrict__ visits,
                                int* __restrict__ counts, int2* __restrict__ pos, int* seq_log,
                                unsigned long long* seq_pos, long long seq_cap, int leaf_lo = 0,
                                int leaf_hi = -1, int* __restrict__ park = nullptr, int* park_n = nullptr) {
  // the top tree's split values in shared memory when they fit (dynamic smem)
  extern __shared__ float s_fl_split[];
  const int ntree = start_tree_smem(top.h);
  for (int i = threadIdx.x; i < ntree; i += blockDim.x) s_fl_split[i] = __ldg(top.split + i);
  __syncthreads();
  const int n = ctl->active;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int qi = work[i];
    const float* qp = q + (long long)qi * D;
    auto qget = [qp](int j) { return __ldg(qp + j); };
    float kth = key_dist(keys[(long long)qi * k + k - 1]);
    uint32_t st = state[qi];
    uint32_t lf = st & 0xFFFFu, pend = st >> 16;
    int nxt;
    if (ntree) nxt = find_next_leaf_with(top.h, top.d, [](uint32_t node) { return s_fl_split[node]; }, qget, kth, lf, pend);
    else nxt = find_next_leaf(top, qget, kth, lf, pend);
    state[qi] = (pend << 16) | lf;
    next[qi] = nxt;
    int rk = 0;
    if (nxt >= 0) {
      uint32_t v = visits[qi] + 1;
      visits[qi] = v;
      if (seq_log) {
        unsigned long long p = atomicAdd(seq_pos, 1ull);
        if ((long long)p < seq_cap) {
          seq_log[3 * p] = qi; seq_log[3 * p + 1] = (int)v; seq_log[3 * p + 2] = nxt;
        }
      }
    }
    // out-of-core drain (park != null): a next leaf outside the resident unit
    // parks the query for a later unit
    const bool parked = park && nxt >= 0 && (nxt < leaf_lo || nxt > leaf_hi);
    if (park) park_append(parked, qi, park, park_n);
    if (nxt >= 0 && !parked) rk = warp_reserve(counts, nxt);  // next round's bucket (key = leaf) and slot
    pos[i] = make_int2(parked ? -1 : nxt, rk);
  }
}

// Query renumbering (engine.cu search_batch): the batch is searched in home-
// bucket order -- query j of the search is query perm[j] of the caller -- so
// that queries with neighbouring ids are spatial neighbours and the per-query
// arrays of every round are read in runs instead of scattered sectors.
__global__ void gather_rows_kernel(const float* __restrict__ src, const int* __restrict__ perm, int D, long long m,
                                   float* __restrict__ dst) {
  const long long total = m * D;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long j = t / D;
    dst[t] = __ldg(src + (long long)__ldg(perm + j) * D + (t - j * D));
  }
}
__global__ void unpermute_keys_kernel(const uint64_t* __restrict__ src, const int* __restrict__ perm, int k, long long m,
                                      uint64_t* __restrict__ dst) {
  const long long total = m * k;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long j = t / k;
    dst[(long long)__ldg(perm + j) * k + (t - j * k)] = src[t];
  }
}
__global__ void unpermute_u32_kernel(const uint32_t* __restrict__ src, const int* __restrict__ perm, long long m,
                                     uint32_t* __restrict__ dst) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < m; j += (long long)gridDim.x * blockDim.x)
    dst[__ldg(perm + j)] = src[j];
}
__global__ void remap_seq_kernel(int* seq_log, const unsigned long long* seq_pos, long long seq_cap,
                                 const int* __restrict__ perm) {
  const long long n = min((long long)*seq_pos, seq_cap);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    seq_log[3 * p] = __ldg(perm + seq_log[3 * p]);
}

// m x d host layout -> m x D kernel layout (zero padded; exact: +0 dims add 0).
__global__ void pad_rows_kernel(const float* __restrict__ src, int d, float* __restrict__ dst, int D, long long m) {
  long long total = m * D;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    long long i = t / D;
    int j = (int)(t - i * D);
    dst[t] = (j < d) ? src[i * d + j] : 0.0f;
  }
}

// Tail finisher.  Warp w takes the queries work[w], work[w + W], ... of the
// round just scanned (length ctl->active); a query with a next leaf runs
// the rest of its traversal here: scan the leaf (lanes stride over its
// quads, reference arithmetic core.py:108-122, FMA variant when !exact),
// insert every candidate whose key beats the current k-th key into the
// warp's sorted top-k row (shared memory), then FindLeaf with the new k-th
// distance (buffer_tree.py:330-349) -- the same per-visit semantics as a
// round (the top-k after a visit is the best k of the list and the leaf), so
// results, visit counts, pairs and leaf sequences are unchanged.
constexpr int kFinishWarps = 8;
// Finishers inside an out-of-core drain walk only the resident unit's leaves
// (pts/pidx hold quads [origin, ...)); a query whose next leaf lies outside
// it keeps that leaf in next[] and is parked.  Default: the whole structure.
struct FinishUnit {
  long long origin = 0;
  int leaf_lo = 0, leaf_hi = 0x7fffffff;
  int* park = nullptr;
  int* park_n = nullptr;
  float* kth = nullptr;  // per-query k-th distance kept by the tensor-core scan (drain)
};

template <bool FMA>
__global__ void __launch_bounds__(kFinishWarps * 32) finish_kernel(
    const int* __restrict__ work, RoundCtl* ctl, const float* __restrict__ q, int D, int k, TopTreeView top,
    uint64_t* __restrict__ keys, uint32_t* __restrict__ state, int* __restrict__ next, uint32_t* __restrict__ visits,
    const float* __restrict__ pts, const uint32_t* __restrict__ pidx, const long long* __restrict__ quad_base,
    const int* __restrict__ leaf_size, unsigned long long* pairs, int* seq_log, unsigned long long* seq_pos,
    long long seq_cap, FinishUnit fu) {
  __shared__ uint64_t s_row[kFinishWarps][64];
  __shared__ float s_q[kFinishWarps][32];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int d = top.d;
  uint64_t* row = s_row[wl];
  float* sq = s_q[wl];
  const int n = ctl->active;
  const int nw = gridDim.x * kFinishWarps;
  unsigned long long pairs_acc = 0, scans_acc = 0;
  for (int i = blockIdx.x * kFinishWarps + wl; i < n; i += nw) {
    const int qi = __ldg(work + i);
    int leaf = next[qi];
    if (leaf < 0) continue;
    if (lane < d) sq[lane] = __ldg(q + (long long)qi * D + lane);
    uint64_t* kp = keys + (long long)qi * k;
    for (int j = lane; j < k; j += 32) row[j] = kp[j];
    __syncwarp();
    float qv[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) qv[j] = j < d ? sq[j] : 0.0f;
    uint32_t st = state[qi];
    uint32_t lf = st & 0xFFFFu, pend = st >> 16;
    uint32_t vis = visits[qi];
    while (leaf >= fu.leaf_lo && leaf <= fu.leaf_hi) {
      const long long g0 = __ldg(quad_base + leaf), g1 = __ldg(quad_base + leaf + 1);
      uint64_t kkey = row[k - 1];
      for (long long gb = g0; gb < g1; gb += 32) {
        const long long g = gb + lane;
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        bool has = g < g1;
        if (has) {
          const float4* pq = reinterpret_cast<const float4*>(pts + (g - fu.origin) * 4 * D);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
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
          // candidates: keys below the current k-th key (ties by original index)
          const uint64_t key = has ? pack_key(acc[t], __ldg(pidx + (g - fu.origin) * 4 + t)) : ~0ull;
          unsigned bal = __ballot_sync(0xffffffffu, key < kkey);
          while (bal) {
            const int src = __ffs(bal) - 1;
            bal &= bal - 1;
            const uint64_t c = __shfl_sync(0xffffffffu, key, src);
            if (lane == 0 && c < row[k - 1]) {
              int j = k - 1;
              while (j > 0 && row[j - 1] > c) {
                row[j] = row[j - 1];
                --j;
              }
              row[j] = c;
            }
            __syncwarp();
            kkey = row[k - 1];
          }
        }
      }
      pairs_acc += (unsigned long long)__ldg(leaf_size + leaf);
      scans_acc += 1;
      // FindLeaf with the k-th distance after this leaf (every lane computes it)
      const float kth = key_dist(row[k - 1]);
      const float* sp = top.split;
      leaf = find_next_leaf_with(top.h, d, [sp](uint32_t node) { return __ldg(sp + node); },
                                 [sq](int j) { return sq[j]; }, kth, lf, pend);
      if (leaf >= 0) {
        ++vis;
        if (seq_log && lane == 0) {
          const unsigned long long p = atomicAdd(seq_pos, 1ull);
          if ((long long)p < seq_cap) {
            seq_log[3 * p] = qi; seq_log[3 * p + 1] = (int)vis; seq_log[3 * p + 2] = leaf;
          }
        }
      }
    }
    for (int j = lane; j < k; j += 32) kp[j] = row[j];
    if (lane == 0) {
      state[qi] = (pend << 16) | lf;
      next[qi] = leaf < 0 ? -1 : leaf;
      visits[qi] = vis;
      if (leaf >= 0) fu.park[atomicAdd(fu.park_n, 1)] = qi;  // left the resident unit
      if (fu.kth) fu.kth[qi] = key_dist(row[k - 1]);
    }
    __syncwarp();
  }
  if (lane == 0 && (pairs_acc || scans_acc)) {
    if (pairs) atomicAdd(pairs, pairs_acc);
    atomicAdd(reinterpret_cast<unsigned long long*>(&ctl->scans), scans_acc);
  }
}

// Tail finisher, one CTA per query: the leaf's quads are spread over the
// CTA's threads (one quad each per slice), candidates below the current k-th
// key are appended to a shared list and inserted by thread 0 after each
// slice; thread 0 runs FindLeaf.  Same per-visit semantics as finish_kernel,
// a quarter of its per-leaf latency for long leaves.
constexpr int kFinishT = 256;
template <bool FMA>
__global__ void __launch_bounds__(kFinishT) finish_cta_kernel(
    const int* __restrict__ work, RoundCtl* ctl, const float* __restrict__ q, int D, int k, TopTreeView top,
    uint64_t* __restrict__ keys, uint32_t* __restrict__ state, int* __restrict__ next, uint32_t* __restrict__ visits,
    const float* __restrict__ pts, const uint32_t* __restrict__ pidx, const long long* __restrict__ quad_base,
    const int* __restrict__ leaf_size, unsigned long long* pairs, int* seq_log, unsigned long long* seq_pos,
    long long seq_cap, FinishUnit fu) {
  __shared__ uint64_t s_row[64];
  __shared__ float s_q[32];
  __shared__ uint64_t s_cand[kFinishT * 4];
  __shared__ int s_nc, s_leaf;
  const int tid = threadIdx.x;
  const int d = top.d;
  const int n = ctl->active;
  unsigned long long pairs_acc = 0, scans_acc = 0;
  if (tid == 0) s_nc = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int qi = __ldg(work + i);
    int leaf = next[qi];
    __syncthreads();  // the previous query's shared state is no longer read
    if (leaf < 0) continue;
    if (tid < d) s_q[tid] = __ldg(q + (long long)qi * D + tid);
    uint64_t* kp = keys + (long long)qi * k;
    if (tid < k) s_row[tid] = kp[tid];
    __syncthreads();
    float qv[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) qv[j] = j < d ? s_q[j] : 0.0f;
    uint32_t lf = 0, pend = 0, vis = 0;
    if (tid == 0) {
      const uint32_t st = state[qi];
      lf = st & 0xFFFFu;
      pend = st >> 16;
      vis = visits[qi];
    }
    while (leaf >= fu.leaf_lo && leaf <= fu.leaf_hi) {
      const long long g0 = __ldg(quad_base + leaf), g1 = __ldg(quad_base + leaf + 1);
      for (long long gb = g0; gb < g1; gb += kFinishT) {
        const uint64_t kkey = s_row[k - 1];
        const long long g = gb + tid;
        if (g < g1) {
          float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
          const float4* pq = reinterpret_cast<const float4*>(pts + (g - fu.origin) * 4 * D);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
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
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint64_t key = pack_key(acc[t], __ldg(pidx + (g - fu.origin) * 4 + t));
            if (key < kkey) s_cand[atomicAdd(&s_nc, 1)] = key;
          }
        }
        __syncthreads();
        if (tid == 0) {
          // insert every candidate that beats the current k-th key (any order:
          // the result is the best k of the list and the candidates)
          const int nc = s_nc;
          for (int c = 0; c < nc; ++c) {
            const uint64_t ck = s_cand[c];
            if (ck < s_row[k - 1]) {
              int j = k - 1;
              while (j > 0 && s_row[j - 1] > ck) {
                s_row[j] = s_row[j - 1];
                --j;
              }
              s_row[j] = ck;
            }
          }
          s_nc = 0;
        }
        __syncthreads();
      }
      if (tid == 0) {
        pairs_acc += (unsigned long long)__ldg(leaf_size + leaf);
        scans_acc += 1;
        // FindLeaf with the k-th distance after this leaf
        const float kth = key_dist(s_row[k - 1]);
        const float* sp = top.split;
        const int nxt = find_next_leaf_with(top.h, d, [sp](uint32_t node) { return __ldg(sp + node); },
                                            [](int j) { return s_q[j]; }, kth, lf, pend);
        if (nxt >= 0) {
          ++vis;
          if (seq_log) {
            const unsigned long long p = atomicAdd(seq_pos, 1ull);
            if ((long long)p < seq_cap) {
              seq_log[3 * p] = qi; seq_log[3 * p + 1] = (int)vis; seq_log[3 * p + 2] = nxt;
            }
          }
        }
        s_leaf = nxt;
      }
      __syncthreads();
      leaf = s_leaf;
    }
    if (tid < k) kp[tid] = s_row[tid];
    if (tid == 0) {
      state[qi] = (pend << 16) | lf;
      next[qi] = leaf < 0 ? -1 : leaf;
      visits[qi] = vis;
      if (leaf >= 0) fu.park[atomicAdd(fu.park_n, 1)] = qi;  // left the resident unit
      if (fu.kth) fu.kth[qi] = key_dist(s_row[k - 1]);
    }
  }
  if (tid == 0 && (pairs_acc || scans_acc)) {
    if (pairs) atomicAdd(pairs, pairs_acc);
    atomicAdd(reinterpret_cast<unsigned long long*>(&ctl->scans), scans_acc);
  }
}

}  // namespace bkt
