// bkt_device.cuh -- device-side building blocks for the sm_100a buffer k-d tree engine.
//
// Numeric contract (reference core.py:1-13, 108-160):
//   * squared distance acc = sum_j (q_j - p_j)^2 accumulated left to right in
//     float32.  "exact" mode reproduces the reference's two roundings per
//     dimension bit for bit; "fma" mode fuses the multiply-add (one rounding).
//   * candidates are ordered by the packed key (f32 bits << 32) | orig_index
//     (core.py:152-160); EMPTY_KEY = (inf bits << 32) | 0xFFFFFFFF (core.py:45).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bkt {

constexpr uint64_t kEmptyKey = 0x7F800000FFFFFFFFull;
constexpr uint32_t kIndexSentinel = 0xFFFFFFFFu;
constexpr int kMaxHeight = 16;   // state packs path + pending mask in 2 x 16 bits
constexpr int kMaxWideHeight = 30;  // wide path (wide_search.cuh): path + pending mask in 2 x 32 bits

// ----------------------------------------------------------------------------
// packed float32x2 arithmetic (sm_100a FADD2 / FFMA2; one issue slot, two lanes)
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float f2_lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2_hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t f2_splat(float x) {
  uint32_t b = __float_as_uint(x);
  return ((uint64_t)b << 32) | b;
}

// One dimension of the distance recurrence for two points at once.
//   exact: sq = RN(diff*diff) computed as fma(diff, diff, +0) -- the +0 comes
//          from a runtime value so ptxas cannot contract it with the following
//          add (ptxas 12.9 fuses mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even
//          under --fmad=false, which would break bit-exactness).  RN(d*d + 0)
//          == RN(d*d) for every finite or infinite d.
//   fma:   acc = RN(diff*diff + acc).
template <bool FMA>
__device__ __forceinline__ uint64_t dist_step(uint64_t acc, uint64_t qq, uint64_t pp, uint64_t zero) {
  uint64_t d = f2_sub(qq, pp);
  if constexpr (FMA) {
    return f2_fma(d, d, acc);
  } else {
    return f2_add(acc, f2_fma(d, d, zero));
  }
}

__device__ __forceinline__ uint64_t pack_key(float dist, uint32_t idx) {
  return ((uint64_t)__float_as_uint(dist) << 32) | idx;
}
__device__ __forceinline__ float key_dist(uint64_t key) { return __uint_as_float((uint32_t)(key >> 32)); }

// Top-k kept in registers, DESCENDING: arr[0] is the current k-th best key
// (the pruning radius), arr[k..KB) hold sentinel 0 keys that never leave.
// Precondition: c < arr[0].  Evicts arr[0] and inserts c in order.
template <int KB>
__device__ __forceinline__ void topk_insert(uint64_t (&arr)[KB], uint64_t c) {
#pragma unroll
  for (int i = 0; i < KB - 1; ++i) {
    uint64_t nxt = arr[i + 1];
    uint64_t cur = arr[i];
    arr[i] = (nxt > c) ? nxt : ((cur > c) ? c : cur);
  }
  arr[KB - 1] = (arr[KB - 1] > c) ? c : arr[KB - 1];
}

// ----------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA 1-D), CTA scope
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// Blocks until the barrier's phase `phase` has completed.  The suspend-time
// hint lets the hardware park the warp until the phase flips instead of
// spinning (a spinning producer warp otherwise steals issue slots from the
// compute warps of its SM).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t a = smem_addr(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(phase), "r"(0x989680u)
        : "memory");
  } while (!ok);
}

// Non-blocking probe: has phase `phase` of the barrier completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

// Spinning variant (no suspend): lowest wake-up latency for warps on the
// critical path of a short producer/consumer loop.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t phase) {
  uint32_t a = smem_addr(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(phase)
        : "memory");
  } while (!ok);
}

// ----------------------------------------------------------------------------
// warp-aggregated atomics
// ----------------------------------------------------------------------------
// Reserve one slot per lane in bucket `key` (lanes sharing a key are combined
// into one atomic by their leader); returns this lane's slot.
__device__ __forceinline__ int warp_reserve(int* cursor, int key) {
  unsigned mask = __activemask();
  unsigned peers = __match_any_sync(mask, key);
  int lane = threadIdx.x & 31;
  int leader = __ffs(peers) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(cursor + key, __popc(peers));
  base = __shfl_sync(peers, base, leader);
  return base + __popc(peers & ((1u << lane) - 1u));
}

// Home-round sub-buckets: a leaf of nb blocks maps block b to sub-bucket
// b >> shift with the smallest shift that fits sub_w sub-buckets (consecutive
// blocks are neighbours, so a coarser bucket stays spatially coherent).
__host__ __device__ __forceinline__ int home_block_shift(int nb, int sub_w) {
  int s = 0;
  while (((nb - 1) >> s) >= sub_w) ++s;
  return s;
}

// ----------------------------------------------------------------------------
// traversal state: bits 0..15 current leaf (root-to-leaf path, depth i at bit
// h-1-i), bits 16..31 pending far-child depths (depth i at bit 16+i).  This is
// the reference's far-child stack (buffer_tree.py:258-276, 340-375) in 4 bytes:
// pushes happen in increasing depth along a descent and pops take the deepest,
// so the stack is exactly the set of pending depths relative to the current
// path, and the far child at depth i is the sibling obtained by flipping bit i.
// ----------------------------------------------------------------------------
struct TopTreeView {
  const float* split;  // 2^h - 1 split values, level order (node j: children 2j+1, 2j+2)
  int h;
  int d;               // real dimensionality (split dim = depth % d, buffer_tree.py:345, 369)
};

// Descend from depth `from` to a leaf along q, pushing every far child
// (buffer_tree.py:365-376: go_left = q[sd] < split, strict; equal goes right).
// SFn(node) returns split value `node` (global or shared memory).
template <typename QFn, typename SFn>
__device__ __forceinline__ void descend_with(int h, int d, SFn sget, QFn qget, uint32_t& leaf, uint32_t& pend,
                                             int from) {
  for (int j = from; j < h; ++j) {
    uint32_t node = (1u << j) - 1u + (leaf >> (h - j));
    float qv = qget(j % d);
    uint32_t right = (qv < sget(node)) ? 0u : 1u;
    uint32_t bit = 1u << (h - 1 - j);
    leaf = (leaf & ~bit) | (right ? bit : 0u);
    pend |= 1u << j;
  }
}

// FindLeaf for a resumed query (buffer_tree.py:330-349): pop the deepest
// pending far child, prune while (q[sd]-split)^2 > kth in float32 (ties are
// visited), descend into the first survivor.  Returns the leaf id or -1 (DONE).
template <typename QFn, typename SFn>
__device__ __forceinline__ int find_next_leaf_with(int h, int d, SFn sget, QFn qget, float kth, uint32_t& leaf,
                                                   uint32_t& pend) {
  while (pend) {
    int di = 31 - __clz(pend);
    pend &= ~(1u << di);
    uint32_t parent = (1u << di) - 1u + (leaf >> (h - di));
    float hp = __fsub_rn(qget(di % d), sget(parent));
    if (!(__fmul_rn(hp, hp) > kth)) {
      leaf ^= 1u << (h - 1 - di);
      descend_with(h, d, sget, qget, leaf, pend, di + 1);
      return (int)leaf;
    }
  }
  return -1;
}

template <typename QFn>
__device__ __forceinline__ void descend(const TopTreeView& T, QFn qget, uint32_t& leaf, uint32_t& pend,
                                        int from) {
  const float* sp = T.split;
  descend_with(T.h, T.d, [sp](uint32_t node) { return __ldg(sp + node); }, qget, leaf, pend, from);
}

template <typename QFn>
__device__ __forceinline__ int find_next_leaf(const TopTreeView& T, QFn qget, float kth, uint32_t& leaf,
                                              uint32_t& pend) {
  const float* sp = T.split;
  return find_next_leaf_with(T.h, T.d, [sp](uint32_t node) { return __ldg(sp + node); }, qget, kth, leaf, pend);
}

}  // namespace bkt
