// build_tree.cpp -- native host build of the buffer k-d tree (bkt_build_tree).
//
// Replaces build_buffer_tree's split loop (reference buffer_tree.py:149-197)
// and median_split (kdtree.py:55-70): level by level, every subset is cut at
// the positional median of coordinate (depth % d) under the total order
// key = order_bits(coord) << 32 | original_index (kdtree.py:46-52, 66-70); the
// split value is the coordinate of the element at position s//2, which goes
// right.  nth_element on the unique packed keys yields exactly the reference's
// left/right sets; the order inside a leaf is not part of the contract.
// Subsets of one level are independent and are split on parallel threads.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bkt.h"

namespace {

inline uint32_t order_bits(float v) {
  uint32_t b;
  std::memcpy(&b, &v, 4);
  return (b & 0x80000000u) ? ~b : (b ^ 0x80000000u);
}

}  // namespace

extern "C" int bkt_build_tree(const float* refs, int64_t n, int32_t d, int32_t h, float* split_out,
                              int64_t* order_out, int64_t* leaf_starts_out, int32_t nthreads) {
  if (!refs || !split_out || !order_out || !leaf_starts_out) return BKT_EINVAL;
  if (h < 1 || h > 30 || d < 1) return BKT_EINVAL;
  if (n < (int64_t(1) << h) || n >= int64_t(0xFFFFFFFFll)) return BKT_EINVAL;
  if (nthreads < 1) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());

  std::vector<uint64_t> keys((size_t)n);
  std::vector<int64_t> starts{0, n}, nstarts;
  // keys carry the original index in their low 32 bits; the high half is
  // refreshed for the split dimension of each level
  for (int64_t i = 0; i < n; ++i) keys[i] = (uint64_t)i;

  int64_t node = 0;
  for (int depth = 0; depth < h; ++depth) {
    const int dim = depth % d;
    const int64_t nsub = (int64_t)starts.size() - 1;
    nstarts.assign(2 * nsub + 1, 0);
    std::vector<float> sv((size_t)nsub);
    std::atomic<int64_t> next_sub{0};
    auto work = [&]() {
      for (;;) {
        int64_t s = next_sub.fetch_add(1);
        if (s >= nsub) break;
        const int64_t lo = starts[s], hi = starts[s + 1], mid = (hi - lo) / 2;
        uint64_t* k = keys.data() + lo;
        for (int64_t t = 0; t < hi - lo; ++t) {
          uint32_t idx = (uint32_t)(k[t] & 0xFFFFFFFFull);
          k[t] = ((uint64_t)order_bits(refs[(int64_t)idx * d + dim]) << 32) | idx;
        }
        std::nth_element(k, k + mid, k + (hi - lo));
        uint32_t med = (uint32_t)(k[mid] & 0xFFFFFFFFull);
        sv[s] = refs[(int64_t)med * d + dim];
        nstarts[2 * s] = lo;
        nstarts[2 * s + 1] = lo + mid;
      }
    };
    const int nt = (int)std::min<int64_t>(nthreads, nsub);
    if (nt <= 1) {
      work();
    } else {
      std::vector<std::thread> th;
      for (int w = 0; w < nt; ++w) th.emplace_back(work);
      for (auto& t : th) t.join();
    }
    nstarts[2 * nsub] = n;
    for (int64_t s = 0; s < nsub; ++s) split_out[node++] = sv[s];
    starts.swap(nstarts);
  }
  for (int64_t i = 0; i < n; ++i) order_out[i] = (int64_t)(keys[i] & 0xFFFFFFFFull);
  std::memcpy(leaf_starts_out, starts.data(), sizeof(int64_t) * starts.size());
  return BKT_OK;
}
