// dims.h -- kernel dimensionalities compiled ahead of time.  Data of any other
// d <= 32 runs on the next larger kernel D with zero-padded coordinates
// (a +0 dimension adds exactly 0 to the accumulator, so results are unchanged).
#pragma once
#include <cuda_runtime.h>
#include "leafscan.cuh"

#define BKT_DIM_LIST(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) \
  X(20) X(24) X(27) X(28) X(32)

// top-k register buckets: k is served by the smallest KB >= k
#define BKT_KB_LIST(X) X(1) X(2) X(4) X(8) X(10) X(16) X(32) X(64)

namespace bkt {
constexpr int kMaxKernelDim = 32;
constexpr int kMaxK = 64;
// occ != nullptr: only report max resident CTAs per SM, do not launch.
#define BKT_DECL_LAUNCH(D) \
  cudaError_t launch_leafscan_d##D(int kb, bool fma, int grid, cudaStream_t s, const ScanArgs& a, int* occ);
BKT_DIM_LIST(BKT_DECL_LAUNCH)
#undef BKT_DECL_LAUNCH
}  // namespace bkt
