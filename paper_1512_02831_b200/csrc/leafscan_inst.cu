// leafscan_inst.cu -- compiled once per kernel dimensionality with -DBKT_D=<D>
// (see build.py); instantiates leafscan_kernel<D, KB, FMA> for every top-k bucket.
#include <atomic>

#include "dims.h"

#ifndef BKT_D
#error "compile with -DBKT_D=<dimensionality>"
#endif
#define BKT_CAT_(a, b) a##b
#define BKT_CAT(a, b) BKT_CAT_(a, b)

namespace bkt {
namespace {
template <int KB, bool FMA>
cudaError_t launch_one(int grid, cudaStream_t s, const ScanArgs& a, int* occ) {
  auto fn = leafscan_kernel<BKT_D, KB, FMA>;
  constexpr int smem = ScanSmem<BKT_D>::kBytes;
  // function attributes are per device: set them once per (instantiation, device)
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
    }
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, kThreads, smem);
  fn<<<grid, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}
}  // namespace

cudaError_t BKT_CAT(launch_leafscan_d, BKT_D)(int kb, bool fma, int grid, cudaStream_t s, const ScanArgs& a,
                                              int* occ) {
  switch (kb) {
#define BKT_CASE(KB) \
  case KB:           \
    return fma ? launch_one<KB, true>(grid, s, a, occ) : launch_one<KB, false>(grid, s, a, occ);
    BKT_KB_LIST(BKT_CASE)
#undef BKT_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
}  // namespace bkt
