// leafscan_tc_inst.cu -- instantiates the tensor-core leaf filter kernel for
// K tiles of 16 and 32 (d + 1 <= KT) and every top-k bucket.
#include <atomic>

#include "dims.h"
#include "leafscan_tc.cuh"

namespace bkt {
namespace {
template <int KT, int KB, bool FMA, int NR>
cudaError_t launch_tc_one(int grid, cudaStream_t s, const TcArgs& a, int* occ) {
  auto fn = leafscan_tc_kernel<KT, KB, FMA, NR>;
  // at least 76 KB so that no more than two CTAs (2 x 256 TMEM columns) share an SM
  constexpr int smem = TcSmem<KT, NR>::kBytes > 78 * 1024 ? TcSmem<KT, NR>::kBytes : 78 * 1024;
  // function attributes are per device: set them once per (instantiation, device)
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, kTcThreads, smem);
  fn<<<grid, kTcThreads, smem, s>>>(a);
  return cudaGetLastError();
}
template <int KT, int NR>
cudaError_t launch_tc_kt(int kb, bool fma, int grid, cudaStream_t s, const TcArgs& a, int* occ) {
  switch (kb) {
#define BKT_CASE(KB) \
  case KB:           \
    return fma ? launch_tc_one<KT, KB, true, NR>(grid, s, a, occ) : launch_tc_one<KT, KB, false, NR>(grid, s, a, occ);
    BKT_KB_LIST(BKT_CASE)
#undef BKT_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
}  // namespace

cudaError_t launch_leafscan_tc(int kt, int kb, bool fma, int grid, cudaStream_t s, const TcArgs& a, int* occ,
                               int nr) {
  if (nr == 128) {
    if (kt == 16) return launch_tc_kt<16, 128>(kb, fma, grid, s, a, occ);
    if (kt == 32) return launch_tc_kt<32, 128>(kb, fma, grid, s, a, occ);
  } else {
    if (kt == 16) return launch_tc_kt<16, 64>(kb, fma, grid, s, a, occ);
    if (kt == 32) return launch_tc_kt<32, 64>(kb, fma, grid, s, a, occ);
  }
  return cudaErrorInvalidValue;
}
}  // namespace bkt
