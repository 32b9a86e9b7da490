// split_launch.cuh -- launch wrappers of the split (leaf, window) rounds (split_scan.cuh).
// Included by engine.cu only (round_kernels.cuh defines non-template kernels).
#pragma once
#include <atomic>

#include "split_scan.cuh"

namespace bkt {

inline cudaError_t launch_splitscan_one(int grid, cudaStream_t s, const SplitScanArgs& a, bool configure_only = false) {
  auto fn = splitscan_tc_kernel;
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SplitSmem::kBytes);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  if (configure_only) return cudaSuccess;
  fn<<<grid, kSplitThreads, SplitSmem::kBytes, s>>>(a);
  return cudaGetLastError();
}

// kernel attributes of the split rounds' kernels, set outside any stream capture
inline cudaError_t configure_split_kernels(bool fma, int kb, int h, int d) {
  (void)fma;
  SplitScanArgs dummy{};
  cudaError_t e = launch_splitscan_one(0, nullptr, dummy, true);
  if (e != cudaSuccess) return e;
  const int smem = advance_smem_bytes(h, d);
  if (smem <= 48 * 1024) return cudaSuccess;
  switch (kb) {
#define BKT_CASE(KB) \
  case KB:           \
    return cudaFuncSetAttribute(advance_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    BKT_KB_LIST(BKT_CASE)
#undef BKT_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

// (the split scan has no arithmetic mode: survivors are evaluated in advance_kernel)
inline cudaError_t launch_splitscan(bool /*fma*/, int grid, cudaStream_t s, const SplitScanArgs& a) {
  return launch_splitscan_one(grid, s, a);
}

template <int KB>
inline cudaError_t launch_advance_kb(int grid, cudaStream_t s, const AdvanceArgs& a) {
  const int smem = advance_smem_bytes(a.top.h, a.top.d);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(advance_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  advance_kernel<KB><<<grid, kAdvThreads, smem, s>>>(a);
  return cudaGetLastError();
}

inline cudaError_t launch_advance(int kb, int grid, cudaStream_t s, const AdvanceArgs& a) {
  switch (kb) {
#define BKT_CASE(KB) \
  case KB:           \
    return launch_advance_kb<KB>(grid, s, a);
    BKT_KB_LIST(BKT_CASE)
#undef BKT_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

inline cudaError_t launch_plan_split(cudaStream_t s, int* counts, int* key_off, int nkeys, int* toff, RoundCtl* ctl) {
  plan_split_kernel<<<1, kPlanThreads, 0, s>>>(counts, key_off, nkeys, toff, ctl, kNT);
  return cudaGetLastError();
}

inline cudaError_t launch_route(int grid, cudaStream_t s, const RouteArgs& a) {
  route_kernel<<<grid, kRouteThreads, 0, s>>>(a);
  return cudaGetLastError();
}

inline cudaError_t launch_place(int grid, cudaStream_t s, const RouteArgs& a) {
  place_kernel<<<grid, kRouteThreads, 0, s>>>(a);
  return cudaGetLastError();
}

inline cudaError_t launch_rescan(bool fma, int grid, cudaStream_t s, const int* ovf, const RoundCtl* ctl, const float* q,
                          int D, int k, int d, uint64_t* keys, int4* qs, const float* pts,
                          const uint32_t* pidx, const long long* quad_base, uint8_t* ccnt, int NW, int* ovflag) {
  if (fma)
    rescan_kernel<true><<<grid, kFinishWarps * 32, 0, s>>>(ovf, ctl, q, D, k, d, keys, qs, pts, pidx,
                                                           quad_base, ccnt, NW, ovflag);
  else
    rescan_kernel<false><<<grid, kFinishWarps * 32, 0, s>>>(ovf, ctl, q, D, k, d, keys, qs, pts, pidx,
                                                            quad_base, ccnt, NW, ovflag);
  return cudaGetLastError();
}

}  // namespace bkt
