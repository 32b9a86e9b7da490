// leafscan_tc_inst.cu -- instantiates the tensor-core leaf filter kernel for
// every top-k bucket.  Compiled once per (KT, NR, CPS, FMA) part
// (-DBKT_TC_KT=.. -DBKT_TC_NR=.. -DBKT_TC_CPS=.. -DBKT_TC_FMA=..) so the parts
// build in parallel; the part built with -DBKT_TC_DISPATCH also defines
// launch_leafscan_tc().
#include <atomic>

#include "dims.h"
#include "leafscan_tc.cuh"

namespace bkt {

#define BKT_TC_PART_DECL(KT, NR, CPS, FMA) \
  cudaError_t launch_tc_##KT##_##NR##_##CPS##_##FMA(int kb, int grid, cudaStream_t s, const TcArgs& a, int* occ);
BKT_TC_PART_DECL(16, 64, 2, 0)
BKT_TC_PART_DECL(16, 64, 2, 1)
BKT_TC_PART_DECL(16, 64, 3, 0)
BKT_TC_PART_DECL(16, 64, 3, 1)
BKT_TC_PART_DECL(16, 128, 3, 0)
BKT_TC_PART_DECL(16, 128, 3, 1)
BKT_TC_PART_DECL(16, 256, 2, 0)
BKT_TC_PART_DECL(16, 256, 2, 1)
BKT_TC_PART_DECL(16, 128, 2, 0)
BKT_TC_PART_DECL(16, 128, 2, 1)
BKT_TC_PART_DECL(32, 64, 2, 0)
BKT_TC_PART_DECL(32, 64, 2, 1)
#undef BKT_TC_PART_DECL

#ifdef BKT_TC_KT
namespace {
template <int KT, int KB, bool FMA, int NR, int CPS>
cudaError_t launch_tc_one(int grid, cudaStream_t s, const TcArgs& a0, int* occ) {
  using S = TcSmem<KT, NR, CPS>;
  auto fn = leafscan_tc_kernel<KT, KB, FMA, NR, CPS>;
  // at least a (CPS+1)-th of the SM so that no more than CPS CTAs share an SM (TMEM columns)
  constexpr int floor_bytes = tc_smem_per_cta(CPS + 1) + 1024;
  constexpr int base = S::kBytes > floor_bytes ? S::kBytes : floor_bytes;
  constexpr int smem_max = tc_smem_per_cta(CPS);
  // the top tree's split values go to shared memory when they fit beside the operand ring
  TcArgs a = a0;
  const int tree_bytes = ((1 << a.s.top.h) - 1) * 4;
  a.tree_smem = (S::kBytes + tree_bytes <= smem_max) ? 1 : 0;
  const int smem = a.tree_smem ? (base > S::kBytes + tree_bytes ? base : S::kBytes + tree_bytes) : base;
  // function attributes are per device: set them once per (instantiation, device)
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, tc_threads(CPS), smem);
  if (a.pdl) {
    // programmatic stream serialization: the prologue overlaps the previous kernel (griddepcontrol.wait)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tc_threads(CPS));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, a);
  }
  fn<<<grid, tc_threads(CPS), smem, s>>>(a);
  return cudaGetLastError();
}
}  // namespace

#define BKT_TC_PART_NAME2(KT, NR, CPS, FMA) launch_tc_##KT##_##NR##_##CPS##_##FMA
#define BKT_TC_PART_NAME(KT, NR, CPS, FMA) BKT_TC_PART_NAME2(KT, NR, CPS, FMA)
cudaError_t BKT_TC_PART_NAME(BKT_TC_KT, BKT_TC_NR, BKT_TC_CPS, BKT_TC_FMA)(int kb, int grid, cudaStream_t s,
                                                                          const TcArgs& a, int* occ) {
  switch (kb) {
#define BKT_CASE(KB) \
  case KB:           \
    return launch_tc_one<BKT_TC_KT, KB, (BKT_TC_FMA != 0), BKT_TC_NR, BKT_TC_CPS>(grid, s, a, occ);
    BKT_KB_LIST(BKT_CASE)
#undef BKT_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
#endif  // BKT_TC_KT

#ifdef BKT_TC_DISPATCH
// nr selects the chunk width for KT = 16 (64 or 128 columns); KT = 32 always
// runs 64-column chunks.  Two CTAs share an SM.
cudaError_t launch_leafscan_tc(int kt, int kb, bool fma, int grid, cudaStream_t s, const TcArgs& a, int* occ,
                               int nr, int cps) {
  if (kt == 32) return fma ? launch_tc_32_64_2_1(kb, grid, s, a, occ) : launch_tc_32_64_2_0(kb, grid, s, a, occ);
  if (kt != 16) return cudaErrorInvalidValue;
  if (cps == 3 && nr == 128)
    return fma ? launch_tc_16_128_3_1(kb, grid, s, a, occ) : launch_tc_16_128_3_0(kb, grid, s, a, occ);
  if (cps == 3) return fma ? launch_tc_16_64_3_1(kb, grid, s, a, occ) : launch_tc_16_64_3_0(kb, grid, s, a, occ);
  if (nr == 256) return fma ? launch_tc_16_256_2_1(kb, grid, s, a, occ) : launch_tc_16_256_2_0(kb, grid, s, a, occ);
  if (nr == 128) return fma ? launch_tc_16_128_2_1(kb, grid, s, a, occ) : launch_tc_16_128_2_0(kb, grid, s, a, occ);
  return fma ? launch_tc_16_64_2_1(kb, grid, s, a, occ) : launch_tc_16_64_2_0(kb, grid, s, a, occ);
}
#endif  // BKT_TC_DISPATCH
}  // namespace bkt
