// chunk_cost.cu -- fixed cost of the TC epilogue's per-chunk protocol, without
// MMA or TMA: which of {mbarrier wait on a completed phase, tcgen05 fences,
// the two tcgen05.ld pairs + min trees, the vote, the release arrive} sets the
// ~900 SM-cycles per 128-column chunk seen in leafscan_tc_kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/chunk_cost tools/chunk_cost.cu && tools/chunk_cost
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1;} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define LD32(taddr, v)                                                                                       \
  asm volatile(                                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"       \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                            \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),      \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),            \
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),            \
        "=r"(v[30]), "=r"(v[31])                                                                             \
      : "r"(taddr))
#define WAITLD(v)                                                                                          \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                            \
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),       \
                 "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]),    \
                 "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), \
                 "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), \
                 "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])                                         \
               :                                                                                           \
               : "memory")
#define TOUCH(v)                                                                                           \
  asm volatile(""                                                                                          \
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),       \
                 "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]),    \
                 "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), \
                 "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), \
                 "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])                                         \
               :                                                                                           \
               : "memory")

__device__ __forceinline__ float min32(const uint32_t (&v)[32]) {
  float m[11];
#pragma unroll
  for (int i = 0; i < 10; ++i)
    m[i] = fminf(fminf(__uint_as_float(v[3 * i]), __uint_as_float(v[3 * i + 1])), __uint_as_float(v[3 * i + 2]));
  m[10] = fminf(__uint_as_float(v[30]), __uint_as_float(v[31]));
  float a = fminf(fminf(m[0], m[1]), m[2]), b = fminf(fminf(m[3], m[4]), m[5]);
  float c = fminf(fminf(m[6], m[7]), m[8]), d = fminf(m[9], m[10]);
  return fminf(fminf(a, b), fminf(c, d));
}

__device__ __forceinline__ bool try_wait(uint64_t* bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph), "r"(0x989680u) : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph) : "memory");
  return ok != 0;
}

// MODE bits: 1 = wait on a completed barrier (try_wait), 2 = tcgen05 fences,
// 4 = release (syncwarp + lane-0 arrive x2), 8 = test_wait instead of try_wait,
// 16 = two groups only (64 columns)
template <int MODE>
__global__ void chunk(int reps, long long* cycles, float* sink, float thr) {
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bars[3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncols = 512 / (int)(blockDim.x / 128);  // TMEM columns per CTA (CTAs per SM = blocks/148)
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[1])), "r"((1 << 20) - 1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[2])), "r"((1 << 20) - 1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t st;
    asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(smem_u32(&bars[0])) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  (void)ncols;
  const uint32_t tbase = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * ((warp >> 2) & 1);
  float acc = 0.f;
  int hits = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (MODE & 1) {
      if (MODE & 8) { while (!test_wait(&bars[0], 0)) {} }
      else { while (!try_wait(&bars[0], 0)) {} }
    }
    if (MODE & 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t va[32], vb[32];
    LD32(tbase, va);
    LD32(tbase + 32, vb);
    WAITLD(va);
    TOUCH(vb);
    float m = fminf(min32(va), min32(vb));
    if (!(MODE & 16)) {
      LD32(tbase + 64, va);
      LD32(tbase + 96, vb);
      WAITLD(va);
      TOUCH(vb);
      m = fminf(m, fminf(min32(va), min32(vb)));
    }
    if (__any_sync(0xffffffffu, m <= thr)) { hits++; acc += m; }
    if (MODE & 2) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (MODE & 4) {
      __syncwarp();
      if (lane == 0) {
        uint64_t st;
        asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(smem_u32(&bars[1])) : "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(smem_u32(&bars[2])) : "memory");
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (hits == 12345) sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256));
}

template <int MODE>
int run(const char* name, int ctas_per_sm, int warps, long long* dc, float* ds) {
  const int reps = 4000;
  const int grid = 148 * ctas_per_sm;
  chunk<MODE><<<grid, warps * 32>>>(reps, dc, ds, -1e30f);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  chunk<MODE><<<grid, warps * 32>>>(reps, dc, ds, -1e30f);
  CK(cudaDeviceSynchronize());
  static long long cyc[148 * 4];
  CK(cudaMemcpy(cyc, dc, sizeof(long long) * grid, cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
  // chunks per SM = reps x ctas_per_sm x (warps / 4) warp-groups
  const double chunks = (double)reps * ctas_per_sm * (warps / 4);
  printf("%-34s ctas/SM %d warps %2d : %6.0f cycles per chunk per warp-group, %6.1f SM-cycles per chunk\n", name,
         ctas_per_sm, warps, (double)mx / reps, (double)mx / chunks);
  return 0;
}

int main() {
  long long* dc;
  float* ds;
  CK(cudaMalloc(&dc, 148 * 4 * sizeof(long long)));
  CK(cudaMalloc(&ds, 1024 * sizeof(float)));
  for (int c : {1, 2}) {
    for (int w : {4, 8}) {
      run<0>("loads+min+vote", c, w, dc, ds);
      run<16>("64 cols: loads+min+vote", c, w, dc, ds);
      run<2>("+fences", c, w, dc, ds);
      run<4>("+release", c, w, dc, ds);
      run<1>("+try_wait(done)", c, w, dc, ds);
      run<9>("+test_wait(done)", c, w, dc, ds);
      run<7>("full protocol (try_wait)", c, w, dc, ds);
      run<15>("full protocol (test_wait)", c, w, dc, ds);
      run<23>("full protocol, 64 cols", c, w, dc, ds);
    }
  }
  return 0;
}
