// mbar_pingpong.cu -- round-trip latency of an mbarrier hand-off between two
// warps of one CTA (the release -> MMA warp -> commit -> epilogue chain of
// leafscan_tc_kernel has two such hand-offs per chunk), for the three wait
// styles: try_wait with a suspend-time hint (mbar_wait), try_wait without a
// hint (mbar_wait_spin), and a test_wait spin loop.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbar_pingpong tools/mbar_pingpong.cu && tools/mbar_pingpong
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1;} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STYLE>
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  uint32_t ok = 0;
  do {
    if (STYLE == 0)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph), "r"(0x989680u) : "memory");
    else if (STYLE == 1)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph) : "memory");
    else
      asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void arrive(uint64_t* bar) {
  uint64_t st;
  asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(smem_u32(bar)) : "memory");
}

// warp 0 lane 0 and warp 1 lane 0 bounce a token `reps` times; the other
// `busy` warps run an ALU loop (the epilogue warps sharing the SM)
template <int STYLE>
__global__ void pingpong(int reps, long long* out, int busy_iters) {
  __shared__ __align__(8) uint64_t bars[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[1])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0 && lane == 0) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      arrive(&bars[0]);
      wait<STYLE>(&bars[1], r & 1);
    }
    out[blockIdx.x] = clock64() - t0;
  } else if (warp == 1 && lane == 0) {
    for (int r = 0; r < reps; ++r) {
      wait<STYLE>(&bars[0], r & 1);
      arrive(&bars[1]);
    }
  } else if (warp >= 2) {
    float x = threadIdx.x;
    for (int i = 0; i < busy_iters; ++i) x = fminf(fmaxf(x * 1.0001f, 0.5f), 1e6f);
    if (x == 12345.f) out[1000 + threadIdx.x] = 1;
  }
}

template <int STYLE>
int run(const char* name, int warps, int busy) {
  long long* d;
  CK(cudaMalloc(&d, 8 * 4096));
  const int reps = 20000;
  pingpong<STYLE><<<148, warps * 32>>>(reps, d, busy);
  CK(cudaDeviceSynchronize());
  pingpong<STYLE><<<148, warps * 32>>>(reps, d, busy);
  CK(cudaDeviceSynchronize());
  long long h;
  CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
  printf("%-28s warps %2d busy %6d : %6.1f cycles per round trip (2 hand-offs)\n", name, warps, busy, (double)h / reps);
  CK(cudaFree(d));
  return 0;
}

int main() {
  for (int w : {2, 8}) {
    const int busy = w > 2 ? 200000 : 0;
    run<0>("try_wait + suspend hint", w, busy);
    run<1>("try_wait (no hint)", w, busy);
    run<2>("test_wait spin", w, busy);
  }
  return 0;
}
