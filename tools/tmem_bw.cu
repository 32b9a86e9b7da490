// tmem_bw.cu -- TMEM -> register read throughput on one SM (the ceiling of the
// tensor-core leaf filter's epilogue: one f32 accumulator read per distance pair).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bw tools/tmem_bw.cu && tools/tmem_bw
//
// Variants: warps per CTA (4/8/16), loads per wait (1/2/4, x32 each), with and
// without a 3-input-min reduction of the loaded values.
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

template <int PER_WAIT, bool REDUCE>
__global__ void bw(int reps, long long* cycles, float* sink) {
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * ((warp >> 2) & 3);
  float acc = 0.f;
  uint32_t x = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < 4; c += PER_WAIT) {
      uint32_t v[PER_WAIT][32];
#pragma unroll
      for (int p = 0; p < PER_WAIT; ++p) LD32(tbase + 32 * (c + p), v[p]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int p = 0; p < PER_WAIT; ++p) {
        if (REDUCE) acc = fminf(acc, min32(v[p]));
        else {
#pragma unroll
          for (int j = 0; j < 32; j += 8) x ^= v[p][j];
        }
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 1234.5f || x == 0x12345u) sink[threadIdx.x] = acc + x;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

template <int PER_WAIT, bool REDUCE>
int run(int warps, long long* dc, float* ds) {
  const int reps = 2000;
  bw<PER_WAIT, REDUCE><<<148, warps * 32>>>(reps, dc, ds);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  bw<PER_WAIT, REDUCE><<<148, warps * 32>>>(reps, dc, ds);
  CK(cudaDeviceSynchronize());
  long long cyc[148];
  CK(cudaMemcpy(cyc, dc, sizeof(cyc), cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
  const double bytes = (double)reps * warps * 32 * 128 * 4;  // per CTA (= per SM)
  printf("warps %2d loads/wait %d reduce %d : %7.1f B/clk/SM  (%.1f f32 values/clk/SM)\n", warps, PER_WAIT,
         (int)REDUCE, bytes / mx, bytes / mx / 4);
  return 0;
}

int main() {
  long long* dc;
  float* ds;
  CK(cudaMalloc(&dc, 148 * sizeof(long long)));
  CK(cudaMalloc(&ds, 1024 * sizeof(float)));
  for (int w : {4, 8, 12, 16}) {
    run<1, false>(w, dc, ds);
    run<2, false>(w, dc, ds);
    run<4, false>(w, dc, ds);
    run<1, true>(w, dc, ds);
    run<2, true>(w, dc, ds);
  }
  return 0;
}
