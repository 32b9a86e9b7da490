// Microbenchmark: FP32 pipe throughput on sm_100a for scalar vs packed f32x2 ops,
// and bit-exactness of the exact-mode distance formulation.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 sub2(u64 a, u64 b){ u64 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 add2(u64 a, u64 b){ u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){ u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

#define ITERS 4096
__global__ void k_ffma(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0+1, x2 = x0+2, x3 = x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_ffma2(float* out, u64 a, u64 b) {
  u64 x[8];
  for (int j = 0; j < 8; ++j) x[j] = (u64)(threadIdx.x + j) * 0x100000001ull;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int t = 0; t < 8; ++t) x[t] = fma2(x[t], a, b);
    }
  }
  u64 s = 0; for (int j = 0; j < 8; ++j) s ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(s & 0xffff);
}
__global__ void k_fadd2(float* out, u64 a) {
  u64 x[8];
  for (int j = 0; j < 8; ++j) x[j] = (u64)(threadIdx.x + j) * 0x100000001ull;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int t = 0; t < 8; ++t) x[t] = add2(x[t], a);
    }
  }
  u64 s = 0; for (int j = 0; j < 8; ++j) s ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(s & 0xffff);
}
// exact-mode distance: diff = q - p ; sq = fma(diff, diff, +0 runtime) ; acc = acc + sq
__global__ void k_exact(const float* q, const float* p, int n, int d, u64 zero, float* out_exact, float* out_fma) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
  // pair the i-th point with itself in both halves: (p_i, p_i)
  u64 acc = 0, accf = 0;
  for (int j = 0; j < d; ++j) {
    float qv = q[j], pv = p[i * d + j];
    u64 qq, pp; unsigned qb = __float_as_uint(qv), pb = __float_as_uint(pv);
    qq = ((u64)qb << 32) | qb; pp = ((u64)pb << 32) | pb;
    u64 df = sub2(qq, pp);
    u64 sq = fma2(df, df, zero);
    acc = add2(acc, sq);
    accf = fma2(df, df, accf);
  }
  out_exact[i] = __uint_as_float((unsigned)(acc & 0xffffffffu));
  out_fma[i] = __uint_as_float((unsigned)(accf & 0xffffffffu));
}
int main() {
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("gpu %s sms %d clock_khz %d\n", prop.name, prop.multiProcessorCount, clk);
  int blocks = prop.multiProcessorCount * 8, threads = 256;
  float* out; cudaMalloc(&out, blocks * threads * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double ops = (double)blocks * threads * ITERS * 4 * 8;  // per-lane op count
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(e0); k_ffma<<<blocks, threads>>>(out, 1.0001f, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA : %.3f ms  %.2f Tlane-op/s  %.2f TFLOP/s\n", ms, ops / ms / 1e9, 2 * ops / ms / 1e9);
    u64 a2 = 0x3f8000d13f8000d1ull, b2 = 0x3f0000003f000000ull;
    cudaEventRecord(e0); k_ffma2<<<blocks, threads>>>(out, a2, b2); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2: %.3f ms  %.2f Tinstr-lane/s  %.2f TFLOP/s\n", ms, ops / ms / 1e9, 4 * ops / ms / 1e9);
    cudaEventRecord(e0); k_fadd2<<<blocks, threads>>>(out, b2); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FADD2: %.3f ms  %.2f Tinstr-lane/s  %.2f Tflop/s\n", ms, ops / ms / 1e9, 2 * ops / ms / 1e9);
  }
  // exactness check
  const int n = 1 << 20, d = 10;
  float *hq = new float[d], *hp = new float[n * d];
  uint64_t s = 12345;
  auto rnd = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (float)((s >> 40) & 0xffffff) / 16777216.0f; };
  for (int j = 0; j < d; ++j) hq[j] = rnd();
  for (int i = 0; i < n * d; ++i) hp[i] = rnd() * (i % 7 == 0 ? 1e-20f : 1.0f);
  float *dq, *dp, *de, *df; cudaMalloc(&dq, d * 4); cudaMalloc(&dp, n * d * 4); cudaMalloc(&de, n * 4); cudaMalloc(&df, n * 4);
  cudaMemcpy(dq, hq, d * 4, cudaMemcpyHostToDevice); cudaMemcpy(dp, hp, n * d * 4, cudaMemcpyHostToDevice);
  k_exact<<<(n + 255) / 256, 256>>>(dq, dp, n, d, 0ull, de, df);
  float* he = new float[n]; float* hf = new float[n];
  cudaMemcpy(he, de, n * 4, cudaMemcpyDeviceToHost); cudaMemcpy(hf, df, n * 4, cudaMemcpyDeviceToHost);
  long bad = 0, fdiff = 0; double maxrel = 0;
  for (int i = 0; i < n; ++i) {
    volatile float acc = 0.0f;
    for (int j = 0; j < d; ++j) { volatile float df_ = hq[j] - hp[i * d + j]; volatile float sq = df_ * df_; acc = acc + sq; }
    float a = acc;
    if (memcmp(&a, &he[i], 4)) ++bad;
    if (memcmp(&a, &hf[i], 4)) { ++fdiff; double r = fabs((double)hf[i] - a) / (a > 0 ? a : 1); if (r > maxrel) maxrel = r; }
  }
  printf("exact-mode mismatches vs host scalar: %ld of %d ; fma-mode differing: %ld (max rel %.3g)\n", bad, n, fdiff, maxrel);
  cudaError_t err = cudaGetLastError(); printf("cuda: %s\n", cudaGetErrorString(err));
  return bad != 0;
}
