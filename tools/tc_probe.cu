// tc_probe.cu -- validate the tcgen05 building blocks used by the tensor-core
// leaf filter: TF32 MMA (M=128, N=256, K=16 as 2 x K=8) with SWIZZLE_NONE
// K-major smem descriptors, TMEM alloc/dealloc, tcgen05.ld 32x32b.x32, and
// measure the TMEM->register read throughput.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, SWIZZLE_NONE canonical layout: core matrix = 8 rows x 16 B; rows 16 B
// apart, K-chunks (16 B) LBO apart, 8-row groups SBO apart.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

constexpr uint32_t kIdescTF32 = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0,1,0,p; }"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(ph), "r"(0x989680u) : "memory");
  } while (!ok);
}

__global__ void __launch_bounds__(128, 1) probe(const float* A, const float* B, float* D, int reps, long long* cycles) {
  // A: 128 x 16 row-major (queries), B: 256 x 16 row-major (points); D: 128 x 256
  __shared__ __align__(1024) float sA[128 * 16];
  __shared__ __align__(1024) float sB[256 * 16];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  // canonical layout: row r, k -> group r/8, chunk k/4, row-in-group r%8, elem k%4
  for (int i = tid; i < 128 * 16; i += 128) {
    int r = i / 16, k = i % 16;
    sA[(r / 8) * 128 + (k / 4) * 32 + (r % 8) * 4 + (k % 4)] = A[i];
  }
  for (int i = tid; i < 256 * 16; i += 128) {
    int r = i / 16, k = i % 16;
    sB[(r / 8) * 128 + (k / 4) * 32 + (r % 8) * 4 + (k % 4)] = B[i];
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // st.shared -> visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int h = 0; h < 2; ++h) {
      uint64_t da = make_desc(a0 + 256 * h, 128, 512);
      uint64_t db = make_desc(b0 + 256 * h, 128, 512);
      uint32_t acc = h > 0 ? 1u : 0u;
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                   ::"r"(tbase), "l"(da), "l"(db), "r"(kIdescTF32), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // each warp reads its 32 lanes, 256 columns in 8 chunks of 32
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
  for (int c = 0; c < 8; ++c) {
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tbase + lane_base + 32 * c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) D[tid * 256 + 32 * c + j] = __uint_as_float(v[j]);
  }
  // TMEM read throughput: reps x (128 lanes x 256 cols)
  __syncthreads();
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(tbase + lane_base + 32 * c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= v[j];
    }
  }
  long long t1 = clock64();
  if (tid == 0) cycles[0] = t1 - t0;
  if (acc == 0x12345678u) D[0] = 0;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
}

int main() {
  std::vector<float> A(128 * 16), B(256 * 16), D(128 * 256);
  srand(1);
  // mixed magnitudes (scales 2^-6..2^6 per element) and near-cancelling rows
  for (auto& x : A) x = ((rand() / (float)RAND_MAX) - 0.5f) * ldexpf(1.0f, (rand() % 13) - 6);
  for (auto& x : B) x = ((rand() / (float)RAND_MAX) - 0.5f) * ldexpf(1.0f, (rand() % 13) - 6);
  if (getenv("PROBE_UNIFORM")) {
    for (auto& x : A) x = (rand() / (float)RAND_MAX) - 0.5f;
    for (auto& x : B) x = (rand() / (float)RAND_MAX) - 0.5f;
  }
  if (getenv("PROBE_PREROUND")) {
    // operands already tf32 (round to nearest, ties away, as cvt.rna.tf32): the
    // residual error is then the tensor core's accumulation alone
    auto rna = [](float& x) {
      uint32_t u;
      memcpy(&u, &x, 4);
      u = (u + 0x1000u) & 0xFFFFE000u;
      memcpy(&x, &u, 4);
    };
    for (auto& x : A) rna(x);
    for (auto& x : B) rna(x);
  }
  float *dA, *dB, *dD; long long* dc;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4)); CK(cudaMalloc(&dc, 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  int reps = 1000;
  probe<<<1, 128>>>(dA, dB, dD, reps, dc);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long long cyc; CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0, maxratio = 0; int bad = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 256; ++j) {
      double s = 0, sa = 0;
      for (int k = 0; k < 16; ++k) { s += (double)A[i * 16 + k] * B[j * 16 + k]; sa += fabs((double)A[i * 16 + k] * B[j * 16 + k]); }
      double e = fabs(D[i * 256 + j] - s);
      if (e > maxerr) maxerr = e;
      if (sa > 0) maxratio = fmax(maxratio, e / sa);
      if (e > sa * (1.0 / 256) + 1e-6) ++bad;
      maxref = fmax(maxref, fabs(s));
    }
  printf("max |err| / sum|a_k b_k| = %.3e (= 2^%.2f); tf32 operand rounding alone allows 2^-10\n", maxratio,
         log2(maxratio));
  printf("tf32 mma: max abs err %.3e (max |ref| %.3f), bad %d of %d\n", maxerr, maxref, bad, 128 * 256);
  printf("D[0][0..3] = %f %f %f %f\n", D[0], D[1], D[2], D[3]);
  double bytes = (double)reps * 128 * 256 * 4;
  printf("tmem read: %lld cycles for %d reps -> %.1f B/clk/SM (one CTA, 4 warps)\n", cyc, reps, bytes / cyc);
  return bad != 0;
}
