// mma_latency.cu -- issue -> tcgen05.commit -> mbarrier latency of the leaf
// filter's MMA (kind::tf32, M=128, N in {64,128,256}, K=16 as two K=8 steps),
// one CTA per SM, optionally two CTAs sharing the SM's tensor core.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1512_02831_b200/csrc -I include \
//        --expt-relaxed-constexpr -o tools/mma_latency tools/mma_latency.cu && tools/mma_latency
#include <cstdio>
#include "leafscan_tc.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1;} } while (0)

using namespace bkt;

template <int N, int KT>
__global__ void mma_lat(int reps, int back_to_back, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  float* A = reinterpret_cast<float*>(sm);
  float* B = A + 128 * KT;
  for (int i = threadIdx.x; i < 128 * KT + N * KT; i += blockDim.x) A[i] = 0.0f;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&s_tmem)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t tmem = s_tmem;
    const uint32_t idesc = idesc_tf32(N);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int j = 0; j < back_to_back; ++j) {
#pragma unroll
        for (int h = 0; h < KT / 8; ++h) {
          const uint64_t da = umma_desc(smem_addr(A) + h * 256, 128, KT * 32);
          const uint64_t db = umma_desc(smem_addr(B) + h * 256, 128, KT * 32);
          const uint32_t acc = h > 0 ? 1u : 0u;
          asm volatile(
              "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(&bar))
                   : "memory");
      mbar_wait_spin(&bar, r & 1);
    }
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(256));
  }
}

template <int N>
int run(int ctas_per_sm, int btb) {
  long long* d;
  CK(cudaMalloc(&d, 8 * 1024));
  const int smem = (128 + N) * 16 * 4 + 1024;
  CK(cudaFuncSetAttribute(mma_lat<N, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int reps = 2000;
  mma_lat<N, 16><<<148 * ctas_per_sm, 128, smem>>>(reps, btb, d);
  CK(cudaDeviceSynchronize());
  mma_lat<N, 16><<<148 * ctas_per_sm, 128, smem>>>(reps, btb, d);
  CK(cudaDeviceSynchronize());
  long long h;
  CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
  printf("N %3d ctas/SM %d mma per commit %d : %7.1f cycles per commit round trip\n", N, ctas_per_sm, btb,
         (double)h / reps);
  CK(cudaFree(d));
  return 0;
}

int main() {
  for (int c : {1, 2}) {
    for (int b : {1, 2, 4}) {
      run<64>(c, b);
      run<128>(c, b);
      run<256>(c, b);
    }
  }
  return 0;
}
