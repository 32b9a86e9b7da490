// build_tree_gpu.cu -- device-side build of the buffer k-d tree (bkt_build_tree_device).
//
// Same contract as the host build (build_tree.cpp) and the reference
// (buffer_tree.py:149-197, kdtree.py:46-70): level by level every subset is
// cut at its positional median of coordinate (depth % d) under the unique
// key  order_bits(coord) << 32 | original_index; the element of rank s/2 is
// the split value and goes right.  The subset sizes only depend on n
// (s -> s/2, s - s/2), so every level's segment bounds are known up front.
//
// Per level, on the GPU:
//   keys     : key[i] = order_bits(refs[idx[i], dim]) << 32 | idx[i]   (gather)
//   select   : 8 MSB-first radix passes of 8 bits find each segment's key of
//              rank s/2 (per-CTA shared-memory histograms of the segment
//              runs a CTA's element range covers, flushed with atomics; one
//              thread per segment then picks the digit bucket holding the rank)
//   partition: flag = key < pivot; a device-wide exclusive scan of the flags
//              gives every element its slot left (rank among the segment's
//              smaller keys) or right of the segment's cut (stable)
// The leaf-sorted points are gathered on the device at the end.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/bkt.h"

namespace {

constexpr int kBT = 256;      // threads per CTA
constexpr int kPerCta = 4096; // elements per CTA in the histogram / scan passes

__device__ __forceinline__ uint32_t order_bits_dev(float v) {
  const uint32_t b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b ^ 0x80000000u);
}

// segment of position i: seg_lo is ascending, nseg entries (+ sentinel n)
__device__ __forceinline__ int seg_of(const long long* __restrict__ seg_lo, int nseg, long long i) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg_lo[mid] <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void make_keys(const float* __restrict__ refs, int d, int dim, const uint32_t* __restrict__ idx,
                          unsigned long long* __restrict__ key, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t r = idx[i];
    key[i] = ((unsigned long long)order_bits_dev(__ldg(refs + (long long)r * d + dim)) << 32) | r;
  }
}

// One radix pass: histogram of digit (key >> shift) & 255 over the elements
// of each segment whose bits above the digit equal the segment's prefix.
__global__ void __launch_bounds__(kBT) radix_hist(const unsigned long long* __restrict__ key, long long n,
                                                  const long long* __restrict__ seg_lo, int nseg,
                                                  const unsigned long long* __restrict__ prefix, int shift,
                                                  unsigned int* __restrict__ hist) {
  __shared__ unsigned int h[256];
  const long long a = (long long)blockIdx.x * kPerCta, b = min(n, a + kPerCta);
  if (a >= b) return;
  int s = seg_of(seg_lo, nseg, a);
  long long s_end = (s + 1 < nseg) ? seg_lo[s + 1] : n;
  long long pos = a;
  while (pos < b) {
    const long long run_end = min(b, s_end);
    for (int t = threadIdx.x; t < 256; t += kBT) h[t] = 0;
    __syncthreads();
    const unsigned long long pre = prefix[s];
    const int hs = shift + 8;  // bits above the digit must match
    for (long long i = pos + threadIdx.x; i < run_end; i += kBT) {
      const unsigned long long k = key[i];
      if (hs >= 64 || (k >> hs) == (pre >> hs)) atomicAdd(&h[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 256; t += kBT)
      if (h[t]) atomicAdd(hist + (size_t)s * 256 + t, h[t]);
    __syncthreads();
    pos = run_end;
    if (pos < b) {
      ++s;
      s_end = (s + 1 < nseg) ? seg_lo[s + 1] : n;
    }
  }
}

// One thread per segment: the digit bucket holding the remaining rank.
__global__ void radix_pick(unsigned int* __restrict__ hist, int nseg, unsigned long long* __restrict__ prefix,
                           long long* __restrict__ rank, int shift) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  unsigned int* h = hist + (size_t)s * 256;
  long long r = rank[s];
  unsigned long long digit = 0;
  for (int t = 0; t < 256; ++t) {
    const long long c = h[t];
    if (r < c) { digit = (unsigned long long)t; break; }
    r -= c;
  }
  for (int t = 0; t < 256; ++t) h[t] = 0;  // ready for the next pass
  rank[s] = r;
  prefix[s] |= digit << shift;
}

// flags + per-CTA sums for the partition scan
__global__ void __launch_bounds__(kBT) part_flags(const unsigned long long* __restrict__ key, long long n,
                                                  const long long* __restrict__ seg_lo, int nseg,
                                                  const unsigned long long* __restrict__ pivot,
                                                  unsigned int* __restrict__ flag, unsigned int* __restrict__ cta_sum) {
  __shared__ unsigned int ws[kBT / 32];
  const long long a = (long long)blockIdx.x * kPerCta, b = min(n, a + kPerCta);
  unsigned int cnt = 0;
  if (a < b) {
    int s = seg_of(seg_lo, nseg, a + threadIdx.x < b ? a + threadIdx.x : a);
    for (long long i = a + threadIdx.x; i < b; i += kBT) {
      while (s + 1 < nseg && seg_lo[s + 1] <= i) ++s;
      const unsigned int f = key[i] < pivot[s] ? 1u : 0u;
      flag[i] = f;
      cnt += f;
    }
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = 0;
    for (int w = 0; w < kBT / 32; ++w) t += ws[w];
    cta_sum[blockIdx.x] = t;
  }
}

// exclusive scan of the per-CTA sums (one CTA, sequential chunks of kBT)
__global__ void __launch_bounds__(kBT) scan_cta_sums(unsigned int* __restrict__ cta_sum, int ncta,
                                                     unsigned long long* __restrict__ cta_off) {
  __shared__ unsigned long long carry;
  __shared__ unsigned long long ws[kBT / 32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < ncta; base += kBT) {
    const int i = base + threadIdx.x;
    unsigned long long v = i < ncta ? cta_sum[i] : 0, x = v;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    unsigned long long wpre = 0;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) wpre += ws[w];
    if (i < ncta) cta_off[i] = carry + wpre + x - v;
    __syncthreads();
    if (threadIdx.x == kBT - 1) carry += wpre + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) cta_off[ncta] = carry;
}

// global exclusive prefix of flags at every element, then the scatter
__global__ void __launch_bounds__(kBT) part_scatter(const unsigned int* __restrict__ flag, long long n,
                                                    const unsigned long long* __restrict__ cta_off,
                                                    unsigned long long* __restrict__ pre_out) {
  // per-CTA in-order scan of its kPerCta flags (kPerCta / kBT per thread, contiguous)
  __shared__ unsigned long long ws[kBT / 32];
  constexpr int per = kPerCta / kBT;
  const long long a = (long long)blockIdx.x * kPerCta;
  const long long t0 = a + (long long)threadIdx.x * per;
  unsigned int loc[per];
  unsigned long long sum = 0;
#pragma unroll
  for (int j = 0; j < per; ++j) {
    loc[j] = (t0 + j < n) ? flag[t0 + j] : 0u;
    sum += loc[j];
  }
  unsigned long long x = sum;
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
  __syncthreads();
  unsigned long long wpre = 0;
  for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) wpre += ws[w];
  unsigned long long run = cta_off[blockIdx.x] + wpre + x - sum;
#pragma unroll
  for (int j = 0; j < per; ++j) {
    if (t0 + j < n) pre_out[t0 + j] = run;
    run += loc[j];
  }
}

__global__ void part_move(const unsigned long long* __restrict__ key, const unsigned int* __restrict__ flag,
                          const unsigned long long* __restrict__ pre, long long n,
                          const long long* __restrict__ seg_lo, int nseg, const long long* __restrict__ mid,
                          uint32_t* __restrict__ idx_out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int s = seg_of(seg_lo, nseg, i);
    const long long lo = seg_lo[s];
    const long long left_before = (long long)(pre[i] - pre[lo]);
    const long long dst = flag[i] ? lo + left_before : lo + mid[s] + ((i - lo) - left_before);
    idx_out[dst] = (uint32_t)(key[i] & 0xFFFFFFFFull);
  }
}

__global__ void gather_rows(const float* __restrict__ refs, int d, const uint32_t* __restrict__ idx, long long n,
                            float* __restrict__ out, long long* __restrict__ order) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * d; t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / d;
    const int j = (int)(t - i * d);
    const uint32_t r = idx[i];
    out[t] = __ldg(refs + (long long)r * d + j);
    if (j == 0) order[i] = (long long)r;
  }
}

thread_local std::string g_build_err;

}  // namespace

extern "C" const char* bkt_build_tree_device_error(void) { return g_build_err.c_str(); }

// Device build: refs (n x d, host), outputs as bkt_build_tree plus the
// leaf-sorted points (n x d, host; optional).  cuda_device selects the GPU.
extern "C" int bkt_build_tree_device(int cuda_device, const float* refs, int64_t n, int32_t d, int32_t h,
                                     float* split_out, int64_t* order_out, int64_t* leaf_starts_out,
                                     float* points_out) {
  g_build_err.clear();
  if (!refs || !split_out || !order_out || !leaf_starts_out || d < 1 || h < 1 || h > 24) {
    g_build_err = "invalid arguments";
    return BKT_EINVAL;
  }
  if (n < (int64_t(1) << h) || n >= int64_t(0xFFFFFFFFll)) {
    g_build_err = "height needs at least 2^h points (and n < 2^32 - 1)";
    return BKT_EINVAL;
  }
  cudaError_t e = cudaSetDevice(cuda_device);
#define CK(call)                                                                            \
  do {                                                                                      \
    e = (call);                                                                             \
    if (e != cudaSuccess) {                                                                 \
      g_build_err = std::string("CUDA error: ") + cudaGetErrorString(e) + " (" #call ")";   \
      goto fail;                                                                            \
    }                                                                                       \
  } while (0)
  {
    float* d_refs = nullptr;
    float* d_pts = nullptr;
    uint32_t* d_idx[2] = {nullptr, nullptr};
    unsigned long long *d_key = nullptr, *d_prefix = nullptr, *d_pre = nullptr, *d_cta_off = nullptr;
    unsigned int *d_hist = nullptr, *d_flag = nullptr, *d_cta_sum = nullptr;
    long long *d_seg = nullptr, *d_rank = nullptr, *d_mid = nullptr, *d_order = nullptr;
    cudaStream_t st = nullptr;
    const int maxseg = 1 << (h - 1);
    const int ncta = (int)((n + kPerCta - 1) / kPerCta);
    const int grid = 148 * 8;
    std::vector<long long> seg{0, (long long)n}, nseg_lo;
    std::vector<long long> mids, ranks;
    std::vector<unsigned long long> pivots;
    std::vector<float> sv;
    std::vector<uint32_t> hidx;
    long long node = 0;
    int cur = 0;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaMalloc(&d_refs, sizeof(float) * n * d));
    CK(cudaMemcpyAsync(d_refs, refs, sizeof(float) * n * d, cudaMemcpyHostToDevice, st));
    CK(cudaMalloc(&d_idx[0], sizeof(uint32_t) * n));
    CK(cudaMalloc(&d_idx[1], sizeof(uint32_t) * n));
    CK(cudaMalloc(&d_key, sizeof(unsigned long long) * n));
    CK(cudaMalloc(&d_flag, sizeof(unsigned int) * n));
    CK(cudaMalloc(&d_pre, sizeof(unsigned long long) * n));
    CK(cudaMalloc(&d_cta_sum, sizeof(unsigned int) * ncta));
    CK(cudaMalloc(&d_cta_off, sizeof(unsigned long long) * (ncta + 1)));
    CK(cudaMalloc(&d_hist, sizeof(unsigned int) * 256 * maxseg));
    CK(cudaMemsetAsync(d_hist, 0, sizeof(unsigned int) * 256 * maxseg, st));
    CK(cudaMalloc(&d_prefix, sizeof(unsigned long long) * maxseg));
    CK(cudaMalloc(&d_seg, sizeof(long long) * (2 * maxseg + 1)));
    CK(cudaMalloc(&d_rank, sizeof(long long) * maxseg));
    CK(cudaMalloc(&d_mid, sizeof(long long) * maxseg));
    hidx.resize(n);
    for (int64_t i = 0; i < n; ++i) hidx[i] = (uint32_t)i;
    CK(cudaMemcpyAsync(d_idx[0], hidx.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st));
    for (int depth = 0; depth < h; ++depth) {
      const int dim = depth % d;
      const int nseg = (int)seg.size() - 1;
      mids.assign(nseg, 0);
      for (int s = 0; s < nseg; ++s) mids[s] = (seg[s + 1] - seg[s]) / 2;
      CK(cudaMemcpyAsync(d_seg, seg.data(), sizeof(long long) * (nseg + 1), cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(d_rank, mids.data(), sizeof(long long) * nseg, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(d_mid, mids.data(), sizeof(long long) * nseg, cudaMemcpyHostToDevice, st));
      CK(cudaMemsetAsync(d_prefix, 0, sizeof(unsigned long long) * nseg, st));
      make_keys<<<grid, kBT, 0, st>>>(d_refs, d, dim, d_idx[cur], d_key, n);
      CK(cudaGetLastError());
      for (int shift = 56; shift >= 0; shift -= 8) {
        radix_hist<<<ncta, kBT, 0, st>>>(d_key, n, d_seg, nseg, d_prefix, shift, d_hist);
        CK(cudaGetLastError());
        radix_pick<<<(nseg + 127) / 128, 128, 0, st>>>(d_hist, nseg, d_prefix, d_rank, shift);
        CK(cudaGetLastError());
      }
      // d_prefix now holds each segment's pivot key (rank s/2)
      part_flags<<<ncta, kBT, 0, st>>>(d_key, n, d_seg, nseg, d_prefix, d_flag, d_cta_sum);
      CK(cudaGetLastError());
      scan_cta_sums<<<1, kBT, 0, st>>>(d_cta_sum, ncta, d_cta_off);
      CK(cudaGetLastError());
      part_scatter<<<ncta, kBT, 0, st>>>(d_flag, n, d_cta_off, d_pre);
      CK(cudaGetLastError());
      part_move<<<grid, kBT, 0, st>>>(d_key, d_flag, d_pre, n, d_seg, nseg, d_mid, d_idx[cur ^ 1]);
      CK(cudaGetLastError());
      cur ^= 1;
      pivots.resize(nseg);
      CK(cudaMemcpyAsync(pivots.data(), d_prefix, sizeof(unsigned long long) * nseg, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      sv.resize(nseg);
      for (int s = 0; s < nseg; ++s) {
        const uint32_t r = (uint32_t)(pivots[s] & 0xFFFFFFFFull);
        split_out[node++] = refs[(int64_t)r * d + dim];
      }
      nseg_lo.assign(2 * nseg + 1, 0);
      for (int s = 0; s < nseg; ++s) {
        nseg_lo[2 * s] = seg[s];
        nseg_lo[2 * s + 1] = seg[s] + mids[s];
      }
      nseg_lo[2 * nseg] = n;
      seg.swap(nseg_lo);
    }
    CK(cudaMalloc(&d_order, sizeof(long long) * n));
    if (points_out) {
      CK(cudaMalloc(&d_pts, sizeof(float) * n * d));
      gather_rows<<<grid, kBT, 0, st>>>(d_refs, d, d_idx[cur], n, d_pts, d_order);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(points_out, d_pts, sizeof(float) * n * d, cudaMemcpyDeviceToHost, st));
    } else {
      CK(cudaMemcpyAsync(hidx.data(), d_idx[cur], sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, st));
    }
    if (points_out) {
      CK(cudaMemcpyAsync(order_out, d_order, sizeof(long long) * n, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    } else {
      CK(cudaStreamSynchronize(st));
      for (int64_t i = 0; i < n; ++i) order_out[i] = (int64_t)hidx[i];
    }
    std::memcpy(leaf_starts_out, seg.data(), sizeof(int64_t) * seg.size());
    cudaFree(d_refs); cudaFree(d_pts); cudaFree(d_idx[0]); cudaFree(d_idx[1]); cudaFree(d_key);
    cudaFree(d_flag); cudaFree(d_pre); cudaFree(d_cta_sum); cudaFree(d_cta_off); cudaFree(d_hist);
    cudaFree(d_prefix); cudaFree(d_seg); cudaFree(d_rank); cudaFree(d_mid); cudaFree(d_order);
    cudaStreamDestroy(st);
    return BKT_OK;
  }
fail:
  return BKT_ECUDA;
#undef CK
}
