// misc.cu -- the reference's fine-grained device plugin seam (bkt_scan_groups)
// and the FP32 pipe probe used as the measured roofline denominator.
#include <cstring>
#include <string>
#include <vector>

#include <algorithm>
#include <numeric>

#include "../../include/bkt.h"
#include "bkt_device.cuh"
#include "seam.h"

using namespace bkt;

// defined in engine.cu
struct bkt_ctx;
namespace bkt_internal {
int ctx_device(bkt_ctx* c);
cudaStream_t ctx_stream(bkt_ctx* c);
int ctx_fail(bkt_ctx* c, int code, const std::string& msg);
}  // namespace bkt_internal

namespace {

// One thread per query row of a group: scan chunk rows [lo, hi) and merge into
// the row's ascending top-k held in global memory.  Reference
// device.py:316-321 (scan) -> core.py:138-146, 152-160, 251-262.
__global__ void groups_kernel(const float* __restrict__ pts, const uint32_t* __restrict__ ids, int d,
                              const float* __restrict__ q, int k, uint64_t* __restrict__ keys, int ngroups,
                              const long long* __restrict__ gptr, const long long* __restrict__ grows,
                              const long long* __restrict__ glo, const long long* __restrict__ ghi,
                              long long total_rows, int exact) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total_rows;
       t += (long long)gridDim.x * blockDim.x) {
    // group of entry t (binary search over gptr)
    int lo = 0, hi = ngroups - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (gptr[mid] <= t) lo = mid; else hi = mid - 1;
    }
    const long long row = grows[t];
    const float* qp = q + row * d;
    uint64_t* kp = keys + row * k;
    for (long long r = glo[lo]; r < ghi[lo]; ++r) {
      const float* pp = pts + r * d;
      float acc = 0.0f;
      if (exact) {
        for (int j = 0; j < d; ++j) {
          float df = __fsub_rn(qp[j], pp[j]);
          acc = __fadd_rn(acc, __fmul_rn(df, df));
        }
      } else {
        for (int j = 0; j < d; ++j) {
          float df = __fsub_rn(qp[j], pp[j]);
          acc = __fmaf_rn(df, df, acc);
        }
      }
      uint64_t c = pack_key(acc, ids[r]);
      if (c < kp[k - 1]) {
        int i = k - 1;
        while (i > 0 && kp[i - 1] > c) {
          kp[i] = kp[i - 1];
          --i;
        }
        kp[i] = c;
      }
    }
  }
}

// One warp per distinct query row of a seam scan: its top-k row (k <= 64)
// lives across the lanes (lane j: entries j and 32 + j, ascending); the lanes
// stride over each of the row's chunk ranges, and every point whose key beats
// the k-th key is inserted at its rank by a one-lane shift -- the best k of
// (row, ranges), NeighborBatch.update_rows (core.py:251-262).
template <bool EXACT>
__global__ void seam_rows_kernel(const float* __restrict__ pts, const uint32_t* __restrict__ ids, int d,
                                 const float* __restrict__ q, int k, uint64_t* __restrict__ keys, int nrows,
                                 const long long* __restrict__ rptr, const long long* __restrict__ rlo,
                                 const long long* __restrict__ rhi) {
  const uint32_t full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < nrows; r += gridDim.x * wpb) {
    uint64_t* kp = keys + (long long)r * k;
    uint64_t r0 = lane < k ? kp[lane] : ~0ull;
    uint64_t r1 = lane + 32 < k ? kp[lane + 32] : ~0ull;
    uint64_t kk = k <= 32 ? __shfl_sync(full, r0, k - 1) : __shfl_sync(full, r1, k - 33);
    const float* qp = q + (long long)r * d;
    for (long long g = rptr[r]; g < rptr[r + 1]; ++g) {
      for (long long p0 = rlo[g]; p0 < rhi[g]; p0 += 32) {
        const long long p = p0 + lane;
        uint64_t key = ~0ull;
        if (p < rhi[g]) {
          const float* pp = pts + p * d;
          float acc = 0.0f;
          for (int j = 0; j < d; ++j) {
            const float df = __fsub_rn(__ldg(qp + j), __ldg(pp + j));
            acc = EXACT ? __fadd_rn(acc, __fmul_rn(df, df)) : __fmaf_rn(df, df, acc);
          }
          key = pack_key(acc, __ldg(ids + p));
        }
        unsigned todo = __ballot_sync(full, key < kk);
        while (todo) {
          const int e = __ffs(todo) - 1;
          todo &= todo - 1;
          const uint64_t cv = __shfl_sync(full, key, e);
          if (!(cv < kk)) continue;
          const int pos = __popc(__ballot_sync(full, r0 < cv)) + __popc(__ballot_sync(full, r1 < cv));
          const uint64_t up0 = __shfl_up_sync(full, r0, 1), up1 = __shfl_up_sync(full, r1, 1);
          const uint64_t last0 = __shfl_sync(full, r0, 31);
          const uint64_t n1 = lane + 32 > pos ? (lane == 0 ? last0 : up1) : (lane + 32 == pos ? cv : r1);
          r0 = lane > pos ? up0 : (lane == pos ? cv : r0);
          r1 = n1;
          kk = k <= 32 ? __shfl_sync(full, r0, k - 1) : __shfl_sync(full, r1, k - 33);
        }
      }
    }
    if (lane < k) kp[lane] = r0;
    if (lane + 32 < k) kp[lane + 32] = r1;
  }
}

#define ITERS 2048
__global__ void ffma_probe(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

}  // namespace

#define CU(call)                                                                                         \
  do {                                                                                                   \
    cudaError_t e_ = (call);                                                                             \
    if (e_ != cudaSuccess)                                                                               \
      return bkt_internal::ctx_fail(ctx, BKT_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                                        " (" #call ")");                                 \
  } while (0)

extern "C" int bkt_scan_groups(bkt_ctx* ctx, const float* points, const int64_t* ids, int64_t L, int32_t d,
                               const float* queries, int64_t m, int32_t k, uint64_t* keys, int32_t ngroups,
                               const int64_t* group_ptr, const int64_t* group_rows, const int64_t* group_lo,
                               const int64_t* group_hi, int32_t exact) {
  if (!ctx) return bkt_internal::ctx_fail(nullptr, BKT_EINVAL, "ctx is NULL");
  if (L < 0 || d < 1 || m < 0 || k < 1 || ngroups < 0)
    return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "invalid scan_groups sizes");
  if (ngroups == 0) return BKT_OK;
  for (int g = 0; g < ngroups; ++g) {
    if (!(0 <= group_lo[g] && group_lo[g] < group_hi[g] && group_hi[g] <= L))
      return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "group range outside chunk");
    if (group_ptr[g + 1] <= group_ptr[g]) return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "empty query group");
  }
  const long long total = group_ptr[ngroups];
  for (long long t = 0; t < total; ++t)
    if (group_rows[t] < 0 || group_rows[t] >= m)
      return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "group row outside the query block");
  CU(cudaSetDevice(bkt_internal::ctx_device(ctx)));
  cudaStream_t s = bkt_internal::ctx_stream(ctx);
  std::vector<uint32_t> ids32((size_t)L);
  for (long long i = 0; i < L; ++i) ids32[i] = (uint32_t)ids[i];
  float *dp = nullptr, *dq = nullptr;
  uint32_t* di = nullptr;
  uint64_t* dk = nullptr;
  long long *dptr = nullptr, *drows = nullptr, *dlo = nullptr, *dhi = nullptr;
  CU(cudaMallocAsync(&dp, sizeof(float) * std::max<long long>(1, L * d), s));
  CU(cudaMallocAsync(&di, sizeof(uint32_t) * std::max<long long>(1, L), s));
  CU(cudaMallocAsync(&dq, sizeof(float) * std::max<long long>(1, m * d), s));
  CU(cudaMallocAsync(&dk, sizeof(uint64_t) * std::max<long long>(1, m * k), s));
  CU(cudaMallocAsync(&dptr, sizeof(long long) * (ngroups + 1), s));
  CU(cudaMallocAsync(&drows, sizeof(long long) * std::max<long long>(1, total), s));
  CU(cudaMallocAsync(&dlo, sizeof(long long) * ngroups, s));
  CU(cudaMallocAsync(&dhi, sizeof(long long) * ngroups, s));
  CU(cudaMemcpyAsync(dp, points, sizeof(float) * L * d, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(di, ids32.data(), sizeof(uint32_t) * L, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(dq, queries, sizeof(float) * m * d, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(dk, keys, sizeof(uint64_t) * m * k, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(dptr, group_ptr, sizeof(long long) * (ngroups + 1), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(drows, group_rows, sizeof(long long) * total, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(dlo, group_lo, sizeof(long long) * ngroups, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(dhi, group_hi, sizeof(long long) * ngroups, cudaMemcpyHostToDevice, s));
  int blocks = (int)std::min<long long>(4096, (total + 127) / 128);
  groups_kernel<<<std::max(1, blocks), 128, 0, s>>>(dp, di, d, dq, k, dk, ngroups, dptr, drows, dlo, dhi, total,
                                                     exact);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(keys, dk, sizeof(uint64_t) * m * k, cudaMemcpyDeviceToHost, s));
  CU(cudaFreeAsync(dp, s)); CU(cudaFreeAsync(di, s)); CU(cudaFreeAsync(dq, s)); CU(cudaFreeAsync(dk, s));
  CU(cudaFreeAsync(dptr, s)); CU(cudaFreeAsync(drows, s)); CU(cudaFreeAsync(dlo, s)); CU(cudaFreeAsync(dhi, s));
  CU(cudaStreamSynchronize(s));
  return BKT_OK;
}

extern "C" int bkt_fp32_peak(bkt_ctx* ctx, double* tflops) {
  if (!ctx || !tflops) return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "ctx/tflops is NULL");
  CU(cudaSetDevice(bkt_internal::ctx_device(ctx)));
  cudaStream_t s = bkt_internal::ctx_stream(ctx);
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, bkt_internal::ctx_device(ctx)));
  const int blocks = sms * 8, threads = 256;
  float* out = nullptr;
  CU(cudaMallocAsync(&out, sizeof(float) * blocks * threads, s));
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    CU(cudaEventRecord(e0, s));
    ffma_probe<<<blocks, threads, 0, s>>>(out, 1.0001f, 0.5f);
    CU(cudaEventRecord(e1, s));
    CU(cudaEventSynchronize(e1));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * blocks * threads * (double)ITERS * 4 * 8;
    if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CU(cudaFreeAsync(out, s));
  CU(cudaStreamSynchronize(s));
  *tflops = best;
  return BKT_OK;
}

extern "C" void* bkt_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (bytes <= 0 || cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocPortable) != cudaSuccess) return nullptr;
  return p;
}

extern "C" void bkt_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

// ---------------------------------------------------------------------------
// Fine device-plugin seam with device-resident chunk slots (SimulatedDevice
// enqueue_copy / enqueue_brute_kernel, device.py:256-337)
// ---------------------------------------------------------------------------
extern "C" int bkt_seam_copy(bkt_ctx* ctx, int32_t slot, const float* points, const int64_t* ids, int64_t L,
                             int32_t d) {
  if (!ctx) return bkt_internal::ctx_fail(nullptr, BKT_EINVAL, "ctx is NULL");
  bkt_internal::SeamSlot* sl = bkt_internal::ctx_seam_slot(ctx, slot);
  if (!sl) return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "seam slot must be 0 or 1");
  if (L < 1 || d < 1) return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "invalid seam chunk sizes");
  CU(cudaSetDevice(bkt_internal::ctx_device(ctx)));
  cudaStream_t cs = bkt_internal::ctx_copy_stream(ctx);
  if (!sl->ready) CU(cudaEventCreateWithFlags(&sl->ready, cudaEventDisableTiming));
  // the slot may still be read by a scan on the compute stream
  CU(cudaStreamSynchronize(bkt_internal::ctx_stream(ctx)));
  if (sl->cap < L * d || sl->L < 0) {
    CU(cudaStreamSynchronize(cs));
    if (sl->pts) cudaFree(sl->pts);
    if (sl->ids) cudaFree(sl->ids);
    sl->pts = nullptr;
    sl->ids = nullptr;
    CU(cudaMalloc(&sl->pts, sizeof(float) * L * d));
    CU(cudaMalloc(&sl->ids, sizeof(uint32_t) * L));
    sl->cap = L * d;
  }
  std::vector<uint32_t> ids32((size_t)L);
  for (long long i = 0; i < L; ++i) {
    if (ids[i] < 0 || ids[i] >= (int64_t)kIndexSentinel)
      return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "point id outside [0, 2^32 - 1)");
    ids32[i] = (uint32_t)ids[i];
  }
  // points: asynchronous when the caller's array is page-locked (the pipeline's staging buffers)
  CU(cudaMemcpyAsync(sl->pts, points, sizeof(float) * L * d, cudaMemcpyHostToDevice, cs));
  CU(cudaMemcpyAsync(sl->ids, ids32.data(), sizeof(uint32_t) * L, cudaMemcpyHostToDevice, cs));
  CU(cudaEventRecord(sl->ready, cs));
  // ids32 is pageable: the copy of it is complete when cudaMemcpyAsync returns
  sl->L = L;
  sl->d = d;
  return BKT_OK;
}

extern "C" int bkt_seam_sync(bkt_ctx* ctx, int32_t slot) {
  if (!ctx) return bkt_internal::ctx_fail(nullptr, BKT_EINVAL, "ctx is NULL");
  bkt_internal::SeamSlot* sl = bkt_internal::ctx_seam_slot(ctx, slot);
  if (!sl) return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "seam slot must be 0 or 1");
  if (sl->ready) CU(cudaEventSynchronize(sl->ready));
  return BKT_OK;
}

extern "C" int bkt_seam_scan(bkt_ctx* ctx, int32_t slot, const float* queries, int64_t m, int32_t k,
                             uint64_t* keys, int32_t ngroups, const int64_t* group_ptr, const int64_t* group_rows,
                             const int64_t* group_lo, const int64_t* group_hi, int32_t exact) {
  if (!ctx) return bkt_internal::ctx_fail(nullptr, BKT_EINVAL, "ctx is NULL");
  bkt_internal::SeamSlot* sl = bkt_internal::ctx_seam_slot(ctx, slot);
  if (!sl || !sl->pts) return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "seam slot holds no chunk");
  if (m < 0 || k < 1 || ngroups < 0) return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "invalid seam scan sizes");
  if (k > 64) {
    // larger rows: the general scan of the same groups (host-resident chunk copy not needed: gather back)
    std::vector<float> pts((size_t)sl->L * sl->d);
    std::vector<uint32_t> ids32((size_t)sl->L);
    CU(cudaMemcpy(pts.data(), sl->pts, sizeof(float) * pts.size(), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(ids32.data(), sl->ids, sizeof(uint32_t) * ids32.size(), cudaMemcpyDeviceToHost));
    std::vector<int64_t> ids64(ids32.begin(), ids32.end());
    return bkt_scan_groups(ctx, pts.data(), ids64.data(), sl->L, sl->d, queries, m, k, keys, ngroups, group_ptr,
                           group_rows, group_lo, group_hi, exact);
  }
  if (ngroups == 0) return BKT_OK;
  const int d = sl->d;
  // (row, lo, hi) triples grouped by distinct row: one warp merges all of a row's ranges
  std::vector<long long> order;
  std::vector<long long> trow, tlo, thi;
  for (int g = 0; g < ngroups; ++g) {
    if (!(0 <= group_lo[g] && group_lo[g] < group_hi[g] && group_hi[g] <= sl->L))
      return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "group range outside chunk");
    if (group_ptr[g + 1] <= group_ptr[g]) return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "empty query group");
    for (long long t = group_ptr[g]; t < group_ptr[g + 1]; ++t) {
      if (group_rows[t] < 0 || group_rows[t] >= m)
        return bkt_internal::ctx_fail(ctx, BKT_EINVAL, "group row outside the query block");
      trow.push_back(group_rows[t]);
      tlo.push_back(group_lo[g]);
      thi.push_back(group_hi[g]);
    }
  }
  order.resize(trow.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](long long a, long long b) { return trow[a] < trow[b]; });
  std::vector<long long> urow, rptr(1, 0), rlo, rhi;
  for (long long i : order) {
    if (urow.empty() || urow.back() != trow[i]) {
      urow.push_back(trow[i]);
      rptr.push_back(rptr.back());
    }
    rlo.push_back(tlo[i]);
    rhi.push_back(thi[i]);
    ++rptr.back();
  }
  const long long nr = (long long)urow.size();
  // only the rows the groups name move: their coordinates and their top-k rows
  std::vector<float> qrows((size_t)nr * d);
  std::vector<uint64_t> krows((size_t)nr * k);
  for (long long i = 0; i < nr; ++i) {
    std::memcpy(&qrows[(size_t)i * d], queries + urow[i] * d, sizeof(float) * d);
    std::memcpy(&krows[(size_t)i * k], keys + urow[i] * k, sizeof(uint64_t) * k);
  }
  CU(cudaSetDevice(bkt_internal::ctx_device(ctx)));
  cudaStream_t s = bkt_internal::ctx_stream(ctx);
  CU(cudaStreamWaitEvent(s, sl->ready, 0));  // the slot's copy (copy stream) before the scan
  float* dq = nullptr;
  uint64_t* dk = nullptr;
  long long *dptr = nullptr, *dlo = nullptr, *dhi = nullptr;
  CU(cudaMallocAsync(&dq, sizeof(float) * nr * d, s));
  CU(cudaMallocAsync(&dk, sizeof(uint64_t) * nr * k, s));
  CU(cudaMallocAsync(&dptr, sizeof(long long) * (nr + 1), s));
  CU(cudaMallocAsync(&dlo, sizeof(long long) * rlo.size(), s));
  CU(cudaMallocAsync(&dhi, sizeof(long long) * rhi.size(), s));
  CU(cudaMemcpyAsync(dq, qrows.data(), sizeof(float) * nr * d, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(dk, krows.data(), sizeof(uint64_t) * nr * k, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(dptr, rptr.data(), sizeof(long long) * (nr + 1), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(dlo, rlo.data(), sizeof(long long) * rlo.size(), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(dhi, rhi.data(), sizeof(long long) * rhi.size(), cudaMemcpyHostToDevice, s));
  const int blocks = (int)std::max<long long>(1, std::min<long long>(4096, (nr + 7) / 8));
  if (exact)
    seam_rows_kernel<true><<<blocks, 256, 0, s>>>(sl->pts, sl->ids, d, dq, k, dk, (int)nr, dptr, dlo, dhi);
  else
    seam_rows_kernel<false><<<blocks, 256, 0, s>>>(sl->pts, sl->ids, d, dq, k, dk, (int)nr, dptr, dlo, dhi);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(krows.data(), dk, sizeof(uint64_t) * nr * k, cudaMemcpyDeviceToHost, s));
  CU(cudaFreeAsync(dq, s)); CU(cudaFreeAsync(dk, s)); CU(cudaFreeAsync(dptr, s));
  CU(cudaFreeAsync(dlo, s)); CU(cudaFreeAsync(dhi, s));
  CU(cudaStreamSynchronize(s));
  for (long long i = 0; i < nr; ++i) std::memcpy(keys + urow[i] * k, &krows[(size_t)i * k], sizeof(uint64_t) * k);
  return BKT_OK;
}
