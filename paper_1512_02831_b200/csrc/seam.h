// seam.h -- device-resident chunk slots of the fine device-plugin seam
// (bkt_seam_copy / bkt_seam_sync / bkt_seam_scan, misc.cu), owned by the context.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

struct bkt_ctx;

namespace bkt_internal {
struct SeamSlot {
  float* pts = nullptr;      // L x d chunk points
  uint32_t* ids = nullptr;   // L original ids
  long long L = 0, cap = 0;  // rows held / allocated
  int d = 0;
  cudaEvent_t ready = nullptr;  // the slot's last copy
};
constexpr int kSeamSlots = 2;
SeamSlot* ctx_seam_slot(bkt_ctx* c, int slot);
cudaStream_t ctx_copy_stream(bkt_ctx* c);
}  // namespace bkt_internal
