// kernel_cluster.cuh -- batch-1 persistent cluster kernel: residency plan + launch.
//
// One thread-block cluster (<= 16 CTAs, one per SM) holds the whole model on
// chip and generates every sample of one utterance in a single launch.  CTA
// roles:
//   chain CTAs  c = 0..nc-1 : layers [3c, 3c+3): W_cur, the folded W_cur W_res and
//                             W_res in tensor memory, W_prev in shared memory;
//                             CTA 0 also samples and embeds
//   head CTAs   h = 0..3    : W_skip^(l) / W_relu / W_out row blocks in tensor
//                             memory, W_skip^(l-1) in shared memory
//   skip CTAs   k = 0..nk-1 : W_skip^(j) for j < l-2, tensor + shared memory
// Hand-offs are DSMEM st.async stores that complete transaction bytes on the
// receiver's mbarrier (data and signal in one message), replacing the paper's
// L2 spin-locks (App. D).
#pragma once
#include "dvw_internal.cuh"

namespace dvw {

constexpr int kCMaxCta = 16;
constexpr int kCMaxLayers = 64;
constexpr int kCMaxSkip = 8;
constexpr int kCMaxSlot = 12;

struct ClusterPlan {
  bool ok = false;
  const char* why = "not planned";
  int L = 0, r = 0, s = 0;
  int nc = 0, nh = 0, nk = 0, size = 0;
  int chain_first[kCMaxCta] = {};
  int chain_nl[kCMaxCta] = {};
  int skip_n[kCMaxSkip] = {};     // layers owned by skip CTA k
  int skip_nsm[kCMaxSkip] = {};   // of which the first nsm live in shared memory, the rest in registers
  int layer_skip_cta[kCMaxLayers] = {};   // cluster rank owning W_skip^(j) (j < L-1)
  int layer_skip_slot[kCMaxLayers] = {};  // slot inside that CTA
  int64_t pk_off[kCMaxCta] = {};  // float offset of each CTA's tensor-memory image [column][128 lanes]
  int tm_cols[kCMaxCta] = {};     // columns of that image
  int64_t pk_smem_off[kCMaxCta] = {};  // float offset of its shared-memory image (inside the block)
  int pk_smem_floats[kCMaxCta] = {};   // size of that image
  int64_t embp_off = 0;           // W_emb_prev transposed [256][r]
  int64_t pk_total = 0;           // floats
  int smem_bytes = 0;
};

ClusterPlan plan_cluster(int L, int r, int s, int device);
size_t packed_bytes(const ClusterPlan& p);
// Build the residency layout on the host from the raw roster-order blob and upload it.
cudaError_t pack_cluster_weights(const ClusterPlan& p, const float* host_blob, const Offsets& o, void* packed);
cudaError_t launch_cluster_kernel(const RunArgs& a, const ClusterPlan& p, const void* packed, cudaStream_t st,
                                  LaunchInfo* info);

}  // namespace dvw
