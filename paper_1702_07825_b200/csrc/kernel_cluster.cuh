// kernel_cluster.cuh -- batch-1 persistent cluster kernel: residency plan + launch.
//
// One thread-block cluster (<= 16 CTAs, one per SM) holds the whole model on
// chip and generates every sample of one utterance in a single launch; a batch of
// streams launches one cluster per stream (up to max_clusters run at once).  CTA
// roles:
//   chain CTAs  c = 0..nc-1 : layers [lp c, lp c + lp), lp = 3 or 4: W_cur and the folded
//                             W_cur W_res in tensor memory, W_res in tensor memory (lp 3)
//                             or shared memory (lp 4), W_prev streamed
//                             from L2 (off the critical chain); CTA 0 also samples
//                             and embeds; skip layers that no skip CTA holds are
//                             applied by their chain CTA from L2, after the pass
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
constexpr int kCMaxSkip = 10;  // skip-partial senders into the heads: skip CTAs + chain CTAs
constexpr int kCMaxSlot = 12;

struct ClusterPlan {
  bool ok = false;
  const char* why = "not planned";
  int L = 0, r = 0, s = 0;
  int lpc = 3;                    // layers per chain CTA (3: all chain weights in TMEM; 4: W_res in SMEM)
  int nc = 0, nh = 0, nk = 0, size = 0;
  int chain_first[kCMaxCta] = {};
  int chain_nl[kCMaxCta] = {};
  int skip_n[kCMaxSkip] = {};     // layers owned by skip CTA k
  int skip_nsm[kCMaxSkip] = {};   // of which the first nsm live in shared memory, the rest in registers
  int layer_skip_cta[kCMaxLayers] = {};   // cluster rank owning W_skip^(j) (j < L-2); -1: the chain CTA
                                          // of layer j applies it from L2 ("chain-skip" layers j < nxs)
  int layer_skip_slot[kCMaxLayers] = {};  // slot inside that CTA
  int nxs = 0;                    // chain-skip layers: j in [0, nxs)
  int npart = 0;                  // skip partials each head receives (nk skip CTAs + chain senders)
  int xpart_slot[kCMaxCta] = {};  // heads' partial slot of chain CTA c (-1: none)
  int64_t wprev_off = 0;          // W_prev_j, [L][16 (k/4)][128 (i)][4], read by the chain CTAs' aux warps
  int64_t wskx_off = 0;           // W_skip_j for j < nxs, [nxs][16 (k/4)][s (row)][4]
  int64_t pk_off[kCMaxCta] = {};  // float offset of each CTA's tensor-memory image [column][128 lanes]
  int tm_cols[kCMaxCta] = {};     // columns of that image
  int64_t pk_smem_off[kCMaxCta] = {};  // float offset of its shared-memory image (inside the block)
  int pk_smem_floats[kCMaxCta] = {};   // size of that image
  int64_t embp_off = 0;           // W_emb_prev transposed [256][r]
  int64_t pk_total = 0;           // floats
  int smem_bytes = 0;
  int max_clusters = 0;           // co-resident clusters on the device (one stream each)
  // multi-stream variant (several streams' samples interleaved per cluster; kernel_cluster.cu PIPE)
  bool pipe_ok = false;
  int smem_pipe = 0;              // its dynamic shared memory (Mail + per-stream mailboxes + image)
  int max_clusters_pipe = 0;
  int sw_off_pipe[kCMaxCta] = {}; // byte offset of each CTA's weights image in that layout
  int nwp[kCMaxCta] = {};         // LP = 4 chain CTAs: W_prev layers resident in shared memory (the rest stream from L2)
  int xnb[kCMaxCta] = {};         // LP = 4 chain CTAs: buffers of the aux warps' weight-stream ring
};

ClusterPlan plan_cluster(int L, int r, int s, int device);
size_t packed_bytes(const ClusterPlan& p);
// Build the residency layout on the host from the raw roster-order blob and upload it.
cudaError_t pack_cluster_weights(const ClusterPlan& p, const float* host_blob, const Offsets& o, void* packed);
// Latency-floor microbenchmarks of the batch-1 critical path's pieces (dvw_measure_floor).
struct FloorProbe {
  double layer_cycles, hop_cycles, head_stage_cycles, sampler_cycles, sm_ghz;
};
cudaError_t measure_floor(int device, FloorProbe* out);

cudaError_t launch_cluster_kernel(const RunArgs& a, const ClusterPlan& p, const void* packed, cudaStream_t st,
                                  LaunchInfo* info);

}  // namespace dvw
