// kernel_batch.cuh -- batched multi-stream kernel (tcgen05): plan, packing, launch.
//
// Many independent utterances advance in lockstep, one sample per step
// ("auto-regressive process"; SURVEY.md §8(a) "Batched mode").
// With 128 streams per stream block the per-layer projections of §8(a) a3/a4/a6/a7
// and the head a8 become real GEMMs, M = 128 streams x N = a tile of output
// channels x K = input channels, issued as tcgen05.mma kind::tf32 with three
// passes (hi*hi + hi*lo + lo*hi; each fp32 operand split into a tf32 head and
// its exact residual) so the products keep ~fp32 accuracy.  The accumulators live
// in tensor memory; the epilogue warps own one stream each (TMEM lane = stream),
// so the gate, residual update and sampler are thread-local per stream.
//
// One persistent launch runs every step; a stream block of 128 streams is one
// thread-block cluster holding all of its tiles, and the steps' phases (one per
// layer, then z_s, z_a, logits, sample) are separated by the cluster barrier.  Weight tiles and activations are staged into shared memory with
// 1-D bulk copies (cp.async.bulk) from global memory, where they are kept in the
// K-major "core matrix" order the MMA descriptors read.
#pragma once
#include "dvw_internal.cuh"

namespace dvw {

constexpr int kBMaxLayers = 64;

struct BatchPlan {
  bool ok = false;
  const char* why = "not planned";
  int L = 0, r = 0, s = 0;
  int TA = 0, TQ = 0, TH = 0;  // CTAs per stream block: layer tiles (16 channels), skip tiles, head tiles (64 rows)
  int per_sb = 0;              // TA + TQ + TH = the cluster size (<= 16)
  int max_sb = 0;              // stream blocks (clusters, 128 streams each) per launch: one co-resident wave
  // packed weights (floats)
  int64_t la_off = 0, la_floats = 0;    // [L][TA] layer-tile blocks
  int64_t q_off = 0, q_floats = 0;      // [L][TQ] skip-tile blocks
  int64_t hr_off = 0, hr_floats = 0;    // [TH] W_relu tile blocks
  int64_t ho_off = 0, ho_floats = 0;    // [TH] W_out tile blocks
  int64_t bias_off = 0;                 // [L][2r] folded gate bias B^(j) + W_cur^(j) B_res^(j-1)
  int64_t total = 0;
  int smem_bytes = 0;
};

// How a batch of n_streams is laid out: `groups` launches of up to per_group streams, each over
// nsb stream blocks (clusters) of rpb <= 128 streams.
struct BatchGrouping {
  int groups = 0, per_group = 0, nsb = 0, rpb = 0;
};

BatchPlan plan_batch(int L, int r, int s, int device);
BatchGrouping batch_grouping(const BatchPlan& p, int n_streams);
cudaError_t pack_batch_weights(const BatchPlan& p, const float* host_blob, const Offsets& o, void* packed);
// Workspace of one launch group of an n_streams call with dilations `dil` (host array, length L).
size_t batch_workspace_bytes(const BatchPlan& p, const int32_t* dil, int n_streams);
// Workspace a streaming session keeps for n_streams: one region per launch group.
size_t batch_session_bytes(const BatchPlan& p, const int32_t* dil, int n_streams);
// Runs n_streams (any count; the launch groups of batch_grouping run back to back on `st`).
// fast: one tf32 pass (DVW_PRECISION_TF32) instead of the fp32-faithful split.
// session: `ws` holds every group's region (batch_session_bytes), zeroed only when a.n0 == 0,
// and the kernel continues from the queues and code history left there (global index a.n0 + n);
// otherwise all groups share one region, zeroed per launch.
cudaError_t launch_batch_kernel(const RunArgs& a, const BatchPlan& p, const void* packed, void* ws, size_t ws_bytes,
                                const int32_t* dil_host, bool fast, cudaStream_t st, LaunchInfo* info,
                                bool session = false);

}  // namespace dvw
