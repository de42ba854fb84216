// dvw_api.cu -- the C ABI declared in include/dvw.h.
//
// Host-side bookkeeping only: argument validation, the library-owned device
// copies of the weights (raw roster layout + each kernel's packed residency
// layout), the per-stream dilation-queue workspace, kernel selection and error
// reporting.  Every step of the generation itself runs in the kernels.
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "dvw_internal.cuh"
#include "kernel_batch.cuh"
#include "kernel_cluster.cuh"

using namespace dvw;

// A streaming session (include/dvw.h dvw_session_*): the state one-shot calls rebuild from
// zero -- the dilation queues of every stream and the last two codes -- kept between calls.
struct dvw_session {
  int device = 0;
  int n_streams = 0;
  int64_t ring_floats = 0;
  float* d_ring = nullptr;  // [S][ring_floats]
  int* d_y = nullptr;       // [S][2]: y_{n-1}, y_{n-2}
  int64_t n_done = 0;
  int hop = 0;
  int kernel = 0;             // the kernel the session's first call ran on (state layouts differ)
  void* d_bws = nullptr;      // TC kernel: every launch group's workspace (queues, x^(0), codes)
  size_t bws_bytes = 0;
};

struct dvw_model {
  int device = 0;
  int L = 0, r = 0, s = 0, a = 0;
  std::vector<int32_t> dil;
  std::vector<int64_t> ring_off;  // floats, per layer, within one stream's ring
  int64_t ring_floats = 0;
  Offsets off{};
  bool loaded = false;
  int kernel = DVW_KERNEL_AUTO;
  int precision = DVW_PRECISION_FP32;
  int weight_bits = 0;  // dvw_set_weight_bits: applied by dvw_load_weights
  int quant_scheme = DVW_QUANT_PER_ROW;
  int samp_kind = DVW_SAMPLER_DIRECT;
  float samp_inv_t = 1.0f;
  int samp_topk = kLevels;
  // device buffers
  float* d_w = nullptr;
  int32_t* d_dil = nullptr;
  int64_t* d_ring_off = nullptr;
  float* d_ring = nullptr;
  int64_t ring_streams = 0;  // streams the workspace is sized for
  int* d_err = nullptr;       // device view of the mapped, pinned error word
  volatile int* h_err = nullptr;  // host view (read without synchronizing)
  ClusterPlan cplan{};
  void* d_packed = nullptr;  // cluster-kernel residency layout
  size_t packed_bytes = 0;
  BatchPlan bplan{};
  void* d_bpacked = nullptr;  // batched-kernel tile layout
  size_t bpacked_bytes = 0;
  void* d_bws = nullptr;      // batched-kernel workspace (activations, queues, barrier)
  size_t bws_bytes = 0;
  void* d_pws = nullptr;      // parallel teacher-forced workspace (x, x', q for a group of streams)
  void* d_ptc = nullptr;      // parallel teacher-forced: tensor-core layer images (r = 64)
  size_t ptc_bytes = 0;
  size_t pws_bytes = 0;
  // host-call staging
  void* d_stage = nullptr;
  size_t stage_bytes = 0;
  dvw_info info{};
  uint64_t* trace = nullptr;
  int64_t trace_n0 = 0;
  int trace_count = 0;
};

namespace {

thread_local std::string g_err;

dvw_status fail(dvw_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
dvw_status fail(dvw_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

}  // namespace

void dvw::note_error(const char* text) { g_err = text; }

namespace {

dvw_status cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return fail(DVW_E_OOM, "%s: %s", what, cudaGetErrorString(e));
  }
  return fail(DVW_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define DVW_CUDA(call, what)                        \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

dvw_status check_config(const dvw_config* c) {
  if (!c) return fail(DVW_E_INVALID_ARG, "config is NULL");
  if (c->n_layers < 1) return fail(DVW_E_SHAPE, "n_layers must be >= 1 (got %d)", c->n_layers);
  if (c->levels != kLevels) return fail(DVW_E_UNSUPPORTED, "levels must be 256 (got %d)", c->levels);
  if (c->residual != 32 && c->residual != 64 && c->residual != 128)
    return fail(DVW_E_UNSUPPORTED, "residual must be 32, 64 or 128 (got %d)", c->residual);
  if (c->skip != 128 && c->skip != 256)
    return fail(DVW_E_UNSUPPORTED, "skip must be 128 or 256 (got %d)", c->skip);
  if (c->dilations) {
    for (int j = 0; j < c->n_layers; ++j)
      if (c->dilations[j] < 1) return fail(DVW_E_SHAPE, "dilation[%d] = %d < 1", j, c->dilations[j]);
  }
  return DVW_OK;
}

dvw_status ensure_ring(dvw_model* m, int n_streams) {
  if (m->ring_streams >= n_streams) return DVW_OK;
  if (m->d_ring) cudaFree(m->d_ring);
  m->d_ring = nullptr;
  m->ring_streams = 0;
  const size_t bytes = sizeof(float) * (size_t)m->ring_floats * n_streams;
  DVW_CUDA(cudaMalloc(&m->d_ring, bytes), "allocating dilation queues");
  m->ring_streams = n_streams;
  m->info.workspace_bytes = (int64_t)bytes;
  return DVW_OK;
}

// The error word is mapped pinned host memory written by the kernels' watchdogs,
// so checking it never synchronizes the stream.
dvw_status check_device_error(dvw_model* m) {
  const int h = *m->h_err;
  if (h != 0) {
    *m->h_err = 0;
    return fail(DVW_E_DEVICE_TIMEOUT, "device watchdog fired (code %d): a persistent kernel spin-wait timed out", h);
  }
  return DVW_OK;
}

// AUTO: batches up to this many streams run on the cluster kernel; larger batches on the batched
// tensor-core kernel (or the stream kernel).  Up to max_clusters streams get one cluster each; more
// streams run interleaved, up to 8 per cluster (the multi-stream variant, exact gate only), whose
// aggregate is flat from ~56 streams on while the batched kernel's grows with the batch.  Crossover
// measured on B200 (profiles/r2_auto_crossover.txt): C2 shape (LP = 3) cluster 2.48 M vs tc 1.64 M
// samples/s at 256 streams, 2.70 M vs 2.85 M at 448; C5 shape (LP = 4) 1.09 M vs 0.87 M at 256,
// 1.09 M vs 1.70 M at 512 -- hence 60 (LP = 3) / 48 (LP = 4) streams per co-resident cluster.
constexpr int kClusterWaves = 16;
int cluster_streams(const dvw_model* m, bool session = false) {
  if (!m->cplan.ok) return 0;
  if (m->trace) return 1;
  if (m->cplan.pipe_ok && m->precision == DVW_PRECISION_FP32 && !session)  // sessions: one stream per cluster
    return (m->cplan.lpc == 3 ? 60 : 48) * m->cplan.max_clusters_pipe;
  return kClusterWaves * m->cplan.max_clusters;
}

dvw_status run(dvw_model* m, const float* cond, int64_t n_frames, int32_t hop, const float* uniforms,
               const uint8_t* forced, int64_t n_samples, int32_t n_streams, uint8_t* out_codes,
               float* out_logits, void* stream, dvw_session* sess = nullptr) {
  if (!m) return fail(DVW_E_INVALID_ARG, "model is NULL");
  if (!m->loaded) return fail(DVW_E_STATE, "weights not loaded (call dvw_load_weights first)");
  if (n_samples < 0) return fail(DVW_E_SHAPE, "n_samples must be >= 0");
  if (n_streams < 1) return fail(DVW_E_SHAPE, "n_streams must be >= 1 (got %d)", n_streams);
  if (hop < 1) return fail(DVW_E_SHAPE, "hop must be >= 1 (got %d)", hop);
  const int64_t n0 = sess ? sess->n_done : 0;  // sessions: cond holds the whole utterance
  if (n_samples > 0 && n_frames < (n0 + n_samples + hop - 1) / hop)
    return fail(DVW_E_SHAPE, "n_frames = %lld < ceil(%s / hop) = %lld", (long long)n_frames,
                sess ? "(samples so far + n_samples)" : "n_samples", (long long)((n0 + n_samples + hop - 1) / hop));
  if (n_samples == 0) return DVW_OK;
  if (!cond) return fail(DVW_E_INVALID_ARG, "cond is NULL");
  if (forced) {
    if (!out_logits) return fail(DVW_E_INVALID_ARG, "out_logits is NULL");
  } else {
    if (!uniforms) return fail(DVW_E_INVALID_ARG, "uniforms is NULL");
    if (!out_codes) return fail(DVW_E_INVALID_ARG, "out_codes is NULL");
  }
  DeviceGuard g(m->device);
  dvw_status st = check_device_error(m);
  if (st != DVW_OK) return st;
  int kern = m->kernel;
  const bool direct = forced != nullptr || m->samp_kind == DVW_SAMPLER_DIRECT;
  if (kern == DVW_KERNEL_CLUSTER && !direct)
    return fail(DVW_E_UNSUPPORTED, "the cluster kernel samples directly only (dvw_set_sampler)");
  if (kern == DVW_KERNEL_PARALLEL && !forced)
    return fail(DVW_E_UNSUPPORTED, "the parallel kernel computes teacher-forced logits only (dvw_logits)");
  if (kern == DVW_KERNEL_AUTO && forced) kern = DVW_KERNEL_PARALLEL;
  if (sess) {
    // the cluster kernel's session variant evaluates the exact gate only
    const bool exact = m->precision == DVW_PRECISION_FP32 || m->precision == DVW_PRECISION_TF32;
    if (kern == DVW_KERNEL_CLUSTER && !exact)
      return fail(DVW_E_UNSUPPORTED, "cluster-kernel sessions run the exact gate (use the STREAM kernel)");
    if (kern == DVW_KERNEL_AUTO) {
      // re-resolved on every call: CLUSTER and STREAM share the queue and code-history layout,
      // so a session that started on CLUSTER moves to STREAM when the sampler or precision
      // changes to something the cluster kernel's session variant does not run (and back)
      if (sess->kernel == DVW_KERNEL_TC) kern = DVW_KERNEL_TC;
      else if (sess->kernel == DVW_KERNEL_STREAM && n_streams > 1) kern = DVW_KERNEL_STREAM;
      else if (n_streams <= cluster_streams(m, true) && direct && exact) kern = DVW_KERNEL_CLUSTER;
      else if (n_streams > 1 && m->bplan.ok && m->precision != DVW_PRECISION_APPC) kern = DVW_KERNEL_TC;
      else kern = DVW_KERNEL_STREAM;
    }
    // a session's state (queues, code history) is laid out by the kernel that started it
    if (sess->kernel != 0 && kern != sess->kernel &&
        !((kern == DVW_KERNEL_CLUSTER || kern == DVW_KERNEL_STREAM) &&
          (sess->kernel == DVW_KERNEL_CLUSTER || sess->kernel == DVW_KERNEL_STREAM)))
      return fail(DVW_E_STATE, "this session was started on kernel %d and cannot continue on kernel %d",
                  sess->kernel, kern);
  }
  if (kern == DVW_KERNEL_TC && m->precision == DVW_PRECISION_APPC)
    return fail(DVW_E_UNSUPPORTED, "the App. C tier runs on the CLUSTER, STREAM and PARALLEL kernels");
  if (kern == DVW_KERNEL_AUTO) {
    if (n_streams <= cluster_streams(m) && direct) kern = DVW_KERNEL_CLUSTER;
    else if (n_streams > 1 && m->bplan.ok && m->precision != DVW_PRECISION_APPC) kern = DVW_KERNEL_TC;
    else kern = DVW_KERNEL_STREAM;
  }
  if (kern == DVW_KERNEL_CLUSTER && m->trace &&
      (m->precision == DVW_PRECISION_APPROX || m->precision == DVW_PRECISION_APPC))
    return fail(DVW_E_UNSUPPORTED, "tracing runs the exact-gate cluster kernel only (dvw_set_trace)");
  if (kern == DVW_KERNEL_CLUSTER && m->trace && n_streams > 1)
    return fail(DVW_E_UNSUPPORTED, "tracing records one stream (dvw_set_trace)");
  int pgroup = 0;  // parallel kernel: streams per workspace group
  if (kern == DVW_KERNEL_PARALLEL) {
    const size_t per = parallel_workspace_bytes(m->r, m->s, n_samples, 1);
    const size_t cap = std::max(per, (size_t)2 << 30);  // bound the workspace to ~2 GiB
    pgroup = (int)std::min<size_t>((size_t)n_streams, cap / per);
    const size_t need = per * pgroup;
    if (m->pws_bytes < need) {
      if (m->d_pws) cudaFree(m->d_pws);
      m->d_pws = nullptr;
      m->pws_bytes = 0;
      DVW_CUDA(cudaMalloc(&m->d_pws, need), "allocating parallel workspace");
      m->pws_bytes = need;
    }
  } else if (kern == DVW_KERNEL_TC && sess) {
    if (!sess->d_bws) {
      const size_t need = batch_session_bytes(m->bplan, m->dil.data(), n_streams);
      DVW_CUDA(cudaMalloc(&sess->d_bws, need), "allocating the session's batched workspace");
      sess->bws_bytes = need;
    }
  } else if (kern == DVW_KERNEL_TC) {
    const size_t need = batch_workspace_bytes(m->bplan, m->dil.data(), n_streams);
    if (m->bws_bytes < need) {
      if (m->d_bws) cudaFree(m->d_bws);
      m->d_bws = nullptr;
      m->bws_bytes = 0;
      DVW_CUDA(cudaMalloc(&m->d_bws, need), "allocating batched workspace");
      m->bws_bytes = need;
      m->info.workspace_bytes = (int64_t)need;
    }
  } else if (!sess) {
    st = ensure_ring(m, n_streams);
    if (st != DVW_OK) return st;
  }

  RunArgs A{};
  A.w = m->d_w;
  A.off = m->off;
  A.L = m->L;
  A.r = m->r;
  A.s = m->s;
  A.dil = m->d_dil;
  A.ring_off = m->d_ring_off;
  A.ring_floats = m->ring_floats;
  A.cond = cond;
  A.n_frames = n_frames;
  A.hop = hop;
  A.uniforms = uniforms;
  A.forced = forced;
  A.N = n_samples;
  A.n_streams = n_streams;
  A.out_codes = out_codes;
  A.out_logits = out_logits;
  A.ring = sess ? sess->d_ring : m->d_ring;
  A.n0 = n0;
  A.ystate = sess ? sess->d_y : nullptr;
  A.err = m->d_err;
  A.approx = m->precision == DVW_PRECISION_APPROX ? 1 : m->precision == DVW_PRECISION_APPC ? 2 : 0;
  A.samp_kind = forced ? DVW_SAMPLER_DIRECT : m->samp_kind;
  A.samp_inv_t = m->samp_inv_t;
  A.samp_topk = m->samp_topk;
  A.trace = m->trace;
  A.trace_n0 = m->trace_n0;
  A.trace_count = m->trace_count;
  // watchdog test hook: honoured only by the TRACE instantiation of the cluster kernel
  A.fault = (m->trace && getenv("DVW_FAULT_INJECT")) ? atoi(getenv("DVW_FAULT_INJECT")) : 0;

  LaunchInfo li{};
  cudaError_t e;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (kern == DVW_KERNEL_CLUSTER) {
    e = launch_cluster_kernel(A, m->cplan, m->d_packed, cs, &li);
  } else if (kern == DVW_KERNEL_STREAM) {
    e = launch_stream_kernel(A, cs, &li);
  } else if (kern == DVW_KERNEL_PARALLEL) {
    e = cudaSuccess;
    int64_t launches = 0;
    for (int g0 = 0; g0 < n_streams && e == cudaSuccess; g0 += pgroup) {
      RunArgs G = A;
      G.n_streams = std::min(pgroup, n_streams - g0);
      G.cond = cond + (int64_t)g0 * n_frames * m->L * 2 * m->r;
      G.forced = forced + (int64_t)g0 * n_samples;
      G.out_logits = out_logits + (int64_t)g0 * n_samples * kLevels;
      e = launch_parallel_logits(G, m->d_pws, cs, &li, static_cast<const float*>(m->d_ptc));
      launches += li.launches;
    }
    li.launches = launches;
  } else if (kern == DVW_KERNEL_TC) {
    e = sess ? launch_batch_kernel(A, m->bplan, m->d_bpacked, sess->d_bws, sess->bws_bytes, m->dil.data(),
                                   m->precision != DVW_PRECISION_FP32, cs, &li, true)
             : launch_batch_kernel(A, m->bplan, m->d_bpacked, m->d_bws, m->bws_bytes, m->dil.data(),
                                   m->precision != DVW_PRECISION_FP32, cs, &li);
  } else {
    return fail(DVW_E_UNSUPPORTED, "kernel %d is not available in this build", kern);
  }
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  if (sess) sess->kernel = kern;
  m->info.last_kernel = kern;
  m->info.last_grid = li.grid;
  m->info.last_cluster = li.cluster;
  m->info.last_threads = li.threads;
  m->info.last_launches = li.launches;
  m->info.streams_per_cluster = kern == DVW_KERNEL_CLUSTER ? li.rows_per_block : 0;
  return DVW_OK;
}

// Symmetric per-row quantisation of one row-major matrix to `bits`-bit integers and back
// (reading R32): s = max|row| / (2^(bits-1) - 1), W := rint(W / s) * s, fp32.
void quantize_rows(float* w, int64_t rows, int64_t cols, int bits) {
  const float qmax = (float)((1 << (bits - 1)) - 1);
  for (int64_t i = 0; i < rows; ++i) {
    float* row = w + i * cols;
    float mx = 0.0f;
    for (int64_t c = 0; c < cols; ++c) mx = std::max(mx, std::fabs(row[c]));
    if (mx == 0.0f) continue;
    const float sc = mx / qmax;
    for (int64_t c = 0; c < cols; ++c) row[c] = std::rint(row[c] / sc) * sc;
  }
}

// One scale for the whole matrix (reading R33, SPEC.md's QuantizedWeightSet): s = max|W| /
// (2^(bits-1) - 1), 1 for an all-zero matrix; W := rint(W / s) * s, fp32.
void quantize_tensor(float* w, int64_t rows, int64_t cols, int bits) {
  const float qmax = (float)((1 << (bits - 1)) - 1);
  float mx = 0.0f;
  for (int64_t i = 0; i < rows * cols; ++i) mx = std::max(mx, std::fabs(w[i]));
  const float sc = mx == 0.0f ? 1.0f : mx / qmax;
  for (int64_t i = 0; i < rows * cols; ++i) w[i] = std::rint(w[i] / sc) * sc;
}

void quantize_matrices(float* w, const Offsets& o, int L, int r, int s, int bits, int scheme) {
  auto q = [&](float* p, int64_t rows, int64_t cols) {
    if (scheme == DVW_QUANT_PER_TENSOR) quantize_tensor(p, rows, cols, bits);
    else quantize_rows(p, rows, cols, bits);
  };
  for (int j = 0; j < L; ++j) {
    float* lw = w + (int64_t)j * o.layer_stride;
    q(lw + o.w_prev, 2 * r, r);
    q(lw + o.w_cur, 2 * r, r);
    q(lw + o.w_res, r, r);
    q(lw + o.w_skip, s, r);
  }
  q(w + o.emb_prev, r, kLevels);
  q(w + o.emb_cur, r, kLevels);
  q(w + o.w_relu, kLevels, s);
  q(w + o.w_out, kLevels, kLevels);
}

}  // namespace

extern "C" {

DVW_API int64_t dvw_weights_numel(const dvw_config* cfg) {
  if (!cfg || cfg->n_layers < 1 || cfg->residual < 1 || cfg->skip < 1 || cfg->levels != kLevels) return -1;
  return make_offsets(cfg->n_layers, cfg->residual, cfg->skip).numel;
}

DVW_API dvw_status dvw_create(const dvw_config* cfg, dvw_model** out) {
  if (!out) return fail(DVW_E_INVALID_ARG, "out is NULL");
  dvw_status st = check_config(cfg);
  if (st != DVW_OK) return st;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (cfg->device < 0 || cfg->device >= ndev)
    return fail(DVW_E_INVALID_ARG, "device %d out of range (%d devices)", cfg->device, ndev);
  DeviceGuard g(cfg->device);
  dvw_model* m = new (std::nothrow) dvw_model();
  if (!m) return fail(DVW_E_OOM, "host allocation failed");
  m->device = cfg->device;
  m->L = cfg->n_layers;
  m->r = cfg->residual;
  m->s = cfg->skip;
  m->a = cfg->levels;
  m->dil.resize(m->L);
  m->ring_off.resize(m->L);
  int64_t acc = 0;
  for (int j = 0; j < m->L; ++j) {
    m->dil[j] = cfg->dilations ? cfg->dilations[j] : (1 << (j % 10));
    m->ring_off[j] = acc;
    acc += (int64_t)m->dil[j] * m->r;
  }
  m->ring_floats = acc;
  m->off = make_offsets(m->L, m->r, m->s);
  e = cudaMalloc(&m->d_dil, sizeof(int32_t) * m->L);
  if (e == cudaSuccess) e = cudaMalloc(&m->d_ring_off, sizeof(int64_t) * m->L);
  if (e == cudaSuccess) {
    int* hp = nullptr;
    e = cudaHostAlloc(reinterpret_cast<void**>(&hp), sizeof(int), cudaHostAllocMapped);
    if (e == cudaSuccess) {
      *hp = 0;
      m->h_err = hp;
      e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&m->d_err), hp, 0);
    }
  }
  if (e == cudaSuccess) e = cudaMemcpy(m->d_dil, m->dil.data(), sizeof(int32_t) * m->L, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(m->d_ring_off, m->ring_off.data(), sizeof(int64_t) * m->L, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    dvw_destroy(m);
    return cuda_fail(e, "dvw_create device setup");
  }
  m->cplan = plan_cluster(m->L, m->r, m->s, m->device);
  m->info.chain_ctas = m->cplan.ok ? m->cplan.nc : 0;
  m->info.max_clusters = m->cplan.ok ? m->cplan.max_clusters : 0;
  m->info.max_clusters_pipe = m->cplan.ok && m->cplan.pipe_ok ? m->cplan.max_clusters_pipe : 0;
  m->bplan = plan_batch(m->L, m->r, m->s, m->device);
  *out = m;
  return DVW_OK;
}

DVW_API dvw_status dvw_load_weights(dvw_model* m, const float* blob, int64_t numel, int32_t blob_on_device) {
  if (!m) return fail(DVW_E_INVALID_ARG, "model is NULL");
  if (!blob) return fail(DVW_E_INVALID_ARG, "blob is NULL");
  if (numel != m->off.numel)
    return fail(DVW_E_SHAPE, "weight blob has %lld floats, expected %lld", (long long)numel,
                (long long)m->off.numel);
  DeviceGuard g(m->device);
  std::vector<float> host;
  const float* hp = blob;
  if (blob_on_device) {
    host.resize(numel);
    DVW_CUDA(cudaMemcpy(host.data(), blob, sizeof(float) * numel, cudaMemcpyDeviceToHost), "reading device blob");
    hp = host.data();
  }
  for (int64_t i = 0; i < numel; ++i)
    if (!std::isfinite(hp[i])) return fail(DVW_E_INVALID_ARG, "weight %lld is not finite", (long long)i);
  if (m->weight_bits != 0) {  // row f4: quantise the matrices (include/dvw.h dvw_set_weight_bits)
    if (host.empty()) host.assign(blob, blob + numel);
    quantize_matrices(host.data(), m->off, m->L, m->r, m->s, m->weight_bits, m->quant_scheme);
    hp = host.data();
  }
  if (!m->d_w) DVW_CUDA(cudaMalloc(&m->d_w, sizeof(float) * numel), "allocating weights");
  DVW_CUDA(cudaMemcpy(m->d_w, hp, sizeof(float) * numel, cudaMemcpyHostToDevice), "uploading weights");
  int64_t wb = sizeof(float) * numel;
  if (m->cplan.ok) {
    size_t need = packed_bytes(m->cplan);
    if (m->d_packed && m->packed_bytes < need) {
      cudaFree(m->d_packed);
      m->d_packed = nullptr;
    }
    if (!m->d_packed) {
      DVW_CUDA(cudaMalloc(&m->d_packed, need), "allocating packed weights");
      m->packed_bytes = need;
    }
    DVW_CUDA(pack_cluster_weights(m->cplan, hp, m->off, m->d_packed), "packing weights");
    wb += (int64_t)need;
  }
  if (m->r == 64 || m->r == 128) {  // tensor-core images for the parallel teacher-forced pass
    const size_t need = sizeof(float) * (size_t)parallel_tc_packed_floats(m->L, m->r, m->s);
    if (m->d_ptc && m->ptc_bytes < need) {
      cudaFree(m->d_ptc);
      m->d_ptc = nullptr;
    }
    if (!m->d_ptc) {
      DVW_CUDA(cudaMalloc(&m->d_ptc, need), "allocating tensor-core layer images");
      m->ptc_bytes = need;
    }
    DVW_CUDA(pack_parallel_tc(hp, m->off, m->L, m->r, m->s, m->d_ptc), "packing tensor-core layer images");
    wb += (int64_t)need;
  }
  if (m->bplan.ok) {
    const size_t need = sizeof(float) * (size_t)m->bplan.total;
    if (m->d_bpacked && m->bpacked_bytes < need) {
      cudaFree(m->d_bpacked);
      m->d_bpacked = nullptr;
    }
    if (!m->d_bpacked) {
      DVW_CUDA(cudaMalloc(&m->d_bpacked, need), "allocating batched tile weights");
      m->bpacked_bytes = need;
    }
    DVW_CUDA(pack_batch_weights(m->bplan, hp, m->off, m->d_bpacked), "packing batched tile weights");
    wb += (int64_t)need;
  }
  m->info.weight_bytes = wb;
  m->loaded = true;
  return DVW_OK;
}

DVW_API dvw_status dvw_generate(dvw_model* m, const float* cond, int64_t n_frames, int32_t hop,
                                const float* uniforms, int64_t n_samples, int32_t n_streams,
                                uint8_t* out_codes, void* cuda_stream) {
  return run(m, cond, n_frames, hop, uniforms, nullptr, n_samples, n_streams, out_codes, nullptr, cuda_stream);
}

DVW_API dvw_status dvw_logits(dvw_model* m, const float* cond, int64_t n_frames, int32_t hop,
                              const uint8_t* codes, int64_t n_samples, int32_t n_streams, float* out_logits,
                              void* cuda_stream) {
  if (!codes && n_samples > 0) return fail(DVW_E_INVALID_ARG, "codes is NULL");
  return run(m, cond, n_frames, hop, nullptr, codes, n_samples, n_streams, nullptr, out_logits, cuda_stream);
}

DVW_API dvw_status dvw_generate_host(dvw_model* m, const float* cond_host, int64_t n_frames, int32_t hop,
                                     const float* uniforms_host, int64_t n_samples, int32_t n_streams,
                                     uint8_t* out_codes_host, void* cuda_stream) {
  if (!m) return fail(DVW_E_INVALID_ARG, "model is NULL");
  if (!cond_host || !uniforms_host || !out_codes_host) return fail(DVW_E_INVALID_ARG, "host buffer is NULL");
  if (n_streams < 1 || n_samples < 0 || n_frames < 0) return fail(DVW_E_SHAPE, "bad sizes");
  DeviceGuard g(m->device);
  const size_t cb = sizeof(float) * (size_t)n_streams * n_frames * m->L * 2 * m->r;
  const size_t ub = sizeof(float) * (size_t)n_streams * n_samples;
  const size_t ob = (size_t)n_streams * n_samples;
  const size_t need = ((cb + 255) & ~size_t(255)) + ((ub + 255) & ~size_t(255)) + ob + 256;
  if (m->stage_bytes < need) {
    if (m->d_stage) cudaFree(m->d_stage);
    m->d_stage = nullptr;
    m->stage_bytes = 0;
    DVW_CUDA(cudaMalloc(&m->d_stage, need), "allocating staging buffers");
    m->stage_bytes = need;
  }
  char* base = static_cast<char*>(m->d_stage);
  float* dc = reinterpret_cast<float*>(base);
  float* du = reinterpret_cast<float*>(base + ((cb + 255) & ~size_t(255)));
  uint8_t* dout = reinterpret_cast<uint8_t*>(base + ((cb + 255) & ~size_t(255)) + ((ub + 255) & ~size_t(255)));
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(cuda_stream);
  DVW_CUDA(cudaMemcpyAsync(dc, cond_host, cb, cudaMemcpyHostToDevice, cs), "H2D cond");
  DVW_CUDA(cudaMemcpyAsync(du, uniforms_host, ub, cudaMemcpyHostToDevice, cs), "H2D uniforms");
  dvw_status st = dvw_generate(m, dc, n_frames, hop, du, n_samples, n_streams, dout, cuda_stream);
  if (st != DVW_OK) return st;
  DVW_CUDA(cudaMemcpyAsync(out_codes_host, dout, ob, cudaMemcpyDeviceToHost, cs), "D2H codes");
  DVW_CUDA(cudaStreamSynchronize(cs), "synchronizing");
  return check_device_error(m);
}

DVW_API dvw_status dvw_session_create(dvw_model* m, int32_t n_streams, dvw_session** out) {
  if (!m || !out) return fail(DVW_E_INVALID_ARG, "NULL argument");
  if (n_streams < 1) return fail(DVW_E_SHAPE, "n_streams must be >= 1 (got %d)", n_streams);
  DeviceGuard g(m->device);
  dvw_session* s = new (std::nothrow) dvw_session();
  if (!s) return fail(DVW_E_OOM, "host allocation failed");
  s->device = m->device;
  s->n_streams = n_streams;
  s->ring_floats = m->ring_floats;
  cudaError_t e = cudaMalloc(&s->d_ring, sizeof(float) * (size_t)m->ring_floats * n_streams);
  if (e == cudaSuccess) e = cudaMemset(s->d_ring, 0, sizeof(float) * (size_t)m->ring_floats * n_streams);
  if (e == cudaSuccess) e = cudaMalloc(&s->d_y, sizeof(int) * 2 * n_streams);
  if (e == cudaSuccess) {
    std::vector<int> y(2 * (size_t)n_streams, kLevels / 2);  // codes at negative times: 128 (R4)
    e = cudaMemcpy(s->d_y, y.data(), sizeof(int) * y.size(), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    cudaFree(s->d_ring);
    cudaFree(s->d_y);
    delete s;
    return cuda_fail(e, "creating session");
  }
  *out = s;
  return DVW_OK;
}

DVW_API dvw_status dvw_session_generate(dvw_model* m, dvw_session* s, const float* cond, int64_t n_frames,
                                        int32_t hop, const float* uniforms, int64_t n_samples, uint8_t* out_codes,
                                        void* cuda_stream) {
  if (!m || !s) return fail(DVW_E_INVALID_ARG, "NULL argument");
  if (s->device != m->device || s->ring_floats != m->ring_floats)
    return fail(DVW_E_INVALID_ARG, "session belongs to another model");
  if (s->hop != 0 && hop != s->hop) return fail(DVW_E_SHAPE, "hop changed within a session (%d -> %d)", s->hop, hop);
  dvw_status st = run(m, cond, n_frames, hop, uniforms, nullptr, n_samples, s->n_streams, out_codes, nullptr,
                      cuda_stream, s);
  if (st == DVW_OK) {
    s->hop = hop;
    s->n_done += n_samples;
  }
  return st;
}

DVW_API int64_t dvw_session_position(const dvw_session* s) { return s ? s->n_done : -1; }

DVW_API void dvw_session_destroy(dvw_session* s) {
  if (!s) return;
  DeviceGuard g(s->device);
  cudaFree(s->d_ring);
  cudaFree(s->d_y);
  cudaFree(s->d_bws);
  delete s;
}

DVW_API dvw_status dvw_set_kernel(dvw_model* m, int32_t kernel) {
  if (!m) return fail(DVW_E_INVALID_ARG, "model is NULL");
  if (kernel < DVW_KERNEL_AUTO || kernel > DVW_KERNEL_PARALLEL) return fail(DVW_E_INVALID_ARG, "unknown kernel %d", kernel);
  if (kernel == DVW_KERNEL_CLUSTER && !m->cplan.ok)
    return fail(DVW_E_UNSUPPORTED, "cluster kernel cannot hold this model: %s", m->cplan.why);
  if (kernel == DVW_KERNEL_TC && !m->bplan.ok)
    return fail(DVW_E_UNSUPPORTED, "batched kernel cannot run this model: %s", m->bplan.why);
  m->kernel = kernel;
  return DVW_OK;
}

DVW_API dvw_status dvw_set_weight_bits(dvw_model* m, int32_t bits) {
  if (!m) return fail(DVW_E_INVALID_ARG, "model is NULL");
  if (bits != 0 && bits != 8 && bits != 16) return fail(DVW_E_INVALID_ARG, "weight bits must be 0, 8 or 16 (got %d)", bits);
  m->weight_bits = bits;
  m->quant_scheme = DVW_QUANT_PER_ROW;
  return DVW_OK;
}

DVW_API dvw_status dvw_set_weight_quant(dvw_model* m, int32_t bits, int32_t scheme) {
  if (!m) return fail(DVW_E_INVALID_ARG, "model is NULL");
  if (scheme != DVW_QUANT_PER_ROW && scheme != DVW_QUANT_PER_TENSOR)
    return fail(DVW_E_INVALID_ARG, "unknown quantisation scheme %d", scheme);
  dvw_status st = dvw_set_weight_bits(m, bits);
  if (st == DVW_OK) m->quant_scheme = scheme;
  return st;
}

DVW_API dvw_status dvw_set_precision(dvw_model* m, int32_t precision) {
  if (!m) return fail(DVW_E_INVALID_ARG, "model is NULL");
  if (precision != DVW_PRECISION_FP32 && precision != DVW_PRECISION_TF32 && precision != DVW_PRECISION_APPROX &&
      precision != DVW_PRECISION_APPC)
    return fail(DVW_E_INVALID_ARG, "unknown precision %d", precision);
  m->precision = precision;
  return DVW_OK;
}

DVW_API dvw_status dvw_set_sampler(dvw_model* m, int32_t kind, float temperature, int32_t top_k) {
  if (!m) return fail(DVW_E_INVALID_ARG, "model is NULL");
  if (kind < DVW_SAMPLER_DIRECT || kind > DVW_SAMPLER_TOP_K) return fail(DVW_E_INVALID_ARG, "unknown sampler %d", kind);
  if (kind == DVW_SAMPLER_TEMPERATURE && !(std::isfinite(temperature) && temperature > 0.0f))
    return fail(DVW_E_INVALID_ARG, "temperature must be finite and > 0 (got %g)", (double)temperature);
  if (kind == DVW_SAMPLER_TOP_K && (top_k < 1 || top_k > kLevels))
    return fail(DVW_E_INVALID_ARG, "top_k must be in [1, 256] (got %d)", top_k);
  m->samp_kind = kind;
  m->samp_inv_t = kind == DVW_SAMPLER_TEMPERATURE ? 1.0f / temperature : 1.0f;
  m->samp_topk = kind == DVW_SAMPLER_TOP_K ? top_k : kLevels;
  return DVW_OK;
}

DVW_API dvw_status dvw_set_trace(dvw_model* m, uint64_t* device_buf, int64_t first_sample, int32_t n_samples) {
  if (!m) return fail(DVW_E_INVALID_ARG, "model is NULL");
  if (device_buf && (first_sample < 0 || n_samples < 1)) return fail(DVW_E_SHAPE, "bad trace window");
  m->trace = device_buf;
  m->trace_n0 = first_sample;
  m->trace_count = device_buf ? n_samples : 0;
  return DVW_OK;
}

DVW_API dvw_status dvw_measure_floor(int32_t device, dvw_floor* out) {
  if (!out) return fail(DVW_E_INVALID_ARG, "out is NULL");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return fail(DVW_E_INVALID_ARG, "device %d not available", device);
  }
  FloorProbe f{};
  DVW_CUDA(measure_floor(device, &f), "latency-floor probes");
  out->layer_cycles = f.layer_cycles;
  out->hop_cycles = f.hop_cycles;
  out->head_stage_cycles = f.head_stage_cycles;
  out->sampler_cycles = f.sampler_cycles;
  out->sm_ghz = f.sm_ghz;
  return DVW_OK;
}

DVW_API dvw_status dvw_get_info(const dvw_model* m, dvw_info* out) {
  if (!m || !out) return fail(DVW_E_INVALID_ARG, "NULL argument");
  *out = m->info;
  return DVW_OK;
}

DVW_API dvw_status dvw_sync(dvw_model* m) {
  if (!m) return fail(DVW_E_INVALID_ARG, "model is NULL");
  DeviceGuard g(m->device);
  DVW_CUDA(cudaDeviceSynchronize(), "synchronizing");
  return check_device_error(m);
}

DVW_API void dvw_destroy(dvw_model* m) {
  if (!m) return;
  DeviceGuard g(m->device);
  cudaFree(m->d_w);
  cudaFree(m->d_dil);
  cudaFree(m->d_ring_off);
  cudaFree(m->d_ring);
  if (m->h_err) cudaFreeHost(const_cast<int*>(m->h_err));
  cudaFree(m->d_packed);
  cudaFree(m->d_bpacked);
  cudaFree(m->d_bws);
  cudaFree(m->d_pws);
  cudaFree(m->d_ptc);
  cudaFree(m->d_stage);
  delete m;
}

DVW_API const char* dvw_last_error(void) { return g_err.c_str(); }

}  // extern "C"
