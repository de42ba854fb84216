// conditioner.cu -- the conditioning network on the GPU (App. A.2;
// SURVEY.md §8(f) row f2): two bidirectional fo-pooling QRNN layers with 2x1 convolutions,
// channel interleave, and a per-WaveNet-layer projection to the L^(j) the generator adds
// inside every layer (at frame rate; the generator repeats frame f for hop samples,
// PAPER.md:477).  The whole utterance is known up front, so everything but the pooling
// recurrence is parallel over frames:
//   k_gates : for every frame t, direction and gate, the 2x1 convolution over the input
//             sequence (forward taps x_{t-1}, x_t; backward taps x_{t+1}, x_t -- reading R28)
//             followed by tanh / sigmoid; a [T x 2 C_in] x [2 C_in x 3H] product per direction,
//             frames staged in shared memory, weights read through L1/L2;
//   k_pool  : one thread per (stream, direction, channel) runs h_t = f h_{t-1} + (1-f) h~_t,
//             z_t = o h_t over time (forward or reversed) -- the only sequential part;
//   k_proj  : interleave (channel 2i = forward i, 2i+1 = backward i, reading R29) and
//             L^(j)_t = P^(j) out_t + B^(j) (reading R30).
// fp32 with fixed summation orders (bitwise deterministic), accurate tanhf/expf.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <new>
#include <string>
#include <vector>

#include "dvw_internal.cuh"

namespace dvw {
namespace {

constexpr int kTT = 16;       // frames per k_gates / k_proj block
constexpr int kGThreads = 256;

// Offsets (floats) of the conditioner blob (include/dvw.h dvwc_load_weights).
struct COff {
  int64_t w[2][2], b[2][2];  // [qrnn layer][direction]
  int64_t P, BP, numel;
};

COff coff(int cin, int H, int L, int r) {
  COff o{};
  int64_t p = 0;
  for (int q = 0; q < 2; ++q) {
    const int c = q == 0 ? cin : 2 * H;
    for (int d = 0; d < 2; ++d) {
      o.w[q][d] = p;
      p += 3LL * 2 * H * c;
      o.b[q][d] = p;
      p += 3LL * H;
    }
  }
  o.P = p;
  p += (int64_t)L * 2 * r * 2 * H;
  o.BP = p;
  p += (int64_t)L * 2 * r;
  o.numel = p;
  return o;
}

// gates[s][d][t][3][H] (h~ = tanh, o and f = sigmoid) of one QRNN layer over x [S][T][C].
// Block: stream s, frames [t0, t0 + kTT); the frames t0-1 .. t0+kTT are staged in shared
// memory; thread -> (gate row = 3H x 2 directions, frame) pairs.
__global__ void __launch_bounds__(kGThreads) k_gates(const float* __restrict__ x, int T, int C, int H,
                                                       const float* __restrict__ W, int64_t wf, int64_t bf,
                                                       int64_t wb, int64_t bb, float* __restrict__ gates) {
  extern __shared__ float xs[];  // [kTT + 2][C]
  const int s = blockIdx.y, t0 = blockIdx.x * kTT;
  const float* xsrc = x + (int64_t)s * T * C;
  for (int i = threadIdx.x; i < (kTT + 2) * C; i += blockDim.x) {
    const int tt = t0 - 1 + i / C, c = i % C;
    xs[i] = (tt >= 0 && tt < T) ? xsrc[(int64_t)tt * C + c] : 0.0f;  // x_{-1} = x_T = 0 (h_0 = 0 start)
  }
  __syncthreads();
  const int d = blockIdx.z / 3, gate = blockIdx.z % 3;  // this block's direction and gate
  for (int job = threadIdx.x; job < H * kTT; job += blockDim.x) {
    const int ch = job % H, tl = job / H, t = t0 + tl;
    if (t >= T) continue;
    const int gh = gate * H + ch;
    const float* w = W + (d == 0 ? wf : wb);
    const float* w_old = w + (int64_t)(gh / H) * 2 * H * C + (int64_t)(gh % H) * C;  // tap 0: x_{t-1} / x_{t+1}
    const float* w_now = w_old + (int64_t)H * C;                                       // tap 1: x_t
    const float* x_old = xs + (d == 0 ? tl : tl + 2) * C;  // staged row of t-1 (forward) or t+1 (backward)
    const float* x_now = xs + (tl + 1) * C;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int c = 0;
    for (; c + 1 < C; c += 2) {
      a0 = fmaf(__ldg(w_old + c), x_old[c], a0);
      a1 = fmaf(__ldg(w_now + c), x_now[c], a1);
      a2 = fmaf(__ldg(w_old + c + 1), x_old[c + 1], a2);
      a3 = fmaf(__ldg(w_now + c + 1), x_now[c + 1], a3);
    }
    if (c < C) {
      a0 = fmaf(__ldg(w_old + c), x_old[c], a0);
      a1 = fmaf(__ldg(w_now + c), x_now[c], a1);
    }
    const float v = ((a0 + a2) + (a1 + a3)) + __ldg(W + (d == 0 ? bf : bb) + gh);
    const float g = (gh < H) ? tanhf(v) : 1.0f / (1.0f + expf(-v));  // h~ | o | f
    gates[(((int64_t)s * 2 + d) * T + t) * 3 * H + gh] = g;
  }
}

// fo-pooling: thread (s, d, channel); forward runs t = 0..T-1, backward
// t = T-1..0 (the forward rule on the reversed copy).  Output z [S][T][2H] = [forward | backward].
__global__ void k_pool(const float* __restrict__ gates, int S, int T, int H, float* __restrict__ z) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= S * 2 * H) return;
  const int s = id / (2 * H), d = (id / H) % 2, c = id % H;
  const float* g = gates + ((int64_t)s * 2 + d) * T * 3 * H;
  float h = 0.0f;
  int t = d == 0 ? 0 : T - 1;
  const int step = d == 0 ? 1 : -1;
  float ht = g[(int64_t)t * 3 * H + c], o = g[(int64_t)t * 3 * H + H + c], f = g[(int64_t)t * 3 * H + 2 * H + c];
  for (int k = 0; k < T; ++k, t += step) {
    float nht = 0.f, no = 0.f, nf = 0.f;
    if (k + 1 < T) {  // next frame's gates in flight while this one is pooled
      const float* gn = g + (int64_t)(t + step) * 3 * H;
      nht = gn[c];
      no = gn[H + c];
      nf = gn[2 * H + c];
    }
    h = f * h + (1.0f - f) * ht;
    z[((int64_t)s * T + t) * 2 * H + d * H + c] = o * h;
    ht = nht;
    o = no;
    f = nf;
  }
}

// L[s][t][j][i] = sum_k P[j][i][k] out_t[k] + B[j][i], out_t[2m] = z[t][m], out_t[2m+1] = z[t][H+m].
__global__ void __launch_bounds__(kGThreads) k_proj(const float* __restrict__ z, int T, int H, int L, int r2,
                                                      const float* __restrict__ P, const float* __restrict__ BP,
                                                      float* __restrict__ out) {
  extern __shared__ float zs[];  // [kTT][2H] interleaved
  const int s = blockIdx.y, t0 = blockIdx.x * kTT;
  for (int i = threadIdx.x; i < kTT * 2 * H; i += blockDim.x) {
    const int tl = i / (2 * H), k = i % (2 * H), t = t0 + tl;
    const int src = (k & 1) ? H + (k >> 1) : (k >> 1);
    zs[i] = t < T ? z[((int64_t)s * T + t) * 2 * H + src] : 0.0f;
  }
  __syncthreads();
  const int rows = L * r2, j = blockIdx.z;  // this block's WaveNet layer
  for (int job = threadIdx.x; job < r2 * kTT; job += blockDim.x) {
    const int row = j * r2 + job % r2, tl = job / r2, t = t0 + tl;
    if (t >= T) continue;
    const float* p = P + (int64_t)row * 2 * H;
    const float* v = zs + tl * 2 * H;
    float a0 = 0.f, a1 = 0.f;
    for (int k = 0; k < 2 * H; k += 2) {
      a0 = fmaf(__ldg(p + k), v[k], a0);
      a1 = fmaf(__ldg(p + k + 1), v[k + 1], a1);
    }
    out[((int64_t)s * T + t) * rows + row] = (a0 + a1) + __ldg(BP + row);
  }
}

dvw_status cfail(dvw_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
dvw_status cfail(dvw_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  note_error(buf);  // dvw_last_error() reports it
  return st;
}

}  // namespace
}  // namespace dvw

using namespace dvw;

struct dvwc_model {
  int cin = 0, H = 0, L = 0, r = 0, device = 0;
  COff off{};
  bool loaded = false;
  float* d_w = nullptr;
  float* d_ws = nullptr;  // gates + two z buffers
  size_t ws_bytes = 0;
};

extern "C" {

DVW_API int64_t dvwc_weights_numel(const dvwc_config* c) {
  if (!c || c->in_channels < 1 || c->hidden < 1 || c->n_layers < 1 || c->residual < 1) return -1;
  return coff(c->in_channels, c->hidden, c->n_layers, c->residual).numel;
}

DVW_API dvw_status dvwc_create(const dvwc_config* c, dvwc_model** out) {
  if (!c || !out) return cfail(DVW_E_INVALID_ARG, "NULL argument");
  if (c->in_channels < 1 || c->hidden < 1 || c->n_layers < 1 || c->residual < 1)
    return cfail(DVW_E_SHAPE, "conditioner sizes must be >= 1");
  // k_gates stages (kTT + 2) frames of C = in_channels (layer 1) or 2 hidden (layer 2) floats
  // in one block's shared memory (<= 227 KB on sm_100)
  constexpr int kMaxC = 232448 / (4 * (kTT + 2));
  if (c->hidden > 1024 || c->in_channels > kMaxC)
    return cfail(DVW_E_UNSUPPORTED, "hidden <= 1024, in_channels <= %d (shared-memory staging)", kMaxC);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || c->device < 0 || c->device >= ndev) {
    cudaGetLastError();
    return cfail(DVW_E_INVALID_ARG, "device %d not available", c->device);
  }
  dvwc_model* m = new (std::nothrow) dvwc_model();
  if (!m) return cfail(DVW_E_OOM, "host allocation failed");
  m->cin = c->in_channels;
  m->H = c->hidden;
  m->L = c->n_layers;
  m->r = c->residual;
  m->device = c->device;
  m->off = coff(m->cin, m->H, m->L, m->r);
  *out = m;
  return DVW_OK;
}

DVW_API dvw_status dvwc_load_weights(dvwc_model* m, const float* blob, int64_t numel, int32_t on_device) {
  if (!m || !blob) return cfail(DVW_E_INVALID_ARG, "NULL argument");
  if (numel != m->off.numel)
    return cfail(DVW_E_SHAPE, "conditioner blob has %lld floats, expected %lld", (long long)numel,
                 (long long)m->off.numel);
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  std::vector<float> host;
  const float* hp = blob;
  cudaError_t e = cudaSuccess;
  if (on_device) {
    host.resize(numel);
    e = cudaMemcpy(host.data(), blob, sizeof(float) * numel, cudaMemcpyDeviceToHost);
    hp = host.data();
  }
  for (int64_t i = 0; e == cudaSuccess && i < numel; ++i)
    if (!std::isfinite(hp[i])) {
      if (prev >= 0) cudaSetDevice(prev);
      return cfail(DVW_E_INVALID_ARG, "conditioner weight %lld is not finite", (long long)i);
    }
  if (e == cudaSuccess && !m->d_w) e = cudaMalloc(&m->d_w, sizeof(float) * numel);
  if (e == cudaSuccess) e = cudaMemcpy(m->d_w, hp, sizeof(float) * numel, cudaMemcpyHostToDevice);
  if (prev >= 0) cudaSetDevice(prev);
  if (e != cudaSuccess) return cfail(DVW_E_CUDA, "conditioner weights: %s", cudaGetErrorString(e));
  m->loaded = true;
  return DVW_OK;
}

DVW_API dvw_status dvwc_run(dvwc_model* m, const float* features, int64_t n_frames, int32_t n_streams,
                            float* out_cond, void* cuda_stream) {
  if (!m) return cfail(DVW_E_INVALID_ARG, "model is NULL");
  if (!m->loaded) return cfail(DVW_E_STATE, "conditioner weights not loaded");
  if (n_frames < 0 || n_streams < 1) return cfail(DVW_E_SHAPE, "n_frames >= 0 and n_streams >= 1 required");
  if (n_frames == 0) return DVW_OK;
  if (!features || !out_cond) return cfail(DVW_E_INVALID_ARG, "NULL buffer");
  if (n_frames > (1LL << 30)) return cfail(DVW_E_SHAPE, "too many frames");
  const int T = (int)n_frames, S = n_streams, H = m->H;
  const size_t gates = (size_t)S * 2 * T * 3 * H, zsz = (size_t)S * T * 2 * H;
  const size_t need = sizeof(float) * (gates + 2 * zsz);
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  cudaError_t e = cudaSuccess;
  if (m->ws_bytes < need) {
    cudaFree(m->d_ws);
    m->d_ws = nullptr;
    m->ws_bytes = 0;
    e = cudaMalloc(&m->d_ws, need);
    if (e == cudaSuccess) m->ws_bytes = need;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  if (e == cudaSuccess) {
    float* g = m->d_ws;
    float* z[2] = {m->d_ws + gates, m->d_ws + gates + zsz};
    const float* in = features;
    int C = m->cin;
    const dim3 grid((T + kTT - 1) / kTT, S);
    const dim3 ggrid((T + kTT - 1) / kTT, S, 6);  // x (direction, gate)
    for (int q = 0; q < 2 && e == cudaSuccess; ++q) {
      const size_t sm = sizeof(float) * (kTT + 2) * C;
      if (sm > 48 * 1024) e = cudaFuncSetAttribute(k_gates, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) break;
      k_gates<<<ggrid, kGThreads, sm, st>>>(in, T, C, H, m->d_w, m->off.w[q][0], m->off.b[q][0], m->off.w[q][1],
                                           m->off.b[q][1], g);
      k_pool<<<(S * 2 * H + 127) / 128, 128, 0, st>>>(g, S, T, H, z[q]);
      e = cudaGetLastError();
      in = z[q];
      C = 2 * H;
    }
    if (e == cudaSuccess) {
      const size_t sm = sizeof(float) * kTT * 2 * H;
      if (sm > 48 * 1024) e = cudaFuncSetAttribute(k_proj, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e == cudaSuccess) {
        k_proj<<<dim3(grid.x, grid.y, m->L), kGThreads, sm, st>>>(z[1], T, H, m->L, 2 * m->r, m->d_w + m->off.P, m->d_w + m->off.BP,
                                            out_cond);
        e = cudaGetLastError();
      }
    }
  }
  if (prev >= 0) cudaSetDevice(prev);
  if (e != cudaSuccess) return cfail(DVW_E_CUDA, "conditioner launch: %s", cudaGetErrorString(e));
  return DVW_OK;
}

DVW_API void dvwc_destroy(dvwc_model* m) {
  if (!m) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  cudaFree(m->d_w);
  cudaFree(m->d_ws);
  if (prev >= 0) cudaSetDevice(prev);
  delete m;
}

}  // extern "C"
