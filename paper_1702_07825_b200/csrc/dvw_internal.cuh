// dvw_internal.cuh -- shared declarations of the CUDA path (never of the oracle).
//
// Everything here is the product side: weight-blob offsets (restated from
// include/dvw.h, independently of oracle/dvw_oracle.c), the device helpers the
// kernels share (gate, sampler) and the launch entry points of each kernel.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dvw.h"

namespace dvw {

constexpr int kLevels = 256;  // a

// Offsets (in floats) into the raw roster-order blob (include/dvw.h "Load the weights").
struct Offsets {
  int64_t layer_stride;                          // floats per layer block
  int64_t w_prev, w_cur, b, w_res, b_res, w_skip;  // within a layer block
  int64_t emb_prev, emb_cur, b_emb, b_skip, w_relu, b_relu, w_out, b_out;  // global section
  int64_t numel;
};

inline Offsets make_offsets(int L, int r, int s) {
  Offsets o{};
  int64_t p = 0;
  o.w_prev = p; p += 2LL * r * r;
  o.w_cur = p;  p += 2LL * r * r;
  o.b = p;      p += 2LL * r;
  o.w_res = p;  p += 1LL * r * r;
  o.b_res = p;  p += r;
  o.w_skip = p; p += 1LL * s * r;
  o.layer_stride = p;
  p = o.layer_stride * L;
  o.emb_prev = p; p += 1LL * r * kLevels;
  o.emb_cur = p;  p += 1LL * r * kLevels;
  o.b_emb = p;    p += r;
  o.b_skip = p;   p += s;
  o.w_relu = p;   p += 1LL * kLevels * s;
  o.b_relu = p;   p += kLevels;
  o.w_out = p;    p += 1LL * kLevels * kLevels;
  o.b_out = p;    p += kLevels;
  o.numel = p;
  return o;
}

// Arguments common to every generation kernel.  All pointers are device pointers.
struct RunArgs {
  const float* w;        // raw roster-order weights
  Offsets off;
  int L, r, s;
  const int32_t* dil;    // [L]
  const int64_t* ring_off;  // [L] float offset of layer j's queue inside one stream's ring
  int64_t ring_floats;   // floats of ring state per stream (sum_j d_j * r)
  const float* cond;     // [S][F][L][2r]
  int64_t n_frames;
  int hop;
  const float* uniforms; // [S][N] (free running) or nullptr
  const uint8_t* forced; // [S][N] (teacher forced) or nullptr
  int64_t N;
  int n_streams;
  uint8_t* out_codes;    // [S][N] or nullptr
  float* out_logits;     // [S][N][256] or nullptr
  float* ring;           // [S][ring_floats] workspace
  int* err;              // device error word (0 = ok)
  uint64_t* trace;       // optional %globaltimer trace [trace_count][16 CTAs][32 events] (dvw_set_trace)
  int64_t trace_n0;
  int trace_count;
};

// ---------------------------------------------------------------- device helpers
#ifdef __CUDACC__
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Gated activation h = tanh(a_h) * sigma(a_g) (§5.1 step 2c).
// Accurate libdevice tanhf/expf: no fast-math (reading R13).
__device__ __forceinline__ float gate(float ah, float ag) {
  return tanhf(ah) * (1.0f / (1.0f + expf(-ag)));
}

// h = tanh(a) * sigma(g): tanh(a) = 1 - 2 / (1 + 2^(2a log2 e)),
// sigma(g) = 1 / (1 + 2^(-g log2 e)); MUFU ex2/rcp (rel. err ~2^-22) keep the
// result within ~1e-7 of the exact value; saturates correctly at +-inf.
__device__ __forceinline__ float gate_fast(float a, float g) {
  float ea, eg, ra, rg;
  const float xa = 2.8853900817779268f * a, xg = -1.4426950408889634f * g;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ea) : "f"(xa));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(eg) : "f"(xg));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(ea + 1.0f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rg) : "f"(eg + 1.0f));
  return fmaf(-2.0f, ra, 1.0f) * rg;
}

// Inverse-CDF direct sampling over a = 256 logits held one per thread by a
// 256-thread group ("Sample randomly from P(y)"; reading R11):
//   e_k = exp(l_k - max l) in fp32, P_k = fp64 inclusive running sum in ascending k,
//   y = min{k : u * P_255 < P_k}  (= number of k with P_k <= u * P_255, since P is
//   non-decreasing); fallback: the largest k with e_k > 0.
// `scratch` is >= 8 doubles + 8 floats of shared memory; `bar_id`/`nthreads`
// select the named barrier the 256 threads use (nthreads == 256).
// Fixed reduction order -> bitwise deterministic.
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ int sample_256(float logit, float u, double* dscratch, float* fscratch,
                                          int* iscratch, int k, int bar_id) {
  const int lane = k & 31, warp = k >> 5;
  float m = warp_max(logit);
  if (lane == 0) fscratch[warp] = m;
  named_sync(bar_id, 256);
  m = fscratch[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) m = fmaxf(m, fscratch[w]);
  const float e = expf(logit - m);
  // inclusive fp64 scan: warp level, then warp totals
  double p = (double)e;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_up_sync(0xffffffffu, p, o);
    if (lane >= o) p += t;
  }
  if (lane == 31) dscratch[warp] = p;
  named_sync(bar_id, 256);
  double base = 0.0, S = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const double t = dscratch[w];
    if (w < warp) base += t;
    S += t;
  }
  p += base;
  const double thr = (double)u * S;
  const unsigned below = __ballot_sync(0xffffffffu, !(thr < p));
  const unsigned pos = __ballot_sync(0xffffffffu, e > 0.0f);
  if (lane == 0) {
    iscratch[warp] = __popc(below);
    iscratch[8 + warp] = pos ? (warp * 32 + 31 - __clz(pos)) : -1;
  }
  named_sync(bar_id, 256);
  int cnt = 0, last = -1;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    cnt += iscratch[w];
    last = max(last, iscratch[8 + w]);
  }
  return cnt < 256 ? cnt : last;
}
#endif

// ---------------------------------------------------------------- kernel entry points
// Each returns cudaSuccess or the launch error; grid/cluster/threads are reported back.
struct LaunchInfo {
  int grid = 0, cluster = 1, threads = 0;
  int64_t launches = 0;
};

cudaError_t launch_stream_kernel(const RunArgs& a, cudaStream_t st, LaunchInfo* info);

}  // namespace dvw
