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

// Records the thread-local text dvw_last_error() returns (dvw_api.cu).
void note_error(const char* text);

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
  int64_t n0;            // streaming sessions: global index of this call's first sample (0 otherwise)
  int* ystate;           // streaming sessions: [S][2] codes y_{n0-1}, y_{n0-2} in, y_{n0+N-1}, y_{n0+N-2}
                         // out; the dilation queues are flushed at the end (nullptr: one-shot call)
  uint8_t* out_codes;    // [S][N] or nullptr
  float* out_logits;     // [S][N][256] or nullptr
  float* ring;           // [S][ring_floats] workspace
  int* err;              // device error word (0 = ok)
  int approx;            // 1: DVW_PRECISION_APPROX (hardware tanh gate); 2: DVW_PRECISION_APPC (App. C)
  int samp_kind;         // App. A.4 strategy (dvw_sampler): 0 direct, 1 temperature, 2 mean, 3 mode, 4 top-k
  float samp_inv_t;      // 1 / temperature
  int samp_topk;         // k of top-k
  uint64_t* trace;       // optional %globaltimer trace [trace_count][16 CTAs][32 events] (dvw_set_trace)
  int64_t trace_n0;
  int trace_count;
  int fault;             // test hook (TRACE instantiation only): 1 = the heads drop sample trace_n0's
                         // logits hand-off, so CTA 0's spin-wait must end in the watchdog
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

// The approximate tier (DVW_PRECISION_APPROX; the GPU analogue of the paper's App. C
// approximations): the hardware tanh unit (tanh.approx.f32, relative
// error ~2^-11) for both halves, sigma(g) = 0.5 tanh(g / 2) + 0.5.  Two MUFU operations in
// parallel instead of two dependent pairs: a shorter gate on the critical chain, at the
// price of bit-exact sampling (measured per-step mismatch rate reported by bench.py).
__device__ __forceinline__ float gate_approx(float a, float g) {
  float ta, tg;
  asm("tanh.approx.f32 %0, %1;" : "=f"(ta) : "f"(a));
  asm("tanh.approx.f32 %0, %1;" : "=f"(tg) : "f"(0.5f * g));
  return ta * fmaf(0.5f, tg, 0.5f);
}

// The paper's own approximations (DVW_PRECISION_APPC; App. C, row f4;
// reading R31).  e~(x) = 1 + |x| + 0.5658 x^2 + 0.143 x^4;
//   tanh(x) ~ sign(x) (e~ - 1/e~) / (e~ + 1/e~), evaluated as
//             sign(x) (1 - r^2) / (1 + r^2) with r = 1/e~ (the same value; no inf/inf)
//   sigma(x) ~ e~ / (1 + e~) (x >= 0), 1 / (1 + e~) (x <= 0), i.e.
//             1 / (1 + r) and r / (1 + r)
// The divisions are the hardware reciprocal (rcp.approx, ~1 ulp): the approximation's own
// error is 1.5e-3 / 2.5e-3, and the GPU still evaluates the oracle's formula to ~1e-7
// (IEEE division here cost 0.9 us per C2 sample on the critical chain).
__device__ __forceinline__ float appc_etilde(float x) {
  const float x2 = x * x;
  return fmaf(0.143f * x2, x2, fmaf(0.5658f, x2, 1.0f + fabsf(x)));
}
__device__ __forceinline__ float fast_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float tanh_appc(float x) {
  const float r = fast_rcp(appc_etilde(x)), r2 = r * r;
  return copysignf((1.0f - r2) * fast_rcp(1.0f + r2), x);
}
__device__ __forceinline__ float sigmoid_appc(float x) {
  const float r = fast_rcp(appc_etilde(x)), d = fast_rcp(1.0f + r);
  return x >= 0.0f ? d : r * d;
}
__device__ __forceinline__ float gate_appc(float a, float g) { return tanh_appc(a) * sigmoid_appc(g); }

// e^x for x <= 0 by App. C.2: 2^x' with x' = x / ln 2 written straight
// into an fp32 bit pattern, I = (x' + 126 + g(z)) 2^23, z = x' - floor(x'),
// g(z) ~ -4.7259162 + 27.7280233 / (4.84252568 - z) - 1.49012907 z.  Evaluated as
// (floor(x') + 127) 2^23 + trunc((z + g(z) - 1) 2^23) so the integer part is exact (a carry
// out of the fraction near z -> 1 moves into the exponent, as in the paper's formula);
// x' < -126 (below the normal range) -> 0 (reading R31).
__device__ __forceinline__ float appc_exp(float x) {
  const float xl = x * 1.44269504f;
  if (!(xl >= -126.0f)) return 0.0f;
  const float fl = floorf(xl);
  const float z = xl - fl;
  const float g = __fsub_rn(__fadd_rn(-4.7259162f, __fdiv_rn(27.7280233f, 4.84252568f - z)), __fmul_rn(1.49012907f, z));
  const float t = __fsub_rn(__fadd_rn(z, g), 1.0f);
  return __int_as_float(((int)fl + 127) * 8388608 + (int)(t * 8388608.0f));
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
  int rows_per_block = 0;  // batched kernel: streams per stream block (cluster)
};

cudaError_t launch_stream_kernel(const RunArgs& a, cudaStream_t st, LaunchInfo* info);
// Teacher-forced logits in parallel over time (kernel_parallel.cu): workspace for a group of
// streams, then one call per group.
size_t parallel_workspace_bytes(int r, int s, int64_t n_samples, int n_streams);
// pk_tc: the tensor-core images (pack_parallel_tc), r = 64 or 128; nullptr -> SIMT layers and head.
cudaError_t launch_parallel_logits(const RunArgs& a, void* ws, cudaStream_t st, LaunchInfo* info,
                                   const float* pk_tc = nullptr);
// Tensor-core layer pass (kernel_parallel_tc.cu, r = 64 or 128): packed image size, host packing, one layer.
int64_t parallel_tc_packed_floats(int L, int r, int s);
cudaError_t pack_parallel_tc(const float* w, const Offsets& o, int L, int r, int s, void* dst);
cudaError_t launch_parallel_layer_tc(const RunArgs& a, int j, const float* xin, float* xout, float* q,
                                     const float* pk, cudaStream_t st);
cudaError_t launch_parallel_head_tc(const RunArgs& a, const float* q, const float* pk, cudaStream_t st);

#ifdef __CUDACC__
// ---------------------------------------------------------------- App. A.4 strategies (row f3)
// One warp draws from 256 logits, lane owns codes 8 lane .. 8 lane + 7 (l[i] = code 8 lane + i).
// fp64 running sums of e in ascending code order, then an fp64 warp scan of the lane totals;
// y = #{k : P_k <= u * P_255}; fallback the largest k with e_k > 0 (reading R11).
__device__ __forceinline__ int warp_cdf_draw(const float (&e)[8], float u, int lane) {
  double p[8];
  p[0] = (double)e[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) p[i] = p[i - 1] + (double)e[i];
  double incl = p[7];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const double base = incl - p[7];
  const double S = __shfl_sync(0xffffffffu, incl, 31);
  const double thr = (double)u * S;
  int cnt = 0, lastpos = -1;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    cnt += (base + p[i] <= thr) ? 1 : 0;
    if (e[i] > 0.0f) lastpos = 8 * lane + i;
  }
  const int y = __reduce_add_sync(0xffffffffu, cnt);
  return y < kLevels ? y : (int)__reduce_max_sync(0xffffffffu, (unsigned)(lastpos + 1)) - 1;
}

// float -> unsigned key with the same order (larger float, larger key)
__device__ __forceinline__ unsigned ordered_key(float v) {
  const unsigned b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// The draw under strategy `kind` (readings R24-R27, as the oracle):
// direct: e = exp(l - max l); temperature: e = exp((l - max l) / t); top-k: e = exp(l - max l)
// on the k largest logits (ties by lower code), 0 elsewhere -- each then drawn with u by
// warp_cdf_draw; mode: argmax (lowest code on ties); mean: floor(sum k e_k / sum e_k + 0.5).
// Every reduction has a fixed order (bitwise deterministic).
__device__ __forceinline__ int warp_sample_policy(const float (&l)[8], float u, int kind, float inv_t, int topk,
                                                  int lane, bool appc = false) {
  auto ex = [appc](float v) { return appc ? appc_exp(v) : expf(v); };  // App. C.2 under DVW_PRECISION_APPC
  float mx = fmaxf(fmaxf(fmaxf(l[0], l[1]), fmaxf(l[2], l[3])), fmaxf(fmaxf(l[4], l[5]), fmaxf(l[6], l[7])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float e[8];
  if (kind == 3) {  // mode
    float bv = l[0];
    int bi = 8 * lane;
#pragma unroll
    for (int i = 1; i < 8; ++i)
      if (l[i] > bv) { bv = l[i]; bi = 8 * lane + i; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    return bi;
  }
  if (kind == 2) {  // mean
    double S = 0.0, M = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double ei = (double)ex(l[i] - mx);
      S += ei;
      M += (double)(8 * lane + i) * ei;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      S += __shfl_xor_sync(0xffffffffu, S, o);
      M += __shfl_xor_sync(0xffffffffu, M, o);
    }
    const double y = floor(M / S + 0.5);
    return y < 0.0 ? 0 : (y > kLevels - 1 ? kLevels - 1 : (int)y);
  }
  if (kind == 1) {
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = ex((l[i] - mx) * inv_t);
    return warp_cdf_draw(e, u, lane);
  }
  if (kind == 4) {  // top-k: the k-th largest key by bisection on the ordered key, then ties by code
    unsigned key[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) key[i] = ordered_key(l[i]);
    unsigned T = 0;
#pragma unroll 1
    for (int bit = 31; bit >= 0; --bit) {
      const unsigned cand = T | (1u << bit);
      int c = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) c += key[i] >= cand ? 1 : 0;
      if ((int)__reduce_add_sync(0xffffffffu, (unsigned)c) >= topk) T = cand;
    }
    int gt = 0, eq = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      gt += key[i] > T ? 1 : 0;
      eq += key[i] == T ? 1 : 0;
    }
    const int need = topk - (int)__reduce_add_sync(0xffffffffu, (unsigned)gt);  // equal keys to keep
    int eq_before = eq;  // exclusive prefix of equal keys over lower lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, eq_before, o);
      if (lane >= o) eq_before += t;
    }
    eq_before -= eq;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      bool keep = key[i] > T;
      if (key[i] == T) {
        keep = eq_before < need;
        ++eq_before;
      }
      e[i] = keep ? ex(l[i] - mx) : 0.0f;
    }
    return warp_cdf_draw(e, u, lane);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) e[i] = ex(l[i] - mx);
  return warp_cdf_draw(e, u, lane);
}
#endif

}  // namespace dvw
