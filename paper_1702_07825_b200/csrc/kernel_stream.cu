// kernel_stream.cu -- the general "one CTA per stream" generation kernel.
//
// One persistent CTA of 256 threads owns one utterance (stream) and runs the
// whole autoregressive loop (§5.1 steps 1-3) for all N
// samples in a single launch.  Weights stay in the raw roster layout in HBM and
// are re-read every sample through L2 (they are 2.8-10 MB, far below the 126 MB
// L2), so this kernel is L2-latency-bound at batch 1; it exists as the
// general-shape path (every supported l, r, s) and as the independent second
// implementation the cluster kernel is checked against.  Warps issue the loads
// of 8 weight rows before reducing any of them so each L2 round trip is paid
// once per 8 rows, not once per row.
//
// Per sample n (warp-per-row matvecs, lanes over columns, vectors in registers):
//   a1  x = W_emb_prev[:, y_{n-2}] + W_emb_cur[:, y_{n-1}] + B_emb
//   per layer j:
//   a2  xp = x^{(j-1)}_{n-d_j} from the dilation queue (0 if n < d_j), then
//       queue slot n mod d_j := x^{(j-1)}_n
//   a3-a5 a = W_prev xp + W_cur x + B + L^{(j)}_{n/hop};  h = tanh * sigma
//   a6  x += W_res h + B_res
//   a7  q += W_skip h
//   a8  z_s = relu(q); z_a = relu(W_relu z_s + B_relu); l = W_out z_a + B_out
//   a9  y = inverse-CDF draw (or the forced code)
#include "dvw_internal.cuh"

namespace dvw {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRB = 8;  // rows per batch of outstanding loads

template <int K>
struct Vec {  // a K-vector spread over a warp: lane holds elements [lane*E, lane*E+E)
  static constexpr int E = K / 32;
  float v[E];
  __device__ __forceinline__ void load_smem(const float* p, int lane) {
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = p[lane * E + e];
  }
};

template <int E>
__device__ __forceinline__ void ld_row(const float* p, float (&dst)[E]) {
  if constexpr (E == 4) {
    float4 t = __ldg(reinterpret_cast<const float4*>(p));
    dst[0] = t.x; dst[1] = t.y; dst[2] = t.z; dst[3] = t.w;
  } else if constexpr (E == 2) {
    float2 t = __ldg(reinterpret_cast<const float2*>(p));
    dst[0] = t.x; dst[1] = t.y;
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) dst[e] = __ldg(p + e);
  }
}

// out(row, dot(W1[row], v1) [+ dot(W2[row], v2)]) for rows = warp, warp+8, ... < nrows.
// Deterministic: per-lane FMA order fixed, then a fixed butterfly.
template <int K, bool TWO, typename Epi>
__device__ __forceinline__ void warp_rows(const float* W1, const float* W2, int nrows, const Vec<K>& v1,
                                          const Vec<K>& v2, int warp, int lane, Epi epi) {
  constexpr int E = K / 32;
  for (int base = warp; base < nrows; base += kWarps * kRB) {
    float a[kRB][E], b[kRB][E];
#pragma unroll
    for (int i = 0; i < kRB; ++i) {
      const int row = base + i * kWarps;
      if (row < nrows) {
        ld_row<E>(W1 + (int64_t)row * K + lane * E, a[i]);
        if (TWO) ld_row<E>(W2 + (int64_t)row * K + lane * E, b[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < kRB; ++i) {
      const int row = base + i * kWarps;
      if (row < nrows) {
        float acc = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) acc = fmaf(a[i][e], v1.v[e], acc);
        if (TWO) {
#pragma unroll
          for (int e = 0; e < E; ++e) acc = fmaf(b[i][e], v2.v[e], acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) epi(row, acc);
      }
    }
  }
}

template <int R, int S>
__global__ void __launch_bounds__(kThreads, 1) k_stream(RunArgs A) {
  const int st = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int L = A.L;
  const Offsets& o = A.off;

  __shared__ double dscr[8];
  __shared__ int iscr[16];
  __shared__ float fscr[8];
  __shared__ __align__(16) float x[R], xp[R], av[2 * R], h[R], q[S], za[kLevels], lg[kLevels];

  const float* W = A.w;
  const float* cond = A.cond + (int64_t)st * A.n_frames * L * 2 * R;
  float* ring = A.ring + (int64_t)st * A.ring_floats;
  const float* uni = A.uniforms ? A.uniforms + (int64_t)st * A.N : nullptr;
  const uint8_t* forced = A.forced ? A.forced + (int64_t)st * A.N : nullptr;

  // codes at negative times: mu-law(0) = 128 (R4); a streaming session continues its history
  int y1 = A.ystate ? A.ystate[2 * st] : kLevels / 2, y2 = A.ystate ? A.ystate[2 * st + 1] : kLevels / 2;
  for (int64_t n = 0; n < A.N; ++n) {
    const int64_t ng = A.n0 + n;  // global sample index (queues, conditioning frame)
    const int64_t f = ng / A.hop;
    for (int i = tid; i < R; i += kThreads)
      x[i] = W[o.emb_prev + (int64_t)i * kLevels + y2] + W[o.emb_cur + (int64_t)i * kLevels + y1] +
             W[o.b_emb + i];
    for (int i = tid; i < S; i += kThreads) q[i] = W[o.b_skip + i];
    __syncthreads();

    for (int j = 0; j < L; ++j) {
      const float* Wl = W + (int64_t)j * o.layer_stride;
      const int d = A.dil[j];
      float* slot = ring + A.ring_off[j] + (int64_t)(ng % d) * R;
      for (int i = tid; i < R; i += kThreads) xp[i] = (ng >= d) ? slot[i] : 0.0f;
      __syncthreads();
      for (int i = tid; i < R; i += kThreads) slot[i] = x[i];
      const float* Lj = cond + (f * L + j) * 2 * R;
      {
        Vec<R> vx, vp;
        vx.load_smem(x, lane);
        vp.load_smem(xp, lane);
        warp_rows<R, true>(Wl + o.w_prev, Wl + o.w_cur, 2 * R, vp, vx, warp, lane,
                           [&](int row, float acc) { av[row] = acc + Wl[o.b + row] + Lj[row]; });
      }
      __syncthreads();
      for (int i = tid; i < R; i += kThreads) h[i] = A.approx == 0 ? gate(av[i], av[R + i])
                  : A.approx == 1 ? gate_approx(av[i], av[R + i]) : gate_appc(av[i], av[R + i]);
      __syncthreads();
      {
        Vec<R> vh;
        vh.load_smem(h, lane);
        warp_rows<R, false>(Wl + o.w_res, nullptr, R, vh, vh, warp, lane,
                            [&](int row, float acc) { x[row] = x[row] + (acc + Wl[o.b_res + row]); });
        warp_rows<R, false>(Wl + o.w_skip, nullptr, S, vh, vh, warp, lane,
                            [&](int row, float acc) { q[row] += acc; });
      }
      __syncthreads();
    }

    // head (a8)
    for (int i = tid; i < S; i += kThreads) q[i] = fmaxf(q[i], 0.0f);
    __syncthreads();
    {
      Vec<S> vz;
      vz.load_smem(q, lane);
      warp_rows<S, false>(W + o.w_relu, nullptr, kLevels, vz, vz, warp, lane,
                          [&](int row, float acc) { za[row] = fmaxf(acc + W[o.b_relu + row], 0.0f); });
    }
    __syncthreads();
    {
      Vec<kLevels> va;
      va.load_smem(za, lane);
      warp_rows<kLevels, false>(W + o.w_out, nullptr, kLevels, va, va, warp, lane,
                                [&](int row, float acc) { lg[row] = acc + W[o.b_out + row]; });
    }
    __syncthreads();

    // sampler / feedback (a9, a10)
    int y;
    const float l = lg[tid];
    if (forced) {
      A.out_logits[((int64_t)st * A.N + n) * kLevels + tid] = l;
      y = forced[n];
    } else {
      if (A.samp_kind == 0 && A.approx != 2) {
        y = sample_256(l, uni[n], dscr, fscr, iscr, tid, 1);
      } else {  // App. A.4 strategies (row f3) and App. C.2's exp (row f4): one warp
        if (tid < 32) {
          float lv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) lv[i] = lg[8 * tid + i];
          const int yy = warp_sample_policy(lv, uni[n], A.samp_kind, A.samp_inv_t, A.samp_topk, tid, A.approx == 2);
          if (tid == 0) iscr[0] = yy;
        }
        __syncthreads();
        y = iscr[0];
      }
      if (tid == 0) A.out_codes[(int64_t)st * A.N + n] = (uint8_t)y;
    }
    y2 = y1;
    y1 = y;
    __syncthreads();
  }
  if (A.ystate && !forced && tid == 0) {  // the code history for the session's next call
    A.ystate[2 * st] = y1;
    A.ystate[2 * st + 1] = y2;
  }
}

template <int R, int S>
cudaError_t launch_rs(const RunArgs& a, cudaStream_t st) {
  k_stream<R, S><<<a.n_streams, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_stream_kernel(const RunArgs& a, cudaStream_t st, LaunchInfo* info) {
  cudaError_t e;
  if (a.r == 32 && a.s == 128) e = launch_rs<32, 128>(a, st);
  else if (a.r == 32 && a.s == 256) e = launch_rs<32, 256>(a, st);
  else if (a.r == 64 && a.s == 128) e = launch_rs<64, 128>(a, st);
  else if (a.r == 64 && a.s == 256) e = launch_rs<64, 256>(a, st);
  else if (a.r == 128 && a.s == 128) e = launch_rs<128, 128>(a, st);
  else if (a.r == 128 && a.s == 256) e = launch_rs<128, 256>(a, st);
  else return cudaErrorInvalidValue;
  info->grid = a.n_streams;
  info->cluster = 1;
  info->threads = kThreads;
  info->launches = 1;
  return e;
}

}  // namespace dvw
