// kernel_parallel.cu -- teacher-forced logits in parallel over time (dvw_logits).
//
// With the codes given (logits[n] depends on codes[0..n-1]), nothing in the
// network is recurrent any more: layer j's input at every timestep is known once layer
// j-1 is done for all timesteps.  So instead of running the autoregressive kernels sample
// by sample, each layer is one pass over the whole utterance (the same arithmetic as
// PAPER.md:340-375, with dilated inputs read at t - d_j):
//   k_embed : x_0[t] = W_emb_prev[:, y_{t-2}] + W_emb_cur[:, y_{t-1}] + B_emb (y_{<0} = 128, R4);
//             q[t] = B_skip
//   k_layer : per 64-timestep tile, a = [W_prev | W_cur] [x_j(t-d) ; x_j(t)] + B + L(t/hop)
//             -> h = tanh(a_0:r) sigma(a_r:2r) -> x_{j+1} = x_j + W_res h + B_res,
//             q += W_skip h   (three block GEMMs sharing the h tile in shared memory)
//   k_head  : z_s = relu(q), z_a = relu(W_relu z_s + B_relu), logits = W_out z_a + B_out
// Block GEMMs: 256 threads, 64 timesteps; activations staged k-major [K][64] in shared
// memory, weights staged in 32-wide K chunks [32][N]; each thread owns a TPT x NPT
// register tile.  fp32 FMA in a fixed order (bitwise deterministic), accurate tanhf/expf.
// One launch per layer plus two: ~l + 2 short launches per call.
#include "dvw_internal.cuh"

namespace dvw {
namespace {

constexpr int kTile = 64;  // timesteps per block
constexpr int kPT = 256;   // threads per block
constexpr int kKC = 32;    // K chunk of the staged weights

// One 32-wide K chunk of weights in registers (same thread -> element map as stage_w), so
// the next chunk's global loads are in flight while the current chunk is multiplied.
template <int N>
struct WChunk {
  static constexpr int kPer = N * (kKC / 4) / kPT;
  static_assert(kPer >= 1 && N * (kKC / 4) % kPT == 0, "chunk does not tile the block");
  float4 v[kPer];
  __device__ __forceinline__ void load(const float* W, int ld, int k0, int kmax) {
#pragma unroll
    for (int p = 0; p < kPer; ++p) {
      const int i = threadIdx.x + p * kPT, n = i % N, k = k0 + 4 * (i / N);
      v[p] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k + 3 < kmax) {
        v[p] = __ldg(reinterpret_cast<const float4*>(W + (int64_t)n * ld + k));
      } else {
        if (k < kmax) v[p].x = __ldg(W + (int64_t)n * ld + k);
        if (k + 1 < kmax) v[p].y = __ldg(W + (int64_t)n * ld + k + 1);
        if (k + 2 < kmax) v[p].z = __ldg(W + (int64_t)n * ld + k + 2);
      }
    }
  }
  __device__ __forceinline__ void store(float* Bs) const {
#pragma unroll
    for (int p = 0; p < kPer; ++p) {
      const int i = threadIdx.x + p * kPT, n = i % N, kq = i / N;
      Bs[(4 * kq) * N + n] = v[p].x;
      Bs[(4 * kq + 1) * N + n] = v[p].y;
      Bs[(4 * kq + 2) * N + n] = v[p].z;
      Bs[(4 * kq + 3) * N + n] = v[p].w;
    }
  }
};

// acc[i][j] += sum_k At[k][t_i] * Bs[k][c_j] over the staged chunk (t_i = t0 + i, c_j = col[j]).
template <int TPT, int NPT, int N>
__device__ __forceinline__ void fma_chunk(const float* At, int kbase, const float* Bs, int t0, const int (&col)[NPT],
                                          float (&acc)[TPT][NPT]) {
#pragma unroll 4
  for (int kk = 0; kk < kKC; ++kk) {
    float a[TPT], b[NPT];
#pragma unroll
    for (int i = 0; i < TPT; ++i) a[i] = At[(kbase + kk) * kTile + t0 + i];
#pragma unroll
    for (int j = 0; j < NPT; ++j) b[j] = Bs[kk * N + col[j]];
#pragma unroll
    for (int i = 0; i < TPT; ++i)
#pragma unroll
      for (int j = 0; j < NPT; j += 2) {  // packed FFMA2: the same two fmaf, ~1.4x the issue rate
        const float2 r = __ffma2_rn(make_float2(a[i], a[i]), make_float2(b[j], b[j + 1]),
                                    make_float2(acc[i][j], acc[i][j + 1]));
        acc[i][j] = r.x;
        acc[i][j + 1] = r.y;
      }
  }
}

// acc += sum over K of At[kbase + k][t] * W[col][k]: the weights come through Bs chunk by chunk,
// chunk k0 + 32 loading into registers while chunk k0 is multiplied.  `src(k0, wc)` loads
// chunk k0 into wc; `pf` holds chunk 0 on entry (issued early by the caller).
template <int TPT, int NPT, int N, typename Src>
__device__ __forceinline__ void gemm_pipelined(const float* At, int kbase, int K, Src src, WChunk<N>& pf, float* Bs,
                                               int t0, const int (&col)[NPT], float (&acc)[TPT][NPT]) {
  for (int k0 = 0; k0 < K; k0 += kKC) {
    __syncthreads();  // the previous chunk's readers are done with Bs
    pf.store(Bs);
    __syncthreads();
    if (k0 + kKC < K) src(k0 + kKC, pf);
    fma_chunk<TPT, NPT, N>(At, kbase + k0, Bs, t0, col, acc);
  }
}

// Load rows [t0 - shift, t0 - shift + 64) (zero outside [0, T)) of X [T][C] into At[koff + c][t].
// Thread -> (timestep t, 4 consecutive channels): a 16-byte read, and writes in which
// consecutive threads hit consecutive t (conflict-free).  C is a multiple of 4.
__device__ __forceinline__ void load_act(float* At, int koff, const float* X, int C, int T, int t0, int shift) {
  for (int i = threadIdx.x; i < kTile * (C / 4); i += kPT) {
    const int t = i % kTile, c = 4 * (i / kTile), tg = t0 - shift + t;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tg >= 0 && tg < T) v = *reinterpret_cast<const float4*>(X + (int64_t)tg * C + c);
    At[(koff + c) * kTile + t] = v.x;
    At[(koff + c + 1) * kTile + t] = v.y;
    At[(koff + c + 2) * kTile + t] = v.z;
    At[(koff + c + 3) * kTile + t] = v.w;
  }
}

template <int R, int S>
__global__ void __launch_bounds__(kPT) k_embed(RunArgs A, float* X0, float* Q) {
  const int st = blockIdx.y;
  const int64_t T = A.N;
  const uint8_t* codes = A.forced + (int64_t)st * T;
  const float* ep = A.w + A.off.emb_prev;
  const float* ec = A.w + A.off.emb_cur;
  for (int64_t i = (int64_t)blockIdx.x * kPT + threadIdx.x; i < T * R; i += (int64_t)gridDim.x * kPT) {
    const int64_t t = i / R;
    const int c = (int)(i % R);
    const int y1 = t >= 1 ? codes[t - 1] : kLevels / 2, y2 = t >= 2 ? codes[t - 2] : kLevels / 2;
    X0[(int64_t)st * T * R + i] =
        (__ldg(ep + (int64_t)c * kLevels + y2) + __ldg(ec + (int64_t)c * kLevels + y1)) + __ldg(A.w + A.off.b_emb + c);
  }
  for (int64_t i = (int64_t)blockIdx.x * kPT + threadIdx.x; i < T * S; i += (int64_t)gridDim.x * kPT)
    Q[(int64_t)st * T * S + i] = __ldg(A.w + A.off.b_skip + (int)(i % S));
}

// One layer over a 64-timestep tile.  Xin/Xout [streams][T][R], Q [streams][T][S].
template <int R, int S>
__global__ void __launch_bounds__(kPT, 2) k_layer(RunArgs A, int j, const float* Xin, float* Xout, float* Q) {
  extern __shared__ float sm[];
  float* Xt = sm;                    // [2R][64]: rows 0..R-1 x(t - d), R..2R-1 x(t)
  float* Ht = Xt + 2 * R * kTile;    // [R][64]
  float* Bs = Ht + R * kTile;        // [kKC][max(2R, S)]
  const int st = blockIdx.y, t0 = blockIdx.x * kTile;
  const int T = (int)A.N;
  const int64_t lo = (int64_t)j * A.off.layer_stride;
  const float* xin = Xin + (int64_t)st * T * R;
  const int d = A.dil[j];
  const float* wprev = A.w + lo + A.off.w_prev;
  const float* wcur = A.w + lo + A.off.w_cur;
  // [W_prev | W_cur] as one 2R x 2R matrix: column k < R from W_prev, else W_cur
  auto src1 = [&](int k0, WChunk<2 * R>& wc) {
    if (k0 < R) wc.load(wprev, R, k0, R);
    else wc.load(wcur, R, k0 - R, R);
  };
  WChunk<2 * R> pf1;
  src1(0, pf1);  // in flight while the activations load
  load_act(Xt, 0, xin, R, T, t0, d);
  load_act(Xt, R, xin, R, T, t0, 0);
  // ---- a = W_prev x(t-d) + W_cur x(t): thread (tg, og): timesteps [tg TPT, +TPT), channels
  //      og*4..og*4+3 of the tanh half and the same of the sigmoid half
  constexpr int OG = R / 4, TPT = kTile * OG / kPT;  // R=64: 16 groups x 4 timesteps
  const int og = threadIdx.x % OG, tg = threadIdx.x / OG, tb = tg * TPT;
  int col1[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    col1[q] = 4 * og + q;
    col1[4 + q] = R + 4 * og + q;
  }
  float acc[TPT][8];
#pragma unroll
  for (int i = 0; i < TPT; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[i][q] = 0.0f;
  gemm_pipelined<TPT, 8, 2 * R>(Xt, 0, 2 * R, src1, pf1, Bs, tb, col1, acc);
  const float* wres = A.w + lo + A.off.w_res;
  auto src2 = [&](int k0, WChunk<R>& wc) { wc.load(wres, R, k0, R); };
  WChunk<R> pf2;
  src2(0, pf2);  // in flight during the gate
  // ---- gate: + B + L(t / hop)
  const float* bj = A.w + lo + A.off.b;
#pragma unroll
  for (int i = 0; i < TPT; ++i) {
    const int t = t0 + tb + i;
    const float* L = A.cond + (((int64_t)st * A.n_frames + (t < T ? t : 0) / A.hop) * A.L + j) * 2 * R;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = 4 * og + q;
      const float ah = acc[i][q] + __ldg(bj + c) + (t < T ? __ldg(L + c) : 0.0f);
      const float ag = acc[i][4 + q] + __ldg(bj + R + c) + (t < T ? __ldg(L + R + c) : 0.0f);
      Ht[c * kTile + tb + i] = A.approx == 0 ? gate(ah, ag) : A.approx == 1 ? gate_approx(ah, ag) : gate_appc(ah, ag);
    }
  }
  // ---- x_{j+1} = x_j + W_res h + B_res: same (tg, og) map, 4 channels
  float acc2[TPT][4];
#pragma unroll
  for (int i = 0; i < TPT; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc2[i][q] = 0.0f;
  int col2[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) col2[q] = 4 * og + q;
  gemm_pipelined<TPT, 4, R>(Ht, 0, R, src2, pf2, Bs, tb, col2, acc2);
  const float* wskip = A.w + lo + A.off.w_skip;
  auto src3 = [&](int k0, WChunk<S>& wc) { wc.load(wskip, R, k0, R); };
  WChunk<S> pf3;
  src3(0, pf3);  // in flight during the residual epilogue
  float* xout = Xout + (int64_t)st * T * R;
#pragma unroll
  for (int i = 0; i < TPT; ++i) {
    const int t = t0 + tb + i;
    if (t >= T) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = 4 * og + q;
      xout[(int64_t)t * R + c] = Xt[(R + c) * kTile + tb + i] + (acc2[i][q] + __ldg(A.w + lo + A.off.b_res + c));
    }
  }
  // ---- q += W_skip h: thread (tg2, cg): timesteps [4 tg2, +4), channels [cg S/16, +S/16)
  constexpr int NS = S / 16;
  const int cg = threadIdx.x % 16, tg2 = threadIdx.x / 16;
  int col3[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) col3[q] = cg * NS + q;
  float acc3[4][NS];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < NS; ++q) acc3[i][q] = 0.0f;
  gemm_pipelined<4, NS, S>(Ht, 0, R, src3, pf3, Bs, 4 * tg2, col3, acc3);
  float* q = Q + (int64_t)st * T * S;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + 4 * tg2 + i;
    if (t >= T) continue;
#pragma unroll
    for (int c = 0; c < NS; ++c) q[(int64_t)t * S + col3[c]] += acc3[i][c];
  }
}

// z_s = relu(q); z_a = relu(W_relu z_s + B_relu); logits = W_out z_a + B_out.
template <int S>
__global__ void __launch_bounds__(kPT, 2) k_head(RunArgs A, const float* Q) {
  extern __shared__ float sm[];
  float* Zs = sm;                   // [S][64]
  float* Za = Zs + S * kTile;       // [256][64]
  float* Bs = Za + kLevels * kTile; // [kKC][256]
  const int st = blockIdx.y, t0 = blockIdx.x * kTile;
  const int T = (int)A.N;
  const float* q = Q + (int64_t)st * T * S;
  for (int i = threadIdx.x; i < kTile * S; i += kPT) {
    const int t = i % kTile, c = i / kTile;  // consecutive threads: consecutive t (conflict-free)
    Zs[c * kTile + t] = (t0 + t < T) ? fmaxf(q[(int64_t)(t0 + t) * S + c], 0.0f) : 0.0f;
  }
  const int cg = threadIdx.x % 16, tg = threadIdx.x / 16;
  int col[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) col[c] = cg * 16 + c;
  float acc[4][16];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[i][c] = 0.0f;
  const float* wrelu = A.w + A.off.w_relu;
  const float* wout = A.w + A.off.w_out;
  auto srcr = [&](int k0, WChunk<kLevels>& wc) { wc.load(wrelu, S, k0, S); };
  auto srco = [&](int k0, WChunk<kLevels>& wc) { wc.load(wout, kLevels, k0, kLevels); };
  WChunk<kLevels> pf;
  srcr(0, pf);
  gemm_pipelined<4, 16, kLevels>(Zs, 0, S, srcr, pf, Bs, 4 * tg, col, acc);
  srco(0, pf);  // in flight during the relu epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      Za[col[c] * kTile + 4 * tg + i] = fmaxf(acc[i][c] + __ldg(A.w + A.off.b_relu + col[c]), 0.0f);
      acc[i][c] = 0.0f;
    }
  gemm_pipelined<4, 16, kLevels>(Za, 0, kLevels, srco, pf, Bs, 4 * tg, col, acc);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + 4 * tg + i;
    if (t >= T) continue;
    float* o = A.out_logits + ((int64_t)st * T + t) * kLevels;
#pragma unroll
    for (int c = 0; c < 16; c += 4)
      *reinterpret_cast<float4*>(o + col[c]) =
          make_float4(acc[i][c] + __ldg(A.w + A.off.b_out + col[c]), acc[i][c + 1] + __ldg(A.w + A.off.b_out + col[c + 1]),
                      acc[i][c + 2] + __ldg(A.w + A.off.b_out + col[c + 2]),
                      acc[i][c + 3] + __ldg(A.w + A.off.b_out + col[c + 3]));
  }
}

template <int R, int S>
cudaError_t run_rs(const RunArgs& a, float* ws, cudaStream_t st, LaunchInfo* info, const float* pk_tc) {
  const int64_t T = a.N, nS = a.n_streams;
  float* X[2] = {ws, ws + nS * T * R};
  float* Q = ws + 2 * nS * T * R;
  const dim3 eg((unsigned)std::min<int64_t>((T * R + kPT - 1) / kPT, 4096), (unsigned)nS);
  k_embed<R, S><<<eg, kPT, 0, st>>>(a, X[0], Q);
  const dim3 grid((unsigned)((T + kTile - 1) / kTile), (unsigned)nS);
  const int lsm = (int)sizeof(float) * (3 * R * kTile + kKC * std::max(2 * R, S));
  cudaError_t e = cudaFuncSetAttribute(k_layer<R, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, lsm);
  for (int j = 0; e == cudaSuccess && j < a.L; ++j) {
    if ((R == 64 || R == 128) && pk_tc) e = launch_parallel_layer_tc(a, j, X[j & 1], X[(j + 1) & 1], Q, pk_tc, st);
    else k_layer<R, S><<<grid, kPT, lsm, st>>>(a, j, X[j & 1], X[(j + 1) & 1], Q);
  }
  const int hsm = (int)sizeof(float) * ((S + kLevels) * kTile + kKC * kLevels);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_head<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm);
  if (e == cudaSuccess) {
    if ((R == 64 || R == 128) && pk_tc) e = launch_parallel_head_tc(a, Q, pk_tc, st);
    else k_head<S><<<grid, kPT, hsm, st>>>(a, Q);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  info->grid = (int)(grid.x * grid.y);
  info->cluster = 1;
  info->threads = kPT;
  info->launches = a.L + 2;
  return e;
}

}  // namespace

size_t parallel_workspace_bytes(int r, int s, int64_t n_samples, int n_streams) {
  return sizeof(float) * (size_t)n_streams * (size_t)n_samples * (size_t)(2 * r + s);
}

cudaError_t launch_parallel_logits(const RunArgs& a, void* ws, cudaStream_t st, LaunchInfo* info,
                                   const float* pk_tc) {
  float* w = static_cast<float*>(ws);
  if (a.r == 32 && a.s == 128) return run_rs<32, 128>(a, w, st, info, nullptr);
  if (a.r == 32 && a.s == 256) return run_rs<32, 256>(a, w, st, info, nullptr);
  if (a.r == 64 && a.s == 128) return run_rs<64, 128>(a, w, st, info, pk_tc);
  if (a.r == 64 && a.s == 256) return run_rs<64, 256>(a, w, st, info, pk_tc);
  if (a.r == 128 && a.s == 128) return run_rs<128, 128>(a, w, st, info, pk_tc);
  if (a.r == 128 && a.s == 256) return run_rs<128, 256>(a, w, st, info, pk_tc);
  return cudaErrorNotSupported;
}

}  // namespace dvw
