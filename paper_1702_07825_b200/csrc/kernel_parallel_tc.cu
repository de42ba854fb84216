// kernel_parallel_tc.cu -- the teacher-forced layer pass of dvw_logits on the tensor cores
// (r = 64; the SIMT k_layer in kernel_parallel.cu serves the other widths).
//
// Same arithmetic as k_layer (SURVEY.md §8(a) a3-a7 for all timesteps
// of a layer at once, codes given), per 128-timestep tile (M = 128, TMEM lane = timestep):
//   GEMM 1  a[t][0:2r] = [W_prev | W_cur] [x_j(t-d); x_j(t)]       K = 2r = 128 in two 64-chunks
//   gate    h = tanh(a_0:r + B + L) sigma(a_r:2r + B + L)            (epilogue, thread = timestep)
//   GEMM 2  [x_{j+1} - x_j - B_res ; dq] = [W_res ; W_skip] h        K = r = 64, N = r + s rows in
//                                                                      chunks of <= 128 rows
// fp32-faithful on the tf32 pipe (reading R23): each operand x is split into x (the MMA reads
// its tf32 head) and lo = x - tf32(x); per K-step of 8: D[:, 0:2N) += A_hi [W_hi; W_lo]^T and
// D[:, 0:N) += A_lo W_hi^T, the epilogue adds column c and c + N (the dropped lo lo term is
// <= 2^-22 relative).  Operands in shared memory in the K-major core-matrix order (umma.cuh):
// activations written by the threads (with their lo halves), weight chunks pre-packed at load
// time and fetched with one bulk copy each.  One elected thread issues the MMAs.
#include <algorithm>
#include <cstring>
#include <vector>

#include "dvw_internal.cuh"
#include "ptx.cuh"
#include "umma.cuh"

namespace dvw {
namespace {

constexpr int R = 64;            // residual channels this kernel is built for
constexpr int kTM = 128;         // timesteps per tile (= MMA M = TMEM lanes)
constexpr int kLThr = 256;       // two threads per timestep (warps w and w + 4 share TMEM lanes)
constexpr int kActF = 16 * kTM * 4;  // one 64-channel activation operand [16][128][4] (floats)
constexpr int kW1F = 16 * 256 * 4;   // one GEMM-1 weight chunk: 64 K x (128 hi + 128 lo rows)
constexpr int kLBP = 2 * R + 1;      // padded row of the per-timestep (L + B) table
constexpr int kSmemF = 2 * kActF + kW1F + kTM * kLBP;

// floats of one layer's packed weights: two GEMM-1 chunks, then GEMM-2 chunks of [16][2n][4]
__host__ __device__ constexpr int64_t tc_layer_floats(int s) { return 2 * kW1F + 128 * (R + s); }

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// mbarrier wait with a 2 s watchdog: a lost completion traps (the launch fails with an error
// the host reports) instead of hanging the device.
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t parity) {
  if (ptx::mbar_try_wait_cta(bar, parity)) return;
  const uint64_t t0 = ptx::globaltimer();
  while (!ptx::mbar_try_wait_cta(bar, parity))
    if (ptx::globaltimer() - t0 > 2000000000ull) asm volatile("trap;");
}

// Rows t0 - shift + i (zero outside [0, T)) of X [T][64] into the operand pair (hi, lo).
// Thread (row i, half hf) loads 8 of the row's 16 channel groups (all in flight at once:
// load_row), then writes them into the operand pair (store_row).
__device__ __forceinline__ void load_row(float4 (&v)[8], const float* X, int T, int t0, int shift, int i, int hf) {
  const int tg = t0 - shift + i;
  const bool in = tg >= 0 && tg < T;
  const float4* src = reinterpret_cast<const float4*>(X + (int64_t)(in ? tg : 0) * R) + 8 * hf;
#pragma unroll
  for (int g = 0; g < 8; ++g) v[g] = in ? __ldg(src + g) : make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void store_row(float* hi, float* lo, const float4 (&v)[8], int i, int hf) {
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const int o = ((8 * hf + g) * kTM + i) * 4;
    *reinterpret_cast<float4*>(hi + o) = v[g];
    *reinterpret_cast<float4*>(lo + o) =
        make_float4(tf32_lo(v[g].x), tf32_lo(v[g].y), tf32_lo(v[g].z), tf32_lo(v[g].w));
  }
}

struct Sync {
  uint32_t bar_w, bar_m;
  uint32_t ph_w = 0, ph_m = 0;
};

// D[:, 0:2n) = / += A (K = 64, operand pair at a_hi/a_lo) times the staged weight chunk
// (n real rows + their n lo rows).  Thread 0 issues (mma_issue); everybody waits (mma_wait).
__device__ __forceinline__ void mma_issue(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint32_t wsm, int n, bool acc,
                                          Sync& sy) {
  if (threadIdx.x == 0) {
    wait_bar(sy.bar_w, sy.ph_w);
    ptx::tmem_fence_after();
    const uint32_t id2 = idesc_tf32(2 * n), id1 = idesc_tf32(n);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const uint32_t ao = ks * 2 * kTM * 16, bo = ks * 2 * (2 * n) * 16;
      const uint64_t dah = sdesc(a_hi + ao, kTM * 16, 128), dal = sdesc(a_lo + ao, kTM * 16, 128);
      const uint64_t db = sdesc(wsm + bo, 2 * n * 16, 128);
      mma_tf32(d, dah, db, id2, (acc || ks > 0) ? 1u : 0u);
      mma_tf32(d, dal, db, id1, 1u);
    }
    mma_commit(sy.bar_m);
  }
  sy.ph_w ^= 1;
}
__device__ __forceinline__ void mma_wait(Sync& sy) {
  wait_bar(sy.bar_m, sy.ph_m);
  sy.ph_m ^= 1;
  ptx::tmem_fence_after();
}
__device__ __forceinline__ void mma_chunk(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint32_t wsm, int n, bool acc,
                                          Sync& sy) {
  mma_issue(d, a_hi, a_lo, wsm, n, acc, sy);
  mma_wait(sy);
}

__device__ __forceinline__ void fetch_w(uint32_t wsm, const float* src, int floats, const Sync& sy) {
  if (threadIdx.x == 0) {
    ptx::mbar_arm(sy.bar_w, (uint32_t)floats * 4);
    bulk_g2s(wsm, src, (uint32_t)floats * 4, sy.bar_w);
  }
}

// TMEM reads of this thread's lane must be complete before the next MMA overwrites D.
__device__ __forceinline__ void release_tmem() {
  ptx::tmem_fence_before();
  __syncthreads();
}

template <int S>
__global__ void __launch_bounds__(kLThr, 1) k_layer_tc(RunArgs A, int j, const float* Xin, float* Xout, float* Q,
                                                       const float* pk) {
  extern __shared__ __align__(1024) float sm[];
  float* a_hi = sm;            // [16][128][4]
  float* a_lo = sm + kActF;    // [16][128][4]
  float* wsm = sm + 2 * kActF; // one weight chunk, <= [16][256][4]
  float* lb = wsm + kW1F;      // [128][2R + 1]: L^(j)(t / hop) + B for this thread's timestep
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x & (kTM - 1), hf = threadIdx.x >> 7;  // timestep row, half of the work
  const int st = blockIdx.y, t0 = blockIdx.x * kTM;
  const int T = (int)A.N;
  const int tg = t0 + t;
  const int64_t lo = (int64_t)j * A.off.layer_stride;
  const float* xin = Xin + (int64_t)st * T * R;
  const float* pl = pk + (int64_t)j * tc_layer_floats(S);
  if (threadIdx.x < 32) ptx::tmem_alloc(ptx::smem_u32(&tmem_base), 256);
  Sync sy;
  sy.bar_w = ptx::smem_u32(&bars[0]);
  sy.bar_m = ptx::smem_u32(&bars[1]);
  if (threadIdx.x == 0) {
    ptx::mbar_init(sy.bar_w, 1);
    ptx::mbar_init(sy.bar_m, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  ptx::tmem_fence_before();
  __syncthreads();
  ptx::tmem_fence_after();
  const uint32_t d = tmem_base;
  const uint32_t s_hi = ptx::smem_u32(a_hi), s_lo = ptx::smem_u32(a_lo), s_w = ptx::smem_u32(wsm);
  const uint32_t lane_addr = d + ((uint32_t)(32 * (t >> 5)) << 16);  // warp w: lanes 32 (w % 4) ..
  const float* bj = A.w + lo + A.off.b;
  // ---- GEMM 1: chunk 0 = W_prev with x_j(t - d), chunk 1 = W_cur with x_j(t).  While chunk 0's
  //      MMAs run: the x_j(t) rows load into registers and the gate's (L + B) table fills.
  const float* w2 = pl + 2 * kW1F;
  {
    float4 v[8];
    fetch_w(s_w, pl, kW1F, sy);
    load_row(v, xin, T, t0, A.dil[j], t, hf);
    store_row(a_hi, a_lo, v, t, hf);
    fence_proxy_async_smem();
    __syncthreads();
    mma_issue(d, s_hi, s_lo, s_w, 128, false, sy);
    load_row(v, xin, T, t0, 0, t, hf);
    const float* Lr = A.cond + (((int64_t)st * A.n_frames + (tg < T ? tg : 0) / A.hop) * A.L + j) * 2 * R;
#pragma unroll 8
    for (int c = R * hf; c < R * hf + R; c += 4) {  // the row's half hf; read back after the barriers
      const float4 lv = tg < T ? __ldg(reinterpret_cast<const float4*>(Lr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 bv = __ldg(reinterpret_cast<const float4*>(bj + c));
      float* o = lb + t * kLBP + c;
      o[0] = bv.x + lv.x;
      o[1] = bv.y + lv.y;
      o[2] = bv.z + lv.z;
      o[3] = bv.w + lv.w;
    }
    mma_wait(sy);
    fetch_w(s_w, pl + kW1F, kW1F, sy);
    store_row(a_hi, a_lo, v, t, hf);
    fence_proxy_async_smem();
    __syncthreads();
    mma_chunk(d, s_hi, s_lo, s_w, 128, true, sy);
  }
  fetch_w(s_w, w2, 16 * 2 * 128 * 4, sy);  // GEMM 2's first chunk, during the gate
  // ---- gate: + B + L(t / hop); h -> operand pair for GEMM 2
#pragma unroll 1
  for (int cc = 2 * hf; cc < 2 * hf + 2; ++cc) {  // channels 16 cc .. 16 cc + 15 (this thread's half)
    float ah[16], ah2[16], ag[16], ag2[16];
    ptx::tmem_ld16(lane_addr + 16 * cc, ah);
    ptx::tmem_ld16(lane_addr + 128 + 16 * cc, ah2);
    ptx::tmem_ld16(lane_addr + 64 + 16 * cc, ag);
    ptx::tmem_ld16(lane_addr + 192 + 16 * cc, ag2);
    ptx::tmem_wait_ld<16>(ah);
    ptx::tmem_wait_ld<16>(ah2);
    ptx::tmem_wait_ld<16>(ag);
    ptx::tmem_wait_ld<16>(ag2);
    float h[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int c = 16 * cc + e;
      const float xh = (ah[e] + ah2[e]) + lb[t * kLBP + c];
      const float xg = (ag[e] + ag2[e]) + lb[t * kLBP + R + c];
      // exact tier: the branch-free MUFU form of tanh / sigma (reading R13, abs. error ~1e-7, as
      // the cluster kernel); libdevice tanhf/expf cost ~200 cycles per channel here
      h[e] = A.approx == 0 ? gate_fast(xh, xg) : A.approx == 1 ? gate_approx(xh, xg) : gate_appc(xh, xg);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int o = ((4 * cc + q) * kTM + t) * 4;
      const float4 v = make_float4(h[4 * q], h[4 * q + 1], h[4 * q + 2], h[4 * q + 3]);
      *reinterpret_cast<float4*>(a_hi + o) = v;
      *reinterpret_cast<float4*>(a_lo + o) = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
    }
  }
  ptx::tmem_fence_before();  // GEMM 2 overwrites D after every lane has read it
  fence_proxy_async_smem();
  __syncthreads();
  // ---- GEMM 2: rows [W_res (64); W_skip (S)] in chunks of <= 128 rows; the next chunk's
  //      bulk copy overlaps this chunk's epilogue
  const float* bres = A.w + lo + A.off.b_res;
  float* xout = Xout + (int64_t)st * T * R;
  float* q = Q + (int64_t)st * T * S;
  int r0 = 0;
#pragma unroll 1
  for (int ci = 0; r0 < R + S; ++ci) {
    const int n = std::min(128, R + S - r0);
    const bool live = tg < T;
    const int tr = live ? tg : 0;
    // the addends of this chunk's rows (x_j for rows < R, the running q above), in flight
    // while the MMAs run
    float4 base[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int g = hf + 2 * k;  // this thread's 16-row groups
      if (16 * g < n) {
        const int row = r0 + 16 * g;  // 16 rows, all on one side of R
        const float4* src = row < R ? reinterpret_cast<const float4*>(xin + (int64_t)tr * R + row)
                                    : reinterpret_cast<const float4*>(q + (int64_t)tr * S + (row - R));
#pragma unroll
        for (int e = 0; e < 4; ++e) base[k][e] = row < R ? __ldg(src + e) : src[e];
      }
    }
    mma_chunk(d, s_hi, s_lo, s_w, n, false, sy);
    if (r0 + n < R + S) fetch_w(s_w, w2 + 16 * 2 * n * 4, 16 * 2 * std::min(128, R + S - r0 - n) * 4, sy);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int g = hf + 2 * k;
      if (16 * g < n) {
        const int row = r0 + 16 * g;
        float v[16], v2[16];
        ptx::tmem_ld16(lane_addr + 16 * g, v);
        ptx::tmem_ld16(lane_addr + n + 16 * g, v2);
        ptx::tmem_wait_ld<16>(v);
        ptx::tmem_wait_ld<16>(v2);
        if (live) {
          float4* dst = row < R ? reinterpret_cast<float4*>(xout + (int64_t)tg * R + row)
                                : reinterpret_cast<float4*>(q + (int64_t)tg * S + (row - R));
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float4 o = base[k][e];
            if (row < R) {  // x_{j+1} = x_j + W_res h + B_res
              const float4 br = __ldg(reinterpret_cast<const float4*>(bres + row) + e);
              o.x += (v[4 * e] + v2[4 * e]) + br.x;
              o.y += (v[4 * e + 1] + v2[4 * e + 1]) + br.y;
              o.z += (v[4 * e + 2] + v2[4 * e + 2]) + br.z;
              o.w += (v[4 * e + 3] + v2[4 * e + 3]) + br.w;
            } else {  // q += W_skip h
              o.x += v[4 * e] + v2[4 * e];
              o.y += v[4 * e + 1] + v2[4 * e + 1];
              o.z += v[4 * e + 2] + v2[4 * e + 2];
              o.w += v[4 * e + 3] + v2[4 * e + 3];
            }
            dst[e] = o;
          }
        }
      }
    }
    release_tmem();
    w2 += 16 * 2 * n * 4;
    r0 += n;
  }
  if (threadIdx.x < 32) ptx::tmem_dealloc(d, 256);
}

// ---------------------------------------------------------------------------- the head
// z_s = relu(q); z_a = relu(W_relu z_s + B_relu); logits = W_out z_a + B_out
// per 128-timestep tile: two K = s and K = 256 GEMMs with N = 256.  Here the three tf32 passes
// are three MMAs into the same columns (A_hi W_hi, A_hi W_lo, A_lo W_hi), so z_a and the
// logits each take 256 TMEM columns and both fit; weight chunks are [16][256][4] hi images
// followed by their lo images, 128 KB, one bulk copy each.
constexpr int kHW = 16 * 256 * 4;  // floats of one 64-K x 256-row image

__device__ __forceinline__ void mma3(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint32_t w_hi, uint32_t w_lo,
                                     bool acc, Sync& sy, int n = 256) {
  if (threadIdx.x == 0) {
    wait_bar(sy.bar_w, sy.ph_w);
    ptx::tmem_fence_after();
    const uint32_t id = idesc_tf32(n);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const uint32_t ao = ks * 2 * kTM * 16, bo = ks * 2 * n * 16;
      const uint64_t dah = sdesc(a_hi + ao, kTM * 16, 128), dal = sdesc(a_lo + ao, kTM * 16, 128);
      const uint64_t dbh = sdesc(w_hi + bo, n * 16, 128), dbl = sdesc(w_lo + bo, n * 16, 128);
      mma_tf32(d, dah, dbh, id, (acc || ks > 0) ? 1u : 0u);
      mma_tf32(d, dah, dbl, id, 1u);
      mma_tf32(d, dal, dbh, id, 1u);
    }
    mma_commit(sy.bar_m);
  }
  sy.ph_w ^= 1;
  wait_bar(sy.bar_m, sy.ph_m);
  sy.ph_m ^= 1;
  ptx::tmem_fence_after();
}

// 32 values (channel groups 8 hf .. 8 hf + 7) of row i into the operand pair (hi, lo).
__device__ __forceinline__ void put_row32(float* hi, float* lo, const float (&v)[32], int i, int hf) {
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const int o = ((8 * hf + g) * kTM + i) * 4;
    *reinterpret_cast<float4*>(hi + o) = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
    *reinterpret_cast<float4*>(lo + o) = make_float4(tf32_lo(v[4 * g]), tf32_lo(v[4 * g + 1]),
                                                     tf32_lo(v[4 * g + 2]), tf32_lo(v[4 * g + 3]));
  }
}

template <int S>
__global__ void __launch_bounds__(kLThr, 1) k_head_tc(RunArgs A, const float* Q, const float* ph) {
  extern __shared__ __align__(1024) float sm[];
  float* a_hi = sm;
  float* a_lo = sm + kActF;
  float* w = sm + 2 * kActF;  // [hi image | lo image]
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x & (kTM - 1), hf = threadIdx.x >> 7;  // timestep row, half of the work
  const int st = blockIdx.y, t0 = blockIdx.x * kTM;
  const int T = (int)A.N;
  const int tg = t0 + t;
  const bool live = tg < T;
  if (threadIdx.x < 32) ptx::tmem_alloc(ptx::smem_u32(&tmem_base), 512);
  Sync sy;
  sy.bar_w = ptx::smem_u32(&bars[0]);
  sy.bar_m = ptx::smem_u32(&bars[1]);
  if (threadIdx.x == 0) {
    ptx::mbar_init(sy.bar_w, 1);
    ptx::mbar_init(sy.bar_m, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  ptx::tmem_fence_before();
  __syncthreads();
  ptx::tmem_fence_after();
  const uint32_t d_za = tmem_base, d_lg = tmem_base + 256;
  const uint32_t lane = (uint32_t)(32 * (t >> 5)) << 16;
  const uint32_t s_hi = ptx::smem_u32(a_hi), s_lo = ptx::smem_u32(a_lo), s_w = ptx::smem_u32(w);
  const float* qrow = Q + ((int64_t)st * T + (live ? tg : 0)) * S;
  // ---- z_a pre-activation = W_relu relu(q), K = s in 64-chunks
#pragma unroll 1
  for (int kc = 0; kc < S / 64; ++kc) {
    fetch_w(s_w, ph + (int64_t)kc * 2 * kHW, 2 * kHW, sy);
    float v[32];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const float4 x = live ? *reinterpret_cast<const float4*>(qrow + 64 * kc + 32 * hf + 4 * g)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      v[4 * g] = fmaxf(x.x, 0.0f);
      v[4 * g + 1] = fmaxf(x.y, 0.0f);
      v[4 * g + 2] = fmaxf(x.z, 0.0f);
      v[4 * g + 3] = fmaxf(x.w, 0.0f);
    }
    put_row32(a_hi, a_lo, v, t, hf);
    fence_proxy_async_smem();
    __syncthreads();
    mma3(d_za, s_hi, s_lo, s_w, s_w + kHW * 4, kc > 0, sy);
  }
  // ---- logits = W_out z_a, K = 256 in 64-chunks; z_a = relu(pre + B_relu) chunk by chunk
  const float* wout = ph + (int64_t)(S / 64) * 2 * kHW;
  const float* brelu = A.w + A.off.b_relu;
#pragma unroll 1
  for (int kc = 0; kc < 4; ++kc) {
    fetch_w(s_w, wout + (int64_t)kc * 2 * kHW, 2 * kHW, sy);
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; c += 16) ptx::tmem_ld16(d_za + lane + 64 * kc + 32 * hf + c, v + c);
    ptx::tmem_wait_ld<32>(v);
#pragma unroll
    for (int c = 0; c < 32; c += 4) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(brelu + 64 * kc + 32 * hf + c));
      v[c] = fmaxf(v[c] + b.x, 0.0f);
      v[c + 1] = fmaxf(v[c + 1] + b.y, 0.0f);
      v[c + 2] = fmaxf(v[c + 2] + b.z, 0.0f);
      v[c + 3] = fmaxf(v[c + 3] + b.w, 0.0f);
    }
    put_row32(a_hi, a_lo, v, t, hf);
    ptx::tmem_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    mma3(d_lg, s_hi, s_lo, s_w, s_w + kHW * 4, kc > 0, sy);
  }
  const float* bout = A.w + A.off.b_out;
  float* out = A.out_logits + ((int64_t)st * T + (live ? tg : 0)) * kLevels;
#pragma unroll 1
  for (int c = 128 * hf; c < 128 * hf + 128; c += 16) {
    float v[16];
    ptx::tmem_ld16(d_lg + lane + c, v);
    ptx::tmem_wait_ld<16>(v);
    if (live) {
#pragma unroll
      for (int e = 0; e < 16; e += 4) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(bout + c + e));
        *reinterpret_cast<float4*>(out + c + e) = make_float4(v[e] + b.x, v[e + 1] + b.y, v[e + 2] + b.z, v[e + 3] + b.w);
      }
    }
  }
  ptx::tmem_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tmem_base, 512);
}

// ------------------------------------------------------------------ r = 128 (C4) layers
// The same layer pass for r = 128, 256 threads, three tf32 passes into the same TMEM columns
// (as the head): GEMM 1 K = 256 in four 64-chunks, N = 256 (D columns [0, 256)); the gate's
// h stays in registers -- thread half hf holds channels 64 hf .. 64 hf + 63, exactly GEMM 2's
// K-chunk hf -- so GEMM 2 (K = 128, rows [W_res; W_skip] in chunks of <= 256) can reuse GEMM
// 1's columns.  Packed per layer: GEMM-1 chunks (hi | lo [16][256][4]), then for each GEMM-2
// K-chunk its row chunks (hi | lo [16][n][4]).
constexpr int R2 = 128;
__host__ __device__ constexpr int64_t tc128_layer_floats(int s) { return 8 * (int64_t)kHW + 256 * (int64_t)(R2 + s); }

template <int S>
__global__ void __launch_bounds__(kLThr, 1) k_layer_tc128(RunArgs A, int j, const float* Xin, float* Xout, float* Q,
                                                          const float* pk) {
  extern __shared__ __align__(1024) float sm[];
  float* a_hi = sm;
  float* a_lo = sm + kActF;
  float* w = sm + 2 * kActF;  // [hi image | lo image], <= 2 x [16][256][4]
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x & (kTM - 1), hf = threadIdx.x >> 7;
  const int st = blockIdx.y, t0 = blockIdx.x * kTM;
  const int T = (int)A.N;
  const int tg = t0 + t;
  const bool live = tg < T;
  const int64_t lo = (int64_t)j * A.off.layer_stride;
  const float* xin = Xin + (int64_t)st * T * R2;
  const float* pl = pk + (int64_t)j * tc128_layer_floats(S);
  if (threadIdx.x < 32) ptx::tmem_alloc(ptx::smem_u32(&tmem_base), 512);
  Sync sy;
  sy.bar_w = ptx::smem_u32(&bars[0]);
  sy.bar_m = ptx::smem_u32(&bars[1]);
  if (threadIdx.x == 0) {
    ptx::mbar_init(sy.bar_w, 1);
    ptx::mbar_init(sy.bar_m, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  ptx::tmem_fence_before();
  __syncthreads();
  ptx::tmem_fence_after();
  const uint32_t d = tmem_base, lane = (uint32_t)(32 * (t >> 5)) << 16;
  const uint32_t s_hi = ptx::smem_u32(a_hi), s_lo = ptx::smem_u32(a_lo), s_w = ptx::smem_u32(w);
  // ---- GEMM 1: K-chunks 0, 1 = W_prev with x_j(t - d); 2, 3 = W_cur with x_j(t)
#pragma unroll 1
  for (int kc = 0; kc < 4; ++kc) {
    fetch_w(s_w, pl + (int64_t)kc * 2 * kHW, 2 * kHW, sy);
    const int tr = t0 - (kc < 2 ? A.dil[j] : 0) + t;
    const bool in = tr >= 0 && tr < T;
    const float4* src = reinterpret_cast<const float4*>(xin + (int64_t)(in ? tr : 0) * R2 + 64 * (kc & 1)) + 8 * hf;
    float4 v[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) v[g] = in ? __ldg(src + g) : make_float4(0.f, 0.f, 0.f, 0.f);
    store_row(a_hi, a_lo, v, t, hf);
    fence_proxy_async_smem();
    __syncthreads();
    mma3(d, s_hi, s_lo, s_w, s_w + kHW * 4, kc > 0, sy);
  }
  // ---- gate: this thread's 64 channels, h kept in registers
  const float* bj = A.w + lo + A.off.b;
  const float* L = A.cond + (((int64_t)st * A.n_frames + (live ? tg : 0) / A.hop) * A.L + j) * 2 * R2;
  float h[64];
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    const int c0 = 64 * hf + 16 * cc;
    float ah[16], ag[16];
    ptx::tmem_ld16(d + lane + c0, ah);
    ptx::tmem_ld16(d + lane + R2 + c0, ag);
    ptx::tmem_wait_ld<16>(ah);
    ptx::tmem_wait_ld<16>(ag);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int c = c0 + e;
      const float xh = ah[e] + __ldg(bj + c) + (live ? __ldg(L + c) : 0.0f);
      const float xg = ag[e] + __ldg(bj + R2 + c) + (live ? __ldg(L + R2 + c) : 0.0f);
      h[16 * cc + e] = A.approx == 0 ? gate_fast(xh, xg) : A.approx == 1 ? gate_approx(xh, xg) : gate_appc(xh, xg);
    }
  }
  ptx::tmem_fence_before();  // every lane has read GEMM 1's columns before GEMM 2 overwrites them
  __syncthreads();
  // ---- GEMM 2: K-chunk kc2 = h channels 64 kc2 .. (held by the threads with hf = kc2)
  const float* w2 = pl + 8 * (int64_t)kHW;
#pragma unroll 1
  for (int kc2 = 0; kc2 < 2; ++kc2) {
    if (hf == kc2) {
#pragma unroll
      for (int g = 0; g < 16; ++g) {
        const int o = (g * kTM + t) * 4;
        *reinterpret_cast<float4*>(a_hi + o) = make_float4(h[4 * g], h[4 * g + 1], h[4 * g + 2], h[4 * g + 3]);
        *reinterpret_cast<float4*>(a_lo + o) =
            make_float4(tf32_lo(h[4 * g]), tf32_lo(h[4 * g + 1]), tf32_lo(h[4 * g + 2]), tf32_lo(h[4 * g + 3]));
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
#pragma unroll 1
    for (int r0 = 0; r0 < R2 + S; r0 += 256) {
      const int n = std::min(256, R2 + S - r0);
      fetch_w(s_w, w2, 2 * 16 * n * 4, sy);
      mma3(d + r0, s_hi, s_lo, s_w, s_w + 16 * n * 4 * 4, kc2 > 0, sy, n);
      w2 += 2 * 16 * n * 4;
    }
  }
  // ---- epilogue: rows r of D = [W_res; W_skip] h (column r)
  const float* bres = A.w + lo + A.off.b_res;
  float* xout = Xout + (int64_t)st * T * R2;
  float* q = Q + (int64_t)st * T * S;
#pragma unroll 1
  for (int g = hf; g < (R2 + S) / 16; g += 2) {
    const int row = 16 * g;
    float v[16];
    ptx::tmem_ld16(d + lane + row, v);
    ptx::tmem_wait_ld<16>(v);
    if (!live) continue;
    if (row < R2) {  // x_{j+1} = x_j + W_res h + B_res
      const float4* xr = reinterpret_cast<const float4*>(xin + (int64_t)tg * R2 + row);
      float4* xo = reinterpret_cast<float4*>(xout + (int64_t)tg * R2 + row);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float4 x = __ldg(xr + e), b = __ldg(reinterpret_cast<const float4*>(bres + row) + e);
        xo[e] = make_float4(x.x + (v[4 * e] + b.x), x.y + (v[4 * e + 1] + b.y), x.z + (v[4 * e + 2] + b.z),
                            x.w + (v[4 * e + 3] + b.w));
      }
    } else {  // q += W_skip h
      float4* qq = reinterpret_cast<float4*>(q + (int64_t)tg * S + (row - R2));
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float4 a = qq[e];
        a.x += v[4 * e];
        a.y += v[4 * e + 1];
        a.z += v[4 * e + 2];
        a.w += v[4 * e + 3];
        qq[e] = a;
      }
    }
  }
  ptx::tmem_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(d, 512);
}

}  // namespace

__host__ __device__ constexpr int64_t tc_head_floats(int s) { return (int64_t)(s / 64 + 4) * 2 * kHW; }

static int64_t layer_floats(int r, int s) { return r == R2 ? tc128_layer_floats(s) : tc_layer_floats(s); }

int64_t parallel_tc_packed_floats(int L, int r, int s) { return (int64_t)L * layer_floats(r, s) + tc_head_floats(s); }

// [K/4][rows][4] operand images of every layer (host, once per dvw_load_weights): GEMM-1
// chunks kc = 0 (W_prev) and 1 (W_cur), each 128 rows of the weight and 128 rows of its
// tf32 residual; then GEMM-2 chunks of <= 128 rows of [W_res; W_skip] and their residuals.
cudaError_t pack_parallel_tc(const float* w, const Offsets& o, int L, int r, int s, void* dst) {
  if (r != R && r != R2) return cudaErrorInvalidValue;
  auto lo_of = [](float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    float h;
    std::memcpy(&h, &u, 4);
    return x - h;
  };
  const int64_t per = layer_floats(r, s);
  std::vector<float> h((size_t)(L * per + tc_head_floats(s)), 0.0f);
  if (r == R2) {  // r = 128: GEMM-1 64-K chunks (hi | lo [16][256][4]), GEMM-2 (K-chunk, row chunk)
    for (int j = 0; j < L; ++j) {
      const float* lw = w + (int64_t)j * o.layer_stride;
      float* c = h.data() + (int64_t)j * per;
      for (int kc = 0; kc < 4; ++kc, c += 2 * kHW) {
        const float* W = lw + (kc < 2 ? o.w_prev : o.w_cur);  // [2r][r]
        for (int k = 0; k < 64; ++k)
          for (int n = 0; n < 2 * R2; ++n) {
            const float v = W[(int64_t)n * R2 + 64 * (kc & 1) + k];
            c[((k / 4) * 256 + n) * 4 + k % 4] = v;
            c[kHW + ((k / 4) * 256 + n) * 4 + k % 4] = lo_of(v);
          }
      }
      for (int kc2 = 0; kc2 < 2; ++kc2)
        for (int r0 = 0; r0 < R2 + s; r0 += 256) {
          const int n = std::min(256, R2 + s - r0);
          for (int k = 0; k < 64; ++k)
            for (int i = 0; i < n; ++i) {
              const int row = r0 + i, kk = 64 * kc2 + k;
              const float v = row < R2 ? lw[o.w_res + (int64_t)row * R2 + kk] : lw[o.w_skip + (int64_t)(row - R2) * R2 + kk];
              c[((k / 4) * n + i) * 4 + k % 4] = v;
              c[16 * n * 4 + ((k / 4) * n + i) * 4 + k % 4] = lo_of(v);
            }
          c += 2 * 16 * n * 4;
        }
    }
  }
  for (int j = 0; r == R && j < L; ++j) {
    const float* lw = w + (int64_t)j * o.layer_stride;
    float* out = h.data() + (int64_t)j * per;
    for (int kc = 0; kc < 2; ++kc) {
      const float* W = lw + (kc == 0 ? o.w_prev : o.w_cur);  // [2R][R]
      float* c = out + kc * kW1F;
      for (int k = 0; k < R; ++k)
        for (int n = 0; n < 2 * R; ++n) {
          const float v = W[(int64_t)n * R + k];
          c[((k / 4) * 256 + n) * 4 + k % 4] = v;
          c[((k / 4) * 256 + 128 + n) * 4 + k % 4] = lo_of(v);
        }
    }
    float* c = out + 2 * kW1F;
    for (int r0 = 0; r0 < R + s;) {
      const int n = std::min(128, R + s - r0);
      for (int k = 0; k < R; ++k)
        for (int i = 0; i < n; ++i) {
          const int row = r0 + i;
          const float v = row < R ? lw[o.w_res + (int64_t)row * R + k] : lw[o.w_skip + (int64_t)(row - R) * R + k];
          c[((k / 4) * 2 * n + i) * 4 + k % 4] = v;
          c[((k / 4) * 2 * n + n + i) * 4 + k % 4] = lo_of(v);
        }
      c += 16 * 2 * n * 4;
      r0 += n;
    }
  }
  // the head: W_relu [256][s] (K = s) then W_out [256][256], 64-K chunks of hi | lo images
  float* hd = h.data() + (int64_t)L * per;
  auto put = [&](const float* W, int K) {
    for (int kc = 0; kc < K / 64; ++kc, hd += 2 * kHW)
      for (int k = 0; k < 64; ++k)
        for (int n = 0; n < kLevels; ++n) {
          const float v = W[(int64_t)n * K + 64 * kc + k];
          hd[((k / 4) * 256 + n) * 4 + k % 4] = v;
          hd[kHW + ((k / 4) * 256 + n) * 4 + k % 4] = lo_of(v);
        }
  };
  put(w + o.w_relu, s);
  put(w + o.w_out, kLevels);
  return cudaMemcpy(dst, h.data(), sizeof(float) * h.size(), cudaMemcpyHostToDevice);
}

cudaError_t launch_parallel_head_tc(const RunArgs& a, const float* q, const float* pk, cudaStream_t st) {
  const dim3 grid((unsigned)((a.N + kTM - 1) / kTM), (unsigned)a.n_streams);
  const int smem = (int)sizeof(float) * (2 * kActF + 2 * kHW);
  const float* ph = pk + (int64_t)a.L * layer_floats(a.r, a.s);
  cudaError_t e;
  if (a.s == 256) {
    e = cudaFuncSetAttribute(k_head_tc<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) k_head_tc<256><<<grid, kLThr, smem, st>>>(a, q, ph);
  } else if (a.s == 128) {
    e = cudaFuncSetAttribute(k_head_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) k_head_tc<128><<<grid, kLThr, smem, st>>>(a, q, ph);
  } else {
    return cudaErrorInvalidValue;
  }
  return e == cudaSuccess ? cudaGetLastError() : e;
}

cudaError_t launch_parallel_layer_tc(const RunArgs& a, int j, const float* xin, float* xout, float* q,
                                     const float* pk, cudaStream_t st) {
  const dim3 grid((unsigned)((a.N + kTM - 1) / kTM), (unsigned)a.n_streams);
  cudaError_t e;
  if (a.r == R2) {
    const int smem128 = (int)sizeof(float) * (2 * kActF + 2 * kHW);
    if (a.s == 256) {
      e = cudaFuncSetAttribute(k_layer_tc128<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem128);
      if (e == cudaSuccess) k_layer_tc128<256><<<grid, kLThr, smem128, st>>>(a, j, xin, xout, q, pk);
    } else if (a.s == 128) {
      e = cudaFuncSetAttribute(k_layer_tc128<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem128);
      if (e == cudaSuccess) k_layer_tc128<128><<<grid, kLThr, smem128, st>>>(a, j, xin, xout, q, pk);
    } else {
      return cudaErrorInvalidValue;
    }
    return e == cudaSuccess ? cudaGetLastError() : e;
  }
  const int smem = (int)sizeof(float) * kSmemF;
  if (a.s == 256) {
    e = cudaFuncSetAttribute(k_layer_tc<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) k_layer_tc<256><<<grid, kLThr, smem, st>>>(a, j, xin, xout, q, pk);
  } else if (a.s == 128) {
    e = cudaFuncSetAttribute(k_layer_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) k_layer_tc<128><<<grid, kLThr, smem, st>>>(a, j, xin, xout, q, pk);
  } else {
    return cudaErrorInvalidValue;
  }
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace dvw
