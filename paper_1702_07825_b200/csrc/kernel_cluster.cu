// kernel_cluster.cu -- batch-1 persistent cluster kernel (r = 64, s in {128, 256}).
//
// The paper's GPU kernel (App. D) put two layers per SM in
// registers and passed each sample round-robin through 23 SMs with spin-locks in
// L2.  This kernel keeps the idea "one launch, weights on chip" and redesigns the
// rest for sm_100a:
//   * one thread-block cluster; every hand-off is a DSMEM st.async whose
//     transaction bytes complete on the receiver's mbarrier (no L2 round trip);
//   * chain CTAs own 3 consecutive layers.  Only ONE matvec per layer sits on
//     the critical path: a_cur^(j+1) = W_cur^(j+1) x^(j) is evaluated as
//     M^(j) h^(j) + R^(j+1), with M^(j) = W_cur^(j+1) W_res^(j) folded on the host
//     (fp64, rounded once) and R^(j+1) = W_cur^(j+1) x^(j-1) + W_cur^(j+1) B_res^(j)
//     computed concurrently by another warpgroup (same linear map as PAPER.md:
//     354 + 437, different fp32 rounding order).  Warpgroup A runs the chain
//     (a, gate), B keeps x up to date (x^(j) = x^(j-1) + W_res h + B_res, for the
//     queues and the next CTA), C computes R.  Each thread holds a (rows x
//     16-column) tile and reuses every loaded vector element across its rows;
//     partial sums meet in a transposing shuffle reduction that leaves the tanh
//     row and its sigmoid partner in one lane for the gate;
//   * all per-thread weight tiles live in tensor memory (TMEM, 256 KB per SM) and
//     are pulled into registers with tcgen05.ld right before use;
//   * the third warpgroup of a chain CTA does the off-chain work of the coming
//     sample (Fig. 2's aux threads): dilation-queue read/write in L2,
//     conditioning fetch, W_prev x_{n+1-d} + B + L from shared memory;
//   * skip CTAs accumulate W_skip^(j) h^(j) as h arrives; head CTAs
//     own 64 output rows each of relu -> W_relu -> relu -> W_out
//     plus W_skip^(l); CTA 0 samples (App. A.4) and embeds the next input (step 1).
// Shared-memory vectors are stored in padded chunks (16 floats -> stride 20) so
// the chunks a warp reads at once fall in different banks.
// Numerics: fp32 FMA; gate from ex2.approx/rcp.approx (|err| ~ 1e-7, R13);
// fp64 CDF scan (R11); every reduction has a fixed order (bitwise deterministic).
#include <algorithm>
#include <cstring>
#include <vector>

#include <cstdlib>

#include "kernel_cluster.cuh"
#include "ptx.cuh"
#include "umma.cuh"

// Timing diagnostics only (codes become wrong): build with -DDVW_DIAG=<mask> into a scratch
// copy (tools/diag_c2.sh).  1: X skips the W_prev matvec; 2: C skips its matvec; 4: B skips
// its matvec; 8: X skips the queue / conditioning / W_prev work; 16: the draw is floor(256 u);
// 32: skip CTAs skip their matvecs; 64: head CTAs skip theirs; 256: X skips the chain-skip matvec;
// 512: X's weight stream (LP = 4 multi-stream) copies but does not compute; 1024: computes, no copies.
#ifndef DVW_DIAG
#define DVW_DIAG 0
#endif
// Accumulator-chain variants under A/B measurement (profiles/r2_experiments.md): bit 1: A's matvec
// with four float2 chains per row (always at LP = 4); bit 2: B's and C's with one (default).
#ifndef DVW_EXP
#define DVW_EXP 2
#endif

namespace dvw {
namespace {

constexpr int R = 64;       // residual channels the kernel is built for
constexpr int LPC = 4;      // most layers per chain CTA (template LP = 3 or 4 per model)
constexpr int NH = 4;       // head CTAs (64 output rows each)
constexpr int kAux = 128;   // threads [0,128): warpgroup X, off-chain work
constexpr int kMain = 256;  // head / skip math threads: warpgroups A and B, [128,384)
constexpr int kMath = 384;  // warpgroups A, B, C: [128,512)
constexpr int kThreads = kAux + kMath;
constexpr int kTmemCols = 512;
// Multi-stream variant (PIPE): up to kWP streams per cluster, their samples interleaved item by item
// (item i = stream i % wc, sample i / wc), so up to wc samples are in flight along the chain at once.
constexpr int kWP = 8;
// multi-stream variant: X's pre terms live in a ring of kPR slots (item i in slot i mod kPR), computed
// kPB <= kPR - 1 items at a time (one W_prev pass and one memory latency per batch); chain-skip
// partials of up to kXH items are computed together (one W_skip pass from L2 per batch)
constexpr int kPR = 4;
constexpr int kPB = kPR - 1;
constexpr int kXH = 4;
// LP = 4 multi-stream: X streams W_prev and the chain-skip W_skip from L2 through a ring of up to kWNB
// shared-memory buffers of kWChunk floats (16 KB: 8 of a row block's 16 column quads), filled by 1-D
// bulk copies (cp.async.bulk, mbarrier complete_tx) -- many KB in flight and no registers held
constexpr int kWNB = 4;
constexpr int kWChunk = 8 * 128 * 4;
// A/B switch (profiles/r2_experiments.md): 1 = the bulk-copy weight stream above; 0 (default) = every X
// thread loads its row's 16 float4 from L2 straight into registers (measured faster: C5 shape, 256
// streams, 1.10 vs 0.96 M samples/s)
#ifndef DVW_XSTREAM
#define DVW_XSTREAM 0
#endif
constexpr bool kXStream = DVW_XSTREAM != 0;
// Timing diagnostic of the multi-stream variant (build with -DDVW_PTRACE=1 into a scratch copy,
// tools/ptrace_pipe.py): %globaltimer stamps of cluster 0's items [kPT0, kPT0 + 64) per CTA and
// event, read back with dvw_diag_ptrace.  Not compiled into the production library.
#ifndef DVW_PTRACE
#define DVW_PTRACE 0
#endif
#if DVW_PTRACE
constexpr int kPT0 = 256;
__device__ unsigned long long g_pt[kCMaxCta][64][16];
#endif
__device__ __forceinline__ void ptr(int64_t it, int ev) {
#if DVW_PTRACE
  if (it >= kPT0 && it < kPT0 + 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x == ptx::cluster_rank()) g_pt[ptx::cluster_rank()][it - kPT0][ev] = t;  // cluster 0
  }
#endif
}
constexpr uint64_t kTimeoutNs = 2000000000ull;

// named barriers (0 is __syncthreads).  A producer that only arrives gets one id per use
// within a sample, so it can never lap its consumer on one barrier.
constexpr int kBarMath = 1;  // A + B + C, 384 threads (CTA 0 sampler hand-off, teardown)
constexpr int kBarH = 2;     // chain: A and B sync (h of a non-final local layer ready), 256
constexpr int kBarAux = 3;   // X, 128
__device__ __forceinline__ constexpr int bar_xr(int jl) { return 4 + jl; }  // chain: B arrives x_{j0+jl}
                                                                            // (jl = 0..2), C syncs, 256
__device__ __forceinline__ constexpr int bar_ra(int jl) { return 7 + jl; }  // chain: C arrives R_{j0+jl}
                                                                            // (jl = 0..3), A syncs, 256
constexpr int kBarHX = 11;   // chain: A arrives (h of local layer jl in hs), X syncs and forwards it,
                             // 256; one id per local layer (11..14)
constexpr int kBarHS = 4;    // head / skip CTAs only (aliases a chain-only id): A + B, 256

// chain TMEM columns (per lane), local layer jl of layers j0..j0+LP-1:
//   A [0, 64 LP)       : W_cur_0 (CTA 0, jl = 0) or M_j = W_cur_j W_res_{j-1}   (64 each)
//   C [64 LP, 128 LP)  : W_cur_j                                                 (64 each)
//   B [384, 480), LP = 3 only : W_res_{j-1}                                      (32 each)
constexpr int kColA = 0;

enum Role { kChain = 0, kHead = 1, kSkip = 2, kIdle = 3 };

// Vectors are read in column chunks of C floats; chunk c starts at c (C + 4), so the
// (up to 8) chunks one warp instruction touches occupy distinct bank groups.
template <int C>
__device__ __forceinline__ int cpad(int i) { return i + (i / C) * 4; }
__device__ __forceinline__ int pad16(int i) { return i + ((i >> 4) << 2); }
constexpr int kHLen = 80;   // 64-vector in 4 chunks of 16
constexpr int kVLen = 320;  // 256-vector in 16 chunks of 16 (or 8)

struct __align__(16) Mail {
  uint64_t bar_hin, bar_xin, bar_logits, bar_pre, bar_done, bar_part, bar_za, bar_exit;
  uint64_t bar_h[kCMaxSlot];
  int abort_flag;
  uint32_t tmem_base;                       // tensor-memory allocation (column 0, lane 0)
  // chain CTA with layers j0..j0+nl-1 (x_j = input of layer j, h_j = its gate output):
  alignas(16) float hin[kHLen];             // h_{j0-1} from the previous chain CTA (pad16)
  alignas(16) float xin[kHLen];             // x_{j0-1} from the previous chain CTA (pad16)
  alignas(16) float xs[2][LPC][kHLen];      // [sample parity][jl] x_{j0+jl} (pad16); CTA 0: xs[.][0] = embedding
  alignas(16) float hs[2][LPC][kHLen];      // [sample parity][jl] h_{j0+jl} (pad16)
  float rr[LPC][2 * R];                     // R_j = W_cur_j x_{j-1} + W_cur_j B_res_{j-1}, from C
  float pre[LPC][2 * R];                    // W_prev x_{n-d} + B + L for the coming sample, from X
  float xp[R];                              // X scratch
  float logits_in[kLevels];                 // CTA 0: inbound logits
  float hbuf[kCMaxSlot][kHLen];             // skip: h^(j) per owned slot; head: slot 0 = h^(l) (pad16)
  float part[kCMaxSkip][256];               // head: skip partials
  float za_in[kVLen];                       // head: all-gathered z_a (pad16)
  float zs[kVLen];                          // head: z_s (cpad<s/16>); skip: partial staging
  double dscr[8];
  float fscr[8];
  int iscr[16];
  // multi-stream variant (PIPE): one mailbox barrier per stream of the cluster (the data live in the
  // mailbox region after Mail, see mb_*), and CTA 0's code history per stream
  uint64_t pb_hin[kWP], pb_xin[kWP], pb_logits[kWP], pb_part[kWP], pb_za[kWP];
  uint64_t pb_h[kCMaxSlot][kWP];
  int ys[kWP][2];
  // PIPE: one barrier per slot of X's pre ring (the ring itself is in the chain's mailbox region)
  uint64_t bar_pre2[kPR];
  uint64_t wfull[kWNB];  // PIPE, LP = 4: X's weight-stream buffers (bulk copy landed)
};

struct Params {
  RunArgs a;
  ClusterPlan p;
  const float* pk;
  int wmax;  // streams per cluster (1, or up to kWP for the multi-stream variant)
  int xpb;   // PIPE: X's pre batch (1..kPB; capped at streams - 1 per cluster)
  int xsb;   // PIPE: chain-skip batch (1..kXH)
};

struct Ctx {
  Mail* mail;
  int* err;
  int size;
  int64_t sidx;  // the stream this cluster generates (one cluster per stream: cluster index)
  // per thread (every thread builds its own Ctx): set by the thread's first failed wait.  From then on
  // the thread never re-arms a barrier: after an abort a barrier can stay in one phase, and a later
  // parity probe of the other phase succeeds spuriously -- arming it again would arrive twice in
  // that phase (an mbarrier fault).  The roles still run every sample, so named barriers between
  // warpgroups stay matched.
  mutable bool dead;
  float* mb;  // PIPE: this CTA's mailbox region (per-stream inbound data; same offset in every CTA)
  int wc;     // streams this cluster generates (1 unless PIPE)
};

// Coordinates of item `it` of a cluster's interleaved sequence: stream s (the mailbox slot), sample
// n of that stream (mailbox barriers flip phase once per sample of their stream: parity n & 1),
// and p = it & 1, the parity of the CTA-local double buffers (xs, hs, pre; one item after another).
struct Item {
  int64_t n;
  int s, p;
  uint32_t par;
};
template <bool PIPE>
__device__ __forceinline__ Item item_of(int64_t it, int wc) {
  Item x;
  if constexpr (PIPE) {  // 32-bit division: the host keeps N x wc < 2^31 for this variant
    const uint32_t iu = (uint32_t)it, w = (uint32_t)wc;
    x.s = (int)(iu % w);
    x.n = (int64_t)(iu / w);
  } else {
    x.s = 0;
    x.n = it;
  }
  x.p = (int)(it & 1);
  x.par = (uint32_t)(x.n & 1);
  return x;
}

// Inbound mailboxes: single buffers in Mail (one stream), or per-stream slots in the mailbox region.
// Region layout (floats): chain: hin [kWP][kHLen], xin [kWP][kHLen], logits [kWP][256];
// head: hbuf slots 0-1 [2][kWP][kHLen], za [kWP][kVLen], part [npart][kWP][256]; skip: hbuf [slots][kWP][kHLen].
template <bool PIPE>
__device__ __forceinline__ float* mb_hin(const Ctx& cx, int s) {
  if constexpr (PIPE) return cx.mb + s * kHLen; else return cx.mail->hin;
}
template <bool PIPE>
__device__ __forceinline__ float* mb_xin(const Ctx& cx, int s) {
  if constexpr (PIPE) return cx.mb + (kWP + s) * kHLen; else return cx.mail->xin;
}
template <bool PIPE>
__device__ __forceinline__ float* mb_logits(const Ctx& cx, int s) {
  if constexpr (PIPE) return cx.mb + 2 * kWP * kHLen + s * kLevels; else return cx.mail->logits_in;
}
// chain mailbox region, after the logits: X's pre ring [kPR][LPC][2R], its queue-entry staging
// [kPB][LPC][R], and (LP = 4) the chain-skip history [kXH][LPC][kHLen] + partial staging [kXH][256]
constexpr int kMbPre = 2 * kWP * kHLen + kWP * kLevels;
constexpr int kMbXst = kMbPre + kPR * LPC * 2 * R;
constexpr int kMbHist = kMbXst + kPB * LPC * R;
constexpr int kMbXstage = kMbHist + kXH * LPC * kHLen;
constexpr int kMbChainEnd3 = kMbHist;                 // LP = 3: no chain-skip layers
constexpr int kMbChainEnd4 = kMbXstage + kXH * 256;  // then (LP = 4) the weight-stream ring [xnb][kWChunk]
__device__ __forceinline__ float* mb_pre(const Ctx& cx, int slot) { return cx.mb + kMbPre + slot * LPC * 2 * R; }
__device__ __forceinline__ float* mb_xst(const Ctx& cx, int k) { return cx.mb + kMbXst + k * LPC * R; }
__device__ __forceinline__ float* mb_hist(const Ctx& cx, int k) { return cx.mb + kMbHist + k * LPC * kHLen; }
__device__ __forceinline__ float* mb_xstage(const Ctx& cx, int k) { return cx.mb + kMbXstage + k * 256; }
template <bool PIPE>
__device__ __forceinline__ float* mb_hbuf(const Ctx& cx, int sl, int s) {
  if constexpr (PIPE) return cx.mb + (sl * kWP + s) * kHLen; else return cx.mail->hbuf[sl];
}
template <bool PIPE>
__device__ __forceinline__ float* mb_za(const Ctx& cx, int s) {
  if constexpr (PIPE) return cx.mb + 2 * kWP * kHLen + s * kVLen; else return cx.mail->za_in;
}
template <bool PIPE>
__device__ __forceinline__ float* mb_part(const Ctx& cx, int kk, int s) {
  if constexpr (PIPE) return cx.mb + 2 * kWP * kHLen + kWP * kVLen + (kk * kWP + s) * 256; else return cx.mail->part[kk];
}
template <bool PIPE>
__device__ __forceinline__ uint64_t* b_hin(const Ctx& cx, int s) {
  if constexpr (PIPE) return &cx.mail->pb_hin[s]; else return &cx.mail->bar_hin;
}
template <bool PIPE>
__device__ __forceinline__ uint64_t* b_xin(const Ctx& cx, int s) {
  if constexpr (PIPE) return &cx.mail->pb_xin[s]; else return &cx.mail->bar_xin;
}
template <bool PIPE>
__device__ __forceinline__ uint64_t* b_logits(const Ctx& cx, int s) {
  if constexpr (PIPE) return &cx.mail->pb_logits[s]; else return &cx.mail->bar_logits;
}
template <bool PIPE>
__device__ __forceinline__ uint64_t* b_part(const Ctx& cx, int s) {
  if constexpr (PIPE) return &cx.mail->pb_part[s]; else return &cx.mail->bar_part;
}
template <bool PIPE>
__device__ __forceinline__ uint64_t* b_za(const Ctx& cx, int s) {
  if constexpr (PIPE) return &cx.mail->pb_za[s]; else return &cx.mail->bar_za;
}
template <bool PIPE>
__device__ __forceinline__ uint64_t* b_h(const Ctx& cx, int sl, int s) {
  if constexpr (PIPE) return &cx.mail->pb_h[sl][s]; else return &cx.mail->bar_h[sl];
}

// This cluster's stream inside the [S][...] caller buffers.
// (s: the stream within a multi-stream cluster)
__device__ __forceinline__ const float* s_uniforms(const RunArgs& A, const Ctx& cx, int s = 0) {
  return A.uniforms ? A.uniforms + (cx.sidx + s) * A.N : nullptr;
}
__device__ __forceinline__ const uint8_t* s_forced(const RunArgs& A, const Ctx& cx, int s = 0) {
  return A.forced ? A.forced + (cx.sidx + s) * A.N : nullptr;
}
__device__ __forceinline__ float* s_logits(const RunArgs& A, const Ctx& cx, int s = 0) {
  return A.out_logits + (cx.sidx + s) * A.N * kLevels;
}
__device__ __forceinline__ uint8_t* s_codes(const RunArgs& A, const Ctx& cx, int s = 0) {
  return A.out_codes + (cx.sidx + s) * A.N;
}
__device__ __forceinline__ int* s_ystate(const RunArgs& A, const Ctx& cx) { return A.ystate + 2 * cx.sidx; }

__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void raise_abort(const Ctx& cx, int code) {
  *reinterpret_cast<volatile int*>(cx.err) = code;  // mapped host memory
  __threadfence_system();
  const uint32_t a = ptx::smem_u32(&cx.mail->abort_flag);
#pragma unroll 1
  for (int r = 0; r < cx.size; ++r) {
    const uint32_t ra = ptx::mapa(a, r);
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(1) : "memory");
  }
}

// Wait for phase `parity` of a local mbarrier (try_wait suspends the warp in
// hardware).  On the watchdog (2 s without progress) or a cluster-wide abort,
// return false: the caller runs on without blocking so every CTA reaches the
// final cluster barrier, and the host sees DVW_E_DEVICE_TIMEOUT.
// CTA-scope acquire: every hand-off into this CTA is a st.async into its own shared memory,
// tracked by the mbarrier's transaction count, so observing the phase makes the data visible;
// a cluster-scope acquire would also invalidate L1 (CCTL.IVALL) on every wake-up.
__device__ __forceinline__ bool wait(const Ctx& cx, uint64_t* bar, uint32_t parity, int code) {
  const uint32_t b = ptx::smem_u32(bar);
  if (ptx::mbar_try_wait_cta(b, parity)) return true;
  const uint64_t t0 = ptx::globaltimer();
#pragma unroll 1
  for (uint32_t i = 1;; ++i) {
    if (ptx::mbar_try_wait_cta(b, parity)) return true;
    if ((i & 7) == 0) {
      if (*reinterpret_cast<volatile int*>(&cx.mail->abort_flag)) {
        cx.dead = true;
        return false;
      }
      if (ptx::globaltimer() - t0 > kTimeoutNs) {
        raise_abort(cx, code);
        cx.dead = true;
        return false;
      }
    }
  }
}

__device__ __forceinline__ uint32_t remote(const void* local, int rank) {
  return ptx::mapa(ptx::smem_u32(local), (uint32_t)rank);
}

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// Optional %globaltimer stamps (dvw_set_trace).  Compiled only into the TRACE
// instantiation of the kernel, so the production kernel carries no trace code.
template <bool TRACE>
__device__ __forceinline__ void trace(const RunArgs& A, int64_t n, int ev) {
  if constexpr (TRACE) {
    const int64_t i = n - A.trace_n0;
    if (i >= 0 && i < A.trace_count) A.trace[(i * kCMaxCta + ptx::cluster_rank()) * 32 + ev] = ptx::globaltimer();
  }
}

// Per-sample slot of this CTA in the trace buffer (nullptr outside the window), so an
// event inside the chain costs one clock read and one store.
template <bool TRACE>
__device__ __forceinline__ uint64_t* trace_slot(const RunArgs& A, int64_t n) {
  if constexpr (TRACE) {
    const int64_t i = n - A.trace_n0;
    if (i >= 0 && i < A.trace_count) return A.trace + (i * kCMaxCta + ptx::cluster_rank()) * 32;
  }
  return nullptr;
}
template <bool TRACE>
__device__ __forceinline__ void stamp(uint64_t* tp, int ev) {
  if constexpr (TRACE) {
    if (tp) tp[ev] = clock64();
  }
}

template <bool TRACE>
__device__ __forceinline__ void trace_clk(const RunArgs& A, int64_t n, int ev) {
  if constexpr (TRACE) {
    const int64_t i = n - A.trace_n0;
    if (i >= 0 && i < A.trace_count) A.trace[(i * kCMaxCta + ptx::cluster_rank()) * 32 + ev] = clock64();
  }
}

// Packed fp32 FMA (FFMA2, sm_100): {c.x + a.x b.x, c.y + a.y b.y}, each rounded exactly
// like fmaf -- the same results as two scalar FMAs at ~1.4x the issue rate (measured
// 118 vs 85 FMA/clk/SM, tools/ffma2_probe.cu), so every matvec below pairs its two
// independent accumulator chains into one FFMA2.
__device__ __forceinline__ float2 ffma2(float a0, float a1, float b0, float b1, float2 c) {
  return __ffma2_rn(make_float2(a0, a1), make_float2(b0, b1), c);
}

// Register tile x vector chunk: acc[m] = sum_c w[m*C + c] * v[c] for RQ rows and a
// C-float chunk of a shared vector; two accumulators per row (even/odd c) for ILP.
// Summation order is fixed (bitwise deterministic).
template <int RQ, int C>
__device__ __forceinline__ void tile_dot(const float* w, const float* v, float (&acc)[RQ]) {
  float2 eo[RQ];  // (even, odd) accumulators
#pragma unroll
  for (int m = 0; m < RQ; ++m) eo[m] = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int c = 0; c < C; c += 4) {
    const float4 x = lds4(v + c);
#pragma unroll
    for (int m = 0; m < RQ; ++m) {
      eo[m] = ffma2(w[m * C + c], w[m * C + c + 1], x.x, x.y, eo[m]);
      eo[m] = ffma2(w[m * C + c + 2], w[m * C + c + 3], x.z, x.w, eo[m]);
    }
  }
#pragma unroll
  for (int m = 0; m < RQ; ++m) acc[m] = eo[m].x + eo[m].y;
}

// Register tile x one 32-column half of a padded 64-vector (two 16-float chunks at v and
// v + 20): acc[m] = sum_c w[m*32 + c] * vec[c]; four accumulators per row (c % 4) for ILP,
// combined in a fixed order (bitwise deterministic).
template <int RQ>
__device__ __forceinline__ void tile_dot_half(const float* w, const float* v, float (&acc)[RQ]) {
  float2 s01[RQ], s23[RQ];
#pragma unroll
  for (int m = 0; m < RQ; ++m) s01[m] = s23[m] = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int c = 0; c < 32; c += 4) {
    const float4 x = lds4(v + c + ((c >> 4) << 2));
#pragma unroll
    for (int m = 0; m < RQ; ++m) {
      s01[m] = ffma2(w[m * 32 + c], w[m * 32 + c + 1], x.x, x.y, s01[m]);
      s23[m] = ffma2(w[m * 32 + c + 2], w[m * 32 + c + 3], x.z, x.w, s23[m]);
    }
  }
#pragma unroll
  for (int m = 0; m < RQ; ++m) acc[m] = (s01[m].x + s01[m].y) + (s23[m].x + s23[m].y);
}

// tile_dot_half with four (NCH = 4) or one (NCH = 1) float2 accumulator chains per row instead
// of two; fixed combine order (bitwise deterministic).  One chain makes B's and C's matvecs
// yield issue slots to A's (C2 7.45 vs 7.51 us); four make A's faster at LP = 4 (C3).
template <int RQ, int NCH>
__device__ __forceinline__ void tile_dot_half_n(const float* w, const float* v, float (&acc)[RQ]) {
  float2 s[RQ][NCH];
#pragma unroll
  for (int m = 0; m < RQ; ++m)
#pragma unroll
    for (int i = 0; i < NCH; ++i) s[m][i] = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int c = 0; c < 32; c += 8) {
    const float4 x0 = lds4(v + c + ((c >> 4) << 2));
    const float4 x1 = lds4(v + c + 4 + ((c >> 4) << 2));
#pragma unroll
    for (int m = 0; m < RQ; ++m) {
      s[m][0] = ffma2(w[m * 32 + c], w[m * 32 + c + 1], x0.x, x0.y, s[m][0]);
      s[m][1 % NCH] = ffma2(w[m * 32 + c + 2], w[m * 32 + c + 3], x0.z, x0.w, s[m][1 % NCH]);
      s[m][2 % NCH] = ffma2(w[m * 32 + c + 4], w[m * 32 + c + 5], x1.x, x1.y, s[m][2 % NCH]);
      s[m][3 % NCH] = ffma2(w[m * 32 + c + 6], w[m * 32 + c + 7], x1.z, x1.w, s[m][3 % NCH]);
    }
  }
#pragma unroll
  for (int m = 0; m < RQ; ++m) {
    if constexpr (NCH == 4)
      acc[m] = ((s[m][0].x + s[m][0].y) + (s[m][1].x + s[m][1].y)) + ((s[m][2].x + s[m][2].y) + (s[m][3].x + s[m][3].y));
    else
      acc[m] = s[m][0].x + s[m][0].y;
  }
}

// One transposing level of a butterfly reduction: lanes whose `bit` is set keep
// the upper half of the row values and send the lower half to their partner,
// which keeps the lower half.  Halves the row count per lane with N/2 shuffles.
template <int N>
__device__ __forceinline__ void xpose_level(float (&v)[N], int lane, int bit) {
  const bool up = (lane & bit) != 0;
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const float send = up ? v[i] : v[i + N / 2];
    const float keep = up ? v[i + N / 2] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
  }
}

// ------------------------------------------------------------------ chain CTA 0: sample + embed
// Inverse-CDF direct sampling (reading R11) by ONE warp, 8 logits per
// lane, no block barriers: m = max l; e_k = exp(l_k - m) (fp32); P_k = running sums in
// ascending k; y = #{k : P_k <= u * P_255}; fallback the largest k with e_k > 0.
// The decision is defined by fp64 running sums (R11).  It is first taken with fp32 sums
// (d = 2^-24): a lane's prefix sums carry <= 7 d T_lane, the 5-level scan <= 5 d S (each
// level's adds cover disjoint lanes), so the fp32 lane base is within 20 d S and each fp32
// P_k within 28 d S of its exact value, and u * S within 13 d S; when no P_k lies within
// M = 64 d S > 41 d S of the threshold the fp32 count equals the fp64 count exactly;
// otherwise (about 2 * 256 * M / S ~ 0.2 % of draws) the fp64 sums decide.  Bitwise the
// same codes as the fp64-only sampler.
// The fp64 decision (reading R11): out of line, it runs for ~0.1 % of draws only.
__device__ __noinline__ int sample_fp64(float e0, float e1, float e2, float e3, float e4, float e5, float e6,
                                        float e7, float u, int lane) {
  const float e[8] = {e0, e1, e2, e3, e4, e5, e6, e7};
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
  const double base = incl - p[7];  // exclusive prefix of the lane totals
  const double S = __shfl_sync(0xffffffffu, incl, 31);
  const double thr = (double)u * S;
  int cnt = 0, lastpos = -1;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    cnt += (base + p[i] <= thr) ? 1 : 0;
    if (e[i] > 0.0f) lastpos = 8 * lane + i;
  }
  const int y = __reduce_add_sync(0xffffffffu, cnt);
  return y < kLevels ? y : __reduce_max_sync(0xffffffffu, (unsigned)(lastpos + 1)) - 1;
}

template <int NL>
__device__ __forceinline__ int sample_warp(const float* logits, float u, int lane) {
  float l[8];
  {
    const float4 a = lds4(logits + 8 * lane), b = lds4(logits + 8 * lane + 4);
    l[0] = a.x; l[1] = a.y; l[2] = a.z; l[3] = a.w; l[4] = b.x; l[5] = b.y; l[6] = b.z; l[7] = b.w;
  }
  const float lmx = fmaxf(fmaxf(fmaxf(l[0], l[1]), fmaxf(l[2], l[3])), fmaxf(fmaxf(l[4], l[5]), fmaxf(l[6], l[7])));
  // warp max in one redux.sync on order-preserving integer keys (exact: the key map is a
  // bijection that keeps the order of finite floats), instead of five shuffle + max steps
  const unsigned kmx = __reduce_max_sync(0xffffffffu, ordered_key(lmx));
  const float mx = __uint_as_float((kmx & 0x80000000u) ? (kmx & 0x7fffffffu) : ~kmx);
  float e[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if constexpr (NL == 2) {
      e[i] = appc_exp(l[i] - mx);  // App. C.2 (R31)
    } else if constexpr ((DVW_EXP & 8) != 0) {  // A/B: exp as one MUFU ex2 of (l - m) log2(e)
      float r;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((l[i] - mx) * 1.4426950408889634f));
      e[i] = r;
    } else {
      e[i] = expf(l[i] - mx);
    }
  }
  // fp32 pass
  float q[8];
  q[0] = e[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) q[i] = q[i - 1] + e[i];
  float inc = q[7];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  const float fbase = inc - q[7];
  const float fS = __shfl_sync(0xffffffffu, inc, 31);
  const float fthr = u * fS;
  const float M = 3.8146973e-06f * fS;  // 64 * 2^-24 * S
  int fcnt = 0;
  bool near = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float P = fbase + q[i];
    fcnt += (P <= fthr) ? 1 : 0;
    near |= fabsf(P - fthr) <= M;
  }
  const int fy = __reduce_add_sync(0xffffffffu, fcnt);
  if (!__any_sync(0xffffffffu, near) && fy < kLevels) return fy;
  return sample_fp64(e[0], e[1], e[2], e[3], e[4], e[5], e[6], e[7], u, lane);
}

// Draw y_{n-1} from the inbound logits (App. A.4) and write x^(0)_n (step 1) into xs[n&1][0]
// with the first warp of warpgroup A; warpgroups A, B, C wait at the closing barrier.
template <bool TRACE, int NL = 0, bool PIPE = false>
__device__ __forceinline__ void sample_and_embed(const Params& P, const Ctx& cx, const Item& I, int k, int& y1,
                                                 int& y2, const float* wembc, const float* bemb) {
  const RunArgs& A = P.a;
  Mail& m = *cx.mail;
  const int64_t n = I.n;
  if (k < 32) {
    if constexpr (PIPE) {  // this stream's code history
      y1 = m.ys[I.s][0];
      y2 = m.ys[I.s][1];
    }
    const float* embp_g = P.pk + P.p.embp_off;  // W_emb_prev^T [256][R] in global memory
    float ep0, ep1;
    if (n > 0) {
      const float* ub = s_uniforms(A, cx, I.s);
      const uint8_t* fb = s_forced(A, cx, I.s);
      const float u = ub ? __ldg(ub + n - 1) : 0.0f;
      const int yf = fb ? (int)__ldg(fb + n - 1) : 0;
      ep0 = __ldg(embp_g + y1 * R + k);  // W_emb_prev[:, y_{n-2}] (= y1 before the update)
      ep1 = __ldg(embp_g + y1 * R + k + 32);
      uint64_t* tp = (k == 0) ? trace_slot<TRACE>(A, n) : nullptr;
      const float* lin = mb_logits<PIPE>(cx, I.s);
      if (wait(cx, b_logits<PIPE>(cx, I.s), (uint32_t)((n - 1) & 1), 11) && k == 0 && !cx.dead)
        ptx::mbar_arm(ptx::smem_u32(b_logits<PIPE>(cx, I.s)), kLevels * 4);
      stamp<TRACE>(tp, 1);
      if (PIPE && k == 0) ptr(n * cx.wc + I.s, 6);
      if (k == 0) trace<TRACE>(A, n - 1, 3);
      int y;
      if (fb) {
        float4* o = reinterpret_cast<float4*>(s_logits(A, cx, I.s) + (n - 1) * kLevels) + 2 * k;
        o[0] = lds4(lin + 8 * k);
        o[1] = lds4(lin + 8 * k + 4);
        y = yf;
      } else {
        stamp<TRACE>(tp, 4);
        if constexpr ((DVW_DIAG & 16) != 0) y = min((int)(u * 256.0f) + (lin[0] > 1e30f), 255);
        else y = sample_warp<NL>(lin, u, k);
        stamp<TRACE>(tp, 6);
        if (k == 0) s_codes(A, cx, I.s)[n - 1] = (uint8_t)y;
      }
      if (k == 0) trace<TRACE>(A, n, 20);
      if (PIPE && k == 0) ptr(n * cx.wc + I.s, 7);
      y2 = y1;
      y1 = y;
    } else {
      ep0 = __ldg(embp_g + y2 * R + k);
      ep1 = __ldg(embp_g + y2 * R + k + 32);
    }
    if constexpr (PIPE) {
      __syncwarp();
      if (k == 0) {
        m.ys[I.s][0] = y1;
        m.ys[I.s][1] = y2;
      }
    }
    // x^(0)_n = W_emb_prev[:, y_{n-2}] + W_emb_cur[:, y_{n-1}] + B_emb
    float* x0 = m.xs[I.p][0];
    x0[pad16(k)] = (ep0 + wembc[y1 * R + k]) + bemb[k];
    x0[pad16(k + 32)] = (ep1 + wembc[y1 * R + k + 32]) + bemb[k + 32];
    if (k == 0) stamp<TRACE>(trace_slot<TRACE>(A, n), 7);
  }
  ptx::bar_sync(kBarMath, kMath);
  if (k == 0) stamp<TRACE>(trace_slot<TRACE>(A, n), 30);
}

// The final draw (sample N-1) after the last layer pass (first warp of A); returns it.
template <int NL = 0, bool PIPE = false>
__device__ __forceinline__ int final_draw(const Params& P, const Ctx& cx, int k, int s = 0) {
  const RunArgs& A = P.a;
  if (k >= 32) return 0;
  const int64_t n = A.N;
  const float* ub = s_uniforms(A, cx, s);
  const float u = ub ? __ldg(ub + n - 1) : 0.0f;
  const float* lin = mb_logits<PIPE>(cx, s);
  wait(cx, b_logits<PIPE>(cx, s), (uint32_t)((n - 1) & 1), 11);
  int y = 0;
  if (A.forced) {
    float4* o = reinterpret_cast<float4*>(s_logits(A, cx, s) + (n - 1) * kLevels) + 2 * k;
    o[0] = lds4(lin + 8 * k);
    o[1] = lds4(lin + 8 * k + 4);
  } else {
    y = sample_warp<NL>(lin, u, k);
    if (k == 0) s_codes(A, cx, s)[n - 1] = (uint8_t)y;
  }
  return y;
}

// TMEM address of this thread's lane (warp w of a warpgroup owns lanes 32w..32w+31)
__device__ __forceinline__ uint32_t tmem_lane_addr(const Mail& m) {
  return m.tmem_base + ((uint32_t)(32 * ((threadIdx.x >> 5) & 3)) << 16);
}

// Shared-memory image of a chain CTA (floats), local layer jl of layer j = j0 + jl:
// (LP = 4 only) W_res_{j-1} [LPC][8 (q/4)][128 (B thread)][4] (B's row-pair tiles, one
// conflict-free LDS.128 per 4 columns), B_j [LPC][2R], B_res_{j-1} [LPC][R], c_j = W_cur_j B_res_{j-1} [LPC][2R]; CTA 0 adds
// W_emb_cur^T [256][R], B_emb [R].  W_prev streams from L2 (the aux warps, off the chain).
constexpr int kSmWres = 0;
// LP = 4: W_res tiles; LP = 3: W_prev [3][16][128][4] (at LP = 4 it streams from L2)
__host__ __device__ constexpr int sm_b(int lp) { return lp == 4 ? LPC * 32 * 128 : 3 * 16 * 128 * 4; }
__host__ __device__ constexpr int sm_bres(int lp) { return sm_b(lp) + LPC * 2 * R; }
__host__ __device__ constexpr int sm_fold(int lp) { return sm_bres(lp) + LPC * R; }
__host__ __device__ constexpr int sm_emb(int lp) { return sm_fold(lp) + LPC * 2 * R; }
// floats of a chain CTA's shared-memory image (see sm_*; LP = 4 appends nwp W_prev layers)
__host__ __device__ constexpr int smem_chain(int c, int lp) { return sm_emb(lp) + (c == 0 ? kLevels * R + R : 0); }
// TMEM: A [0, 64 LP), C [64 LP, 128 LP); at LP = 3 B's W_res tiles sit in [384, 480)
__host__ __device__ constexpr int col_c(int lp) { return 64 * lp; }
constexpr int kColB3 = 384;

// The chain, per chain CTA c with layers j0..j0+nl-1 (x_j = input of layer j, h_j = its gate
// output, a_j = W_cur_j x_j + pre_j, x_{j+1} = x_j + W_res_j h_j + B_res_j):
// a_j is evaluated as M_j h_{j-1} + R_j with M_j = W_cur_j W_res_{j-1} (folded on the host, R22)
// and R_j = W_cur_j x_{j-1} + W_cur_j B_res_{j-1}, so only ONE matvec per layer (A) sits on the
// sample's critical chain, also across CTAs: CTA c >= 1 receives h_{j0-1} (from the previous A,
// the critical hop) and x_{j0-1} (from the previous B, one layer earlier).  CTA 0 starts from the
// embedding x_0 and evaluates a_0 = W_cur_0 x_0 directly.
//   A: a_j, gate -> h_j (and for the CTA's last layer: h straight to the next CTA / the heads)
//   B: x_{j0+jl} = x_{j0+jl-1} + W_res h_{j0+jl-1} + B_res (queues, C, next CTA)
//   C: R_{j0+jl} from x_{j0+jl-1}
//   X: forwards h to skip / head CTAs, dilation queues, pre for the coming sample
// Warpgroups A, C: thread a owns rows {g, R+g} (tanh g, sigmoid g), g = a / 2, columns
// [32 half, 32 half + 32), half = a % 2 -- one shuffle finishes both rows in both lanes of the
// pair, where the gate runs.  B: row g of W_res, same columns.

// ------------------------------------------------------------------ chain CTA, warpgroup A (the chain)
template <int LP, bool TRACE, int NL, bool SESS, bool PIPE>
__device__ void chain_A(const Params& P, const Ctx& cx, int c, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int a = threadIdx.x - kAux;  // 0..127 (also the sampler's thread index)
  const int hrow = a >> 1, half = a & 1;  // rows hrow (tanh) and R + hrow (sigmoid), columns [32 half, +32)
  const bool writer = half == 0;
  const int voff = 40 * half;             // padded offset of column 32 half
  const int nl = pl.chain_nl[c];
  const bool last_cta = (c == pl.nc - 1);
  const uint32_t tm = tmem_lane_addr(m) + kColA;
  const float* wembc = sw + sm_emb(LP);  // CTA 0: [256][R]
  const float* bemb = wembc + kLevels * R;
  int y1 = SESS ? s_ystate(A, cx)[0] : kLevels / 2, y2 = SESS ? s_ystate(A, cx)[1] : kLevels / 2;
  float w[64];

  for (int64_t it = 0; it < A.N * cx.wc; ++it) {
    const Item I = item_of<PIPE>(it, cx.wc);
    const int64_t n = I.n;
    const int p = I.p;
    const float* hinb = mb_hin<PIPE>(cx, I.s);
    ptx::tmem_load_async<64>(tm, w);  // layer j0's tile, hidden behind the waits
    if (c == 0) {
      sample_and_embed<TRACE, NL, PIPE>(P, cx, I, a, y1, y2, wembc, bemb);
    } else {
      if (wait(cx, b_hin<PIPE>(cx, I.s), I.par, 12) && a == 0 && !cx.dead) ptx::mbar_arm(ptx::smem_u32(b_hin<PIPE>(cx, I.s)), R * 4);
    }
    if (a == 0) trace<TRACE>(A, n, 0);
    if (PIPE && a == 0) ptr(it, 1);
    uint64_t* tp = (a == 0) ? trace_slot<TRACE>(A, n) : nullptr;
    if constexpr (PIPE) wait(cx, &m.bar_pre2[it % kPR], (uint32_t)((it / kPR) & 1), 13);
    else wait(cx, &m.bar_pre, (uint32_t)p, 13);
    if (PIPE && a == 0) ptr(it, 0);
    const float* prev_pre = PIPE ? mb_pre(cx, (int)(it % kPR)) : &m.pre[0][0];
    ptx::tmem_wait_ld<64>(w);
#pragma unroll
    for (int jl = 0; jl < LP; ++jl) {
      if (jl < nl) {
        const bool direct = (c == 0 && jl == 0);  // a_0 = W_cur_0 x_0
        stamp<TRACE>(tp, 8 + 2 * jl);
        const float pre0 = prev_pre[jl * 2 * R + hrow], pre1 = prev_pre[jl * 2 * R + R + hrow];
        float v[2];
        if constexpr ((DVW_EXP & 1) != 0 || LP == 4)
          tile_dot_half_n<2, 4>(w, (direct ? m.xs[p][0] : (jl == 0 ? hinb : m.hs[p][jl - 1])) + voff, v);
        else
          tile_dot_half<2>(w, (direct ? m.xs[p][0] : (jl == 0 ? hinb : m.hs[p][jl - 1])) + voff, v);
        if (jl + 1 < nl) ptx::tmem_load_async<64>(tm + 64 * (jl + 1), w);  // next layer's tile
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);  // both lanes of the pair: full (tanh, sigmoid) rows
        v[1] += __shfl_xor_sync(0xffffffffu, v[1], 1);
        if (!direct) {
          stamp<TRACE>(tp, 14 + jl);
          ptx::bar_sync(bar_ra(jl), kMain);  // R_j from C
          stamp<TRACE>(tp, 17 + jl);
          v[0] += m.rr[jl][hrow];
          v[1] += m.rr[jl][R + hrow];
        }
        // a = a_cur + (W_prev x_{n-d} + B + L); h = tanh(a_h) sigma(a_g)
        const float hv = NL == 1   ? gate_approx(v[0] + pre0, v[1] + pre1)
                         : NL == 2 ? gate_appc(v[0] + pre0, v[1] + pre1)
                                   : gate_fast(v[0] + pre0, v[1] + pre1);
        stamp<TRACE>(tp, 27 + jl);
        if (PIPE && a == 0) ptr(it, 2 + jl);
        if (jl + 1 == nl) {
          // the CTA's last layer: h goes straight to the next chain CTA (or, for layer l, to the
          // four heads) -- the only hop on the critical chain between two CTAs
          // four heads: X sends one 16-byte st.async per thread (one instruction)
          if (writer) {
            if (!last_cta)
              ptx::st_async(remote(mb_hin<PIPE>(cx, I.s) + pad16(hrow), c + 1), hv, remote(b_hin<PIPE>(cx, I.s), c + 1));
            m.hs[p][jl][pad16(hrow)] = hv;
          }
          bar_arrive(kBarHX + jl, kMain);  // X forwards h_{L-1}, h_{L-2} / skip-layer h
          stamp<TRACE>(tp, 9 + 2 * jl);
        } else {
          if (writer) m.hs[p][jl][pad16(hrow)] = hv;
          ptx::bar_sync(kBarH, kMain);     // h_j complete for A (next layer) and B
          bar_arrive(kBarHX + jl, kMain);  // ... and for X, which forwards it to the skip / head CTAs
          stamp<TRACE>(tp, 9 + 2 * jl);
          ptx::tmem_wait_ld<64>(w);
        }
      }
    }
  }
  if (c == 0 && A.N > 0) {
    for (int s = 0; s < cx.wc; ++s) {
      const int y = final_draw<NL, PIPE>(P, cx, a, s);
      if (SESS && a == 0 && !A.forced) {  // streaming session: the code history for the next call
        s_ystate(A, cx)[0] = y;
        s_ystate(A, cx)[1] = y1;
      }
    }
  }
}

// ------------------------------------------------------------------ chain CTA, warpgroup B (x updates)
// x_{j0+jl} = x_{j0+jl-1} + W_res_{j0+jl-1} h_{j0+jl-1} + B_res_{j0+jl-1} for
// jl >= xb (CTA 0 starts from the embedding): for the dilation queues, for C, and (jl = nl-1)
// for the next chain CTA.
template <int LP, bool TRACE, bool SESS, bool PIPE>
__device__ void chain_B(const Params& P, const Ctx& cx, int c, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int b = threadIdx.x - kAux - 128;  // 0..127
  const int k = threadIdx.x - kAux;        // sampler thread index (>= 128: waits only)
  const int row = b >> 1, half = b & 1;    // row of x this lane pair finishes, columns [32 half, +32)
  const bool writer = half == 0;
  const int voff = 40 * half;
  const int nl = pl.chain_nl[c];
  const int xb = (c == 0) ? 1 : 0;
  const bool last_cta = (c == pl.nc - 1);
  const float* wres = sw + kSmWres;  // LP = 4: [LPC][8][128][4] in shared memory
  const uint32_t tmb = tmem_lane_addr(m) + kColB3;  // LP = 3: tensor memory
  const float* bres = sw + sm_bres(LP);  // [LPC][R]: B_res_{j0+jl-1}
  const float* wembc = sw + sm_emb(LP);
  const float* bemb = wembc + kLevels * R;
  int y1 = SESS ? s_ystate(A, cx)[0] : kLevels / 2, y2 = SESS ? s_ystate(A, cx)[1] : kLevels / 2;
  float wr[32];

  for (int64_t it = 0; it < A.N * cx.wc; ++it) {
    const Item I = item_of<PIPE>(it, cx.wc);
    const int64_t n = I.n;
    const int p = I.p;
    if (c == 0) sample_and_embed<TRACE, 0, PIPE>(P, cx, I, k, y1, y2, wembc, bemb);
#pragma unroll
    for (int jl = 0; jl < LP; ++jl) {
      if (jl < nl && jl >= xb) {
        if constexpr (LP == 3) {
          ptx::tmem_load_async<32>(tmb + 32 * jl, wr);
        } else {
#pragma unroll
          for (int q = 0; q < 32; q += 4) {  // W_res tile into registers before the wait
            const float4 t4 = lds4(wres + ((jl * 8 + q / 4) * 128 + b) * 4);
            wr[q] = t4.x; wr[q + 1] = t4.y; wr[q + 2] = t4.z; wr[q + 3] = t4.w;
          }
        }
        const float* hv;
        const float* xv;
        if (jl == 0) {  // inbound h_{j0-1}, x_{j0-1}
          wait(cx, b_xin<PIPE>(cx, I.s), I.par, 16);
          wait(cx, b_hin<PIPE>(cx, I.s), I.par, 17);
          hv = mb_hin<PIPE>(cx, I.s);
          xv = mb_xin<PIPE>(cx, I.s);
        } else {
          if (b == 0) stamp<TRACE>(trace_slot<TRACE>(A, n), 24 + jl - 1);  // B arrives for h_{j0+jl-1}
          ptx::bar_sync(kBarH, kMain);  // h_{j0+jl-1} from A
          hv = m.hs[p][jl - 1];
          xv = m.xs[p][jl - 1];
        }
        const float xi = xv[pad16(row)];
        if constexpr (LP == 3) ptx::tmem_wait_ld<32>(wr);
        float v[1];
        if constexpr ((DVW_DIAG & 4) != 0) v[0] = hv[voff] * wr[0];
        else if constexpr ((DVW_EXP & 2) != 0) tile_dot_half_n<1, 1>(wr, hv + voff, v);
        else tile_dot_half<1>(wr, hv + voff, v);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        const float xn = xi + (v[0] + bres[jl * R + row]);
        if (writer) {
          m.xs[p][jl][pad16(row)] = xn;
          if (jl + 1 == nl && !last_cta)
            ptx::st_async(remote(mb_xin<PIPE>(cx, I.s) + pad16(row), c + 1), xn, remote(b_xin<PIPE>(cx, I.s), c + 1));
        }
        if (jl + 1 < nl) bar_arrive(bar_xr(jl), kMain);  // x_{j0+jl} ready: C computes R_{j0+jl+1}
      }
    }
    // the sample's x are all in xs[p]: the aux warpgroup may read them
    // every warp of B arrives once its own rows of xs[p] are stored (4 arrivals complete the phase):
    // X reads all 64 rows for the queues
    __syncwarp();
    if (PIPE && b == 0) ptr(it, 13);
    if ((b & 31) == 0) {
      if (b == 0) trace<TRACE>(A, n, 2);
      ptx::mbar_arrive(ptx::smem_u32(&m.bar_done));
    }
  }
}

// ------------------------------------------------------------------ chain CTA, warpgroup C (R terms)
// R_{j0+jl} = W_cur_{j0+jl} x_{j0+jl-1} + c_{j0+jl} for jl >= xb: jl = 0 from the inbound x_{j0-1},
// jl >= 1 from x_{j0+jl-1} (B, or the embedding on CTA 0).
template <int LP, bool TRACE, bool SESS, bool PIPE>
__device__ void chain_C(const Params& P, const Ctx& cx, int c, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int ct = threadIdx.x - kAux - 256;  // 0..127
  const int k = threadIdx.x - kAux;         // sampler thread index (>= 256: waits only)
  const int hrow = ct >> 1, half = ct & 1;  // same mapping as A
  const bool writer = half == 0;
  const int voff = 40 * half;
  const int nl = pl.chain_nl[c];
  const int xb = (c == 0) ? 1 : 0;
  const uint32_t tm = tmem_lane_addr(m) + col_c(LP);
  const float* cf = sw + sm_fold(LP);  // [LPC][2R]
  const float* wembc = sw + sm_emb(LP);
  const float* bemb = wembc + kLevels * R;
  int y1 = SESS ? s_ystate(A, cx)[0] : kLevels / 2, y2 = SESS ? s_ystate(A, cx)[1] : kLevels / 2;
  float w[64];

  for (int64_t it = 0; it < A.N * cx.wc; ++it) {
    const Item I = item_of<PIPE>(it, cx.wc);
    const int64_t n = I.n;
    const int p = I.p;
    if (nl > xb) ptx::tmem_load_async<64>(tm + 64 * xb, w);
    if (c == 0) sample_and_embed<TRACE, 0, PIPE>(P, cx, I, k, y1, y2, wembc, bemb);
#pragma unroll
    for (int jl = 0; jl < LP; ++jl) {
      if (jl < nl && jl >= xb) {
        const float* xv;
        if (jl == 0) {
          if (wait(cx, b_xin<PIPE>(cx, I.s), I.par, 15) && ct == 0 && !cx.dead)
            ptx::mbar_arm(ptx::smem_u32(b_xin<PIPE>(cx, I.s)), R * 4);
          if (PIPE && ct == 0) ptr(it, 14);
          xv = mb_xin<PIPE>(cx, I.s);
        } else {
          if (jl - 1 >= xb) ptx::bar_sync(bar_xr(jl - 1), kMain);  // x_{j0+jl-1} from B
          xv = m.xs[p][jl - 1];
        }
        ptx::tmem_wait_ld<64>(w);
        float v[2];
        if constexpr ((DVW_DIAG & 2) != 0) { v[0] = xv[voff] * w[0]; v[1] = xv[voff + 1] * w[1]; }
        else if constexpr ((DVW_EXP & 2) != 0) tile_dot_half_n<2, 1>(w, xv + voff, v);
        else tile_dot_half<2>(w, xv + voff, v);
        if (jl + 1 < nl) ptx::tmem_load_async<64>(tm + 64 * (jl + 1), w);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        v[1] += __shfl_xor_sync(0xffffffffu, v[1], 1);
        if (writer) {
          m.rr[jl][hrow] = v[0] + cf[jl * 2 * R + hrow];
          m.rr[jl][R + hrow] = v[1] + cf[jl * 2 * R + R + hrow];
        }
        if (ct == 0) stamp<TRACE>(trace_slot<TRACE>(A, n), 21 + jl);
        // sync, not arrive: C's next matvec (R_{j+1}) then starts only once A is past this
        // layer's matvec, so it overlaps A's gate instead of competing with A's FMAs
        ptx::bar_sync(bar_ra(jl), kMain);
      }
    }
  }
}

// ------------------------------------------------------------------ chain CTA, warpgroup X (aux)
// Forward h of sample n-1 as A publishes it: layers l-1 and l-2 to the heads' slots 0 and 1,
// every other layer's to its skip CTA (16 x 16 B per
// destination; a DSMEM store holds its warp for about one hop, hence not on A).
template <bool PIPE>
__device__ __forceinline__ void aux_forward(const ClusterPlan& pl, const Ctx& cx, int first, int nl, int at, int p,
                                            int s) {
  Mail& m = *cx.mail;
  for (int jl = 0; jl < nl; ++jl) {
    const int j = first + jl;
    ptx::bar_sync(kBarHX + jl, kMain);
    if (j >= pl.L - 2) {
      const int sl = pl.L - 1 - j;
      if (at < 16 * NH) {
        const int hh = at >> 4, e = at & 15, off = 20 * (e >> 2) + 4 * (e & 3);
        ptx::st_async4(remote(mb_hbuf<PIPE>(cx, sl, s) + off, pl.nc + hh), lds4(&m.hs[p][jl][off]),
                       remote(b_h<PIPE>(cx, sl, s), pl.nc + hh));
      }
    } else if (at < 16 && pl.layer_skip_cta[j] >= 0) {
      const int off = 20 * (at >> 2) + 4 * (at & 3);
      const int kk = pl.layer_skip_cta[j], sl = pl.layer_skip_slot[j];
      ptx::st_async4(remote(mb_hbuf<PIPE>(cx, sl, s) + off, kk), lds4(&m.hs[p][jl][off]), remote(b_h<PIPE>(cx, sl, s), kk));
    }
  }
}

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// Chain-skip layers (those no skip CTA holds, j < nxs): this CTA's partial
// sum_j W_skip_j h_j of sample n-1, W_skip streamed from L2 ([16][S][4], rows at and
// at + 128), then sent to every head's partial slot.  Off the critical chain: these are the
// earliest layers, at least two chain CTAs before the heads need the sum.
template <int S, bool PIPE>
__device__ __forceinline__ void aux_chain_skip(const Params& P, const Ctx& cx, int c, int at, int pp, int s) {
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int first = pl.chain_first[c], nl = pl.chain_nl[c];
  constexpr int RR = S / 128;  // rows per thread
  float part[RR];
#pragma unroll
  for (int rr = 0; rr < RR; ++rr) part[rr] = 0.0f;
  for (int jl = 0; jl < nl; ++jl) {
    const int j = first + jl;
    if (j >= pl.nxs) break;
    if constexpr ((DVW_DIAG & 256) != 0) continue;
    const float* wsk = P.pk + pl.wskx_off + (int64_t)j * 16 * S * 4;
    const float* h = m.hs[pp][jl];
#pragma unroll
    for (int rr = 0; rr < RR; ++rr) {
      float4 wv[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) wv[q] = ldg4(wsk + ((int64_t)(rr * 16 + q) * 128 + at) * 4);
      float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float4 x = lds4(h + pad16(4 * q));
        s01 = ffma2(wv[q].x, wv[q].y, x.x, x.y, s01);
        s23 = ffma2(wv[q].z, wv[q].w, x.z, x.w, s23);
      }
      part[rr] += (s01.x + s01.y) + (s23.x + s23.y);
    }
  }
#pragma unroll
  for (int rr = 0; rr < RR; ++rr) m.zs[at + 128 * rr] = part[rr];
  ptx::bar_sync(kBarAux, kAux);
  const int slot = pl.xpart_slot[c];
#pragma unroll
  for (int i = at; i < (S / 4) * NH; i += kAux) {  // S / 4 float4 per head
    const int hh = i / (S / 4), e = i % (S / 4);
    ptx::st_async4(remote(mb_part<PIPE>(cx, slot, s) + 4 * e, pl.nc + hh), lds4(&m.zs[4 * e]),
                   remote(b_part<PIPE>(cx, s), pl.nc + hh));
  }
}

// For the coming sample n: queue write of x_j(n-1), queue read of x_j(n-d),
// pre = B + L_j(n/hop) + W_prev x_j(n-d)  (Fig. 2 aux threads),
// W_prev streamed from L2 ([16][128][4]; thread at = row of a).
template <int S, int LP, bool TRACE, bool SESS, bool PIPE>
__device__ void chain_aux(const Params& P, const Ctx& cx, int c, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int at = threadIdx.x;  // 0..127 = row of a (2r rows)
  const int first = pl.chain_first[c], nl = pl.chain_nl[c];
  const float* bj = sw + sm_b(LP);  // [LPC][2R]
  const int L = A.L;
  const bool xskip = LP == 4 && first < pl.nxs;  // LP = 3 plans never have chain-skip layers
  const int64_t nit = A.N * cx.wc;

  for (int64_t it = 0; it < nit; ++it) {
    const Item I = item_of<PIPE>(it, cx.wc);
    const int64_t n = I.n;
    const int sp = PIPE ? (int)((it + cx.wc - 1) % cx.wc) : 0;  // stream of the previous item
    const int64_t np = PIPE ? (it - 1) / cx.wc : n - 1;         // its sample
    // this item's stream (one cluster per stream unless PIPE)
    const float* condb = A.cond + (cx.sidx + I.s) * A.n_frames * L * 2 * R;
    float* ringb = A.ring + (cx.sidx + I.s) * A.ring_floats;
    float* ringp = A.ring + (cx.sidx + sp) * A.ring_floats;
    const int pp = (int)((it - 1) & 1);  // local buffer parity of the previous item
    if (it > 0) {
      aux_forward<PIPE>(pl, cx, first, nl, at, pp, sp);
      wait(cx, &m.bar_done, (uint32_t)pp, 14);
      if constexpr (LP == 4)
        if (xskip) aux_chain_skip<S, PIPE>(P, cx, c, at, pp, sp);
    }
    const int64_t ng = SESS ? A.n0 + n : n;  // global sample index (streaming sessions continue at n0)
    const int64_t f = ng / A.hop;
    for (int jl = 0; jl < nl; ++jl) {
      if constexpr ((DVW_DIAG & 8) != 0) { m.pre[jl][at] = 0.0f; continue; }
      const int j = first + jl;
      const int d = A.dil[j];
      float4 wv[16];
      if constexpr ((DVW_DIAG & 1) != 0) {
#pragma unroll
        for (int q = 0; q < 16; ++q) wv[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else if constexpr (LP == 3) {
        const float* wp = sw + jl * 16 * 128 * 4;  // shared memory
#pragma unroll
        for (int q = 0; q < 16; ++q) wv[q] = lds4(wp + (q * 128 + at) * 4);
      } else if (jl < pl.nwp[c]) {  // LP = 4: the first nwp layers' W_prev in shared memory
        const float* wp = sw + smem_chain(c, LP) + jl * 16 * 128 * 4;
#pragma unroll
        for (int q = 0; q < 16; ++q) wv[q] = lds4(wp + (q * 128 + at) * 4);
      } else {
        const float* wp = P.pk + pl.wprev_off + (int64_t)j * 16 * 128 * 4;  // L2
#pragma unroll
        for (int q = 0; q < 16; ++q) wv[q] = ldg4(wp + (q * 128 + at) * 4);
      }
      const float lv = __ldg(condb + (f * L + j) * 2 * R + at);
      if (at < R) {
        float* ring = ringb + A.ring_off[j];
        const float xc = m.xs[pp][jl][pad16(at)];  // x_j of the previous item (unused at it = 0)
        float xpv = 0.0f;
        if constexpr (PIPE) {
          // the previous item (another stream unless wc = 1) into its stream's queue, slot np mod d;
          // then this stream's x_j(n - d) from slot n mod d (written wc items or more ago)
          if (it > 0) ringp[A.ring_off[j] + (int64_t)(np % d) * R + at] = xc;
          if (n - d >= 0) xpv = ring[(int64_t)(n % d) * R + at];
        } else {
          // x_j(ng - d): slot (ng - d) mod d = ng mod d; at n = 0 of a continued session x_j(ng - 1)
          // was flushed to the queue by the previous call
          if (ng - d >= 0) xpv = (d == 1 && n > 0) ? xc : ring[(int64_t)(ng % d) * R + at];
          if (n > 0 && d >= 2) ring[(int64_t)((ng - 1) % d) * R + at] = xc;
        }
        m.xp[at] = xpv;
      }
      ptx::bar_sync(kBarAux, kAux);
      float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < ((DVW_DIAG & 1) ? 0 : 16); ++q) {
        const float4 x = lds4(&m.xp[4 * q]);
        a01 = ffma2(wv[q].x, wv[q].y, x.x, x.y, a01);
        a23 = ffma2(wv[q].z, wv[q].w, x.z, x.w, a23);
      }
      m.pre[jl][at] = (bj[jl * 2 * R + at] + lv) + ((a01.x + a01.y) + (a23.x + a23.y));
      ptx::bar_sync(kBarAux, kAux);
    }
    if (at == 0) {
      trace<TRACE>(A, n, 5);
      ptx::mbar_arrive(ptx::smem_u32(&m.bar_pre));
    }
  }
  if (A.N > 0) {  // the last item's h and chain-skip partial
    const int pp = (int)((nit - 1) & 1);
    const int sl = PIPE ? cx.wc - 1 : 0;
    float* ringb = A.ring + cx.sidx * A.ring_floats;
    aux_forward<PIPE>(pl, cx, first, nl, at, pp, sl);
    if (xskip || SESS) wait(cx, &m.bar_done, (uint32_t)pp, 14);
    if constexpr (LP == 4) {
      if (xskip) aux_chain_skip<S, PIPE>(P, cx, c, at, pp, sl);
    }
    if (SESS && at < R) {  // streaming session: x_j of the last sample into its queue slot
      const int64_t ng = A.n0 + A.N - 1;
      for (int jl = 0; jl < nl; ++jl) {
        const int d = A.dil[first + jl];
        ringb[A.ring_off[first + jl] + (int64_t)(ng % d) * R + at] = m.xs[pp][jl][pad16(at)];
      }
    }
  }
}

// Multi-stream variant of the aux warpgroup.  Item i = (stream s, sample n).  X computes the pre terms
// of the next kPB items at once (P.xpb, capped at wc - 1) while A and B work on item i: one W_prev
// pass (L2 at LP = 4) and one memory latency (conditioning, queue entries) per batch instead of per
// item.  X retires item i (forwards its h, writes its x into its stream's queues), then releases item
// i + 1 to A -- so A can never run two items ahead of X's forwarding (the named barriers kBarHX + jl
// are shared by consecutive items).  The queue entries x_j(n - d) of items i + 1 .. i + kPB belong to
// items <= i + kPB - wc d <= i - 1 (kPB <= wc - 1), already retired; a cluster with one stream (a
// ragged last cluster) writes item i's queues before computing pre for i + 1.  At LP = 4 the
// chain-skip partials (layers < nxs, W_skip from L2) are computed for P.xsb items at a time.
template <int S, int LP>
__device__ void chain_aux_pipe(const Params& P, const Ctx& cx, int c, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int at = threadIdx.x;  // 0..127 = row of a (2r rows)
  const int first = pl.chain_first[c], nl = pl.chain_nl[c];
  const float* bj = sw + sm_b(LP);  // [LPC][2R]
  const int L = A.L;
  const bool xskip = LP == 4 && first < pl.nxs;
  const int64_t nit = A.N * cx.wc;
  const bool early = cx.wc >= 2;
  const int pb = early ? max(1, min(P.xpb, cx.wc - 1)) : 1;
  // a chain-skip batch holds items of distinct streams (xsb <= wc): the partial of item i waits
  // for item i + xsb - 1, which must not be a later sample of i's own stream
  const int xsb = max(1, min(min(P.xsb, kXH), cx.wc));
  // LP = 4: weight stream.  A job is a list of nch 16-KB chunks (src(i)); chunk g of the CTA's
  // running count uses buffer g mod nb (phase (g / nb) & 1).  Thread 0 keeps nb copies in flight;
  // after body(i, buffer) every X thread passes kBarAux, so the buffer is free for chunk i + nb.
  const int nb = pl.xnb[c];
  uint32_t wg = 0;
  auto stream_job = [&](int nch, auto&& src, auto&& body) {
    auto issue = [&](int i) {
      const int sl = (int)((wg + i) % nb);
      const uint32_t bar = ptx::smem_u32(&m.wfull[sl]);
      ptx::mbar_arm(bar, kWChunk * 4);
      bulk_g2s(ptx::smem_u32(cx.mb + kMbChainEnd4 + sl * kWChunk), src(i), kWChunk * 4, bar);
    };
    constexpr bool kCopy = (DVW_DIAG & 1024) == 0, kBody = (DVW_DIAG & 512) == 0;  // timing diagnostics
    if (at == 0 && kCopy)
      for (int i = 0; i < min(nb, nch); ++i) issue(i);
    for (int i = 0; i < nch; ++i) {
      const int sl = (int)((wg + i) % nb);
      if (kCopy) wait(cx, &m.wfull[sl], ((wg + i) / nb) & 1, 19);
      if (kBody) body(i, (const float*)(cx.mb + kMbChainEnd4 + sl * kWChunk));
      ptx::bar_sync(kBarAux, kAux);
      if (at == 0 && i + nb < nch && kCopy) issue(i + nb);
    }
    wg += nch;
  };

  // pre of items [i0, i0 + cnt) (cnt <= kPB) into their ring slots; ordered before the releases by
  // the caller's next kBarAux barrier
  auto make_pre = [&](int64_t i0, int cnt) {
    if constexpr ((DVW_DIAG & 8) != 0) {  // timing diagnostic: no queue / conditioning / W_prev work
      for (int k = 0; k < cnt; ++k)
        for (int jl = 0; jl < nl; ++jl) mb_pre(cx, (int)((i0 + k) % kPR))[jl * 2 * R + at] = 0.0f;
      return;
    }
    // every item's conditioning and queue entries in flight at once (all loads issued before the
    // first store): B + L into the item's slot, x_j(n - d) into the staging rows
    float lv[kPB][LPC], xv[kPB][LPC];
#pragma unroll
    for (int k = 0; k < kPB; ++k) {
      const Item I = item_of<true>(i0 + k, cx.wc);
      const float* condb = A.cond + ((cx.sidx + I.s) * A.n_frames + (uint32_t)I.n / (uint32_t)A.hop) * L * 2 * R;
      const float* ringb = A.ring + (cx.sidx + I.s) * A.ring_floats;
#pragma unroll
      for (int jl = 0; jl < LPC; ++jl) {
        lv[k][jl] = xv[k][jl] = 0.0f;
        if (k < cnt && jl < nl) {
          const int j = first + jl;
          const int d = A.dil[j];
          lv[k][jl] = __ldg(condb + j * 2 * R + at);
          if (at < R && I.n - d >= 0) xv[k][jl] = ringb[A.ring_off[j] + ((uint32_t)I.n % (uint32_t)d) * R + at];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kPB; ++k) {
      float* ps = mb_pre(cx, (int)((i0 + k) % kPR));
      float* xs = mb_xst(cx, k);
#pragma unroll
      for (int jl = 0; jl < LPC; ++jl) {
        if (k < cnt && jl < nl) {
          ps[jl * 2 * R + at] = bj[jl * 2 * R + at] + lv[k][jl];
          if (at < R) xs[jl * R + at] = xv[k][jl];
        }
      }
    }
    ptx::bar_sync(kBarAux, kAux);
    // pre += W_prev x_j(n - d): each W_prev row loaded once per batch; k innermost:
    // one weight float4 is live at a time, not every item's x rows
    if constexpr (LP == 3 || !kXStream) {
#pragma unroll
      for (int jl = 0; jl < LPC; ++jl) {
        if (jl >= nl) break;
        float4 wv[16];
        if constexpr (LP == 3) {
          const float* wp = sw + jl * 16 * 128 * 4;
#pragma unroll
          for (int q = 0; q < 16; ++q) wv[q] = lds4(wp + (q * 128 + at) * 4);
        } else if (jl < pl.nwp[c]) {  // LP = 4: resident in shared memory
          const float* wp = sw + smem_chain(c, LP) + jl * 16 * 128 * 4;
#pragma unroll
          for (int q = 0; q < 16; ++q) wv[q] = lds4(wp + (q * 128 + at) * 4);
        } else {  // LP = 4: from L2, the row's 16 float4 in flight at once
          const float* wp = P.pk + pl.wprev_off + (int64_t)(first + jl) * 16 * 128 * 4;
#pragma unroll
          for (int q = 0; q < 16; ++q) wv[q] = ldg4(wp + (q * 128 + at) * 4);
        }
        float2 a01[kPB], a23[kPB];
#pragma unroll
        for (int k = 0; k < kPB; ++k) a01[k] = a23[k] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
#pragma unroll
          for (int k = 0; k < kPB; ++k) {
            if (k < cnt) {
              const float4 x = lds4(mb_xst(cx, k) + jl * R + 4 * q);
              a01[k] = ffma2(wv[q].x, wv[q].y, x.x, x.y, a01[k]);
              a23[k] = ffma2(wv[q].z, wv[q].w, x.z, x.w, a23[k]);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < kPB; ++k) {
          if (k < cnt) {
            float* ps = mb_pre(cx, (int)((i0 + k) % kPR)) + jl * 2 * R + at;
            *ps = *ps + ((a01[k].x + a01[k].y) + (a23[k].x + a23[k].y));
          }
        }
      }
    } else {
      // W_prev_j streamed through the weight ring: chunk 2 jl + hq = column quads [8 hq, 8 hq + 8)
      float2 a01[kPB], a23[kPB];
      stream_job(
          2 * nl, [&](int i) { return P.pk + pl.wprev_off + (int64_t)(first + i / 2) * 16 * 128 * 4 + (i & 1) * kWChunk; },
          [&](int i, const float* wb) {
            const int jl = i >> 1;
            if ((i & 1) == 0) {
#pragma unroll
              for (int k = 0; k < kPB; ++k) a01[k] = a23[k] = make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 wq = lds4(wb + (q * 128 + at) * 4);
              const int qq = 8 * (i & 1) + q;
#pragma unroll
              for (int k = 0; k < kPB; ++k) {
                if (k < cnt) {
                  const float4 x = lds4(mb_xst(cx, k) + jl * R + 4 * qq);
                  a01[k] = ffma2(wq.x, wq.y, x.x, x.y, a01[k]);
                  a23[k] = ffma2(wq.z, wq.w, x.z, x.w, a23[k]);
                }
              }
            }
            if ((i & 1) == 1) {
#pragma unroll
              for (int k = 0; k < kPB; ++k) {
                if (k < cnt) {
                  float* ps = mb_pre(cx, (int)((i0 + k) % kPR)) + jl * 2 * R + at;
                  *ps = *ps + ((a01[k].x + a01[k].y) + (a23[k].x + a23[k].y));
                }
              }
            }
          });
    }
  };
  auto release = [&](int64_t it) {
    if (at == 0 && it < nit) ptx::mbar_arrive(ptx::smem_u32(&m.bar_pre2[it % kPR]));
  };
  // chain-skip partials sum_{j < nxs} W_skip_j h_j of the last `cnt` retired items
  // (their h in the history slots), W_skip rows streamed from L2 once per batch, then sent to every
  // head's partial slot of each item's stream
  auto chain_skip = [&](int64_t ilast, int cnt) {
    constexpr int RR = S / 128;  // rows per thread
    float part[kXH][RR];
#pragma unroll
    for (int k = 0; k < kXH; ++k)
#pragma unroll
      for (int rr = 0; rr < RR; ++rr) part[k][rr] = 0.0f;
    if constexpr (!kXStream) {
      // W_skip_j row block rr ([nxs][RR][16][128][4]) from L2, the thread's 16 float4 in flight at
      // once, applied to every item of the batch; partials accumulate layer by layer (oracle order).
      // Row blocks outermost: one block's item partials live at a time (register pressure)
#pragma unroll
      for (int rr = 0; rr < RR; ++rr) {
        float pr[kXH];
#pragma unroll
        for (int k = 0; k < kXH; ++k) pr[k] = 0.0f;
        for (int jl = 0; jl < nl; ++jl) {
          const int j = first + jl;
          if (j >= pl.nxs) break;
          if constexpr ((DVW_DIAG & 256) != 0) continue;
          const float* wsk = P.pk + pl.wskx_off + ((int64_t)j * RR + rr) * 16 * 128 * 4;
          float2 s01[kXH], s23[kXH];
#pragma unroll
          for (int k = 0; k < kXH; ++k) s01[k] = s23[k] = make_float2(0.f, 0.f);
          // the row in two halves of 8 float4 (register pressure; same accumulation order)
#pragma unroll
          for (int hq = 0; hq < 2; ++hq) {
            float4 wv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) wv[q] = ldg4(wsk + ((8 * hq + q) * 128 + at) * 4);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
#pragma unroll
              for (int k = 0; k < kXH; ++k) {
                if (k < cnt) {
                  const float4 x = lds4(mb_hist(cx, (int)((ilast - k) % kXH)) + jl * kHLen + pad16(4 * (8 * hq + q)));
                  s01[k] = ffma2(wv[q].x, wv[q].y, x.x, x.y, s01[k]);
                  s23[k] = ffma2(wv[q].z, wv[q].w, x.z, x.w, s23[k]);
                }
              }
            }
          }
#pragma unroll
          for (int k = 0; k < kXH; ++k)
            if (k < cnt) pr[k] += (s01[k].x + s01[k].y) + (s23[k].x + s23[k].y);
        }
#pragma unroll
        for (int k = 0; k < kXH; ++k) part[k][rr] = pr[k];
      }
    } else {
    // W_skip_j row block rr ([nxs][RR][16][128][4]) in chunks of 8 column quads: chunk
    // (jl RR + rr) 2 + hq; every item's partial accumulates layer by layer in the oracle's order
    const int nsk = (DVW_DIAG & 256) ? 0 : max(0, min(nl, pl.nxs - first));
    float2 s01[kXH], s23[kXH];
    stream_job(
        2 * RR * nsk, [&](int i) { return P.pk + pl.wskx_off + (int64_t)(first * RR + i / 2) * 16 * 128 * 4 + (i & 1) * kWChunk; },
        [&](int i, const float* wb) {
          const int jl = i / (2 * RR), rr = (i / 2) % RR;
          if ((i & 1) == 0) {
#pragma unroll
            for (int k = 0; k < kXH; ++k) s01[k] = s23[k] = make_float2(0.f, 0.f);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 wq = lds4(wb + (q * 128 + at) * 4);
            const int qq = 8 * (i & 1) + q;
#pragma unroll
            for (int k = 0; k < kXH; ++k) {
              if (k < cnt) {
                const float4 x = lds4(mb_hist(cx, (int)((ilast - k) % kXH)) + jl * kHLen + pad16(4 * qq));
                s01[k] = ffma2(wq.x, wq.y, x.x, x.y, s01[k]);
                s23[k] = ffma2(wq.z, wq.w, x.z, x.w, s23[k]);
              }
            }
          }
          if ((i & 1) == 1) {
#pragma unroll
            for (int k = 0; k < kXH; ++k)
              if (k < cnt) {
#pragma unroll
                for (int r2 = 0; r2 < RR; ++r2)
                  if (r2 == rr) part[k][r2] += (s01[k].x + s01[k].y) + (s23[k].x + s23[k].y);
              }
          }
        });
    }
#pragma unroll
    for (int k = 0; k < kXH; ++k)
      if (k < cnt)
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) mb_xstage(cx, k)[at + 128 * rr] = part[k][rr];
    ptx::bar_sync(kBarAux, kAux);
    const int slot = pl.xpart_slot[c];
    for (int k = cnt - 1; k >= 0; --k) {  // oldest item first
      const int s = item_of<true>(ilast - k, cx.wc).s;
      const float* st = mb_xstage(cx, k);
#pragma unroll
      for (int i = at; i < (S / 4) * NH; i += kAux) {  // S / 4 float4 per head
        const int hh = i / (S / 4), e = i % (S / 4);
        ptx::st_async4(remote(mb_part<true>(cx, slot, s) + 4 * e, pl.nc + hh), lds4(st + 4 * e),
                       remote(b_part<true>(cx, s), pl.nc + hh));
      }
    }
  };
  // item `it` published by A and finished by B: forward its h layer by layer, then its x into its
  // stream's queues; release item it + 1 to A when `rel`
  // forward layer jl's h of item I to its skip CTA or (last two layers) the heads.  Consecutive
  // layers' hand-offs from different warps: an st.async holds its warp for about one hop, so the
  // sends of layers jl and jl + 1 overlap instead of queueing on one warp
  auto forward = [&](const Item& I, int jl) {
    const int j = first + jl;
    if (j >= pl.L - 2) {
      const int sl = pl.L - 1 - j;
      const int ht = at - 64 * (jl & 1);
      if (ht >= 0 && ht < 16 * NH) {
        const int hh = ht >> 4, e = ht & 15, off = 20 * (e >> 2) + 4 * (e & 3);
        ptx::st_async4(remote(mb_hbuf<true>(cx, sl, I.s) + off, pl.nc + hh), lds4(&m.hs[I.p][jl][off]),
                       remote(b_h<true>(cx, sl, I.s), pl.nc + hh));
      }
    } else if ((at >> 5) == (jl & 3) && (at & 31) < 16 && pl.layer_skip_cta[j] >= 0) {
      const int st = at & 31, off = 20 * (st >> 2) + 4 * (st & 3);
      const int kk = pl.layer_skip_cta[j], sl = pl.layer_skip_slot[j];
      ptx::st_async4(remote(mb_hbuf<true>(cx, sl, I.s) + off, kk), lds4(&m.hs[I.p][jl][off]),
                     remote(b_h<true>(cx, sl, I.s), kk));
    }
  };
  // item `it` published by A and finished by B: forward its h layer by layer, its x into its
  // stream's queues.  With `rel`, item it + 1 is released to A as soon as X holds everything it
  // still needs from item it's buffers (its x rows in registers, its h in the history ring):
  // the last layer's forward and the queue stores follow the release.  A overwrites hs[p] / B
  // xs[p] (p = it's parity) only for item it + 2, released after retire(it + 1).
  auto retire = [&](int64_t it, bool rel) {
    const Item I = item_of<true>(it, cx.wc);
    if (at == 0) ptr(it, 8);
    for (int jl = 0; jl < nl; ++jl) {
      ptx::bar_sync(kBarHX + jl, kMain);
      if (jl + 1 < nl || !rel) forward(I, jl);
    }
    if (at == 0) ptr(it, 9);
    wait(cx, &m.bar_done, (uint32_t)I.p, 14);
    if (at == 0) ptr(it, 10);
    if constexpr (LP == 4) {
      if (xskip) {  // h of the item for its chain-skip batch (hs[p] is reused two items later)
        float* hh = mb_hist(cx, (int)(it % kXH));
        for (int i = at; i < nl * kHLen; i += kAux) hh[i] = m.hs[I.p][i / kHLen][i % kHLen];
      }
    }
    float xq[LPC];
#pragma unroll
    for (int jl = 0; jl < LPC; ++jl) xq[jl] = (at < R && jl < nl) ? m.xs[I.p][jl][pad16(at)] : 0.0f;
    ptx::bar_sync(kBarAux, kAux);
    if (rel) {
      release(it + 1);
      if (at == 0) ptr(it, 11);
      forward(I, nl - 1);
    }
    if (at < R) {
      float* ringb = A.ring + (cx.sidx + I.s) * A.ring_floats;
#pragma unroll
      for (int jl = 0; jl < LPC; ++jl) {
        if (jl < nl) {
          const int d = A.dil[first + jl];
          ringb[A.ring_off[first + jl] + ((uint32_t)I.n % (uint32_t)d) * R + at] = xq[jl];
        }
      }
    }
  };
  if (nit == 0) return;
  // chain-skip batch ending at item `it` (after its retirement; the history slots are X-private)
  auto skip_batch = [&](int64_t it) {
    if constexpr (LP == 4) {
      if (xskip) {
        const int k = (int)(it % xsb);
        if (k == xsb - 1 || it == nit - 1) chain_skip(it, k + 1);
      }
    }
  };
  if (early) {
    // Item i + 1 is released as soon as item i is retired (its h forwarded, its x in the queues);
    // X then computes the next pre batch and the chain-skip batch while A and B run item i + 1.
    // Items 0 .. min(kPB, wc) - 1 are sample 0 of their streams (no queue entries yet); later
    // batches [it + 2, it + 2 + pb) are computed after retiring item it, and item it + 1 + k needs
    // items <= it + 1 + k - wc <= it retired (k <= pb <= wc - 1).  Pre slots in use: it + 1 (A) and
    // the batch, pb + 1 <= kPR (item it's slot is free once it is retired).
    int64_t nx = min((int64_t)min(kPB, cx.wc), nit);
    make_pre(0, (int)nx);
    ptx::bar_sync(kBarAux, kAux);
    release(0);
    for (int64_t it = 0; it < nit; ++it) {
      retire(it, true);
      if (nx == it + 2 && nx < nit) {
        const int cnt = (int)min((int64_t)pb, nit - nx);
        make_pre(nx, cnt);
        nx += cnt;
        if (at == 0) ptr(it, 12);
      }
      skip_batch(it);
    }
  } else {
    // one stream: item it + 1 = sample n + 1 needs item it's x in the queues (d = 1)
    make_pre(0, 1);
    ptx::bar_sync(kBarAux, kAux);
    release(0);
    for (int64_t it = 0; it < nit; ++it) {
      retire(it, false);
      skip_batch(it);
      if (it + 1 < nit) {
        make_pre(it + 1, 1);
        ptx::bar_sync(kBarAux, kAux);
        release(it + 1);
      }
    }
  }
}

// ------------------------------------------------------------------ head CTA (rows [64h, 64h+64))
// Thread k (0..255):
//   q   : rows {g + 64 m} (m < S/64), columns [16 cc, +16) of W_skip^(l); g = k/4, cc = k%4
//   z_a : rows 64h + 4 (k/16) + m (m < 4), columns [(k%16) S/16, +S/16) of W_relu
//   out : rows 64h + 4 (k/16) + m (m < 4), columns [16 (k%16), +16) of W_out
template <int S, bool TRACE, bool PIPE>
__device__ void head_main(const Params& P, const Ctx& cx, int hidx, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int k = threadIdx.x - kAux;  // 0..255
  constexpr int RQ = S / 64;         // q rows per thread
  constexpr int CZ = S / 16;         // z_s columns per thread
  // TMEM tiles (this thread's lane): W_skip^(l) [RQ*16], W_relu [4*CZ], W_out [64]
  const uint32_t tm = tmem_lane_addr(m) + (k < 128 ? 0 : 256);
  constexpr int cRelu = RQ * 16, cOut = RQ * 16 + 4 * CZ, cSk2 = RQ * 16 + 4 * CZ + 64;
  const float* bskip = sw;          // [S]
  const float* brelu = sw + S;      // [64]
  const float* bout = sw + S + 64;  // [64]
  const bool has2 = pl.L >= 2;
  const int g = k >> 2, cc = k & 3;
  const int qrow = g + 64 * ((RQ == 4) ? cc : (cc >> 1));  // q row this lane finishes
  const bool qwriter = (RQ == 4) || ((cc & 1) == 0);
  const int c16 = k & 15;
  const int orow = 4 * (k >> 4) + ((k >> 2) & 3);  // z_a / logits row (within the head) this lane finishes
  const bool owriter = (k & 3) == 0;
  const int np = pl.npart;
  float w[64];

  auto finish = [&](float (&v)[RQ]) -> float {
    xpose_level<RQ>(v, cc, 2);
    if constexpr (RQ == 4) {
      xpose_level<2>(*reinterpret_cast<float(*)[2]>(v), cc, 1);
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    }
    return v[0];
  };

  for (int64_t it = 0; it < A.N * cx.wc; ++it) {
    const Item I = item_of<PIPE>(it, cx.wc);
    const int64_t n = I.n;
    const uint32_t par = I.par;
    const float* hb0 = mb_hbuf<PIPE>(cx, 0, I.s);
    const float* hb1 = mb_hbuf<PIPE>(cx, 1, I.s);
    const float* zin = mb_za<PIPE>(cx, I.s);
    // q = B_skip + sum_k partial_k + W_skip^(l-1) h^(l-1) + W_skip^(l) h^(l); z_s = relu(q)
    // (PAPER.md:365-372).  W_skip^(l-1) is applied here, from tensor memory, while the last
    // layer runs, so no skip CTA sits between the chain and the head (and the head's shared
    // memory stays free for the inbound DSMEM traffic).
    float d2 = 0.0f;
    if (has2) {
      ptx::tmem_load_async<RQ * 16>(tm + cSk2, w);  // W_skip^(l-1) tile
      if (wait(cx, b_h<PIPE>(cx, 1, I.s), par, 24) && k == 0 && !cx.dead)
        ptx::mbar_arm(ptx::smem_u32(b_h<PIPE>(cx, 1, I.s)), R * 4);
      if (PIPE && k == 0) ptr(it, 0);
      if (k == 0) trace<TRACE>(A, n, 4);
      ptx::tmem_wait_ld<RQ * 16>(w);
      float v2[RQ];
      if constexpr ((DVW_DIAG & 64) != 0) { for (int r = 0; r < RQ; ++r) v2[r] = w[r] * hb1[20 * cc]; } else tile_dot<RQ, 16>(w, hb1 + 20 * cc, v2);
      d2 = finish(v2);
      if (k == 0) trace<TRACE>(A, n, 6);
    }
    ptx::tmem_load_async<RQ * 16>(tm, w);  // W_skip^(l) tile, hidden behind the wait
    if (wait(cx, b_h<PIPE>(cx, 0, I.s), par, 21) && k == 0 && !cx.dead)
      ptx::mbar_arm(ptx::smem_u32(b_h<PIPE>(cx, 0, I.s)), R * 4);
    if (PIPE && k == 0) ptr(it, 1);
    if (k == 0) trace<TRACE>(A, n, 0);
    ptx::tmem_wait_ld<RQ * 16>(w);
    float v[RQ];
    if constexpr ((DVW_DIAG & 64) != 0) { for (int r = 0; r < RQ; ++r) v[r] = w[r] * hb0[20 * cc]; } else tile_dot<RQ, 16>(w, hb0 + 20 * cc, v);
    ptx::tmem_load_async<4 * CZ>(tm + cRelu, w);
    v[0] = finish(v);
    if (np > 0) {
      if (wait(cx, b_part<PIPE>(cx, I.s), par, 22) && k == 0 && !cx.dead)
        ptx::mbar_arm(ptx::smem_u32(b_part<PIPE>(cx, I.s)), np * S * 4);
    }
    if (PIPE && k == 0) ptr(it, 2);
    if (k == 0) trace<TRACE>(A, n, 1);
    if (qwriter) {
      float qv = bskip[qrow];
      for (int kk = 0; kk < np; ++kk) qv += mb_part<PIPE>(cx, kk, I.s)[qrow];
      qv += d2;
      qv += v[0];
      m.zs[cpad<CZ>(qrow)] = fmaxf(qv, 0.0f);
    }
    ptx::bar_sync(kBarHS, kMain);
    if (k == 0) trace<TRACE>(A, n, 7);
    // z_a = relu(W_relu z_s + B_relu)
    ptx::tmem_wait_ld<4 * CZ>(w);
    float za[4];
    if constexpr ((DVW_DIAG & 64) != 0) { for (int r = 0; r < 4; ++r) za[r] = w[r] * m.zs[(CZ + 4) * c16]; } else tile_dot<4, CZ>(w, &m.zs[(CZ + 4) * c16], za);
    ptx::tmem_load_async<64>(tm + cOut, w);
    xpose_level<4>(za, k, 8);
    xpose_level<2>(*reinterpret_cast<float(*)[2]>(za), k, 4);
    za[0] += __shfl_xor_sync(0xffffffffu, za[0], 2);
    za[0] += __shfl_xor_sync(0xffffffffu, za[0], 1);
    const float zav = fmaxf(za[0] + brelu[orow], 0.0f);
    {  // all four lanes of a quad hold z_a[orow]: lane k%4 sends it to head k%4 (one st.async
       // per lane -- a st.async holds its warp for about one hop, so never several in a row)
      const int dst = pad16(64 * hidx + orow);
      ptx::st_async(remote(mb_za<PIPE>(cx, I.s) + dst, pl.nc + (k & 3)), zav, remote(b_za<PIPE>(cx, I.s), pl.nc + (k & 3)));
    }
    if (k == 0) trace<TRACE>(A, n, 9);
    if (wait(cx, b_za<PIPE>(cx, I.s), par, 23) && k == 0 && !cx.dead)
      ptx::mbar_arm(ptx::smem_u32(b_za<PIPE>(cx, I.s)), kLevels * 4);
    if (PIPE && k == 0) ptr(it, 4);
    if (k == 0) trace<TRACE>(A, n, 2);
    // logits = W_out z_a + B_out
    ptx::tmem_wait_ld<64>(w);
    float lg[4];
    if constexpr ((DVW_DIAG & 64) != 0) { for (int r = 0; r < 4; ++r) lg[r] = w[r] * zin[20 * c16]; } else tile_dot<4, 16>(w, zin + 20 * c16, lg);
    xpose_level<4>(lg, k, 8);
    xpose_level<2>(*reinterpret_cast<float(*)[2]>(lg), k, 4);
    lg[0] += __shfl_xor_sync(0xffffffffu, lg[0], 2);
    lg[0] += __shfl_xor_sync(0xffffffffu, lg[0], 1);
    bool drop = false;  // watchdog test hook (TRACE instantiation only; DVW_FAULT_INJECT=1)
    if constexpr (TRACE) drop = A.fault == 1 && n == A.trace_n0;
    if (owriter && !drop)
      ptx::st_async(remote(mb_logits<PIPE>(cx, I.s) + 64 * hidx + orow, 0), lg[0] + bout[orow],
                    remote(b_logits<PIPE>(cx, I.s), 0));
    if (k == 0) trace<TRACE>(A, n, 3);
    if (PIPE && k == 0) ptr(it, 5);
  }
}

// ------------------------------------------------------------------ skip CTA
// partial_k = sum over owned layers j (ascending) of W_skip^(j) h^(j).
// Thread t: rows {g + 64 m} (m < S/64), columns [16 cc, +16); g = t/4, cc = t%4.
template <int S, bool TRACE, bool PIPE>
__device__ void skip_main(const Params& P, const Ctx& cx, int k, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int t = threadIdx.x - kAux;     // 0..255
  constexpr int RQ = S / 64;
  constexpr int QS = RQ * 16;           // floats of one layer's tile per thread
  constexpr int LSTRIDE = QS * kMain;   // floats per shared-memory layer ([q/4][t][4])
  const int nown = pl.skip_n[k], nsm = pl.skip_nsm[k];
  const uint32_t tm = tmem_lane_addr(m) + (t < 128 ? 0 : 256);  // TMEM layers: [QS] each
  const int g = t >> 2, cc = t & 3;
  const int row = g + 64 * ((RQ == 4) ? cc : (cc >> 1));
  const bool writer = (RQ == 4) || ((cc & 1) == 0);
  float wl[QS];

  auto finish = [&](float (&v)[RQ]) -> float {
    xpose_level<RQ>(v, cc, 2);
    if constexpr (RQ == 4) {
      xpose_level<2>(*reinterpret_cast<float(*)[2]>(v), cc, 1);
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    }
    return v[0];
  };

  for (int64_t it = 0; it < A.N * cx.wc; ++it) {
    const Item I = item_of<PIPE>(it, cx.wc);
    const int64_t n = I.n;
    const uint32_t par = I.par;
    float part = 0.0f;
#pragma unroll 1
    for (int sl = 0; sl < nown; ++sl) {
      const bool in_tmem = sl >= nsm;
      if (in_tmem) ptx::tmem_load_async<QS>(tm + (sl - nsm) * QS, wl);
      if (wait(cx, b_h<PIPE>(cx, sl, I.s), par, 31) && t == 0 && !cx.dead)
        ptx::mbar_arm(ptx::smem_u32(b_h<PIPE>(cx, sl, I.s)), R * 4);
      if (PIPE && t == 0 && (sl == 0 || sl == nown - 1)) ptr(it, sl == 0 ? 0 : 1);
      if (in_tmem) {
        ptx::tmem_wait_ld<QS>(wl);
      } else {
        const float* ws = sw + sl * LSTRIDE;
#pragma unroll
        for (int q = 0; q < QS; q += 4) {
          const float4 x = lds4(ws + (q / 4 * kMain + t) * 4);
          wl[q] = x.x; wl[q + 1] = x.y; wl[q + 2] = x.z; wl[q + 3] = x.w;
        }
      }
      float v[RQ];
      if constexpr ((DVW_DIAG & 32) != 0) {
#pragma unroll
        for (int r = 0; r < RQ; ++r) v[r] = wl[r] * mb_hbuf<PIPE>(cx, sl, I.s)[20 * cc];
      } else {
        tile_dot<RQ, 16>(wl, mb_hbuf<PIPE>(cx, sl, I.s) + 20 * cc, v);
      }
      part += finish(v);
    }
    // staged by sample parity (a skip CTA's own part[] is otherwise unused): the next sample's
    // writes can never meet this sample's reads (compute-sanitizer racecheck), with no second barrier
    float* stage = m.part[I.p];
    if (writer) stage[row] = part;
    if (t == 0) trace<TRACE>(A, n, 1);
    ptx::bar_sync(kBarHS, kMain);
    if (t < (S / 4) * NH) {
      const int hh = t / (S / 4), e = t % (S / 4);
      ptx::st_async4(remote(mb_part<PIPE>(cx, k, I.s) + 4 * e, pl.nc + hh), lds4(&stage[4 * e]),
                     remote(b_part<PIPE>(cx, I.s), pl.nc + hh));
    }
    if (PIPE && t == 0) ptr(it, 2);
  }
}

template <int S, int LP, bool TRACE, int NL = 0, bool SESS = false, bool PIPE = false>
__global__ void __launch_bounds__(kThreads, 1) k_cluster(const __grid_constant__ Params P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Mail* mail = reinterpret_cast<Mail*>(smem_raw);
  const ClusterPlan& pl = P.p;
  const int rank = (int)ptx::cluster_rank();
  const int t = threadIdx.x;
  constexpr size_t kMailBytes = (sizeof(Mail) + 127) & ~size_t(127);
  // PIPE: [Mail][this role's mailbox region][weights image]; otherwise [Mail][weights image]
  float* sw = reinterpret_cast<float*>(smem_raw + (PIPE ? (size_t)pl.sw_off_pipe[rank] : kMailBytes));
  const int64_t sidx = (int64_t)(blockIdx.x / pl.size) * (PIPE ? P.wmax : 1);
  const int wc = PIPE ? (int)min((int64_t)P.wmax, (int64_t)P.a.n_streams - sidx) : 1;
  Ctx cx{mail, P.a.err, pl.size, sidx, false, reinterpret_cast<float*>(smem_raw + kMailBytes), wc};

  int role = kIdle, idx = 0;
  if (rank < pl.nc) { role = kChain; idx = rank; }
  else if (rank < pl.nc + NH) { role = kHead; idx = rank - pl.nc; }
  else if (rank < pl.nc + NH + pl.nk) { role = kSkip; idx = rank - pl.nc - NH; }

  if (t < 32) ptx::tmem_alloc(ptx::smem_u32(&mail->tmem_base), kTmemCols);
  if (t == 0) {
    mail->abort_flag = 0;
    ptx::mbar_init(ptx::smem_u32(&mail->bar_hin), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_xin), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_logits), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_pre), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_done), 4);  // one arrival per warp of B
    ptx::mbar_init(ptx::smem_u32(&mail->bar_part), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_za), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_exit), 1);
    for (int i = 0; i < kCMaxSlot; ++i) ptx::mbar_init(ptx::smem_u32(&mail->bar_h[i]), 1);
    ptx::fence_mbar_init();
    // arm phase 0 of every transaction barrier a role receives on
    ptx::mbar_arm(ptx::smem_u32(&mail->bar_hin), R * 4);
    ptx::mbar_arm(ptx::smem_u32(&mail->bar_xin), R * 4);
    ptx::mbar_arm(ptx::smem_u32(&mail->bar_logits), kLevels * 4);
    ptx::mbar_arm(ptx::smem_u32(&mail->bar_part), pl.npart * S * 4);
    ptx::mbar_arm(ptx::smem_u32(&mail->bar_za), kLevels * 4);
    for (int i = 0; i < kCMaxSlot; ++i) ptx::mbar_arm(ptx::smem_u32(&mail->bar_h[i]), R * 4);
    if constexpr (PIPE) {  // one barrier per stream of the cluster for every inbound mailbox
      for (int q = 0; q < kWP; ++q) {
        ptx::mbar_init(ptx::smem_u32(&mail->pb_hin[q]), 1);
        ptx::mbar_init(ptx::smem_u32(&mail->pb_xin[q]), 1);
        ptx::mbar_init(ptx::smem_u32(&mail->pb_logits[q]), 1);
        ptx::mbar_init(ptx::smem_u32(&mail->pb_part[q]), 1);
        ptx::mbar_init(ptx::smem_u32(&mail->pb_za[q]), 1);
        for (int i = 0; i < kCMaxSlot; ++i) ptx::mbar_init(ptx::smem_u32(&mail->pb_h[i][q]), 1);
        mail->ys[q][0] = mail->ys[q][1] = kLevels / 2;  // R4
      }
      for (int q = 0; q < kPR; ++q) ptx::mbar_init(ptx::smem_u32(&mail->bar_pre2[q]), 1);
      for (int q = 0; q < kWNB; ++q) ptx::mbar_init(ptx::smem_u32(&mail->wfull[q]), 1);
      ptx::fence_mbar_init();
      for (int q = 0; q < kWP; ++q) {
        ptx::mbar_arm(ptx::smem_u32(&mail->pb_hin[q]), R * 4);
        ptx::mbar_arm(ptx::smem_u32(&mail->pb_xin[q]), R * 4);
        ptx::mbar_arm(ptx::smem_u32(&mail->pb_logits[q]), kLevels * 4);
        ptx::mbar_arm(ptx::smem_u32(&mail->pb_part[q]), pl.npart * S * 4);
        ptx::mbar_arm(ptx::smem_u32(&mail->pb_za[q]), kLevels * 4);
        for (int i = 0; i < kCMaxSlot; ++i) ptx::mbar_arm(ptx::smem_u32(&mail->pb_h[i][q]), R * 4);
      }
    }
  }
  if (role != kIdle) {
    const float4* src = reinterpret_cast<const float4*>(P.pk + pl.pk_smem_off[rank]);
    float4* dst = reinterpret_cast<float4*>(sw);
    for (int i = t; i < pl.pk_smem_floats[rank] / 4; i += kThreads) dst[i] = __ldg(src + i);
  }
  ptx::tmem_fence_before();
  __syncthreads();
  ptx::tmem_fence_after();
  // Tensor-memory image: [column][128 lanes]; each math thread fills the columns its role
  // uses in its own lane (chain: A [0,192) C [192,320) B [320,416); head / skip: A-half
  // [0,256) B-half [256,512)).
  if (t >= kAux && role != kIdle) {
    const int wg = (t - kAux) >> 7;  // 0 = A, 1 = B, 2 = C
    int c0 = 0, c1 = 0;
    if (role == kChain) {
      if (wg == 0) { c0 = kColA; c1 = col_c(LP); }
      else if (wg == 2) { c0 = col_c(LP); c1 = 2 * col_c(LP); }
      else if (LP == 3) { c0 = kColB3; c1 = kColB3 + 3 * 32; }
    } else if (wg < 2) {
      c0 = 256 * wg;
      c1 = c0 + 256;
    }
    c1 = min(c1, pl.tm_cols[rank]);
    const int lane = (t - kAux) & 127;
    const float* img = P.pk + pl.pk_off[rank];
    const uint32_t ta = tmem_lane_addr(*mail);
    for (int col = c0; col < c1; col += 16) {
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = __ldg(img + (int64_t)(col + i) * 128 + lane);
      ptx::tmem_st16(ta + col, v);
    }
    ptx::tmem_wait_st();
  }
  ptx::tmem_fence_before();
  __syncthreads();
  ptx::tmem_fence_after();
  ptx::cluster_sync();

  if (t >= kAux) {
    if (role == kChain) {
      if (t < kAux + 128) chain_A<LP, TRACE, NL, SESS, PIPE>(P, cx, idx, sw);
      else if (t < kAux + 256) chain_B<LP, TRACE, SESS, PIPE>(P, cx, idx, sw);
      else chain_C<LP, TRACE, SESS, PIPE>(P, cx, idx, sw);
    } else if (role == kHead) {
      if (t < kAux + kMain) head_main<S, TRACE, PIPE>(P, cx, idx, sw);
    } else if (role == kSkip) {
      if (t < kAux + kMain) skip_main<S, TRACE, PIPE>(P, cx, idx, sw);
    }
    ptx::tmem_fence_before();
    ptx::bar_sync(kBarMath, kMath);
    if (t == kAux) ptx::mbar_arrive(ptx::smem_u32(&mail->bar_exit));
    __syncwarp();
    ptx::cluster_sync();
    return;
  }
  if constexpr (PIPE) {
    if (role == kChain) chain_aux_pipe<S, LP>(P, cx, idx, sw);
  } else {
    if (role == kChain) chain_aux<S, LP, TRACE, SESS, PIPE>(P, cx, idx, sw);
  }
  // Park until the math warps are done (try_wait suspends the warp), then free TMEM.
  while (!ptx::mbar_try_wait_cta(ptx::smem_u32(&mail->bar_exit), 0)) {
  }
  ptx::tmem_fence_after();
  if (t < 32) ptx::tmem_dealloc(mail->tmem_base, kTmemCols);
  __syncwarp();
  ptx::cluster_sync();
}

template <int S, int LP, bool TRACE, int NL = 0, bool SESS = false, bool PIPE = false>
cudaError_t configure(int smem) {
  cudaError_t e = cudaFuncSetAttribute(k_cluster<S, LP, TRACE, NL, SESS, PIPE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_cluster<S, LP, TRACE, NL, SESS, PIPE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}

template <int S, int LP>
int max_active_clusters(int size, int smem) {
  if (configure<S, LP, false>(smem) != cudaSuccess || configure<S, LP, true>(smem) != cudaSuccess ||
      configure<S, LP, false, 1>(smem) != cudaSuccess || configure<S, LP, false, 2>(smem) != cudaSuccess ||
      configure<S, LP, false, 0, true>(smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(size);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = size;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_cluster<S, LP, false>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// The multi-stream variant (production gate only): co-resident clusters at its shared-memory size.
template <int S, int LP>
int max_active_pipe(int size, int smem) {
  if (configure<S, LP, false, 0, false, true>(smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(size);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = size;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_cluster<S, LP, false, 0, false, true>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}


}  // namespace

namespace {
// One residency plan with `lp` layers per chain CTA.
ClusterPlan plan_lp(int L, int r, int s, int device, int lp) {
  ClusterPlan p;
  p.L = L;
  p.r = r;
  p.s = s;
  p.lpc = lp;
  if (r != R) { p.why = "cluster kernel is built for r = 64"; return p; }
  if (s != 128 && s != 256) { p.why = "cluster kernel needs s in {128, 256}"; return p; }
  if (L > kCMaxLayers) { p.why = "too many layers"; return p; }
  p.nc = (L + lp - 1) / lp;
  for (int c = 0; c < p.nc; ++c) {
    p.chain_first[c] = c * lp;
    p.chain_nl[c] = std::min(lp, L - c * lp);
    p.xpart_slot[c] = -1;
  }
  p.nh = NH;
  if (p.nc + p.nh > kCMaxCta) { p.why = "model does not fit one 16-CTA cluster"; return p; }
  const int nskip = std::max(0, L - 2);  // W_skip^(l) and W_skip^(l-1) live in the head CTAs
  const int qs = s / 4;                   // floats of one skip layer's tile per thread
  const int maxtm = 256 / qs;             // skip layers in tensor memory per thread half
  const int lstride = qs * kMain;         // floats per shared-memory skip layer
  const int maxsm = std::min(kCMaxSlot - maxtm, (int)((190 * 1024) / (lstride * 4)));
  const int cap = maxtm + maxsm;
  // skip CTAs take the latest layers; what they cannot hold (the earliest layers) is applied
  // by each layer's own chain CTA from L2 after its pass
  p.nk = nskip > 0 ? std::min(kCMaxCta - p.nc - p.nh, (nskip + cap - 1) / cap) : 0;
  p.nxs = std::max(0, nskip - p.nk * cap);
  if (p.nxs > 0 && p.nxs > nskip - 2 * lp) {
    p.why = "model does not fit one 16-CTA cluster (chain-skip layers too close to the head)";
    return p;
  }
  const int nxp = (p.nxs + lp - 1) / lp;  // chain CTAs that send a partial
  p.npart = p.nk + nxp;
  if (p.npart > kCMaxSkip) { p.why = "too many skip partials"; return p; }
  for (int c = 0; c < nxp; ++c) p.xpart_slot[c] = p.nk + c;
  p.size = p.nc + p.nh + p.nk;
  for (int k = 0; k < p.nk; ++k) p.skip_n[k] = 0;
  for (int j = 0; j < p.nxs; ++j) {
    p.layer_skip_cta[j] = -1;
    p.layer_skip_slot[j] = 0;
  }
  // Skip CTA k takes a contiguous block of layers (DVW_SKIP_RR=1: round robin, A/B).  With several
  // streams in flight (the multi-stream variant) a skip CTA holds an item from its first owned layer
  // to its last, so a block spanning a third of the chain instead of all of it triples how many
  // items it can serve per chain traversal; at batch 1 a block keeps up as well (one 64 x 256 matvec
  // per arriving layer).
  const char* rr = std::getenv("DVW_SKIP_RR");
  const bool round_robin = rr && std::atoi(rr) == 1;
  const int nsk = nskip - p.nxs, per = p.nk > 0 ? (nsk + p.nk - 1) / p.nk : 0;
  for (int j = p.nxs; j < nskip; ++j) {
    const int k = round_robin ? (j - p.nxs) % p.nk : (j - p.nxs) / per;
    p.layer_skip_cta[j] = p.nc + p.nh + k;
    p.layer_skip_slot[j] = p.skip_n[k]++;
  }
  for (int k = 0; k < p.nk; ++k) {
    if (p.skip_n[k] > cap) { p.why = "skip capacity"; return p; }
    p.skip_nsm[k] = std::max(0, p.skip_n[k] - maxtm);  // latest layers in tensor memory
  }
  int dev_smem = 0;
  cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  int64_t off = 0;
  int max_sw = 0;
  for (int rank = 0; rank < p.size; ++rank) {
    int swf = 0;
    p.nwp[rank] = 0;
    if (rank < p.nc && lp == 4 && !kXStream) {
      swf = smem_chain(rank, lp);
      // W_prev of the CTA's first layers into the shared memory left free in the (larger)
      // multi-stream layout, so neither variant streams them from L2
      const int64_t used = (int64_t)((sizeof(Mail) + 127) & ~size_t(127)) + (int64_t)kMbChainEnd4 * 4 + (int64_t)swf * 4;
      p.nwp[rank] = (int)std::max<int64_t>(0, std::min<int64_t>(p.chain_nl[rank], ((int64_t)dev_smem - used) / (16 * 128 * 4 * 4)));
      swf += p.nwp[rank] * 16 * 128 * 4;
    } else if (rank < p.nc) swf = smem_chain(rank, lp);
    else if (rank < p.nc + p.nh) swf = s + 128;
    else swf = p.skip_nsm[rank - p.nc - p.nh] * lstride;
    p.pk_off[rank] = off;
    p.tm_cols[rank] = kTmemCols;
    off += (int64_t)kTmemCols * 128;
    p.pk_smem_off[rank] = off;
    p.pk_smem_floats[rank] = swf;
    off += (swf + 3) & ~3;
    max_sw = std::max(max_sw, swf);
  }
  p.embp_off = off;
  off += (int64_t)kLevels * R;
  p.wprev_off = off;
  off += (int64_t)L * 16 * 128 * 4;
  p.wskx_off = off;
  off += (int64_t)p.nxs * 16 * s * 4;
  p.pk_total = off;
  p.smem_bytes = (int)(((sizeof(Mail) + 127) & ~size_t(127)) + (size_t)max_sw * 4);
  if (p.smem_bytes > dev_smem) { p.why = "shared memory"; return p; }
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  int nclus;
  if (s == 256) nclus = lp == 3 ? max_active_clusters<256, 3>(p.size, p.smem_bytes) : max_active_clusters<256, 4>(p.size, p.smem_bytes);
  else nclus = lp == 3 ? max_active_clusters<128, 3>(p.size, p.smem_bytes) : max_active_clusters<128, 4>(p.size, p.smem_bytes);
  if (prev >= 0) cudaSetDevice(prev);
  if (nclus < 1) { p.why = "cluster cannot be scheduled on this device"; return p; }
  p.max_clusters = nclus;
  // multi-stream variant: [Mail][per-stream inbound mailboxes of the CTA's role][weights image]
  {
    const size_t mailb = (sizeof(Mail) + 127) & ~size_t(127);
    int smem_pipe = 0;
    for (int rank = 0; rank < p.size; ++rank) {
      int64_t mbf;
      p.xnb[rank] = 0;
      if (rank < p.nc && lp == 4 && kXStream) {  // weight-stream ring: as many 16-KB buffers as fit (<= kWNB)
        const int64_t used = (int64_t)mailb + (int64_t)kMbChainEnd4 * 4 + (int64_t)p.pk_smem_floats[rank] * 4;
        p.xnb[rank] = (int)std::min<int64_t>(kWNB, ((int64_t)dev_smem - used) / (kWChunk * 4));
        if (p.xnb[rank] < 1) p.xnb[rank] = -1;  // does not fit: no multi-stream variant
      }
      if (rank < p.nc) mbf = lp == 4 ? kMbChainEnd4 + (int64_t)std::max(0, p.xnb[rank]) * kWChunk : kMbChainEnd3;
      else if (rank < p.nc + p.nh) mbf = 2 * kWP * kHLen + kWP * kVLen + (int64_t)p.npart * kWP * 256;
      else mbf = (int64_t)p.skip_n[rank - p.nc - p.nh] * kWP * kHLen;
      const int64_t off = (int64_t)mailb + ((mbf * 4 + 127) & ~int64_t(127));
      p.sw_off_pipe[rank] = (int)off;
      smem_pipe = std::max(smem_pipe, (int)(off + (int64_t)p.pk_smem_floats[rank] * 4));
    }
    p.smem_pipe = smem_pipe;
    bool fits = smem_pipe <= dev_smem;
    for (int rank = 0; rank < p.nc; ++rank) fits = fits && p.xnb[rank] >= 0;
    if (fits) {
      cudaGetDevice(&prev);
      cudaSetDevice(device);
      int np = 0;
      if (s == 256) np = lp == 3 ? max_active_pipe<256, 3>(p.size, smem_pipe) : max_active_pipe<256, 4>(p.size, smem_pipe);
      else np = lp == 3 ? max_active_pipe<128, 3>(p.size, smem_pipe) : max_active_pipe<128, 4>(p.size, smem_pipe);
      if (prev >= 0) cudaSetDevice(prev);
      p.max_clusters_pipe = np;
      p.pipe_ok = np >= 1;
    }
  }
  p.ok = true;
  p.why = "ok";
  return p;
}
}  // namespace

// 3 layers per chain CTA (every weight of the chain in tensor memory) when the model fits
// one cluster that way with no chain-skip layers; else 4 (W_res in shared memory).
ClusterPlan plan_cluster(int L, int r, int s, int device) {
  // tuning override for A/B measurements (tools/sweep_layers.py): DVW_CLUSTER_LP=3|4
  if (const char* e = std::getenv("DVW_CLUSTER_LP")) {
    const int lp = std::atoi(e);
    if (lp == 3 || lp == 4) return plan_lp(L, r, s, device, lp);
  }
  ClusterPlan p3 = plan_lp(L, r, s, device, 3);
  if (p3.ok && p3.nxs == 0) return p3;
  ClusterPlan p4 = plan_lp(L, r, s, device, 4);
  return p4.ok ? p4 : p3;
}

size_t packed_bytes(const ClusterPlan& p) { return sizeof(float) * (size_t)p.pk_total; }

// Residency layout, built on the host from the raw roster-order blob: the tensor-memory
// images [column][lane], the shared-memory images, W_emb_prev^T.  Index shuffling plus
// the fold M^(j) = W_cur^(j+1) W_res^(j) and c^(j) = W_cur^(j+1) B_res^(j), computed in
// double precision and rounded once to fp32.
cudaError_t pack_cluster_weights(const ClusterPlan& p, const float* w, const Offsets& o, void* packed) {
  const int s = p.s, qs = s / 4, rq = s / 64, cz = s / 16;
  std::vector<float> h((size_t)p.pk_total, 0.0f);
  auto W = [&](int j, int64_t off_in_layer, int row, int col, int ncol) {
    return w[(int64_t)j * o.layer_stride + off_in_layer + (int64_t)row * ncol + col];
  };
  auto fold = [&](int j, std::vector<float>& M, std::vector<float>& cvec) {  // j: the W_res layer
    M.assign(2 * R * R, 0.0f);
    cvec.assign(2 * R, 0.0f);
    for (int i = 0; i < 2 * R; ++i) {
      double cs = 0.0;
      for (int k = 0; k < R; ++k) {
        double acc = 0.0;
        for (int t = 0; t < R; ++t) acc += (double)W(j + 1, o.w_cur, i, t, R) * (double)W(j, o.w_res, t, k, R);
        M[i * R + k] = (float)acc;
      }
      for (int t = 0; t < R; ++t) cs += (double)W(j + 1, o.w_cur, i, t, R) * (double)w[(int64_t)j * o.layer_stride + o.b_res + t];
      cvec[i] = (float)cs;
    }
  };
  for (int rank = 0; rank < p.size; ++rank) {
    float* img = h.data() + p.pk_off[rank];  // [col][128]
    float* sm = h.data() + p.pk_smem_off[rank];
    auto put = [&](int col, int lane, float v) { img[(int64_t)col * 128 + lane] = v; };
    if (rank < p.nc) {
      const int first = p.chain_first[rank], nl = p.chain_nl[rank], lp = p.lpc;
      const int xb = (rank == 0) ? 1 : 0;  // CTA 0's layer 0 takes the embedding directly
      // local layer jl (layer j = first + jl) with jl >= xb: M_j = W_cur_j W_res_{j-1}, c_j = W_cur_j B_res_{j-1}
      std::vector<std::vector<float>> M(LPC), cf(LPC);
      for (int jl = xb; jl < nl; ++jl) fold(first + jl - 1, M[jl], cf[jl]);
      for (int lane = 0; lane < 128; ++lane) {
        const int g = lane >> 1, half = lane & 1;  // rows g (tanh), R + g (sigmoid); columns [32 half, +32)
        for (int jl = 0; jl < nl; ++jl)
          for (int q = 0; q < 64; ++q) {
            const int row = (q < 32) ? g : R + g, col = 32 * half + (q & 31);
            put(kColA + 64 * jl + q, lane, jl < xb ? W(first, o.w_cur, row, col, R) : M[jl][row * R + col]);
            if (jl >= xb) put(col_c(lp) + 64 * jl + q, lane, W(first + jl, o.w_cur, row, col, R));
          }
        for (int jl = xb; jl < nl; ++jl)  // B's W_res_{j-1} row-pair tile: TMEM (LP 3) or shared memory (LP 4)
          for (int q = 0; q < 32; ++q) {
            const float v = W(first + jl - 1, o.w_res, g, 32 * half + q, R);
            if (lp == 3) put(kColB3 + 32 * jl + q, lane, v);
            else sm[kSmWres + ((jl * 8 + q / 4) * 128 + lane) * 4 + q % 4] = v;
          }
      }
      for (int jl = 0; jl < nl; ++jl) {
        const int j = first + jl;
        if (lp == 3)  // W_prev_j [16][128][4] in shared memory
          for (int i = 0; i < 2 * R; ++i)
            for (int k = 0; k < R; ++k) sm[(jl * 16 * 128 + (k / 4) * 128 + i) * 4 + k % 4] = W(j, o.w_prev, i, k, R);
        if (lp == 4 && jl < p.nwp[rank])  // LP = 4: the first nwp layers' W_prev after the image
          for (int i = 0; i < 2 * R; ++i)
            for (int k = 0; k < R; ++k)
              sm[smem_chain(rank, lp) + (jl * 16 * 128 + (k / 4) * 128 + i) * 4 + k % 4] = W(j, o.w_prev, i, k, R);
        for (int i = 0; i < 2 * R; ++i) sm[sm_b(lp) + jl * 2 * R + i] = w[(int64_t)j * o.layer_stride + o.b + i];
        if (jl >= xb) {
          for (int i = 0; i < R; ++i) sm[sm_bres(lp) + jl * R + i] = w[(int64_t)(j - 1) * o.layer_stride + o.b_res + i];
          for (int i = 0; i < 2 * R; ++i) sm[sm_fold(lp) + jl * 2 * R + i] = cf[jl][i];
        }
      }
      if (rank == 0) {
        float* we = sm + sm_emb(lp);
        for (int y = 0; y < kLevels; ++y)
          for (int i = 0; i < R; ++i) we[y * R + i] = w[o.emb_cur + (int64_t)i * kLevels + y];
        for (int i = 0; i < R; ++i) we[kLevels * R + i] = w[o.b_emb + i];
      }
    } else if (rank < p.nc + p.nh) {
      const int hidx = rank - p.nc;
      const int jl = p.L - 1;
      for (int k = 0; k < kMain; ++k) {
        const int lane = k & 127, cbase = (k < 128) ? 0 : 256;
        const int g = k >> 2, cc = k & 3, c16 = k & 15, rbase = 64 * hidx + 4 * (k >> 4);
        for (int mm = 0; mm < rq; ++mm)
          for (int q = 0; q < 16; ++q) put(cbase + mm * 16 + q, lane, W(jl, o.w_skip, g + 64 * mm, 16 * cc + q, R));
        for (int mm = 0; mm < 4; ++mm)
          for (int q = 0; q < cz; ++q)
            put(cbase + rq * 16 + mm * cz + q, lane, w[o.w_relu + (int64_t)(rbase + mm) * s + c16 * cz + q]);
        for (int mm = 0; mm < 4; ++mm)
          for (int q = 0; q < 16; ++q)
            put(cbase + rq * 16 + 4 * cz + mm * 16 + q, lane, w[o.w_out + (int64_t)(rbase + mm) * kLevels + 16 * c16 + q]);
      }
      for (int i = 0; i < s; ++i) sm[i] = w[o.b_skip + i];
      for (int i = 0; i < 64; ++i) {
        sm[s + i] = w[o.b_relu + 64 * hidx + i];
        sm[s + 64 + i] = w[o.b_out + 64 * hidx + i];
      }
      if (p.L >= 2)  // W_skip^(l-1) in tensor memory after W_out
        for (int k = 0; k < kMain; ++k) {
          const int lane = k & 127, cbase = (k < 128) ? 0 : 256;
          const int g = k >> 2, cc = k & 3;
          for (int mm = 0; mm < rq; ++mm)
            for (int q = 0; q < 16; ++q)
              put(cbase + rq * 16 + 4 * cz + 64 + mm * 16 + q, lane, W(p.L - 2, o.w_skip, g + 64 * mm, 16 * cc + q, R));
        }
    } else {
      const int k = rank - p.nc - p.nh;
      std::vector<int> layers;
      for (int j = 0; j < p.L - 2; ++j)
        if (p.layer_skip_cta[j] == rank) layers.push_back(j);
      const int nsm = p.skip_nsm[k];
      const int lstride = qs * kMain;
      for (int sl = 0; sl < (int)layers.size(); ++sl) {
        const int j = layers[sl];
        for (int t = 0; t < kMain; ++t) {
          const int g = t >> 2, cc = t & 3;
          for (int mm = 0; mm < rq; ++mm)
            for (int q = 0; q < 16; ++q) {
              const float v = W(j, o.w_skip, g + 64 * mm, 16 * cc + q, R);
              const int qq = mm * 16 + q;
              if (sl < nsm) sm[sl * lstride + ((qq / 4) * kMain + t) * 4 + (qq % 4)] = v;
              else put((t < 128 ? 0 : 256) + (sl - nsm) * qs + qq, t & 127, v);
            }
        }
      }
    }
  }
  float* ep = h.data() + p.embp_off;
  for (int y = 0; y < kLevels; ++y)
    for (int i = 0; i < R; ++i) ep[y * R + i] = w[o.emb_prev + (int64_t)i * kLevels + y];
  for (int j = 0; j < p.L; ++j) {  // W_prev_j [16][128][4] (streamed by the chain aux warps)
    float* wp = h.data() + p.wprev_off + (int64_t)j * 16 * 128 * 4;
    for (int i = 0; i < 2 * R; ++i)
      for (int k = 0; k < R; ++k) wp[((k / 4) * 128 + i) * 4 + k % 4] = W(j, o.w_prev, i, k, R);
  }
  for (int j = 0; j < p.nxs; ++j) {  // chain-skip W_skip_j [s/128 (row block)][16][128][4]
    float* ws = h.data() + p.wskx_off + (int64_t)j * 16 * s * 4;
    for (int i = 0; i < s; ++i)
      for (int k = 0; k < R; ++k) ws[(((i / 128) * 16 + k / 4) * 128 + i % 128) * 4 + k % 4] = W(j, o.w_skip, i, k, R);
  }
  return cudaMemcpy(packed, h.data(), sizeof(float) * h.size(), cudaMemcpyHostToDevice);
}

cudaError_t launch_cluster_kernel(const RunArgs& a, const ClusterPlan& p, const void* packed, cudaStream_t st,
                                  LaunchInfo* info) {
  if (!p.ok) return cudaErrorNotSupported;
  if (a.n_streams < 1 || (a.trace && a.n_streams != 1)) return cudaErrorInvalidValue;
  Params P;
  P.a = a;
  P.p = p;
  P.pk = static_cast<const float*>(packed);
  P.wmax = 1;
  P.xpb = 1;
  P.xsb = 1;
  const bool tr = a.trace != nullptr;
  const bool ss = a.ystate != nullptr;
  const bool ap = a.approx == 1 && !tr && !ss;
  const bool pc = a.approx == 2 && !tr && !ss;
  // Streams per cluster: one (cluster c generates stream c, Ctx::sidx), or -- for more streams than
  // clusters fit at once, production gate, no session / trace -- up to kWP interleaved per cluster
  // (the multi-stream variant), spread evenly.  DVW_CLUSTER_W=k forces k (A/B measurements).
  int w = 1;
  if (p.pipe_ok && !tr && !ss && a.approx == 0 && a.N * kWP < (int64_t(1) << 31)) {
    const int cap = std::max(1, p.max_clusters_pipe);
    if (a.n_streams > p.max_clusters) w = std::min(kWP, (a.n_streams + cap - 1) / cap);
    if (const char* ev = std::getenv("DVW_CLUSTER_W")) w = std::max(1, std::min(kWP, std::atoi(ev)));
  }
  P.wmax = w;
  P.xpb = kPB;
  P.xsb = kXH;
  if (const char* ev = std::getenv("DVW_XPB")) P.xpb = std::max(1, std::min(kPB, std::atoi(ev)));
  if (const char* ev = std::getenv("DVW_XSB")) P.xsb = std::max(1, std::min(kXH, std::atoi(ev)));
  const int nclu = (a.n_streams + w - 1) / w;
  cudaLaunchConfig_t cfg{};
  // clusters never wait for each other, so more clusters than fit at once simply run in waves
  cfg.gridDim = dim3(p.size * nclu);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = w > 1 ? p.smem_pipe : p.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.size;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e;
  // variants: production (exact gate), TRACE (exact gate + timestamps), NL = 1 (hardware tanh),
  // NL = 2 (App. C gate and exp), SESS (streaming session: continues the queues and code
  // history; exact gate -- the API routes approximate-tier sessions to the stream kernel)
#define DVW_LAUNCH(S_, LP_)                                                         \
  e = w > 1 ? cudaLaunchKernelEx(&cfg, k_cluster<S_, LP_, false, 0, false, true>, P) \
      : ss ? cudaLaunchKernelEx(&cfg, k_cluster<S_, LP_, false, 0, true>, P)       \
      : tr ? cudaLaunchKernelEx(&cfg, k_cluster<S_, LP_, true>, P)                 \
      : ap ? cudaLaunchKernelEx(&cfg, k_cluster<S_, LP_, false, 1>, P)             \
      : pc ? cudaLaunchKernelEx(&cfg, k_cluster<S_, LP_, false, 2>, P)             \
           : cudaLaunchKernelEx(&cfg, k_cluster<S_, LP_, false>, P)
  if (p.s == 256 && p.lpc == 3) {
    DVW_LAUNCH(256, 3);
  } else if (p.s == 256) {
    DVW_LAUNCH(256, 4);
  } else if (p.lpc == 3) {
    DVW_LAUNCH(128, 3);
  } else {
    DVW_LAUNCH(128, 4);
  }
#undef DVW_LAUNCH
  info->grid = p.size * nclu;
  info->cluster = p.size;
  info->rows_per_block = w;
  info->threads = kThreads;
  info->launches = 1;
  return e;
}

// ------------------------------------------------------------------ latency-floor microbenchmarks
// (dvw_measure_floor; SURVEY.md §8(d) "measured latency floor").  Each kernel times, with clock64
// on one SM, the minimal dependent form of one piece of the batch-1 critical path, built from the
// same device functions the cluster kernel runs:
//   layer   : one chain layer with nothing else on the SM -- LDS of h, the 128 x 64 matvec
//             (tile_dot_half<2>, 32 FFMA2 per thread), the pair shuffle, gate_fast, STS of h and
//             the named barrier that publishes it (warpgroup A alone)
//   hop     : one DSMEM hand-off -- st.async of 4 bytes completing transaction bytes on the peer
//             CTA's mbarrier, observed by the peer's try_wait (ping-pong / 2)
//   head    : one head stage -- 64-row x 256-column slice (tile_dot<4,16>), 4 transposing shuffle
//             levels, STS and a 256-thread named barrier
//   sampler : one inverse-CDF draw by one warp (sample_warp), each draw dependent on the last
namespace {
__global__ void __launch_bounds__(128, 1) k_probe_layer(int iters, unsigned long long* out) {
  __shared__ __align__(16) float hs[2][kHLen];
  const int a = threadIdx.x, hrow = a >> 1, half = a & 1, voff = 40 * half;
  float w[64];
#pragma unroll
  for (int q = 0; q < 64; ++q) w[q] = 0.01f * (float)((q * 7 + a * 13) % 17 - 8);
  const float pre0 = 0.01f * (a % 5), pre1 = -0.02f * (a % 3);
  for (int i = a; i < 2 * kHLen; i += 128) (&hs[0][0])[i] = 0.1f;
  __syncthreads();
  long long t0 = 0;
  float acc = 0.0f;
#pragma unroll 1
  for (int n = -64; n < iters; ++n) {
    if (n == 0) t0 = clock64();
    const int p = n & 1;
    float v[2];
    tile_dot_half<2>(w, hs[p] + voff, v);
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    v[1] += __shfl_xor_sync(0xffffffffu, v[1], 1);
    const float hv = gate_fast(v[0] + pre0, v[1] + pre1);
    if (half == 0) hs[p ^ 1][pad16(hrow)] = hv;
    acc += hv;
    ptx::bar_sync(1, 128);
  }
  const long long t1 = clock64();
  if (a == 0) {
    out[0] = (unsigned long long)(t1 - t0);
    out[1] = __float_as_uint(acc);
  }
}

__global__ void __launch_bounds__(32, 1) k_probe_hop(int iters, unsigned long long* out) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(16) float box[4];
  const uint32_t rank = ptx::cluster_rank();
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
    ptx::mbar_arm(ptx::smem_u32(&bar), 4);
  }
  __syncwarp();
  ptx::cluster_sync();
  const uint32_t peer = rank ^ 1u;
  const uint32_t rbox = ptx::mapa(ptx::smem_u32(&box[0]), peer), rbar = ptx::mapa(ptx::smem_u32(&bar), peer);
  long long t0 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
      if (rank == 0) {
        ptx::st_async(rbox, (float)i, rbar);
        while (!ptx::mbar_try_wait_cta(ptx::smem_u32(&bar), (uint32_t)(i & 1))) {
        }
        ptx::mbar_arm(ptx::smem_u32(&bar), 4);
      } else {
        while (!ptx::mbar_try_wait_cta(ptx::smem_u32(&bar), (uint32_t)(i & 1))) {
        }
        ptx::mbar_arm(ptx::smem_u32(&bar), 4);
        ptx::st_async(rbox, box[0] + 1.0f, rbar);
      }
    }
    if (rank == 0) out[2] = (unsigned long long)(clock64() - t0);
  }
  __syncwarp();
  ptx::cluster_sync();
}

__global__ void __launch_bounds__(256, 1) k_probe_head(int iters, unsigned long long* out) {
  __shared__ __align__(16) float zb[2][kVLen];
  const int k = threadIdx.x, c16 = k & 15, orow = 4 * (k >> 4) + ((k >> 2) & 3);
  float w[64];
#pragma unroll
  for (int q = 0; q < 64; ++q) w[q] = 0.003f * (float)((q * 5 + k * 11) % 13 - 6);
  for (int i = k; i < 2 * kVLen; i += 256) (&zb[0][0])[i] = 0.05f;
  __syncthreads();
  long long t0 = 0;
  float acc = 0.0f;
#pragma unroll 1
  for (int n = -32; n < iters; ++n) {
    if (n == 0) t0 = clock64();
    const int p = n & 1;
    float lg[4];
    tile_dot<4, 16>(w, &zb[p][20 * c16], lg);
    xpose_level<4>(lg, k, 8);
    xpose_level<2>(*reinterpret_cast<float(*)[2]>(lg), k, 4);
    lg[0] += __shfl_xor_sync(0xffffffffu, lg[0], 2);
    lg[0] += __shfl_xor_sync(0xffffffffu, lg[0], 1);
    const float z = fmaxf(lg[0], 0.0f) * 0.5f;
    if ((k & 3) == 0) zb[p ^ 1][pad16(64 * (n & 3) + orow)] = z;
    acc += z;
    ptx::bar_sync(1, 256);
  }
  const long long t1 = clock64();
  if (k == 0) {
    out[3] = (unsigned long long)(t1 - t0);
    out[4] = __float_as_uint(acc);
  }
}

__global__ void __launch_bounds__(32, 1) k_probe_sampler(int iters, unsigned long long* out) {
  __shared__ __align__(16) float lg[kLevels];
  const int lane = threadIdx.x;
  for (int i = lane; i < kLevels; i += 32) lg[i] = 0.05f * (float)((i * 37) % 23) - 0.5f;
  __syncwarp();
  long long t0 = 0;
  int y = 0;
#pragma unroll 1
  for (int n = -16; n < iters; ++n) {
    if (n == 0) t0 = clock64();
    const float u = (float)((n * 2654435761u + (unsigned)y * 97u) >> 8) * 5.9604645e-08f;
    y = sample_warp<0>(lg, u, lane);
    if (lane == 0) lg[y] += 1e-3f;  // the next draw depends on this one
    __syncwarp();
  }
  const long long t1 = clock64();
  if (lane == 0) {
    out[5] = (unsigned long long)(t1 - t0);
    out[6] = (unsigned long long)y;
  }
}

__global__ void k_probe_clock(int spin, unsigned long long* out) {
  const uint64_t g0 = ptx::globaltimer();
  const long long c0 = clock64();
  while (clock64() - c0 < spin) {
  }
  out[7] = (unsigned long long)(clock64() - c0);
  out[8] = (unsigned long long)(ptx::globaltimer() - g0);
}
}  // namespace

cudaError_t measure_floor(int device, FloorProbe* f) {
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  unsigned long long* d = nullptr;
  unsigned long long h[16] = {};
  constexpr int kIters = 20000;
  cudaError_t e = cudaMalloc(&d, sizeof(h));
  if (e == cudaSuccess) e = cudaMemset(d, 0, sizeof(h));
  if (e == cudaSuccess) {
    k_probe_clock<<<1, 1>>>(20000000, d);  // ~10 ms: the SM clock under this (latency-bound) load
    k_probe_layer<<<1, 128>>>(kIters, d);
    k_probe_head<<<1, 256>>>(kIters, d);
    k_probe_sampler<<<1, 32>>>(kIters / 4, d);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(32);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k_probe_hop, kIters, d);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (d) cudaFree(d);
  if (e == cudaSuccess) {
    f->layer_cycles = (double)h[0] / kIters;
    f->hop_cycles = (double)h[2] / (2.0 * kIters);
    f->head_stage_cycles = (double)h[3] / kIters;
    f->sampler_cycles = (double)h[5] / (kIters / 4);
    f->sm_ghz = h[8] ? (double)h[7] / (double)h[8] : 0.0;
  }
  if (prev >= 0) cudaSetDevice(prev);
  return e;
}

}  // namespace dvw

#if DVW_PTRACE
extern "C" __attribute__((visibility("default"))) int dvw_diag_ptrace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, dvw::g_pt, sizeof(dvw::g_pt));
}
#endif
