// kernel_batch.cu -- batched multi-stream kernel: tcgen05 (kind::tf32, 3 passes)
// projections; one persistent launch per launch group, one thread-block cluster per
// stream block of 128 streams, the hardware cluster barrier between phases.
//
// Step n of every stream, as phases (0-based layer j; §5.1):
//   phase j (0 <= j < l): layer tile t of stream block sb computes, for channels
//       [16t, 16t+16),
//         a^(j) = W_prev^(j) x^(j)_{n-d_j} + W_cur^(j) x^(j)_n + B^(j) + L^(j)_n
//         h^(j) = tanh(a_tanh) * sigma(a_sigma)
//       where, for j >= 1, W_cur^(j) x^(j) is evaluated as
//         W_cur^(j) x^(j-1) + M^(j) h^(j-1) + W_cur^(j) B_res^(j-1),  M^(j) = W_cur^(j) W_res^(j-1)
//       (the residual update of PAPER.md:437 folded in, M formed in fp64 on the host;
//       reading R22), so a layer needs only the PREVIOUS phase's outputs and one barrier
//       per layer suffices.  The same CTA also finishes the residual update of layer j-1,
//         x^(j) = x^(j-1) + W_res^(j-1) h^(j-1) + B_res^(j-1)
//       and stores it into layer j's dilation queue ("never recompute").
//       Skip tile u accumulates q += W_skip^(j-1) h^(j-1) in TMEM.
//   phase l    : skip tiles add W_skip^(l-1) h^(l-1); z_s = relu(q), q_0 = B_skip
//   phase l+1  : head tile v: z_a = relu(W_relu z_s + B_relu), rows [64v, 64v+64)
//   phase l+2  : head tile v: logits = W_out z_a + B_out
//   phase l+3  : one warp per stream: inverse-CDF draw (R11), then the
//                embedding x^(0)_{n+1} = W_emb_prev[:, y_{n-1}] + W_emb_cur[:, y_n] + B_emb
//                 into x^(0) and layer 0's queue.
// One thread-block cluster per stream block of 128 streams holds all of its tiles
// (r/16 layer tiles + s/64 skip tiles + 4 head tiles <= 16 CTAs); stream blocks never
// wait for each other.  Operands: A = activations of 128 streams (M = 128, TMEM lane =
// stream), B = a weight tile (N = 32 or 48 or 64 rows, stacked with its tf32 residual
// rows), K staged 32 channels at a time through a kStages-deep ring of shared-memory
// stages filled by cp.async.bulk; every fp32 operand is split into hi = x (the MMA reads
// its tf32 truncation) and lo = x - tf32(x), and each K-step issues hi*[hi; lo] (one MMA
// over the stacked rows) and lo*hi (reading R23).
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "kernel_batch.cuh"
#include "umma.cuh"
#include "ptx.cuh"

namespace dvw {
namespace {

constexpr int kBT = 256;  // 8 warps; warp w reads TMEM lanes [32(w%4), +32) = its streams, half w/4 of the columns
constexpr int kMaxStages = 8;  // ring depth: as many stages as fit (4 at 128 rows per block, up to 8)
constexpr int kChunk = 32;                   // K channels per staged chunk
constexpr int kActChunk = 128 * kChunk;      // floats of one activation chunk slot (hi or lo), up to 128 rows
constexpr int kMaxN = 64;
// one stage = [A_hi: r8 x 32][A_lo: r8 x 32][W: up to 2 kMaxN rows x 32] floats
__host__ __device__ constexpr int stage_floats(int r8) { return 2 * r8 * kChunk + kMaxN * kChunk * 2; }
constexpr int kCtlBytes = 256;  // Ctl (mbarriers) ahead of the stages
constexpr int kSmemBytes = kCtlBytes + 4 * stage_floats(128) * 4;  // 4 stages at 128 rows: 192 KB + control
constexpr int kTmemCols = 128;
// TMEM accumulator columns (a CTA has one role).  Each tile accumulates hi*hi + lo*hi in
// its first block of columns and hi*lo in a second block (the stacked-B pass below):
//   layer: [0,48) = tanh 16 | sigmoid 16 | residual 16, [48,96) the hi*lo partner
//   skip / head (64 rows): [0,64) and [64,128)
constexpr uint32_t kColA = 0, kColA2 = 48, kColQ = 0, kColQ2 = 64, kColH = 0;
constexpr int kTileRows = 64;  // rows of a skip or head tile

constexpr uint64_t kTimeoutNs = 4000000000ull;

struct BParams {
  RunArgs a;
  const float* pk;
  int L, r, s, TA, TQ, TH, per_sb, nsb;
  int rpb, r8;    // streams per stream block (<= 128) and the image's row count (rpb rounded up to 8)
  int nst;        // ring depth (stages of stage_floats(r8) that fit the shared memory)
  int64_t la_off, la_floats, q_off, q_floats, hr_off, hr_floats, ho_off, ho_floats, bias_off;

  float* hb[2];   // h^(k) in hb[k & 1]
  float* zs;      // [hi | lo] nsb x [s/32][8][r8][4]
  float* za;      // [hi | lo] nsb x [8][8][r8][4]
  float* logits;  // [nsb*rpb][256]
  float* ring;    // per layer j: (d_j + 1) slots of [hi | lo] nsb x [r/32][8][r8][4]
  int* yh;        // [nsb*rpb][2]: y_{n-1}, y_{n-2}
  int* abort_flag;  // [nsb]: per stream block (cluster)
  int32_t dil[kBMaxLayers];
  int64_t ring_off[kBMaxLayers];  // floats
};

struct __align__(8) Ctl {
  uint64_t full[kMaxStages], freeb[kMaxStages], done;
  uint32_t tmem;
  int abort;
};

// (channel c, stream row i) inside one stream block's [C/32][8][r8][4] image: only the block's rows
// are stored and staged; the MMA's M = 128 rows past r8 read other data and are never used
__device__ __forceinline__ int canon(int c, int i, int r8) {
  return ((c >> 5) * 8 + ((c & 31) >> 2)) * (r8 * 4) + i * 4 + (c & 3);
}

__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }


// The abort word of this CTA's stream block (one cluster); the host error word is shared.
__device__ __forceinline__ int* abort_word(const BParams& P) { return P.abort_flag + blockIdx.x / P.per_sb; }

__device__ __forceinline__ void raise_abort(const BParams& P, Ctl& c, int code) {
  c.abort = 1;
  if (atomicExch(abort_word(P), 1) == 0) *(volatile int*)P.a.err = code;  // mapped host word
}

// mbarrier wait with watchdog; false on abort / timeout.  The spin touches only the
// barrier; the abort flags and the clock are looked at every 256 probes, so a
// completed phase is seen within one probe.
__device__ __forceinline__ bool mwait(const BParams& P, Ctl& c, uint64_t* bar, uint32_t parity, int code) {
  const uint32_t b = ptx::smem_u32(bar);
  if (ptx::mbar_test_wait_cta(b, parity)) return true;
  const uint64_t t0 = ptx::globaltimer();
  for (uint32_t it = 1;; ++it) {
    if (ptx::mbar_test_wait_cta(b, parity)) return true;
    if ((it & 255) == 0) {
      if (*(volatile int*)&c.abort || *(volatile int*)abort_word(P)) {
        c.abort = 1;
        return false;
      }
      if (ptx::globaltimer() - t0 > kTimeoutNs) {
        raise_abort(P, c, code);
        return false;
      }
    }
  }
}

// Barrier between phases of one stream block: the hardware cluster barrier (release /
// acquire at cluster scope), with every CTA's generic global stores made visible to the
// async proxy (the next phase's bulk copies) on both sides.  Every CTA of the cluster
// passes every barrier, aborted or not.
__device__ __forceinline__ bool phase_sync(const BParams& P, Ctl& c) {
  (void)P;
  (void)c;
  fence_proxy_async_global();
  __syncthreads();
  ptx::cluster_sync();
  fence_proxy_async_global();
  return true;
}

enum BRole { kLayer = 0, kSkipT = 1, kHeadT = 2 };

// Optional %globaltimer trace (dvw_set_trace): [sample][CTA < 16][32 events].
__device__ __forceinline__ void btrace(const BParams& P, int64_t n, int ev) {
  const RunArgs& A = P.a;
  if (A.trace == nullptr || blockIdx.x >= 16) return;
  const int64_t k = n - A.trace_n0;
  if (k < 0 || k >= A.trace_count) return;
  A.trace[(k * 16 + blockIdx.x) * 32 + ev] = ptx::globaltimer();
}

// One staged K-chunk of a tile job: activation image (hi, lo), weight block
// (hi then lo, N rows each), destination TMEM column and whether it starts the
// accumulation.
struct Chunk {
  const float* ah;
  const float* al;
  const float* w;
  int N;   // rows of the hi block (lo*hi pass)
  int NS;  // rows of the stacked [hi; (0); lo] block (hi*[hi; lo] pass)
  uint32_t dcol;
  uint32_t acc;
};

// x^(j)_n (this step's input of layer j) lives in layer j's dilation queue, slot n mod (d_j + 1):
// the epilogue of phase j (or the embedding, j = 0) writes it there once and phase j + 1 reads
// it back from the same place.  [hi | lo] halves, stream block sb.
__device__ __forceinline__ const float* x_now(const BParams& P, int j, int64_t n) {
  const int d = P.dil[j];
  return P.ring + P.ring_off[j] + (int64_t)(n % (d + 1)) * 2 * ((int64_t)P.nsb * P.r * P.r8);
}

__device__ __forceinline__ int job_chunks(const BParams& P, int role, int ph) {
  const int nR = P.r / kChunk;
  if (role == kLayer) return ph < P.L ? (ph >= 1 ? 3 * nR : 2 * nR) : 0;
  if (role == kSkipT) return (ph >= 1 && ph <= P.L) ? nR : 0;
  if (ph == P.L + 1) return P.s / kChunk;
  if (ph == P.L + 2) return kLevels / kChunk;
  return 0;
}

__device__ __forceinline__ Chunk job_chunk(const BParams& P, int role, int idx, int sb, int ph, int64_t n, int c) {
  const int r = P.r, nR = r / kChunk;
  const int64_t actR = (int64_t)P.nsb * r * P.r8;  // floats of one [hi | lo] half
  Chunk k{};
  if (role == kLayer) {
    const int j = ph;
    const float* wb = P.pk + P.la_off + ((int64_t)j * P.TA + idx) * P.la_floats;
    int part = 0, kc = c;
    if (j >= 1) {
      // order: H chunks first (their first MMA zeroes D_a and D_x), then R, then X
      if (c < nR) part = 2;
      else if (c < 2 * nR) { part = 0; kc = c - nR; }
      else { part = 1; kc = c - 2 * nR; }
    } else {
      if (c < nR) part = 0;
      else { part = 1; kc = c - nR; }
    }
    const float* src;
    if (part == 0) {  // x^(j)_{n-d_j} from layer j's queue, slot (n - d) mod (d + 1)
      const int d = P.dil[j];
      const int64_t slot = ((n - d) % (d + 1) + (d + 1)) % (d + 1);
      src = P.ring + P.ring_off[j] + slot * 2 * actR;
      k.w = wb + (int64_t)kc * 80 * 32;
      k.N = 32;
      k.NS = 80;
    } else if (part == 1) {  // x^(j-1) (j >= 1) or x^(0) (j = 0)
      src = x_now(P, j >= 1 ? j - 1 : 0, n);
      k.w = wb + (int64_t)nR * 80 * 32 + (int64_t)kc * 80 * 32;
      k.N = 32;
      k.NS = 80;
    } else {  // h^(j-1)
      src = P.hb[(j - 1) & 1];
      k.w = wb + (int64_t)2 * nR * 80 * 32 + (int64_t)kc * 96 * 32;
      k.N = 48;
      k.NS = 96;
    }
    k.ah = src + ((int64_t)sb * r + kc * kChunk) * P.r8;
    k.al = k.ah + actR;
    k.dcol = kColA;
    k.acc = c > 0;
  } else if (role == kSkipT) {
    const int j = ph - 1;
    const float* src = P.hb[j & 1];
    k.ah = src + ((int64_t)sb * r + c * kChunk) * P.r8;
    k.al = k.ah + actR;
    k.w = P.pk + P.q_off + ((int64_t)j * P.TQ + idx) * P.q_floats + (int64_t)c * 2 * kTileRows * 32;
    k.N = kTileRows;
    k.NS = 2 * kTileRows;
    k.dcol = kColQ;
    k.acc = (j > 0 || c > 0);
  } else {
    const bool relu = ph == P.L + 1;
    const int C = relu ? P.s : kLevels;
    const float* src = relu ? P.zs : P.za;
    k.ah = src + ((int64_t)sb * C + c * kChunk) * P.r8;
    k.al = k.ah + (int64_t)P.nsb * C * P.r8;
    k.w = P.pk + (relu ? P.hr_off + idx * P.hr_floats : P.ho_off + idx * P.ho_floats) +
          (int64_t)c * 2 * kTileRows * 32;
    k.N = kTileRows;
    k.NS = 2 * kTileRows;
    k.dcol = kColH;
    k.acc = c > 0;
  }
  return k;
}

// Producer (warp 1, one lane): stage every chunk of the job through the ring.
template <bool FAST>
__device__ __forceinline__ bool produce(const BParams& P, Ctl& cl, float* stages, int role, int idx, int sb, int ph,
                                        int64_t n, int nch, uint32_t cseq) {
  for (int c = 0; c < nch; ++c) {
    const uint32_t g = cseq + c, st = g % P.nst, use = g / P.nst;
    if (use > 0 && !mwait(P, cl, &cl.freeb[st], (use - 1) & 1, 42)) return false;
    const Chunk k = job_chunk(P, role, idx, sb, ph, n, c);
    float* sbase = stages + (int64_t)st * stage_floats(P.r8);
    const uint32_t bar = ptx::smem_u32(&cl.full[st]);
    const uint32_t wbytes = (uint32_t)k.NS * kChunk * 4;
    const uint32_t abytes = (uint32_t)P.r8 * kChunk * 4;  // the block's rows only
    ptx::mbar_arm(bar, (FAST ? 1 : 2) * abytes + wbytes);
    bulk_g2s(ptx::smem_u32(sbase), k.ah, abytes, bar);
    if (!FAST) bulk_g2s(ptx::smem_u32(sbase + P.r8 * kChunk), k.al, abytes, bar);
    bulk_g2s(ptx::smem_u32(sbase + 2 * P.r8 * kChunk), k.w, wbytes, bar);
  }
  if (ph == 3) btrace(P, n, 12);
  return true;
}

// MMA issuer (warp 0, one lane): 4 K-steps of 8 per chunk, 3 passes each.
template <bool FAST>
__device__ __forceinline__ bool issue(const BParams& P, Ctl& cl, float* stages, int role, int idx, int sb, int ph,
                                      int64_t n, int nch, uint32_t cseq) {
  for (int c = 0; c < nch; ++c) {
    const uint32_t g = cseq + c, st = g % P.nst, use = g / P.nst;
    if (!mwait(P, cl, &cl.full[st], use & 1, 43)) return false;
    if (c == 0 && ph == 3) btrace(P, n, 13);
    ptx::tmem_fence_after();
    const Chunk k = job_chunk(P, role, idx, sb, ph, n, c);
    const uint32_t a_hi = ptx::smem_u32(stages + (int64_t)st * stage_floats(P.r8));
    const uint32_t a_lo = a_hi + P.r8 * kChunk * 4;
    const uint32_t wb = a_hi + 2 * P.r8 * kChunk * 4;
    const uint32_t id2 = idesc_tf32(k.NS), id1 = idesc_tf32(k.N);
    const uint32_t d = cl.tmem + k.dcol;
#pragma unroll
    for (int ks = 0; ks < kChunk / 8; ++ks) {
      // D[:, 0:NS) += A_hi . [W_hi; (0); W_lo]^T ; D[:, 0:N) += A_lo . W_hi^T (reading R23)
      const uint32_t ao = ks * 2 * P.r8 * 16, bo = ks * 2 * k.NS * 16;
      const uint64_t dah = sdesc(a_hi + ao, P.r8 * 16, 128), dal = sdesc(a_lo + ao, P.r8 * 16, 128);
      const uint64_t db = sdesc(wb + bo, k.NS * 16, 128);
      if constexpr (FAST) {  // DVW_PRECISION_TF32: D[:, 0:N) += A_hi . W_hi^T only
        mma_tf32(d, dah, db, id1, (k.acc || ks > 0) ? 1u : 0u);
      } else {
        mma_tf32(d, dah, db, id2, (k.acc || ks > 0) ? 1u : 0u);
        mma_tf32(d, dal, db, id1, 1u);
      }
    }
    mma_commit(ptx::smem_u32(&cl.freeb[st]));
  }
  if (ph == 3) btrace(P, n, 14);
  mma_commit(ptx::smem_u32(&cl.done));
  return true;
}

__device__ __forceinline__ void st_act(float* base_hi, int64_t half, int c, int i, const float (&v)[4],
                                       bool with_lo, int r8) {
  // 4 consecutive channels c..c+3 (c % 4 == 0) of stream row i < r8; the lo half is not read
  // in the one-pass tf32 mode
  const int o = canon(c, i, r8);
  float4 hi = make_float4(v[0], v[1], v[2], v[3]);
  __stcg(reinterpret_cast<float4*>(base_hi + o), hi);
  if (with_lo) {
    float4 lo = make_float4(tf32_lo(v[0]), tf32_lo(v[1]), tf32_lo(v[2]), tf32_lo(v[3]));
    __stcg(reinterpret_cast<float4*>(base_hi + half + o), lo);
  }
}

// Loads that must be issued where they are written (before a wait), not sunk to
// their first use: volatile asm keeps them ordered with the waits.
__device__ __forceinline__ float4 ld4_early_nc(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld4_early_cg(const float* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

// The draw for one stream by one warp (App. A.4 strategy of RunArgs; direct sampling is the
// cluster kernel's sampler arithmetic: fp32 exp, fp64 running sums in ascending k; R11).
__device__ __forceinline__ int sample_warp_g(const RunArgs& A, const float* logits, float u, int lane) {
  float l[8];
  const float4 a = __ldcg(reinterpret_cast<const float4*>(logits + 8 * lane));
  const float4 b = __ldcg(reinterpret_cast<const float4*>(logits + 8 * lane + 4));
  l[0] = a.x; l[1] = a.y; l[2] = a.z; l[3] = a.w; l[4] = b.x; l[5] = b.y; l[6] = b.z; l[7] = b.w;
  return warp_sample_policy(l, u, A.samp_kind, A.samp_inv_t, A.samp_topk, lane);
}

// x^(0)_{n+1} = W_emb_prev[:, y_{n-1}] + W_emb_cur[:, y_n] + B_emb
// into layer 0's queue slot (n+1) mod (d_0+1) (where phase 0 reads it); one warp, stream g.
__device__ __forceinline__ void embed(const BParams& P, int g, int64_t n1, int yprev, int ycur, int lane) {
  const RunArgs& A = P.a;
  const int r = P.r, sb = g / P.rpb, i = g % P.rpb;
  const int64_t half = (int64_t)P.nsb * r * P.r8;
  const float* ep = A.w + A.off.emb_prev;
  const float* ec = A.w + A.off.emb_cur;
  const float* be = A.w + A.off.b_emb;
  const int d = P.dil[0];
  float* q = P.ring + P.ring_off[0] + (int64_t)(n1 % (d + 1)) * 2 * half + (int64_t)sb * r * P.r8;
  for (int c = lane; c < r; c += 32) {
    const float v = (__ldg(ep + (int64_t)c * kLevels + yprev) + __ldg(ec + (int64_t)c * kLevels + ycur)) + __ldg(be + c);
    const int o = canon(c, i, P.r8);
    __stcg(q + o, v);
    __stcg(q + half + o, tf32_lo(v));
  }
}

template <int NC>
__device__ __forceinline__ void tmem_cols(uint32_t taddr, float (&v)[NC]);
template <>
__device__ __forceinline__ void tmem_cols<8>(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_cols<16>(uint32_t taddr, float (&v)[16]) {
  ptx::tmem_ld16(taddr, v);
}

// Epilogue inputs that do not depend on the MMA: issued before waiting for it.
struct Pre {
  float L[16];  // conditioning: 8 tanh + 8 sigmoid channels
  float b[16];  // folded gate bias, same channels
  float x[8];   // x^(j-1) for the residual update
  float br[8];  // B_res^(j-1)
};

__device__ __forceinline__ void prefetch(const BParams& P, int role, int idx, int sb, int ph, int64_t n, Pre& pre) {
  const RunArgs& A = P.a;
  if (role != kLayer || ph >= P.L) return;
  const int t = threadIdx.x, i = t & 127, half = t >> 7;
  const int g = sb * P.rpb + i, r = P.r, j = ph;
  const int c0 = 16 * idx + 8 * half;
  const float* bias = P.pk + P.bias_off + (int64_t)j * 2 * r;
  float* bv = pre.b;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const float4 a = ld4_early_nc(bias + c0 + 4 * q), b = ld4_early_nc(bias + r + c0 + 4 * q);
    bv[4 * q] = a.x; bv[4 * q + 1] = a.y; bv[4 * q + 2] = a.z; bv[4 * q + 3] = a.w;
    bv[8 + 4 * q] = b.x; bv[8 + 4 * q + 1] = b.y; bv[8 + 4 * q + 2] = b.z; bv[8 + 4 * q + 3] = b.w;
  }
  if (i < P.rpb && g < A.n_streams) {
    const float* cp = A.cond + (((int64_t)g * A.n_frames + n / A.hop) * P.L + j) * 2 * r;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float4 a = ld4_early_nc(cp + c0 + 4 * q);
      const float4 b = ld4_early_nc(cp + r + c0 + 4 * q);
      pre.L[4 * q] = a.x; pre.L[4 * q + 1] = a.y; pre.L[4 * q + 2] = a.z; pre.L[4 * q + 3] = a.w;
      pre.L[8 + 4 * q] = b.x; pre.L[8 + 4 * q + 1] = b.y; pre.L[8 + 4 * q + 2] = b.z; pre.L[8 + 4 * q + 3] = b.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 16; ++q) pre.L[q] = 0.0f;
  }
  if (j >= 1) {
    const float* xin = x_now(P, j - 1, n) + (int64_t)sb * r * P.r8;
    const float* bres = A.w + A.off.b_res + (int64_t)(j - 1) * A.off.layer_stride + c0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float4 v = ld4_early_cg(xin + canon(c0 + 4 * q, i < P.r8 ? i : 0, P.r8));
      const float4 bb = ld4_early_nc(bres + 4 * q);
      pre.x[4 * q] = v.x; pre.x[4 * q + 1] = v.y; pre.x[4 * q + 2] = v.z; pre.x[4 * q + 3] = v.w;
      pre.br[4 * q] = bb.x; pre.br[4 * q + 1] = bb.y; pre.br[4 * q + 2] = bb.z; pre.br[4 * q + 3] = bb.w;
    }
  }
}

// Thread t: stream row i = t % 128 (its TMEM lane), column half t / 128 of the tile.
template <bool FAST>
__device__ void epilogue(const BParams& P, Ctl& cl, int role, int idx, int sb, int ph, int64_t n, const Pre& pre) {
  const RunArgs& A = P.a;
  const int t = threadIdx.x, w = t >> 5, i = t & 127, half = t >> 7;
  const int g = sb * P.rpb + i;
  const bool live = i < P.rpb && g < A.n_streams;
  const bool row = i < P.r8;  // a row of the block's image (padding rows past rpb are stored too)
  const uint32_t lane_base = cl.tmem + ((uint32_t)(32 * (w & 3)) << 16);
  const int r = P.r;
  if (t == 0 && ph == 3) btrace(P, n, 19);
  __syncwarp();  // tcgen05.ld is warp-collective
  if (t == 0 && ph == 3) btrace(P, n, 15);
  if (role == kLayer) {
    const int j = ph, c0 = 16 * idx + 8 * half;
    float Dt[8], Ds[8], Dx[8] = {}, Et[8], Es[8], Ex[8] = {};
    tmem_cols<8>(lane_base + kColA + 8 * half, Dt);
    tmem_cols<8>(lane_base + kColA + 16 + 8 * half, Ds);
    tmem_cols<8>(lane_base + kColA2 + 8 * half, Et);
    tmem_cols<8>(lane_base + kColA2 + 16 + 8 * half, Es);
    if (j >= 1) {
      tmem_cols<8>(lane_base + kColA + 32 + 8 * half, Dx);
      tmem_cols<8>(lane_base + kColA2 + 32 + 8 * half, Ex);
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("" : "+f"(Dt[q]), "+f"(Ds[q]), "+f"(Dx[q]), "+f"(Et[q]), "+f"(Es[q]), "+f"(Ex[q]));
    if constexpr (FAST) {  // the hi*lo partner columns were not written this phase
#pragma unroll
      for (int q = 0; q < 8; ++q) Et[q] = Es[q] = Ex[q] = 0.0f;
    }
    if (t == 0 && ph == 3) btrace(P, n, 16);
    const int64_t half_f = (int64_t)P.nsb * r * P.r8;
    float* hdst = P.hb[j & 1] + (int64_t)sb * r * P.r8;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float hv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = 4 * q + e;
        hv[e] = gate_fast(((Dt[c] + Et[c]) + pre.b[c]) + pre.L[c], ((Ds[c] + Es[c]) + pre.b[8 + c]) + pre.L[8 + c]);
      }
      if (row) st_act(hdst, half_f, c0 + 4 * q, i, hv, !FAST, P.r8);
    }
    if (t == 0 && ph == 3) btrace(P, n, 17);
    if (j >= 1) {
      const int d = P.dil[j];
      float* qd = P.ring + P.ring_off[j] + (int64_t)(n % (d + 1)) * 2 * half_f + (int64_t)sb * r * P.r8;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float xv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) xv[e] = pre.x[4 * q + e] + ((Dx[4 * q + e] + Ex[4 * q + e]) + pre.br[4 * q + e]);
        if (row) st_act(qd, half_f, c0 + 4 * q, i, xv, !FAST, P.r8);
      }
    }
  } else {
    if (role == kSkipT && ph != P.L) return;  // accumulation continues in TMEM
    // 64-row tile: thread (stream i, half) finishes rows [64 idx + 32 half, +32)
    float D[32], E[32];
    const uint32_t c0t = kColQ + 32 * half, c1t = kColQ2 + 32 * half;  // kColQ == kColH
    tmem_cols<16>(lane_base + c0t, *reinterpret_cast<float(*)[16]>(D));
    tmem_cols<16>(lane_base + c0t + 16, *reinterpret_cast<float(*)[16]>(D + 16));
    tmem_cols<16>(lane_base + c1t, *reinterpret_cast<float(*)[16]>(E));
    tmem_cols<16>(lane_base + c1t + 16, *reinterpret_cast<float(*)[16]>(E + 16));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 32; ++q) asm volatile("" : "+f"(D[q]), "+f"(E[q]));
    if constexpr (!FAST) {
#pragma unroll
      for (int q = 0; q < 32; ++q) D[q] += E[q];
    }
    const int c0 = kTileRows * idx + 32 * half;
    if (role == kSkipT) {  // z_s = relu(q + B_skip)
      const float* bsk = A.w + A.off.b_skip + c0;
      const int64_t half_f = (int64_t)P.nsb * P.s * P.r8;
      float* dst = P.zs + (int64_t)sb * P.s * P.r8;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = fmaxf(D[4 * q + e] + __ldg(bsk + 4 * q + e), 0.0f);
        if (row) st_act(dst, half_f, c0 + 4 * q, i, v, !FAST, P.r8);
      }
    } else if (ph == P.L + 1) {  // z_a = relu(W_relu z_s + B_relu)
      const float* bb = A.w + A.off.b_relu + c0;
      const int64_t half_f = (int64_t)P.nsb * kLevels * P.r8;
      float* dst = P.za + (int64_t)sb * kLevels * P.r8;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = fmaxf(D[4 * q + e] + __ldg(bb + 4 * q + e), 0.0f);
        if (row) st_act(dst, half_f, c0 + 4 * q, i, v, !FAST, P.r8);
      }
    } else {  // logits = W_out z_a + B_out
      const float* bb = A.w + A.off.b_out + c0;
      float* lg = P.logits + (int64_t)g * kLevels + c0;
      float* ol = (A.forced && live) ? A.out_logits + ((int64_t)g * A.N + (n - A.n0)) * kLevels + c0 : nullptr;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 v = make_float4(D[4 * q] + __ldg(bb + 4 * q), D[4 * q + 1] + __ldg(bb + 4 * q + 1),
                               D[4 * q + 2] + __ldg(bb + 4 * q + 2), D[4 * q + 3] + __ldg(bb + 4 * q + 3));
        if (i < P.rpb) __stcg(reinterpret_cast<float4*>(lg) + q, v);
        if (ol) reinterpret_cast<float4*>(ol)[q] = v;
      }
    }
  }
}

template <bool FAST>
__global__ void __launch_bounds__(kBT, 1) k_batch(const __grid_constant__ BParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Ctl& cl = *reinterpret_cast<Ctl*>(smem_raw);
  static_assert(sizeof(Ctl) <= kCtlBytes, "Ctl");
  float* stages = reinterpret_cast<float*>(smem_raw + kCtlBytes);
  const RunArgs& A = P.a;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int b = blockIdx.x;
  const int sb = b / P.per_sb, k = b % P.per_sb;
  int role, idx;
  if (k < P.TA) { role = kLayer; idx = k; }
  else if (k < P.TA + P.TQ) { role = kSkipT; idx = k - P.TA; }
  else { role = kHeadT; idx = k - P.TA - P.TQ; }

  if (w == 0) ptx::tmem_alloc(ptx::smem_u32(&cl.tmem), kTmemCols);
  if (t == 0) {
    cl.abort = 0;
    for (int s = 0; s < kMaxStages; ++s) {
      ptx::mbar_init(ptx::smem_u32(&cl.full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&cl.freeb[s]), 1);
    }
    ptx::mbar_init(ptx::smem_u32(&cl.done), 1);
    ptx::fence_mbar_init();
  }
  ptx::tmem_fence_before();
  __syncthreads();
  ptx::tmem_fence_after();

  uint32_t cseq = 0, jseq = 0;
  // the warps of this cluster serve the streams of its stream block (sampler, embedding)
  const int nwarps = P.per_sb * (kBT / 32);
  const int gw = k * (kBT / 32) + w;
  const int g_end = min(A.n_streams, (sb + 1) * P.rpb);

  // x^(0)_0 from y_{-1} = y_{-2} = 128 (R4).  A streaming session (n0 > 0) continues from
  // the queues, x^(0)_{n0} and the code history its previous call left in the workspace.
  if (A.n0 == 0) {
    for (int g = sb * P.rpb + gw; g < g_end; g += nwarps) {
      embed(P, g, 0, kLevels / 2, kLevels / 2, lane);
      if (lane == 0) {
        P.yh[2 * g] = kLevels / 2;
        P.yh[2 * g + 1] = kLevels / 2;
      }
    }
  }
  phase_sync(P, cl);
  // A CTA whose pipeline failed (watchdog) stops working but keeps passing every cluster
  // barrier, so the other CTAs of its stream block never wait forever; the host sees the
  // error word.
  bool ok = true;

  // n: the global sample index (queue slots, conditioning frames); n - n0 indexes this call's
  // uniforms, codes and logits
  for (int64_t n = A.n0; n < A.n0 + A.N; ++n) {
    const int64_t nl = n - A.n0;
    for (int ph = 0; ph < P.L + 4; ++ph) {
      const int tev = ph == 3 ? 0 : ph == P.L + 2 ? 8 : ph == P.L + 3 ? 4 : -1;
      if (t == 0 && tev >= 0) btrace(P, n, tev);
      if (ph < P.L + 3) {
        const int nch = ok ? job_chunks(P, role, ph) : 0;
        if (nch > 0) {
          bool good = true;
          if (t == 32) good = produce<FAST>(P, cl, stages, role, idx, sb, ph, n, nch, cseq);
          else if (t == 0) good = issue<FAST>(P, cl, stages, role, idx, sb, ph, n, nch, cseq);
          if (!good) cl.abort = 1;
          __syncwarp();
          Pre pre;
          prefetch(P, role, idx, sb, ph, n, pre);
          bool dn = true;
          if (lane == 0) dn = mwait(P, cl, &cl.done, jseq & 1, 44);
          dn = __shfl_sync(0xffffffffu, dn ? 1 : 0, 0) != 0;
          if (dn) {
            if (t == 0 && tev >= 0) btrace(P, n, tev + 1);
            ptx::tmem_fence_after();
            if (t == 0 && ph == 3) btrace(P, n, 18);
            epilogue<FAST>(P, cl, role, idx, sb, ph, n, pre);
            if (t == 0 && tev >= 0) btrace(P, n, tev + 2);
          }
          ptx::tmem_fence_before();
          cseq += nch;
          ++jseq;
        }
      } else if (ok) {
        // sample y_n and embed x^(0)_{n+1}; one warp per stream
        for (int g = sb * P.rpb + gw; g < g_end; g += nwarps) {
          const int y1 = __ldcg(P.yh + 2 * g);
          int y;
          if (A.forced) {
            y = __ldg(A.forced + (int64_t)g * A.N + nl);
          } else {
            y = sample_warp_g(A, P.logits + (int64_t)g * kLevels, __ldg(A.uniforms + (int64_t)g * A.N + nl), lane);
            if (lane == 0) A.out_codes[(int64_t)g * A.N + nl] = (uint8_t)y;
          }
          // x^(0)_{n+1}, also after the call's last sample (a session's next call starts from it)
          embed(P, g, n + 1, y1, y, lane);
          __syncwarp();
          if (lane == 0) {
            __stcg(P.yh + 2 * g, y);
            __stcg(P.yh + 2 * g + 1, y1);
          }
        }
      }
      if (t == 0 && ph == P.L + 3) btrace(P, n, 5);
      __syncthreads();
      ok = ok && !cl.abort;
      phase_sync(P, cl);
      if (t == 0 && tev >= 0) btrace(P, n, tev == 4 ? 6 : tev + 3);
    }
  }
  ptx::tmem_fence_before();
  __syncthreads();
  ptx::tmem_fence_after();
  if (w == 0) ptx::tmem_dealloc(cl.tmem, kTmemCols);
}

inline float tf32_lo_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  float h;
  std::memcpy(&h, &u, 4);
  return x - h;
}

}  // namespace

BatchPlan plan_batch(int L, int r, int s, int device) {
  BatchPlan p;
  p.L = L;
  p.r = r;
  p.s = s;
  if (L > kBMaxLayers) { p.why = "more than 64 layers"; return p; }
  if (r % kChunk != 0 || r > 128) { p.why = "residual channels must be 32, 64 or 128"; return p; }
  if (s % kTileRows != 0) { p.why = "skip channels must be a multiple of 64"; return p; }
  p.TA = r / 16;
  p.TQ = s / kTileRows;
  p.TH = kLevels / kTileRows;
  p.per_sb = p.TA + p.TQ + p.TH;  // one cluster per stream block
  if (p.per_sb > 16) { p.why = "a stream block needs more than 16 CTAs"; return p; }
  const int nR = r / kChunk;
  int64_t off = 0;
  p.la_off = off;
  p.la_floats = (int64_t)nR * (80 * 32 + 80 * 32 + 96 * 32);
  off += (int64_t)L * p.TA * p.la_floats;
  p.q_off = off;
  p.q_floats = (int64_t)nR * 2 * kTileRows * 32;
  off += (int64_t)L * p.TQ * p.q_floats;
  p.hr_off = off;
  p.hr_floats = (int64_t)(s / kChunk) * 2 * kTileRows * 32;
  off += (int64_t)p.TH * p.hr_floats;
  p.ho_off = off;
  p.ho_floats = (int64_t)(kLevels / kChunk) * 2 * kTileRows * 32;
  off += (int64_t)p.TH * p.ho_floats;
  p.bias_off = off;
  off += (int64_t)L * 2 * r;
  p.total = off;
  p.smem_bytes = kSmemBytes;
  // stream blocks per launch = clusters that are co-resident (one wave)
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaError_t e = cudaSuccess;
  for (auto fn : {k_batch<false>, k_batch<true>}) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_bytes);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  int ncl = 0;
  if (e == cudaSuccess) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.per_sb);
    cfg.blockDim = dim3(kBT);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.per_sb;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaOccupancyMaxActiveClusters(&ncl, k_batch<false>, &cfg);
  }
  if (prev >= 0) cudaSetDevice(prev);
  if (e != cudaSuccess || ncl < 1) {
    cudaGetLastError();
    p.why = "a stream-block cluster cannot be scheduled on this device";
    return p;
  }
  p.max_sb = ncl;
  p.ok = true;
  p.why = "ok";
  return p;
}

cudaError_t pack_batch_weights(const BatchPlan& p, const float* w, const Offsets& o, void* packed) {
  const int L = p.L, r = p.r, s = p.s, nR = r / kChunk;
  std::vector<float> pk((size_t)p.total, 0.0f);
  // One K-chunk block of a B operand in the K-major core-matrix order [8][NS][4]:
  // rows [0, N) = the weight rows (hi: fp32 value), rows [lo0, lo0 + N) = their tf32
  // residuals, other rows zero (the kernel's stacked-B pass, reading R23).
  auto put_block = [&](float* dst, int N, int NS, const std::vector<float>& rows /* N x 32 */) {
    const int lo0 = NS - N;
    for (int rr = 0; rr < N; ++rr)
      for (int kk = 0; kk < kChunk; ++kk) {
        const float v = rows[(size_t)rr * kChunk + kk];
        dst[((size_t)(kk >> 2) * NS + rr) * 4 + (kk & 3)] = v;
        dst[((size_t)(kk >> 2) * NS + lo0 + rr) * 4 + (kk & 3)] = tf32_lo_host(v);
      }
  };
  auto W = [&](int j, int64_t base, int row, int col, int ncol) -> float {
    return w[(int64_t)j * o.layer_stride + base + (int64_t)row * ncol + col];
  };
  std::vector<double> M((size_t)2 * r * r);
  std::vector<float> rows;
  for (int j = 0; j < L; ++j) {
    if (j >= 1) {  // M^(j) = W_cur^(j) W_res^(j-1) in fp64, rounded once
      for (int a = 0; a < 2 * r; ++a)
        for (int c = 0; c < r; ++c) {
          double acc = 0.0;
          for (int k = 0; k < r; ++k) acc += (double)W(j, o.w_cur, a, k, r) * (double)W(j - 1, o.w_res, k, c, r);
          M[(size_t)a * r + c] = acc;
        }
    }
    // folded bias B^(j) + W_cur^(j) B_res^(j-1)
    for (int a = 0; a < 2 * r; ++a) {
      double acc = (double)w[(int64_t)j * o.layer_stride + o.b + a];
      if (j >= 1)
        for (int k = 0; k < r; ++k)
          acc += (double)W(j, o.w_cur, a, k, r) * (double)w[(int64_t)(j - 1) * o.layer_stride + o.b_res + k];
      pk[(size_t)p.bias_off + (size_t)j * 2 * r + a] = (float)acc;
    }
    for (int t = 0; t < p.TA; ++t) {
      float* blk = pk.data() + p.la_off + ((int64_t)j * p.TA + t) * p.la_floats;
      auto arow = [&](int rho) { return rho < 16 ? 16 * t + rho : r + 16 * t + rho - 16; };
      for (int kc = 0; kc < nR; ++kc) {
        rows.assign(32 * kChunk, 0.0f);
        for (int rho = 0; rho < 32; ++rho)
          for (int kk = 0; kk < kChunk; ++kk) rows[rho * kChunk + kk] = W(j, o.w_prev, arow(rho), 32 * kc + kk, r);
        put_block(blk + (int64_t)kc * 80 * 32, 32, 80, rows);
        for (int rho = 0; rho < 32; ++rho)
          for (int kk = 0; kk < kChunk; ++kk) rows[rho * kChunk + kk] = W(j, o.w_cur, arow(rho), 32 * kc + kk, r);
        put_block(blk + (int64_t)nR * 80 * 32 + (int64_t)kc * 80 * 32, 32, 80, rows);
        if (j >= 1) {
          rows.assign(48 * kChunk, 0.0f);
          for (int rho = 0; rho < 48; ++rho)
            for (int kk = 0; kk < kChunk; ++kk)
              rows[rho * kChunk + kk] = rho < 32 ? (float)M[(size_t)arow(rho) * r + 32 * kc + kk]
                                                 : W(j - 1, o.w_res, 16 * t + rho - 32, 32 * kc + kk, r);
          put_block(blk + (int64_t)2 * nR * 80 * 32 + (int64_t)kc * 96 * 32, 48, 96, rows);
        }
      }
    }
    for (int u = 0; u < p.TQ; ++u) {
      float* blk = pk.data() + p.q_off + ((int64_t)j * p.TQ + u) * p.q_floats;
      for (int kc = 0; kc < nR; ++kc) {
        rows.assign(kTileRows * kChunk, 0.0f);
        for (int rho = 0; rho < kTileRows; ++rho)
          for (int kk = 0; kk < kChunk; ++kk)
            rows[rho * kChunk + kk] = W(j, o.w_skip, kTileRows * u + rho, 32 * kc + kk, r);
        put_block(blk + (int64_t)kc * 2 * kTileRows * 32, kTileRows, 2 * kTileRows, rows);
      }
    }
  }
  for (int v = 0; v < p.TH; ++v) {
    for (int kc = 0; kc < s / kChunk; ++kc) {
      rows.assign(kTileRows * kChunk, 0.0f);
      for (int rho = 0; rho < kTileRows; ++rho)
        for (int kk = 0; kk < kChunk; ++kk)
          rows[rho * kChunk + kk] = w[o.w_relu + (int64_t)(kTileRows * v + rho) * s + 32 * kc + kk];
      put_block(pk.data() + p.hr_off + v * p.hr_floats + (int64_t)kc * 2 * kTileRows * 32, kTileRows, 2 * kTileRows,
                rows);
    }
    for (int kc = 0; kc < kLevels / kChunk; ++kc) {
      rows.assign(kTileRows * kChunk, 0.0f);
      for (int rho = 0; rho < kTileRows; ++rho)
        for (int kk = 0; kk < kChunk; ++kk)
          rows[rho * kChunk + kk] = w[o.w_out + (int64_t)(kTileRows * v + rho) * kLevels + 32 * kc + kk];
      put_block(pk.data() + p.ho_off + v * p.ho_floats + (int64_t)kc * 2 * kTileRows * 32, kTileRows, 2 * kTileRows,
                rows);
    }
  }
  return cudaMemcpy(packed, pk.data(), sizeof(float) * pk.size(), cudaMemcpyHostToDevice);
}

namespace {
struct WsLayout {
  int64_t hb[2], zs, za, logits, ring, yh, abort, total;  // byte offsets
  int64_t ring_off[kBMaxLayers];                                 // floats from ring
};
WsLayout ws_layout(const BatchPlan& p, const int32_t* dil, int nsb, int rpb) {
  WsLayout l{};
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t o = off;
    off += (bytes + 255) & ~int64_t(255);
    return o;
  };
  const int r8 = (rpb + 7) & ~7;
  const int64_t act = (int64_t)2 * nsb * p.r * r8 * 4;
  l.hb[0] = take(act);
  l.hb[1] = take(act);
  l.zs = take((int64_t)2 * nsb * p.s * r8 * 4);
  l.za = take((int64_t)2 * nsb * kLevels * r8 * 4);
  l.logits = take((int64_t)nsb * rpb * kLevels * 4);
  l.yh = take((int64_t)nsb * rpb * 2 * 4);
  l.abort = take((int64_t)nsb * 4);
  int64_t rf = 0;
  for (int j = 0; j < p.L; ++j) {
    l.ring_off[j] = rf;
    rf += (int64_t)(dil[j] + 1) * 2 * nsb * p.r * r8;
  }
  l.ring = take(rf * 4);
  l.total = off;
  return l;
}
}  // namespace

// Launch groups of a batch (the same for every call with this n_streams, so a session's per-group
// workspace stays valid): as few groups as co-resident clusters allow, the streams spread evenly
// over up to max_sb stream blocks per group (fewer rows per block, more clusters busy).
BatchGrouping batch_grouping(const BatchPlan& p, int n_streams) {
  BatchGrouping g;
  const int cap = p.max_sb * 128;
  g.groups = (n_streams + cap - 1) / cap;
  g.per_group = (n_streams + g.groups - 1) / g.groups;
  g.nsb = std::min(p.max_sb, g.per_group);
  g.rpb = (g.per_group + g.nsb - 1) / g.nsb;
  // A/B switch: DVW_BATCH_BALANCE=0 packs full 128-stream blocks (round 1)
  if (const char* e = std::getenv("DVW_BATCH_BALANCE"))
    if (std::atoi(e) == 0) {
      g.per_group = std::min(cap, n_streams);
      g.rpb = 128;
    }
  g.nsb = (g.per_group + g.rpb - 1) / g.rpb;
  return g;
}

size_t batch_workspace_bytes(const BatchPlan& p, const int32_t* dil, int n_streams) {
  const BatchGrouping g = batch_grouping(p, n_streams);
  return (size_t)ws_layout(p, dil, g.nsb, g.rpb).total;
}

size_t batch_session_bytes(const BatchPlan& p, const int32_t* dil, int n_streams) {
  const BatchGrouping g = batch_grouping(p, n_streams);
  return (size_t)g.groups * (size_t)ws_layout(p, dil, g.nsb, g.rpb).total;
}

cudaError_t launch_batch_kernel(const RunArgs& a, const BatchPlan& p, const void* packed, void* ws, size_t ws_bytes,
                                const int32_t* dil_host, bool fast, cudaStream_t st, LaunchInfo* info,
                                bool session) {
  if (!p.ok) return cudaErrorNotSupported;
  // (plan_batch set the kernel's shared-memory and cluster-size attributes)
  const BatchGrouping gr = batch_grouping(p, a.n_streams);
  const WsLayout l = ws_layout(p, dil_host, gr.nsb, gr.rpb);
  int64_t launches = 0;
  int grid = 0;
  size_t wsoff = 0;  // a session keeps every launch group's workspace (queues, x^(0), codes)
  for (int g0 = 0; g0 < a.n_streams; g0 += gr.per_group) {
    const int ns = std::min(gr.per_group, a.n_streams - g0);
    const int nsb = (ns + gr.rpb - 1) / gr.rpb;
    if (wsoff + (size_t)l.total > ws_bytes) return cudaErrorInvalidValue;
    char* gws = static_cast<char*>(ws) + wsoff;
    if (session) wsoff += (size_t)l.total;
    cudaError_t e = cudaSuccess;
    if (!session || a.n0 == 0) e = cudaMemsetAsync(gws, 0, (size_t)l.total, st);
    if (e != cudaSuccess) return e;
    BParams P{};
    P.a = a;
    P.a.n_streams = ns;
    P.a.cond = a.cond + (int64_t)g0 * a.n_frames * a.L * 2 * a.r;
    if (a.uniforms) P.a.uniforms = a.uniforms + (int64_t)g0 * a.N;
    if (a.forced) P.a.forced = a.forced + (int64_t)g0 * a.N;
    if (a.out_codes) P.a.out_codes = a.out_codes + (int64_t)g0 * a.N;
    if (a.out_logits) P.a.out_logits = a.out_logits + (int64_t)g0 * a.N * kLevels;
    P.pk = static_cast<const float*>(packed);
    P.L = p.L; P.r = p.r; P.s = p.s;
    P.TA = p.TA; P.TQ = p.TQ; P.TH = p.TH; P.per_sb = p.per_sb;
    P.nsb = gr.nsb;  // image layout (the workspace holds gr.nsb blocks; this group runs nsb of them)
    P.rpb = gr.rpb;
    P.r8 = (gr.rpb + 7) & ~7;
    P.nst = std::min(kMaxStages, (p.smem_bytes - kCtlBytes) / (stage_floats(P.r8) * 4));
    // a deeper ring measured slower (C4 at 37 streams per block, 7 stages: 1.14 M vs 1.26 M samples/s):
    // 4 stages unless DVW_BATCH_STAGES says otherwise (A/B)
    {
      const char* e = std::getenv("DVW_BATCH_STAGES");
      P.nst = std::min(P.nst, e ? std::max(2, std::atoi(e)) : 4);
    }

    P.la_off = p.la_off; P.la_floats = p.la_floats;
    P.q_off = p.q_off; P.q_floats = p.q_floats;
    P.hr_off = p.hr_off; P.hr_floats = p.hr_floats;
    P.ho_off = p.ho_off; P.ho_floats = p.ho_floats;
    P.bias_off = p.bias_off;
    char* base = gws;
    for (int q = 0; q < 2; ++q) {
      P.hb[q] = reinterpret_cast<float*>(base + l.hb[q]);
    }
    P.zs = reinterpret_cast<float*>(base + l.zs);
    P.za = reinterpret_cast<float*>(base + l.za);
    P.logits = reinterpret_cast<float*>(base + l.logits);
    P.ring = reinterpret_cast<float*>(base + l.ring);
    P.yh = reinterpret_cast<int*>(base + l.yh);
    P.abort_flag = reinterpret_cast<int*>(base + l.abort);
    for (int j = 0; j < p.L; ++j) {
      P.dil[j] = dil_host[j];
      P.ring_off[j] = l.ring_off[j];
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nsb * p.per_sb);  // one cluster of per_sb CTAs per stream block
    cfg.blockDim = dim3(kBT);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.per_sb;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = fast ? cudaLaunchKernelEx(&cfg, k_batch<true>, P) : cudaLaunchKernelEx(&cfg, k_batch<false>, P);
    if (e != cudaSuccess) return e;
    ++launches;
    grid = std::max(grid, nsb * p.per_sb);
  }
  info->grid = grid;
  info->cluster = p.per_sb;
  info->threads = kBT;
  info->launches = launches;
  info->rows_per_block = gr.rpb;
  return cudaSuccess;
}

}  // namespace dvw
