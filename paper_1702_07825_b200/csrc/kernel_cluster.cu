// kernel_cluster.cu -- batch-1 persistent cluster kernel (r = 64, s in {128, 256}).
//
// The paper's GPU kernel (App. D) put two layers per SM in
// registers and passed each sample round-robin through 23 SMs with spin-locks in
// L2.  This kernel keeps the idea "one launch, weights on chip" and redesigns the
// rest for sm_100a:
//   * one thread-block cluster; every hand-off is a DSMEM st.async whose
//     transaction bytes complete on the receiver's mbarrier (no L2 round trip);
//   * the critical chain (steps 2b-2c + residual) holds W_cur
//     and W_res in registers (192 per thread, setmaxnreg 232) four layers per SM;
//   * everything off the chain runs concurrently elsewhere: W_prev x_{n+1-d} for
//     the next sample (Fig. 2's "aux threads") in a dedicated
//     warpgroup of each chain CTA, the skip projections in
//     skip CTAs, the ring buffers in L2;
//   * the head is split by output rows over 4 CTAs, and CTA 0
//     samples (App. A.4) and embeds the next input (step 1).
// Numerics: fp32 FMA everywhere, accurate tanhf/expf, fp64 CDF scan (R11-R13);
// every reduction has a fixed order, so results are bitwise deterministic.
#include <algorithm>
#include <cstring>
#include <vector>

#include "kernel_cluster.cuh"
#include "ptx.cuh"

namespace dvw {
namespace {

constexpr int R = 64;       // residual channels the kernel is built for
constexpr int LPC = 4;      // layers per chain CTA
constexpr int NH = 4;       // head CTAs (64 output rows each)
constexpr int kMain = 256;  // warps 0-7: chain / head / skip math
constexpr int kAux = 128;   // warps 8-11: off-chain work of chain CTAs
constexpr int kThreads = kMain + kAux;
constexpr int kMainRegs = 232;
constexpr int kAuxRegs = 40;  // 8 warps x 232 + 4 warps x 40 = 384 x 168 (the launch allocation)
constexpr int kChainRegs = LPC * 48;  // W_cur (2 rows x 16) + W_res (16) per layer
constexpr uint64_t kTimeoutNs = 2000000000ull;

enum Role { kChain = 0, kHead = 1, kSkip = 2, kIdle = 3 };

struct __align__(16) Mail {
  uint64_t bar_xin, bar_logits, bar_pre, bar_done, bar_part, bar_za;
  uint64_t bar_h[kCMaxSlot];
  int abort_flag;
  int pad_[3];
  float xs[LPC + 1][R];       // chain: layer inputs; xs[0] is the inbound x
  float xsave[LPC][R];        // chain: x^(j-1)_n for the aux warpgroup (ring + a_prev)
  float pre[LPC][2 * R];      // chain: W_prev x_{n-d} + B + L for the coming sample
  float xp[R];                // chain aux scratch
  float hs[R];                // chain: h exchange inside the CTA
  float logits_in[kLevels];   // CTA 0: inbound logits
  float hbuf[kCMaxSlot][R];   // skip: h^(j) per owned slot; head: slot 0 = h^(l)
  float part[kCMaxSkip][256]; // head: skip partials
  float za_in[kLevels];       // head: all-gathered z_a
  float zs[256];              // head: z_s; skip: partial staging
  double dscr[8];
  float fscr[8];
  int iscr[16];
};

struct Params {
  RunArgs a;
  ClusterPlan p;
  const float* pk;
};

struct Ctx {
  Mail* mail;
  int* err;
  int size;
};

__device__ __forceinline__ void raise_abort(const Ctx& cx, int code) {
  *reinterpret_cast<volatile int*>(cx.err) = code;  // mapped host memory
  __threadfence_system();
  const uint32_t a = ptx::smem_u32(&cx.mail->abort_flag);
  for (int r = 0; r < cx.size; ++r) {
    const uint32_t ra = ptx::mapa(a, r);
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(1) : "memory");
  }
}

// Wait for phase `parity` of a local mbarrier; on the watchdog (2 s without
// progress) or a cluster-wide abort, return false and let the caller run on
// without blocking so every CTA reaches the final cluster barrier.
__device__ __forceinline__ bool wait(const Ctx& cx, uint64_t* bar, uint32_t parity, int code) {
  const uint32_t b = ptx::smem_u32(bar);
  if (ptx::mbar_try_wait(b, parity)) return true;
  const uint64_t t0 = ptx::globaltimer();
  for (uint32_t i = 1;; ++i) {
    if (ptx::mbar_try_wait(b, parity)) return true;
    if ((i & 7) == 0) {
      if (*reinterpret_cast<volatile int*>(&cx.mail->abort_flag)) return false;
      if (ptx::globaltimer() - t0 > kTimeoutNs) {
        raise_abort(cx, code);
        return false;
      }
    }
  }
}

__device__ __forceinline__ uint32_t remote(const void* local, int rank) {
  return ptx::mapa(ptx::smem_u32(local), (uint32_t)rank);
}

// Optional per-event %globaltimer stamps (dvw_set_trace); one predicated branch when off.
__device__ __forceinline__ void trace(const RunArgs& A, int64_t n, int ev) {
  if (A.trace) {
    const int64_t i = n - A.trace_n0;
    if (i >= 0 && i < A.trace_count) A.trace[(i * kCMaxCta + ptx::cluster_rank()) * 32 + ev] = ptx::globaltimer();
  }
}

// Same, but the SM-local cycle counter (cheap; for events inside one CTA).
__device__ __forceinline__ void trace_clk(const RunArgs& A, int64_t n, int ev) {
  if (A.trace) {
    const int64_t i = n - A.trace_n0;
    if (i >= 0 && i < A.trace_count) A.trace[(i * kCMaxCta + ptx::cluster_rank()) * 32 + ev] = clock64();
  }
}

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// ------------------------------------------------------------------ chain CTA, main warps
template <int S>
__device__ void chain_main(const Params& P, const Ctx& cx, int c, const float* blk, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int t = threadIdx.x;
  const int pr = t >> 2, ch = t & 3;  // row pair (i, i + r) and 16-column chunk
  const int first = pl.chain_first[c], nl = pl.chain_nl[c];
  const bool last_cta = (c == pl.nc - 1);

  float wc[LPC][32], wr[LPC][16];
#pragma unroll
  for (int jl = 0; jl < LPC; ++jl) {
#pragma unroll
    for (int q = 0; q < 32; ++q) wc[jl][q] = blk[(jl * 48 + q) * kMain + t];
#pragma unroll
    for (int q = 0; q < 16; ++q) wr[jl][q] = blk[(jl * 48 + 32 + q) * kMain + t];
  }
  const float* bres = sw + LPC * R * 2 * R + LPC * 2 * R;  // [LPC][R]
  const float* wembc = bres + LPC * R;                     // CTA 0: [256][R]
  const float* bemb = wembc + kLevels * R;                 // CTA 0: [R]
  const float* embp_g = P.pk + pl.embp_off;                // [256][R] in global

  const float* uni = A.uniforms;
  const uint8_t* forced = A.forced;
  int y1 = kLevels / 2, y2 = kLevels / 2;

  for (int64_t n = 0; n < A.N; ++n) {
    if (c == 0) {
      float ep = 0.0f;
      if (n > 0) {
        const float u = uni ? __ldg(uni + n - 1) : 0.0f;
        const int yf = forced ? (int)__ldg(forced + n - 1) : 0;
        if (t < R) ep = __ldg(embp_g + y1 * R + t);  // W_emb_prev[:, y_{n-2}] (y1 before the update)
        if (wait(cx, &m.bar_logits, (uint32_t)((n - 1) & 1), 11) && t == 0)
          ptx::mbar_arm(ptx::smem_u32(&m.bar_logits), kLevels * 4);
        if (t == 0) trace(A, n - 1, 3);
        const float l = m.logits_in[t];
        int y;
        if (forced) {
          A.out_logits[(n - 1) * kLevels + t] = l;
          y = yf;
        } else {
          y = sample_256(l, u, m.dscr, m.fscr, m.iscr, t, 1);
          if (t == 0) A.out_codes[n - 1] = (uint8_t)y;
        }
        y2 = y1;
        y1 = y;
      } else {
        if (t < R) ep = __ldg(embp_g + y2 * R + t);
      }
      // step 1: x^(0)_n = W_emb_prev[:, y_{n-2}] + W_emb_cur[:, y_{n-1}] + B_emb
      if (t < R) m.xs[0][t] = (ep + wembc[y1 * R + t]) + bemb[t];
      ptx::bar_sync(1, kMain);
    } else {
      if (wait(cx, &m.bar_xin, (uint32_t)(n & 1), 12) && t == 0) ptx::mbar_arm(ptx::smem_u32(&m.bar_xin), R * 4);
    }
    if (t == 0) trace(A, n, 0);
    wait(cx, &m.bar_pre, (uint32_t)(n & 1), 13);
    if (t == 0) trace(A, n, 1);

#pragma unroll
    for (int jl = 0; jl < LPC; ++jl) {
      if (jl < nl) {
        const int j = first + jl;
        if (t == 0) trace_clk(A, n, 8 + 5 * jl);
        const float* xin = m.xs[jl];
        float xv[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 v = lds4(xin + ch * 16 + 4 * k);
          xv[4 * k] = v.x; xv[4 * k + 1] = v.y; xv[4 * k + 2] = v.z; xv[4 * k + 3] = v.w;
        }
        const float ph = m.pre[jl][pr], pg = m.pre[jl][R + pr];
        const float xi = xin[pr];
        // a_cur = W_cur x, both gate halves of row pair pr
        float h0 = 0.f, h1 = 0.f, g0 = 0.f, g1 = 0.f;
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
          h0 = fmaf(wc[jl][q], xv[q], h0);
          g0 = fmaf(wc[jl][16 + q], xv[q], g0);
          h1 = fmaf(wc[jl][q + 1], xv[q + 1], h1);
          g1 = fmaf(wc[jl][16 + q + 1], xv[q + 1], g1);
        }
        float ah = h0 + h1, ag = g0 + g1;
        ah += __shfl_xor_sync(0xffffffffu, ah, 1);
        ag += __shfl_xor_sync(0xffffffffu, ag, 1);
        ah += __shfl_xor_sync(0xffffffffu, ah, 2);
        ag += __shfl_xor_sync(0xffffffffu, ag, 2);
        // a = a_prev + a_cur + B + L ; h = tanh(a_h) sigma(a_g)
        const float hv = gate(ah + ph, ag + pg);
        if (t == 0) trace_clk(A, n, 9 + 5 * jl);
        if (ch == 0) {
          m.hs[pr] = hv;
          m.xsave[jl][pr] = xi;
          if (j == pl.L - 1) {
#pragma unroll
            for (int hh = 0; hh < NH; ++hh)
              ptx::st_async(remote(&m.hbuf[0][pr], pl.nc + hh), hv, remote(&m.bar_h[0], pl.nc + hh));
          } else {
            const int k = pl.layer_skip_cta[j], sl = pl.layer_skip_slot[j];
            ptx::st_async(remote(&m.hbuf[sl][pr], k), hv, remote(&m.bar_h[sl], k));
          }
        }
        ptx::bar_sync(1, kMain);
        if (t == 0) trace_clk(A, n, 10 + 5 * jl);
        if (j < pl.L - 1) {
          // x^(j) = x^(j-1) + W_res h + B_res
          float hvv[16];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float4 v = lds4(m.hs + ch * 16 + 4 * k);
            hvv[4 * k] = v.x; hvv[4 * k + 1] = v.y; hvv[4 * k + 2] = v.z; hvv[4 * k + 3] = v.w;
          }
          float r0 = 0.f, r1 = 0.f;
#pragma unroll
          for (int q = 0; q < 16; q += 2) {
            r0 = fmaf(wr[jl][q], hvv[q], r0);
            r1 = fmaf(wr[jl][q + 1], hvv[q + 1], r1);
          }
          float rr = r0 + r1;
          rr += __shfl_xor_sync(0xffffffffu, rr, 1);
          rr += __shfl_xor_sync(0xffffffffu, rr, 2);
          const float xn = xi + (rr + bres[jl * R + pr]);
          if (t == 0) trace_clk(A, n, 11 + 5 * jl);
          if (ch == 0) {
            if (jl + 1 < nl) m.xs[jl + 1][pr] = xn;
            else if (!last_cta) ptx::st_async(remote(&m.xs[0][pr], c + 1), xn, remote(&m.bar_xin, c + 1));
          }
        }
        ptx::bar_sync(1, kMain);
      }
    }
    if (t == 0) {
      trace(A, n, 2);
      ptx::mbar_arrive(ptx::smem_u32(&m.bar_done));
    }
  }

  if (c == 0 && A.N > 0) {  // draw the last sample
    const int64_t n = A.N;
    const float u = uni ? __ldg(uni + n - 1) : 0.0f;
    const int yf = forced ? (int)__ldg(forced + n - 1) : 0;
    wait(cx, &m.bar_logits, (uint32_t)((n - 1) & 1), 11);
    const float l = m.logits_in[t];
    if (forced) {
      A.out_logits[(n - 1) * kLevels + t] = l;
      (void)yf;
    } else {
      const int y = sample_256(l, u, m.dscr, m.fscr, m.iscr, t, 1);
      if (t == 0) A.out_codes[n - 1] = (uint8_t)y;
    }
  }
}

// ------------------------------------------------------------------ chain CTA, aux warpgroup
// For the coming sample n: queue write of x^(j-1)_{n-1}, queue read of x^(j-1)_{n-d},
// pre = B + L^(j)_{n/hop} + W_prev x^(j-1)_{n-d}  (Fig. 2 aux threads).
__device__ void chain_aux(const Params& P, const Ctx& cx, int c, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int at = threadIdx.x - kMain;  // 0..127 = row of a (2r rows)
  const int first = pl.chain_first[c], nl = pl.chain_nl[c];
  const float* wprev = sw;                    // [LPC][R (k)][2R (i)]
  const float* bj = sw + LPC * R * 2 * R;     // [LPC][2R]
  const int L = A.L;

  for (int64_t n = 0; n < A.N; ++n) {
    if (n > 0) wait(cx, &m.bar_done, (uint32_t)((n - 1) & 1), 14);
    if (at == 0) trace(A, n, 4);
    const int64_t f = n / A.hop;
    for (int jl = 0; jl < nl; ++jl) {
      const int j = first + jl;
      const int d = A.dil[j];
      const float lv = __ldg(A.cond + (f * L + j) * 2 * R + at);
      if (at < R) {
        float* ring = A.ring + A.ring_off[j];
        const float xc = m.xsave[jl][at];  // x^(j-1)_{n-1}
        float xpv = 0.0f;
        if (n - d >= 0) xpv = (d == 1) ? xc : ring[(int64_t)(n % d) * R + at];  // slot of n-d
        if (n > 0 && d >= 2) ring[(int64_t)((n - 1) % d) * R + at] = xc;
        m.xp[at] = xpv;
      }
      ptx::bar_sync(2, kAux);
      const float* w = wprev + jl * R * 2 * R;
      float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
      for (int k = 0; k < R; k += 2) {
        a0 = fmaf(w[k * 2 * R + at], m.xp[k], a0);
        a1 = fmaf(w[(k + 1) * 2 * R + at], m.xp[k + 1], a1);
      }
      m.pre[jl][at] = (bj[jl * 2 * R + at] + lv) + (a0 + a1);
      ptx::bar_sync(2, kAux);
    }
    if (at == 0) {
      trace(A, n, 5);
      ptx::mbar_arrive(ptx::smem_u32(&m.bar_pre));
    }
  }
}

// ------------------------------------------------------------------ head CTA (rows [64h, 64h+64))
template <int S>
__device__ void head_main(const Params& P, const Ctx& cx, int hidx, const float* blk, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int t = threadIdx.x;
  constexpr int QS = S / 4;  // weights per thread of W_skip^(l) and of W_relu
  float wsk[QS], wrl[QS], wo[64];
#pragma unroll
  for (int q = 0; q < QS; ++q) wsk[q] = blk[q * kMain + t];
#pragma unroll
  for (int q = 0; q < QS; ++q) wrl[q] = blk[(QS + q) * kMain + t];
#pragma unroll
  for (int q = 0; q < 64; ++q) wo[q] = blk[(2 * QS + q) * kMain + t];
  const float* bskip = sw;           // [S]
  const float* brelu = sw + S;       // [64]
  const float* bout = sw + S + 64;   // [64]
  const int row = t >> 2, ch = t & 3;
  const int nk = pl.nk;

  for (int64_t n = 0; n < A.N; ++n) {
    const uint32_t par = (uint32_t)(n & 1);
    if (wait(cx, &m.bar_h[0], par, 21) && t == 0) ptx::mbar_arm(ptx::smem_u32(&m.bar_h[0]), R * 4);
    if (t == 0) trace(A, n, 0);
    // q = B_skip + sum_k partial_k + W_skip^(l) h^(l); z_s = relu(q)
    float dot;
    int qrow;
    if constexpr (S == 256) {
      qrow = t;
      float d0 = 0.f, d1 = 0.f;
#pragma unroll
      for (int q = 0; q < 64; q += 4) {
        const float4 hv = lds4(&m.hbuf[0][q]);
        d0 = fmaf(wsk[q], hv.x, d0);
        d1 = fmaf(wsk[q + 1], hv.y, d1);
        d0 = fmaf(wsk[q + 2], hv.z, d0);
        d1 = fmaf(wsk[q + 3], hv.w, d1);
      }
      dot = d0 + d1;
    } else {
      qrow = t >> 1;
      const int half = t & 1;
      float d0 = 0.f, d1 = 0.f;
#pragma unroll
      for (int q = 0; q < 32; q += 4) {
        const float4 hv = lds4(&m.hbuf[0][32 * half + q]);
        d0 = fmaf(wsk[q], hv.x, d0);
        d1 = fmaf(wsk[q + 1], hv.y, d1);
        d0 = fmaf(wsk[q + 2], hv.z, d0);
        d1 = fmaf(wsk[q + 3], hv.w, d1);
      }
      dot = d0 + d1;
      dot += __shfl_xor_sync(0xffffffffu, dot, 1);
    }
    if (nk > 0) {
      if (wait(cx, &m.bar_part, par, 22) && t == 0) ptx::mbar_arm(ptx::smem_u32(&m.bar_part), nk * S * 4);
    }
    if (t == 0) trace(A, n, 1);
    float qv = bskip[qrow];
    for (int k = 0; k < nk; ++k) qv += m.part[k][qrow];
    qv += dot;
    if (S == 256 || (t & 1) == 0) m.zs[qrow] = fmaxf(qv, 0.0f);
    ptx::bar_sync(1, kMain);
    // z_a = relu(W_relu z_s + B_relu), rows 64h + row
    float r0 = 0.f, r1 = 0.f;
#pragma unroll
    for (int q = 0; q < QS; q += 4) {
      const float4 zv = lds4(&m.zs[ch * QS + q]);
      r0 = fmaf(wrl[q], zv.x, r0);
      r1 = fmaf(wrl[q + 1], zv.y, r1);
      r0 = fmaf(wrl[q + 2], zv.z, r0);
      r1 = fmaf(wrl[q + 3], zv.w, r1);
    }
    float za = r0 + r1;
    za += __shfl_xor_sync(0xffffffffu, za, 1);
    za += __shfl_xor_sync(0xffffffffu, za, 2);
    za = fmaxf(za + brelu[row], 0.0f);
    if (ch == 0) {
#pragma unroll
      for (int hh = 0; hh < NH; ++hh)
        ptx::st_async(remote(&m.za_in[64 * hidx + row], pl.nc + hh), za, remote(&m.bar_za, pl.nc + hh));
    }
    if (wait(cx, &m.bar_za, par, 23) && t == 0) ptx::mbar_arm(ptx::smem_u32(&m.bar_za), kLevels * 4);
    if (t == 0) trace(A, n, 2);
    // logits = W_out z_a + B_out, rows 64h + row
    float o0 = 0.f, o1 = 0.f;
#pragma unroll
    for (int q = 0; q < 64; q += 4) {
      const float4 zv = lds4(&m.za_in[ch * 64 + q]);
      o0 = fmaf(wo[q], zv.x, o0);
      o1 = fmaf(wo[q + 1], zv.y, o1);
      o0 = fmaf(wo[q + 2], zv.z, o0);
      o1 = fmaf(wo[q + 3], zv.w, o1);
    }
    float lg = o0 + o1;
    lg += __shfl_xor_sync(0xffffffffu, lg, 1);
    lg += __shfl_xor_sync(0xffffffffu, lg, 2);
    lg += bout[row];
    if (ch == 0) ptx::st_async(remote(&m.logits_in[64 * hidx + row], 0), lg, remote(&m.bar_logits, 0));
    if (t == 0) trace(A, n, 3);
  }
}

// ------------------------------------------------------------------ skip CTA
// partial_k = sum over owned layers j (ascending) of W_skip^(j) h^(j).
template <int S>
__device__ void skip_main(const Params& P, const Ctx& cx, int k, const float* blk, const float* sw) {
  const RunArgs& A = P.a;
  const ClusterPlan& pl = P.p;
  Mail& m = *cx.mail;
  const int t = threadIdx.x;
  constexpr int QS = S / 4;             // registers per layer per thread
  constexpr int MAXREG = 192 / QS;      // 3 (s=256) or 6 (s=128)
  constexpr int LSTRIDE = (S == 256) ? 64 * 256 : 2 * (32 * 128 + 16);  // floats per smem layer
  const int nown = pl.skip_n[k], nsm = pl.skip_nsm[k], nreg = nown - nsm;
  float w[MAXREG][QS];
#pragma unroll
  for (int rl = 0; rl < MAXREG; ++rl)
#pragma unroll
    for (int q = 0; q < QS; ++q) w[rl][q] = (rl < nreg) ? blk[(rl * QS + q) * kMain + t] : 0.0f;
  const int row = (S == 256) ? t : (t >> 1);
  const int half = (S == 256) ? 0 : (t & 1);

  for (int64_t n = 0; n < A.N; ++n) {
    const uint32_t par = (uint32_t)(n & 1);
    float part = 0.0f;
    for (int sl = 0; sl < nsm; ++sl) {
      if (wait(cx, &m.bar_h[sl], par, 31) && t == 0) ptx::mbar_arm(ptx::smem_u32(&m.bar_h[sl]), R * 4);
      const float* ws = sw + sl * LSTRIDE;
      float d0 = 0.f, d1 = 0.f;
      if constexpr (S == 256) {
#pragma unroll 8
        for (int q = 0; q < 64; q += 2) {
          d0 = fmaf(ws[q * 256 + row], m.hbuf[sl][q], d0);
          d1 = fmaf(ws[(q + 1) * 256 + row], m.hbuf[sl][q + 1], d1);
        }
      } else {
        const float* wh = ws + half * (32 * 128 + 16);
#pragma unroll 8
        for (int q = 0; q < 32; q += 2) {
          d0 = fmaf(wh[q * 128 + row], m.hbuf[sl][32 * half + q], d0);
          d1 = fmaf(wh[(q + 1) * 128 + row], m.hbuf[sl][32 * half + q + 1], d1);
        }
      }
      float dot = d0 + d1;
      if (S == 128) dot += __shfl_xor_sync(0xffffffffu, dot, 1);
      part += dot;
    }
#pragma unroll
    for (int rl = 0; rl < MAXREG; ++rl) {
      if (rl < nreg) {
        const int sl = nsm + rl;
        if (wait(cx, &m.bar_h[sl], par, 32) && t == 0) ptx::mbar_arm(ptx::smem_u32(&m.bar_h[sl]), R * 4);
        float d0 = 0.f, d1 = 0.f;
#pragma unroll
        for (int q = 0; q < QS; q += 4) {
          const float4 hv = lds4(&m.hbuf[sl][half * 32 + q]);
          d0 = fmaf(w[rl][q], hv.x, d0);
          d1 = fmaf(w[rl][q + 1], hv.y, d1);
          d0 = fmaf(w[rl][q + 2], hv.z, d0);
          d1 = fmaf(w[rl][q + 3], hv.w, d1);
        }
        float dot = d0 + d1;
        if (S == 128) dot += __shfl_xor_sync(0xffffffffu, dot, 1);
        part += dot;
      }
    }
    if (half == 0) m.zs[row] = part;
    if (t == 0) trace(A, n, 1);
    ptx::bar_sync(1, kMain);
    if (t < (S / 4) * NH) {
      const int hh = t / (S / 4), e = t % (S / 4);
      ptx::st_async4(remote(&m.part[k][4 * e], pl.nc + hh), lds4(&m.zs[4 * e]),
                     remote(&m.bar_part, pl.nc + hh));
    }
  }
}

template <int S>
__global__ void __launch_bounds__(kThreads, 1) k_cluster(const __grid_constant__ Params P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Mail* mail = reinterpret_cast<Mail*>(smem_raw);
  float* sw = reinterpret_cast<float*>(smem_raw + ((sizeof(Mail) + 127) & ~size_t(127)));
  const ClusterPlan& pl = P.p;
  const int rank = (int)ptx::cluster_rank();
  const int t = threadIdx.x;
  Ctx cx{mail, P.a.err, pl.size};

  int role = kIdle, idx = 0;
  if (rank < pl.nc) { role = kChain; idx = rank; }
  else if (rank < pl.nc + NH) { role = kHead; idx = rank - pl.nc; }
  else if (rank < pl.nc + NH + pl.nk) { role = kSkip; idx = rank - pl.nc - NH; }

  // barriers + abort flag, then the shared-memory weight image
  if (t == 0) {
    mail->abort_flag = 0;
    ptx::mbar_init(ptx::smem_u32(&mail->bar_xin), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_logits), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_pre), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_done), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_part), 1);
    ptx::mbar_init(ptx::smem_u32(&mail->bar_za), 1);
    for (int i = 0; i < kCMaxSlot; ++i) ptx::mbar_init(ptx::smem_u32(&mail->bar_h[i]), 1);
    ptx::fence_mbar_init();
    // arm phase 0 of every transaction barrier this role receives on
    ptx::mbar_arm(ptx::smem_u32(&mail->bar_xin), R * 4);
    ptx::mbar_arm(ptx::smem_u32(&mail->bar_logits), kLevels * 4);
    ptx::mbar_arm(ptx::smem_u32(&mail->bar_part), pl.nk * S * 4);
    ptx::mbar_arm(ptx::smem_u32(&mail->bar_za), kLevels * 4);
    for (int i = 0; i < kCMaxSlot; ++i) ptx::mbar_arm(ptx::smem_u32(&mail->bar_h[i]), R * 4);
  }
  const float* blk = P.pk + pl.pk_off[rank < kCMaxCta ? rank : 0];
  if (role != kIdle) {
    const float4* src = reinterpret_cast<const float4*>(P.pk + pl.pk_smem_off[rank]);
    float4* dst = reinterpret_cast<float4*>(sw);
    for (int i = t; i < pl.pk_smem_floats[rank] / 4; i += kThreads) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  ptx::cluster_sync();

  // Register split: the two math warpgroups grow to 232 registers (W_cur/W_res,
  // head or skip weights live there), the aux warpgroup shrinks to 48.  Each
  // branch ends with its own cluster barrier so no code is shared across budgets.
  if (t < kMain) {
    ptx::setmaxnreg_inc<kMainRegs>();
    if (role == kChain) chain_main<S>(P, cx, idx, blk, sw);
    else if (role == kHead) head_main<S>(P, cx, idx, blk, sw);
    else if (role == kSkip) skip_main<S>(P, cx, idx, blk, sw);
    __syncwarp();
    ptx::cluster_sync();
    return;
  }
  ptx::setmaxnreg_dec<kAuxRegs>();
  if (role == kChain) chain_aux(P, cx, idx, sw);
  __syncwarp();
  ptx::cluster_sync();
}

template <int S>
cudaError_t configure(int smem) {
  cudaError_t e = cudaFuncSetAttribute(k_cluster<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_cluster<S>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}

template <int S>
int max_active_clusters(int size, int smem) {
  if (configure<S>(smem) != cudaSuccess) {
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
  if (cudaOccupancyMaxActiveClusters(&n, k_cluster<S>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int smem_chain(const ClusterPlan& p, int c) {
  int f = LPC * R * 2 * R + LPC * 2 * R + LPC * R;
  if (c == 0) f += kLevels * R + R;
  (void)p;
  return f;
}

}  // namespace

ClusterPlan plan_cluster(int L, int r, int s, int device) {
  ClusterPlan p;
  p.L = L;
  p.r = r;
  p.s = s;
  if (r != R) { p.why = "cluster kernel is built for r = 64"; return p; }
  if (s != 128 && s != 256) { p.why = "cluster kernel needs s in {128, 256}"; return p; }
  if (L > kCMaxLayers) { p.why = "too many layers"; return p; }
  p.nc = (L + LPC - 1) / LPC;
  for (int c = 0; c < p.nc; ++c) {
    p.chain_first[c] = c * LPC;
    p.chain_nl[c] = std::min(LPC, L - c * LPC);
  }
  p.nh = NH;
  const int nskip = L - 1;  // W_skip^(l) lives in the head CTAs
  const int qs = s / 4, maxreg = 192 / qs;
  const int lstride = (s == 256) ? 64 * 256 : 2 * (32 * 128 + 16);
  const int maxsm = std::min(kCMaxSlot - maxreg, (int)((200 * 1024) / (lstride * 4)));
  const int cap = maxreg + maxsm;
  p.nk = nskip > 0 ? (nskip + cap - 1) / cap : 0;
  if (p.nk > kCMaxSkip) { p.why = "too many skip CTAs"; return p; }
  p.size = p.nc + p.nh + p.nk;
  if (p.size > kCMaxCta) { p.why = "model does not fit one 16-CTA cluster"; return p; }
  for (int k = 0; k < p.nk; ++k) p.skip_n[k] = 0;
  for (int j = 0; j < nskip; ++j) {  // round robin: consecutive layers go to different CTAs
    const int k = j % p.nk;
    p.layer_skip_cta[j] = p.nc + p.nh + k;
    p.layer_skip_slot[j] = p.skip_n[k]++;
  }
  for (int k = 0; k < p.nk; ++k) {
    if (p.skip_n[k] > cap) { p.why = "skip capacity"; return p; }
    p.skip_nsm[k] = std::max(0, p.skip_n[k] - maxreg);  // latest layers in registers
  }
  // packed layout
  int64_t off = 0;
  int max_sw = 0;
  for (int rank = 0; rank < p.size; ++rank) {
    int regs = 0, swf = 0;
    if (rank < p.nc) { regs = kChainRegs; swf = smem_chain(p, rank); }
    else if (rank < p.nc + p.nh) { regs = 2 * qs + 64; swf = s + 128; }
    else { const int k = rank - p.nc - p.nh; regs = (p.skip_n[k] - p.skip_nsm[k]) * qs; swf = p.skip_nsm[k] * lstride; }
    p.pk_off[rank] = off;
    off += (int64_t)regs * kMain;
    p.pk_smem_off[rank] = off;
    p.pk_smem_floats[rank] = swf;
    off += (swf + 3) & ~3;
    max_sw = std::max(max_sw, swf);
  }
  p.embp_off = off;
  off += (int64_t)kLevels * R;
  p.pk_total = off;
  p.smem_bytes = (int)(((sizeof(Mail) + 127) & ~size_t(127)) + (size_t)max_sw * 4);
  int dev_smem = 0;
  cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (p.smem_bytes > dev_smem) { p.why = "shared memory"; return p; }
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  const int nclus = (s == 256) ? max_active_clusters<256>(p.size, p.smem_bytes)
                               : max_active_clusters<128>(p.size, p.smem_bytes);
  if (prev >= 0) cudaSetDevice(prev);
  if (nclus < 1) { p.why = "cluster cannot be scheduled on this device"; return p; }
  p.ok = true;
  p.why = "ok";
  return p;
}

size_t packed_bytes(const ClusterPlan& p) { return sizeof(float) * (size_t)p.pk_total; }

cudaError_t pack_cluster_weights(const ClusterPlan& p, const float* w, const Offsets& o, void* packed) {
  const int s = p.s, qs = s / 4;
  std::vector<float> h((size_t)p.pk_total, 0.0f);
  auto W = [&](int j, int64_t off_in_layer, int row, int col, int ncol) {
    return w[(int64_t)j * o.layer_stride + off_in_layer + (int64_t)row * ncol + col];
  };
  for (int rank = 0; rank < p.size; ++rank) {
    float* blk = h.data() + p.pk_off[rank];
    float* sm = h.data() + p.pk_smem_off[rank];
    if (rank < p.nc) {
      const int first = p.chain_first[rank], nl = p.chain_nl[rank];
      for (int t = 0; t < kMain; ++t) {
        const int pr = t >> 2, ch = t & 3;
        for (int jl = 0; jl < nl; ++jl) {
          const int j = first + jl;
          for (int q = 0; q < 16; ++q) {
            blk[(jl * 48 + q) * kMain + t] = W(j, o.w_cur, pr, ch * 16 + q, R);
            blk[(jl * 48 + 16 + q) * kMain + t] = W(j, o.w_cur, R + pr, ch * 16 + q, R);
            blk[(jl * 48 + 32 + q) * kMain + t] = W(j, o.w_res, pr, ch * 16 + q, R);
          }
        }
      }
      for (int jl = 0; jl < nl; ++jl) {
        const int j = first + jl;
        for (int k = 0; k < R; ++k)
          for (int i = 0; i < 2 * R; ++i) sm[jl * R * 2 * R + k * 2 * R + i] = W(j, o.w_prev, i, k, R);
        for (int i = 0; i < 2 * R; ++i) sm[LPC * R * 2 * R + jl * 2 * R + i] = w[(int64_t)j * o.layer_stride + o.b + i];
        for (int i = 0; i < R; ++i)
          sm[LPC * R * 2 * R + LPC * 2 * R + jl * R + i] = w[(int64_t)j * o.layer_stride + o.b_res + i];
      }
      if (rank == 0) {
        float* we = sm + LPC * R * 2 * R + LPC * 2 * R + LPC * R;
        for (int y = 0; y < kLevels; ++y)
          for (int i = 0; i < R; ++i) we[y * R + i] = w[o.emb_cur + (int64_t)i * kLevels + y];
        for (int i = 0; i < R; ++i) we[kLevels * R + i] = w[o.b_emb + i];
      }
    } else if (rank < p.nc + p.nh) {
      const int hidx = rank - p.nc;
      const int jl = p.L - 1;
      for (int t = 0; t < kMain; ++t) {
        const int row = t >> 2, ch = t & 3;
        for (int q = 0; q < qs; ++q) {
          if (s == 256) blk[q * kMain + t] = W(jl, o.w_skip, t, q, R);
          else blk[q * kMain + t] = W(jl, o.w_skip, t >> 1, 32 * (t & 1) + q, R);
          blk[(qs + q) * kMain + t] = w[o.w_relu + (int64_t)(64 * hidx + row) * s + ch * qs + q];
        }
        for (int q = 0; q < 64; ++q)
          blk[(2 * qs + q) * kMain + t] = w[o.w_out + (int64_t)(64 * hidx + row) * kLevels + ch * 64 + q];
      }
      for (int i = 0; i < s; ++i) sm[i] = w[o.b_skip + i];
      for (int i = 0; i < 64; ++i) {
        sm[s + i] = w[o.b_relu + 64 * hidx + i];
        sm[s + 64 + i] = w[o.b_out + 64 * hidx + i];
      }
    } else {
      const int k = rank - p.nc - p.nh;
      std::vector<int> layers;
      for (int j = 0; j < p.L - 1; ++j)
        if (p.layer_skip_cta[j] == rank) layers.push_back(j);
      const int nsm = p.skip_nsm[k];
      const int lstride = (s == 256) ? 64 * 256 : 2 * (32 * 128 + 16);
      for (int sl = 0; sl < (int)layers.size(); ++sl) {
        const int j = layers[sl];
        if (sl < nsm) {
          float* ws = sm + sl * lstride;
          for (int i = 0; i < s; ++i)
            for (int c = 0; c < R; ++c) {
              if (s == 256) ws[c * 256 + i] = W(j, o.w_skip, i, c, R);
              else ws[(c >> 5) * (32 * 128 + 16) + (c & 31) * 128 + i] = W(j, o.w_skip, i, c, R);
            }
        } else {
          const int rl = sl - nsm;
          for (int t = 0; t < kMain; ++t)
            for (int q = 0; q < qs; ++q) {
              if (s == 256) blk[(rl * qs + q) * kMain + t] = W(j, o.w_skip, t, q, R);
              else blk[(rl * qs + q) * kMain + t] = W(j, o.w_skip, t >> 1, 32 * (t & 1) + q, R);
            }
        }
      }
    }
  }
  float* ep = h.data() + p.embp_off;
  for (int y = 0; y < kLevels; ++y)
    for (int i = 0; i < R; ++i) ep[y * R + i] = w[o.emb_prev + (int64_t)i * kLevels + y];
  return cudaMemcpy(packed, h.data(), sizeof(float) * h.size(), cudaMemcpyHostToDevice);
}

cudaError_t launch_cluster_kernel(const RunArgs& a, const ClusterPlan& p, const void* packed, cudaStream_t st,
                                  LaunchInfo* info) {
  if (!p.ok) return cudaErrorNotSupported;
  if (a.n_streams != 1) return cudaErrorInvalidValue;
  Params P;
  P.a = a;
  P.p = p;
  P.pk = static_cast<const float*>(packed);
  cudaError_t e = (p.s == 256) ? configure<256>(p.smem_bytes) : configure<128>(p.smem_bytes);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.size);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = p.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.size;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = (p.s == 256) ? cudaLaunchKernelEx(&cfg, k_cluster<256>, P) : cudaLaunchKernelEx(&cfg, k_cluster<128>, P);
  info->grid = p.size;
  info->cluster = p.size;
  info->threads = kThreads;
  info->launches = 1;
  return e;
}

}  // namespace dvw
