/*
 * dvw_oracle.c -- plain, slow, obviously correct CPU oracle of autoregressive
 * WaveNet sample generation (Deep Voice, arXiv 1702.07825).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code with the CUDA path (paper_1702_07825_b200/csrc): it has its
 * own weight-offset bookkeeping, its own sampler, its own everything.
 *
 * Arithmetic: scalar C, double throughout, no SIMD intrinsics, compiled
 * without -ffast-math.  Weights, conditioning and uniforms arrive as the fp32
 * values the GPU receives and are promoted to double.
 *
 * Algorithm, in the paper's order and notation (PAPER.md = /root/reference):
 *   state: ring_j[d_j][r] = 0 ; y_{-1} = y_{-2} = a/2 = 128       (R4)
 *   for n = 0 .. N-1:
 *     f   = floor(n / hop)                                      (App. A.2 repetition)
 *     x   = W_emb_prev[:, y_{n-2}] + W_emb_cur[:, y_{n-1}] + B_emb  (§5.1 step 1; R3)
 *     q   = B_skip                                              (§5.1 step 2d)
 *     for j = 1 .. l:
 *       xp  = ring_j[n mod d_j]          (x^{(j-1)}_{n-d_j}, 0 if n < d_j)   (step 2a)
 *       a   = W_prev xp + W_cur x + B + L^{(j)}_n               (steps 2a-2c)
 *       h   = tanh(a[0:r]) * sigmoid(a[r:2r])                   (step 2c;
 *             oracle_run_nl with nl = 1: App. C's approximations, also for the softmax exp)
 *       ring_j[n mod d_j] = x            (store x^{(j-1)}_n after reading)
 *       x   = x + W_res h + B_res                               (App. A.1; R1)
 *       q   = q + W_skip^{(j)} h                                (step 2d)
 *     z_s = relu(q); z_a = relu(W_relu z_s + B_relu); l = W_out z_a + B_out   (step 3)
 *     p   = softmax(l); y_n = inverse-CDF draw with u_n         (R11)
 *
 * Pins (tests/test_oracle_pins.py, test_appc_oracle.py): mu-law against torchaudio, the
 * receptive field, causality, the softmax (oracle_softmax vs scipy.special.softmax, its sum,
 * and the draw frequencies over a u grid), closed-form draws (zero weights, one-hot and
 * bias-only logits), the independent brute-force oracle (bruteforce.py), the App. A.4
 * strategies' limits (t = 1, k = a), and App. C's printed maximum errors.
 *
 * Weight blob (include/dvw.h, restated here independently):
 *   per layer j: W_prev[2r][r] W_cur[2r][r] B[2r] W_res[r][r] B_res[r] W_skip[s][r]
 *   then W_emb_prev[r][a] W_emb_cur[r][a] B_emb[r] B_skip[s] W_relu[a][s]
 *        B_relu[a] W_out[a][a] B_out[a]
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_API __attribute__((visibility("default")))

ORACLE_API int64_t oracle_weights_numel(int L, int r, int s, int a) {
  int64_t per_layer = (int64_t)2 * r * r + (int64_t)2 * r * r + 2 * r + (int64_t)r * r + r + (int64_t)s * r;
  return L * per_layer + (int64_t)2 * r * a + r + s + (int64_t)a * s + a + (int64_t)a * a + a;
}

/* ---- App. C: the paper's approximate nonlinearities (R31) ----
 * The oracle of the DVW_PRECISION_APPC tier, written as the paper prints it:
 *   e~(x)    = 1 + |x| + 0.5658 x^2 + 0.143 x^4
 *   tanh(x) ~ sign(x) (e~(x) - 1/e~(x)) / (e~(x) + 1/e~(x))
 *   sigma(x) ~ e~(x) / (1 + e~(x)) for x >= 0, 1 / (1 + e~(x)) for x <= 0
 *   e^x = 2^(x / ln 2); for x' = x / ln 2 the fp32 bit pattern of 2^x' is
 *     I = (x' + 126 + g(z)) 2^23, z = x' - floor(x'),
 *     g(z) ~ -4.7259162 + 27.7280233 / (4.84252568 - z) - 1.49012907 z
 *   I is truncated to an integer and read back as a 32-bit float; x' < -126 (no normal
 *   fp32 pattern) gives 0 (reading R31).  Double arithmetic up to the bit pattern. */
static double appc_etilde(double x) { return 1.0 + fabs(x) + 0.5658 * x * x + 0.143 * x * x * x * x; }

static double appc_tanh(double x) {
  const double e = appc_etilde(x);
  const double v = (e - 1.0 / e) / (e + 1.0 / e);
  return x > 0.0 ? v : (x < 0.0 ? -v : 0.0);
}

static double appc_sigmoid(double x) {
  const double e = appc_etilde(x);
  return x >= 0.0 ? e / (1.0 + e) : 1.0 / (1.0 + e);
}

static double appc_exp(double x) {
  const double xl = x / log(2.0);
  if (!(xl >= -126.0)) return 0.0;
  const double z = xl - floor(xl);
  const double g = -4.7259162 + 27.7280233 / (4.84252568 - z) - 1.49012907 * z;
  const int32_t bits = (int32_t)((xl + 126.0 + g) * 8388608.0);  /* truncation toward zero */
  float f;
  memcpy(&f, &bits, sizeof f);
  return (double)f;
}

ORACLE_API double oracle_appc_tanh(double x) { return appc_tanh(x); }
ORACLE_API double oracle_appc_sigmoid(double x) { return appc_sigmoid(x); }
ORACLE_API double oracle_appc_exp(double x) { return appc_exp(x); }

/* the nonlinearity set: nl = 0 exact (reading R13), nl = 1 App. C */
static double nl_exp(int nl, double x) { return nl ? appc_exp(x) : exp(x); }

/* Inverse-CDF direct sampling (App. A.4 "Sample randomly from P(y)";
 * reading R11): e_k = exp(l_k - max l); P_k = sum_{i<=k} e_i in ascending k;
 * y = min{k : u * P_{a-1} < P_k}; fallback the largest k with e_k > 0. */
/* softmax numerators (PAPER.md:374 p = softmax(l)): e_k = exp(l_k - max l); returns S = sum e_k,
 * so p_k = e_k / S (oracle_softmax) */
static double softmax_terms(const double* logit, int a, double* e, int nl) {
  double m = logit[0];
  for (int k = 1; k < a; ++k)
    if (logit[k] > m) m = logit[k];
  double S = 0.0;
  for (int k = 0; k < a; ++k) {
    e[k] = nl_exp(nl, logit[k] - m);
    S += e[k];
  }
  return S;
}

static int sample_inverse_cdf(const double* logit, int a, double u, double* e, int nl) {
  const double S = softmax_terms(logit, a, e, nl);
  double t = u * S, P = 0.0;
  for (int k = 0; k < a; ++k) {
    P += e[k];
    if (t < P) return k;
  }
  for (int k = a - 1; k >= 0; --k)
    if (e[k] > 0.0) return k;
  return a - 1;
}

/* The draw under each of the paper's sampling strategies (App. A.4);
 * kind: 0 direct, 1 temperature, 2 mean, 3 mode, 4 top-k.  Details the paper leaves open
 * follow SPEC's sample() post-conditions (readings R24-R27):
 *   temperature t : P_t(y) = P(y)^(1/t) / Z, i.e. e_k = exp((l_k - max l) / t), then the
 *                   direct inverse-CDF rule with u (t = 1 is direct sampling)
 *   mean          : round(sum_y y P(y)) = floor(E_P[y] + 0.5), clamped to [0, a-1]; no u
 *   mode          : argmax_y P(y) = argmax l, lowest index on ties; no u
 *   top-k         : keep the k largest P(y) (ties by lower index), zero the rest,
 *                   renormalise (implicitly), then the direct rule with u */
static int sample_policy(const double* logit, int a, int kind, double t, int topk, double u, double* e, int nl) {
  if (kind == 0) return sample_inverse_cdf(logit, a, u, e, nl);
  double m = logit[0];
  int am = 0;
  for (int k = 1; k < a; ++k)
    if (logit[k] > m) { m = logit[k]; am = k; }
  if (kind == 3) return am;  /* first index reaching the max */
  if (kind == 2) {
    double S = 0.0, M = 0.0;
    for (int k = 0; k < a; ++k) {
      const double ek = nl_exp(nl, logit[k] - m);
      S += ek;
      M += (double)k * ek;
    }
    double y = floor(M / S + 0.5);
    if (y < 0.0) y = 0.0;
    if (y > a - 1) y = a - 1;
    return (int)y;
  }
  for (int k = 0; k < a; ++k) {
    if (kind == 1) {
      e[k] = nl_exp(nl, (logit[k] - m) / t);
    } else { /* top-k: rank of k among all codes, larger first, ties by lower index */
      int rank = 0;
      for (int j = 0; j < a; ++j)
        if (logit[j] > logit[k] || (logit[j] == logit[k] && j < k)) ++rank;
      e[k] = rank < topk ? nl_exp(nl, logit[k] - m) : 0.0;
    }
  }
  double S = 0.0;
  for (int k = 0; k < a; ++k) S += e[k];
  double thr = u * S, P = 0.0;
  for (int k = 0; k < a; ++k) {
    P += e[k];
    if (thr < P) return k;
  }
  for (int k = a - 1; k >= 0; --k)
    if (e[k] > 0.0) return k;
  return a - 1;
}

ORACLE_API int oracle_sample(const double* logits, int a, float u) {
  double* e = (double*)malloc(sizeof(double) * a);
  int y = sample_inverse_cdf(logits, a, (double)u, e, 0);
  free(e);
  return y;
}

/* p = softmax(l) with the sampler's own numerators: p_k = e_k / S. */
ORACLE_API void oracle_softmax(const double* logits, int a, double* p) {
  const double S = softmax_terms(logits, a, p, 0);
  for (int k = 0; k < a; ++k) p[k] /= S;
}

ORACLE_API int oracle_sample_policy(const double* logits, int a, int kind, double t, int topk, float u) {
  if (kind < 0 || kind > 4 || (kind == 1 && !(t > 0.0)) || (kind == 4 && (topk < 1 || topk > a))) return -1;
  double* e = (double*)malloc(sizeof(double) * a);
  int y = sample_policy(logits, a, kind, t, topk, (double)u, e, 0);
  free(e);
  return y;
}

static double sigmoid(double v) { return 1.0 / (1.0 + exp(-v)); }

/* y[i] = sum_k W[i][k] x[k], W row-major rows x cols (plain definition). */
static void matvec(const double* W, int rows, int cols, const double* x, double* y) {
  for (int i = 0; i < rows; ++i) {
    double acc = 0.0;
    for (int k = 0; k < cols; ++k) acc += W[(int64_t)i * cols + k] * x[k];
    y[i] = acc;
  }
}

/*
 * One utterance.  Returns 0 on success, negative on bad arguments.
 *   dilations   : length L, each >= 1 (NULL -> 2^((j-1) mod 10))
 *   weights     : fp32 blob, numel must equal oracle_weights_numel
 *   cond        : fp32 [n_frames][L][2r]; frame for sample n is n / hop
 *   uniforms    : fp32 [N] (may be NULL only when forced != NULL)
 *   forced      : uint8 [N] teacher-forced history, or NULL for free running
 *   out_codes   : uint8 [N] the code fed back at step n (forced[n] or the draw)
 *   out_logits  : double [N][a] pre-softmax logits (may be NULL)
 *   out_sampled : uint8 [N] the draw with u_n even when teacher-forced (may be NULL)
 */
ORACLE_API int oracle_run_nl(int L, int r, int s, int a, const int32_t* dilations,
                             const float* weights, int64_t numel, const float* cond,
                             int64_t n_frames, int hop, const float* uniforms,
                             const uint8_t* forced, int64_t N, uint8_t* out_codes,
                             double* out_logits, uint8_t* out_sampled, int kind, double temp,
                             int topk, int nl) {
  if (nl < 0 || nl > 1) return -6;
  if (L < 1 || r < 1 || s < 1 || a < 2 || a > 256 || hop < 1 || N < 0) return -1;
  if (kind < 0 || kind > 4 || (kind == 1 && !(temp > 0.0)) || (kind == 4 && (topk < 1 || topk > a))) return -5;
  if (numel != oracle_weights_numel(L, r, s, a)) return -2;
  if (N > 0 && n_frames < (N + hop - 1) / hop) return -3;
  if (!forced && !uniforms) return -4;

  int* d = (int*)malloc(sizeof(int) * L);
  int64_t ring_total = 0;
  for (int j = 0; j < L; ++j) {
    d[j] = dilations ? dilations[j] : (1 << (j % 10));
    if (d[j] < 1) { free(d); return -5; }
    ring_total += d[j];
  }

  /* promote the blob to double once */
  double* W = (double*)malloc(sizeof(double) * numel);
  for (int64_t i = 0; i < numel; ++i) W[i] = (double)weights[i];

  /* offsets, written out from the roster */
  int64_t per_layer = (int64_t)4 * r * r + 2 * r + (int64_t)r * r + r + (int64_t)s * r;
  const double** Wprev = (const double**)malloc(sizeof(double*) * L);
  const double** Wcur = (const double**)malloc(sizeof(double*) * L);
  const double** Bj = (const double**)malloc(sizeof(double*) * L);
  const double** Wres = (const double**)malloc(sizeof(double*) * L);
  const double** Bres = (const double**)malloc(sizeof(double*) * L);
  const double** Wskip = (const double**)malloc(sizeof(double*) * L);
  for (int j = 0; j < L; ++j) {
    const double* p = W + j * per_layer;
    Wprev[j] = p;            p += (int64_t)2 * r * r;
    Wcur[j] = p;             p += (int64_t)2 * r * r;
    Bj[j] = p;               p += 2 * r;
    Wres[j] = p;             p += (int64_t)r * r;
    Bres[j] = p;             p += r;
    Wskip[j] = p;
  }
  const double* g = W + L * per_layer;
  const double* Wemb_prev = g; g += (int64_t)r * a;
  const double* Wemb_cur = g;  g += (int64_t)r * a;
  const double* Bemb = g;      g += r;
  const double* Bskip = g;     g += s;
  const double* Wrelu = g;     g += (int64_t)a * s;
  const double* Brelu = g;     g += a;
  const double* Wout = g;      g += (int64_t)a * a;
  const double* Bout = g;

  double* ring = (double*)calloc(ring_total * r, sizeof(double));
  int64_t* ring_off = (int64_t*)malloc(sizeof(int64_t) * L);
  int64_t acc_off = 0;
  for (int j = 0; j < L; ++j) { ring_off[j] = acc_off; acc_off += (int64_t)d[j] * r; }

  double* x = (double*)malloc(sizeof(double) * r);
  double* xnew = (double*)malloc(sizeof(double) * r);
  double* ap = (double*)malloc(sizeof(double) * 2 * r);
  double* ac = (double*)malloc(sizeof(double) * 2 * r);
  double* h = (double*)malloc(sizeof(double) * r);
  double* rh = (double*)malloc(sizeof(double) * r);
  double* q = (double*)malloc(sizeof(double) * s);
  double* sk = (double*)malloc(sizeof(double) * s);
  double* zs = (double*)malloc(sizeof(double) * s);
  double* za = (double*)malloc(sizeof(double) * a);
  double* lg = (double*)malloc(sizeof(double) * a);
  double* e = (double*)malloc(sizeof(double) * a);

  /* y_{n-1}, y_{n-2}: codes at negative times are mu-law(0) = a/2 (= 128 at a = 256; R4) */
  int y1 = a / 2, y2 = a / 2;
  for (int64_t n = 0; n < N; ++n) {
    int64_t f = n / hop;
    /* step 1: sample embedding, two column lookups */
    for (int i = 0; i < r; ++i)
      x[i] = Wemb_prev[(int64_t)i * a + y2] + Wemb_cur[(int64_t)i * a + y1] + Bemb[i];
    for (int i = 0; i < s; ++i) q[i] = Bskip[i];
    /* step 2: layers */
    for (int j = 0; j < L; ++j) {
      double* slot = ring + ring_off[j] + (int64_t)(n % d[j]) * r;
      const float* Lj = cond + ((int64_t)f * L + j) * 2 * r;
      matvec(Wprev[j], 2 * r, r, slot, ap);
      matvec(Wcur[j], 2 * r, r, x, ac);
      for (int i = 0; i < r; ++i) {
        double ah = ap[i] + ac[i] + Bj[j][i] + (double)Lj[i];
        double ag = ap[r + i] + ac[r + i] + Bj[j][r + i] + (double)Lj[r + i];
        h[i] = nl ? appc_tanh(ah) * appc_sigmoid(ag) : tanh(ah) * sigmoid(ag);
      }
      memcpy(slot, x, sizeof(double) * r);
      matvec(Wres[j], r, r, h, rh);
      for (int i = 0; i < r; ++i) xnew[i] = x[i] + rh[i] + Bres[j][i];
      memcpy(x, xnew, sizeof(double) * r);
      matvec(Wskip[j], s, r, h, sk);
      for (int i = 0; i < s; ++i) q[i] += sk[i];
    }
    /* step 3: output */
    for (int i = 0; i < s; ++i) zs[i] = q[i] > 0.0 ? q[i] : 0.0;
    matvec(Wrelu, a, s, zs, za);
    for (int i = 0; i < a; ++i) {
      double v = za[i] + Brelu[i];
      za[i] = v > 0.0 ? v : 0.0;
    }
    matvec(Wout, a, a, za, lg);
    for (int i = 0; i < a; ++i) lg[i] += Bout[i];
    if (out_logits) memcpy(out_logits + n * a, lg, sizeof(double) * a);
    int drawn = -1;
    if (uniforms) drawn = sample_policy(lg, a, kind, temp, topk, (double)uniforms[n], e, nl);
    if (out_sampled) out_sampled[n] = (uint8_t)(drawn < 0 ? 0 : drawn);
    int y = forced ? (int)forced[n] : drawn;
    out_codes[n] = (uint8_t)y;
    y2 = y1;
    y1 = y;
  }

  free(x); free(xnew); free(ap); free(ac); free(h); free(rh); free(q); free(sk);
  free(zs); free(za); free(lg); free(e); free(ring); free(ring_off);
  free(Wprev); free(Wcur); free(Bj); free(Wres); free(Bres); free(Wskip);
  free(W); free(d);
  return 0;
}

ORACLE_API int oracle_run_policy(int L, int r, int s, int a, const int32_t* dilations,
                                 const float* weights, int64_t numel, const float* cond,
                                 int64_t n_frames, int hop, const float* uniforms,
                                 const uint8_t* forced, int64_t N, uint8_t* out_codes,
                                 double* out_logits, uint8_t* out_sampled, int kind, double temp,
                                 int topk) {
  return oracle_run_nl(L, r, s, a, dilations, weights, numel, cond, n_frames, hop, uniforms, forced, N,
                       out_codes, out_logits, out_sampled, kind, temp, topk, 0);
}

ORACLE_API int oracle_run(int L, int r, int s, int a, const int32_t* dilations, const float* weights,
                          int64_t numel, const float* cond, int64_t n_frames, int hop, const float* uniforms,
                          const uint8_t* forced, int64_t N, uint8_t* out_codes, double* out_logits,
                          uint8_t* out_sampled) {
  return oracle_run_policy(L, r, s, a, dilations, weights, numel, cond, n_frames, hop, uniforms, forced, N,
                           out_codes, out_logits, out_sampled, 0, 1.0, 1);
}
