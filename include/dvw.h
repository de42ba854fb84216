/*
 * dvw.h -- C ABI of the B200-native autoregressive WaveNet sample generator
 * (Deep Voice, arXiv 1702.07825).  libdvw.so exports exactly these symbols.
 *
 * The operation (PAPER.md = the paper's LaTeX source):
 *   PAPER.md:416 (App. A)  "auto-regressive process P(y_i | c, y_{i-1}, ..., y_{i-R})"
 *   PAPER.md:340-377 (§5.1 steps 1-3) and PAPER.md:427-457 (App. A.1): per generated
 *     sample, the input 2x1 convolution done as two embedding lookups, l gated
 *     dilated 2x1 convolution layers with residual (r) and skip (s) projections,
 *     relu -> 1x1 -> relu -> 1x1 -> softmax over a = 256 mu-law levels,
 *   PAPER.md:376, 501 (App. A.4 direct sampling): draw y from p, feed it back.
 *   Conditioning is taken already computed, at frame rate, and upsampled by
 *   repetition inside the kernel (App. A.2).
 * DESIGN.md lists every reading of a point the paper leaves open (R1..R34);
 * the ones that fix the ABI's semantics are cited below.
 *
 * Conventions for every entry point:
 *   - returns dvw_status; DVW_OK = 0.  On any other status the thread-local
 *     text from dvw_last_error() says what was wrong.  No C++ exception ever
 *     crosses this boundary.
 *   - all tensors are row-major, little-endian, contiguous.
 *   - pointers are DEVICE pointers on the model's device unless the entry point
 *     name ends in _host or the argument says otherwise.  The caller owns every
 *     buffer it passes; the library never frees or retains them past the call.
 *   - calls are asynchronous on `cuda_stream` (a cudaStream_t, NULL = legacy
 *     default stream).  Argument errors and launch errors are returned
 *     immediately; device-side faults (a spin-wait watchdog firing) surface at
 *     dvw_sync() or at the next call on the handle.
 *   - a handle is not re-entrant: one call at a time.  Handles are independent.
 */
#ifndef DVW_H_
#define DVW_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DVW_API __attribute__((visibility("default")))
#else
#define DVW_API
#endif

typedef struct dvw_model dvw_model; /* opaque, owned by the library */

typedef enum {
  DVW_OK = 0,
  DVW_E_INVALID_ARG = 1,    /* null pointer, non-finite weights, bad enum value */
  DVW_E_SHAPE = 2,          /* sizes inconsistent: numel, n_frames < ceil(N/hop), hop < 1 ... */
  DVW_E_UNSUPPORTED = 3,    /* (r, s, a) or kernel choice this build does not implement */
  DVW_E_STATE = 4,          /* generate/logits before load_weights */
  DVW_E_OOM = 5,            /* device allocation failed */
  DVW_E_CUDA = 6,           /* CUDA runtime error (text has cudaGetErrorString) */
  DVW_E_DEVICE_TIMEOUT = 7  /* a persistent kernel's spin-wait watchdog fired */
} dvw_status;

/* Model sizes (§3.4: l layers, r residual, s skip channels;
 * a = 256 mu-law levels).
 *   n_layers  l >= 1
 *   residual  r in {32, 64, 128}
 *   skip      s in {128, 256}
 *   levels    a, must be 256
 *   dilations length l, each >= 1, copied at create time; NULL selects
 *             d_j = 2^((j-1) mod 10) (reading R2: the only cycle consistent with
 *             PAPER.md:166's 83 ms receptive field for l = 40 at 48 kHz)
 *   device    CUDA ordinal the handle lives on */
typedef struct {
  int32_t n_layers;
  int32_t residual;
  int32_t skip;
  int32_t levels;
  const int32_t* dilations;
  int32_t device;
} dvw_config;

/* Kernel selection.  AUTO: dvw_generate picks CLUSTER when the model
 * fits its residency plan, the sampler is direct and n_streams is at most the number of
 * clusters the device runs at once times 16 (one cluster per stream, the rest in waves),
 * TC for larger batches, else STREAM; dvw_logits picks PARALLEL.  A pinned CLUSTER kernel
 * takes any n_streams (clusters beyond the co-resident count run in waves). */
typedef enum {
  DVW_KERNEL_AUTO = 0,
  DVW_KERNEL_STREAM = 1,   /* one CTA per stream, weights read from L2 every sample */
  DVW_KERNEL_CLUSTER = 2,  /* batch-1 persistent cluster kernel, weights on chip */
  DVW_KERNEL_TC = 3,       /* batched streams, tcgen05 projections */
  DVW_KERNEL_PARALLEL = 4  /* dvw_logits only: all timesteps of a layer at once (codes known) */
} dvw_kernel;

typedef struct {
  int32_t last_kernel;       /* dvw_kernel that ran the last generate/logits call */
  int32_t last_grid;         /* CTAs launched */
  int32_t last_cluster;      /* cluster size (1 = none) */
  int32_t last_threads;      /* threads per CTA */
  int64_t last_launches;     /* kernel launches issued by the last call */
  int64_t weight_bytes;      /* bytes of packed device weights the handle owns */
  int64_t workspace_bytes;   /* bytes of per-stream state (dilation rings) */
  int32_t chain_ctas;        /* cluster kernel's plan: chain CTAs (layers per CTA = ceil(l / chain_ctas)); 0 if none */
  int32_t max_clusters;      /* cluster kernel's plan: clusters co-resident on the device */
  int32_t streams_per_cluster;  /* cluster kernel, last call: streams interleaved per cluster (1 = one each) */
  int32_t max_clusters_pipe;    /* cluster kernel's plan: co-resident clusters of the multi-stream variant (0: none) */
} dvw_info;

/* Create a handle on cfg->device.  Validates sizes (DVW_E_SHAPE / DVW_E_UNSUPPORTED).
 * *out is set only on DVW_OK. */
DVW_API dvw_status dvw_create(const dvw_config* cfg, dvw_model** out);

/* Expected weight-blob length in floats (no handle needed):
 *   l (5 r^2 + 3 r + r s) + 2 r a + r + s + a s + a + a^2 + a.
 * Returns -1 for an invalid config. */
DVW_API int64_t dvw_weights_numel(const dvw_config* cfg);

/* Load the weights.  blob: fp32, numel floats, in this order:
 *   for j = 1..l: W_prev[2r][r]  W_cur[2r][r]  B[2r]  W_res[r][r]  B_res[r]  W_skip[s][r]
 *   then W_emb_prev[r][a]  W_emb_cur[r][a]  B_emb[r]  B_skip[s]
 *        W_relu[a][s]  B_relu[a]  W_out[a][a]  B_out[a]
 *   Rows 0..r-1 of W_prev, W_cur, B feed tanh, rows r..2r-1 feed the sigmoid
 *   (reading R7).  One bias B per layer (reading R8).
 * blob_on_device != 0: blob is a device pointer on the model's device, else host.
 * The library builds its own packed device copy (residency layout); the caller may
 * free blob when this returns.  Synchronous.  Non-finite values -> DVW_E_INVALID_ARG;
 * numel mismatch -> DVW_E_SHAPE. */
DVW_API dvw_status dvw_load_weights(dvw_model* m, const float* blob, int64_t numel,
                                    int32_t blob_on_device);

/* Free-running generation (App. A.4 direct sampling).
 *   cond      fp32 [n_streams][n_frames][l][2r]: L^(j) for frame f; sample n uses
 *             frame n / hop (repetition upsampling; readings R5, R6).
 *             Requires n_frames >= ceil(n_samples / hop) and hop >= 1.
 *   uniforms  fp32 [n_streams][n_samples] in [0, 1): u_n for the inverse-CDF draw
 *             y_n = min{k : u_n * P_255 < P_k}, P_k the fp64 running sum of
 *             exp(l_i - max l) in ascending code order (reading R11).  Values
 *             outside [0,1) are not validated (precondition).
 *   out_codes uint8 [n_streams][n_samples]: the emitted mu-law codes.
 * Every call starts from the fresh state: dilation queues zero, codes at negative
 * times 128 = mu-law(0) (reading R4).  Results are bitwise deterministic for the
 * same inputs, independent of n_streams and of the stream's position (R20). */
DVW_API dvw_status dvw_generate(dvw_model* m, const float* cond, int64_t n_frames, int32_t hop,
                                const float* uniforms, int64_t n_samples, int32_t n_streams,
                                uint8_t* out_codes, void* cuda_stream);

/* Teacher-forced evaluation: the same network, but the code fed back after step n
 * is codes[n] (uint8 [n_streams][n_samples]); writes the PRE-softmax logits
 * l = W_out z_a + B_out (reading R15) to
 * out_logits fp32 [n_streams][n_samples][256].  logits[n] depends on codes[0..n-1]. */
DVW_API dvw_status dvw_logits(dvw_model* m, const float* cond, int64_t n_frames, int32_t hop,
                              const uint8_t* codes, int64_t n_samples, int32_t n_streams,
                              float* out_logits, void* cuda_stream);

/* dvw_generate with HOST buffers (pageable or pinned): copies cond and uniforms
 * to library-owned device staging, generates, copies the codes back, and
 * synchronizes before returning.  Used for end-to-end timing. */
DVW_API dvw_status dvw_generate_host(dvw_model* m, const float* cond_host, int64_t n_frames,
                                     int32_t hop, const float* uniforms_host, int64_t n_samples,
                                     int32_t n_streams, uint8_t* out_codes_host,
                                     void* cuda_stream);

/* Streaming (stateful) generation: one utterance in consecutive chunks, the output of the
 * chunks bitwise equal to a single dvw_generate over their concatenation (SURVEY.md §8(f)
 * "streaming/stateful generation across calls").  The session owns the state a one-shot call
 * rebuilds from zero (reading R4): every stream's dilation queues and its last two codes.
 *   dvw_session_create   : state for n_streams utterances of model m (queues zero, codes 128)
 *   dvw_session_generate : the next n_samples of every stream.  cond covers the WHOLE
 *                          utterance, fp32 [n_streams][n_frames][l][2r] with
 *                          n_frames >= ceil((position + n_samples) / hop); uniforms and
 *                          out_codes are the chunk's, [n_streams][n_samples].  hop must not
 *                          change within a session.  AUTO runs up to the co-resident
 *                          cluster count of streams on the CLUSTER kernel (direct sampler,
 *                          exact gate), larger batches on the batched TC kernel (the session
 *                          then keeps its workspace: queues, x^(0) and codes of every launch
 *                          group), else the STREAM kernel -- re-resolved on every call, since
 *                          CLUSTER and STREAM share one state layout (a session moves between
 *                          them when the sampler or precision changes).  A TC session stays
 *                          on TC; a call pinned to a kernel with another state layout ->
 *                          DVW_E_STATE.  Calls on one session must be ordered
 *                          (same CUDA stream).
 *   dvw_session_position : samples generated so far (-1 for NULL)
 * The session is bound to the model's device and dilation schedule. */
typedef struct dvw_session dvw_session;
DVW_API dvw_status dvw_session_create(dvw_model* m, int32_t n_streams, dvw_session** out);
DVW_API dvw_status dvw_session_generate(dvw_model* m, dvw_session* s, const float* cond, int64_t n_frames,
                                        int32_t hop, const float* uniforms, int64_t n_samples,
                                        uint8_t* out_codes, void* cuda_stream);
DVW_API int64_t dvw_session_position(const dvw_session* s);
DVW_API void dvw_session_destroy(dvw_session* s);

/* Pin the kernel used by later calls (DVW_KERNEL_AUTO restores the default).
 * DVW_E_UNSUPPORTED if that kernel cannot run this model. */
DVW_API dvw_status dvw_set_kernel(dvw_model* m, int32_t kernel);

/* Arithmetic precision of the batched tcgen05 kernel:
 *   DVW_PRECISION_FP32 (default) : every fp32 operand is split into a tf32 head and its
 *     exact residual and each product is issued as hi*[hi; lo] + lo*hi (reading R23):
 *     teacher-forced logits within ~1e-6 of the fp64 oracle, codes bit-exact.
 *   DVW_PRECISION_TF32           : one pass, A_hi * W_hi (inputs rounded to tf32,
 *     10-bit mantissa; fp32 accumulation): half the staged activation bytes and a third
 *     of the MMAs.  Logits stay within the north_star's 1e-3 teacher-forced gate
 *     (measured error reported by bench.py / tests), but free-running codes are NOT
 *     bit-exact with the fp64 oracle: they diverge at a measured per-step rate.
 * The batch-1 kernels (CLUSTER, STREAM) are fp32 FMA kernels and ignore the setting.
 * Unknown value -> DVW_E_INVALID_ARG. */
/*   DVW_PRECISION_APPROX         : the GPU analogue of the paper's approximate
 *     nonlinearities (App. C): the batch-1 kernels
 *     (CLUSTER, STREAM) evaluate the gate with the hardware tanh unit (tanh.approx.f32,
 *     relative error ~2^-11; sigma(g) = (1 + tanh(g/2)) / 2) -- a shorter gate on the
 *     critical chain; logits within the 1e-3 gate, codes not bit-exact (measured rate
 *     reported).  The batched kernel runs as DVW_PRECISION_TF32 under this setting. */
/*   DVW_PRECISION_APPC           : the paper's own approximations (App. C, PAPER.md:551-592;
 *     reading R31): tanh and sigma from e~(x) = 1 + |x| + 0.5658 x^2 + 0.143 x^4 in every
 *     gate, and the softmax's e^x by the 2^x bit-pattern construction with the rational
 *     g(z) in the sampler (all strategies).  CLUSTER, STREAM (generation, sessions) and
 *     PARALLEL (logits) kernels; TC -> DVW_E_UNSUPPORTED (AUTO picks CLUSTER, else STREAM,
 *     for batches).
 *     Parity is with the oracle's App. C mode (oracle.run(..., nonlin="appc")). */
typedef enum {
  DVW_PRECISION_FP32 = 0,
  DVW_PRECISION_TF32 = 1,
  DVW_PRECISION_APPROX = 2,
  DVW_PRECISION_APPC = 3
} dvw_precision;
DVW_API dvw_status dvw_set_precision(dvw_model* m, int32_t precision);

/* Weight quantisation ("inference with weight matrices quantized to int16";
 * SURVEY.md §8(f) row f4; reading R32).  bits = 16 or 8: at the NEXT
 * dvw_load_weights every weight matrix (W_prev, W_cur, W_res, W_skip per layer; W_emb_prev,
 * W_emb_cur, W_relu, W_out) is quantised symmetrically per row, in fp32 arithmetic:
 *   s = max_c |W[row][c]| / (2^(bits-1) - 1),  q = rint(W / s) (half to even),  W := q s
 * (rows of zeros stay zero); biases stay fp32.  Every kernel then runs on the quantised
 * values (fp32 storage: the weights are resident on chip, so the batch-1 path gains no
 * bandwidth from narrower storage -- the tier measures what the quantisation costs in
 * accuracy).  bits = 0 (default) loads the blob unchanged.  Other values ->
 * DVW_E_INVALID_ARG. */
DVW_API dvw_status dvw_set_weight_bits(dvw_model* m, int32_t bits);

/* The same quantisation with a choice of scale granularity (reading R33):
 *   scheme DVW_QUANT_PER_ROW    (0): one scale per matrix row, as dvw_set_weight_bits;
 *   scheme DVW_QUANT_PER_TENSOR (1): one scale per weight matrix, s = max|W| / (2^(bits-1) - 1)
 *     (an all-zero matrix keeps s = 1), q = rint(W / s), W := q s -- SPEC.md's
 *     QuantizedWeightSet scheme (e.g. [0, 1, -1] -> q = [0, 32767, -32767] at 16 bits,
 *     s = 1/32767); |W - q s| <= s/2 elementwise.
 * bits as dvw_set_weight_bits (0 turns quantisation off; scheme is then ignored).
 * Unknown scheme or bits -> DVW_E_INVALID_ARG. */
typedef enum { DVW_QUANT_PER_ROW = 0, DVW_QUANT_PER_TENSOR = 1 } dvw_quant_scheme;
DVW_API dvw_status dvw_set_weight_quant(dvw_model* m, int32_t bits, int32_t scheme);

/* Sampling strategy for dvw_generate (App. A.4).
 * Details the paper leaves open follow DESIGN.md readings R24-R27:
 *   DVW_SAMPLER_DIRECT      (default) inverse-CDF draw from P with u_n (reading R11)
 *   DVW_SAMPLER_TEMPERATURE from P_t = P^(1/t) / Z, same inverse-CDF rule with u_n
 *   DVW_SAMPLER_MEAN        round(E_P[y]) = floor(sum_y y P(y) + 0.5); u_n unused
 *   DVW_SAMPLER_MODE        argmax P (lowest code on ties); u_n unused
 *   DVW_SAMPLER_TOP_K       the k largest P(y) kept (ties by lower code), renormalised,
 *                           inverse-CDF rule with u_n
 * temperature must be finite and > 0 (used by TEMPERATURE only), 1 <= top_k <= 256 (TOP_K
 * only); otherwise DVW_E_INVALID_ARG.  The batched (TC) and STREAM kernels implement every
 * strategy; the batch-1 CLUSTER kernel only DIRECT (pinning CLUSTER with another strategy
 * makes generate return DVW_E_UNSUPPORTED; AUTO then runs STREAM for a single stream).
 * dvw_logits is unaffected. */
typedef enum {
  DVW_SAMPLER_DIRECT = 0,
  DVW_SAMPLER_TEMPERATURE = 1,
  DVW_SAMPLER_MEAN = 2,
  DVW_SAMPLER_MODE = 3,
  DVW_SAMPLER_TOP_K = 4
} dvw_sampler;
DVW_API dvw_status dvw_set_sampler(dvw_model* m, int32_t kind, float temperature, int32_t top_k);

/* Tracing: when device_buf != NULL, persistent kernels record timestamps at fixed
 * events of samples [first_sample, first_sample + n_samples) into device_buf, uint64
 * [n_samples][16 cluster ranks][32 events] (unwritten slots keep their old value; the
 * caller zero-fills).  Time base per slot: on the cluster kernel's chain CTAs events
 * 0, 2, 3, 5 and 20 are %globaltimer nanoseconds and events 1, 4, 6-19 and 21-30 are
 * that SM's clock64 cycles (one-store stamps inside a layer, comparable only within one
 * CTA and sample); every event of the head and skip CTAs, and of the batched kernel, is
 * %globaltimer ns.  Event meaning per role: tools/trace_c2.py, tools/trace_batch.py.
 * Tracing runs the exact-gate kernels: with DVW_PRECISION_APPROX / APPC the cluster
 * kernel returns DVW_E_UNSUPPORTED.  NULL disables tracing.  Off the hot path when
 * disabled. */
DVW_API dvw_status dvw_set_trace(dvw_model* m, uint64_t* device_buf, int64_t first_sample, int32_t n_samples);

/* Launch bookkeeping of the last call (filled synchronously, host side). */
DVW_API dvw_status dvw_get_info(const dvw_model* m, dvw_info* out);

/* Latency floor of the batch-1 critical path (SURVEY.md §8(d) "measured latency floor";
 * PAPER.md:225-229 per-layer budget, PAPER.md:600-606 synchronisation as the GPU bottleneck).
 * Runs four microbenchmarks on `device` (a few ms, synchronous) built from the cluster
 * kernel's own device functions, each timed with clock64 on one SM:
 *   layer_cycles      one chain layer alone: LDS of h, the 2r x r matvec, pair shuffle, gate,
 *                     STS of h and the named barrier that publishes it (r = 64)
 *   hop_cycles        one DSMEM hand-off between two CTAs of a cluster (st.async completing
 *                     transaction bytes on the peer's mbarrier; ping-pong / 2)
 *   head_stage_cycles one head stage: a 64-row slice of a 256 x 256 matvec, the transposing
 *                     shuffle reduction, STS and a 256-thread barrier
 *   sampler_cycles    one inverse-CDF draw by one warp
 *   sm_ghz            SM clock during the probe (clock64 / %globaltimer over ~10 ms)
 * The floor of a model on the cluster kernel is l x layer + (chain CTAs + 2) x hop +
 * 3 x head_stage + sampler (bench.py "roofline").  Errors: DVW_E_INVALID_ARG (NULL out,
 * bad device), DVW_E_CUDA. */
typedef struct {
  double layer_cycles, hop_cycles, head_stage_cycles, sampler_cycles, sm_ghz;
} dvw_floor;
DVW_API dvw_status dvw_measure_floor(int32_t device, dvw_floor* out);

/* Wait for the handle's outstanding work; returns DVW_E_DEVICE_TIMEOUT if a
 * device watchdog fired, DVW_E_CUDA on an asynchronous CUDA error. */
DVW_API dvw_status dvw_sync(dvw_model* m);

/* Release the handle and everything it owns.  NULL is a no-op. */
DVW_API void dvw_destroy(dvw_model* m);

/* Thread-local text for the last non-OK status ("" if none). */
DVW_API const char* dvw_last_error(void);

/* ---------------------------------------------------------------------------------------
 * Conditioning network (App. A.2): features at
 * frame rate -> the per-layer conditioning `cond` dvw_generate consumes.  Two bidirectional
 * QRNN layers with fo-pooling and 2x1 convolutions,
 *   h~ = tanh(W_h * x + B_h), o = sigma(W_o * x + B_o), f = sigma(W_f * x + B_f),
 *   h_t = f_t h_{t-1} + (1 - f_t) h~_t, z_t = o_t h_t, h_0 = 0,
 * the backward QRNN running on the reversed sequence (its taps are x_{t+1}, x_t; reading
 * R28), channels stacked [forward | backward] per layer, interleaved after the second layer
 * (channel 2i forward i, 2i+1 backward i; R29), then one projection per WaveNet layer,
 * L^(j)_t = P^(j) out_t + B^(j) (R30).  Upsampling by repetition happens inside
 * dvw_generate (hop).  fp32, bitwise deterministic.
 *
 * Weight blob (fp32, this order): for QRNN layer q = 1, 2 (C_in = in_channels, then
 * 2 hidden), for the forward then the backward direction: W [3 gates h,o,f][2 taps: older,
 * current][hidden][C_in], B [3][hidden]; then P [n_layers][2 residual][2 hidden] and
 * B_P [n_layers][2 residual].
 * dvwc_run: features fp32 [n_streams][n_frames][in_channels] (device), out_cond fp32
 * [n_streams][n_frames][n_layers][2 residual] (device) -- exactly dvw_generate's cond layout.
 * Same conventions as the generator: stream-ordered, asynchronous, caller owns buffers,
 * errors via dvw_last_error(). */
typedef struct dvwc_model dvwc_model;
typedef struct {
  int32_t in_channels;  /* feature channels per frame (1..3228: frames are staged in shared memory;
                           larger -> DVW_E_UNSUPPORTED at dvwc_create) */
  int32_t hidden;       /* QRNN channels per direction (1..1024) */
  int32_t n_layers;     /* l of the WaveNet it conditions */
  int32_t residual;     /* r of the WaveNet it conditions */
  int32_t device;
} dvwc_config;
DVW_API dvw_status dvwc_create(const dvwc_config* cfg, dvwc_model** out);
DVW_API int64_t dvwc_weights_numel(const dvwc_config* cfg);
DVW_API dvw_status dvwc_load_weights(dvwc_model* m, const float* blob, int64_t numel, int32_t blob_on_device);
DVW_API dvw_status dvwc_run(dvwc_model* m, const float* features, int64_t n_frames, int32_t n_streams,
                            float* out_cond, void* cuda_stream);
DVW_API void dvwc_destroy(dvwc_model* m);

#ifdef __cplusplus
}
#endif
#endif /* DVW_H_ */
