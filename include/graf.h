/*
 * graf.h — C ABI of the B200 (sm_100a) GRAF ambiguity-function hot path.
 *
 * Operation (BASELINE.json north_star; aperiodic, M-bin, e^{-j} form of the
 * paper's Eq. 2, PAPER.md L121 / Eq. 7, readings R1-R5 in DESIGN.md §2):
 *
 *   A[k,m] = sum_{n} s[n] * conj(s[n-k]) * exp(-2*pi*j*m*n/M),
 *            k in [-(N-1), N-1], m in [0, M), terms with n-k outside [0,N) are 0.
 *
 * computed as delay-lag products (Eqs. 8-10) followed by a
 * length-M Doppler FFT per delay row (Eq. 11; Algorithm 1 steps 1-3,
 * L245-250), its magnitude (Eq. 12; Alg. 1 step 4), the sidelobe losses
 * ISL (Eq. 20) and log-sum-exp soft-PSL (smoothed Eq. 19)
 * over a region mask, and the Wirtinger adjoint dL/ds* (Eqs. 13-15).
 *
 * Conventions shared by every entry point:
 *  - All data pointers (s, surface, dA, grad, loss, partials unless stated,
 *    w_k, w_d, workspace) are DEVICE pointers owned by the caller.  The
 *    library never allocates or frees device memory, never synchronises the
 *    device, and enqueues all work on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream).  Results are complete when the stream
 *    reaches them.
 *  - Complex data are complex64 interleaved (re, im float32), row-major:
 *    s [B][N]; surface / dA [B][k_end-k_begin][M] with row index k-k_begin and
 *    Doppler column m (GRAF_DOPPLER_RAW) or j = d + M/2 with centred Doppler
 *    d = m (m < M/2) else m - M (GRAF_DOPPLER_CENTERED, Alg. 1 step 5 fftshift,
 *    L252).  Pointers must be 16-byte aligned.
 *  - Gradients are Wirtinger cotangents g = dL/ds* (PAPER
 *    L219): dL/dRe s = 2 Re g, dL/dIm s = 2 Im g.  Outputs are overwritten,
 *    never accumulated.  Torch's complex .grad equals 2*g.
 *  - Reentrant: no mutable global state except an immutable per-device table
 *    of M-th roots of unity.  It is filled by a small kernel enqueued on the
 *    stream of the first call on a device (or of graf_init); calls on other
 *    streams are ordered after it with an event wait, and a first call made
 *    inside CUDA-graph capture records the fill into the graph.  No call ever
 *    blocks the host or synchronises the device.
 *  - Deterministic: fixed reduction order, no floating-point atomics; a call
 *    repeated on the same inputs returns bitwise-identical outputs.
 *  - Errors: argument checks happen on the host before any launch and return a
 *    non-OK status with a message in graf_last_error() (thread-local).  A CUDA
 *    launch failure returns GRAF_ECUDA.  Value-dependent problems (E = 0,
 *    NaN/Inf in s) are not detected: they propagate as IEEE NaN.
 *  - v1 device limits: M a power of two with max(N,2) <= M <= 16384; N >= 1.
 */
#ifndef GRAF_H_
#define GRAF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GRAF_ABI_VERSION 6
#define GRAF_MAX_M 16384

typedef enum {
  GRAF_OK = 0,
  GRAF_EINVAL = 1,        /* malformed argument (sizes, ranges, NULL, alignment) */
  GRAF_EUNSUPPORTED = 2,  /* well-formed but outside v1 device limits (M > 16384, M < N, ...) */
  GRAF_ECUDA = 3,         /* a CUDA runtime call or launch failed */
  /* 4 is unused: value-dependent problems are never detected (no host sync), see above */
  GRAF_EWORKSPACE = 5     /* ws_bytes < graf_workspace_bytes(...) */
} graf_status;

typedef enum {
  GRAF_OUT_NONE = 0,
  GRAF_OUT_C64 = 1,       /* A (complex64) */
  GRAF_OUT_ABS_F32 = 2,   /* |A| (float32) */
  GRAF_OUT_POW_F32 = 3    /* chi = |A|^2 (float32), Alg. 1 step 4 */
} graf_out_kind;

typedef enum { GRAF_DOPPLER_RAW = 0, GRAF_DOPPLER_CENTERED = 1 } graf_doppler_layout;

/* Problem geometry and surface output. */
typedef struct {
  int32_t abi_version;      /* must equal GRAF_ABI_VERSION */
  int32_t n;                /* N >= 1: waveform length */
  int32_t m;                /* M: Doppler bins, power of two, max(N,2) <= M <= 16384 */
  int32_t out_kind;         /* graf_out_kind of `surface` (GRAF_OUT_NONE: no surface) */
  int64_t batch;            /* B >= 1 waveforms */
  int32_t k_begin, k_end;   /* surface / dA delay-row window, -(N-1) <= k_begin < k_end <= N */
  int32_t doppler_layout;   /* graf_doppler_layout of surface and dA */
  int32_t normalize_output; /* 1: surface holds A/E, |A|/E, chi/E^2 (Eq. 17 analogue: max chi = E^2, L265-268) */
  int32_t shard_index;      /* delay sharding of the LOSS rows: this call handles the folded */
  int32_t shard_count;      /*   delay rows k >= 0 with k % shard_count == shard_index (0/1 = all) */
  int32_t periodic;         /* 0: aperiodic (above).  1: the paper's circular surface, Eq. 2 (L121)
                               and Algorithm 1 (L239-256) with the FFT's e^{-j} (reading R2):
                               A[k,m] = sum_{n<N} s[n] conj(s[(n-k) mod N]) exp(-2 pi j m n/M);
                               requires M == N.  Rows of the window are delays taken mod N
                               (k_end - k_begin <= N; [-N/2, N/2) with GRAF_DOPPLER_CENTERED is
                               Alg. 1's two-axis fftshift, L252).  The loss region uses the
                               circular delay distance min(k mod N, N - k mod N) <= k_max and
                               weights w_k[k + N - 1] for k in (-N/2, N/2].  (ABI v2) */
  const int32_t* skip;      /* nullable device int32 [B]: waveforms b with skip[b] != 0 are not
                               computed, and every per-waveform output of theirs (surface rows,
                               partials, loss, grad) is left untouched.  A guarded re-run of a
                               batch (the sharded single pass's fallback) costs nothing for the
                               skipped waveforms and needs no host-side decision.  Honoured by
                               graf_af_forward / _loss_grad / _backward; the sp_* and xaf_* entry
                               points return GRAF_EUNSUPPORTED when it is set.  (ABI v6) */
} graf_af_desc;

/* Loss over the sidelobe region Omega_s (never defined by the paper,
 * reading R7):  |k| <= k_max, |d| <= d_max, minus the mainlobe |k| <= ml_k && |d| <= ml_d.
 *   x   = chi/E^2 (normalize = 1, Eqs. 19-20 divide by chi(0,0) = E^2) or chi (0)
 *   ISL = sum_{Omega} w*x,  w = w_k[k+N-1] * w_d[d+M/2] (NULL = 1)        (Eq. 20)
 *   softPSL = T*log sum_{Omega} exp(x/T)                                   (Eq. 19, smoothed)
 *   L   = lambda_isl*ISL + lambda_psl*softPSL per waveform                 (Eq. 23 weights, L313)
 * The row-folding (k >= 0 only) used by the kernels requires symmetric weights:
 * w_k[N-1+k] == w_k[N-1-k] and w_d[M/2+d] == w_d[M/2-d]; the caller guarantees it. */
typedef struct {
  int32_t k_max, d_max;     /* >= 0 */
  int32_t ml_k, ml_d;       /* mainlobe half-widths, >= 0 */
  const float* w_k;         /* optional device [2N-1] delay weights */
  const float* w_d;         /* optional device [M] Doppler weights */
  float lambda_isl, lambda_psl;
  float temperature;        /* T > 0 (read iff lambda_psl != 0), in the units of x.  The kernels
                               form (x - LSE)/T in fp32, so T must be well above the rounding of
                               max x, ~6e-8 max x: with normalize = 1 (x <= 1) any T >= 1e-5 is
                               safe (the configs use 0.01); with raw chi (x ~ E^2) T = 0.01 is
                               below fp32 resolution and the soft-PSL gradient is not reliable
                               (reading R30).  Not checked at run time. */
  int32_t normalize;        /* 1 (default reading R6) or 0 (raw chi) */
  float lambda_hpsl;        /* weight of the HARD PSL = max_{Omega} x (Eq. 19) with its
                               argmax subgradient (the paper's section-7 loss, L416); ties go to
                               the lowest row-major (delay, raw Doppler bin) cell (reading R23).
                               Needs the global max, so it runs pass 1 like soft-PSL.  (ABI v3) */
  float lambda_match;       /* weight of the match loss ||x - target||^2 summed over Omega (
                               reading R24).  Not combinable with soft-PSL (lambda_psl != 0). */
  const float* target;      /* device fp32 target x_target laid out like the surface window of
                               graf_af_desc ([k_end - k_begin][M], doppler_layout; periodic: a full
                               window of N delays); the window must hold every delay of Omega */
  int64_t target_stride;    /* floats between waveforms' targets (0: one target for the batch) (ABI v4) */
} graf_loss_desc;

/* Per-waveform partial sums over the rows a call covered (exactly combinable
 * across delay shards with graf_combine_partials):
 *   isl_sum = sum w*chi (raw numerator);  lse_max = max x (= the hard PSL);
 *   lse_sum = sum exp((x - lse_max)/T);   cen_sum = sum expm1((x - xbar)/T) with
 *   xbar = (M-1)/|Omega| when Omega is constant-sum (reading R13), else 0;
 *   psl_key = row-major key (delay index * M + raw Doppler bin, delays ascending from
 *   the smallest delay of the region) of the argmax cell (lambda_hpsl != 0 only). */
typedef struct { double isl_sum, lse_max, lse_sum, cen_sum, psl_key, reserved; } graf_partials;

int32_t graf_abi_version(void);
const char* graf_status_string(graf_status status);
const char* graf_last_error(void);

/* Optional explicit initialisation of the current device: enqueues the fill of the
 * roots-of-unity table on `stream` (the first entry-point call does the same when it
 * has not happened).  Never blocks.  (ABI v6) */
graf_status graf_init(void* stream);

/* Bytes of device workspace the call with these descriptors needs (0 on
 * invalid descriptors).  Same value for graf_af_forward, graf_af_loss_grad and
 * graf_af_backward with the same descriptors; loss may be NULL. */
size_t graf_workspace_bytes(const graf_af_desc* af, const graf_loss_desc* loss);

/* Forward.  Writes the surface window (if af->out_kind != NONE; `surface` must
 * then be non-NULL) and, if `loss` != NULL, this shard's graf_partials[B] into
 * `partials` (device).  Kernels: lag product -> Stockham FFT -> epilogue. */
graf_status graf_af_forward(const graf_af_desc* af, const graf_loss_desc* loss,
                            const void* s, void* surface, graf_partials* partials,
                            void* ws, size_t ws_bytes, void* stream);

/* Loss and gradient.  `global` = combined partials [B] of ALL shards (device), or
 * NULL to compute them here (unsharded call).  Writes loss[B] (double, may be
 * NULL) and grad[B][N] = dL/ds* restricted to this shard's delay rows, including
 * this shard's share of the normalization term, so the SUM over shards is the
 * full gradient.  Optionally writes the surface window too (af->out_kind).
 * ISL-only losses (lambda_psl == 0) run as ONE fused pass (forward, epilogue,
 * inverse FFT, delay correlation); soft-PSL needs the global LSE and runs two.
 * Sharded calls without `global`: the loss is this shard's part of a sum over shards
 * (ISL and match terms are linear in the rows).  A shard that owns no loss rows writes
 * grad 0 and loss 0 then; with soft-PSL or hard-PSL terms, which need the global
 * statistic, `global` is required (GRAF_EINVAL before any launch otherwise). */
graf_status graf_af_loss_grad(const graf_af_desc* af, const graf_loss_desc* loss,
                              const void* s, const graf_partials* global,
                              double* loss_out, void* grad, void* surface,
                              void* ws, size_t ws_bytes, void* stream);

/* Generic adjoint for arbitrary losses of A:  given dA = dL/dA* over the rows
 * [k_begin, k_end) (complex64 [B][rows][M], af->doppler_layout), write
 * grad[B][N] = dL/ds* = sum_k (term1 + term2) of the inverse Doppler DFT of dA
 * ("IFFT operation (linear)", Eq. 15).  Linear in dA. */
graf_status graf_af_backward(const graf_af_desc* af, const void* s, const void* dA,
                             void* grad, void* ws, size_t ws_bytes, void* stream);

/* Delay-sharded SINGLE pass of the full-plane centred soft-PSL (DESIGN.md readings
 * R13 and R27).  An unsharded graf_af_loss_grad already runs such a
 * loss as one optimistic pass.  Across shards, the scale 1/Z_c and the validity rule
 * need global sums, so the pass is split in two phases around the caller's exchange:
 *   1. graf_af_loss_grad_sp_begin: this shard's rows (af->shard_index / shard_count >= 2)
 *      run once with f' = lambda expm1((x - xbar)/T).  It writes this shard's partials
 *      [B] (device), to be combined over ALL shards in rank order with
 *      graf_combine_partials.  It keeps the unscaled gradient in `ws`.
 *   2. graf_af_loss_grad_sp_end: takes `global` = the combined partials (device [B]).
 *      It applies the R13 rule max x - xbar <= 40 T per waveform.  It writes loss[B]
 *      (nullable) and this shard's grad[B][N], scaled by the global 1/Z_c.  The SUM over
 *      shards is dL/ds*.  valid[B] (int32, nullable) is 1 where the rule holds.  Where it
 *      fails, it writes loss NaN and grad 0; the caller then recomputes that batch with
 *      the two-pass protocol (graf_af_forward partials -> combine -> graf_af_loss_grad
 *      with `global`).  All shards see the same `global`, so they agree.
 * Both phases take the same descriptors and the SAME workspace (graf_workspace_bytes),
 * which must not be reused in between.
 * Errors: GRAF_EINVAL for shard_count < 2, NULL or misaligned buffers, or a small
 * workspace.  GRAF_EUNSUPPORTED unless graf_af_single_pass_eligible(af, loss) holds:
 * the loss region is the full plane with no mainlobe cut, normalize = 1, no weights,
 * lambda_psl != 0, no hard-PSL or match term, and no surface output. */
int32_t graf_af_single_pass_eligible(const graf_af_desc* af, const graf_loss_desc* loss);
graf_status graf_af_loss_grad_sp_begin(const graf_af_desc* af, const graf_loss_desc* loss, const void* s,
                                       graf_partials* partials, void* ws, size_t ws_bytes, void* stream);
graf_status graf_af_loss_grad_sp_end(const graf_af_desc* af, const graf_loss_desc* loss, const void* s,
                                     const graf_partials* global, double* loss_out, void* grad,
                                     int32_t* valid, void* ws, size_t ws_bytes, void* stream);

/* Cross-ambiguity ("cross-ambiguity" for MIMO):
 *   X[k,m] = sum_n s1[n] conj(s2[n-k]) exp(-2 pi j m n / M),  k in [-(N-1), N-1],
 * the same kernels with the second waveform staged beside the first.  Rows are NOT
 * folded (X has no mirror symmetry).  Normalised quantities use E1 E2 in place of
 * E^2 (reading R25: |X| <= sqrt(E1 E2), = E^2 when s1 = s2); the surface with
 * normalize_output holds X / sqrt(E1 E2).  The loss call returns both Wirtinger
 * gradients: grad1 = dL/ds1*, grad2 = dL/ds2* (complex64 [B][N]).  v1 limits
 * (GRAF_EUNSUPPORTED otherwise): aperiodic, unsharded, M <= 4096, unweighted ISL
 * and soft-PSL (no hard PSL / match).  Workspace: graf_xaf_workspace_bytes. */
size_t graf_xaf_workspace_bytes(const graf_af_desc* af, const graf_loss_desc* loss);
graf_status graf_xaf_forward(const graf_af_desc* af, const graf_loss_desc* loss, const void* s1,
                             const void* s2, void* surface, graf_partials* partials, void* ws,
                             size_t ws_bytes, void* stream);
graf_status graf_xaf_loss_grad(const graf_af_desc* af, const graf_loss_desc* loss, const void* s1,
                               const void* s2, const graf_partials* global, double* loss_out,
                               void* grad1, void* grad2, void* surface, void* ws, size_t ws_bytes,
                               void* stream);
graf_status graf_xaf_backward(const graf_af_desc* af, const void* s1, const void* s2, const void* dA,
                              void* grad1, void* grad2, void* ws, size_t ws_bytes, void* stream);

/* Spectral variance of each waveform (the paper's section-7 LPI term, L417):
 *   SV_b = var{ |F s_b|^2 / sum |F s_b|^2 } over the N DFT bins, F the length-N DFT,
 *   var = sum (p - mean p)^2 / (N - ddof): ddof = 0 population variance (SPEC.md L328,
 *   the default of the binding; reading R22), ddof = 1 the unbiased estimator (PyTorch's
 *   var default).  (ABI v6)
 * and its Wirtinger gradient dSV/ds*.  Writes weight*SV_b into loss[b] and
 * weight*dSV/ds* into grad[b][:], or ADDS them when accumulate = 1 (to combine
 * with a graf_af_loss_grad result: the Eq. 26 loss PSL + lambda*alpha*SV).
 * weights: device float [B] per-waveform weights (e.g. lambda_b * alpha for a
 * batched lambda sweep), or NULL to use `weight` for every waveform.
 * s, grad: complex64 [B][N]; loss: double [B] (nullable).  N a power of two,
 * 2 <= N <= 16384.  No workspace. */
graf_status graf_spectral_variance(int64_t batch, int32_t n, const void* s, float weight,
                                   const float* weights, double* loss, void* grad, int32_t accumulate,
                                   int32_t ddof, void* stream);

/* Differentiable mainlobe width:
 *   W_b = sum_tau |tau| sigma(gamma (chi(tau,0) - chi(0,0)/2))
 * over every delay of the zero-Doppler cut (aperiodic tau in +-(N-1), periodic = 1:
 * the residues of (-N/2, N/2]), chi raw (reading R26), and dW/ds*.  Writes (or with
 * accumulate = 1 adds) weight*W_b into loss[b] and weight*dW/ds* into grad[b][:].
 * s, grad: complex64 [B][N]; 1 <= N <= 8192 (v1); no workspace. */
graf_status graf_mainlobe_width(int64_t batch, int32_t n, const void* s, float gamma, float weight,
                                int32_t periodic, double* loss, void* grad, int32_t accumulate, void* stream);

/* One Adam step (L425: Adam, learning rate 0.01) on the phases of phase-coded
 * waveforms s = exp(j*theta):  dL/dtheta = -2 Im(s conj(g)) from g = dL/ds*
 * (complex64 [B][N]); m, v: float [B][N] moments; step: int32 [B] completed steps
 * per waveform (incremented here, so a captured CUDA graph can replay the step);
 * theta updated in place; s_out (complex64 [B][N], may alias nothing else) gets
 * exp(j*theta_new).  Torch's Adam: m = b1 m + (1-b1) d, v = b2 v + (1-b2) d^2,
 * theta -= lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps). */
graf_status graf_phase_adam_step(int64_t batch, int32_t n, float* theta, float* m, float* v,
                                 int32_t* step, const void* grad, void* s_out, float lr, float beta1,
                                 float beta2, float eps, void* stream);

/* Combine per-shard partials shards[G][B] into out[B] in shard order
 * (deterministic).  on_device = 1: both arrays are device pointers and the work
 * is enqueued on `stream`; 0: both are host pointers, computed synchronously. */
graf_status graf_combine_partials(const graf_loss_desc* loss, const graf_partials* shards,
                                  int32_t G, int64_t B, graf_partials* out,
                                  int32_t on_device, void* stream);

/* Diagnostics: number of device operations (kernels and memsets) that the calling
 * thread's most recent entry-point call enqueued (e.g. 1 for a fused single-pass
 * ISL call whose finalize runs inside the row kernel; 2 when it runs separately). */
int32_t graf_last_launch_count(void);

/* Diagnostics (host only, no CUDA call): the CTAs per waveform P that the launch model
 * (choose_P, csrc/graf_launch.cuh) picks for `rows` delay rows per
 * waveform, `slots` row slots per CTA, a batch of `batch` waveforms, `occ` resident CTAs
 * per SM on `nsm` SMs, from the candidates 1..p_bound.  Returns 0 for a non-positive
 * argument.  The production launches call the same function with the kernel's occupancy. */
int32_t graf_plan_ctas_per_waveform(int32_t rows, int32_t slots, int64_t batch, int32_t occ,
                                    int32_t nsm, int32_t p_bound);

/* Diagnostics: with both events non-NULL (cudaEvent_t handles created by the
 * caller), every later entry-point call made by THIS thread records `start` on
 * its stream just before its first delay-row kernel (af_rows_kernel) and `stop`
 * just after its last one, so the caller can time the dominant kernel(s) with
 * cudaEventElapsedTime (works inside CUDA-graph capture).  (NULL, NULL) = off. */
graf_status graf_set_profile_events(void* start, void* stop);

/* Diagnostics: FP32 peak probe.  Enqueues one FFMA-bound kernel (8 independent fmaf chains
 * per thread, 4 CTAs x 256 threads per SM, `iters` x 16 x 8 FFMA per thread) and writes its
 * flop count to *flops (host).  The caller times it with events on `stream`; bench.py uses
 * it as the MEASURED FP32 denominator next to the derived 2 x 128 x SMs x clock.
 * scratch: device float [4 x SMs x 256] (written only in a practically impossible case). */
graf_status graf_probe_fp32(float* scratch, int32_t iters, double* flops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GRAF_H_ */
