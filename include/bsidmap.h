/*
 * bsidmap.h -- C ABI of the B200 batched BSID MAP (forward-backward) decoder,
 * arXiv 1802.08483.  "P:n" cites line n of the paper's LaTeX;
 * equations are cited by label.
 *
 * The decoder computes, for every frame of a batch, the a-posteriori symbol
 * probabilities L_i(D) of eqn:L:
 *
 *   L_i(D) = 1/lambda_N(rho - tau) * sum_{m',m} alpha_i(m') gamma_i(m',m,D) beta_{i+1}(m)
 *
 * with gamma from the corridor-constrained receiver-metric lattice
 * (eqn:gamma P:156-161, eqn:F P:197-204, eqn:F_lastrow P:228-235, corridor
 * P:250-254), alpha/beta from the normalised recursions (eqn:alpha,
 * eqn:beta, eqn:alpha_norm P:257-271), the receiver metric in single and the
 * states in double precision.  Boundary priors are point masses:
 * alpha_0 = delta(0), beta_N = delta(rho - tau) (reading R1).
 *
 * Bit conventions: bit t (LSB = bit 0) of a codeword word is the t-th
 * transmitted bit x_{t+1}; received sequences are packed LSB-first into
 * 32-bit words, y_1 = bit 0 of the frame's first word (reading R15).
 *
 * Every function returns BSIDMAP_OK (0) or a negative error code; the
 * message of the last failure is available from bsidmap_last_error().
 * Per-frame conditions are reported in frame_status[], never as errors.
 * A decoder is used by one host thread at a time; decoders on different
 * devices are independent (one process per GPU).
 */
#ifndef BSIDMAP_H
#define BSIDMAP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bsidmap_decoder bsidmap_decoder; /* opaque; owns the device codebook and workspace */

/* return codes */
#define BSIDMAP_OK 0
#define BSIDMAP_EINVAL (-1)         /* invalid argument (see bsidmap_last_error) */
#define BSIDMAP_ENOTINJECTIVE (-2)  /* some C_i maps two symbols to one codeword */
#define BSIDMAP_ENOMEM (-3)         /* device allocation failed */
#define BSIDMAP_EPLAN (-4)          /* no feasible launch plan (e.g. corridor wider than 32) */
#define BSIDMAP_ECUDA (-5)          /* a CUDA call failed */

/* per-frame status */
#define BSIDMAP_FRAME_OK 0
#define BSIDMAP_FRAME_DRIFT_OUT_OF_RANGE 1 /* rho - tau outside [m_tau^-, m_tau^+]; L rows = 0 */
#define BSIDMAP_FRAME_UNDERFLOW 2          /* an all-zero alpha/beta/L row: Y impossible under the limits; L rows = 0 */

/* storage schedule */
#define BSIDMAP_MODE_AUTO 0      /* planner choice (= GAMMASUM, the fastest on B200) */
#define BSIDMAP_MODE_STORED 1    /* paper's global storage: every gamma stored in HBM, read back for L */
#define BSIDMAP_MODE_RECOMPUTE 2 /* paper's memory-reduced (local storage) schedule: gamma computed in
                                    a forward (alpha) sweep and again in a backward (beta + L) sweep.  On the
                                    specialised / run-time compiled cores: in slabs of symbol indices (Gamma of
                                    two slabs, all alpha rows, beta rows of three slabs; the backward sweep
                                    recomputes gamma only where alpha != 0, R19).  Otherwise (or with
                                    BSIDMAP_SLAB=0) fused per-frame passes keeping only alpha rows: one warp per
                                    frame for M_tau <= 64, one CTA per frame for 64 < M_tau <= 1024; beyond that
                                    the GAMMASUM schedule runs */
#define BSIDMAP_MODE_GAMMASUM 3  /* memory-reduced variant with parallel passes: Gamma = sum_D gamma, alpha and
                                    beta kept; gamma recomputed once for L */

/*
 * Create a decoder on CUDA device `device`.
 *   q, n, N        : alphabet size, codeword length, symbols per frame; 2 <= q <= 2^n,
 *                    1 <= n <= 32, N >= 1.
 *   codebook_host  : HOST pointer, N*q words, C[i*q + D] = C_i(D); copied, caller keeps ownership.
 *                    Each C_i must be injective (else BSIDMAP_ENOTINJECTIVE).
 *   Pi, Pd, Ps     : BSID channel; Pi, Pd, Ps >= 0, Ps <= 1, Pi + Pd < 1.
 *   mn_lo, mn_hi   : per-codeword drift limits m_n^-, m_n^+ (corridor, M_n = mn_hi - mn_lo + 1 <= 32),
 *                    mn_lo <= 0 <= mn_hi, n + mn_hi <= 64.
 *   mt_lo, mt_hi   : trellis drift limits m_tau^-, m_tau^+ (M_tau states), mt_lo <= mn_lo, mt_hi >= mn_hi.
 *   mode           : BSIDMAP_MODE_* (0..3).
 * On success *out receives the decoder.  Allocates the codebook and its symbol visiting orders
 * (about 3 N q * 6 bytes: lexicographic and last-2/3-bit class orders used by the lattice passes);
 * the workspace is allocated lazily by the first decode of a given size.
 *
 * Kernel-variant overrides, read from the environment at create (measurement and testing only;
 * the defaults are the measured-fastest choices):
 *   BSIDMAP_AB_SUB=k   alpha/beta side-stream sub-batches (1 = off; default: 2 when 2F <= #SMs)
 *   BSIDMAP_APP_KP=k   APP prefix-sharing length (0 = off; default ~log2(q) - 1)
 *   BSIDMAP_APP_KS=k   lattice rows folded into the APP weights (1 or 2; default 1 on the pair core,
 *                      2 on the scalar APP core)
 *   BSIDMAP_LIVE_EPS=e live-window threshold (default 2^-128; 0 = skip exactly-zero windows only)
 *   BSIDMAP_APP_G=g    frames per warp of the live-window APP (default: up to 12 / 8 / 4)
 *   BSIDMAP_JIT=0      shapes without a compiled unit run on the generic core (default: compiled at create)
 *   BSIDMAP_SLAB=0     RECOMPUTE runs the per-frame local kernels instead of the slab schedule
 *   BSIDMAP_SLAB_LEN=B symbol indices per slab (default: ~4 waves of pass-1 CTAs per slab)
 *   BSIDMAP_SLAB_ASKIP=0  the backward sweep recomputes Gamma for every window (default: alpha != 0 only)
 *   BSIDMAP_AB_CTA_STAGES=k, BSIDMAP_AB_CTA_THREADS=t  ring depth / block size of the CTA alpha/beta
 *                      kernel (M_tau > 128; defaults: 1 stage when 2F >= 4 #SMs, ~M_tau/2 threads)
 */
int bsidmap_create(bsidmap_decoder **out, int q, int n, int N, const uint32_t *codebook_host,
                   double Pi, double Pd, double Ps, int mn_lo, int mn_hi, int mt_lo, int mt_hi,
                   int mode, int device);

/*
 * Decode num_frames frames.  All pointers are DEVICE pointers on the decoder's device,
 * caller-owned, and must stay valid until `cuda_stream` (a cudaStream_t; NULL = legacy
 * default stream) reaches the end of the call.  The call is asynchronous: it only
 * enqueues work (it may block once to grow the workspace).
 *   rx_words        : packed received bits (LSB-first); frame f starts at word rx_word_offset[f]
 *                     and owns ceil(rho[f]/32) words.
 *   rx_word_offset  : [num_frames] int64.
 *   rho             : [num_frames] int32 received lengths.
 *   priors          : [num_frames][N][q] FP32 P(D_i = D) weights, or NULL for uniform 1/q
 *                     (P:166-170); rows need not sum to 1; entries >= 0.
 *   L_out           : [num_frames][N][q] FP32 APPs L_i(D); each row sums to 1 (0 for failed frames).
 *   frame_status    : [num_frames] int32 BSIDMAP_FRAME_*.
 */
int bsidmap_decode_batch(bsidmap_decoder *d, int num_frames, const uint32_t *rx_words,
                         const int64_t *rx_word_offset, const int32_t *rho, const float *priors,
                         float *L_out, int32_t *frame_status, void *cuda_stream);

/*
 * Options of bsidmap_decode_batch_opts (all DEVICE pointers, caller-owned; NULL = default).
 *   alpha0, betaN : [num_frames][M_tau] FP64 frame-boundary priors alpha_0(m), beta_N(m), state m at
 *                   index m - m_tau^- ("set as the prior probabilities of the frame boundaries",
 *                   P:152-154; e.g. Phi_T from bsidmap_phi).  Default: alpha_0 = delta(0) and
 *                   beta_N = delta(rho - tau).  With betaN given, rho - tau need not be a state
 *                   (no DRIFT_OUT_OF_RANGE), as in stream decoding.  Any positive scale.
 *   extrinsic     : [num_frames][N][q] FP32 output E_i(D) = L_i(D) / P(D_i = D) normalised over D
 *                   (0 where the prior is 0; = L for uniform priors): the extrinsic information
 *                   for an outer decoder in iterative decoding.
 */
typedef struct bsidmap_decode_opts {
  const double *alpha0;
  const double *betaN;
  float *extrinsic;
} bsidmap_decode_opts;

/* bsidmap_decode_batch with options (opts may be NULL). */
int bsidmap_decode_batch_opts(bsidmap_decoder *d, int num_frames, const uint32_t *rx_words,
                              const int64_t *rx_word_offset, const int32_t *rho, const float *priors,
                              const bsidmap_decode_opts *opts, float *L_out, int32_t *frame_status,
                              void *cuda_stream);

/*
 * Same computation with HOST buffers (end-to-end path): copies the inputs to the
 * device (pinned memory gives async copies), decodes, copies L and the status back and
 * synchronises `cuda_stream` before returning.  rx_words_total = number of words in rx_words.
 */
int bsidmap_decode_batch_host(bsidmap_decoder *d, int num_frames, const uint32_t *rx_words,
                              size_t rx_words_total, const int64_t *rx_word_offset, const int32_t *rho,
                              const float *priors, float *L_out, int32_t *frame_status, void *cuda_stream);

/* Release the decoder and all its device memory (synchronises its device). NULL is a no-op. */
void bsidmap_destroy(bsidmap_decoder *d);

/* Message of the last failure on this decoder ("" if none); valid until the next call. NULL d: global message. */
const char *bsidmap_last_error(const bsidmap_decoder *d);

/* Device workspace bytes needed to decode num_frames frames in `mode` without chunking
   (the paper's memory estimate).  Returns 0 for an invalid mode. */
size_t bsidmap_workspace_bytes(const bsidmap_decoder *d, int num_frames, int mode);

/* Cap the workspace (bytes; 0 = automatic, 85% of free memory); larger batches are chunked. */
int bsidmap_set_workspace_limit(bsidmap_decoder *d, size_t bytes);

/* Override the storage schedule of subsequent decodes (BSIDMAP_MODE_*). */
int bsidmap_set_mode(bsidmap_decoder *d, int mode);

/*
 * Per-phase device timing of the next decodes (CUDA events on the decode stream).
 * bsidmap_phase_times writes up to n_max entries of the LAST decode_batch, in ms:
 *   [0] status init + accumulator clear, [1] lattice pass 1 (gamma / Gamma),
 *   [2] alpha/beta recursions, [3] lattice pass 2 / stored APP, [4] finalize,
 *   [5] alpha/beta busy time,
 * and returns the number written.  It synchronises the decode stream.  In the Gamma-sum
 * schedule the batch is split into sub-batches whose alpha/beta recursions run on a
 * high-priority side stream, overlapped with the lattice passes of the other sub-batches
 * (automatic: 2 sub-batches when the alpha/beta grid cannot fill the GPU, else off; the
 * environment variable BSIDMAP_AB_SUB read at create overrides it, 1 = off);
 * then [1] and [3] span all sub-batches' lattice launches, [2] is the exposed part of
 * alpha/beta on the decode stream and [5] its busy time on the side stream.
 */
int bsidmap_set_timing(bsidmap_decoder *d, int enable);
int bsidmap_phase_times(bsidmap_decoder *d, float *ms, int n_max);

/* Kernel launches issued by the last decode_batch call. */
long bsidmap_last_launch_count(const bsidmap_decoder *d);

/*
 * Human/JSON-readable launch plan for num_frames frames (mode, chunking, grid and block
 * sizes, lattice core: "spec" fully unrolled and compiled into the library, "jit" fully unrolled
 * and compiled at create, or "generic"), written to buf (NUL-terminated).
 * Returns the length, or a negative error code.
 */
int bsidmap_plan_info(bsidmap_decoder *d, int num_frames, char *buf, size_t buf_len);

/*
 * Corridor nodes per lattice of this decoder's shape, n M_n - m_n^-(m_n^- - 1)/2,
 * and the number of lattices with a valid window (0 <= n i + m' <= rho) for the given
 * host rho[] -- the algorithmic work counters used by the roofline.
 */
long bsidmap_lattice_nodes(const bsidmap_decoder *d);

/*
 * Run-time compiled lattice cores (the paper's templates over the code and channel sizes,
 * P:1055-1079, for any shape).  bsidmap_create compiles the fully unrolled kernels of a shape
 * (n, m_n^-, M_n) that has no compiled unit with NVRTC for sm_100a, caches the cubins on disk
 * (BSIDMAP_JIT_CACHE, default ~/.cache/bsidmap) and loads them once per process; BSIDMAP_JIT=0
 * keeps the generic core.  This entry only compiles (no device needed): BSIDMAP_OK, or
 * BSIDMAP_EPLAN with the reason in err (err may be NULL; len bytes incl. NUL).
 */
int bsidmap_jit_compile(int n, int mn_lo, int Mn, char *err, size_t len);
long long bsidmap_valid_lattices(const bsidmap_decoder *d, int num_frames, const int32_t *rho_host);

/*
 * Debug/parity: gamma_i(m', m, D) of symbol index i for every frame, true scale, FP64,
 * gamma_out[f][m' - m_tau^-][m - m' - m_n^-][D] (DEVICE pointer, num_frames*M_tau*M_n*q
 * doubles).  Uses the same lattice core as the decode.  Inputs as in decode_batch.
 * Synchronous.
 */
int bsidmap_debug_gamma(bsidmap_decoder *d, int num_frames, const uint32_t *rx_words,
                        const int64_t *rx_word_offset, const int32_t *rho, const float *priors, int i,
                        double *gamma_out, void *cuda_stream);

/*
 * Debug/parity: after a decode_batch whose workspace held all frames (no chunking), copy
 * the normalised FP64 alpha and beta rows [num_frames][N+1][M_tau] to DEVICE pointers.
 * Synchronous.  Returns BSIDMAP_EINVAL if the last decode was chunked or smaller.
 */
int bsidmap_debug_states(bsidmap_decoder *d, int num_frames, double *alpha_out, double *beta_out,
                         void *cuda_stream);

/* ---------------------------------------------------------------------------------------
 * State-space sizing.  Host functions, no device needed.
 * The drift S_T after T transmitted bits is the T-fold convolution of the per-bit
 * change: k insertions then deletion (k-1, prob Pi^k Pd) or transmission (k, prob Pi^k Pt).
 */
/* pmf[m - lo] = P(S_T = m) for m in [lo, hi] (FP64; mass outside the range is dropped). */
int bsidmap_drift_pmf(int T, double Pi, double Pd, int lo, int hi, double *pmf);
/* Limits with exclusion probability Pr (reading R8; the paper defers the rule to
 * bbw14joe, and names P_r at P:1747-1750): the smallest [lo, hi] containing 0 with
 * P(S_T < lo) + P(S_T > hi) < Pr, grown from [0, 0] one state at a time on the side with more
 * excluded mass, ties to the positive side.  BSIDMAP_EINVAL for bad arguments or
 * when the PMF's own truncation loss (insertions per bit cut at Pi^k < 1e-17) is >= Pr. */
int bsidmap_drift_limits(int T, double Pi, double Pd, double Pr, int *lo, int *hi);
/* The per-tail rule (round 1's default): lo = max{m : P(S_T < m) <= Pr/2},
 * hi = min{m : P(S_T > m) <= Pr/2}, clamped to -T <= lo <= 0 <= hi. */
int bsidmap_drift_limits_tails(int T, double Pi, double Pd, double Pr, int *lo, int *hi);
/* m_n^± from T = n and m_tau^± from T = n N, widened to contain m_n (bsidmap_create's rule). */
int bsidmap_state_space(int n, int N, double Pi, double Pd, double Pr, int *mn_lo, int *mn_hi, int *mt_lo,
                        int *mt_hi);
/* Phi_T (named but undefined in the paper; read as the drift PMF over T bits) written
 * on the device for num_frames frames: out_dev[f][m - lo] = P(S_T = m).  Synchronous. */
int bsidmap_phi(int T, double Pi, double Pd, int lo, int hi, int num_frames, double *out_dev, void *cuda_stream);

/* ---------------------------------------------------------------------------------------
 * Monte-Carlo symbol/frame error rates on the device (the decoder inside the
 * paper's simulator).  Messages D_i ~ U[0,q), encoding with the
 * decoder's codebook and the literal BSID event loop use the counter-based
 * stream of the host generator (bsidgen), so frame (seed, index) is bit-identical on host and
 * device; frames with rho - tau outside [m_tau^-, m_tau^+] are redrawn and counted.
 */
/* Generate frames [first_frame, first_frame + num_frames) into DEVICE buffers: msg [F][N] int32,
 * rx [F][words_per_frame] packed LSB-first (frame f at word f * words_per_frame), rho [F];
 * *redraws (device counter) is incremented.  Asynchronous. */
int bsidmap_mc_generate(bsidmap_decoder *d, uint64_t seed, int64_t first_frame, int num_frames, int words_per_frame,
                        int32_t *msg, uint32_t *rx, int32_t *rho, unsigned long long *redraws, void *cuda_stream);
/* Hard decisions argmax_D L_i(D) (lowest D on ties) against msg: counters (DEVICE, accumulated):
 * [0] symbol errors, [1] frame errors, [2] failed frames (status != OK; all their symbols count as
 * errors).  Asynchronous. */
int bsidmap_count_errors(bsidmap_decoder *d, int num_frames, const float *L, const int32_t *msg,
                         const int32_t *frame_status, unsigned long long *counters, void *cuda_stream);
/* Generate, decode (uniform priors) and count num_frames frames in batches of `batch` frames.
 * results (HOST, 4 entries): frames, symbol errors, frame errors, channel redraws.  Synchronous. */
int bsidmap_mc_run(bsidmap_decoder *d, uint64_t seed, int64_t first_frame, int num_frames, int batch,
                   unsigned long long *results, void *cuda_stream);

#ifdef __cplusplus
}
#endif

#endif /* BSIDMAP_H */
