// k_states.cu -- frame status, the alpha/beta drift-trellis recursions and the
// APP row normalisation (sm_100a).
//
//   k_frame_init : end drift rho - tau outside [m_tau^-, m_tau^+] -> status
//                  DRIFT_OUT_OF_RANGE.
//   k_alpha_beta_cta (k_alphabeta_cta.cuh) : a2/a3 -- one CTA per (frame, direction), persistent over i
//                  (TMA-fed Gamma ring, one barrier per step, see below):
//                  alpha'_{i+1}(m) = sum_k alpha_i(m-k) Gamma_i(m-k, k)
//                  (eqn:alpha_prenorm with sum_D folded into Gamma),
//                  alpha_{i+1} = alpha'/sum_m alpha' (eqn:alpha_norm); the
//                  mirror for beta (eqn:beta, "similar argument" P:271).
//                  FP64 states.  Boundaries alpha_0 = delta(0),
//                  beta_N = delta(rho - tau) (reading R1).  A zero normaliser
//                  marks the frame UNDERFLOW.  Replaces the paper's 2N+
//                  per-step launches by one launch.
//   k_finalize   : L_i(D) = Lacc_i(D) / sum_D Lacc_i(D) -- equal to the literal
//                  1/lambda_N(rho - tau) of eqn:L in exact arithmetic
//                  (reading R2); FP32 output.
#include "common.cuh"
#include "tma.cuh"
#include "k_alphabeta_cta.cuh"

namespace bsidmap {

__global__ void k_frame_init(const DecodeParams p) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= p.F) return;
  const int drift = p.rho[f] - p.n * p.N;
  // with soft beta_N weights the end drift need not be a state (stream decoding)
  p.status[f] = (p.betaN || (drift >= p.mt_lo && drift <= p.mt_hi)) ? kFrameOk : kFrameDriftOutOfRange;
}

// generic-M_n instance of the CTA recursion (k_alphabeta_cta.cuh); spec shapes instantiate their own
template __global__ void k_alpha_beta_cta<0>(const DecodeParams p, int stages);
template __global__ void k_alpha_beta_cta<0, false>(const DecodeParams p, int stages);

// Frames that failed (status != OK) get all-zero L rows (contract of bsidmap_decode_batch);
// also catches an UNDERFLOW raised by a late row after other rows were written.
__global__ void k_zero_failed(const DecodeParams p) {
  const int f = blockIdx.x;
  if (p.status[f] == kFrameOk) return;
  float* L = p.L + (size_t)f * p.N * p.q;
  for (long k = threadIdx.x; k < (long)p.N * p.q; k += blockDim.x) L[k] = 0.f;
}

// Extrinsic output (NEXT-4): E_i(D) = L_i(D) / P(D_i = D), normalised,
// 0 where the prior is 0; uniform priors give E = L.  One warp per (frame, i) row.
__global__ void k_extrinsic(const DecodeParams p, float* E) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= (long)p.F * p.N) return;
  const float* Lr = p.L + row * p.q;
  const float* Pr = p.priors ? p.priors + row * p.q : nullptr;
  float* Er = E + row * p.q;
  float s = 0.f;
  for (int D = lane; D < p.q; D += 32) {
    const float P = Pr ? Pr[D] : 1.f;
    s += P > 0.f ? Lr[D] / P : 0.f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float inv = s > 0.f ? 1.f / s : 0.f;
  for (int D = lane; D < p.q; D += 32) {
    const float P = Pr ? Pr[D] : 1.f;
    Er[D] = P > 0.f ? Lr[D] / P * inv : 0.f;
  }
}

// Live windows of the APP pass (row a4, eqn:L).  Window (i, m') adds
//   sum_k alpha_i(m') gamma_i(m', m'+k, D) beta_{i+1}(m'+k)
// to S_i(D); summed over D and k that is alpha_i(m') beta~_i(m'), beta~_i the unnormalised beta_i of
// eqn:beta -- c_i alpha_i(m') beta_i(m'), the posterior mass of drift m' at symbol boundary i times
// the row constant c_i sum_m alpha_i beta_i = sum_D S_i(D).  A window with
// alpha_i(m') beta_i(m') <= eps sum_m alpha_i(m) beta_i(m) therefore moves every L_i(D) by at most eps,
// and all skipped windows together by at most M_tau eps (reading R18: eps = 2^-128, M_tau eps
// < 1e-35, far below the 1e-4 relative gate at its 1e-30 floor; eps = 0 skips exact zeros only).
// Writes the smallest state range holding every live window, its length rounded up to even (the pair
// core runs two adjacent windows per lane).  One warp per (frame, i) row.
__global__ void k_live(const DecodeParams p) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int ni = p.i_end - p.i_base;  // symbol indices [i_base, i_end) of this launch
  if (row >= (long)p.F * ni) return;
  const int f = (int)(row / ni), i = p.i_base + (int)(row - (long)f * ni);
  int2 out = make_int2(0, 0);
  if (p.status[f] == kFrameOk) {
    const double* a = p.alpha + ((size_t)f * (p.N + 1) + i) * p.Mt;
    const double* b = beta_row(p, f, i);
    double s = 0.0;
    for (int m = lane; m < p.Mt; m += 32) s += a[m] * b[m];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double thr = s * p.live_eps;
    int lo = 0x7fffffff, hi = -1;
    for (int m = lane; m < p.Mt; m += 32) {
      if (a[m] * b[m] > thr) {
        lo = min(lo, m);
        hi = max(hi, m);
      }
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (s > 0.0 && hi >= lo) out = make_int2(lo, (hi - lo + 2) & ~1);
  }
  if (lane == 0) p.live[(size_t)f * p.N + i] = out;
}

// One warp per (frame, i) row.
__global__ void k_finalize(const DecodeParams p) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= (long)p.F * p.N) return;
  const int f = (int)(row / p.N);
  const double* a = p.Lacc + row * p.q;
  float* out = p.L + row * p.q;
  const bool ok = p.status[f] == kFrameOk;
  double s = 0.0;
  for (int D = lane; D < p.q; D += 32) s += ok ? a[D] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const double inv = (ok && s > 0.0) ? 1.0 / s : 0.0;
  for (int D = lane; D < p.q; D += 32) out[D] = (float)(a[D] * inv);
  if (ok && !(s > 0.0) && lane == 0) p.status[f] = kFrameUnderflow;
}

}  // namespace bsidmap
