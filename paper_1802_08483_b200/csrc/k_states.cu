// k_states.cu -- frame status, the alpha/beta drift-trellis recursions and the
// APP row normalisation (sm_100a).
//
//   k_frame_init : end drift rho - tau outside [m_tau^-, m_tau^+] -> status
//                  DRIFT_OUT_OF_RANGE.
//   k_alpha_beta : a2/a3 -- one CTA per (frame, direction), persistent over i:
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

namespace bsidmap {

__global__ void k_frame_init(const DecodeParams p) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= p.F) return;
  const int drift = p.rho[f] - p.n * p.N;
  p.status[f] = (drift >= p.mt_lo && drift <= p.mt_hi) ? kFrameOk : kFrameDriftOutOfRange;
}

__device__ __forceinline__ double block_sum(double v, double* s_red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nw ? s_red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) s_red[32] = t;
  }
  __syncthreads();
  return s_red[32];
}

// blockIdx.x = frame, blockIdx.y = 0 (alpha, forward) / 1 (beta, backward).
__global__ void __launch_bounds__(1024) k_alpha_beta(const DecodeParams p) {
  extern __shared__ __align__(16) double s_st[];  // cur[Mt] | nxt[Mt] | red[33]
  double* cur = s_st;
  double* nxt = s_st + p.Mt;
  double* red = s_st + 2 * p.Mt;
  const int f = blockIdx.x;
  const bool fwd = blockIdx.y == 0;
  if (p.status[f] != kFrameOk) return;
  const int Mt = p.Mt, Mn = p.Mn, N = p.N, lo = p.mn_lo;
  const int end_idx = p.rho[f] - p.n * N - p.mt_lo;
  double* rows = (fwd ? p.alpha : p.beta) + (size_t)f * (N + 1) * Mt;
  const float* Gf = p.Gsum + (size_t)f * N * Mn * p.Mtp;

  const int i0 = fwd ? 0 : N;
  const int boundary = fwd ? -p.mt_lo : end_idx;  // alpha_0 = delta(0), beta_N = delta(rho - tau)
  for (int m = threadIdx.x; m < Mt; m += blockDim.x) {
    const double v = (m == boundary) ? 1.0 : 0.0;
    cur[m] = v;
    rows[(size_t)i0 * Mt + m] = v;
  }
  __syncthreads();

  for (int step = 0; step < N; step++) {
    const int i = fwd ? step : N - 1 - step;  // Gamma_i used by this step
    const float* G = Gf + (size_t)i * Mn * p.Mtp;  // [k][m']
    double part = 0.0;
    for (int m = threadIdx.x; m < Mt; m += blockDim.x) {
      // issue all M_n loads of Gamma_i first (independent, one latency per step)
      float g[kMaxMn];
#pragma unroll
      for (int e = 0; e < kMaxMn; e++) {
        const int idx = fwd ? m - lo - e : m;  // alpha reads Gamma_i(m - k, k); beta reads Gamma_i(m', k)
        g[e] = (e < Mn && idx >= 0 && idx < Mt) ? __ldg(G + (size_t)e * p.Mtp + idx) : 0.f;
      }
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int e = 0; e < kMaxMn; e += 2) {
        // alpha'_{i+1}(m) = sum_k alpha_i(m - k) Gamma_i(m - k, k);  beta'_i(m') = sum_k Gamma_i(m', k) beta_{i+1}(m' + k)
        const int j0 = fwd ? m - lo - e : m + lo + e;
        const int j1 = fwd ? j0 - 1 : j0 + 1;
        if (e < Mn && j0 >= 0 && j0 < Mt) acc0 = fma(cur[j0], (double)g[e], acc0);
        if (e + 1 < Mn && j1 >= 0 && j1 < Mt) acc1 = fma(cur[j1], (double)g[e + 1], acc1);
      }
      const double acc = acc0 + acc1;
      nxt[m] = acc;
      part += acc;
    }
    const double c = block_sum(part, red);
    const int row = fwd ? i + 1 : i;
    if (!(c > 0.0)) {  // all-zero row: Y impossible under the limits (reading R14)
      if (threadIdx.x == 0) p.status[f] = kFrameUnderflow;
      return;
    }
    const double inv = 1.0 / c;
    for (int m = threadIdx.x; m < Mt; m += blockDim.x) {
      const double v = nxt[m] * inv;
      cur[m] = v;
      rows[(size_t)row * Mt + m] = v;
    }
    __syncthreads();
  }
}

// Frames that failed (status != OK) get all-zero L rows (contract of bsidmap_decode_batch);
// also catches an UNDERFLOW raised by a late row after other rows were written.
__global__ void k_zero_failed(const DecodeParams p) {
  const int f = blockIdx.x;
  if (p.status[f] == kFrameOk) return;
  float* L = p.L + (size_t)f * p.N * p.q;
  for (long k = threadIdx.x; k < (long)p.N * p.q; k += blockDim.x) L[k] = 0.f;
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
