// k_states.cu -- frame status, the alpha/beta drift-trellis recursions and the
// APP row normalisation (sm_100a).
//
//   k_frame_init : end drift rho - tau outside [m_tau^-, m_tau^+] -> status
//                  DRIFT_OUT_OF_RANGE.
//   k_alpha_beta : a2/a3 -- one CTA per (frame, direction), persistent over i
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

namespace bsidmap {

__global__ void k_frame_init(const DecodeParams p) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= p.F) return;
  const int drift = p.rho[f] - p.n * p.N;
  // with soft beta_N weights the end drift need not be a state (stream decoding)
  p.status[f] = (p.betaN || (drift >= p.mt_lo && drift <= p.mt_hi)) ? kFrameOk : kFrameDriftOutOfRange;
}

// Shared memory of k_alpha_beta: ring[stages][M_n][Mtp] floats | R[2][Mtp] doubles |
// part[2][32] doubles | bars[stages].
__host__ __device__ size_t ab_cta_smem(int Mn, int Mtp, int stages) {
  return (size_t)stages * Mn * Mtp * 4 + 2 * (size_t)Mtp * 8 + 2 * 32 * 8 + (size_t)stages * 8;
}

// blockIdx.x = frame, blockIdx.y = 0 (alpha, forward) / 1 (beta, backward).
//
// One CTA per (frame, direction), persistent over the N steps, ONE block barrier
// per step: the row is kept unnormalised, R_{i+1} = (1/c_i) sum_k R_i Gamma_i with
// c_i = sum_m R_i(m) taken from the previous step's per-warp partial sums, and rows
// are ping-ponged so no thread overwrites a row another thread may still read.  The
// Gamma_i blocks (M_n x Mtp FP32, contiguous) stream through a `stages`-deep ring
// via TMA bulk copies (one thread issues, an mbarrier per stage signals arrival).
__global__ void __launch_bounds__(1024) k_alpha_beta(const DecodeParams p, int stages) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int Mt = p.Mt, Mn = p.Mn, Mtp = p.Mtp, N = p.N, lo = p.mn_lo;
  float* ring = reinterpret_cast<float*>(smem);
  double* R = reinterpret_cast<double*>(smem + (size_t)stages * Mn * Mtp * 4);
  double* part = R + 2 * Mtp;
  uint64_t* bars = reinterpret_cast<uint64_t*>(part + 64);
  const int f = blockIdx.x;
  const bool fwd = blockIdx.y == 0;
  if (p.status[f] != kFrameOk) return;  // uniform over the CTA
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = (nt + 31) >> 5;
  double* rows = (fwd ? p.alpha : p.beta) + (size_t)f * (N + 1) * Mt;
  const float* Gf = p.Gsum + (size_t)f * N * Mn * Mtp;
  const uint32_t blk = (uint32_t)(Mn * Mtp * 4);
  auto gblock = [&](int step) { return Gf + (size_t)(fwd ? step : N - 1 - step) * Mn * Mtp; };
  if (tid == 0) {
    for (int s = 0; s < stages; s++) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < stages && s < N; s++) {
      mbar_expect_tx(bars + s, blk);
      tma_bulk_g2s(ring + (size_t)s * Mn * Mtp, gblock(s), blk, bars + s);
    }
  }
  const int i0 = fwd ? 0 : N;
  for (int m = tid; m < Mt; m += nt) {
    const double v = boundary_row(p, f, m, fwd);  // alpha_0 / beta_N
    R[m] = v;
    rows[(size_t)i0 * Mt + m] = v;
  }
  __syncthreads();
  double inv_c = 1.0;  // scale of R_cur (any constant: every row is normalised by its own sum)
  for (int step = 0; step < N; step++) {
    const int stage = step % stages;
    mbar_wait(bars + stage, (uint32_t)(step / stages) & 1u);
    const float* G = ring + (size_t)stage * Mn * Mtp;
    const double* cur = R + (step & 1) * Mtp;
    double* nxt = R + ((step + 1) & 1) * Mtp;
    double ps = 0.0;
    for (int m = tid; m < Mt; m += nt) {
      double a0 = 0.0, a1 = 0.0;
      for (int e = 0; e < Mn; e++) {
        // alpha: R(m - k) Gamma_i(m - k, k); beta: Gamma_i(m', k) R(m' + k)
        const int j = fwd ? m - lo - e : m + lo + e;
        const int idx = fwd ? j : m;
        if (j >= 0 && j < Mt) {
          const double t = cur[j] * (double)G[e * Mtp + idx];
          if (e & 1) a1 += t; else a0 += t;
        }
      }
      const double v = (a0 + a1) * inv_c;
      nxt[m] = v;
      ps += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
    double* pp = part + ((step + 1) & 1) * 32;
    if (lane == 0) pp[warp] = ps;
    __syncthreads();  // nxt and the partials are complete; the ring stage is consumed
    if (tid == 0 && step + stages < N) {
      mbar_expect_tx(bars + stage, blk);
      tma_bulk_g2s(ring + (size_t)stage * Mn * Mtp, gblock(step + stages), blk, bars + stage);
    }
    double c = 0.0;
    for (int w = 0; w < nw; w++) c += pp[w];
    if (!(c > 0.0)) {  // all-zero row: Y impossible under the limits (reading R14)
      if (tid == 0) {
        p.status[f] = kFrameUnderflow;
        for (int t = step + 1; t < N && t <= step + stages; t++)  // drain issued copies
          mbar_wait(bars + t % stages, (uint32_t)(t / stages) & 1u);
      }
      return;
    }
    inv_c = 1.0 / c;
    const int r = fwd ? step + 1 : N - 1 - step;
    for (int m = tid; m < Mt; m += nt) rows[(size_t)r * Mt + m] = nxt[m] * inv_c;  // eqn:alpha_norm
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
