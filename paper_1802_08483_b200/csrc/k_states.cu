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
template <int LPR>
__device__ __forceinline__ void live_body(const DecodeParams& p) {
  // LPR lanes per (frame, i) row, 32 / LPR rows per warp (M_tau <= 64: 8 lanes, so the reductions and
  // the per-row index work serve four rows at once; the kernel is issue-bound)
  constexpr int RPW = 32 / LPR;
  const int lane = threadIdx.x & 31, sl = lane % LPR;
  const long row = ((long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW + lane / LPR;
  const int ni = p.i_end - p.i_base;  // symbol indices [i_base, i_end) of this launch
  const bool valid = row < (long)p.F * ni;
  int f = 0, i = p.i_base;
  if (valid) row_fi(row, ni, p.i_base, &f, &i);
  const bool ok = valid && p.status[f] == kFrameOk;
  const double* a = p.alpha + ((size_t)f * (p.N + 1) + i) * p.Mt;
  const double* b = beta_row(p, f, i);
  double s = 0.0;
  if (ok)
    for (int m = sl; m < p.Mt; m += LPR) s += a[m] * b[m];
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);  // within the row's lanes
  const double thr = s * p.live_eps;
  int lo = 0x7fffffff, hi = -1;
  if (ok) {
    for (int m = sl; m < p.Mt; m += LPR) {
      if (a[m] * b[m] > thr) {
        lo = min(lo, m);
        hi = max(hi, m);
      }
    }
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (valid && sl == 0)
    p.live[(size_t)f * p.N + i] = (ok && s > 0.0 && hi >= lo) ? make_int2(lo, (hi - lo + 2) & ~1) : make_int2(0, 0);
}
__global__ void __launch_bounds__(256) k_live8(const DecodeParams p) { live_body<8>(p); }
__global__ void __launch_bounds__(256) k_live16(const DecodeParams p) { live_body<16>(p); }
__global__ void __launch_bounds__(256) k_live32(const DecodeParams p) { live_body<32>(p); }

// The slab schedule's backward sweep: per (frame, i) row of symbol indices [i_base, i_end), the state
// range [first, first + count) holding every alpha_i(m') != 0 (count 0: none), into p.live (which the
// live-window APP's k_live overwrites for the same rows afterwards).  One warp per row.
__global__ void k_alpha_support(const DecodeParams p) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int ni = p.i_end - p.i_base;
  if (row >= (long)p.F * ni) return;
  int f, i;
  row_fi(row, ni, p.i_base, &f, &i);
  int lo = 0x7fffffff, hi = -1;
  if (p.status[f] == kFrameOk) {
    const double* a = p.alpha + ((size_t)f * (p.N + 1) + i) * p.Mt;
    for (int m = lane; m < p.Mt; m += 32) {
      if (a[m] != 0.0) {
        lo = min(lo, m);
        hi = max(hi, m);
      }
    }
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if (lane == 0) p.live[(size_t)f * p.N + i] = hi >= lo ? make_int2(lo, hi - lo + 1) : make_int2(0, 0);
}

// Packing of the slab backward sweep's pass 1 (win_base_packed), per symbol-index group g (p.i_steps
// indices from p.i_base): per frame the union [lo, hi] of the group's alpha-support rows
// (k_alpha_support), its width, and the exclusive scan of the widths over frames, in two passes --
// pack1: grid (groups, ceil(F / 256)), a block scan of 256 frames, block totals to spack_blk;
// pack2: one block per group, scans the block totals, adds them, writes the total at [F].
__device__ __forceinline__ int block_scan_incl(int v, int* s_w) {  // blockDim.x = 256
  s_w[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const int t = threadIdx.x >= (unsigned)o ? s_w[threadIdx.x - o] : 0;
    __syncthreads();
    s_w[threadIdx.x] += t;
    __syncthreads();
  }
  return s_w[threadIdx.x];
}
__global__ void __launch_bounds__(256) k_support_pack1(const DecodeParams p) {
  __shared__ int s_w[256];
  const int g = blockIdx.x, f = blockIdx.y * 256 + threadIdx.x;
  const int i0 = p.i_base + g * p.i_steps, i1 = min(i0 + p.i_steps, p.i_end);
  int lo = 0x7fffffff, hi = -1;
  if (f < p.F) {
    for (int i = i0; i < i1; i++) {
      const int2 r = p.live[(size_t)f * p.N + i];
      if (r.y > 0) {
        lo = min(lo, r.x);
        hi = max(hi, r.x + r.y - 1);
      }
    }
  }
  const int w = hi >= lo ? hi - lo + 1 : 0;
  const int incl = block_scan_incl(w, s_w);
  if (f < p.F) p.spack[(size_t)g * (p.F + 1) + f] = make_int2(incl - w, w > 0 ? lo : 0);
  if (threadIdx.x == blockDim.x - 1) p.spack_blk[(size_t)g * gridDim.y + blockIdx.y] = incl;
}
__global__ void __launch_bounds__(256) k_support_pack2(const DecodeParams p, int nblk) {
  __shared__ int s_w[256];
  __shared__ int s_carry;
  const int g = blockIdx.x;
  int2* pk = p.spack + (size_t)g * (p.F + 1);
  int* bt = p.spack_blk + (size_t)g * nblk;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nblk; b0 += blockDim.x) {  // exclusive scan of the block totals
    const int b = b0 + threadIdx.x;
    const int v = b < nblk ? bt[b] : 0;
    const int incl = block_scan_incl(v, s_w);
    const int carry = s_carry;
    __syncthreads();
    if (b < nblk) bt[b] = carry + incl - v;
    if (threadIdx.x == blockDim.x - 1) s_carry = carry + incl;
    __syncthreads();
  }
  for (int f = threadIdx.x; f < p.F; f += blockDim.x) pk[f].x += bt[f >> 8];
  if (threadIdx.x == 0) pk[p.F] = make_int2(s_carry, 0);
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
