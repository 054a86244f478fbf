// k_local_x2.cuh -- the paper's memory-reduced ("local storage") schedule, P:483-627:
// gamma_i is computed inside the alpha pass and computed again inside the
// combined beta + L pass ("combining the computation of L with that of beta",
// P:520-521); only the alpha rows are stored (O(N M_tau) per frame instead of
// O(N M_tau M_n q) for stored gamma).
//
// B200 form, for M_tau <= 64: one warp owns one frame for the whole pass (no
// block barrier, no per-step launch -- the paper needs 2N+ launches and a
// 4-stream pipeline for this).  Lane t owns start drifts m' = 2t, 2t+1
// (packed-pair lattice core, lattice_x2.cuh).
//
//   k_local_fwd : for i = 0..N-1: Gamma_i(m', k) = sum_D P(D) G(m', k, D) in
//                 registers -> warp smem -> alpha_{i+1}(m) = sum_k alpha_i(m-k)
//                 Gamma_i(m-k, k) (eqn:alpha_prenorm), normalised (eqn:alpha_norm),
//                 row written to HBM (FP64).
//   k_local_bwd : for i = N-1..0: t(m', D) = sum_k G(m', k, D) beta~_{i+1}(m'+k);
//                 L_i(D) from sum_{m'} alpha_i(m') t(m', D) (eqn:L, written normalised)
//                 and beta_i(m') = sum_D P(D) t(m', D) (eqn:beta), normalised.
#pragma once
#include "k_lattice_x2.cuh"

namespace bsidmap {

constexpr int kLocalWarps = 4;  // frames per CTA

// smem per warp: s_G[max(M_n * 64, 2 q)] floats (fwd: Gamma_i [k][slot]; bwd: S(D) as doubles) |
//                s_row[64] doubles | s_C[q] words
__host__ __device__ __forceinline__ int local_g_floats(int Mn, int q) { return Mn * 64 > 2 * q ? Mn * 64 : 2 * q; }
__host__ __device__ __forceinline__ size_t local_warp_smem(int Mn, int q) {
  // rounded to 16 bytes: the next warp's FP64 row must stay 8-byte aligned for odd q
  return ((size_t)local_g_floats(Mn, q) * 4 + 64 * 8 + (size_t)q * 4 + 15) & ~size_t(15);
}

template <class Core>
__global__ void __launch_bounds__(kLocalWarps * 32, Core::kMinBlocks) k_local_fwd(const DecodeParams p) {
  using f32x2 = typename Core::P2;
  constexpr int MN = Core::Mn;
  extern __shared__ __align__(128) unsigned char s_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = s_raw + (size_t)warp * local_warp_smem(MN, p.q);
  float* sG = reinterpret_cast<float*>(base);                 // Gamma_i [k][slot]
  double* row = reinterpret_cast<double*>(sG + local_g_floats(MN, p.q));  // alpha_i [slot]
  uint32_t* sC = reinterpret_cast<uint32_t*>(row + 64);       // C_i(0..q-1)
  const int f = blockIdx.x * kLocalWarps + warp;
  if (f >= p.F || p.status[f] != kFrameOk) return;  // warp-uniform
  const int Mt = p.Mt, N = p.N, lo = p.mn_lo;
  double* rows_g = p.alpha + (size_t)f * (N + 1) * Mt;
  const int ma = 2 * lane, mb = 2 * lane + 1;
  // alpha_0 (delta(0) by default, reading R1)
  {
    const double va = boundary_row(p, f, ma, true), vb = boundary_row(p, f, mb, true);
    row[ma] = va;
    row[mb] = vb;
    if (ma < Mt) rows_g[ma] = va;
    if (mb < Mt) rows_g[mb] = vb;
  }
  const float sc = p.priors ? 1.f : 1.f / p.q;
  for (int i = 0; i < N; i++) {
    for (int t = lane; t < p.q; t += 32) sC[t] = p.C[(size_t)i * p.q + t];
    __syncwarp();
    const LaneGeom A = geom_fm(p, i, f, ma, ma < Mt), B = geom_fm(p, i, f, mb, mb < Mt);
    f32x2 acc[MN];
#pragma unroll
    for (int e = 0; e < MN; e++) acc[e] = Core::f2z();
    if (__any_sync(0xffffffffu, A.active || B.active)) {
      typename Core::Lane lt;
      Core::init(lt, A.active ? load_window(p, f, A.s, A.rho) : 0ull, B.active ? load_window(p, f, B.s, B.rho) : 0ull,
                 p);
      const float* pri = p.priors ? p.priors + ((size_t)f * N + i) * p.q : nullptr;
      for (int D = 0; D < p.q; D++) {
        const float P = pri ? __ldg(pri + D) : 1.f;
        f32x2 fo[MN];
        Core::template run<true>(lt, sC[D], p, fo);
        const f32x2 P2 = Core::pk(P, P);
#pragma unroll
        for (int e = 0; e < MN; e++) acc[e] = ffma2(P2, fo[e], acc[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < MN; e++) {
      sG[e * 64 + ma] = out_valid(p, A, e) ? sc * lo_of(acc[e]) : 0.f;
      sG[e * 64 + mb] = out_valid(p, B, e) ? sc * hi_of(acc[e]) : 0.f;
    }
    __syncwarp();
    // alpha'_{i+1}(m) = sum_k alpha_i(m - k) Gamma_i(m - k, k)
    double na = 0.0, nb = 0.0;
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const int ja = ma - lo - e, jb = mb - lo - e;
      if (ma < Mt && ja >= 0 && ja < Mt) na = fma(row[ja], (double)sG[e * 64 + ja], na);
      if (mb < Mt && jb >= 0 && jb < Mt) nb = fma(row[jb], (double)sG[e * 64 + jb], nb);
    }
    double c = na + nb;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (!(c > 0.0)) {  // all-zero row (reading R14)
      if (lane == 0) p.status[f] = kFrameUnderflow;
      return;
    }
    const double inv = 1.0 / c;
    __syncwarp();  // all reads of the old row done
    row[ma] = na * inv;
    row[mb] = nb * inv;
    double* out = rows_g + (size_t)(i + 1) * Mt;
    if (ma < Mt) out[ma] = na * inv;
    if (mb < Mt) out[mb] = nb * inv;
    __syncwarp();
  }
}

// 5 CTAs/SM where the pair core allows 3 (as the round-1 tiled APP kernel it derives from)
template <class Core>
__global__ void __launch_bounds__(kLocalWarps * 32, Core::kMinBlocks > 2 ? 5 : 2) k_local_bwd(const DecodeParams p) {
  using f32x2 = typename Core::P2;
  constexpr int MN = Core::Mn;
  extern __shared__ __align__(128) unsigned char s_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = s_raw + (size_t)warp * local_warp_smem(MN, p.q);
  double* sS = reinterpret_cast<double*>(base);               // S(D), q doubles
  double* row = reinterpret_cast<double*>(base + (size_t)local_g_floats(MN, p.q) * 4);  // beta_{i+1} [slot]
  uint32_t* sC = reinterpret_cast<uint32_t*>(row + 64);
  const int f = blockIdx.x * kLocalWarps + warp;
  if (f >= p.F) return;
  const int Mt = p.Mt, N = p.N, lo = p.mn_lo;
  float* Lf = p.L + (size_t)f * N * p.q;
  if (p.status[f] != kFrameOk) {  // failed frame: zero rows (k_zero_failed also covers late failures)
    for (long k = lane; k < (long)N * p.q; k += 32) Lf[k] = 0.f;
    return;
  }
  const double* alpha_f = p.alpha + (size_t)f * (N + 1) * Mt;
  const int ma = 2 * lane, mb = 2 * lane + 1;
  row[ma] = boundary_row(p, f, ma, false);  // beta_N (delta(rho - tau) by default)
  row[mb] = boundary_row(p, f, mb, false);
  __syncwarp();
  for (int i = N - 1; i >= 0; i--) {
    for (int t = lane; t < p.q; t += 32) sC[t] = p.C[(size_t)i * p.q + t];
    const LaneGeom A = geom_fm(p, i, f, ma, ma < Mt), B = geom_fm(p, i, f, mb, mb < Mt);
    // per-window beta_{i+1}(m'+k) scaled by 2^-E (exact) and weight alpha_i(m') 2^E
    f32x2 bt[MN];
    int Ea, Eb;
    double da, db;
    {
      double bm_a = 0.0, bm_b = 0.0;
#pragma unroll
      for (int e = 0; e < MN; e++) {
        const int j = ma + lo + e;  // state m' + k of window a; window b is j + 1
        const double va = ((A.vmask >> e) & 1u) ? row[min(max(j, 0), 63)] : 0.0;
        const double vb = ((B.vmask >> e) & 1u) ? row[min(max(j + 1, 0), 63)] : 0.0;
        bm_a = fmax(bm_a, va);
        bm_b = fmax(bm_b, vb);
      }
      Ea = bm_a > 0.0 ? exp2_of(bm_a) : 0;
      Eb = bm_b > 0.0 ? exp2_of(bm_b) : 0;
      const double sa = pow2d(-Ea), sb = pow2d(-Eb);
#pragma unroll
      for (int e = 0; e < MN; e++) {
        const int j = ma + lo + e;
        const double va = ((A.vmask >> e) & 1u) ? row[min(max(j, 0), 63)] : 0.0;
        const double vb = ((B.vmask >> e) & 1u) ? row[min(max(j + 1, 0), 63)] : 0.0;
        bt[e] = Core::pk((float)(va * sa), (float)(vb * sb));
      }
      da = (A.active && bm_a > 0.0) ? alpha_f[(size_t)i * Mt + ma] * pow2d(Ea) : 0.0;
      db = (B.active && bm_b > 0.0) ? alpha_f[(size_t)i * Mt + mb] * pow2d(Eb) : 0.0;
    }
    const double dm = fmax(da, db);
    const int Emax = __reduce_max_sync(0xffffffffu, dm > 0.0 ? exp2_of(dm) + 2048 : 0) - 2048;
    const double wsc = pow2d(-Emax);
    const float wa = (float)(da * wsc), wb = (float)(db * wsc);
    // windows with a non-zero beta part feed beta_i even where alpha_i = 0
    const bool live = __any_sync(0xffffffffu, A.active || B.active);
    __syncwarp();
    float ba = 0.f, bb = 0.f;  // sum_D P(D) t(m', D) for beta_i
    if (live) {
      typename Core::Lane lt;
      Core::init(lt, A.active ? load_window(p, f, A.s, A.rho) : 0ull, B.active ? load_window(p, f, B.s, B.rho) : 0ull,
                 p);
      const float* pri = p.priors ? p.priors + ((size_t)f * N + i) * p.q : nullptr;
      for (int D = 0; D < p.q; D++) {
        f32x2 fo[MN];
        Core::template run<BSIDMAP_APP_GROUP>(lt, sC[D], p, fo);
        f32x2 t0 = Core::f2z(), t1 = Core::f2z();
#pragma unroll
        for (int e = 0; e < MN; e += 2) {
          t0 = ffma2(fo[e], bt[e], t0);
          if (e + 1 < MN) t1 = ffma2(fo[e + 1], bt[e + 1], t1);
        }
        const float ta = lo_of(t0) + lo_of(t1), tb = hi_of(t0) + hi_of(t1);
        const float P = pri ? __ldg(pri + D) : 1.f;
        ba = fmaf(P, ta, ba);
        bb = fmaf(P, tb, bb);
        double c = (double)fmaf(wa, ta, wb * tb);  // the sum over the windows in FP64
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) sS[D] = c * (double)P;
      }
    }
    __syncwarp();
    // L_i(D) = S(D) / sum_D S(D)   (eqn:L; equal to the literal 1/lambda_N, reading R2)
    {
      double tot = 0.0;
      if (live)
        for (int D = lane; D < p.q; D += 32) tot += sS[D];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      const bool ok = live && tot > 0.0;
      const double inv = ok ? 1.0 / tot : 0.0;
      float* Lrow = Lf + (size_t)i * p.q;
      for (int D = lane; D < p.q; D += 32) Lrow[D] = ok ? (float)(sS[D] * inv) : 0.f;
      if (!ok) {
        if (lane == 0) p.status[f] = kFrameUnderflow;
        return;
      }
    }
    // beta_i(m') = 2^E sum_D P(D) t(m', D), normalised (eqn:beta)
    const double na = (double)ba * pow2d(Ea), nb = (double)bb * pow2d(Eb);
    double c = (ma < Mt ? na : 0.0) + (mb < Mt ? nb : 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (!(c > 0.0)) {
      if (lane == 0) p.status[f] = kFrameUnderflow;
      return;
    }
    const double inv = 1.0 / c;
    __syncwarp();
    row[ma] = ma < Mt ? na * inv : 0.0;
    row[mb] = mb < Mt ? nb * inv : 0.0;
    __syncwarp();
  }
}

template <class Core>
CoreKernels make_core_kernels_x2(long nodes) {
  CoreKernels k = make_core_kernels_x2_base<Core>(nodes);
  k.local_fwd = k_local_fwd<Core>;
  k.local_bwd = k_local_bwd<Core>;
  return k;
}

}  // namespace bsidmap
