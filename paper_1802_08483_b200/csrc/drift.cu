// drift.cu -- drift distribution and state-space sizing.
//
// The drift S_T after T transmitted bits is a sum of T i.i.d. per-bit
// changes: k insertions (probability Pi each, the channel stays at the bit)
// followed by a deletion (change k - 1, probability Pi^k Pd) or a transmission
// (change k, probability Pi^k Pt).  Its PMF is the T-fold convolution, computed by
// repeated squaring in FP64.  The limits follow DESIGN.md reading R8 (the paper
// defers the rule to bbw14joe; exclusion probability P_r):
// the smallest interval around 0 whose excluded mass is below P_r, grown one state at
// a time on the side with more excluded mass; the older per-tail rule
// (each tail <= P_r/2) stays available as bsidmap_drift_limits_tails.
//
// Phi_T (the paper names a "Compute Phi_T" kernel but never
// defines it) is read as this drift PMF over T bits; k_phi writes it, restricted to a
// state range, into device arrays (soft frame-boundary priors, NEXT-1).
#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/bsidmap.h"
#include "common.cuh"

namespace {

struct Pmf {
  long off = 0;              // pmf[j] = P(S = off + j)
  std::vector<double> p{1.0};
};

void trim(Pmf& a, double floor_) {
  size_t b = 0, e = a.p.size();
  while (b < e && a.p[b] <= floor_) b++;
  while (e > b && a.p[e - 1] <= floor_) e--;
  if (b == e) return;
  a.p = std::vector<double>(a.p.begin() + b, a.p.begin() + e);
  a.off += (long)b;
}

Pmf conv(const Pmf& a, const Pmf& b) {
  Pmf r;
  r.off = a.off + b.off;
  r.p.assign(a.p.size() + b.p.size() - 1, 0.0);
  for (size_t i = 0; i < a.p.size(); i++)
    for (size_t j = 0; j < b.p.size(); j++) r.p[i + j] += a.p[i] * b.p[j];
  return r;
}

Pmf bit_pmf(double Pi, double Pd) {
  const double Pt = 1.0 - Pi - Pd;
  int K = 0;  // truncate the insertion count at the first Pi^k < 1e-17 (cap 64)
  while (K < 64 && Pi > 0 && std::pow(Pi, K + 1) >= 1e-17) K++;
  Pmf r;
  r.off = -1;
  r.p.assign(K + 2, 0.0);
  for (int k = 0; k <= K; k++) {
    r.p[k] += std::pow(Pi, k) * Pd;      // change k - 1 at index k
    r.p[k + 1] += std::pow(Pi, k) * Pt;  // change k at index k + 1
  }
  return r;
}

Pmf drift_pmf(long T, double Pi, double Pd) {
  Pmf res, base = bit_pmf(Pi, Pd);
  for (long t = T; t > 0; t >>= 1) {
    if (t & 1) {
      res = conv(res, base);
      trim(res, 1e-300);
    }
    if (t > 1) {
      base = conv(base, base);
      trim(base, 1e-300);
    }
  }
  return res;
}

bool valid_channel(double Pi, double Pd) { return Pi >= 0 && Pd >= 0 && Pi + Pd < 1; }

}  // namespace

namespace bsidmap {

// Phi_T on the device: out[f][m - lo] = P(S_T = m) for m in [lo, hi] (pmf copied once per frame).
__global__ void k_phi_fill(const double* pmf, int width, int frames, double* out) {
  const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < (long)frames * width) out[k] = pmf[k % width];
}

}  // namespace bsidmap

extern "C" {

int bsidmap_drift_pmf(int T, double Pi, double Pd, int lo, int hi, double* pmf) {
  if (T < 0 || hi < lo || !pmf || !valid_channel(Pi, Pd)) return BSIDMAP_EINVAL;
  const Pmf d = drift_pmf(T, Pi, Pd);
  for (int m = lo; m <= hi; m++) {
    const long j = m - d.off;
    pmf[m - lo] = (j >= 0 && j < (long)d.p.size()) ? d.p[j] : 0.0;
  }
  return BSIDMAP_OK;
}

int bsidmap_drift_limits(int T, double Pi, double Pd, double Pr, int* lo, int* hi) {
  if (T < 0 || !lo || !hi || !valid_channel(Pi, Pd) || !(Pr > 0 && Pr < 1)) return BSIDMAP_EINVAL;
  const Pmf d = drift_pmf(T, Pi, Pd);
  const long W = (long)d.p.size();
  // the excluded mass must be resolvable: the PMF's own truncation loss stays below Pr
  double mass = 0.0;
  for (long j = 0; j < W; j++) mass += d.p[j];
  if (!(1.0 - mass < Pr)) return BSIDMAP_EINVAL;
  // tail sums accumulated from the far ends (small terms first): left[j] = P(S < off + j),
  // right[j] = P(S > off + j)
  std::vector<double> left(W + 1, 0.0), right(W + 1, 0.0);
  for (long j = 0; j < W; j++) left[j + 1] = left[j] + d.p[j];
  for (long j = W - 1; j >= 0; j--) right[j] = (j + 1 < W ? right[j + 1] + d.p[j + 1] : 0.0);
  auto below = [&](long m) { const long j = m - d.off; return j <= 0 ? 0.0 : j >= W ? mass : left[j]; };
  auto above = [&](long m) { const long j = m - d.off; return j >= W ? 0.0 : j < 0 ? mass : right[j]; };
  // grow [0, 0] one state at a time on the side with more excluded mass (ties: the positive
  // side) until the excluded mass is below Pr (reading R8)
  long mlo = 0, mhi = 0;
  while (below(mlo) + above(mhi) >= Pr) {
    if (above(mhi) >= below(mlo)) mhi++;
    else mlo--;
  }
  *lo = (int)mlo;
  *hi = (int)mhi;
  return BSIDMAP_OK;
}

int bsidmap_drift_limits_tails(int T, double Pi, double Pd, double Pr, int* lo, int* hi) {
  if (T < 0 || !lo || !hi || !valid_channel(Pi, Pd) || !(Pr > 0 && Pr < 1)) return BSIDMAP_EINVAL;
  const Pmf d = drift_pmf(T, Pi, Pd);
  const size_t W = d.p.size();
  // m^- = max{m : P(S < m) <= Pr/2},  m^+ = min{m : P(S > m) <= Pr/2}  (the round-1 rule)
  long mlo = d.off, mhi = d.off + (long)W - 1;
  double below = 0.0;
  for (size_t j = 0; j < W; j++) {
    if (below <= Pr / 2) mlo = d.off + (long)j; else break;
    below += d.p[j];
  }
  double above = 0.0;
  for (size_t j = W; j-- > 0;) {
    if (above <= Pr / 2) mhi = d.off + (long)j; else break;
    above += d.p[j];
  }
  mlo = std::max(std::min(mlo, 0L), -(long)T);
  mhi = std::max(mhi, 0L);
  *lo = (int)mlo;
  *hi = (int)mhi;
  return BSIDMAP_OK;
}

int bsidmap_state_space(int n, int N, double Pi, double Pd, double Pr, int* mn_lo, int* mn_hi, int* mt_lo,
                        int* mt_hi) {
  if (n < 1 || N < 1 || !mn_lo || !mn_hi || !mt_lo || !mt_hi) return BSIDMAP_EINVAL;
  int rc = bsidmap_drift_limits(n, Pi, Pd, Pr, mn_lo, mn_hi);
  if (rc) return rc;
  if ((rc = bsidmap_drift_limits(n * N, Pi, Pd, Pr, mt_lo, mt_hi))) return rc;
  *mt_lo = std::min(*mt_lo, *mn_lo);  // m_tau must contain m_n (create() requires it)
  *mt_hi = std::max(*mt_hi, *mn_hi);
  return BSIDMAP_OK;
}

int bsidmap_phi(int T, double Pi, double Pd, int lo, int hi, int num_frames, double* out_dev, void* stream) {
  if (num_frames < 1 || !out_dev || hi < lo) return BSIDMAP_EINVAL;
  std::vector<double> h(hi - lo + 1);
  int rc = bsidmap_drift_pmf(T, Pi, Pd, lo, hi, h.data());
  if (rc) return rc;
  double* tmp = nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMallocAsync(&tmp, h.size() * sizeof(double), s) != cudaSuccess) return BSIDMAP_ENOMEM;
  cudaMemcpyAsync(tmp, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, s);
  const long tot = (long)num_frames * (long)h.size();
  bsidmap::k_phi_fill<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(tmp, (int)h.size(), num_frames, out_dev);
  cudaFreeAsync(tmp, s);
  cudaError_t e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? BSIDMAP_OK : BSIDMAP_ECUDA;
}

}  // extern "C"
