// mc.cu -- Monte-Carlo symbol/frame error-rate workload on the device:
// encoder + BSID channel generated in HBM, the batched decoder, and an
// error counter, so a simulation never round-trips frames through the host (the paper's use
// of the decoder in its simulator).
//
// The generator is the SAME counter-based stream as the host generator (bsidgen/bsidgen.c:
// SplitMix64 keyed by (seed, stream, frame index)), implemented again here so that device
// frames are bit-identical to host frames (tests/test_gpu_mc.py).  One thread per frame runs
// the literal per-time-step event loop; frames whose end drift leaves [m_tau^-, m_tau^+] are
// redrawn from the continuing stream and counted.
#include <cstdint>

#include "../../include/bsidmap.h"
#include "common.cuh"

namespace bsidmap {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
struct Rng {
  uint64_t key, ctr;
};
__device__ __forceinline__ Rng rng_make(uint64_t seed, uint64_t stream, uint64_t index) {
  Rng r;
  r.key = splitmix64(splitmix64(seed ^ 0x1802084830000000ull) ^ splitmix64(stream * 0x632BE59BD9B4E019ull + 1)) ^
          splitmix64(index + 0x2545F4914F6CDD1Dull);
  r.ctr = 0;
  return r;
}
__device__ __forceinline__ uint64_t rng_next(Rng& r) { return splitmix64(r.key + 0x9E3779B97F4A7C15ull * (++r.ctr)); }
__device__ __forceinline__ double rng_unif(Rng& r) {
  return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ uint64_t rng_below(Rng& r, uint64_t bound) {
  const uint64_t lim = UINT64_MAX - (UINT64_MAX % bound);
  uint64_t v;
  do {
    v = rng_next(r);
  } while (v >= lim);
  return v % bound;
}
constexpr uint64_t kStreamMessage = 2, kStreamChannel = 3;

}  // namespace

struct McParams {
  uint64_t seed;
  long first;
  int F, N, q, n, wpf, mt_lo, mt_hi;
  double Pi, Pd, Ps;
  const uint32_t* C;
  int32_t* msg;
  uint32_t* rx;
  int32_t* rho;
  unsigned long long* redraws;
};

__global__ void k_mc_generate(const McParams P) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= P.F) return;
  const uint64_t gf = (uint64_t)(P.first + f);
  Rng rm = rng_make(P.seed, kStreamMessage, gf), rc = rng_make(P.seed, kStreamChannel, gf);
  int32_t* m = P.msg + (size_t)f * P.N;
  uint32_t* w = P.rx + (size_t)f * P.wpf;
  for (int i = 0; i < P.N; i++) m[i] = (int32_t)rng_below(rm, (uint64_t)P.q);
  const long tau = (long)P.n * P.N, cap = (long)P.wpf * 32;
  unsigned long long red = 0;
  for (;;) {
    long out = 0;
    for (int k = 0; k < P.wpf; k++) w[k] = 0u;
    for (int i = 0; i < P.N; i++) {
      const uint32_t word = P.C[(size_t)i * P.q + m[i]];
      for (int t = 0; t < P.n; t++) {
        const uint32_t xb = (word >> t) & 1u;
        for (;;) {  // events at time t
          const double u = rng_unif(rc);
          uint32_t ob;
          if (u < P.Pi) {
            ob = (uint32_t)(rng_next(rc) >> 63);  // insertion: uniform random bit, stay at t
          } else if (u < P.Pi + P.Pd) {
            break;  // deletion
          } else {
            ob = xb ^ (uint32_t)(rng_unif(rc) < P.Ps);  // transmission (+ substitution)
          }
          if (out < cap) w[out >> 5] |= ob << (out & 31);
          out++;
          if (u >= P.Pi) break;
        }
      }
    }
    if (out - tau >= P.mt_lo && out - tau <= P.mt_hi) {
      P.rho[f] = (int32_t)out;
      break;
    }
    red++;
  }
  if (red) atomicAdd(P.redraws, red);
}

// counters[0] symbol errors, [1] frame errors, [2] failed frames (status != OK, counted as frame errors)
__global__ void k_mc_count(const float* L, const int32_t* msg, const int32_t* status, int F, int N, int q,
                           unsigned long long* counters) {
  const int f = blockIdx.x;
  if (f >= F) return;
  const bool ok = status[f] == kFrameOk;
  unsigned long long errs = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const float* row = L + ((size_t)f * N + i) * q;
    int best = 0;
    float bv = row[0];
    for (int D = 1; D < q; D++)
      if (row[D] > bv) {  // argmax, lowest D on ties (reading R12)
        bv = row[D];
        best = D;
      }
    errs += (!ok || best != msg[(size_t)f * N + i]) ? 1ull : 0ull;
  }
  for (int o = 16; o > 0; o >>= 1) errs += __shfl_xor_sync(0xffffffffu, errs, o);
  __shared__ unsigned long long s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = errs;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < (int)(blockDim.x + 31) / 32; k++) t += s[k];
    atomicAdd(counters + 0, t);
    if (t) atomicAdd(counters + 1, 1ull);
    if (!ok) atomicAdd(counters + 2, 1ull);
  }
}

}  // namespace bsidmap
