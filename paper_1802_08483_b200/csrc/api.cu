// api.cu -- the C ABI (include/bsidmap.h): argument validation, the launch
// planner (row a6: storage schedule from the memory estimate, chunking,
// grid/block geometry for 148 SMs) and the launch sequence of one decode.
//
// Launch sequence per chunk of frames (all on the caller's stream):
//   k_frame_init -> memset(Lacc) -> lattice pass 1 (Gamma; STORED: + gamma)
//   -> k_alpha_beta -> lattice pass 2 (RECOMPUTE) | k_app_stored (STORED)
//   -> k_finalize
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "../../include/bsidmap.h"
#include "k_local_x2.cuh"
#include "k_alphabeta_cta.cuh"
#include "k_local_cta.cuh"

namespace bsidmap {
__global__ void k_frame_init(const DecodeParams p);
__global__ void k_finalize(const DecodeParams p);
__global__ void k_zero_failed(const DecodeParams p);
__global__ void k_extrinsic(const DecodeParams p, float* E);
__global__ void k_live8(const DecodeParams p);
__global__ void k_live16(const DecodeParams p);
__global__ void k_live32(const DecodeParams p);
__global__ void k_alpha_support(const DecodeParams p);
__global__ void k_support_pack1(const DecodeParams p);
__global__ void k_support_pack2(const DecodeParams p, int nblk);
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
__global__ void k_mc_generate(const McParams P);
__global__ void k_mc_count(const float* L, const int32_t* msg, const int32_t* status, int F, int N, int q,
                           unsigned long long* counters);
}  // namespace bsidmap

namespace {
__global__ void k_iota_offsets(int64_t* off, int F, int wpf) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < F) off[f] = (int64_t)f * wpf;
}
}  // namespace

using namespace bsidmap;

namespace {
constexpr int kPhases = 5;
constexpr int kHostSub = 12;  // sub-batches of the host-buffer pipeline (at most 8 + 3)
constexpr int kMaxAbSub = 4;  // sub-batches of the alpha/beta-overlapped Gamma-sum pipeline
std::string g_err;  // failures without a decoder (create)
}  // namespace

struct bsidmap_decoder {
  int device = 0;
  int q = 0, n = 0, N = 0, mn_lo = 0, mn_hi = 0, mt_lo = 0, mt_hi = 0, Mn = 0, Mt = 0;
  double Pi = 0, Pd = 0, Ps = 0;
  int mode = BSIDMAP_MODE_AUTO;
  uint32_t* d_C = nullptr;
  void* d_orders = nullptr;  // symbol visiting orders (DecodeParams::Cp/Dp/Cs/Ds/Cst), one allocation
  size_t ord_off[8] = {};    // byte offsets: Cp, Dp, Cs2, Ds2, Cst2, Cs3, Ds3, Cst3
  CoreKernels kern{};
  bool spec = false;
  bool jit = false;                     // spec kernels compiled at run time (jit.cu)
  bool slab_ok = false;                 // RECOMPUTE may run the slab schedule (spec cores)
  int slab_fixed = 0;                   // symbol indices per slab (0 = automatic)
  bool slab_askip = true;               // backward sweep: Gamma only where alpha != 0 (BSIDMAP_SLAB_ASKIP)
  std::string jit_err;                  // why a shape without a unit runs on the generic core
  LatticeConst lc{};
  // workspace
  void* ws = nullptr;
  size_t ws_bytes = 0;
  size_t ws_limit = 0;
  int last_chunk = 0, last_frames = 0, last_sched = 0;
  // host-path staging and the D2H pipeline
  void* hs = nullptr;
  size_t hs_bytes = 0;
  cudaStream_t s_copy = nullptr;
  cudaEvent_t ev_sub[kHostSub] = {};
  // host-side caches: the free-memory query and the smem opt-ins cost ~1 ms per call,
  // which would dominate single-frame latency (C1)
  size_t budget_cache = 0;
  int budget_frames = -1, budget_mode = -1;
  std::vector<std::pair<const void*, size_t>> smem_set;
  // alpha/beta overlap: sub-batch k's alpha/beta recursions run on a high-priority side
  // stream while the lattice passes of the other sub-batches run on the decode stream
  int ab_sub = 0;                       // sub-batches per chunk (0 = automatic, 1 = no overlap)
  int ab_stages = 0, ab_threads = 0;    // CTA alpha/beta ring depth and block size (0 = automatic)
  int num_sms = 148;
  int app_kp = -1;                      // pass-2 prefix length override (-1 = automatic)
  int app_ks = -1;                      // rows folded into the APP weights (-1 = automatic; BSIDMAP_APP_KS)
  double live_eps = 0x1p-128;           // live-window threshold of the APP pass (reading R18; BSIDMAP_LIVE_EPS)
  int app_G = 0;                        // its frames per warp (0 = automatic; BSIDMAP_APP_G)
  cudaStream_t s_ab = nullptr;
  cudaEvent_t ev_p1[kMaxAbSub] = {}, ev_ab[kMaxAbSub] = {};
  cudaEvent_t ev_abt[2] = {};           // alpha/beta stream busy time (timed decodes)
  bool ab_overlapped = false;           // last decode used the side stream
  // timing
  bool timing = false;
  cudaEvent_t ev[kPhases + 1] = {};
  cudaStream_t ev_stream = nullptr;
  bool ev_valid = false;
  long launches = 0;
  std::string err;
};

namespace {

int fail(bsidmap_decoder* d, int code, const std::string& msg) {
  if (d) d->err = msg; else g_err = msg;
  return code;
}

// Launch a kernel of the core table through cudaLaunchKernel: the table holds either the address
// of a statically compiled __global__ function or a cudaKernel_t of a run-time compiled shape
// (jit.cu, cast to the same pointer type), which the runtime accepts in the same place.
template <class... A>
void launch_k(void (*fn)(A...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A... args) {
  void* argv[] = {static_cast<void*>(&args)...};
  cudaLaunchKernel(reinterpret_cast<const void*>(fn), grid, block, argv, smem, s);
}

int cuda_fail(bsidmap_decoder* d, cudaError_t e, const char* what) {
  return fail(d, BSIDMAP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t gsum, gamma, alpha, beta, lacc, live, spack, sblk, total;
};


// Bytes per frame of each workspace array (the paper's memory estimate).
// Storage schedules.  kSchedLocal is the paper's local storage: gamma computed in
// the alpha pass and again in the beta + L pass, only alpha rows kept.  kSchedGammaSum keeps
// Gamma = sum_D gamma between two parallel lattice passes.  kSchedStored keeps every gamma.
// kSchedLocalCta is the same schedule with one CTA per frame (M_tau > 64).
// kSchedSlab is the local storage in slabs of B symbol indices (the B200 form of P:483-522; DESIGN
// 5): a forward sweep computes Gamma for one slab at a time (the fully parallel pass-1 kernel) and
// runs alpha through it, a backward sweep recomputes Gamma only where alpha_i(m') != 0 (reading R19),
// runs beta through it and the live-window APP over it; alpha and beta rows are kept, Gamma only
// for two slabs in flight.
enum Sched { kSchedStored = 1, kSchedLocal = 2, kSchedGammaSum = 3, kSchedLocalCta = 4, kSchedSlab = 5 };

// Windows per Gamma slab: pass 1 of one slab is ~16 waves of 3 CTAs (256 windows x 8 symbol indices
// each) on every SM; the slab length is a multiple of the pass-1 CTA's 8 symbol indices, and the
// two-slab ring at most a quarter of the Gamma-sum schedule's Gamma (slabs of <= N/8).  Measured (C5,
// 32 frames; tools/exp_slab.py): slabs of 64 / 128 / 256 / 512 symbol indices 375 / 362 / 311 / 299 ms
// (the last two with the packed backward sweep); C2 (65536 frames): 8 / 100 indices 125.8 / 126.5 ms.
constexpr long kSlabWindows = 16L * 3 * 256 * 8 * 148;
int slab_len(const bsidmap_decoder* d, long F) {
  if (d->slab_fixed > 0) return std::min(d->slab_fixed, d->N);  // BSIDMAP_SLAB_LEN (tests: many slabs at small N)
  const long per_i = std::max(1L, F * d->Mt);
  long B = (kSlabWindows + per_i - 1) / per_i;
  B = std::min(B, std::max(8L, (long)d->N / 8));
  B = (B + 7) / 8 * 8;
  return (int)std::max(1L, std::min<long>(B, d->N));
}
// beta rows the slab schedule keeps per frame: a ring of three slabs (the backward sweep writes slab
// b while the APP of slab b + 1 reads its rows and the first row of slab b + 2), or all N + 1
int slab_beta_rows(const bsidmap_decoder* d, int B) { return std::min(d->N + 1, 3 * B); }

int resolve_sched(const bsidmap_decoder* d, int mode) {
  if (mode == BSIDMAP_MODE_STORED) return kSchedStored;
  // AUTO: Gamma-sum -- fully parallel lattice passes; measured fastest on B200 (C2: 140.6 ms vs
  // 148.4 ms for the fused local schedule per 65536 frames, profiles/r01_*)
  if (mode == BSIDMAP_MODE_GAMMASUM || mode == BSIDMAP_MODE_AUTO) return kSchedGammaSum;
  // RECOMPUTE: the slab schedule on the spec cores (the live-window APP), else the paper's local
  // schedule where a frame fits one warp tile or one CTA, else Gamma-sum
  if (d->slab_ok && mode == BSIDMAP_MODE_RECOMPUTE) return kSchedSlab;
  if (d->kern.local_fwd && d->Mt <= kTileSlots) return kSchedLocal;
  if (d->kern.local_cta_bwd[0] && d->Mt <= 4 * kLocalCtaThreads &&
      local_cta_fwd_smem(d->Mn, gsum_stride(d->Mt)) <= 227u * 1024 &&
      local_cta_bwd_smem(d->Mn, gsum_stride(d->Mt), d->q) <= 227u * 1024)
    return kSchedLocalCta;
  return kSchedGammaSum;
}

// One frame per warp of the live-window APP with one folded row fits in shared memory.
bool live_app_smem_fits(const CoreKernels& k, int q, int Mn) {
  const size_t need = k.app_live_W == 2 ? kX2Warps * app_live_x2_warp_smem(q, Mn, 1, 1)
                                        : app_live_x1_cta_tables(Mn, 1) + kX2Warps * app_live_x1_warp_smem(q, 1);
  return need <= 227u * 1024;
}

// The Gamma-sum schedule runs the live-window APP (k_app_live.cuh) on the spec cores.
bool uses_live_app(const bsidmap_decoder* d, int sched) {
  if ((sched != kSchedGammaSum && sched != kSchedSlab) || d->kern.app_live[0][0] == nullptr) return false;
  return live_app_smem_fits(d->kern, d->q, d->Mn);
}

const char* sched_name(int s) {
  return s == kSchedStored ? "stored"
         : s == kSchedLocal ? "recompute-local"
         : s == kSchedLocalCta ? "recompute-local-cta"
         : s == kSchedSlab     ? "recompute-slab"
                               : "recompute-gammasum";
}

Layout layout(const bsidmap_decoder* d, long F, int sched) {
  Layout l{};
  const bool local = sched == kSchedLocal || sched == kSchedLocalCta;
  const size_t blocks = sched == kSchedSlab ? 2 * (size_t)slab_len(d, F) : (size_t)d->N;  // Gamma_i blocks per frame
  l.gsum = local ? 0 : align_up((size_t)F * blocks * d->Mn * gsum_stride(d->Mt) * sizeof(float));
  l.gamma = sched == kSchedStored ? align_up((size_t)F * d->N * d->q * d->Mn * d->Mt * sizeof(float)) : 0;
  l.alpha = align_up((size_t)F * (d->N + 1) * d->Mt * sizeof(double));
  l.beta = local ? 0
         : sched == kSchedSlab ? align_up((size_t)F * slab_beta_rows(d, slab_len(d, F)) * d->Mt * sizeof(double))
                               : l.alpha;
  const bool live = uses_live_app(d, sched);
  l.lacc = (local || live) ? 0 : align_up((size_t)F * d->N * d->q * sizeof(double));
  l.live = live ? align_up((size_t)F * d->N * sizeof(int2)) : 0;
  // slab backward sweep: packed alpha-support windows, (F + 1) entries per symbol-index group
  l.spack = sched == kSchedSlab ? align_up(((size_t)F + 1) * slab_len(d, F) * sizeof(int2)) : 0;
  l.sblk = sched == kSchedSlab ? align_up((size_t)((F + 255) / 256) * slab_len(d, F) * sizeof(int)) : 0;
  l.total = l.gsum + l.gamma + l.alpha + l.beta + l.lacc + l.live + l.spack + l.sblk;
  return l;
}

struct Plan {
  int mode;         // schedule (Sched)
  int chunk;        // frames per chunk
  int nchunks;
  int ab_threads;   // k_alpha_beta block size
  int ab_stages;    // k_alpha_beta TMA ring depth
  size_t ab_smem, app_smem, l1_smem;
  void (*ab_warp)(const DecodeParams);  // warp-per-task alpha/beta kernel or nullptr
  void (*ab_cta)(const DecodeParams, int);  // CTA-per-task alpha/beta kernel (spec M_n instance or generic)
  bool direct_L;                         // APP pass writes normalised L rows itself
  size_t local_smem;                     // k_local_fwd / k_local_bwd dynamic smem
  void (*l1_kernel)(const DecodeParams);  // pass-1 kernel of the recompute schedules
  int ab_sub;                              // sub-batches of the alpha/beta-overlapped pipeline
  void (*app_kernel)(const DecodeParams);  // pass-2 kernel (prefix-sharing instance where available)
  int app_kp;                              // its prefix length (0 = none)
  int app_ks;                              // lattice rows folded into the APP weights (1 or 2)
  bool app_live;                           // app_kernel is the live-window APP (k_app_live.cuh)
  int app_G;                               // its frames per warp
  int slab;                                // symbol indices per Gamma slab (kSchedSlab)
};

size_t budget(const bsidmap_decoder* d) {
  if (d->ws_limit) return d->ws_limit;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return 0;
  return (size_t)((double)(fr + d->ws_bytes) * 0.85);
}

// Budget for a plan of F frames: re-query free memory only when the request changes or the
// current workspace is too small (the query is a synchronous driver call).
size_t budget_for(bsidmap_decoder* d, int F, int mode, size_t need) {
  if (d->ws_limit) return d->ws_limit;
  if (d->budget_cache && d->budget_mode == mode && need <= d->ws_bytes) return d->budget_cache;
  d->budget_cache = budget(d);
  d->budget_frames = F;
  d->budget_mode = mode;
  return d->budget_cache;
}

// Frames per warp of the live-window APP: 12 on the pair core (rounds of 64 windows), 8 / 4 on the
// scalar core (rounds of 32) for q <= 32 / larger, fewer where the grid would not fill the GPU.  Measured (tools/exp_appG*.sh,
// pass 2 ms at G = 4 / 8 / 12): C2 (pair) 35.9 / 36.1 / 32.0, C4 (pair) 36.6 / 35.4 / 36.0,
// C5 (scalar) 27.0 / 29.8 / 32.1, C3 (scalar) 35.4 / 34.5 / 34.6.  Results do not depend on G beyond
// the FP64 association of a frame split over two rounds (test_live_app_independent_of_packing).
int live_frames_per_warp(const bsidmap_decoder* d, long rows) {
  const long gmax = std::max(1L, rows / (32L * d->num_sms));
  return (int)std::min<long>(d->kern.app_live_W == 2 ? 12 : d->q <= 32 ? 8 : 4, gmax);
}

int make_plan(bsidmap_decoder* d, int F, Plan* P) {
  // Stored gamma costs 8 B of HBM traffic per gamma value against ~5n FP32 flops to
  // recompute it; on B200 recomputing is the faster side of the ridge, and
  // the only one whose batches fit for long frames: AUTO = recompute.
  const int mode = resolve_sched(d, d->mode);
  const size_t per = layout(d, 1, mode).total;
  const size_t bud = budget_for(d, F, mode, layout(d, F, mode).total);
  long chunk = per ? (long)(bud / per) : F;
  if (mode == kSchedSlab) {  // the Gamma slabs depend on the chunk (automatic length: ~constant bytes)
    long lo = 0, hi = F;     // largest chunk whose whole layout fits the budget
    while (lo < hi) {
      const long mid = (lo + hi + 1) / 2;
      if (layout(d, mid, mode).total <= bud) lo = mid; else hi = mid - 1;
    }
    chunk = lo;
  }
  if (chunk < 1) return fail(d, BSIDMAP_ENOMEM, "workspace for one frame (" + std::to_string(per) +
                                                    " B) exceeds the budget (" + std::to_string(bud) + " B)");
  chunk = std::min<long>(chunk, F);
  {  // equal chunks (a short tail chunk would leave the GPU half idle)
    const long nch = (F + chunk - 1) / chunk;
    chunk = (F + nch - 1) / nch;
  }
  P->mode = mode;
  P->chunk = (int)chunk;
  P->nchunks = (int)((F + chunk - 1) / chunk);
  P->slab = mode == kSchedSlab ? slab_len(d, chunk) : d->N;
  // CTA alpha/beta: ~2 states per thread (smaller blocks, more of them resident per SM), and a
  // single-stage Gamma ring when the grid has several CTAs per SM -- the other resident CTAs hide
  // each one's copy latency (C3: 11.7 -> 7.7 ms, C4: 14.6 -> 11.9 ms; tools/exp_abcta*.sh).  The
  // block size depends on M_tau only, so chunking does not change the arithmetic.
  P->ab_threads = std::min(1024, std::max(64, ((d->Mt + 1) / 2 + 31) / 32 * 32));
  {  // TMA ring depth: up to 4 stages of Gamma_i blocks within ~200 KB of shared memory
    const int Mtp = gsum_stride(d->Mt);
    const size_t blk = (size_t)d->Mn * Mtp * 4;
    P->ab_stages = (int)std::max<size_t>(1, std::min<size_t>(4, (200u * 1024 - 2 * (size_t)Mtp * 8 - 600) / blk));
    if (2L * chunk >= 4L * d->num_sms) P->ab_stages = 1;
    if (d->ab_stages > 0) P->ab_stages = d->ab_stages;
    if (d->ab_threads > 0) P->ab_threads = std::min(1024, d->ab_threads);
    P->ab_smem = ab_cta_smem(d->Mn, Mtp, P->ab_stages);
    if (P->ab_smem > 227u * 1024) {  // a Gamma_i block beyond shared memory: read it from global (L2)
      P->ab_stages = 0;
      P->ab_smem = ab_cta_smem(d->Mn, Mtp, 0);
      if (mode != kSchedLocal && mode != kSchedLocalCta && P->ab_smem > 227u * 1024)  // (slab too)
        return fail(d, BSIDMAP_EPLAN, "M_tau too large for the alpha/beta state rows in shared memory");
    }
  }
  P->ab_warp = nullptr;
  P->ab_cta = d->kern.ab_cta ? d->kern.ab_cta : k_alpha_beta_cta<0>;
  if (P->ab_stages == 0) P->ab_cta = k_alpha_beta_cta<0, false>;  // Gamma_i read from global memory
  const int spt = (d->Mt + 31) / 32;
  const int spt_k = spt == 3 ? 4 : spt;
  const size_t ab_warp_bytes = (size_t)(kAbWarpThreads / 32) * ab_warp_smem(spt_k, d->Mn, gsum_stride(d->Mt));
  if (d->kern.ab_warp[0] && spt <= 4 && ab_warp_bytes <= 100 * 1024) {
    const int k = spt == 1 ? 0 : spt == 2 ? 1 : 2;
    P->ab_warp = d->kern.ab_warp[k];
    P->ab_smem = ab_warp_bytes;
  }
  P->local_smem = (size_t)kLocalWarps * local_warp_smem(d->Mn, d->q);
  if (mode == kSchedLocalCta) {  // CTA local schedule: the larger of the two passes' smem
    const int Mtp = gsum_stride(d->Mt);
    P->local_smem = std::max(local_cta_fwd_smem(d->Mn, Mtp), local_cta_bwd_smem(d->Mn, Mtp, d->q));
  }
  // pass 1: hoist the last K lattice rows out of the symbol loop (K = 3 for q > 24, else 2)
  P->l1_kernel = (d->q > 24 && d->kern.gamma_sum_k3) ? d->kern.gamma_sum_k3 : d->kern.gamma_sum;
  // pass 2 (APP, row a4).  Local schedules: inside k_local_*_bwd.  Stored gamma: k_app_stored.
  // Gamma-sum on a spec core: the live-window APP (k_app_live.cuh) -- only the windows of each
  // (frame, i) row whose posterior mass exceeds eps (k_live), packed G frames per warp, the warps
  // writing the L rows themselves.  Generic core: k_app (FP64 atomics into Lacc, then k_finalize).
  P->direct_L = mode == kSchedLocal || mode == kSchedLocalCta;
  P->app_kp = 0;
  P->app_ks = 1;
  P->app_live = false;
  P->app_G = 1;
  const size_t nwin = kLatticeThreads;
  P->app_smem = nwin * sizeof(double) + (size_t)kAppSegCap * std::min(d->q, kAppDChunk) * sizeof(double) +
                nwin * app_tstride(d->q) * 4 + (size_t)d->q * 4;
  P->app_kernel = mode == kSchedStored ? d->kern.app_stored : d->kern.app;
  if (uses_live_app(d, mode)) {
    P->app_live = true;
    P->direct_L = true;
    // share lattice rows 1..KP between symbols with equal first KP codeword bits
    P->app_kp = app_prefix_bits(d->q, d->n);
    if (d->app_kp >= 0) P->app_kp = (d->app_kp == 0 || d->app_kp > d->n - 2) ? 0 : std::min(4, std::max(2, d->app_kp));
    // fold the last one or two lattice rows into the weights (the core's app_ks_auto: two on the
    // scalar core, one on the pair core, by measurement; tools/exp_appkpks.sh)
    const int ks = d->app_ks > 0 ? d->app_ks : d->kern.app_ks_auto;
    P->app_ks = (ks == 2 && d->n >= 3) ? 2 : 1;
    auto smem = [&](int ksv, int g) {
      return d->kern.app_live_W == 2 ? kX2Warps * app_live_x2_warp_smem(d->q, d->Mn, ksv, g)
                                     : app_live_x1_cta_tables(d->Mn, ksv) + kX2Warps * app_live_x1_warp_smem(d->q, g);
    };
    if (smem(P->app_ks, 1) > 227u * 1024) P->app_ks = 1;
    // up to 8 frames per warp (fewer partly filled rounds); fewer where the grid would not fill the
    // GPU or the per-frame sums would not fit in shared memory
    // rows of one APP launch: the chunk's, or one slab's (slab schedule)
    const long rows = (long)chunk * (mode == kSchedSlab ? slab_len(d, chunk) : d->N);
    int G = d->app_G > 0 ? std::min(d->app_G, kLiveMaxG) : live_frames_per_warp(d, rows);
    while (G > 1 && smem(P->app_ks, G) > 227u * 1024) G--;
    P->app_kernel = d->kern.app_live[P->app_ks - 1][P->app_kp > 0 ? P->app_kp - 1 : 0];
    P->app_G = G;
    P->app_smem = smem(P->app_ks, G);
  }
  // alpha/beta overlap (Gamma-sum only): measured on B200 it only pays where the alpha/beta grid
  // cannot fill the GPU (one CTA per frame and direction, 2F <= #SMs: C5 at 32 frames/GPU,
  // 401 vs 424 ms); with a full grid the recursions compete with the lattice passes for issue
  // slots and the step time is unchanged (C2, C4) or worse (C3: 212 vs 208 ms) -- tools/exp_ab.sh
  if (mode != kSchedGammaSum)
    P->ab_sub = 1;  // (the slab schedule overlaps alpha/beta with the next slab's pass 1 instead)
  else if (d->ab_sub > 0)
    P->ab_sub = std::min(kMaxAbSub, d->ab_sub);
  else
    P->ab_sub = (!P->ab_warp && 2L * chunk <= d->num_sms) ? 2 : 1;
  if (mode == kSchedSlab && !P->app_live) return fail(d, BSIDMAP_EPLAN, "slab schedule without the live-window APP");
  P->l1_smem = (d->kern.gamma_sum_k3 && mode != kSchedStored)
                   ? (size_t)d->Mn * kLatticeThreads * 8 + (size_t)d->q * 6 + 64 + 16 +
                         d->kern.l1_head_bytes[P->l1_kernel == d->kern.gamma_sum_k3 ? 1 : 0]
                   : (size_t)d->q * 4;
  return BSIDMAP_OK;
}

int ensure_ws(bsidmap_decoder* d, size_t bytes) {
  if (bytes <= d->ws_bytes) return BSIDMAP_OK;
  if (d->ws) {
    cudaDeviceSynchronize();
    cudaFree(d->ws);
    d->ws = nullptr;
    d->ws_bytes = 0;
  }
  cudaError_t e = cudaMalloc(&d->ws, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(d, BSIDMAP_ENOMEM, "cudaMalloc(" + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e));
  }
  d->ws_bytes = bytes;
  return BSIDMAP_OK;
}

int set_smem(bsidmap_decoder* d, const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return BSIDMAP_OK;
  for (auto& fs : d->smem_set)
    if (fs.first == fn && fs.second >= bytes) return BSIDMAP_OK;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return cuda_fail(d, e, "cudaFuncSetAttribute(smem)");
  d->smem_set.emplace_back(fn, bytes);
  return BSIDMAP_OK;
}

void fill_params(const bsidmap_decoder* d, DecodeParams* p) {
  std::memset(p, 0, sizeof(*p));
  p->q = d->q; p->n = d->n; p->N = d->N;
  p->mn_lo = d->mn_lo; p->mn_hi = d->mn_hi; p->Mn = d->Mn;
  p->mt_lo = d->mt_lo; p->mt_hi = d->mt_hi; p->Mt = d->Mt;
  p->Mtp = gsum_stride(d->Mt);
  p->C = d->d_C;
  const char* ob = static_cast<const char*>(d->d_orders);
  p->Cp = reinterpret_cast<const uint32_t*>(ob + d->ord_off[0]);
  p->Dp = reinterpret_cast<const uint16_t*>(ob + d->ord_off[1]);
  for (int k = 0; k < 2; k++) {
    p->Cs[k] = reinterpret_cast<const uint32_t*>(ob + d->ord_off[2 + 3 * k]);
    p->Ds[k] = reinterpret_cast<const uint16_t*>(ob + d->ord_off[3 + 3 * k]);
    p->Cst[k] = reinterpret_cast<const int*>(ob + d->ord_off[4 + 3 * k]);
  }
  p->lc = d->lc;
  p->live_eps = d->live_eps;
  p->gs_N = d->N;  // every Gamma_i block kept (the slab schedule narrows this per slab)
  p->gs_i0 = 0;
  p->ab_r0 = 0;    // alpha/beta: the whole recursion, both directions
  p->ab_r1 = d->N;
  p->ab_dir = -1;
  p->beta_rows = d->N + 1;
}

void bind_ws(const bsidmap_decoder* d, const Layout& l, DecodeParams* p) {
  char* b = static_cast<char*>(d->ws);
  p->Gsum = reinterpret_cast<float*>(b);
  b += l.gsum;
  p->gamma = l.gamma ? reinterpret_cast<float*>(b) : nullptr;
  b += l.gamma;
  p->alpha = reinterpret_cast<double*>(b);
  b += l.alpha;
  p->beta = reinterpret_cast<double*>(b);
  b += l.beta;
  p->Lacc = l.lacc ? reinterpret_cast<double*>(b) : nullptr;
  b += l.lacc;
  p->live = l.live ? reinterpret_cast<int2*>(b) : nullptr;
  b += l.live;
  p->spack = l.spack ? reinterpret_cast<int2*>(b) : nullptr;
  b += l.spack;
  p->spack_blk = l.sblk ? reinterpret_cast<int*>(b) : nullptr;
}

void record(bsidmap_decoder* d, int k, cudaStream_t s) {
  if (d->timing) cudaEventRecord(d->ev[k], s);
}

// Lattice-pass launches over i in slices of <= 65535 (gridDim.y limit).
template <class Fn>
void for_i_slices(int N, Fn fn) {
  for (int i0 = 0; i0 < N; i0 += 65535) fn(i0, std::min(65535, N - i0));
}


// The per-frame slice [f0, f0 + nf) of a chunk's parameters (every per-frame array offset).
DecodeParams sub_params(const DecodeParams& p, int f0, int nf) {
  DecodeParams s = p;
  const size_t N = (size_t)p.N, q = (size_t)p.q, Mt = (size_t)p.Mt;
  s.F = nf;
  s.rx_off += f0;
  s.rho += f0;
  if (s.priors) s.priors += (size_t)f0 * N * q;
  if (s.alpha0) s.alpha0 += (size_t)f0 * Mt;
  if (s.betaN) s.betaN += (size_t)f0 * Mt;
  s.status += f0;
  if (s.Gsum) s.Gsum += (size_t)f0 * p.gs_N * p.Mn * p.Mtp;
  if (s.gamma) s.gamma += (size_t)f0 * N * q * p.Mn * Mt;
  s.alpha += (size_t)f0 * (N + 1) * Mt;
  if (s.beta) s.beta += (size_t)f0 * p.beta_rows * Mt;
  if (s.Lacc) s.Lacc += (size_t)f0 * N * q;
  if (s.live) s.live += (size_t)f0 * N;
  s.L += (size_t)f0 * N * q;
  return s;
}

int ensure_ab_stream(bsidmap_decoder* d) {
  if (d->s_ab) return BSIDMAP_OK;
  int lo = 0, hi = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&d->s_ab, cudaStreamNonBlocking, hi);
  for (int k = 0; e == cudaSuccess && k < kMaxAbSub; k++) {
    e = cudaEventCreateWithFlags(&d->ev_p1[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_ab[k], cudaEventDisableTiming);
  }
  for (int k = 0; e == cudaSuccess && k < 2; k++) e = cudaEventCreate(&d->ev_abt[k]);
  if (e != cudaSuccess) return cuda_fail(d, e, "alpha/beta stream");
  return BSIDMAP_OK;
}

// The pass-1 kernel a decode launches: the stored-gamma kernel, or the plan's class kernel in its
// non-uniform-prior instance when priors are given (the smem opt-in is set on this same pointer).
void (*pass1_kernel(const bsidmap_decoder* d, const Plan& P, bool priors))(const DecodeParams) {
  auto l1 = P.mode == kSchedStored ? d->kern.gamma_store : P.l1_kernel;
  if (P.mode != kSchedStored && priors) {
    if (l1 == d->kern.gamma_sum && d->kern.gamma_sum_pri) l1 = d->kern.gamma_sum_pri;
    if (l1 == d->kern.gamma_sum_k3 && d->kern.gamma_sum_k3_pri) l1 = d->kern.gamma_sum_k3_pri;
  }
  return l1;
}

// Pass-1 grid: x over the windows of F frames, y over groups of `steps` symbol indices of [ib, ie).
// The class kernels walk up to kL1Steps symbol indices per CTA -- fewer where the grid would not fill
// the GPU (small batches: single-frame latency).
unsigned pass1_gx(const bsidmap_decoder* d, long F) {
  const long lanes = F * d->Mt;
  return d->kern.l1_W == 2 ? (unsigned)((lanes + 2 * kLatticeThreads - 1) / (2 * kLatticeThreads))
                           : (unsigned)((lanes + kLatticeThreads - 1) / kLatticeThreads);
}
int pass1_steps(const bsidmap_decoder* d, const Plan& P, long F, int ib, int ie) {
  const bool multi = P.mode != kSchedStored && d->kern.l1_steps;
  const unsigned gx1 = pass1_gx(d, F);
  int steps = multi ? kL1Steps : 1;
  while (steps > 1 && (long)gx1 * ((ie - ib + steps - 1) / steps) < 8L * d->num_sms) steps >>= 1;
  return steps;
}

void launch_pass1(bsidmap_decoder* d, const Plan& P, DecodeParams p, cudaStream_t s, int ib = 0, int ie = -1) {
  if (ie < 0) ie = d->N;  // symbol indices [ib, ie)
  auto l1 = pass1_kernel(d, P, p.priors != nullptr);
  const unsigned gx1 = pass1_gx(d, p.F);
  const int steps = pass1_steps(d, P, p.F, ib, ie);
  p.i_steps = steps;
  for_i_slices(ie - ib, [&](int i0, int ni) {
    p.i_base = ib + i0;
    p.i_end = ib + i0 + ni;
    launch_k(l1, dim3(gx1, (unsigned)((ni + steps - 1) / steps)), kLatticeThreads, P.l1_smem, s, p);
    d->launches++;
  });
}

void launch_alpha_beta(bsidmap_decoder* d, const Plan& P, const DecodeParams& p, cudaStream_t s) {
  if (P.ab_warp) {
    const long tasks = (p.ab_dir < 0 ? 2L : 1L) * p.F, per = kAbWarpThreads / 32;
    launch_k(P.ab_warp, (unsigned)((tasks + per - 1) / per), kAbWarpThreads, P.ab_smem, s, p);
  } else {
    launch_k(P.ab_cta, dim3(p.F, p.ab_dir < 0 ? 2 : 1), P.ab_threads, P.ab_smem, s, p, P.ab_stages);
  }
  d->launches++;
}

void launch_pass2(bsidmap_decoder* d, const Plan& P, DecodeParams p, cudaStream_t s, int ib = 0, int ie = -1) {
  if (ie < 0) ie = d->N;  // symbol indices [ib, ie)
  if (P.app_live) {  // live windows of every (frame, i) row, then the packed APP over them
    const long rows = (long)p.F * (ie - ib);
    p.i_base = ib;
    p.i_end = ie;
    // k_live: 8 / 16 / 32 lanes per row for M_tau <= 64 / 128 / more (rows per 256-thread block: 32 / 16 / 8)
    if (d->Mt <= 64)
      k_live8<<<(unsigned)((rows + 31) / 32), 256, 0, s>>>(p);
    else if (d->Mt <= 128)
      k_live16<<<(unsigned)((rows + 15) / 16), 256, 0, s>>>(p);
    else
      k_live32<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(p);
    d->launches++;
    p.app_G = P.app_G;
    const unsigned gx = (unsigned)(((p.F + P.app_G - 1) / P.app_G + kX2Warps - 1) / kX2Warps);
    for_i_slices(ie - ib, [&](int i0, int ni) {
      p.i_base = ib + i0;
      launch_k(P.app_kernel, dim3(gx, ni), kLatticeThreads, P.app_smem, s, p);
      d->launches++;
    });
    return;
  }
  const long lanes = (long)p.F * d->Mt;
  const unsigned gx_flat = (unsigned)((lanes + kLatticeThreads - 1) / kLatticeThreads);
  auto l2 = P.app_kernel;
  for_i_slices(ie - ib, [&](int i0, int ni) {
    p.i_base = ib + i0;
    launch_k(l2, dim3(gx_flat, ni), kLatticeThreads, P.app_smem, s, p);
    d->launches++;
  });
}

// The slab schedule (kSchedSlab).  Gamma lives in two slab buffers (ring halves); slab b of B
// symbol indices uses half b & 1.  Forward sweep: pass 1 of slab b on the decode stream, alpha
// through it on the side stream (overlapping pass 1 of slab b + 1).  Backward sweep: pass 1 of slab
// b again, only for windows with alpha_i(m') != 0 (askip), beta through it on the side stream, and
// on the decode stream the live-window APP of slab b + 1 (its beta rows are complete by then).
int run_chunk_slab(bsidmap_decoder* d, const Plan& P, DecodeParams p, cudaStream_t s, bool first_chunk,
                   bool last_chunk) {
  int rc = ensure_ab_stream(d);
  if (rc) return rc;
  const int N = d->N, B = P.slab, nsl = (N + B - 1) / B;
  const size_t half = (size_t)p.F * B * d->Mn * p.Mtp;
  p.beta_rows = slab_beta_rows(d, B);  // the bound workspace holds this many rows per frame
  float* const ring = p.Gsum;
  auto slab_params = [&](int b, bool askip) {
    DecodeParams q = p;
    q.Gsum = ring + (b & 1) * half;
    q.gs_N = B;
    q.gs_i0 = b * B;
    q.askip = askip ? 1 : 0;
    return q;
  };
  if (first_chunk) record(d, 1, s);
  for (int b = 0; b < nsl; b++) {  // forward sweep: Gamma slab -> alpha
    const int i0 = b * B, i1 = std::min(N, i0 + B);
    DecodeParams q = slab_params(b, false);
    if (b >= 2) cudaStreamWaitEvent(s, d->ev_ab[b & 1], 0);  // alpha of slab b - 2 read this half
    launch_pass1(d, P, q, s, i0, i1);
    cudaEventRecord(d->ev_p1[b & 1], s);
    cudaStreamWaitEvent(d->s_ab, d->ev_p1[b & 1], 0);
    q.ab_r0 = i0;
    q.ab_r1 = i1;
    q.ab_dir = 0;
    launch_alpha_beta(d, P, q, d->s_ab);
    cudaEventRecord(d->ev_ab[b & 1], d->s_ab);
  }
  cudaStreamWaitEvent(s, d->ev_ab[(nsl - 1) & 1], 0);  // every alpha row (the backward sweep reads them)
  if (first_chunk) record(d, 2, s);
  if (first_chunk) record(d, 3, s);
  for (int b = nsl - 1; b >= 0; b--) {  // backward sweep: Gamma slab (alpha != 0) -> beta -> APP
    const int i0 = b * B, i1 = std::min(N, i0 + B);
    DecodeParams q = slab_params(b, d->slab_askip);
    if (b + 2 < nsl) cudaStreamWaitEvent(s, d->ev_ab[b & 1], 0);  // beta of slab b + 2 read this half
    if (q.askip) {  // alpha support of the slab's rows (p.live; k_live reuses the rows after beta)
      if (d->kern.l1_W != 2) {
        q.askip = 0;  // the pair core's pass 1 packs the windows with alpha != 0; others recompute all
      } else {
        DecodeParams r = q;
        r.i_base = i0;
        r.i_end = i1;
        r.i_steps = pass1_steps(d, P, p.F, i0, i1);  // the pass-1 CTA rows' symbol-index groups
        const unsigned groups = (unsigned)((i1 - i0 + r.i_steps - 1) / r.i_steps);
        const int nblk = (p.F + 255) / 256;
        k_alpha_support<<<(unsigned)(((long)p.F * (i1 - i0) + 7) / 8), 256, 0, s>>>(r);
        k_support_pack1<<<dim3(groups, nblk), 256, 0, s>>>(r);
        k_support_pack2<<<groups, 256, 0, s>>>(r, nblk);
        d->launches += 3;
      }
    }
    launch_pass1(d, P, q, s, i0, i1);
    cudaEventRecord(d->ev_p1[b & 1], s);
    cudaStreamWaitEvent(d->s_ab, d->ev_p1[b & 1], 0);
    q.ab_r0 = N - i1;
    q.ab_r1 = N - i0;
    q.ab_dir = 1;
    launch_alpha_beta(d, P, q, d->s_ab);
    cudaEventRecord(d->ev_ab[b & 1], d->s_ab);
    if (b + 1 < nsl) {  // the APP of slab b + 1: its beta rows are done
      cudaStreamWaitEvent(s, d->ev_ab[(b + 1) & 1], 0);
      launch_pass2(d, P, p, s, i1, std::min(N, i1 + B));
    }
  }
  cudaStreamWaitEvent(s, d->ev_ab[0], 0);
  launch_pass2(d, P, p, s, 0, std::min(N, B));
  if (first_chunk) record(d, 4, s);
  k_zero_failed<<<p.F, 256, 0, s>>>(p);
  d->launches++;
  if (last_chunk) record(d, 5, s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(d, e, "kernel launch");
  return BSIDMAP_OK;
}

int run_chunk(bsidmap_decoder* d, const Plan& P, DecodeParams p, cudaStream_t s, bool first_chunk, bool last_chunk) {
  if (first_chunk) record(d, 0, s);
  k_frame_init<<<(p.F + 255) / 256, 256, 0, s>>>(p);
  d->launches += 1;
  if (P.mode == kSchedLocal) {  // the paper's local schedule: two fused per-frame passes
    const unsigned gl = (unsigned)((p.F + kLocalWarps - 1) / kLocalWarps);
    if (first_chunk) record(d, 1, s);
    launch_k(d->kern.local_fwd, gl, kLocalWarps * 32, P.local_smem, s, p);
    if (first_chunk) record(d, 2, s);
    if (first_chunk) record(d, 3, s);
    launch_k(d->kern.local_bwd, gl, kLocalWarps * 32, P.local_smem, s, p);
    if (first_chunk) record(d, 4, s);
    k_zero_failed<<<p.F, 256, 0, s>>>(p);
    d->launches += 3;
    if (last_chunk) record(d, 5, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(d, e, "kernel launch");
    return BSIDMAP_OK;
  }
  if (P.mode == kSchedLocalCta) {  // the same schedule, one CTA per frame (M_tau > 64)
    const int kk = d->q > 24 ? 1 : 0, pr = p.priors ? 1 : 0;
    if (first_chunk) record(d, 1, s);
    launch_k(d->kern.local_cta_fwd[kk][pr], p.F, kLocalCtaThreads, P.local_smem, s, p);
    if (first_chunk) record(d, 2, s);
    if (first_chunk) record(d, 3, s);
    launch_k(d->kern.local_cta_bwd[pr], p.F, kLocalCtaThreads, P.local_smem, s, p);
    if (first_chunk) record(d, 4, s);
    k_zero_failed<<<p.F, 256, 0, s>>>(p);
    d->launches += 3;
    if (last_chunk) record(d, 5, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(d, e, "kernel launch");
    return BSIDMAP_OK;
  }
  if (P.mode == kSchedSlab) return run_chunk_slab(d, P, p, s, first_chunk, last_chunk);
  if (!P.direct_L) cudaMemsetAsync(p.Lacc, 0, (size_t)p.F * d->N * d->q * sizeof(double), s);
  const int S = std::min(P.ab_sub, p.F);
  if (S > 1) {
    // Sub-batch pipeline: pass 1 of every sub-batch on `s`; the alpha/beta recursions of
    // sub-batch k (HBM/latency-bound) on the high-priority side stream as soon as its Gamma
    // is written, overlapping the (FP32-bound) lattice passes of the other sub-batches;
    // pass 2 of sub-batch k waits for its alpha/beta rows.
    int rc = ensure_ab_stream(d);
    if (rc) return rc;
    if (first_chunk) record(d, 1, s);
    for (int k = 0; k < S; k++) {
      const int f0 = (int)((long)p.F * k / S), f1 = (int)((long)p.F * (k + 1) / S);
      const DecodeParams sp = sub_params(p, f0, f1 - f0);
      launch_pass1(d, P, sp, s);
      cudaEventRecord(d->ev_p1[k], s);
      cudaStreamWaitEvent(d->s_ab, d->ev_p1[k], 0);
      if (first_chunk && k == 0 && d->timing) cudaEventRecord(d->ev_abt[0], d->s_ab);
      launch_alpha_beta(d, P, sp, d->s_ab);
      if (first_chunk && k == S - 1 && d->timing) cudaEventRecord(d->ev_abt[1], d->s_ab);
      cudaEventRecord(d->ev_ab[k], d->s_ab);
    }
    if (first_chunk) record(d, 2, s);
    for (int k = 0; k < S; k++) {
      const int f0 = (int)((long)p.F * k / S), f1 = (int)((long)p.F * (k + 1) / S);
      cudaStreamWaitEvent(s, d->ev_ab[k], 0);
      if (first_chunk && k == 0) record(d, 3, s);  // phase 2 = the exposed part of alpha/beta
      launch_pass2(d, P, sub_params(p, f0, f1 - f0), s);
    }
    if (first_chunk) d->ab_overlapped = true;
  } else {
    if (first_chunk) record(d, 1, s);
    launch_pass1(d, P, p, s);
    if (first_chunk) record(d, 2, s);
    launch_alpha_beta(d, P, p, s);
    if (first_chunk) record(d, 3, s);
    launch_pass2(d, P, p, s);
  }
  if (first_chunk) record(d, 4, s);
  if (!P.direct_L) {
    const long rows = (long)p.F * d->N;
    k_finalize<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(p);
    d->launches++;
  }
  k_zero_failed<<<p.F, 256, 0, s>>>(p);
  d->launches++;
  if (last_chunk) record(d, 5, s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(d, e, "kernel launch");
  return BSIDMAP_OK;
}

// Symbol visiting orders of every C_i, computed once per decoder (they depend on the codebook only):
//  - lexicographic in (x_1, x_2, ..., x_n) -- the APP pass shares lattice rows 1..KP between
//    consecutive symbols with equal first KP bits (every prefix length is contiguous in this order);
//  - grouped by the class of the last K bits (K = 2, 3), stable -- pass 1 runs the last K rows once
//    per class.
cudaError_t upload_orders(bsidmap_decoder* d, const uint32_t* C) {
  const int N = d->N, q = d->q, n = d->n;
  const size_t nq = (size_t)N * q;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  d->ord_off[0] = off; off = al(off + nq * 4);
  d->ord_off[1] = off; off = al(off + nq * 2);
  for (int k = 0; k < 2; k++) {
    const int NC = 1 << (k + 2);
    d->ord_off[2 + 3 * k] = off; off = al(off + nq * 4);
    d->ord_off[3 + 3 * k] = off; off = al(off + nq * 2);
    d->ord_off[4 + 3 * k] = off; off = al(off + (size_t)N * (NC + 1) * 4);
  }
  std::vector<char> h(off, 0);
  auto rev = [n](uint32_t w) {  // bit t -> bit n-1-t: x_1 becomes the most significant
    uint32_t r = 0;
    for (int t = 0; t < n; t++) r |= ((w >> t) & 1u) << (n - 1 - t);
    return r;
  };
  std::vector<int> idx(q);
  for (int i = 0; i < N; i++) {
    const uint32_t* Ci = C + (size_t)i * q;
    for (int D = 0; D < q; D++) idx[D] = D;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return rev(Ci[a]) < rev(Ci[b]); });
    for (int k = 0; k < q; k++) {
      reinterpret_cast<uint32_t*>(h.data() + d->ord_off[0])[(size_t)i * q + k] = Ci[idx[k]];
      reinterpret_cast<uint16_t*>(h.data() + d->ord_off[1])[(size_t)i * q + k] = (uint16_t)idx[k];
    }
    for (int kk = 0; kk < 2; kk++) {
      const int K = kk + 2, NC = 1 << K, sh = n - K;
      auto cls = [&](int D) { return sh >= 0 ? (int)((Ci[D] >> sh) & (uint32_t)(NC - 1)) : 0; };
      for (int D = 0; D < q; D++) idx[D] = D;
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return cls(a) < cls(b); });
      int* st = reinterpret_cast<int*>(h.data() + d->ord_off[4 + 3 * kk]) + (size_t)i * (NC + 1);
      for (int c = 0; c <= NC; c++) st[c] = q;
      for (int k = q - 1; k >= 0; k--) {
        reinterpret_cast<uint32_t*>(h.data() + d->ord_off[2 + 3 * kk])[(size_t)i * q + k] = Ci[idx[k]];
        reinterpret_cast<uint16_t*>(h.data() + d->ord_off[3 + 3 * kk])[(size_t)i * q + k] = (uint16_t)idx[k];
        st[cls(idx[k])] = k;
      }
      for (int c = NC - 1; c >= 0; c--) st[c] = std::min(st[c], st[c + 1]);  // empty classes
    }
  }
  cudaError_t e = cudaMalloc(&d->d_orders, off);
  if (e == cudaSuccess) e = cudaMemcpy(d->d_orders, h.data(), off, cudaMemcpyHostToDevice);
  return e;
}

int check_inputs(bsidmap_decoder* d, int F, const void* rx, const void* off, const void* rho, const void* L,
                 const void* st) {
  if (!d) return fail(nullptr, BSIDMAP_EINVAL, "decoder is NULL");
  if (F < 0) return fail(d, BSIDMAP_EINVAL, "num_frames < 0");
  if (F > 0 && (!rx || !off || !rho || !L || !st))
    return fail(d, BSIDMAP_EINVAL, "rx_words, rx_word_offset, rho, L_out and frame_status must be non-NULL");
  return BSIDMAP_OK;
}

}  // namespace

extern "C" {

int bsidmap_create(bsidmap_decoder** out, int q, int n, int N, const uint32_t* codebook_host, double Pi, double Pd,
                   double Ps, int mn_lo, int mn_hi, int mt_lo, int mt_hi, int mode, int device) {
  if (!out) return fail(nullptr, BSIDMAP_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 1 || n > 32) return fail(nullptr, BSIDMAP_EINVAL, "need 1 <= n <= 32");
  if (q < 2 || (n < 32 && (uint64_t)q > (1ull << n))) return fail(nullptr, BSIDMAP_EINVAL, "need 2 <= q <= 2^n");
  if (N < 1) return fail(nullptr, BSIDMAP_EINVAL, "need N >= 1");
  if (!codebook_host) return fail(nullptr, BSIDMAP_EINVAL, "codebook is NULL");
  if (!(Pi >= 0 && Pd >= 0 && Ps >= 0 && Ps <= 1 && Pi + Pd < 1))
    return fail(nullptr, BSIDMAP_EINVAL, "need Pi, Pd, Ps >= 0, Ps <= 1, Pi + Pd < 1");
  if (!(mn_lo <= 0 && 0 <= mn_hi)) return fail(nullptr, BSIDMAP_EINVAL, "need m_n^- <= 0 <= m_n^+");
  if (!(mt_lo <= mn_lo && mt_hi >= mn_hi)) return fail(nullptr, BSIDMAP_EINVAL, "need m_tau^- <= m_n^-, m_tau^+ >= m_n^+");
  if (n + mn_hi > kMaxWindow) return fail(nullptr, BSIDMAP_EINVAL, "need n + m_n^+ <= 64");
  if (mode < 0 || mode > 3) return fail(nullptr, BSIDMAP_EINVAL, "unknown mode");
  const int Mn = mn_hi - mn_lo + 1;
  if (Mn > kMaxMn) return fail(nullptr, BSIDMAP_EPLAN, "corridor width M_n > 32 is not supported");
  if ((long)(mt_hi - mt_lo + 1) * (N + 1) > (1l << 40)) return fail(nullptr, BSIDMAP_EINVAL, "state space too large");
  const uint32_t mask = n == 32 ? 0xffffffffu : ((1u << n) - 1u);
  for (int i = 0; i < N; i++) {
    std::set<uint32_t> seen;
    for (int D = 0; D < q; D++) {
      const uint32_t w = codebook_host[(size_t)i * q + D];
      if (w & ~mask) return fail(nullptr, BSIDMAP_EINVAL, "codeword has bits above n");
      if (!seen.insert(w).second)
        return fail(nullptr, BSIDMAP_ENOTINJECTIVE, "C_" + std::to_string(i) + " is not injective");
    }
  }
  bsidmap_decoder* d = new bsidmap_decoder();
  d->device = device;
  d->q = q; d->n = n; d->N = N;
  d->mn_lo = mn_lo; d->mn_hi = mn_hi; d->Mn = Mn;
  d->mt_lo = mt_lo; d->mt_hi = mt_hi; d->Mt = mt_hi - mt_lo + 1;
  d->Pi = Pi; d->Pd = Pd; d->Ps = Ps;
  d->mode = mode;
  if (const char* v = std::getenv("BSIDMAP_AB_SUB")) d->ab_sub = std::max(1, std::atoi(v));
  if (const char* v = std::getenv("BSIDMAP_AB_CTA_STAGES")) d->ab_stages = std::max(0, std::atoi(v));
  if (const char* v = std::getenv("BSIDMAP_AB_CTA_THREADS")) d->ab_threads = std::max(0, std::atoi(v)) & ~31;
  if (const char* v = std::getenv("BSIDMAP_APP_KP")) d->app_kp = std::max(0, std::atoi(v));
  if (const char* v = std::getenv("BSIDMAP_APP_KS")) d->app_ks = std::atoi(v) == 2 ? 2 : 1;
  if (const char* v = std::getenv("BSIDMAP_LIVE_EPS")) d->live_eps = std::max(0.0, std::atof(v));
  if (const char* v = std::getenv("BSIDMAP_APP_G")) d->app_G = std::max(0, std::atoi(v));
  // lattice constants (eqn:F, Q-dot); row 0 = insertions only, F_{0,j} = 2^s (Pi/2)^j
  const double Pt = 1.0 - Pi - Pd;
  // G = F / Pd^r grows by at most Pd^-n over the lattice: keep 2^s Pd^-n q M_n below FLT_MAX / 2^10
  const double grow = Pd > 0 ? n * std::log2(1.0 / Pd) : 1e9;
  const bool rescaled = Pd > 0 && grow <= 90.0;
  int seed = kLatticeSeedMaxLog2;
  if (rescaled) seed = std::min(seed, (int)std::floor(118.0 - grow - std::log2((double)q) - std::log2((double)Mn)));
  d->lc.rescaled = rescaled ? 1 : 0;
  d->lc.seed_log2 = seed;
  d->lc.a = (float)(0.5 * Pi);
  d->lc.b = rescaled ? 1.0f : (float)Pd;
  d->lc.qm = (float)(Pt * (1.0 - Ps) / (rescaled ? Pd : 1.0));
  d->lc.qs = (float)(Pt * Ps / (rescaled ? Pd : 1.0));
  d->lc.out_scale = std::ldexp(rescaled ? std::pow(Pd, n) : 1.0, -seed);
  for (int e = 0; e < kMaxMn; e++) {
    const int j = mn_lo + e;
    d->lc.row0[e] = (e < Mn && j >= 0) ? (float)std::ldexp(std::pow(0.5 * Pi, j), seed) : 0.f;
  }
  // the spec cores' APP (k_app_live.cuh) stages per-symbol terms in shared memory: very large
  // alphabets use the generic core, whose APP pass stages symbols in chunks
  const bool unit = rescaled && find_spec_kernels(n, mn_lo, Mn, &d->kern);
  d->spec = unit && live_app_smem_fits(d->kern, q, Mn);
  if (rescaled && !unit) {  // no compiled unit for this shape: compile its unrolled core now
    const char* jv = std::getenv("BSIDMAP_JIT");
    if (jv && std::atoi(jv) == 0) {
      d->jit_err = "BSIDMAP_JIT=0";
    } else if (cudaSetDevice(device) == cudaSuccess && jit_spec_kernels(n, mn_lo, Mn, &d->kern, &d->jit_err, false)) {
      d->spec = d->jit = live_app_smem_fits(d->kern, q, Mn);
      if (!d->jit) d->jit_err = "alphabet too large for the live-window APP's shared memory";
    }
  }
  // RECOMPUTE runs the slab schedule on the spec cores (BSIDMAP_SLAB=0: the per-frame local kernels)
  d->slab_ok = d->spec;
  if (const char* v = std::getenv("BSIDMAP_SLAB")) d->slab_ok = d->slab_ok && std::atoi(v) != 0;
  if (const char* v = std::getenv("BSIDMAP_SLAB_LEN")) d->slab_fixed = std::max(0, std::atoi(v));
  if (const char* v = std::getenv("BSIDMAP_SLAB_ASKIP")) d->slab_askip = std::atoi(v) != 0;
  if (!d->spec && !find_generic_kernels(Mn, &d->kern)) {
    delete d;
    return fail(nullptr, BSIDMAP_EPLAN, "no lattice core for M_n = " + std::to_string(Mn));
  }
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&d->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaMalloc(&d->d_C, sizeof(uint32_t) * (size_t)N * q);
  if (e == cudaSuccess) e = cudaMemcpy(d->d_C, codebook_host, sizeof(uint32_t) * (size_t)N * q, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = upload_orders(d, codebook_host);
  for (int k = 0; e == cudaSuccess && k <= kPhases; k++) e = cudaEventCreate(&d->ev[k]);
  if (e != cudaSuccess) {
    std::string m = std::string("device setup: ") + cudaGetErrorString(e);
    bsidmap_destroy(d);
    return fail(nullptr, BSIDMAP_ECUDA, m);
  }
  *out = d;
  return BSIDMAP_OK;
}

int bsidmap_decode_batch(bsidmap_decoder* d, int F, const uint32_t* rx, const int64_t* off, const int32_t* rho,
                         const float* priors, float* L, int32_t* status, void* stream) {
  return bsidmap_decode_batch_opts(d, F, rx, off, rho, priors, nullptr, L, status, stream);
}

int bsidmap_decode_batch_opts(bsidmap_decoder* d, int F, const uint32_t* rx, const int64_t* off, const int32_t* rho,
                              const float* priors, const bsidmap_decode_opts* opts, float* L, int32_t* status,
                              void* stream) {
  int rc = check_inputs(d, F, rx, off, rho, L, status);
  if (rc) return rc;
  d->launches = 0;
  d->ev_valid = false;
  d->ab_overlapped = false;
  if (F == 0) return BSIDMAP_OK;
  cudaSetDevice(d->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Plan P;
  if ((rc = make_plan(d, F, &P))) return rc;
  const Layout l = layout(d, P.chunk, P.mode);
  if ((rc = ensure_ws(d, l.total))) return rc;
  if ((rc = set_smem(d, P.ab_warp ? (const void*)P.ab_warp : (const void*)P.ab_cta, P.ab_smem))) return rc;
  if ((rc = set_smem(d, (const void*)pass1_kernel(d, P, priors != nullptr), P.l1_smem))) return rc;
  if (P.mode == kSchedLocal) {
    if ((rc = set_smem(d, (const void*)d->kern.local_fwd, P.local_smem))) return rc;
    if ((rc = set_smem(d, (const void*)d->kern.local_bwd, P.local_smem))) return rc;
  } else if (P.mode == kSchedLocalCta) {
    for (int a = 0; a < 2; a++) {
      for (int b = 0; b < 2; b++)
        if ((rc = set_smem(d, (const void*)d->kern.local_cta_fwd[a][b], P.local_smem))) return rc;
      if ((rc = set_smem(d, (const void*)d->kern.local_cta_bwd[a], P.local_smem))) return rc;
    }
  } else if ((rc = set_smem(d, (const void*)P.app_kernel, P.app_smem))) {
    return rc;
  }
  for (int c = 0; c < P.nchunks; c++) {
    const int f0 = c * P.chunk;
    DecodeParams p;
    fill_params(d, &p);
    bind_ws(d, l, &p);
    p.F = std::min(P.chunk, F - f0);
    p.rx = rx;
    p.rx_off = off + f0;
    p.rho = rho + f0;
    p.priors = priors ? priors + (size_t)f0 * d->N * d->q : nullptr;
    p.alpha0 = (opts && opts->alpha0) ? opts->alpha0 + (size_t)f0 * d->Mt : nullptr;
    p.betaN = (opts && opts->betaN) ? opts->betaN + (size_t)f0 * d->Mt : nullptr;
    p.status = status + f0;
    p.L = L + (size_t)f0 * d->N * d->q;
    if ((rc = run_chunk(d, P, p, s, c == 0, c == P.nchunks - 1))) return rc;
    if (opts && opts->extrinsic) {  // NEXT-4: extrinsic APPs for an outer decoder
      const long rows = (long)p.F * d->N;
      k_extrinsic<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(p, opts->extrinsic + (size_t)f0 * d->N * d->q);
      d->launches++;
    }
  }
  d->last_chunk = P.chunk;
  d->last_frames = F;
  d->last_sched = P.mode;
  d->ev_stream = s;
  d->ev_valid = d->timing;
  return BSIDMAP_OK;
}

int bsidmap_decode_batch_host(bsidmap_decoder* d, int F, const uint32_t* rx, size_t rx_words_total,
                              const int64_t* off, const int32_t* rho, const float* priors, float* L, int32_t* status,
                              void* stream) {
  int rc = check_inputs(d, F, rx, off, rho, L, status);
  if (rc) return rc;
  if (F == 0) return BSIDMAP_OK;
  cudaSetDevice(d->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t nL = (size_t)F * d->N * d->q;
  const size_t b_rx = align_up(rx_words_total * 4), b_off = align_up((size_t)F * 8), b_rho = align_up((size_t)F * 4);
  const size_t b_pri = priors ? align_up(nL * 4) : 0, b_L = align_up(nL * 4), b_st = align_up((size_t)F * 4);
  const size_t need = b_rx + b_off + b_rho + b_pri + b_L + b_st;
  if (need > d->hs_bytes) {
    if (d->hs) {
      cudaStreamSynchronize(s);
      cudaFree(d->hs);
    }
    d->hs = nullptr;
    d->hs_bytes = 0;
    cudaError_t e = cudaMalloc(&d->hs, need);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(d, BSIDMAP_ENOMEM, "staging cudaMalloc failed");
    }
    d->hs_bytes = need;
  }
  char* b = static_cast<char*>(d->hs);
  uint32_t* d_rx = reinterpret_cast<uint32_t*>(b); b += b_rx;
  int64_t* d_off = reinterpret_cast<int64_t*>(b); b += b_off;
  int32_t* d_rho = reinterpret_cast<int32_t*>(b); b += b_rho;
  float* d_pri = priors ? reinterpret_cast<float*>(b) : nullptr; b += b_pri;
  float* d_L = reinterpret_cast<float*>(b); b += b_L;
  int32_t* d_st = reinterpret_cast<int32_t*>(b);
  // Pipeline: inputs go up on `s`; the batch is decoded in sub-batches on `s`, and each
  // sub-batch's APPs go back on a second stream while the next sub-batch computes, so the
  // large D2H of L (N q 4 bytes per frame) overlaps the decode instead of following it.
  if (!d->s_copy) {
    cudaError_t e = cudaStreamCreateWithFlags(&d->s_copy, cudaStreamNonBlocking);
    for (int k = 0; e == cudaSuccess && k < kHostSub; k++) e = cudaEventCreateWithFlags(&d->ev_sub[k], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(d, e, "copy stream");
  }
  cudaMemcpyAsync(d_rx, rx, rx_words_total * 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_off, off, (size_t)F * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_rho, rho, (size_t)F * 4, cudaMemcpyHostToDevice, s);
  if (priors) cudaMemcpyAsync(d_pri, priors, nL * 4, cudaMemcpyHostToDevice, s);
  // sub-batches: up to 8 equal ones; the last of them split in halves down to 1/8 (4/2/1/1 eighths),
  // so the D2H left after the last decode is small (C2: 6.5 MB instead of 52 MB)
  const int neq = std::max(1, std::min(8, F / 8192));
  std::vector<int> cut;
  for (int k = 0; k < neq; k++) cut.push_back((int)((long)F * k / neq));
  if (neq >= 2) {
    const int last = cut.back(), len = F - last;
    for (int part : {4, 6, 7}) cut.push_back(last + (int)((long)len * part / 8));
  }
  cut.push_back(F);
  const int nsub = (int)cut.size() - 1;
  const size_t row = (size_t)d->N * d->q;
  long launches = 0;
  for (int k = 0; k < nsub; k++) {
    const int f0 = cut[k], f1 = cut[k + 1];
    if ((rc = bsidmap_decode_batch(d, f1 - f0, d_rx, d_off + f0, d_rho + f0, d_pri ? d_pri + f0 * row : nullptr,
                                   d_L + f0 * row, d_st + f0, stream)))
      return rc;
    launches += d->launches;
    cudaEventRecord(d->ev_sub[k], s);
    cudaStreamWaitEvent(d->s_copy, d->ev_sub[k], 0);
    cudaMemcpyAsync(L + f0 * row, d_L + f0 * row, (size_t)(f1 - f0) * row * 4, cudaMemcpyDeviceToHost, d->s_copy);
    cudaMemcpyAsync(status + f0, d_st + f0, (size_t)(f1 - f0) * 4, cudaMemcpyDeviceToHost, d->s_copy);
  }
  d->launches = launches;
  cudaError_t e = cudaStreamSynchronize(d->s_copy);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(d, e, "decode_batch_host");
  return BSIDMAP_OK;
}

void bsidmap_destroy(bsidmap_decoder* d) {
  if (!d) return;
  cudaSetDevice(d->device);
  cudaDeviceSynchronize();
  if (d->ws) cudaFree(d->ws);
  if (d->hs) cudaFree(d->hs);
  if (d->s_copy) cudaStreamDestroy(d->s_copy);
  if (d->s_ab) cudaStreamDestroy(d->s_ab);
  for (int k = 0; k < kMaxAbSub; k++) {
    if (d->ev_p1[k]) cudaEventDestroy(d->ev_p1[k]);
    if (d->ev_ab[k]) cudaEventDestroy(d->ev_ab[k]);
  }
  for (int k = 0; k < 2; k++)
    if (d->ev_abt[k]) cudaEventDestroy(d->ev_abt[k]);
  for (int k = 0; k < kHostSub; k++)
    if (d->ev_sub[k]) cudaEventDestroy(d->ev_sub[k]);
  if (d->d_C) cudaFree(d->d_C);
  if (d->d_orders) cudaFree(d->d_orders);
  for (int k = 0; k <= kPhases; k++)
    if (d->ev[k]) cudaEventDestroy(d->ev[k]);
  delete d;
}

const char* bsidmap_last_error(const bsidmap_decoder* d) { return d ? d->err.c_str() : g_err.c_str(); }

size_t bsidmap_workspace_bytes(const bsidmap_decoder* d, int F, int mode) {
  if (!d || F < 0) return 0;
  if (mode < 0 || mode > 3) return 0;
  return layout(d, F, resolve_sched(d, mode)).total;
}

int bsidmap_set_workspace_limit(bsidmap_decoder* d, size_t bytes) {
  if (!d) return fail(nullptr, BSIDMAP_EINVAL, "decoder is NULL");
  d->ws_limit = bytes;
  return BSIDMAP_OK;
}

int bsidmap_set_mode(bsidmap_decoder* d, int mode) {
  if (!d) return fail(nullptr, BSIDMAP_EINVAL, "decoder is NULL");
  if (mode < 0 || mode > 3) return fail(d, BSIDMAP_EINVAL, "unknown mode");
  d->mode = mode;
  return BSIDMAP_OK;
}

int bsidmap_set_timing(bsidmap_decoder* d, int enable) {
  if (!d) return fail(nullptr, BSIDMAP_EINVAL, "decoder is NULL");
  d->timing = enable != 0;
  return BSIDMAP_OK;
}

int bsidmap_phase_times(bsidmap_decoder* d, float* ms, int n_max) {
  if (!d || !ms) return fail(d, BSIDMAP_EINVAL, "bad arguments");
  if (!d->ev_valid) return fail(d, BSIDMAP_EINVAL, "no timed decode (enable bsidmap_set_timing first)");
  cudaError_t e = cudaEventSynchronize(d->ev[kPhases]);
  if (e != cudaSuccess) return cuda_fail(d, e, "cudaEventSynchronize");
  int k = 0;
  for (; k < kPhases && k < n_max; k++) {
    // phases 0-3 are the first chunk; the last phase runs to the end of the last chunk
    cudaEventElapsedTime(&ms[k], d->ev[k], d->ev[k + 1]);
  }
  if (k < n_max) {  // [5]: alpha/beta busy time (on the side stream when overlapped)
    if (d->ab_overlapped)
      cudaEventElapsedTime(&ms[k], d->ev_abt[0], d->ev_abt[1]);
    else
      ms[k] = ms[2];
    k++;
  }
  return k;
}

long bsidmap_last_launch_count(const bsidmap_decoder* d) { return d ? d->launches : 0; }

namespace {
// A message as the body of a JSON string: quotes and backslashes dropped, control characters as
// spaces, at most max_len characters.
std::string json_text(const std::string& m, size_t max_len) {
  std::string o;
  for (char c : m) {
    if (o.size() >= max_len) break;
    if (c == '"' || c == '\\') continue;
    o += (static_cast<unsigned char>(c) < 0x20) ? ' ' : c;
  }
  return o;
}
}  // namespace

int bsidmap_plan_info(bsidmap_decoder* d, int F, char* buf, size_t len) {
  if (!d || !buf || F < 1) return fail(d, BSIDMAP_EINVAL, "bad arguments");
  Plan P;
  int rc = make_plan(d, F, &P);
  if (rc) return rc;
  const long lanes = (long)P.chunk * d->Mt;
  int nb = std::snprintf(
      buf, len,
      "{\"mode\": \"%s\", \"frames\": %d, \"chunk\": %d, \"chunks\": %d, \"core\": \"%s\", "
      "\"lattice_grid\": [%ld, %d], \"lattice_block\": %d, \"alpha_beta_grid\": [%d, 2], \"alpha_beta_block\": %d, "
      "\"workspace_bytes\": %zu, \"windows_per_lane\": %d, \"q\": %d, \"n\": %d, \"N\": %d, \"Mn\": %d, \"Mtau\": %d, "
      "\"alpha_beta_overlap_subbatches\": %d, \"app_prefix_bits\": %d, \"app_windows_per_lane\": %d, "
      "\"app_folded_rows\": %d, \"app_live\": %d, \"app_frames_per_warp\": %d, \"live_eps\": %.6g, "
      "\"slab\": %d, \"jit_error\": \"%s\"}",
      sched_name(P.mode), F, P.chunk, P.nchunks, d->jit ? "jit" : d->spec ? "spec" : "generic",
      d->kern.W == 2 ? ((long)P.chunk * tiles_per_frame(d->Mt) + kX2Warps - 1) / kX2Warps
                     : (lanes + kLatticeThreads - 1) / kLatticeThreads,
      d->N, kLatticeThreads, P.chunk, P.ab_warp ? kAbWarpThreads : P.ab_threads,
      layout(d, P.chunk, P.mode).total, d->kern.W, d->q, d->n, d->N, d->Mn, d->Mt, std::min(P.ab_sub, P.chunk), P.app_kp, P.app_live ? d->kern.app_live_W : 1, P.app_ks,
      P.app_live ? 1 : 0, P.app_G, d->live_eps, P.slab, json_text(d->jit_err, 300).c_str());
  return nb;
}

int bsidmap_jit_compile(int n, int mn_lo, int Mn, char* err, size_t len) {
  std::string e;
  CoreKernels k{};
  const bool ok = jit_spec_kernels(n, mn_lo, Mn, &k, &e, true);
  if (err && len) std::snprintf(err, len, "%s", e.c_str());
  return ok ? BSIDMAP_OK : fail(nullptr, BSIDMAP_EPLAN, e);
}

long bsidmap_lattice_nodes(const bsidmap_decoder* d) {
  if (!d) return 0;
  return (long)d->n * d->Mn - (long)d->mn_lo * (d->mn_lo - 1) / 2;
}

long long bsidmap_valid_lattices(const bsidmap_decoder* d, int F, const int32_t* rho) {
  if (!d || !rho) return 0;
  long long tot = 0;
  for (int f = 0; f < F; f++) {
    const int drift = rho[f] - d->n * d->N;
    if (drift < d->mt_lo || drift > d->mt_hi) continue;
    for (int i = 0; i < d->N; i++) {
      // m' in [mt_lo, mt_hi] with 0 <= n i + m' <= rho
      const int lo = std::max(d->mt_lo, -d->n * i), hi = std::min(d->mt_hi, rho[f] - d->n * i);
      if (hi >= lo) tot += hi - lo + 1;
    }
  }
  return tot * d->q;
}

int bsidmap_debug_gamma(bsidmap_decoder* d, int F, const uint32_t* rx, const int64_t* off, const int32_t* rho,
                        const float* priors, int i, double* gamma_out, void* stream) {
  if (!d || F < 1 || !rx || !off || !rho || !gamma_out || i < 0 || i >= d->N)
    return fail(d, BSIDMAP_EINVAL, "bad arguments");
  cudaSetDevice(d->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* st = nullptr;
  cudaError_t e = cudaMalloc(&st, sizeof(int32_t) * F);
  if (e != cudaSuccess) return cuda_fail(d, e, "cudaMalloc");
  DecodeParams p;
  fill_params(d, &p);
  p.F = F; p.rx = rx; p.rx_off = off; p.rho = rho; p.priors = priors; p.status = st;
  p.dbg_gamma = gamma_out; p.dbg_i = i;
  k_frame_init<<<(F + 255) / 256, 256, 0, s>>>(p);
  const unsigned gx = d->kern.W == 2 ? (unsigned)(((long)F * tiles_per_frame(d->Mt) + kX2Warps - 1) / kX2Warps)
                                     : (unsigned)(((long)F * d->Mt + kLatticeThreads - 1) / kLatticeThreads);
  launch_k(d->kern.gamma_dump, gx, kLatticeThreads, (size_t)d->q * 4, s, p);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(st);
  if (e != cudaSuccess) return cuda_fail(d, e, "debug_gamma");
  return BSIDMAP_OK;
}

int bsidmap_debug_states(bsidmap_decoder* d, int F, double* alpha_out, double* beta_out, void* stream) {
  if (!d || !alpha_out || !beta_out) return fail(d, BSIDMAP_EINVAL, "bad arguments");
  if (F != d->last_frames || d->last_chunk < F || !d->ws)
    return fail(d, BSIDMAP_EINVAL, "last decode was chunked or of a different size");
  cudaSetDevice(d->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (d->last_sched == kSchedLocal || d->last_sched == kSchedLocalCta)
    return fail(d, BSIDMAP_EINVAL, "the local schedule keeps no beta rows");
  if (d->last_sched == kSchedSlab && slab_beta_rows(d, slab_len(d, d->last_chunk)) != d->N + 1)
    return fail(d, BSIDMAP_EINVAL, "the slab schedule keeps beta rows for three slabs only");
  const Layout l = layout(d, d->last_chunk, d->last_sched);
  DecodeParams p;
  bind_ws(d, l, &p);
  const size_t bytes = (size_t)F * (d->N + 1) * d->Mt * sizeof(double);
  cudaMemcpyAsync(alpha_out, p.alpha, bytes, cudaMemcpyDeviceToDevice, s);
  cudaMemcpyAsync(beta_out, p.beta, bytes, cudaMemcpyDeviceToDevice, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(d, e, "debug_states");
  return BSIDMAP_OK;
}

int bsidmap_mc_generate(bsidmap_decoder* d, uint64_t seed, int64_t first_frame, int F, int wpf, int32_t* msg,
                        uint32_t* rx, int32_t* rho, unsigned long long* redraws, void* stream) {
  if (!d || F < 1 || !msg || !rx || !rho || !redraws || (long)wpf * 32 < (long)d->n * d->N + d->mt_hi)
    return fail(d, BSIDMAP_EINVAL, "bad arguments");
  cudaSetDevice(d->device);
  McParams P;
  P.seed = seed; P.first = first_frame; P.F = F; P.N = d->N; P.q = d->q; P.n = d->n; P.wpf = wpf;
  P.mt_lo = d->mt_lo; P.mt_hi = d->mt_hi; P.Pi = d->Pi; P.Pd = d->Pd; P.Ps = d->Ps;
  P.C = d->d_C; P.msg = msg; P.rx = rx; P.rho = rho; P.redraws = redraws;
  k_mc_generate<<<(F + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(P);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BSIDMAP_OK : cuda_fail(d, e, "mc_generate");
}

int bsidmap_count_errors(bsidmap_decoder* d, int F, const float* L, const int32_t* msg, const int32_t* status,
                         unsigned long long* counters, void* stream) {
  if (!d || F < 1 || !L || !msg || !status || !counters) return fail(d, BSIDMAP_EINVAL, "bad arguments");
  cudaSetDevice(d->device);
  k_mc_count<<<F, 128, 0, static_cast<cudaStream_t>(stream)>>>(L, msg, status, F, d->N, d->q, counters);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BSIDMAP_OK : cuda_fail(d, e, "count_errors");
}

int bsidmap_mc_run(bsidmap_decoder* d, uint64_t seed, int64_t first_frame, int num_frames, int batch,
                   unsigned long long* results, void* stream) {
  if (!d || num_frames < 1 || batch < 1 || !results) return fail(d, BSIDMAP_EINVAL, "bad arguments");
  cudaSetDevice(d->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  batch = std::min(batch, num_frames);
  const int wpf = (d->n * d->N + d->mt_hi + 31) / 32 + 1;  // as the host generator (bsidgen)
  const size_t nL = (size_t)batch * d->N * d->q;
  char* buf = nullptr;
  const size_t b_msg = align_up((size_t)batch * d->N * 4), b_rx = align_up((size_t)batch * wpf * 4),
               b_rho = align_up((size_t)batch * 4), b_off = align_up((size_t)batch * 8), b_L = align_up(nL * 4),
               b_st = align_up((size_t)batch * 4), b_cnt = 256;
  cudaError_t e = cudaMallocAsync(&buf, b_msg + b_rx + b_rho + b_off + b_L + b_st + b_cnt, s);
  if (e != cudaSuccess) return cuda_fail(d, e, "mc_run alloc");
  int32_t* msg = reinterpret_cast<int32_t*>(buf);
  uint32_t* rx = reinterpret_cast<uint32_t*>(buf + b_msg);
  int32_t* rho = reinterpret_cast<int32_t*>(buf + b_msg + b_rx);
  int64_t* off = reinterpret_cast<int64_t*>(buf + b_msg + b_rx + b_rho);
  float* L = reinterpret_cast<float*>(buf + b_msg + b_rx + b_rho + b_off);
  int32_t* st = reinterpret_cast<int32_t*>(buf + b_msg + b_rx + b_rho + b_off + b_L);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(buf + b_msg + b_rx + b_rho + b_off + b_L + b_st);
  cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), s);
  int rc = BSIDMAP_OK;
  long launches = 0;
  for (int f0 = 0; f0 < num_frames && rc == BSIDMAP_OK; f0 += batch) {
    const int F = std::min(batch, num_frames - f0);
    k_iota_offsets<<<(F + 255) / 256, 256, 0, s>>>(off, F, wpf);
    if ((rc = bsidmap_mc_generate(d, seed, first_frame + f0, F, wpf, msg, rx, rho, cnt + 3, stream))) break;
    if ((rc = bsidmap_decode_batch(d, F, rx, off, rho, nullptr, L, st, stream))) break;
    launches += d->launches + 3;
    if ((rc = bsidmap_count_errors(d, F, L, msg, st, cnt, stream))) break;
  }
  unsigned long long h[4] = {0, 0, 0, 0};
  if (rc == BSIDMAP_OK) {
    cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(d, e, "mc_run");
  }
  cudaFreeAsync(buf, s);
  d->launches = launches;
  results[0] = (unsigned long long)num_frames;
  results[1] = h[0];
  results[2] = h[1];
  results[3] = h[3];
  return rc;
}

}  // extern "C"
