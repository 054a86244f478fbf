// jit.cu -- run-time compiled lattice cores for shapes without a compiled unit.
//
// The paper builds its decoder from templates over the code and channel sizes, split over
// compilation units, so only the sizes compiled in are fast; any other shape here
// used to fall back to the generic core (runtime n, m_n^-; M_n-only template).  bsidmap_create
// now compiles the fully unrolled cores for ANY (n, m_n^-, M_n <= 32) with NVRTC: the same kernel
// templates as the inst_spec_*.cu units (sources embedded in the library at build time), compiled
// for sm_100a in five programs on five host threads, cached on disk (cubin + lowered names) so a
// shape is compiled once per machine.  The kernels come back as cudaKernel_t handles, which the
// runtime launches and configures in place of __global__ function addresses (api.cu launch_k).
//   BSIDMAP_JIT=0          off (the generic core serves every shape without a unit)
//   BSIDMAP_JIT_CACHE=dir  cache directory (default $XDG_CACHE_HOME/bsidmap or ~/.cache/bsidmap)
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "k_lattice_x2.cuh"

namespace {

struct HeaderSrc {
  const char* name;
  const char* src;
};
const HeaderSrc kHeaders[] = {
#include "jit_sources.inc"
};
constexpr int kNumHeaders = sizeof(kHeaders) / sizeof(kHeaders[0]);
constexpr const char* kJitVersion = "bsidmap-jit-1";
// fully unrolled cores up to this many corridor nodes per lattice (C4's 2.6x: longer codes with wide
// corridors unroll into kernels too large to compile quickly and register-bound anyway)
constexpr long kJitMaxNodes = 320;

uint64_t fnv1a(uint64_t h, const void* data, size_t n) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < n; i++) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

std::string cache_dir() {
  if (const char* v = std::getenv("BSIDMAP_JIT_CACHE")) return v;
  if (const char* v = std::getenv("XDG_CACHE_HOME")) return std::string(v) + "/bsidmap";
  if (const char* v = std::getenv("HOME")) return std::string(v) + "/.cache/bsidmap";
  return "/tmp/bsidmap-jit";
}

void mkdirs(const std::string& path) {
  for (size_t i = 1; i <= path.size(); i++)
    if (i == path.size() || path[i] == '/') mkdir(path.substr(0, i).c_str(), 0755);
}

// One NVRTC program: the kernel name expressions, the cubin and their lowered names.
struct Unit {
  std::vector<std::string> exprs;
  std::vector<std::string> lowered;
  std::string cubin;
  std::string err;
};

const char* kOpts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-default-device", "-DBSIDMAP_JIT=1"};
constexpr int kNumOpts = sizeof(kOpts) / sizeof(kOpts[0]);

uint64_t unit_key(const Unit& u) {
  uint64_t h = 1469598103934665603ull;
  h = fnv1a(h, kJitVersion, std::strlen(kJitVersion));
  for (int i = 0; i < kNumHeaders; i++) {
    h = fnv1a(h, kHeaders[i].name, std::strlen(kHeaders[i].name));
    h = fnv1a(h, kHeaders[i].src, std::strlen(kHeaders[i].src));
  }
  for (int i = 0; i < kNumOpts; i++) h = fnv1a(h, kOpts[i], std::strlen(kOpts[i]));
  for (auto& e : u.exprs) h = fnv1a(h, e.c_str(), e.size() + 1);
  return h;
}

// cache file: "BSIDMAPJ" | u32 count | count lowered names ('\0'-terminated) | u64 size | cubin
bool cache_load(const std::string& path, Unit& u) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  char magic[8];
  uint32_t cnt = 0;
  if (!f.read(magic, 8) || std::memcmp(magic, "BSIDMAPJ", 8) != 0 || !f.read(reinterpret_cast<char*>(&cnt), 4) ||
      cnt != u.exprs.size())
    return false;
  u.lowered.clear();
  for (uint32_t i = 0; i < cnt; i++) {
    std::string s;
    if (!std::getline(f, s, '\0')) return false;
    u.lowered.push_back(s);
  }
  uint64_t n = 0;
  if (!f.read(reinterpret_cast<char*>(&n), 8) || n == 0 || n > (1ull << 31)) return false;
  u.cubin.resize(n);
  return static_cast<bool>(f.read(&u.cubin[0], (std::streamsize)n));
}

void cache_store(const std::string& path, const Unit& u) {
  const std::string tmp = path + ".tmp." + std::to_string(getpid());
  {
    std::ofstream f(tmp, std::ios::binary);
    if (!f) return;
    const uint32_t cnt = (uint32_t)u.lowered.size();
    const uint64_t n = u.cubin.size();
    f.write("BSIDMAPJ", 8);
    f.write(reinterpret_cast<const char*>(&cnt), 4);
    for (auto& s : u.lowered) f.write(s.c_str(), (std::streamsize)s.size() + 1);
    f.write(reinterpret_cast<const char*>(&n), 8);
    f.write(u.cubin.data(), (std::streamsize)n);
    if (!f) return;
  }
  std::rename(tmp.c_str(), path.c_str());
}

void compile(Unit& u) {
  std::string src = "#include \"k_local_x2.cuh\"\n#include \"k_local_cta.cuh\"\n#include \"k_alphabeta_cta.cuh\"\n";
  std::vector<const char*> hs, hn;
  for (int i = 0; i < kNumHeaders; i++) {
    hs.push_back(kHeaders[i].src);
    hn.push_back(kHeaders[i].name);
  }
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), "bsidmap_jit.cu", kNumHeaders, hs.data(), hn.data());
  if (r != NVRTC_SUCCESS) {
    u.err = nvrtcGetErrorString(r);
    return;
  }
  for (auto& e : u.exprs) nvrtcAddNameExpression(prog, e.c_str());
  r = nvrtcCompileProgram(prog, kNumOpts, kOpts);
  if (r != NVRTC_SUCCESS) {
    size_t ls = 0;
    nvrtcGetProgramLogSize(prog, &ls);
    std::string log(ls, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    u.err = std::string(nvrtcGetErrorString(r)) + ": " + log.substr(0, 2000);
    nvrtcDestroyProgram(&prog);
    return;
  }
  size_t cs = 0;
  nvrtcGetCUBINSize(prog, &cs);
  u.cubin.resize(cs);
  nvrtcGetCUBIN(prog, &u.cubin[0]);
  u.lowered.clear();
  for (auto& e : u.exprs) {
    const char* ln = nullptr;
    nvrtcGetLoweredName(prog, e.c_str(), &ln);
    u.lowered.push_back(ln ? ln : "");
  }
  nvrtcDestroyProgram(&prog);
}

template <class Fn>
Fn as_fn(cudaKernel_t k) {
  return reinterpret_cast<Fn>(reinterpret_cast<void*>(k));
}

}  // namespace

namespace bsidmap {

// Kernel tables already loaded in this process, by shape: a shape is compiled (or read from the
// disk cache) and loaded once, whatever the number of decoders.
std::mutex g_jit_mu;
std::map<std::string, CoreKernels> g_jit_loaded;

// The kernel table of spec_kernels<n, m_n^-, M_n> (inst.cuh), compiled at run time.  Uses a host
// copy of the register estimate of SpecCoreX2 (lattice_x2.cuh kMinBlocks) and of the scalar-APP
// rule of inst.cuh (BSIDMAP_SCALAR_MN_MAX).  compile_only: NVRTC (and the disk cache) only, no
// device needed.

bool jit_spec_kernels(int n, int lo, int Mn, CoreKernels* out, std::string* err, bool compile_only) {
  const std::string shape_key = std::to_string(n) + "," + std::to_string(lo) + "," + std::to_string(Mn);
  std::lock_guard<std::mutex> lock(g_jit_mu);
  if (!compile_only) {
    auto it = g_jit_loaded.find(shape_key);
    if (it != g_jit_loaded.end()) {
      *out = it->second;
      return true;
    }
  }
  const int J = n + lo + Mn - 1;
  const long nodes = (long)n * Mn - (long)lo * (lo - 1) / 2;
  if (!(Mn >= 1 && Mn <= kMaxMn && lo <= 0 && lo + Mn - 1 >= 0 && J <= kMaxWindow && n >= 3 && nodes <= kJitMaxNodes)) {
    *err = "shape outside the unrolled cores (need M_n <= 32, n + m_n^+ <= 64, n >= 3, <= " +
           std::to_string(kJitMaxNodes) + " corridor nodes)";
    return false;
  }
  const bool minb3 = 4 * J + 4 * Mn + 30 <= 168;
  const bool scalar_app = !minb3 && Mn <= 20;
  const std::string sh = std::to_string(n) + ", " + std::to_string(lo) + ", " + std::to_string(Mn) + ">";
  const std::string px = "bsidmap::SpecCoreX2<" + sh, sc = "bsidmap::SpecCore<" + sh, m = std::to_string(Mn);
  // the pair APP runs the core on 64-bit pairs (lattice_x2.cuh)
  const std::string pxa = "bsidmap::SpecCoreX2<" + std::to_string(n) + ", " + std::to_string(lo) + ", " +
                          std::to_string(Mn) + ", unsigned long long>";
  // slots, in the order of the units below
  std::vector<Unit> units(5);
  auto add = [&](int g, const std::string& e) { units[g].exprs.push_back(e); };
  for (int K = 2; K <= 3; K++)
    for (int pri = 0; pri < 2; pri++)
      add(0, "bsidmap::k_gamma_sum_x2_cls<" + px + ", " + std::to_string(K) + ", " + (pri ? "true" : "false") + ">");
  add(0, "bsidmap::k_gamma_sum_x2<" + px + ", true>");
  add(0, "bsidmap::k_gamma_dump_x2<" + px + ">");
  // prefix lengths KP = 0, 2, 3, 4 (a KP the shape cannot use, KP > n - 2, is never planned:
  // its slot holds the KP = 0 kernel)
  const int kps[4] = {0, 2, 3, 4};
  for (int ks = 1; ks <= 2; ks++)
    for (int k = 0; k < 4; k++)
      add(ks, std::string(scalar_app ? "bsidmap::k_app_live_x1<" + sc : "bsidmap::k_app_live_x2<" + pxa) + ", " +
                  std::to_string(kps[k] <= n - 2 ? kps[k] : 0) + ", " + std::to_string(ks) + ">");
  for (int spt : {1, 2, 4}) add(3, "bsidmap::k_alpha_beta_warp<" + std::to_string(spt) + ", " + m + ">");
  add(3, "bsidmap::k_alpha_beta_cta<" + m + ">");
  add(3, "bsidmap::k_app_stored<" + m + ">");
  add(3, "bsidmap::k_local_fwd<" + px + ">");
  add(3, "bsidmap::k_local_bwd<" + px + ">");
  for (int K = 2; K <= 3; K++)
    for (int pri = 0; pri < 2; pri++)
      add(4, "bsidmap::k_local_cta_fwd<" + sc + ", " + std::to_string(K) + ", " + (pri ? "true" : "false") + ">");
  add(4, "bsidmap::k_local_cta_bwd<" + sc + ", false>");
  add(4, "bsidmap::k_local_cta_bwd<" + sc + ", true>");

  const std::string dir = cache_dir();
  mkdirs(dir);
  std::vector<std::thread> th;
  std::vector<std::string> paths(units.size());
  for (size_t g = 0; g < units.size(); g++) {
    char name[64];
    std::snprintf(name, sizeof(name), "/bsidmap_%016llx.bin", (unsigned long long)unit_key(units[g]));
    paths[g] = dir + name;
    if (cache_load(paths[g], units[g])) continue;
    th.emplace_back([&units, &paths, g] {
      compile(units[g]);
      if (units[g].err.empty()) cache_store(paths[g], units[g]);
    });
  }
  for (auto& t : th) t.join();
  for (auto& u : units)
    if (!u.err.empty()) {
      *err = "NVRTC: " + u.err;
      return false;
    }
  if (compile_only) return true;

  std::vector<cudaKernel_t> ks;
  std::vector<cudaLibrary_t> libs;
  for (auto& u : units) {
    cudaLibrary_t lib = nullptr;
    cudaError_t e = cudaLibraryLoadData(&lib, u.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess) {
      *err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
      cudaGetLastError();
      for (auto l : libs) cudaLibraryUnload(l);
      return false;
    }
    libs.push_back(lib);
    for (auto& ln : u.lowered) {
      cudaKernel_t k = nullptr;
      e = cudaLibraryGetKernel(&k, lib, ln.c_str());
      if (e != cudaSuccess) {
        *err = "cudaLibraryGetKernel(" + ln + "): " + cudaGetErrorString(e);
        cudaGetLastError();
        for (auto l : libs) cudaLibraryUnload(l);
        return false;
      }
      ks.push_back(k);
    }
  }
  using F1 = void (*)(const DecodeParams);
  using F2 = void (*)(const DecodeParams, int);
  CoreKernels k{};
  size_t i = 0;
  k.gamma_sum = as_fn<F1>(ks[i++]);
  k.gamma_sum_pri = as_fn<F1>(ks[i++]);
  k.gamma_sum_k3 = as_fn<F1>(ks[i++]);
  k.gamma_sum_k3_pri = as_fn<F1>(ks[i++]);
  k.gamma_store = as_fn<F1>(ks[i++]);
  k.gamma_dump = as_fn<F1>(ks[i++]);
  for (int a = 0; a < 2; a++)
    for (int b = 0; b < 4; b++) k.app_live[a][b] = as_fn<F1>(ks[i++]);
  for (int a = 0; a < 3; a++) k.ab_warp[a] = as_fn<F1>(ks[i++]);
  k.ab_cta = as_fn<F2>(ks[i++]);
  k.app_stored = as_fn<F1>(ks[i++]);
  k.local_fwd = as_fn<F1>(ks[i++]);
  k.local_bwd = as_fn<F1>(ks[i++]);
  for (int a = 0; a < 2; a++)
    for (int b = 0; b < 2; b++) k.local_cta_fwd[a][b] = as_fn<F1>(ks[i++]);
  k.local_cta_bwd[0] = as_fn<F1>(ks[i++]);
  k.local_cta_bwd[1] = as_fn<F1>(ks[i++]);
  k.app = nullptr;
  k.app_ks_auto = scalar_app ? 2 : 1;  // as spec_kernels<> (inst.cuh) and make_core_kernels_x2_base
  k.app_live_W = scalar_app ? 1 : 2;
  k.nodes = (long)n * Mn - (long)lo * (lo - 1) / 2;
  // pass-1 head tables (k_lattice_x2.cuh l1_head_rows), at the class kernel's CTAs per SM (BSIDMAP_L1C_MINB)
  const int l1_minb = minb3 ? 4 : (Mn <= 20 ? 3 : 2);
  for (int K = 2; K <= 3; K++) k.l1_head_bytes[K - 2] = l1_head_bytes(l1_head_rows(n, lo, Mn, K, l1_minb), lo, Mn);
  k.W = 2;
  k.l1_W = 2;
  k.l1_steps = true;
  *out = k;
  g_jit_loaded[shape_key] = k;  // the libraries stay loaded for the process (driver frees them at exit)
  return true;
}

}  // namespace bsidmap
