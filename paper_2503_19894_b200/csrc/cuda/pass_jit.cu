// JIT-compiled tile passes (NVRTC): the paper's code-generation idea
// (CAST emits a kernel per fused gate through LLVM) applied
// to the B200 tile pass.  The generic k_pass interprets its op table at run
// time: every op of every tile reloads its fields from shared memory and
// branches on its kind.  A JIT pass is the same kernel (k_pass_body) with
// the op table as a constexpr array and the op sequence unrolled into
// straight-line pass_step calls with literal op indices, so every field,
// table offset, loop bound and dispatch folds to a constant; the data the
// ops read (matrices, per-thread tables) still comes from the staged blob.
// Results are bit-identical to the interpreter (same device functions, same
// arithmetic order).
//
// Compiled once per distinct op table (source hash), cached in-process and
// on disk (TSG_JIT_CACHE_DIR, default jit_cache/ beside the library), loaded as a CUDA
// library (cudaLibraryLoadData).  TSG_PASS_JIT=0 disables; passes on states
// below TSG_PASS_JIT_MIN_N qubits (default 24) use the interpreter (a
// compile costs seconds, a small pass microseconds).
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvrtc.h>

#include "gate_launch.hpp"
#include "pass_jit.hpp"
#include "tilesim/pass.hpp"

#include "jit_headers.inc"

namespace tsg {

namespace {

// NVRTC has no C++ standard library: the integer types and the one trait the
// headers use, ahead of them (the headers skip their std includes under
// __CUDACC_RTC__).
const char* const kPreamble = R"tsgjit(
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef signed char int8_t;
typedef short int16_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned long size_t;
namespace std {
template <bool B, class T, class F> struct conditional { using type = T; };
template <class T, class F> struct conditional<false, T, F> { using type = F; };
template <bool B, class T, class F> using conditional_t = typename conditional<B, T, F>::type;
}
struct CUstream_st;
typedef CUstream_st* cudaStream_t;
#define TSG_JIT 1
)tsgjit";

struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  std::string error;
};

// NVRTC is loaded on first use, so the library itself loads without it
const Nvrtc& nvrtc() {
  static Nvrtc api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.error = std::string("cannot load libnvrtc.so.12: ") + dlerror();
      return;
    }
    api.create = reinterpret_cast<decltype(api.create)>(dlsym(h, "nvrtcCreateProgram"));
    api.compile = reinterpret_cast<decltype(api.compile)>(dlsym(h, "nvrtcCompileProgram"));
    api.log_size = reinterpret_cast<decltype(api.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
    api.log = reinterpret_cast<decltype(api.log)>(dlsym(h, "nvrtcGetProgramLog"));
    api.cubin_size = reinterpret_cast<decltype(api.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
    api.cubin = reinterpret_cast<decltype(api.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
    if (!api.create || !api.compile || !api.cubin || !api.destroy) api.error = "libnvrtc.so.12 lacks the program API";
  });
  return api;
}

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ULL) {
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ULL;
  return h;
}

std::string hex16(uint64_t v) {
  char b[17];
  std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(v));
  return b;
}

// TSG_JIT_CACHE_DIR, else jit_cache/ next to this library (in-tree: a cache
// warmed by build() travels with the repository), else /tmp/tsg_jit
std::string cache_dir() {
  const char* d = std::getenv("TSG_JIT_CACHE_DIR");
  if (d && *d) return d;
  static const std::string dir = [] {
    Dl_info info;
    if (dladdr(reinterpret_cast<void*>(&pass_jit_enabled), &info) && info.dli_fname) {
      std::string so = info.dli_fname;
      const size_t slash = so.rfind('/');
      const std::string here = slash == std::string::npos ? "." : so.substr(0, slash);
      const std::string cand = here + "/jit_cache";
      mkdir(cand.c_str(), 0777);
      if (access(cand.c_str(), W_OK) == 0) return cand;
    }
    return std::string("/tmp/tsg_jit");
  }();
  return dir;
}

std::vector<char> compile_cubin(const std::string& src, const std::string& name) {
  const Nvrtc& api = nvrtc();
  if (!api.error.empty()) throw std::runtime_error(api.error);
  nvrtcProgram prog = nullptr;
  if (api.create(&prog, src.c_str(), (name + ".cu").c_str(), kJitHeaderCount, kJitHeaderTexts, kJitHeaderNames) !=
      NVRTC_SUCCESS)
    throw std::runtime_error("nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                        "--fmad=true", "-default-device"};
  const nvrtcResult rc = api.compile(prog, static_cast<int>(sizeof opts / sizeof opts[0]), opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    api.log_size(prog, &n);
    std::string log(n, '\0');
    api.log(prog, log.data());
    api.destroy(&prog);
    throw std::runtime_error("NVRTC compile of " + name + " failed:\n" + log.substr(0, 4000));
  }
  size_t n = 0;
  api.cubin_size(prog, &n);
  std::vector<char> cubin(n);
  api.cubin(prog, cubin.data());
  api.destroy(&prog);
  return cubin;
}

std::vector<char> cached_cubin(const std::string& src, const std::string& name) {
  const std::string path = cache_dir() + "/" + name + ".cubin";
  {
    std::ifstream in(path, std::ios::binary);
    if (in) return std::vector<char>((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  }
  std::vector<char> cubin = compile_cubin(src, name);
  mkdir(cache_dir().c_str(), 0777);
  static std::atomic<unsigned> seq{0};  // unique per writer: threads of one process may compile the same kernel
  const std::string tmp = path + ".tmp" + std::to_string(getpid()) + "." + std::to_string(seq.fetch_add(1));
  {
    std::ofstream out(tmp, std::ios::binary);
    out.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
  }
  std::rename(tmp.c_str(), path.c_str());  // atomic: concurrent compilers of the same pass agree
  return cubin;
}

void emit_op(std::ostringstream& os, const PassOp& op) {
  auto arr = [&](const auto* a, int n) {
    os << '{';
    for (int i = 0; i < n; ++i) os << (i ? "," : "") << static_cast<unsigned long long>(a[i]) << 'u';
    os << '}';
  };
  os << "{" << op.kind << ',' << op.ks << ',' << op.data_off << ',' << op.n_out << ',' << op.log2_groups << ','
     << op.log2_rsplit << ',' << op.aux_off << ',' << op.rmask << ',' << op.ictl_mask << "u," << op.ictl_val << "u,"
     << op.tctl_mask << "u," << op.tctl_val << "u," << static_cast<unsigned long long>(op.cout_mask) << "ull,"
     << static_cast<unsigned long long>(op.cout_val) << "ull,";
  arr(op.out_gbit, 8);
  os << ',';
  arr(op.out_jbit, 8);
  os << ',';
  arr(op.dep, 8);
  os << ',';
  arr(op.xmask, 6);
  os << ',';
  arr(op.tb_pos, 8);
  os << ',';
  arr(op.tb_jbit, 8);
  os << ',' << op.n_tb << ',' << op.n_xmask << ',' << op.thr_off << ',' << op.n_swap << ',';
  arr(op.swap_k, 4);
  os << ',';
  arr(op.swap_l, 4);
  os << ",{}}";
}

// indices of the ops the interpreter visits (a RUN consumes its groups,
// their members and its per-op diagonal ops; kernels_pass.cuh pass_diag_run)
std::vector<int> head_ops(const PassOp* ops, int n_ops) {
  std::vector<int> heads;
  for (int o = 0; o < n_ops;) {
    heads.push_back(o);
    if (ops[o].kind != kPassRun) {
      ++o;
      continue;
    }
    const int n_groups = ops[o].ks, nT = ops[o].log2_groups, nX = ops[o].log2_rsplit;
    int og = o + 1;
    for (int g = 0; g < n_groups; ++g) og += 1 + ops[og].log2_groups;
    o = og + nT + nX;
  }
  return heads;
}

struct Cache {
  std::mutex mu;
  std::map<std::string, const void*> kernels;
};
Cache& cache() {
  static Cache c;
  return c;
}

}  // namespace

bool pass_jit_enabled(int n_qubits) { return tilesim::pass_jit_expected(n_qubits); }

std::string pass_jit_source(int precision_bits, const PassOp* ops, int n_ops, std::string* name) {
  std::ostringstream os;
  os << "#include \"kernels_pass.cuh\"\nnamespace tsg { namespace jit {\n";
  os << "__device__ constexpr PassOp kOps[" << n_ops << "] = {\n";
  for (int o = 0; o < n_ops; ++o) {
    emit_op(os, ops[o]);
    os << ",\n";
  }
  os << "};\nstruct Exec {\n  template <typename Real, int M, int L, typename RG>\n"
        "  static __device__ __forceinline__ void run(const PassOp*, int, const unsigned char* blob, const uint32_t* tcs,"
        " int tid, Real* xr, Real* xi, typename Real2Of<Real>::T* fi_tab, RG& rg) {\n";
  for (int o : head_ops(ops, n_ops))
    os << "    pass_step<Real, M, L>(kOps, " << o << ", " << n_ops << ", blob, tcs, tid, xr, xi, fi_tab, rg);\n";
  os << "  }\n};\n}}  // namespace tsg::jit\n";
  const std::string body = os.str();
  const std::string key =
      hex16(fnv1a(body, fnv1a(std::string(kJitHeaderHash) + (precision_bits == 64 ? "f64" : "f32"))));
  *name = "tsg_pass_jit_" + key;
  std::ostringstream k;
  k << kPreamble << body << "extern \"C\" __global__ void __launch_bounds__(" << kPassThreads << ", 2) " << *name
    << "(const __grid_constant__ tsg::PassParams p) {\n  tsg::k_pass_body<"
    << (precision_bits == 64 ? "double, 11, 5" : "float, 12, 6") << ", 2, tsg::jit::Exec>(p);\n}\n";
  return k.str();
}

std::string dmma_jit_source(int ks, int stages, const uint32_t nz[3], bool tpose, std::string* name) {
  std::ostringstream body;
  body << "complex128 ks=" << ks << " stages=" << stages << " nz=" << nz[0] << "," << nz[1] << "," << nz[2]
       << (tpose ? " tpose" : "");
  const std::string key = hex16(fnv1a(body.str(), fnv1a(std::string(kJitHeaderHash) + "dmma")));
  *name = "tsg_dmma_jit_" + key;
  std::ostringstream k;
  k << kPreamble << "#include \"kernels_dmma.cuh\"\n"
    << "extern \"C\" __global__ void __launch_bounds__(tsg::DShape<double, " << ks << ">::kThreads + 32, "
    << "tsg::DShape<double, " << ks << ">::W >= 16 ? 1 : 2) " << *name
    << "(const __grid_constant__ tsg::DmmaParams<double, " << ks << "> p) {\n"
    << "  tsg::k_stream_dmma_body<double, " << ks << ", " << stages << ", true, false, tsg::DmmaStaticNz<" << nz[0]
    << "u, " << nz[1] << "u, " << nz[2] << "u>, " << (tpose ? "true" : "false") << ">(p);\n}\n";
  return k.str();
}

bool dmma_jit_enabled(int n_qubits) {
  const char* e = std::getenv("TSG_DMMA_JIT");
  if (e && e[0] == '0' && e[1] == '\0') return false;
  return pass_jit_enabled(n_qubits);
}

void pass_jit_cubin(const std::string& source, const std::string& name) { cached_cubin(source, name); }

const void* pass_jit_kernel(const std::string& source, const std::string& name) {
  Cache& c = cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.kernels.find(name);
    if (it != c.kernels.end()) return it->second;
  }
  const std::vector<char> cubin = cached_cubin(source, name);  // outside the lock: compiles run in parallel
  cudaLibrary_t lib = nullptr;
  if (cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess)
    throw std::runtime_error("cudaLibraryLoadData failed for " + name);
  cudaKernel_t k = nullptr;
  if (cudaLibraryGetKernel(&k, lib, name.c_str()) != cudaSuccess)
    throw std::runtime_error("cudaLibraryGetKernel failed for " + name);
  std::lock_guard<std::mutex> lk(c.mu);
  c.kernels.emplace(name, reinterpret_cast<const void*>(k));  // the library stays loaded
  return reinterpret_cast<const void*>(k);
}

}  // namespace tsg
