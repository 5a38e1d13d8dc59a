// Custom cipher specs (cipher.py:57-170, CipherSpec.from_json): kernels compiled for the
// spec at first use.
//
// The built-in ciphers (A5/1, mini567, mini789) have their kernels compiled ahead of time
// with the spec as template parameters (register lengths, taps and clock taps are
// compile-time constants, so the bitsliced step is pure LOP3s).  Any other valid spec
// gets exactly the same kernel templates, instantiated for it at runtime: the device
// parts of walk.cu, kernels.cu and prune.cu are compiled by NVRTC (loaded with dlopen
// only when a custom spec is first used) for sm_100a, with the spec spelled out as
// `lc::Spec<...>`, and loaded as a CUDA library (cudaLibraryLoadData).  The launchers'
// SpecId::CUSTOM cases take the kernels of the calling thread's current custom spec
// (set by the C ABI entry point that validated it).  R3's period through F, which the
// built-ins fold in at compile time, is a launch parameter for these (WalkParams::window).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "jit.h"
#include "lfsr_internal.h"

namespace lc {
namespace {

struct Nvrtc {
  void* h = nullptr;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult (*add_name)(nvrtcProgram, const char*);
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
  nvrtcResult (*log_size)(nvrtcProgram, size_t*);
  nvrtcResult (*log)(nvrtcProgram, char*);
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*);
  nvrtcResult (*cubin)(nvrtcProgram, char*);
  nvrtcResult (*lowered)(nvrtcProgram, const char*, const char**);
  nvrtcResult (*destroy)(nvrtcProgram*);
  bool ok = false;
};

template <class F>
bool sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  return f != nullptr;
}

Nvrtc& nvrtc(std::string* err) {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    // the toolkit's own NVRTC first: a bare soname can resolve to an older copy another
    // library of the process (torch) already loaded
    for (const char* lib : {"/usr/local/cuda/lib64/libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so",
                            "libnvrtc.so.12", "libnvrtc.so"})
      if ((n.h = dlopen(lib, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
    if (!n.h) return;
    n.ok = sym(n.h, "nvrtcCreateProgram", n.create) && sym(n.h, "nvrtcAddNameExpression", n.add_name) &&
           sym(n.h, "nvrtcCompileProgram", n.compile) && sym(n.h, "nvrtcGetProgramLogSize", n.log_size) &&
           sym(n.h, "nvrtcGetProgramLog", n.log) && sym(n.h, "nvrtcGetCUBINSize", n.cubin_size) &&
           sym(n.h, "nvrtcGetCUBIN", n.cubin) && sym(n.h, "nvrtcGetLoweredName", n.lowered) &&
           sym(n.h, "nvrtcDestroyProgram", n.destroy);
  });
  if (!n.ok && err) *err = "NVRTC (libnvrtc.so.12) not available";
  return n;
}

// the kernel sources: <dir of this library>/../csrc (or /../../csrc for _lib/checked/)
std::string csrc_dir() {
  if (const char* env = getenv("LFSR_CSRC")) return env;
  Dl_info info{};
  if (!dladdr(reinterpret_cast<void*>(&csrc_dir), &info) || !info.dli_fname) return "";
  std::string d = info.dli_fname;
  d = d.substr(0, d.rfind('/'));
  for (int up = 0; up < 3; ++up) {
    const std::string c = d + "/csrc";
    if (FILE* f = fopen((c + "/walk.cu").c_str(), "r")) {
      fclose(f);
      return c;
    }
    d = d.substr(0, d.rfind('/'));
  }
  return "";
}

constexpr const char* kPrelude =
    "typedef unsigned char uint8_t;\n"
    "typedef unsigned short uint16_t;\n"
    "typedef unsigned int uint32_t;\n"
    "typedef unsigned long long uint64_t;\n"
    "typedef signed char int8_t;\n"
    "typedef short int16_t;\n"
    "typedef int int32_t;\n"
    "typedef long long int64_t;\n";

// Compile one source file of csrc/ for `names`; returns the library and lowered names.
bool compile_file(const std::string& dir, const char* file, const std::vector<std::string>& names,
                  cudaLibrary_t* lib, std::vector<std::string>* lowered, std::string* err) {
  Nvrtc& nv = nvrtc(err);
  if (!nv.ok) return false;
  const std::string src = std::string(kPrelude) + "#include \"" + file + "\"\n";
  nvrtcProgram prog;
  if (nv.create(&prog, src.c_str(), "lfsr_custom_spec.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    *err = "nvrtcCreateProgram failed";
    return false;
  }
  for (const std::string& n : names) nv.add_name(prog, n.c_str());
  const std::string inc = "-I" + dir, inc2 = "-I" + dir + "/../../include";
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device", "-lineinfo",
                        inc.c_str(), inc2.c_str(), LC_CHECKS ? "-DLC_CHECKS=1" : "-DLC_CHECKS=0"};
  const nvrtcResult rc = nv.compile(prog, static_cast<int>(sizeof(opts) / sizeof(opts[0])), opts);
  if (rc != NVRTC_SUCCESS) {
    size_t ls = 0;
    nv.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) nv.log(prog, &log[0]);
    *err = std::string("NVRTC compile of ") + file + " failed: " + log.substr(0, 2000);
    nv.destroy(&prog);
    return false;
  }
  size_t cs = 0;
  nv.cubin_size(prog, &cs);
  std::vector<char> cubin(cs);
  nv.cubin(prog, cubin.data());
  lowered->clear();
  for (const std::string& n : names) {
    const char* l = nullptr;
    nv.lowered(prog, n.c_str(), &l);
    lowered->push_back(l ? l : "");
  }
  nv.destroy(&prog);
  if (!lib) return true;  // compile-only check
  const cudaError_t e = cudaLibraryLoadData(lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) {
    *err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
    return false;
  }
  return true;
}

std::mutex g_mu;
std::map<std::string, std::unique_ptr<CustomKernels>> g_cache;
thread_local const CustomKernels* tl_current = nullptr;
CustomKernels g_compile_ok;  // build_custom's result for a successful compile-only check

}  // namespace

int custom_spec_error(const lc_spec* s, std::string* err) {
  int total = 0;
  for (int k = 0; k < 3; ++k) {
    const int l = s->lengths[k];
    if (l < 2 || l > 32) {
      *err = "custom spec: register lengths must be in [2, 32]";
      return 1;
    }
    if (s->clock_taps[k] < 0 || s->clock_taps[k] + 1 >= l) {
      *err = "custom spec: clock taps must satisfy 0 <= tap < length - 1 (cipher.py:80-86)";
      return 1;
    }
    const uint64_t m = (l >= 64) ? ~0ull : ((1ull << l) - 1);
    if ((s->tap_masks[k] & ~m) || !((s->tap_masks[k] >> (l - 1)) & 1ull)) {
      *err = "custom spec: taps must lie in the register and include its top bit (cipher.py:72-79)";
      return 1;
    }
    total += l;
  }
  if (total > 64) {
    *err = "custom spec: registers must fit 64 bits";
    return 1;
  }
  return 0;
}

namespace {
const CustomKernels* build_custom(const lc_spec* s, bool load, std::string* err);
}

const CustomKernels* custom_kernels_for(const lc_spec* s, std::string* err) { return build_custom(s, true, err); }

int custom_compile_check(const lc_spec* s, std::string* err) { return build_custom(s, false, err) ? 0 : 1; }

namespace {
// load = false: compile every unit (NVRTC only, no device), return &dummy on success
const CustomKernels* build_custom(const lc_spec* s, bool load, std::string* err) {
  if (custom_spec_error(s, err)) return nullptr;
  char key[256];
  snprintf(key, sizeof key, "%d,%d,%d,%llu,%llu,%llu,%d,%d,%d", s->lengths[0], s->lengths[1], s->lengths[2],
           static_cast<unsigned long long>(s->tap_masks[0]), static_cast<unsigned long long>(s->tap_masks[1]),
           static_cast<unsigned long long>(s->tap_masks[2]), s->clock_taps[0], s->clock_taps[1], s->clock_taps[2]);
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_cache.find(key);
  if (load && it != g_cache.end()) return it->second.get();
  const std::string dir = csrc_dir();
  if (dir.empty()) {
    *err = "kernel sources (csrc/) not found next to the library";
    return nullptr;
  }
  // the spec as template arguments; WINDOW 0 = R3's period is a launch parameter
  char spec[256];
  snprintf(spec, sizeof spec, "lc::Spec<%d, %d, %d, %lluu, %lluu, %lluu, %d, %d, %d, 0u, 0ull>", s->lengths[0],
           s->lengths[1], s->lengths[2], static_cast<unsigned long long>(s->tap_masks[0]),
           static_cast<unsigned long long>(s->tap_masks[1]), static_cast<unsigned long long>(s->tap_masks[2]),
           s->clock_taps[0], s->clock_taps[1], s->clock_taps[2]);
  const std::string S = spec;
  auto k = std::make_unique<CustomKernels>();
  for (int i = 0; i < 3; ++i) {
    k->lengths[i] = s->lengths[i];
    k->taps[i] = s->tap_masks[i];
    k->clock_taps[i] = s->clock_taps[i];
  }
  struct Unit {
    const char* file;
    std::vector<std::string> names;
    std::vector<cudaKernel_t*> out;
  };
  char ring[16], stack3[16];
  snprintf(ring, sizeof ring, "%d", prune2_ring());
  snprintf(stack3, sizeof stack3, "%d", prune3_stack());
  Unit units[] = {
      {"walk.cu",
       {"&lc::walk_kernel<" + S + ", false, false>", "&lc::walk_kernel<" + S + ", false, true>",
        "&lc::mode_probe_kernel<" + S + ">"},
       {&k->walk_plain, &k->walk_rearm, &k->mode_probe}},
      {"kernels.cu",
       {"&lc::is_candidate_kernel<" + S + ">", "&lc::predecessors_kernel<" + S + ">", "&lc::clock_kernel<" + S + ">",
        "&lc::enumerate_plane_kernel<" + S + ">"},
       {&k->is_candidate, &k->predecessors, &k->clock, &k->enumerate}},
      {"prune.cu",
       {"&lc::prune2_kernel<" + S + ", " + ring + ", true>", "&lc::prune2_kernel<" + S + ", " + ring + ", false>",
        "&lc::prune3_kernel<" + S + ", " + stack3 + ", true>", "&lc::prune3_kernel<" + S + ", " + stack3 + ", false>",
        "&lc::probe_expand_kernel<" + S + ">"},
       {&k->prune_dfs, &k->prune_bfs, &k->prune3_dfs, &k->prune3_bfs, &k->probe_expand}},
  };
  for (Unit& u : units) {
    cudaLibrary_t lib;
    std::vector<std::string> lowered;
    if (!compile_file(dir, u.file, u.names, load ? &lib : nullptr, &lowered, err)) return nullptr;
    if (!load) continue;
    for (size_t i = 0; i < u.names.size(); ++i) {
      const cudaError_t e = cudaLibraryGetKernel(u.out[i], lib, lowered[i].c_str());
      if (e != cudaSuccess) {
        *err = "cudaLibraryGetKernel(" + u.names[i] + "): " + cudaGetErrorString(e);
        return nullptr;
      }
    }
  }
  if (!load) return &g_compile_ok;
  const CustomKernels* p = k.get();
  g_cache.emplace(key, std::move(k));
  return p;
}
}  // namespace

void set_current_custom(const CustomKernels* k) { tl_current = k; }
const CustomKernels* current_custom() { return tl_current; }

}  // namespace lc
