// Runtime-compiled kernels for custom cipher specs (csrc/jit.cu).  Host only.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/lfsr_b200.h"

namespace lc {

// One custom spec's kernels (the same templates as the built-ins, instantiated for it).
struct CustomKernels {
  int lengths[3];
  uint64_t taps[3];
  int clock_taps[3];
  cudaKernel_t walk_plain, walk_rearm, mode_probe;         // walk.cu (runtime F)
  cudaKernel_t is_candidate, predecessors, clock, enumerate;  // kernels.cu
  cudaKernel_t prune_dfs, prune_bfs, prune3_dfs, prune3_bfs, probe_expand;  // prune.cu
};

// 0 if the spec is valid for the kernels (cipher.py:72-86 and a 64-bit state), else 1
// with the reason in *err.
int custom_spec_error(const lc_spec* s, std::string* err);
// The kernels for spec s, compiled and loaded at first use (thread safe, cached per
// spec for the life of the process); null with *err on failure.
const CustomKernels* custom_kernels_for(const lc_spec* s, std::string* err);
// 0 if every kernel of spec s compiles (NVRTC only: no device, nothing loaded), else 1
// with the compiler log in *err.
int custom_compile_check(const lc_spec* s, std::string* err);
// The calling thread's current custom spec (set by the C ABI entry point that validated
// it; launchers' SpecId::CUSTOM cases use it).
void set_current_custom(const CustomKernels* k);
const CustomKernels* current_custom();
int prune2_ring();  // shared-memory ring depth the prune kernels are built with (prune.cu)
int prune3_stack();  // shared-memory stack ring of the v3 DFS kernel (prune.cu)

template <class... A>
cudaError_t jit_launch(cudaKernel_t k, dim3 grid, dim3 block, size_t smem, cudaStream_t st, A... args) {
  void* p[] = {&args...};
  return cudaLaunchKernel(reinterpret_cast<const void*>(k), grid, block, p, smem, st);
}

inline int jit_blocks_per_sm(cudaKernel_t k, int threads, size_t smem = 0) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, reinterpret_cast<const void*>(k), threads, smem) != cudaSuccess)
    return 1;
  return b > 0 ? b : 1;
}

}  // namespace lc
