// NVRTC compilation of generated modules for sm_100a, loaded through the CUDA
// runtime's library API (no driver-API link dependency, so the shared library
// also loads on machines without a GPU driver).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace ocg {

struct JitModule {
  cudaLibrary_t lib = nullptr;
  std::string log;
  ~JitModule();
  cudaKernel_t kernel(const char* name) const;
};

// Compiles `source` (cached on disk by content hash) and loads it.
// Throws std::runtime_error with the NVRTC log on failure.
void jit_compile(const std::string& source, bool fma, JitModule& out);

// Load an already compiled cubin.
void jit_load(const std::string& cubin, JitModule& out);

// Compile (or fetch from the cache) without loading; returns the cubin.
void jit_compile_only(const std::string& source, bool fma, std::string& cubin, std::string* log = nullptr);

}  // namespace ocg
