#include "jit.hpp"

#include <nvrtc.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <sys/stat.h>
#include <unistd.h>

#include <thread>

namespace ocg {

namespace {

std::uint64_t fnv1a(const std::string& s) {
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

std::string cache_dir() {
  if (const char* d = std::getenv("OCG_CACHE_DIR")) return d;
  const char* home = std::getenv("HOME");
  return std::string(home ? home : "/tmp") + "/.cache/ocgpu";
}

void mkdirs(const std::string& path) {
  std::string cur;
  std::stringstream ss(path);
  std::string part;
  if (!path.empty() && path[0] == '/') cur = "/";
  while (std::getline(ss, part, '/')) {
    if (part.empty()) continue;
    cur += part + "/";
    ::mkdir(cur.c_str(), 0755);
  }
}

bool read_file(const std::string& path, std::string& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return !out.empty();
}

}  // namespace

JitModule::~JitModule() {
  if (lib) cudaLibraryUnload(lib);
}

cudaKernel_t JitModule::kernel(const char* name) const {
  cudaKernel_t k = nullptr;
  if (cudaLibraryGetKernel(&k, lib, name) != cudaSuccess)
    throw std::runtime_error(std::string("generated kernel not found: ") + name);
  return k;
}

void jit_compile_only(const std::string& source, bool fma, std::string& cubin, std::string* logp) {
  const char* opts[] = {"-arch=sm_100a", "--std=c++17", "-default-device", fma ? "--fmad=true" : "--fmad=false",
                        "-lineinfo", "--extra-device-vectorization", "--ptxas-options=-v"};
  const int nopt = 7;
  std::string key;
  for (int i = 0; i < nopt; ++i) key += std::string(opts[i]) + ";";
  int nv = 0;
  nvrtcVersion(&nv, &nv);
  key += std::to_string(nv) + ";" + source;
  char name[32];
  std::snprintf(name, sizeof name, "%016llx.cubin", static_cast<unsigned long long>(fnv1a(key)));
  const std::string dir = cache_dir();
  const std::string path = dir + "/" + name;

  std::string dummy;
  std::string& outlog = logp ? *logp : dummy;
  if (!std::getenv("OCG_NO_CACHE") && read_file(path, cubin)) {
    if (!read_file(path + ".log", outlog)) outlog = "cache hit " + path;
  } else {
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, source.c_str(), "ocg_generated.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
      throw std::runtime_error("nvrtcCreateProgram failed");
    const nvrtcResult rc = nvrtcCompileProgram(prog, nopt, opts);
    size_t logn = 0;
    nvrtcGetProgramLogSize(prog, &logn);
    std::string log(logn, '\0');
    if (logn) nvrtcGetProgramLog(prog, log.data());
    while (!log.empty() && log.back() == '\0') log.pop_back();
    outlog = log;
    if (rc != NVRTC_SUCCESS) {
      nvrtcDestroyProgram(&prog);
      throw std::runtime_error("NVRTC compile failed: " + log.substr(0, 4000));
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    cubin.resize(n);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    mkdirs(dir);
    const std::string tmp = path + ".tmp" + std::to_string(::getpid()) + "." +
                            std::to_string(std::hash<std::thread::id>{}(std::this_thread::get_id()));
    {
      std::ofstream f(tmp, std::ios::binary);
      f.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
    }
    {
      std::ofstream f(tmp + ".log", std::ios::binary);
      f.write(log.data(), static_cast<std::streamsize>(log.size()));
    }
    std::rename((tmp + ".log").c_str(), (path + ".log").c_str());
    std::rename(tmp.c_str(), path.c_str());
  }
}

void jit_load(const std::string& cubin, JitModule& out) {
  cudaError_t e = cudaLibraryLoadData(&out.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e));
}

void jit_compile(const std::string& source, bool fma, JitModule& out) {
  std::string cubin;
  jit_compile_only(source, fma, cubin, &out.log);
  jit_load(cubin, out);
}

}  // namespace ocg
