// tsm_jit.cpp -- run-time instantiation of the width-specialised kernels.
//
// The AOT build instantiates the benchmark shapes (tools/gen_instances.py).
// Every other (op, dtype, M, N) -- and every explicit configuration the
// autotuner asks for -- is compiled at plan-creation time by NVRTC from the
// SAME template source (csrc/tsm_kernels.cuh, embedded at build time) for
// sm_100a, loaded with cudaLibraryLoadData and launched like the AOT kernels.
// Compiled cubins are memoised in-process and, optionally, on disk
// (TSM_JIT_CACHE_DIR, default $HOME/.cache/libtsm; set to "" to disable).
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <deque>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <unistd.h>
#include <vector>

#include "tsm_internal.h"
#include "tsm_registry.h"

#include "gen/kernel_source.inc"  // static const char* kTsmKernelSource

namespace tsm {

namespace {

std::mutex g_jit_mu;
std::deque<KernelEntry> g_jit_entries;  // stable addresses
std::map<std::string, const KernelEntry*> g_jit_index;

std::string cfg_type(const KernelEntry& ein) {
  // complex-as-real entries instantiate the real kernel on 2M x 2N with ZR = true
  const KernelEntry e = real_view(ein);
  const char* zr = zr_flag(ein.edge) ? "true" : "false";
  std::ostringstream os;
  const char* z = e.dt ? "true" : "false";
  if (e.op == KIND_TSMTTSM && e.impl >= 1)
    os << "tsm::TsmttsmMmaCfg<" << e.M << ", " << e.N << ", " << z << ", " << e.p0 << ", " << e.p1
       << ", " << (e.NT / 32 - 1 - edge_warps(e.edge)) << ", " << e.R << ", " << e.p2 << ", " << e.p3 << ", "
       << (e.impl == 2 ? "true" : "false") << ", " << edge_warps(e.edge) << ", "
       << ((e.edge & 2) ? "true" : "false") << ", " << zr << ", " << (g3_flag(e.edge) ? "true" : "false") << ", "
       << (ei_flag(e.edge) ? "true" : "false") << ", " << (lb_flag(e.edge) ? "true" : "false") << ", "
       << (ga_flag(e.edge) ? "true" : "false") << ">";
  else if (e.op == KIND_TSMTTSM)
    os << "tsm::TsmttsmCfg<" << e.M << ", " << e.N << ", " << z << ", " << e.p0 << ", " << e.p1
       << ", " << e.NT << ", " << e.R << ">";
  else if (e.impl == 4)
    os << "tsm::TsmmCstbCfg<" << e.M << ", " << e.N << ", " << z << ", " << e.p0 << ", " << e.p1
       << ", " << (e.NT / 32 - 1) << ", " << e.R << ", " << ((e.edge & 1) ? e.N % 8 : 0) << ", "
       << (ga_flag(e.edge) ? "true" : "false") << ">";
  else if (e.impl == 3)
    os << "tsm::TsmmCstCfg<" << e.M << ", " << e.N << ", " << z << ", " << e.p0 << ", " << e.p1
       << ", " << (e.NT / 32 - 1) << ", " << e.R << ", " << zr << ", " << ((e.edge & 1) ? e.N % 8 : 0) << ", "
       << (g3_flag(e.edge) ? "true" : "false") << ">";
  else if (e.impl >= 1)
    os << "tsm::TsmmMmaCfg<" << e.M << ", " << e.N << ", " << z << ", " << e.p0 << ", "
       << (e.NT / 32 - 1) << ", " << e.R << ", " << e.p1 << ", " << e.p2 << ", "
       << (e.impl == 2 ? "true" : "false") << ">";
  else
    os << "tsm::TsmmCfg<" << e.M << ", " << e.N << ", " << z << ", " << e.p0 << ", " << e.p1
       << ", " << e.p2 << ", " << e.NT << ", " << e.R << ">";
  return os.str();
}

std::string kernel_name(const KernelEntry& e) {
  const char* fn = e.op == KIND_TSMM ? (e.impl == 4   ? "tsm::tsmm_cstb_kernel<"
                                        : e.impl == 3 ? "tsm::tsmm_cst_kernel<"
                                        : e.impl >= 1 ? "tsm::tsmm_mma_kernel<" : "tsm::tsmm_kernel<")
                   : (e.impl >= 1 ? "tsm::tsmttsm_mma_kernel<" : "tsm::tsmttsm_kernel<");
  return std::string(fn) + cfg_type(e) + ">";
}

unsigned long long fnv1a(const std::string& s, unsigned long long h = 1469598103934665603ull) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

// Default cache: <directory of libtsm.so>/kcache (filled at build time by
// tsm_jit_precompile, travels with the library), else $HOME/.cache/libtsm.
std::string cache_dir() {
  const char* d = getenv("TSM_JIT_CACHE_DIR");
  if (d) return std::string(d);
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&cache_dir), &info) && info.dli_fname) {
    std::string lib(info.dli_fname);
    const size_t slash = lib.rfind('/');
    const std::string dir = (slash == std::string::npos ? std::string(".") : lib.substr(0, slash)) + "/kcache";
    mkdir(dir.c_str(), 0755);
    if (access(dir.c_str(), W_OK) == 0) return dir;
  }
  const char* home = getenv("HOME");
  return home ? std::string(home) + "/.cache/libtsm" : std::string();
}

bool read_file(const std::string& path, std::vector<char>* out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  out->assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  return !out->empty();
}

void write_file_atomic(const std::string& dir, const std::string& name, const std::vector<char>& data) {
  if (dir.empty()) return;
  std::string cur;
  for (size_t i = 0; i <= dir.size(); i++) {  // mkdir -p
    if (i == dir.size() || dir[i] == '/') {
      if (!cur.empty()) mkdir(cur.c_str(), 0755);
    }
    if (i < dir.size()) cur += dir[i];
  }
  const std::string tmp = dir + "/" + name + ".tmp" + std::to_string(getpid());
  {
    std::ofstream f(tmp, std::ios::binary);
    if (!f) return;
    f.write(data.data(), static_cast<std::streamsize>(data.size()));
  }
  std::rename(tmp.c_str(), (dir + "/" + name).c_str());
}

tsm_status compile(const KernelEntry& e, std::vector<char>* cubin, std::string* lowered) {
  const std::string name = kernel_name(e);
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, kTsmKernelSource, "tsm_kernels.cuh", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return fail(TSM_ERR_INTERNAL, std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(r));
  nvrtcAddNameExpression(prog, name.c_str());
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device",
                        "-DTSM_NVRTC", "-lineinfo"};
  r = nvrtcCompileProgram(prog, 5, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    return fail(TSM_ERR_INTERNAL, "NVRTC compile of " + name + " failed:\n" + log);
  }
  const char* low = nullptr;
  nvrtcGetLoweredName(prog, name.c_str(), &low);
  *lowered = low ? low : "";
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin->resize(n);
  nvrtcGetCUBIN(prog, cubin->data());
  nvrtcDestroyProgram(&prog);
  if (lowered->empty() || cubin->empty()) return fail(TSM_ERR_INTERNAL, "NVRTC produced no cubin");
  return TSM_SUCCESS;
}

}  // namespace

// cubin + lowered name of `want`: from the disk cache, else compiled by NVRTC
// (and written to the cache).
tsm_status cubin_for(const KernelEntry& want, std::vector<char>* cubin, std::string* lowered) {
  const std::string key = kernel_name(want);
  // one subdirectory per kernel-source version (stale ones can be pruned whole)
  static const unsigned long long src_hash = fnv1a(kTsmKernelSource);
  char sbuf[32];
  snprintf(sbuf, sizeof sbuf, "/src_%016llx", src_hash);
  std::string dir = cache_dir();
  if (!dir.empty()) dir += sbuf;
  char hbuf[32];
  snprintf(hbuf, sizeof hbuf, "%016llx", fnv1a(key, src_hash));
  const std::string cname = std::string("tsm_") + hbuf + ".cubin";
  const std::string lname = std::string("tsm_") + hbuf + ".name";
  std::vector<char> lowv;
  if (!dir.empty() && read_file(dir + "/" + cname, cubin) && read_file(dir + "/" + lname, &lowv)) {
    lowered->assign(lowv.begin(), lowv.end());
    return TSM_SUCCESS;
  }
  tsm_status st = compile(want, cubin, lowered);
  if (st != TSM_SUCCESS) return st;
  write_file_atomic(dir, cname, *cubin);
  write_file_atomic(dir, lname, std::vector<char>(lowered->begin(), lowered->end()));
  return TSM_SUCCESS;
}

// Build-time: compile `want` into the disk cache (no CUDA device needed).
tsm_status jit_precompile(const KernelEntry& want) {
  std::vector<char> cubin;
  std::string lowered;
  return cubin_for(want, &cubin, &lowered);
}

// Returns a registry entry whose func is a JIT-compiled kernel for `want`.
tsm_status jit_kernel(const KernelEntry& want, const KernelEntry** out) {
  const std::string key = kernel_name(want);
  {
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto it = g_jit_index.find(key);
    if (it != g_jit_index.end()) {
      *out = it->second;
      return TSM_SUCCESS;
    }
  }
  // compile / load outside the lock: independent plans JIT in parallel
  std::vector<char> cubin;
  std::string lowered;
  {
    tsm_status st = cubin_for(want, &cubin, &lowered);
    if (st != TSM_SUCCESS) return st;
  }
  cudaLibrary_t lib;
  cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess)
    return fail(TSM_ERR_CUDA, std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e));
  cudaKernel_t k;
  e = cudaLibraryGetKernel(&k, lib, lowered.c_str());
  if (e != cudaSuccess)
    return fail(TSM_ERR_CUDA, std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e));
  KernelEntry ent = want;
  ent.func = reinterpret_cast<const void*>(k);
  std::lock_guard<std::mutex> lk(g_jit_mu);
  auto it = g_jit_index.find(key);
  if (it != g_jit_index.end()) {  // another thread finished first: keep one entry
    *out = it->second;
    return TSM_SUCCESS;
  }
  g_jit_entries.push_back(ent);
  const KernelEntry* p = &g_jit_entries.back();
  g_jit_index[key] = p;
  *out = p;
  return TSM_SUCCESS;
}

int jit_count() {
  std::lock_guard<std::mutex> lk(g_jit_mu);
  return static_cast<int>(g_jit_entries.size());
}

}  // namespace tsm
