// Runtime code generation for model-specific kernels (the paper's "code
// generator to C++/CUDA").
//
// The Python side lowers a model's pointwise plans (expr.py KernelPlan
// instruction lists, expr.py:363-373) to CUDA device functions, splices them
// into the kernel template csrc/ldg_nl.cuh and hands the source here.  NVRTC
// compiles it for sm_100a to a CUBIN which is loaded into the current
// (PyTorch primary) context.  Kernels take one parameter struct by
// value (__grid_constant__) whose bytes the caller packs.  Loading and
// launching go through the runtime's library API (cudaLibraryLoadData /
// cudaLibraryGetKernel), so the library does not link libcuda directly.

#include <cuda_runtime.h>
#include <nvrtc.h>

#include <cstring>
#include <string>
#include <vector>

#include "ldgb200.h"

namespace {
thread_local std::string g_jit_err;

int jfail(int code, const std::string& what) {
  g_jit_err = what;
  return code;
}

}  // namespace

struct LdgModule {
  cudaLibrary_t lib = nullptr;
  std::vector<char> cubin;
};

extern "C" {

const char* ldg_jit_last_error(void) { return g_jit_err.c_str(); }

int ldg_jit_compile(const char* src, const char* name, const char* const* opts, int nopts,
                    void* cubin_out, int64_t* cubin_size) {
  // compile only (no device needed); cubin_out == NULL queries the size
  if (!src || !cubin_size) return jfail(2, "null argument");
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, src, name ? name : "ldg_nl.cu", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return jfail(4, std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(r));
  std::vector<const char*> o;
  o.push_back("-arch=sm_100a");
  o.push_back("-std=c++17");
  o.push_back("-default-device");
  o.push_back("-lineinfo");
  for (int i = 0; i < nopts; ++i) o.push_back(opts[i]);
  r = nvrtcCompileProgram(prog, (int)o.size(), o.data());
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    return jfail(4, std::string("NVRTC compile failed:\n") + log);
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  if (cubin_out) {
    if ((int64_t)n > *cubin_size) {
      nvrtcDestroyProgram(&prog);
      return jfail(2, "cubin buffer too small");
    }
    nvrtcGetCUBIN(prog, static_cast<char*>(cubin_out));
  }
  *cubin_size = (int64_t)n;
  nvrtcDestroyProgram(&prog);
  return 0;
}

int ldg_jit_load(const void* cubin, int64_t size, LdgModule** out) {
  if (!cubin || size <= 0 || !out) return jfail(2, "null argument");
  cudaError_t ce = cudaFree(nullptr);   // make sure the primary context exists
  if (ce != cudaSuccess) return jfail(3, std::string("cudaFree(0): ") + cudaGetErrorString(ce));
  LdgModule* m = new LdgModule();
  m->cubin.assign(static_cast<const char*>(cubin), static_cast<const char*>(cubin) + size);
  ce = cudaLibraryLoadData(&m->lib, m->cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (ce != cudaSuccess) {
    delete m;
    return jfail(3, std::string("cudaLibraryLoadData: ") + cudaGetErrorString(ce));
  }
  *out = m;
  return 0;
}

int ldg_jit_unload(LdgModule* m) {
  if (!m) return 0;
  if (m->lib) cudaLibraryUnload(m->lib);
  delete m;
  return 0;
}

static int get_kernel(LdgModule* m, const char* name, cudaKernel_t* k) {
  cudaError_t ce = cudaLibraryGetKernel(k, m->lib, name);
  if (ce != cudaSuccess)
    return jfail(2, std::string("no kernel ") + name + ": " + cudaGetErrorString(ce));
  return 0;
}

// Launch kernel `name` with its single by-value parameter block `params`.
int ldg_jit_launch(LdgModule* m, const char* name, int gx, int gy, int bx, int smem,
                   const void* params, int64_t param_size, void* stream) {
  if (!m || !name || !params || param_size <= 0) return jfail(2, "null argument");
  cudaKernel_t k;
  if (int rc = get_kernel(m, name, &k)) return rc;
  cudaError_t ce;
  if (smem > 48 * 1024) {
    ce = cudaFuncSetAttribute(reinterpret_cast<const void*>(k),
                              cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (ce != cudaSuccess) return jfail(3, std::string("smem attribute: ") + cudaGetErrorString(ce));
  }
  void* args[] = {const_cast<void*>(params)};
  ce = cudaLaunchKernel(reinterpret_cast<const void*>(k), dim3(gx, gy, 1), dim3(bx, 1, 1), args,
                        (size_t)smem, static_cast<cudaStream_t>(stream));
  if (ce != cudaSuccess)
    return jfail(3, std::string("launch ") + name + ": " + cudaGetErrorString(ce));
  return 0;
}

// Registers / spill / shared usage of a loaded kernel (for tests and tuning).
int ldg_jit_attr(LdgModule* m, const char* name, int* regs, int* local_bytes, int* static_smem) {
  if (!m || !name) return jfail(2, "null argument");
  cudaKernel_t k;
  if (int rc = get_kernel(m, name, &k)) return rc;
  cudaFuncAttributes a;
  cudaError_t ce = cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(k));
  if (ce != cudaSuccess) return jfail(3, std::string("attributes: ") + cudaGetErrorString(ce));
  if (regs) *regs = a.numRegs;
  if (local_bytes) *local_bytes = (int)a.localSizeBytes;
  if (static_smem) *static_smem = (int)a.sharedSizeBytes;
  return 0;
}

}  // extern "C"
