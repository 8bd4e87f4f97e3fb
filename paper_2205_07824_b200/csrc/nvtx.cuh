// NVTX ranges on the C-ABI entry points: a profiler timeline (Nsight
// Systems / ncu --nvtx) shows the operator passes, the host pipeline and the
// block-Jacobi build / apply by name; no cost without a tool attached.
#pragma once
#include <nvtx3/nvToolsExt.h>

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
