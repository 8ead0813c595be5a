// rt_internal.h -- helpers shared by runtime.cpp (C ABI, device runtime) and
// planner.cpp (kernel planner): error slot, clock, NVTX ranges, the planner
// entry point.  Internal to libperm.
#pragma once
#include <chrono>
#include <future>
#include <string>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a profiler is attached

#include "perm.h"

struct perm_plan_s;

namespace perm {

extern thread_local std::string g_err;  // perm_last_error()

inline int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

inline double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// NVTX ranges around the planner phases and the compute steps (nsys / ncu
// timelines; `ncu --nvtx --nvtx-include perm_compute/` selects one permanent)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

// The planner (planner.cpp) for a validated, structurally nonsingular plan
// whose mode is set: base orderings, elimination searches, candidate kernels,
// NVRTC compiles with the spill gate, optional on-device autotune; fills the
// plan's ordering, spec, code, cubin and info fields.  PERM_OK, or an error
// code with g_err set.  ctx_ready: the CUDA context (created concurrently).
int plan_kernel(perm_plan_s* p, perm_ordering ord, double gr, const std::shared_future<void>& ctx_ready);

}  // namespace perm
