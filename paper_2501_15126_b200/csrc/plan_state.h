// plan_state.h -- the state behind an opaque perm_plan_t (internal to libperm).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "perm_internal.h"

struct perm_plan_s {
  using Csx = perm::Csx;
  using KernelSpec = perm::KernelSpec;
  using KernelCode = perm::KernelCode;
  int n = 0;
  perm_opts opts{};
  Csx ccs, crs, occs;
  std::vector<int> rowp, colp;
  bool singular = false;
  bool trivial1 = false;  // n == 1
  KernelSpec spec;
  KernelCode code;
  std::vector<char> cubin;
  std::string ptxas_log;
  perm_plan_info info{};
  bool is_u128 = false;   // INT01 partials (16 B)
  bool is_c128 = false;   // complex FP64 partials (re, im; 16 B)
  int kind() const { return is_u128 ? 1 : (is_c128 ? 2 : 0); }
  size_t pbytes() const { return (is_u128 || is_c128) ? 16 : 8; }
  // device state
  bool on_device = false;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  void* d_slots = nullptr;
  void* d_counter = nullptr;
  void* d_partial = nullptr;  // 16 bytes
  void* d_scratch = nullptr;  // fold scratch (world entries)
  void* d_rscratch = nullptr; // tree-reduction pass buffers
  // pooled allocation sizes (perm_free returns the buffers to the pool)
  size_t partial_bytes = 64, counter_bytes = 256, slots_bytes = 0, rscratch_bytes = 0, tier_alloc_bytes = 0;
  std::string lib_key;        // cubin bytes: key of the shared loaded library
  bool lib_held = false;
  size_t scratch_bytes = 0;
  void* d_tier = nullptr;     // HYBRID global tier (tier_rows x resident threads)
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // sweep | tree | fold(+collective)
  uint64_t last_first = 0, last_count = 0;
};

namespace perm {
// plan_io.cpp: binary (de)serialisation of the planning output of a plan
// (matrix, orderings, kernel spec/code, cubin, info) -- the on-disk plan cache
// and rank-0 plan broadcast.  `key` is the planner-cache key (matrix content +
// planning options + library build); import checks it byte for byte.
std::string plan_serialize(const perm_plan_s& p, const std::string& key);
// returns false (and leaves p untouched) on a malformed / foreign blob;
// *key_out receives the embedded key
bool plan_deserialize(const void* blob, size_t size, perm_plan_s& p, std::string* key_out);
uint64_t fnv1a64(const std::string& s, uint64_t seed = 1469598103934665603ull);
const char* build_id();
}  // namespace perm
