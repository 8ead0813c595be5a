// runtime.cpp -- libperm C ABI: plan entry (validation, caches, device
// load), launch, deterministic reduction, shards, fold and the collective.
// The kernel planner (searches, codegen candidates, NVRTC, autotune) is in
// planner.cpp.  See include/perm.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <unistd.h>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a profiler is attached

#include "perm_internal.h"
#include "plan_state.h"
#include "rt_internal.h"

namespace {

}  // namespace

extern "C" cudaError_t libperm_launch_tree_reduce(const void* slots, uint64_t count, int kind, void* out,
                                                  void* scratch, cudaStream_t st);
extern "C" size_t libperm_tree_scratch_bytes(uint64_t count, int kind);
extern "C" cudaError_t libperm_launch_fold(const void* partials, int world, int n, int kind, int neg,
                                           void* out, cudaStream_t st);
extern "C" cudaError_t libperm_probe_fp64_peak(int device, int reps, double* ops_per_s, double* ms_best);
// collective.cpp (dlopen'd NCCL)
int libperm_allgather(void* comm, void* recv, size_t bytes, int rank, cudaStream_t st, std::string& msg);
int libperm_comm_unique_id(void* id128, std::string& msg);
int libperm_comm_init(int world, int rank, const void* id128, int device, void** comm, std::string& msg);
int libperm_comm_destroy(void* comm, std::string& msg);

using namespace perm;

namespace perm {
thread_local std::string g_err;
}

namespace {




std::mutex g_cache_mu;

bool all_ones(const Csx& a) {
  for (double v : a.val)
    if (v != 1.0) return false;
  return true;
}

// Bregman-Minc: perm(A) <= prod_i (r_i!)^(1/r_i) for 0/1 A; INT01 needs
// |perm| * 2^(n-1) < 2^127 (T' fits the signed 128-bit range).
bool int01_fits(const Csx& crs) {
  double lg = 0;
  for (int i = 0; i < crs.n; ++i) {
    int r = crs.ptr[i + 1] - crs.ptr[i];
    if (r == 0) return true;  // perm = 0
    lg += std::lgamma((double)r + 1.0) / std::log(2.0) / r;
  }
  return lg + (crs.n - 1) < 126.0;
}

}  // namespace

// struct perm_plan_s: plan_state.h

namespace {

std::map<std::string, perm_plan_s> g_plan_cache;  // guarded by g_cache_mu

#define CUDA_TRY(x)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) return fail(PERM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---- process-wide device resources shared by plans -------------------------
// Loaded sweep libraries are cached by (device, cubin) so re-planning the same
// matrix (planner cache hit) does not reload the module; device buffers are
// recycled through a small per-device pool (perm_free synchronises the plan's
// stream before returning them).  Both are bounded.
struct LibEntry {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int regs = 0, local = 0, bps = 0, refs = 0;
  uint64_t stamp = 0;
};
std::mutex g_dev_mu;
std::map<std::pair<int, std::string>, LibEntry> g_libs;
uint64_t g_lib_clock = 0;
std::multimap<std::pair<int, size_t>, void*> g_pool;
size_t g_pool_bytes = 0;
constexpr size_t kPoolCap = 256ull << 20;
constexpr int kIdleLibs = 16;

cudaError_t pool_alloc(int dev, void** ptr, size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_pool.find({dev, bytes});
    if (it != g_pool.end()) {
      *ptr = it->second;
      g_pool.erase(it);
      g_pool_bytes -= bytes;
      return cudaSuccess;
    }
  }
  return cudaMalloc(ptr, bytes);
}

void pool_free(int dev, void* ptr, size_t bytes) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (g_pool_bytes + bytes > kPoolCap) {
    cudaFree(ptr);
    return;
  }
  g_pool.insert({{dev, bytes}, ptr});
  g_pool_bytes += bytes;
}

void lib_release(int dev, const std::string& key) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_libs.find({dev, key});
  if (it == g_libs.end()) return;
  it->second.refs -= 1;
  it->second.stamp = ++g_lib_clock;
  int idle = 0;
  for (auto& kv : g_libs) idle += kv.second.refs == 0;
  while (idle > kIdleLibs) {  // unload the least recently used idle library
    auto old = g_libs.end();
    for (auto q = g_libs.begin(); q != g_libs.end(); ++q)
      if (q->second.refs == 0 && (old == g_libs.end() || q->second.stamp < old->second.stamp)) old = q;
    cudaLibraryUnload(old->second.lib);
    g_libs.erase(old);
    --idle;
  }
}

int load_device_impl(perm_plan_s* p);
int load_device(perm_plan_s* p) {
  const double t0 = now_ms();
  const int st = load_device_impl(p);
  if (getenv("PERM_DEBUG_TIMING")) fprintf(stderr, "[timing] load_device %.3f ms\n", now_ms() - t0);
  return st;
}
int load_device_impl(perm_plan_s* p) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(PERM_ECUDA, std::string("no CUDA device available (no CPU fallback): ") + cudaGetErrorString(e));
  if (p->opts.device < 0 || p->opts.device >= ndev) return fail(PERM_ECUDA, "device ordinal out of range");
  p->device = p->opts.device;
  CUDA_TRY(cudaSetDevice(p->device));
  // single attributes (cudaGetDeviceProperties costs milliseconds per call)
  int major = 0, minor = 0, sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, p->device));
  CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, p->device));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device));
  if (major != 10 || minor != 0)
    return fail(PERM_ECUDA, "libperm kernels are built for sm_100a (B200); device is sm_" +
                                std::to_string(major) + std::to_string(minor));
  p->info.sms = sms;
  const bool dbg_t = getenv("PERM_DEBUG_TIMING") != nullptr;
  double tq = now_ms();
  auto lap = [&](const char* what) {
    if (!dbg_t) return;
    cudaDeviceSynchronize();
    fprintf(stderr, "[timing]   %s %.3f ms\n", what, now_ms() - tq);
    tq = now_ms();
  };
  lap("attributes");
  if (p->opts.cuda_stream) {
    p->stream = (cudaStream_t)p->opts.cuda_stream;
  } else {
    CUDA_TRY(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    p->own_stream = true;
  }
  for (auto& ev : p->ev) CUDA_TRY(cudaEventCreate(&ev));
  lap("stream+events");
  CUDA_TRY(pool_alloc(p->device, &p->d_partial, p->partial_bytes));
  // the result / partial slots are 16 bytes (complex, u128) and copied back
  // whole; FP64 writes 8 of them: zero them once (compute-sanitizer initcheck)
  CUDA_TRY(cudaMemsetAsync(p->d_partial, 0, p->partial_bytes, p->stream));
  p->scratch_bytes = 16 * 128;
  CUDA_TRY(pool_alloc(p->device, &p->d_scratch, p->scratch_bytes));
  CUDA_TRY(cudaMemsetAsync(p->d_scratch, 0, p->scratch_bytes, p->stream));
  CUDA_TRY(pool_alloc(p->device, &p->d_counter, p->counter_bytes));
  if (!p->singular && !p->trivial1) {
    p->lib_key.assign(p->cubin.begin(), p->cubin.end());
    LibEntry le;
    bool hit = false;
    {
      std::lock_guard<std::mutex> lk(g_dev_mu);
      auto it = g_libs.find({p->device, p->lib_key});
      if (it != g_libs.end()) {
        it->second.refs += 1;
        le = it->second;
        hit = true;
      }
    }
    if (!hit) {
      CUDA_TRY(cudaLibraryLoadData(&le.lib, p->cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
      CUDA_TRY(cudaLibraryGetKernel(&le.kern, le.lib, p->code.name.c_str()));
      if (p->code.smem_bytes > 0)
        CUDA_TRY(cudaFuncSetAttribute((const void*)le.kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      p->code.smem_bytes));
      cudaFuncAttributes fa;
      CUDA_TRY(cudaFuncGetAttributes(&fa, (const void*)le.kern));
      le.regs = fa.numRegs;
      le.local = (int)fa.localSizeBytes;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&le.bps, (const void*)le.kern, p->spec.threads,
                                                             p->code.smem_bytes));
      le.refs = 1;
      std::lock_guard<std::mutex> lk(g_dev_mu);
      auto ins = g_libs.insert({{p->device, p->lib_key}, le});
      if (!ins.second) {  // another thread loaded it meanwhile: use that one
        cudaLibraryUnload(le.lib);
        ins.first->second.refs += 1;
        le = ins.first->second;
      }
    }
    lap(hit ? "library (cached)" : "library load");
    p->lib_held = true;
    p->kern = le.kern;
    p->info.regs_per_thread = le.regs;
    p->info.local_bytes = le.local;
    if (le.bps < 1) return fail(PERM_ECUDA, "generated kernel cannot be resident (occupancy 0)");
    p->info.blocks_per_sm = le.bps;
    p->info.grid = le.bps * p->info.sms;
    p->slots_bytes = std::max<size_t>(p->pbytes() * (size_t)p->info.tasks, 16);
    CUDA_TRY(pool_alloc(p->device, &p->d_slots, p->slots_bytes));
    p->rscratch_bytes = libperm_tree_scratch_bytes(p->info.tasks, p->kind());
    CUDA_TRY(pool_alloc(p->device, &p->d_rscratch, p->rscratch_bytes));
    if (p->code.tier_bytes > 0) {
      p->tier_alloc_bytes = (size_t)p->code.tier_bytes * (size_t)p->info.grid * (size_t)p->spec.threads;
      CUDA_TRY(pool_alloc(p->device, &p->d_tier, p->tier_alloc_bytes));
    }
    lap("buffers");
  }
  p->on_device = true;
  return PERM_OK;
}

// Sweep tasks [first, first+count) and reduce them into p->d_partial.
int run_range(perm_plan_s* p, uint64_t first, uint64_t count, double* sweep_ms, double* reduce_ms) {
  p->last_first = first;
  p->last_count = count;
  if (count == 0) {
    CUDA_TRY(cudaMemsetAsync(p->d_partial, 0, 16, p->stream));
    if (sweep_ms) *sweep_ms = 0;
    if (reduce_ms) *reduce_ms = 0;
    return PERM_OK;
  }
  if (count > 0x7fffffffull)  // the kernel's task counter is 32-bit
    return fail(PERM_EINVAL, "more than 2^31 warp-tasks in one launch: set task_chunks (M) larger");
  CUDA_TRY(cudaMemsetAsync(p->d_counter, 0, sizeof(unsigned), p->stream));
  unsigned long long tb = first;
  unsigned tc = (unsigned)count;
  unsigned long long stride = 1;
  void* args[] = {&tb, &tc, &stride, &p->d_counter, &p->d_slots, &p->d_tier};
  const int grid = (int)std::min<uint64_t>((uint64_t)p->info.grid,
                                           (count * 32 + p->spec.threads - 1) / p->spec.threads);
  CUDA_TRY(cudaEventRecord(p->ev[0], p->stream));
  {
    Nvtx r("perm_sweep");
    CUDA_TRY(cudaLaunchKernel((const void*)p->kern, dim3(grid), dim3(p->spec.threads), args,
                              (size_t)p->code.smem_bytes, p->stream));
  }
  CUDA_TRY(cudaEventRecord(p->ev[1], p->stream));
  {
    Nvtx r("perm_reduce");
    CUDA_TRY(libperm_launch_tree_reduce(p->d_slots, count, p->kind(), p->d_partial, p->d_rscratch, p->stream));
  }
  CUDA_TRY(cudaEventRecord(p->ev[2], p->stream));
  if (sweep_ms || reduce_ms) {
    CUDA_TRY(cudaEventSynchronize(p->ev[2]));
    float a = 0, b = 0;
    CUDA_TRY(cudaEventElapsedTime(&a, p->ev[0], p->ev[1]));
    CUDA_TRY(cudaEventElapsedTime(&b, p->ev[1], p->ev[2]));
    if (sweep_ms) *sweep_ms = a;
    if (reduce_ms) *reduce_ms = b;
  }
  return PERM_OK;
}

int shard_range(perm_plan_s* p, int rank, int world, uint64_t& first, uint64_t& count) {
  if (world < 1 || (world & (world - 1)) || world > 65536)
    return fail(PERM_EINVAL, "world must be a power of two <= 65536");
  if (rank < 0 || rank >= world) return fail(PERM_EINVAL, "rank out of range");
  const uint64_t T = p->info.tasks;
  if (T >= (uint64_t)world) {
    count = T / world;
    first = count * rank;
  } else {
    count = (uint64_t)rank < T ? 1 : 0;
    first = std::min<uint64_t>((uint64_t)rank, T);  // empty shards sit at the end
  }
  return PERM_OK;
}

void fill_result(perm_plan_s* p, perm_result* r, const unsigned char* raw16, bool scaled) {
  std::memset(r, 0, sizeof(*r));
  r->w_plan = p->info.w_plan;
  r->k = p->info.k;
  r->c = p->info.c;
  r->b = p->info.B;
  r->mode = p->info.mode;
  r->K = p->info.K;
  if (p->is_u128) {
    uint64_t lo, hi;
    std::memcpy(&lo, raw16, 8);
    std::memcpy(&hi, raw16 + 8, 8);
    r->exact_lo = lo;
    r->exact_hi = hi;
    r->exact_valid = 1;
    __int128 v = (__int128)(((unsigned __int128)hi << 64) | lo);
    r->value = (double)v;
  } else {
    double v;
    std::memcpy(&v, raw16, 8);
    r->value = v;
    if (p->is_c128) std::memcpy(&r->value_im, raw16 + 8, 8);
  }
  (void)scaled;
}

}  // namespace

extern "C" {

const char* perm_last_error(void) { return g_err.c_str(); }
const char* perm_version(void) { return "libperm 0.1 (sm_100a, arXiv 2501.15126 sweep)"; }

int perm_structural_rank(int n, perm_format fmt, const int32_t* ptr, const int32_t* idx, const double* val) {
  Csx ccs, crs;
  std::string err;
  if (validate_and_convert(n, fmt, ptr, idx, val, ccs, crs, err) != PERM_OK) {
    g_err = err;
    return -1;
  }
  return structural_rank(ccs);
}

int perm_order(int n, perm_format fmt, const int32_t* ptr, const int32_t* idx, const double* val,
               perm_ordering ord, int32_t* row_perm, int32_t* col_perm) {
  Csx ccs, crs;
  std::string err;
  int st = validate_and_convert(n, fmt, ptr, idx, val, ccs, crs, err);
  if (st != PERM_OK) return fail(st, err);
  std::vector<int> rp, cp;
  if (ord == PERM_ORDER_PERMANENT) order_permanent(ccs, crs, rp, cp);
  else if (ord == PERM_ORDER_DEGREE) order_degree(ccs, rp, cp);
  else if (ord == PERM_ORDER_NONE) {
    for (int i = 0; i < n; ++i) { rp.push_back(i); cp.push_back(i); }
  } else return fail(PERM_EINVAL, "perm_order: ordering must be NONE, DEGREE or PERMANENT");
  for (int i = 0; i < n; ++i) { row_perm[i] = rp[i]; col_perm[i] = cp[i]; }
  return PERM_OK;
}

int perm_partition(int n, const int32_t* cptrs, const int32_t* rids, double gr_ratio, int sms, int* k, int* c) {
  if (n < 1 || n > 64 || !cptrs || !k || !c) return fail(PERM_EINVAL, "perm_partition: bad arguments");
  Csx o;
  o.n = n;
  o.ptr.assign(cptrs, cptrs + n + 1);
  o.idx.assign(rids, rids + cptrs[n]);
  o.val.assign(cptrs[n], 1.0);
  partition_alg4(o, gr_ratio > 0 ? gr_ratio : 16.0, sms > 0 ? sms : 148, *k, *c);
  return PERM_OK;
}

int perm_alg2_launch_parameters(uint64_t tau, int n, uint64_t* out, int cap) {
  return alg2_launch_parameters(tau, n, out, cap);
}

}  // extern "C"

static int plan_impl(int n, perm_format fmt, const int32_t* ptr, const int32_t* idx, const double* val,
                     bool complex_input, perm_ordering ord, const perm_opts* opts_in, perm_plan_t* out) {
  if (!out) return fail(PERM_EINVAL, "out is NULL");
  *out = nullptr;
  Nvtx range("perm_plan");
  const double t0 = now_ms();
  auto* p = new perm_plan_s();
  if (opts_in) p->opts = *opts_in;
  if (p->opts.world > 1 && ((p->opts.world & (p->opts.world - 1)) || p->opts.world > 128 || p->opts.rank < 0 ||
                            p->opts.rank >= p->opts.world)) {
    delete p;
    return fail(PERM_EINVAL, "opts.world must be a power of two <= 128 and 0 <= opts.rank < world");
  }
  auto bail = [&](int code) {
    perm_free(p);
    return code;
  };
  // the CUDA context is created on a helper thread while the host planner
  // runs (a cold process spends ~0.3 s in context creation); load_device and
  // the autotune wait for it
  std::shared_future<void> ctx_ready;
  if (!p->opts.no_device) {
    const int dev = p->opts.device;
    ctx_ready = std::async(std::launch::async, [dev] {
                  int nd = 0;
                  if (cudaGetDeviceCount(&nd) == cudaSuccess && dev >= 0 && dev < nd && cudaSetDevice(dev) == cudaSuccess)
                    cudaFree(nullptr);
                  cudaGetLastError();
                }).share();
  }
  std::string err;
  int st = complex_input ? validate_and_convert_c(n, fmt, ptr, idx, val, p->ccs, p->crs, err)
                         : validate_and_convert(n, fmt, ptr, idx, val, p->ccs, p->crs, err);
  if (st != PERM_OK) { delete p; return fail(st, err); }
  p->n = n;
  perm_plan_info& I = p->info;
  I.n = n;
  I.nnz = p->ccs.nnz();
  I.struct_rank = structural_rank(p->ccs);
  I.singular = p->singular = I.struct_rank < n;
  const double gr = p->opts.gr_ratio > 0 ? p->opts.gr_ratio : 16.0;
  if (getenv("PERM_DEBUG_TIMING")) fprintf(stderr, "[timing] validate+rank %.3f ms\n", now_ms() - t0);

  // ---- mode
  int mode = p->opts.mode;
  if (mode < PERM_MODE_AUTO || mode > PERM_MODE_INT01) { delete p; return fail(PERM_EINVAL, "unknown mode"); }
  if (complex_input) {
    if (mode == PERM_MODE_INT01 || mode == PERM_MODE_HYBRID) {
      delete p;
      return fail(PERM_EINVAL, "complex matrices support modes AUTO/REG only");
    }
    mode = PERM_MODE_COMPLEX_INTERNAL;
  }
  if (mode == PERM_MODE_AUTO) mode = (all_ones(p->ccs) && int01_fits(p->crs)) ? PERM_MODE_INT01 : PERM_MODE_REG;
  if (mode == PERM_MODE_INT01) {
    if (!all_ones(p->ccs)) { delete p; return fail(PERM_EINVAL, "INT01 mode needs every value == 1.0"); }
    if (!int01_fits(p->crs)) {
      delete p;
      return fail(PERM_ERANGE, "INT01: Bregman-Minc bound * 2^(n-1) may exceed 2^127");
    }
  }
  I.mode = mode;
  p->is_u128 = mode == PERM_MODE_INT01;
  p->is_c128 = mode == PERM_MODE_COMPLEX_INTERNAL;

  // ---- geometry for a sweep over nb h-bits: B, U, M, tasks (Lemma 1 aligned
  // chunks; DESIGN "Chunk grid").  Depends only on (n, K, opts): identical on
  // every rank, so shards are complete subtrees of the same reduction tree.
  if (p->opts.task_chunks > 0 && (p->opts.task_chunks & (p->opts.task_chunks - 1))) {
    delete p;
    return fail(PERM_EINVAL, "task_chunks must be a power of two");
  }
  if (ord < PERM_ORDER_NONE || ord > PERM_ORDER_AUTO) { delete p; return fail(PERM_EINVAL, "unknown ordering"); }
  // in-process planner cache: same matrix + planning options -> same plan
  std::string pkey;
  {
    auto app = [&](const void* d, size_t nb) { pkey.append((const char*)d, nb); };
    const int hdr[] = {n, mode, (int)ord, p->opts.chunk_log2, p->opts.block_log2, p->opts.task_chunks,
                       p->opts.factor_cols, p->opts.min_blocks, p->opts.threads_per_block,
                       p->opts.hybrid_c, p->opts.zero_skip, p->opts.autotune, p->opts.no_device,
                       p->opts.reseed_log2};
    app(hdr, sizeof hdr);
    // planner knobs read from the environment change plans: part of the key
    for (const char* k : {"PERM_ELIM_CANDS", "PERM_ELIM_MAXSIZE", "PERM_ELIM_BEAM", "PERM_ELIM_VARIANTS", "PERM_NO_CC",
                          "PERM_PLAN_COMPILES", "PERM_NO_AUTOTUNE", "PERM_ALLOW_SPILL", "PERM_PLAN_BUDGET",
                          // codegen post-pass knobs (codegen.cpp post_pass)
                          "PERM_NO_SMEM", "PERM_SMEM_ALL", "PERM_NO_DCE", "PERM_NO_FUSE", "PERM_NO_KC", "PERM_KC_CAP", "PERM_SMEM_VOL_FRAC", "PERM_LADDER_RUNGS",
                          "PERM_NO_ASM_MUL", "PERM_ASM_MUL", "PERM_PIPE_DISPATCH", "PERM_SPILL_OK", "PERM_SCORE_B",
                          "PERM_TASK_BITS", "PERM_NO_SMEM_RO", "PERM_SMEM_RO", "PERM_SMEM_RO_FORCE", "PERM_ELIM_TIER4", "PERM_ELIM_SHIFT", "PERM_GIANT_BEAM", "PERM_ELIM_TIER4_ALL"}) {
      const char* v = getenv(k);
      pkey += k;
      pkey += '=';
      pkey += v ? v : "";
      pkey += ';';
    }
    pkey += build_id();
    app(&gr, sizeof gr);
    app(p->ccs.ptr.data(), p->ccs.ptr.size() * sizeof(int32_t));
    app(p->ccs.idx.data(), p->ccs.idx.size() * sizeof(int32_t));
    app(p->ccs.val.data(), p->ccs.val.size() * sizeof(double));
    app(p->ccs.vim.data(), p->ccs.vim.size() * sizeof(double));
  }
  bool plan_hit = false;
  if (getenv("PERM_DEBUG_TIMING")) fprintf(stderr, "[timing] key %.3f ms\n", now_ms() - t0);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_plan_cache.find(pkey);
    if (it != g_plan_cache.end()) {
      const perm_opts keep = p->opts;
      *p = it->second;  // planning state only (device fields are empty in the cache)
      p->opts = keep;
      I.plan_cached = 1;
      plan_hit = true;
    }
  }
  // on-disk plan cache (opts.cache_dir, else $PERM_CACHE_DIR): planning output
  // of an earlier process with the same key (matrix content, options, build)
  std::string cache_file;
  {
    const char* dir = p->opts.cache_dir ? p->opts.cache_dir : getenv("PERM_CACHE_DIR");
    if (dir && *dir) {
      char nm[64];
      snprintf(nm, sizeof nm, "/perm-%016llx%016llx.plan", (unsigned long long)fnv1a64(pkey),
               (unsigned long long)fnv1a64(pkey, 0x84222325cbf29ce4ull));
      cache_file = std::string(dir) + nm;
    }
  }
  if (!plan_hit && !cache_file.empty()) {
    std::string blob;
    if (FILE* f = fopen(cache_file.c_str(), "rb")) {
      char buf[1 << 16];
      size_t got;
      while ((got = fread(buf, 1, sizeof buf, f)) > 0) blob.append(buf, got);
      fclose(f);
      std::string key;
      const perm_opts keep = p->opts;
      if (plan_deserialize(blob.data(), blob.size(), *p, &key) && key == pkey) {
        p->opts = keep;
        I.disk_cached = 1;
        plan_hit = true;
        std::lock_guard<std::mutex> lk(g_cache_mu);
        if (g_plan_cache.size() > 256) g_plan_cache.clear();
        g_plan_cache[pkey] = *p;
      }
    }
  }
  if (!plan_hit && p->singular) {
    // structural rank < n: perm = 0 exactly with no kernel; nothing to
    // order, eliminate or compile (an all-zero column would otherwise reach
    // the ordering and the generator)
    p->rowp.resize(n);
    p->colp.resize(n);
    for (int i = 0; i < n; ++i) {
      p->rowp[i] = p->colp[i] = i;
      I.row_perm[i] = I.col_perm[i] = i;
    }
    I.ordering = PERM_ORDER_NONE;
    I.K = 0;
    I.candidates_compiled = 0;
    I.w_alg1 = 0;
  }
  if (!plan_hit && !p->singular) {
    // search, candidates, NVRTC compiles, autotune: planner.cpp
    const int pst = plan_kernel(p, ord, gr, ctx_ready);
    if (pst != PERM_OK) return bail(pst);
    std::lock_guard<std::mutex> lk(g_cache_mu);
    if (g_plan_cache.size() > 256) g_plan_cache.clear();
    g_plan_cache[pkey] = *p;
  }
  if (!plan_hit && !p->singular && !cache_file.empty()) {  // atomic publish: write a temp file, rename
    const std::string blob = plan_serialize(*p, pkey);
    const std::string tmp = cache_file + ".tmp." + std::to_string((long long)getpid());
    if (FILE* f = fopen(tmp.c_str(), "wb")) {
      const bool ok = fwrite(blob.data(), 1, blob.size(), f) == blob.size();
      if (fclose(f) == 0 && ok) rename(tmp.c_str(), cache_file.c_str());
      else remove(tmp.c_str());
    }
  }
  I.plan_ms = now_ms() - t0;
  if (getenv("PERM_DEBUG_TIMING")) {
    double gms, pms;
    long long calls;
    codegen_timing(gms, pms, calls);
    fprintf(stderr, "[timing] planning %.3f ms (cached %d); generate_kernel %lld calls, %.1f ms summed (post-pass %.1f)\n",
            I.plan_ms, I.plan_cached, calls, gms, pms);
  }
  if (!p->opts.no_device) {
    if (ctx_ready.valid()) ctx_ready.wait();
    st = load_device(p);
    if (st != PERM_OK) return bail(st);
  }
  I.plan_ms = now_ms() - t0;
  *out = p;
  return PERM_OK;
}

extern "C" {

int perm_plan_ex(int n, perm_format fmt, const int32_t* ptr, const int32_t* idx, const double* val,
                 perm_ordering ord, const perm_opts* opts, perm_plan_t* out) {
  return plan_impl(n, fmt, ptr, idx, val, false, ord, opts, out);
}

int perm_plan_complex(int n, perm_format fmt, const int32_t* ptr, const int32_t* idx, const double* val_re_im,
                      perm_ordering ord, const perm_opts* opts, perm_plan_t* out) {
  return plan_impl(n, fmt, ptr, idx, val_re_im, true, ord, opts, out);
}

int perm_plan(int n, perm_format fmt, const int32_t* ptr, const int32_t* idx, const double* val,
              perm_ordering ord, perm_plan_t* out) {
  return perm_plan_ex(n, fmt, ptr, idx, val, ord, nullptr, out);
}

int perm_partial_bytes(perm_plan_t p) { return p ? (int)p->pbytes() : 8; }

int perm_shard_range(perm_plan_t p, int rank, int world, uint64_t* first_task, uint64_t* ntasks,
                     uint64_t* g_begin, uint64_t* g_end) {
  if (!p || !first_task || !ntasks || !g_begin || !g_end) return fail(PERM_EINVAL, "NULL argument");
  uint64_t first, count;
  int st = shard_range(p, rank, world, first, count);
  if (st) return st;
  *first_task = first;
  *ntasks = count;
  if (p->trivial1 || p->singular) {  // no sweep: rank 0 owns the whole range
    const uint64_t total = p->n >= 2 ? (1ull << (p->n - 1)) : 1;
    *g_begin = rank == 0 ? 0 : total;
    *g_end = total;
    return PERM_OK;
  }
  const uint64_t Lg = ((32ull * (uint64_t)p->info.M) << p->info.B) << p->info.K;  // Gray steps per task
  // small n: one task may span more lanes than the range has chunks (masked
  // lanes); the Gray range itself ends at 2^(n-1)
  const uint64_t total = 1ull << (p->n - 1);
  *g_begin = std::min(first * Lg, total);
  *g_end = std::min((first + count) * Lg, total);
  return PERM_OK;
}

double perm_fold_host(perm_plan_t p, const double* partials, int world) {
  if (!p || !partials || p->is_u128 || p->is_c128 || world < 1 || world > 65536 || (world & (world - 1))) {
    g_err = "perm_fold_host: real FP64 plan and power-of-two world <= 65536 required";
    return std::nan("");
  }
  if (p->singular) return 0.0;
  const int nn = p->trivial1 ? 1 : p->n;
  double st[20];  // same binary-counter pairwise tree as fold_f64 (reduce.cu)
  for (int k = 0; k < world; ++k) {
    double v = partials[k];
    int lvl = 0, kk = k;
    while (kk & 1) { v = st[lvl] + v; kk >>= 1; ++lvl; }
    st[lvl] = v;
  }
  int top = 0;
  while ((1 << top) < world) ++top;
  const double scale = ((nn % 2) ? 2.0 : -2.0) * ((p->info.K & 1) ? -1.0 : 1.0);
  return st[top] * scale;
}

int perm_compute_shard_async(perm_plan_t p, int rank, int world, void* d_partial) {
  if (!p) return fail(PERM_EINVAL, "plan is NULL");
  if (!p->on_device) return fail(PERM_ECUDA, "plan was created with no_device (no CPU fallback)");
  uint64_t first, count;
  int st = shard_range(p, rank, world, first, count);
  if (st) return st;
  CUDA_TRY(cudaSetDevice(p->device));
  const size_t pb = p->pbytes();
  if (p->trivial1 || p->singular) {
    // unscaled partial: singular -> 0.  n == 1: the fold scales by
    // 4(1 mod 2) - 2 = 2 (FP64) or shifts by n-1 = 0 (INT01), so the partial
    // is a00/2 resp. a00.
    unsigned char raw[16] = {0};
    if (p->trivial1 && rank == 0) {
      if (p->is_u128) { __int128 w = (long long)p->ccs.val[0]; std::memcpy(raw, &w, 16); }
      else {
        const double v[2] = {p->ccs.val[0] / 2.0, p->ccs.im(0) / 2.0};
        std::memcpy(raw, v, 16);
      }
    }
    CUDA_TRY(cudaMemcpyAsync(d_partial, raw, pb, cudaMemcpyHostToDevice, p->stream));
    p->last_count = 0;
    return PERM_OK;
  }
  st = run_range(p, first, count, nullptr, nullptr);
  if (st) return st;
  CUDA_TRY(cudaMemcpyAsync(d_partial, p->d_partial, pb, cudaMemcpyDeviceToDevice, p->stream));
  return PERM_OK;
}

int perm_compute_shard(perm_plan_t p, int rank, int world, perm_result* r) {
  if (!p || !r) return fail(PERM_EINVAL, "NULL argument");
  if (!p->on_device) return fail(PERM_ECUDA, "plan was created with no_device (no CPU fallback)");
  uint64_t first, count;
  int st = shard_range(p, rank, world, first, count);
  if (st) return st;
  CUDA_TRY(cudaSetDevice(p->device));
  double sm = 0, rm = 0;
  unsigned char raw[16] = {0};
  if (p->trivial1 || p->singular) {
    st = perm_compute_shard_async(p, rank, world, p->d_scratch);
    if (st) return st;
    CUDA_TRY(cudaMemcpyAsync(raw, p->d_scratch, 16, cudaMemcpyDeviceToHost, p->stream));
  } else {
    st = run_range(p, first, count, &sm, &rm);
    if (st) return st;
    CUDA_TRY(cudaMemcpyAsync(raw, p->d_partial, 16, cudaMemcpyDeviceToHost, p->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  fill_result(p, r, raw, false);
  r->world = world;
  r->rank = rank;
  {
    const uint64_t total = p->n >= 2 ? (1ull << (p->n - 1)) : 1;
    const uint64_t Lg = ((32ull * (uint64_t)p->info.M) << p->info.B) << p->info.K;
    const uint64_t g0 = std::min<uint64_t>(total, first * Lg);
    r->products = std::min<uint64_t>(total - g0, count * Lg);
  }
  r->steps = r->products;
  r->sweep_ms = sm;
  r->reduce_ms = rm;
  r->seconds = (sm + rm) * 1e-3;
  return PERM_OK;
}

int perm_fold_async(perm_plan_t p, const void* d_partials, int world, void* d_out) {
  if (!p) return fail(PERM_EINVAL, "plan is NULL");
  if (world < 1 || world > 65536 || (world & (world - 1)))
    return fail(PERM_EINVAL, "world must be a power of two <= 65536");
  CUDA_TRY(cudaSetDevice(p->device));
  const int nn = p->trivial1 ? 1 : p->n;
  CUDA_TRY(libperm_launch_fold(d_partials, world, nn, p->kind(), p->info.K & 1, d_out, p->stream));
  return PERM_OK;
}

int perm_fold(perm_plan_t p, const perm_result* shards, int world, perm_result* out) {
  if (!p || !shards || !out) return fail(PERM_EINVAL, "NULL argument");
  if (!p->on_device) return fail(PERM_ECUDA, "plan was created with no_device (no CPU fallback)");
  if (world < 1 || world > 65536 || (world & (world - 1)))
    return fail(PERM_EINVAL, "world must be a power of two <= 65536");
  if ((size_t)16 * world > p->scratch_bytes) {  // grow the fold scratch
    CUDA_TRY(cudaSetDevice(p->device));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    CUDA_TRY(cudaFree(p->d_scratch));
    p->scratch_bytes = (size_t)16 * world;
    CUDA_TRY(cudaMalloc(&p->d_scratch, p->scratch_bytes));
  }
  std::vector<unsigned char> raw(16 * world, 0);
  const size_t pb = p->pbytes();
  for (int k = 0; k < world; ++k) {
    if (p->is_u128) {
      std::memcpy(&raw[pb * k], &shards[k].exact_lo, 8);
      std::memcpy(&raw[pb * k + 8], &shards[k].exact_hi, 8);
    } else {
      std::memcpy(&raw[pb * k], &shards[k].value, 8);
      if (p->is_c128) std::memcpy(&raw[pb * k + 8], &shards[k].value_im, 8);
    }
  }
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaMemcpyAsync(p->d_scratch, raw.data(), pb * world, cudaMemcpyHostToDevice, p->stream));
  int st = perm_fold_async(p, p->d_scratch, world, p->d_partial);
  if (st) return st;
  unsigned char res[16];
  CUDA_TRY(cudaMemcpyAsync(res, p->d_partial, 16, cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  fill_result(p, out, res, true);
  if (p->singular) { out->value = 0.0; out->value_im = 0.0; out->exact_lo = out->exact_hi = 0; }
  out->world = world;
  out->products = p->n >= 2 ? (1ull << (p->n - 1)) : 1;
  for (int k = 0; k < world; ++k) {
    out->sweep_ms = std::max(out->sweep_ms, shards[k].sweep_ms);
    out->reduce_ms = std::max(out->reduce_ms, shards[k].reduce_ms);
  }
  return PERM_OK;
}

int perm_compute_async(perm_plan_t p, void* d_out) {
  if (!p || !d_out) return fail(PERM_EINVAL, "NULL argument");
  if (!p->on_device) return fail(PERM_ECUDA, "plan was created with no_device (no CPU fallback)");
  const int world = std::max(1, p->opts.world), rank = p->opts.world > 1 ? p->opts.rank : 0;
  if (world > 128) return fail(PERM_EINVAL, "world > 128");
  if (world > 1 && !p->opts.nccl_comm) return fail(PERM_EINVAL, "opts.world > 1 needs opts.nccl_comm");
  const size_t pb = p->pbytes();
  Nvtx range("perm_compute");
  CUDA_TRY(cudaSetDevice(p->device));
  // this rank's unscaled partial into its slot of the gather buffer
  char* gather = static_cast<char*>(p->d_scratch);
  int st = perm_compute_shard_async(p, rank, world, gather + (size_t)rank * pb);
  if (st) return st;
  if (p->opts.nccl_comm) {  // the path's one exchange step (in-place all-gather)
    std::string msg;
    Nvtx r("perm_allgather");
    st = libperm_allgather(p->opts.nccl_comm, gather, pb, rank, p->stream, msg);
    if (st) return fail(st, msg);
  }
  {
    Nvtx r("perm_fold");
    st = perm_fold_async(p, gather, world, d_out);
  }
  if (st) return st;
  CUDA_TRY(cudaEventRecord(p->ev[3], p->stream));
  return PERM_OK;
}

int perm_compute_ex(perm_plan_t p, perm_result* r) {
  if (!p || !r) return fail(PERM_EINVAL, "NULL argument");
  if (!p->on_device) return fail(PERM_ECUDA, "plan was created with no_device (no CPU fallback)");
  void* d_res = static_cast<char*>(p->d_partial) + 32;  // 16-byte result slot
  int st = perm_compute_async(p, d_res);
  if (st) return st;
  unsigned char raw[16];
  CUDA_TRY(cudaMemcpyAsync(raw, d_res, 16, cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  fill_result(p, r, raw, true);
  if (p->singular) { r->value = 0.0; r->value_im = 0.0; r->exact_lo = r->exact_hi = 0; }
  r->world = std::max(1, p->opts.world);
  r->rank = p->opts.world > 1 ? p->opts.rank : 0;
  r->products = r->steps = p->n >= 2 ? (1ull << (p->n - 1)) : 1;
  if (p->last_count > 0) {
    float a = 0, b = 0, c = 0;
    CUDA_TRY(cudaEventElapsedTime(&a, p->ev[0], p->ev[1]));
    CUDA_TRY(cudaEventElapsedTime(&b, p->ev[1], p->ev[2]));
    CUDA_TRY(cudaEventElapsedTime(&c, p->ev[0], p->ev[3]));
    r->sweep_ms = a;
    r->reduce_ms = b;
    r->seconds = c * 1e-3;
  }
  return PERM_OK;
}

double perm_compute(perm_plan_t p) {
  perm_result r;
  if (perm_compute_ex(p, &r) != PERM_OK) return std::nan("");
  return r.value;
}

int perm_compute_partial(perm_plan_t p, int rank, int world, double* partial) {
  if (!partial) return fail(PERM_EINVAL, "NULL argument");
  perm_result r;
  const int st = perm_compute_shard(p, rank, world, &r);
  if (st) return st;
  partial[0] = r.value;
  if (p->is_c128) partial[1] = r.value_im;
  return PERM_OK;
}

int perm_plan_export(perm_plan_t p, void* buf, size_t* size) {
  if (!p || !size) return fail(PERM_EINVAL, "NULL argument");
  const std::string blob = plan_serialize(*p, "export");
  if (buf && *size >= blob.size()) std::memcpy(buf, blob.data(), blob.size());
  *size = blob.size();
  return PERM_OK;
}

int perm_plan_import(const void* blob, size_t size, const perm_opts* opts, perm_plan_t* out) {
  if (!blob || !out) return fail(PERM_EINVAL, "NULL argument");
  *out = nullptr;
  const double t0 = now_ms();
  auto* p = new perm_plan_s();
  if (opts) p->opts = *opts;
  std::string key;
  if (!plan_deserialize(blob, size, *p, &key) || key != "export") {
    delete p;
    return fail(PERM_EINVAL, "perm_plan_import: not a plan blob of this libperm build");
  }
  p->info.disk_cached = 1;
  p->info.plan_cached = 0;
  if (!p->opts.no_device) {
    const int st = load_device(p);
    if (st != PERM_OK) {
      perm_free(p);
      return st;
    }
  }
  p->info.plan_ms = now_ms() - t0;
  *out = p;
  return PERM_OK;
}

int perm_comm_unique_id(void* id128) {
  if (!id128) return fail(PERM_EINVAL, "NULL argument");
  std::string msg;
  const int st = libperm_comm_unique_id(id128, msg);
  return st ? fail(st, msg) : PERM_OK;
}

int perm_comm_init(int world, int rank, const void* id128, int device, void** comm) {
  if (!id128 || !comm || world < 1 || rank < 0 || rank >= world) return fail(PERM_EINVAL, "bad arguments");
  std::string msg;
  const int st = libperm_comm_init(world, rank, id128, device, comm, msg);
  return st ? fail(st, msg) : PERM_OK;
}

int perm_comm_destroy(void* comm) {
  std::string msg;
  const int st = libperm_comm_destroy(comm, msg);
  return st ? fail(st, msg) : PERM_OK;
}

int perm_probe_fp64_peak(int device, double* lane_ops_per_s, double* ms) {
  if (!lane_ops_per_s) return fail(PERM_EINVAL, "NULL argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(PERM_ECUDA, "no such CUDA device (no CPU fallback)");
  double m = 0;
  CUDA_TRY(libperm_probe_fp64_peak(device, 5, lane_ops_per_s, &m));
  if (ms) *ms = m;
  return PERM_OK;
}

int perm_debug_task_partials(perm_plan_t p, void* host, uint64_t cap, uint64_t* count, uint64_t* first_task) {
  if (!p || !count) return fail(PERM_EINVAL, "NULL argument");
  if (!p->on_device) return fail(PERM_ECUDA, "plan has no device state");
  const uint64_t c = std::min(cap, p->last_count);
  const size_t pb = p->pbytes();
  if (c && host) {
    CUDA_TRY(cudaSetDevice(p->device));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    CUDA_TRY(cudaMemcpy(host, p->d_slots, c * pb, cudaMemcpyDeviceToHost));
  }
  *count = c;
  if (first_task) *first_task = p->last_first;
  return PERM_OK;
}

int perm_last_timing(perm_plan_t p, double* sweep_ms, double* reduce_ms) {
  if (!p || !sweep_ms || !reduce_ms) return fail(PERM_EINVAL, "NULL argument");
  *sweep_ms = *reduce_ms = 0;
  if (!p->on_device || p->last_count == 0) return PERM_OK;
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaEventSynchronize(p->ev[2]));
  float a = 0, b = 0;
  CUDA_TRY(cudaEventElapsedTime(&a, p->ev[0], p->ev[1]));
  CUDA_TRY(cudaEventElapsedTime(&b, p->ev[1], p->ev[2]));
  *sweep_ms = a;
  *reduce_ms = b;
  return PERM_OK;
}

int perm_plan_get_info(perm_plan_t p, perm_plan_info* info) {
  if (!p || !info) return fail(PERM_EINVAL, "NULL argument");
  *info = p->info;
  return PERM_OK;
}

const char* perm_plan_source(perm_plan_t p) { return p ? p->code.source.c_str() : ""; }

int perm_plan_cubin(perm_plan_t p, void* buf, size_t* size) {
  if (!p || !size) return fail(PERM_EINVAL, "NULL argument");
  const size_t need = p->cubin.size();
  if (buf && *size >= need) std::memcpy(buf, p->cubin.data(), need);
  *size = need;
  return PERM_OK;
}

void perm_free(perm_plan_t p) {
  if (!p) return;
  // release every device resource that exists, whether or not load_device
  // completed (a failed plan may hold a stream, events, buffers, a library)
  const bool any = p->stream || p->d_slots || p->d_counter || p->d_rscratch || p->d_partial || p->d_scratch ||
                   p->d_tier || p->lib_held || p->ev[0] || p->ev[1] || p->ev[2] || p->ev[3];
  if (any) {
    cudaSetDevice(p->device);
    if (p->stream) cudaStreamSynchronize(p->stream);
    pool_free(p->device, p->d_slots, p->slots_bytes);
    pool_free(p->device, p->d_counter, p->counter_bytes);
    pool_free(p->device, p->d_rscratch, p->rscratch_bytes);
    pool_free(p->device, p->d_partial, p->partial_bytes);
    if (p->d_scratch) {
      if (p->scratch_bytes == 16 * 128) pool_free(p->device, p->d_scratch, p->scratch_bytes);
      else cudaFree(p->d_scratch);  // grown by perm_fold with cudaMalloc
    }
    pool_free(p->device, p->d_tier, p->tier_alloc_bytes);
    for (auto& e : p->ev)
      if (e) cudaEventDestroy(e);
    if (p->lib_held) lib_release(p->device, p->lib_key);
    if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
  }
  delete p;
}

}  // extern "C"
