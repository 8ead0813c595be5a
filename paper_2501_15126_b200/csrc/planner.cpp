// planner.cpp -- the matrix-specific kernel planner behind perm_plan
// (DESIGN.md 3.6 column elimination, 3.13(f) spill policy, "Planner model"):
// base orderings (Alg. 3 / degree sort), the chunk
// geometry (Lemma 1), elimination searches scored on generated
// code, candidate ranking, NVRTC sm_100a compiles with the spill gate and its
// escalation ladder, on-device autotune, and the chosen plan's fields.
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "perm_internal.h"
#include "plan_state.h"
#include "rt_internal.h"

namespace perm {
namespace {

// Host cores for the planner's CPU work (codegen evaluations, NVRTC): the
// searches fan out into many std::async tasks (hundreds of threads at the
// widest beam step); each task holds one slot only while it computes, never
// while it waits on another task, so the slots bound the CPU contention
// without any risk of deadlock.
struct CpuSlots {
  std::mutex mu;
  std::condition_variable cv;
  int free_ = std::max(1u, std::thread::hardware_concurrency());
  void acquire() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return free_ > 0; });
    --free_;
  }
  void release() {
    { std::lock_guard<std::mutex> lk(mu); ++free_; }
    cv.notify_one();
  }
};
CpuSlots g_cpu_slots;
struct CpuSlot {
  CpuSlot() { g_cpu_slots.acquire(); }
  ~CpuSlot() { g_cpu_slots.release(); }
};

std::mutex g_cubin_mu;
std::map<std::string, std::pair<std::vector<char>, std::string>> g_cubin_cache;  // source -> (cubin, log)

int nvrtc_compile(const std::string& src, std::vector<char>& cubin, std::string& log, bool int128,
                  bool& cached, double& ms) {
  {
    std::lock_guard<std::mutex> lk(g_cubin_mu);
    auto it = g_cubin_cache.find(src);
    if (it != g_cubin_cache.end()) {
      cubin = it->second.first;
      log = it->second.second;
      cached = true;
      ms = 0;
      return PERM_OK;
    }
  }
  cached = false;
  double t0 = now_ms();
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "perm_sweep.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return fail(PERM_ENVRTC, "nvrtcCreateProgram failed");
  // --fmad=false: every arithmetic op the generator emits (and counts in
  // W_plan) is exactly one DADD/DMUL/DFMA; fusions are emitted explicitly.
  std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                                   "--ptxas-options=-v", "-default-device", "--fmad=false"};
  if (int128) opts.push_back("--device-int128");
  nvrtcResult r = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
  size_t ls = 0;
  nvrtcGetProgramLogSize(prog, &ls);
  log.assign(ls, '\0');
  if (ls) nvrtcGetProgramLog(prog, &log[0]);
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return fail(PERM_ENVRTC, std::string("NVRTC compile failed: ") + nvrtcGetErrorString(r) + "\n" + log);
  }
  size_t cs = 0;
  nvrtcGetCUBINSize(prog, &cs);
  cubin.resize(cs);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  ms = now_ms() - t0;
  std::lock_guard<std::mutex> lk(g_cubin_mu);
  g_cubin_cache[src] = {cubin, log};
  return PERM_OK;
}

// parse "Used N registers", "N bytes stack frame", "N bytes spill stores"
void parse_ptxas(const std::string& log, int& regs, int& stack, int& spill) {
  regs = stack = spill = -1;
  size_t p = log.find("Used ");
  if (p != std::string::npos) regs = atoi(log.c_str() + p + 5);
  p = log.find(" bytes stack frame");
  if (p != std::string::npos) {
    size_t b = log.rfind(' ', p - 1);
    stack = atoi(log.c_str() + b + 1);
  }
  p = log.find(" bytes spill stores");
  if (p != std::string::npos) {
    size_t b = log.rfind(' ', p - 1);
    spill = atoi(log.c_str() + b + 1);
  }
}

// Register count and stack frame of the kernel from the cubin itself (the
// .nv.info section's EIATTR_REGCOUNT / EIATTR_FRAME_SIZE entries).  NVRTC 12.9
// serves repeated compiles from the driver's cache without running ptxas, so
// the `-v` log can be empty on a GPU host: the spill gate must not depend on it.
bool cubin_attrs(const std::vector<char>& cub, int& regs, int& frame) {
  regs = frame = -1;
  auto rd = [&](size_t off, size_t n) -> uint64_t {
    uint64_t v = 0;
    if (off + n > cub.size()) return 0;
    std::memcpy(&v, cub.data() + off, n);
    return v;
  };
  if (cub.size() < 64 || std::memcmp(cub.data(), "\x7f" "ELF", 4) != 0 || cub[4] != 2) return false;
  const uint64_t shoff = rd(0x28, 8);
  const uint64_t shentsize = rd(0x3a, 2), shnum = rd(0x3c, 2), shstrndx = rd(0x3e, 2);
  if (shentsize < 64 || shstrndx >= shnum) return false;
  auto sh = [&](uint64_t i, size_t field, size_t n) { return rd(shoff + i * shentsize + field, n); };
  const uint64_t stroff = sh(shstrndx, 0x18, 8);
  for (uint64_t i = 0; i < shnum; ++i) {
    const uint64_t name = sh(i, 0, 4);
    if (stroff + name + 9 > cub.size() || std::strcmp(cub.data() + stroff + name, ".nv.info") != 0) continue;
    const uint64_t off = sh(i, 0x18, 8), size = sh(i, 0x20, 8);
    for (uint64_t q = off; q + 2 <= off + size && q + 2 <= cub.size();) {
      const int fmt = (unsigned char)cub[q], attr = (unsigned char)cub[q + 1];
      if (fmt == 0x04) {  // EIFMT_SVAL: u16 size, payload (u32 symbol, u32 value for these)
        const uint64_t len = rd(q + 2, 2);
        if (len >= 8) {
          const int val = (int)rd(q + 8, 4);
          if (attr == 0x2f) regs = std::max(regs, val);    // EIATTR_REGCOUNT
          if (attr == 0x11) frame = std::max(frame, val);  // EIATTR_FRAME_SIZE
        }
        q += 4 + len;
      } else if (fmt == 0x03) {
        q += 4;  // EIFMT_HVAL
      } else if (fmt == 0x02) {
        q += 4;  // EIFMT_BVAL (padded)
      } else {
        q += 2;  // EIFMT_NVAL
      }
    }
  }
  return regs >= 0;
}


// Ranked kernel candidate: base ordering x elimination prefix K x swept-column
// variant x chunk-bit cap x composite caches, scored W / eff(estimated blocks)
struct Cand { double score, w; int base, K, var, bcap, est; bool cc; int ev; double pskip; };

// One compiled candidate (or the reason it failed): its ordered matrix, spec,
// generated code and cubin.
struct Built {
  int status = PERM_OK;
  std::string err;
  bool ok = false;
  std::vector<int> rp, colp;
  Csx o;
  std::vector<double> xo;
  KernelSpec sp;
  uint64_t tasks = 0;
  KernelCode kc;
  std::vector<char> cubin;
  std::string log;
  int regs = -1;
  int spill = 0;  // bytes of local memory (stack frame / spill stores) the accepted kernel uses
  double nvrtc_ms = 0;
  bool cached = false;
  std::shared_ptr<Built> alt;  // with autotune: the first spill-free rung, measured beside a spilling pick
};
// measured seconds per Gray step of each compiled candidate on `device`:
// one launch over ~4 waves of warp-tasks strided across its whole task
// range (zero skipping depends on the high task bits); candidates are timed in
// interleaved rounds after a warm-up (clock ramp) and the minimum over the
// rounds is kept; < 0 on any CUDA error
struct Timed {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t k = nullptr;
  void *d_cnt = nullptr, *d_slots = nullptr, *d_tier = nullptr;
  uint64_t cnt = 0;
  int S = 0;
  unsigned grid = 0;
  bool ok = false;
};

// The planner for one plan (perm_plan_s) whose matrix is validated and
// structurally nonsingular and whose mode is set.  Phases (run()):
//   search()          elimination sequences per base ordering (DESIGN 3.6),
//                     scored on generated code, shared memo
//   rank_candidates() candidate kernels per sequence, ranked by the model
//                     W / eff(blocks per SM), pruned to the compile set
//   compile()         NVRTC sm_100a builds with the spill gate and its
//                     escalation ladder (DESIGN 3.13(f)), concurrently
//   choose()          model pick, optional on-device autotune, the plan's fields
class Planner {
 public:
  Planner(perm_plan_s* plan, perm_ordering ord, double gr, const std::shared_future<void>& ctx_ready);
  int run();

 private:
  struct Ok { double score; size_t ci; Built b; };

  // the chunk grid for a sweep over n-1-K h-bits: B, U, M and the task count
  // (Lemma 1 aligned chunks; DESIGN "Chunk grid").  Depends only on
  // (n, K, opts): identical on every rank, so shards are complete subtrees of
  // the same reduction tree
  uint64_t geometry(int K, KernelSpec& sp, int bcap) const;
  // HYBRID: tier split from Alg. 4's c on the candidate's ordered matrix
  // (columns 0..K-1 are eliminated, so swept bit b is column K+b), clamped to
  // [U, B] so the tier is touched only at block-boundary flips
  void set_hybrid(KernelSpec& sp, const Csx& o) const;
  // base orderings: Alg. 3 PermanentOrdering, degree sort, identity
  void order_with(int o, std::vector<int>& rp, std::vector<int>& cp) const;
  // Alg. 1 lines 1-5 (reading R1: the true a_{i,n-1})
  std::vector<double> make_x0(const Csx& o) const;
  // FP64-pipe efficiency vs resident 128-thread blocks per SM (1 warp per
  // SMSP each); calibrated on B200
  // (profiles/r1_calibration.md: 3 -> 2 blocks costs 0-5 %; 1 block ~ half)
  static double eff(int bps) { return bps >= 3 ? 1.0 : bps == 2 ? 0.95 : 0.55; }
  static int bps_of(int regs, int threads) {
    const int r8 = (std::max(regs, 16) + 7) / 8 * 8;
    return std::max(1, std::min(16, 65536 / (threads * r8)));
  }
  // INT01 zero tracking at warp-task level (extends Sec. VI-B): the
  // columns of a few even-degree plain rows go to the top swept positions
  // (bits >= B + 5, uniform over the 32 lanes of a warp-task), so those rows
  // are frozen and lane-uniform; whenever one of them is 0 (2y_r = sum of
  // +-1 over its columns balances), F == 0 on every lane and the warp skips
  // the chunk (generated `__all_sync(F == 0)`).  Rows placed only on
  // block-level bits [U, B) are lane-uniform too and constant within a block:
  // when one is 0, S_U == 0 on every lane and the existing block-level skip
  // drops the block.  The placement fills the top (chunk-skip) positions
  // first, then [U, B).  Returns the order and the skipped fraction of chunks.
  std::vector<int> zero_aware(const std::vector<int>& colp, int K, int B, int U, double& pskip);
  // swept order of a candidate: eliminated prefix, then var 0 = base order,
  // 1 = sorted by flip cost, 2/3 = zero-aware placements (INT01)
  std::vector<int> colp_of(const std::vector<int>& cp, const std::vector<int>& picks, int K, int var, int B = 0,
                           double* pskip = nullptr, int U = -1);
  // Elimination sequence per base ordering: greedy (or beam),
  // each step takes the candidate column whose elimination lowers the
  // generated code's exact FP64 op count per Gray step the most (evaluated on
  // a reduced geometry), until no candidate helps.
  std::vector<int> elimination_search(int base, const std::vector<int>& rp, const std::vector<int>& cp, int ev);
  std::vector<double> time_candidates(const std::vector<const Built*>& bs, const std::vector<double>& pskips,
                                      int device, bool wide);
  // one candidate: codegen + NVRTC with the spill gate and escalation
  Built build(const Cand& c);

  void search();
  void rank_candidates();
  int compile();
  int choose();

  perm_plan_s* p;
  const int n, mode;
  perm_plan_info& I;
  const perm_ordering ord;
  const double gr;
  const std::shared_future<void>& ctx_ready;

  // ---- knobs (DESIGN "Planner model"; env overrides for tuning experiments)
  double tc = 0;                 // planning start (codegen_ms)
  int kcap = 0;                  // longest elimination prefix searched
  std::vector<int> bases;        // base orderings
  std::vector<int> bcaps;        // chunk-bit caps of the candidates
  bool fp64_real = false;
  // spill tolerance (real FP64; INT01 under autotune only; complex strict).
  // B200, n=40 K=9 U=4: a 28-byte spill with 12 values in volatile shared
  // memory costs 3.8 % per DP instruction against a spill-free kernel, and
  // its 9 % lower W makes it 5 % faster (profiles/r2_xform_variants_spill.jsonl)
  int spill_ok = 0;
  bool smem_ro_rung = false;
  double spill_pen = 1.04;
  int smem_ro_uses = 6;
  bool will_autotune = false;
  bool cc_allowed = true;        // composite caches (DESIGN 3.12): candidates with and without
  int nvar = 1;                  // swept-column variants: 0 = base order, 1 = sorted by flip cost (AUTO only)
  std::vector<std::vector<int>> row_cols;
  int elim_cands = 6;
  int elim_maxsize = 96, elim_maxsize_big = 160, elim_maxsize_huge = 256, elim_maxsize_giant = 640;
  bool elim_tier4 = false;       // a fourth composite-bound tier (ev / 6 = 3)
  int giant_beam = 4;            // its beam width
  int elim_beam = 4;
  bool dbg_plan = false;
  int task_bits = 17;            // floor of the warp-task count, log2 (geometry)
  int score_b = 8;               // chunk-bit cap the elimination searches score at

  // ---- state shared by the phases
  // ev % 3: how the search scores a sequence -- 0: the kernel as planned
  // (U <= 4); 1: with Alg. 4's register/global split applied (FP64 only);
  // 2: U <= 3.  ev / 3: greedy or beam search.  The W landscape is rugged (a
  // greedy path can end far from the best, and a beam is not a superset of
  // the greedy path), so the sequences of every search become candidates.
  // W of a partial elimination sequence depends on (base ordering, scoring,
  // sequence) only -- not on the search kind or the composite bound -- so
  // the 18 searches per base share one memo (each sequence is generated once)
  std::mutex memo_mu;
  std::map<std::pair<int, std::vector<int>>, std::shared_future<double>> memo;
  std::atomic<int> memo_evals{0}, memo_hits{0};
  std::map<int, std::vector<int>> elim_of_base;  // key: base * 32 + ev
  std::vector<Cand> cands;
  std::vector<Ok> oks;
};

Planner::Planner(perm_plan_s* plan, perm_ordering ord_, double gr_, const std::shared_future<void>& ctx)
    : p(plan), n(plan->n), mode(plan->info.mode), I(plan->info), ord(ord_), gr(gr_), ctx_ready(ctx) {
  tc = now_ms();
  kcap = p->opts.factor_cols < 0 ? 0 : (p->opts.factor_cols > 0 ? p->opts.factor_cols : 16);
  if (p->singular || n < 3) kcap = 0;
  if (ord == PERM_ORDER_AUTO) bases = {PERM_ORDER_PERMANENT, PERM_ORDER_DEGREE};
  else bases = {(int)ord};
  bcaps = {12, 10, 8};
  if (p->opts.chunk_log2 > 0) bcaps = {p->opts.chunk_log2};
  fp64_real = mode == PERM_MODE_REG || mode == PERM_MODE_HYBRID;
  will_autotune = !p->opts.no_device && p->opts.autotune >= 0 &&
                  !(getenv("PERM_NO_AUTOTUNE") && atoi(getenv("PERM_NO_AUTOTUNE")));
  // INT01: spilling kernels only as measured candidates (autotune, beside
  // their spill-free rung).  B200, 0/1 ER n=40: the autotuned pick with a
  // spill (K=8 U=3) runs 9.9 ms against 12.7 ms spill-free, while the model
  // alone would pick a slower spilling kernel (16.1 ms, profiles/r2_spill_policy_ab.jsonl)
  const bool i01_measured = mode == PERM_MODE_INT01 && will_autotune;
  // real FP64 96 bytes: with the giant tier the n=40 plan's U-1 rung keeps an
  // 88-byte frame and runs 6.42 ms against 6.70 ms for its spill-free
  // smem_ro rung; no FP64 config was slower at 96 than at 64
  spill_ok = getenv("PERM_SPILL_OK") ? atoi(getenv("PERM_SPILL_OK")) : (fp64_real ? 96 : (i01_measured ? 64 : 0));
  spill_pen = mode == PERM_MODE_INT01 ? 1.3 : 1.04;
  smem_ro_rung = fp64_real && !(getenv("PERM_NO_SMEM_RO") && atoi(getenv("PERM_NO_SMEM_RO")) == 1);
  smem_ro_uses = getenv("PERM_SMEM_RO") ? std::max(1, atoi(getenv("PERM_SMEM_RO"))) : 6;
  cc_allowed = !(getenv("PERM_NO_CC") && atoi(getenv("PERM_NO_CC")) == 1);
  nvar = ord == PERM_ORDER_AUTO ? 2 : 1;
  row_cols.assign(n, {});
  for (int j = 0; j < n; ++j)
    for (int q = p->ccs.ptr[j]; q < p->ccs.ptr[j + 1]; ++q) row_cols[p->ccs.idx[q]].push_back(j);
  const bool cplx_mode = mode == PERM_MODE_COMPLEX_INTERNAL;
  elim_cands = getenv("PERM_ELIM_CANDS") ? atoi(getenv("PERM_ELIM_CANDS")) : 6;
  // complex values take 4 registers: halve the composite size bound
  elim_maxsize = getenv("PERM_ELIM_MAXSIZE") ? atoi(getenv("PERM_ELIM_MAXSIZE")) : (cplx_mode ? 40 : 96);
  // larger composite-bound tiers (ev / 6 = 1, 2): real (FP64, INT01) 160 / 256, complex 64 / 96
  elim_maxsize_big = cplx_mode ? 64 : 160;
  elim_maxsize_huge = cplx_mode ? 96 : 256;
  elim_maxsize_giant = cplx_mode ? 160 : 640;
  // real FP64: a fourth, "giant" composite tier (640 leaf evaluations; beam
  // searches with scorings 0 and 1 only).  B200, model picks: n=40 p=0.2
  // 7.50 -> 6.71 ms (K=9 U=4, W 0.2239 -> 0.1971), band n=44 0.99 -> 0.75 ms,
  // ER n=48 6.0 -> 5.4 s, n=40 seed 2 -14 %, n=36 seed 2 -12 %
  // (profiles/r2_spill_policy_ab.jsonl); it roughly doubles the search time
  elim_tier4 = getenv("PERM_ELIM_TIER4") ? atoi(getenv("PERM_ELIM_TIER4")) == 1 : fp64_real;
  giant_beam = getenv("PERM_GIANT_BEAM") ? std::max(1, atoi(getenv("PERM_GIANT_BEAM"))) : 4;
  // experiment knob: real FP64 tiers shifted up to 160 / 256 / 640
  if (fp64_real && getenv("PERM_ELIM_SHIFT") && atoi(getenv("PERM_ELIM_SHIFT")) == 1 && !getenv("PERM_ELIM_MAXSIZE")) {
    elim_maxsize = 160;
    elim_maxsize_big = 256;
    elim_maxsize_huge = 640;
  }
  // beam width of the elimination searches (FP64: 4, INT01 / complex: greedy)
  elim_beam = std::max(1, getenv("PERM_ELIM_BEAM") ? atoi(getenv("PERM_ELIM_BEAM")) : (cplx_mode ? 1 : 4));
  dbg_plan = getenv("PERM_DEBUG_PLAN") != nullptr;
  task_bits = getenv("PERM_TASK_BITS") ? atoi(getenv("PERM_TASK_BITS")) : 17;
  score_b = getenv("PERM_SCORE_B") ? atoi(getenv("PERM_SCORE_B")) : 8;
}

int Planner::run() {
  search();
  rank_candidates();
  const int st = compile();
  if (st != PERM_OK) return st;
  return choose();
}

uint64_t Planner::geometry(int K, KernelSpec& sp, int bcap) const {
  const int nb = std::max(0, n - 1 - K);  // h-bits
  // at least 2^17 warp-tasks when the range allows (B >= 8): >= 14 tasks per
  // resident warp on each of 8 GPUs keeps the dynamic-scheduling tail small
  const int btask = std::max(8, nb - 5 - task_bits);
  int B = p->opts.chunk_log2 > 0 ? p->opts.chunk_log2 : std::min(std::min(bcap, btask), std::max(0, nb - 5));
  // exact reseed interval (perm_opts.reseed_log2): every chunk is seeded
  // exactly from x0, so the interval caps the chunk length
  if (p->opts.reseed_log2 > 0) B = std::min(B, p->opts.reseed_log2);
  if (B > nb) B = nb;
  // INT01 keeps 128-bit products: a shorter unrolled block (fewer live
  // 4-register values, faster NVRTC)
  int U = p->opts.block_log2 > 0
              ? p->opts.block_log2
              : ((mode == PERM_MODE_INT01 || mode == PERM_MODE_COMPLEX_INTERNAL) ? 3 : 5);
  if (U > B) U = B;
  const uint64_t nchunks = 1ull << (nb - B);
  const uint64_t warp_chunks = std::max<uint64_t>(1, nchunks / 32);
  uint64_t M = p->opts.task_chunks > 0 ? (uint64_t)p->opts.task_chunks : 0;
  if (M == 0) {
    M = 1;
    while (warp_chunks / (M * 2) >= (1ull << task_bits)) M *= 2;
  }
  if (M > warp_chunks) M = warp_chunks;
  sp.n = n;
  sp.K = K;
  sp.B = B;
  sp.U = U;
  sp.M = (int)M;
  sp.mode = mode;
  sp.threads = p->opts.threads_per_block > 0 ? p->opts.threads_per_block : 128;
  sp.nchunks_total = nchunks;
  sp.zero_skip = mode == PERM_MODE_INT01 && p->opts.zero_skip >= 0;
  return warp_chunks / M;  // tasks
}

void Planner::set_hybrid(KernelSpec& sp, const Csx& o) const {
  if (mode != PERM_MODE_HYBRID) return;
  int cbits = p->opts.hybrid_c;
  if (cbits <= 0) {
    int k4, c4;
    partition_alg4(o, gr, 148, k4, c4);
    cbits = c4 - sp.K;
  }
  sp.hybrid_c = std::max(std::min(cbits, sp.B), std::min(sp.U, sp.B));
}

void Planner::order_with(int o, std::vector<int>& rp, std::vector<int>& cp) const {
  if (o == PERM_ORDER_PERMANENT) order_permanent(p->ccs, p->crs, rp, cp);
  else if (o == PERM_ORDER_DEGREE) order_degree(p->ccs, rp, cp);
  else { rp.resize(n); cp.resize(n); for (int i = 0; i < n; ++i) rp[i] = cp[i] = i; }
}

std::vector<double> Planner::make_x0(const Csx& o) const {
  Csx orr = transpose(o);
  const bool cpx = mode == PERM_MODE_COMPLEX_INTERNAL;
  std::vector<double> x0(cpx ? 2 * n : n);  // complex: (re, im) pairs
  for (int i = 0; i < n; ++i) {
    long double sum = 0, last = 0, sumi = 0, lasti = 0;
    for (int q = orr.ptr[i]; q < orr.ptr[i + 1]; ++q) {
      sum += orr.val[q];
      sumi += orr.im(q);
      if (orr.idx[q] == n - 1) { last = orr.val[q]; lasti = orr.im(q); }
    }
    if (cpx) {
      x0[2 * i] = (double)(last - sum / 2);
      x0[2 * i + 1] = (double)(lasti - sumi / 2);
    } else {
      x0[i] = mode == PERM_MODE_INT01 ? (double)(2 * last - sum) : (double)(last - sum / 2);
    }
  }
  return x0;
}

std::vector<int> Planner::zero_aware(const std::vector<int>& colp, int K, int B, int U, double& pskip) {
  pskip = 0;
  const int nb = n - 1 - K;
  const int top = std::max(0, nb - B - 5), mid = std::max(0, B - std::max(U, 0));
  if (top < 1) return colp;
  const int cap = std::min(top + mid, 31);
  const int last = colp[n - 1];
  std::set<int> elim(colp.begin(), colp.begin() + K);
  struct R { double pz; int r; };
  std::vector<R> rows;
  for (int r = 0; r < n; ++r) {
    const int d = (int)row_cols[r].size();
    if (d < 2 || (d & 1)) continue;
    bool ok = true, has_last = false;
    for (int c : row_cols[r]) { ok &= !elim.count(c); has_last |= c == last; }
    if (!ok) continue;
    // P(sum of the swept signs = -(last column's +1)) or P(sum = 0)
    const int m = has_last ? d - 1 : d, need = has_last ? d / 2 - 1 : d / 2;
    const double pz = std::exp(std::lgamma(m + 1.0) - std::lgamma(need + 1.0) - std::lgamma(m - need + 1.0) -
                               m * std::log(2.0));
    rows.push_back({pz, r});
  }
  std::stable_sort(rows.begin(), rows.end(), [](const R& a, const R& b) { return a.pz > b.pz; });
  std::set<int> chosen_cols;
  std::vector<int> chosen_order;  // priority: columns of the most zero-prone rows first
  double keep = 1.0;
  for (const R& x : rows) {
    std::set<int> u = chosen_cols;
    for (int c : row_cols[x.r]) if (c != last) u.insert(c);
    if ((int)u.size() > cap) continue;
    for (int c : row_cols[x.r])
      if (c != last && !chosen_cols.count(c)) chosen_order.push_back(c);
    chosen_cols.swap(u);
    keep *= 1.0 - x.pz;
  }
  if (chosen_cols.empty()) return colp;
  (void)keep;  // rows sharing columns are correlated: count the skipped fraction exactly
  {
    std::vector<int> cols(chosen_cols.begin(), chosen_cols.end());
    const int c = (int)cols.size();
    std::map<int, int> bit;
    for (int q = 0; q < c; ++q) bit[cols[q]] = q;
    std::vector<std::pair<uint32_t, int>> rm;  // (mask over chosen columns, +1 signs needed)
    for (const R& x : rows) {
      uint32_t m = 0;
      bool fits = true, has_last = false;
      for (int col : row_cols[x.r]) {
        if (col == last) { has_last = true; continue; }
        auto it = bit.find(col);
        if (it == bit.end()) { fits = false; break; }
        m |= 1u << it->second;
      }
      if (!fits) continue;
      const int d = __builtin_popcount(m) + (has_last ? 1 : 0);
      rm.push_back({m, d / 2 - (has_last ? 1 : 0)});  // #(+1) among the swept columns for a zero sum
    }
    uint64_t hit = 0, tot = 0;
    auto count = [&](uint32_t st) {
      ++tot;
      for (auto& q : rm)
        if (__builtin_popcount(st & q.first) == q.second) { ++hit; return; }
    };
    if (c <= 20) {
      for (uint32_t st = 0; st < (1u << c); ++st) count(st);
    } else {  // SplitMix64 sample of the column states
      uint64_t z = 0x9E3779B97F4A7C15ull;
      for (int q = 0; q < (1 << 20); ++q) {
        z += 0x9E3779B97F4A7C15ull;
        uint64_t v = z;
        v = (v ^ (v >> 30)) * 0xBF58476D1CE4E5B9ull;
        v = (v ^ (v >> 27)) * 0x94D049BB133111EBull;
        count((uint32_t)(v ^ (v >> 31)));
      }
    }
    pskip = tot ? (double)hit / (double)tot : 0.0;
  }
  // swept slots: chosen columns on the top positions, the rest of them on
  // [U, B) (highest first); the other columns keep their relative order
  std::vector<int> slot(nb, -1);
  const int ntop = std::min((int)chosen_order.size(), top);
  for (int q = 0; q < ntop; ++q) slot[nb - 1 - q] = chosen_order[q];
  for (int q = ntop; q < (int)chosen_order.size(); ++q) slot[B - 1 - (q - ntop)] = chosen_order[q];
  int w = 0;
  for (int q = K; q < n - 1; ++q) {
    if (chosen_cols.count(colp[q])) continue;
    while (slot[w] >= 0) ++w;
    slot[w] = colp[q];
  }
  std::vector<int> out(colp.begin(), colp.begin() + K);
  out.insert(out.end(), slot.begin(), slot.end());
  out.push_back(last);
  return out;
}

std::vector<int> Planner::colp_of(const std::vector<int>& cp, const std::vector<int>& picks, int K, int var, int B,
                                   double* pskip, int U) {
  std::vector<int> c = factored_columns(cp, picks, K);
  if (var >= 2) {  // zero-aware placement on the cost-sorted order (INT01); 3: also on [U, B)
    c = costsort_swept(p->ccs, c, K);
    double ps = 0;
    c = zero_aware(c, K, B, var == 3 ? U : B, ps);
    if (pskip) *pskip = ps;
    return c;
  }
  return var ? costsort_swept(p->ccs, c, K) : c;
}

std::vector<int> Planner::elimination_search(int base, const std::vector<int>& rp, const std::vector<int>& cp,
                                             int ev) {
  std::vector<int> seq;
  if (kcap == 0) return seq;
  auto evalW_raw = [&, ev](const std::vector<int>& s) {
    const int k = (int)s.size();
    std::vector<int> c = costsort_swept(p->ccs, factored_columns(cp, s, k), k);
    Csx o = permute_ccs(p->ccs, rp, c);
    KernelSpec sp;
    geometry(k, sp, score_b);
    const int sc = ev % 3;  // scoring; (ev / 3) % 2: greedy (0) or beam (1); ev / 6: composite bound tier
    sp.U = std::min(sp.U, sc == 2 ? 3 : 4);
    sp.cc = cc_allowed;
    set_hybrid(sp, o);
    if (sc == 1 && (mode == PERM_MODE_REG || mode == PERM_MODE_HYBRID)) {
      int k4, c4;
      partition_alg4(o, gr, 148, k4, c4);
      sp.mode = PERM_MODE_HYBRID;
      sp.hybrid_c = std::max(std::min(c4 - k, sp.B), std::min(sp.U, sp.B));
    }
    sp.w_only = true;
    CpuSlot slot;
    return generate_kernel(o, make_x0(o), sp).w_plan;
  };
  auto evalW = [&, base, ev](const std::vector<int>& s) {
    const std::pair<int, std::vector<int>> key{base * 4 + ev % 3, s};
    std::promise<double> pr;
    std::shared_future<double> f;
    bool owner = false;
    {
      std::lock_guard<std::mutex> lk(memo_mu);
      auto it = memo.find(key);
      if (it != memo.end()) {
        f = it->second;
      } else {
        f = pr.get_future().share();
        memo.emplace(key, f);
        owner = true;
      }
    }
    if (!owner) {
      ++memo_hits;
      return f.get();
    }
    ++memo_evals;
    const double v = evalW_raw(s);
    pr.set_value(v);
    return v;
  };
  // beam search (width 1 = greedy) over elimination sequences
  std::vector<std::pair<double, std::vector<int>>> beam = {{evalW(seq), seq}};
  std::pair<double, std::vector<int>> best = beam[0];
  while ((int)beam[0].second.size() < kcap && (int)beam[0].second.size() < n - 3) {
    const int k = (int)beam[0].second.size();
    std::vector<std::pair<std::vector<int>, std::future<double>>> jobs;  // evaluated concurrently
    std::set<std::vector<int>> seen;
    for (const auto& st : beam) {
      const std::vector<int>& s = st.second;
      std::vector<int> cand;
      std::vector<int> fc = factored_columns(cp, s, k);
      for (int q = k; q < n - 1 && (int)cand.size() < elim_cands; ++q) cand.push_back(fc[q]);
      std::vector<int> cs = costsort_swept(p->ccs, fc, k);
      for (int q = k, added = 0; q < n - 1 && added < elim_cands; ++q, ++added)
        if (std::find(cand.begin(), cand.end(), cs[q]) == cand.end()) cand.push_back(cs[q]);
      for (int c : cand) {
        std::vector<int> s2 = s;
        s2.push_back(c);
        std::vector<int> key = s2;
        std::sort(key.begin(), key.end());  // the elimination set decides the tree up to order
        if (!seen.insert(key).second) continue;
        // bound the composite factors' evaluation size (code size, registers)
        if (elim_eval_size(p->ccs, factored_columns(cp, s2, k + 1), k + 1) >
            (ev >= 18 ? elim_maxsize_giant
                      : (ev >= 12 ? elim_maxsize_huge : (ev >= 6 ? elim_maxsize_big : elim_maxsize))))
          continue;
        jobs.emplace_back(s2, std::async(std::launch::async, evalW, s2));
      }
    }
    std::vector<std::pair<double, std::vector<int>>> next;
    for (auto& j : jobs) next.push_back({j.second.get(), j.first});
    if (next.empty()) break;
    std::sort(next.begin(), next.end());
    if (!(next[0].first < best.first * 0.995)) break;  // no further gain
    best = next[0];
    const int width = (ev % 6) >= 3 ? (ev >= 18 ? giant_beam : elim_beam) : 1;
    if ((int)next.size() > width) next.resize(width);
    beam.swap(next);
  }
  return best.second;
}

std::vector<double> Planner::time_candidates(const std::vector<const Built*>& bs,
                                             const std::vector<double>& pskips, int device, bool wide) {
  std::vector<double> out(bs.size(), -1.0);
  std::vector<Timed> T(bs.size());
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int sms = 0;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    cudaGetLastError();
    return out;
  }
  for (size_t q = 0; q < bs.size(); ++q) {
    const Built& b = *bs[q];
    Timed& t = T[q];
    int bps = 0;
    if (b.tasks == 0 || b.cubin.empty()) continue;
    if (cudaLibraryLoadData(&t.lib, b.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
        cudaLibraryGetKernel(&t.k, t.lib, b.kc.name.c_str()) != cudaSuccess ||
        (b.kc.smem_bytes > 0 &&
         cudaFuncSetAttribute((const void*)t.k, cudaFuncAttributeMaxDynamicSharedMemorySize, b.kc.smem_bytes) !=
             cudaSuccess) ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, (const void*)t.k, b.sp.threads, b.kc.smem_bytes) !=
            cudaSuccess ||
        bps < 1)
      continue;
    const uint64_t grid = (uint64_t)bps * sms, warps = grid * b.sp.threads / 32;
    // one strided launch: tasks spread over the whole range (every task bit
    // varies); about four waves, one wave when tasks are long (> 2^27 Gray steps)
    const double task_gray = 32.0 * b.sp.M * std::ldexp(1.0, b.sp.B + b.sp.K);
    // zero-skip plans: most tasks are nearly free and the sample's makespan
    // is set by the few full ones, so it needs ~4 waves of *unskipped* tasks
    const double keep = std::max(0.02, 1.0 - pskips[q]);
    const uint64_t waves = task_gray > std::ldexp(1.0, 27) ? 1 : (uint64_t)std::ceil(4.0 / keep);
    t.cnt = 1;
    while (t.cnt * 2 <= std::min<uint64_t>(b.tasks, waves * warps)) t.cnt *= 2;
    t.S = 1;
    t.grid = (unsigned)std::min<uint64_t>(grid, (t.cnt * 32 + b.sp.threads - 1) / b.sp.threads);
    if (cudaMalloc(&t.d_cnt, 256) != cudaSuccess || cudaMalloc(&t.d_slots, t.cnt * (wide ? 16 : 8)) != cudaSuccess)
      continue;
    if (b.kc.tier_bytes > 0 &&
        cudaMalloc(&t.d_tier, (size_t)b.kc.tier_bytes * grid * b.sp.threads) != cudaSuccess)
      continue;
    t.ok = true;
  }
  auto launch = [&](size_t q, uint64_t first) {
    const Built& b = *bs[q];
    Timed& t = T[q];
    // odd stride: the sampled task indices vary in their low bits too (a
    // power-of-two stride pins them, biasing the zero-skip rate); indices
    // past the range wrap in the seed (bits >= n-1-K are ignored): valid states
    unsigned long long tb = first, stride = (b.tasks / t.cnt) | 1ull;
    unsigned tc = (unsigned)t.cnt;
    void* args[] = {&tb, &tc, &stride, &t.d_cnt, &t.d_slots, &t.d_tier};
    cudaMemsetAsync(t.d_cnt, 0, 4, st);
    return cudaLaunchKernel((const void*)t.k, dim3(t.grid), dim3(b.sp.threads), args, (size_t)b.kc.smem_bytes,
                            st);
  };
  auto sample = [&](size_t q) -> double {  // seconds per Gray step of one round
    const Built& b = *bs[q];
    Timed& t = T[q];
    bool okl = cudaEventRecord(e0, st) == cudaSuccess;
    for (int i = 0; i < t.S && okl; ++i) okl = launch(q, (b.tasks / t.S) * i / t.cnt * t.cnt) == cudaSuccess;
    okl = okl && cudaEventRecord(e1, st) == cudaSuccess && cudaEventSynchronize(e1) == cudaSuccess;
    float ms = 0;
    if (!okl || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess) return -1.0;
    return ms * 1e-3 / ((double)t.S * t.cnt * 32.0 * b.sp.M * std::ldexp(1.0, b.sp.B + b.sp.K));
  };
  // warm-up (module load, clock ramp); a candidate whose sample already
  // takes > 50 ms (large n: long tasks) keeps that single measurement
  std::vector<char> long_sample(bs.size(), 0);
  for (size_t q = 0; q < bs.size(); ++q) {
    if (!T[q].ok) continue;
    const auto t0 = std::chrono::steady_clock::now();
    const double v = sample(q);
    if (v < 0) { T[q].ok = false; continue; }
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > 0.05) {
      long_sample[q] = 1;
      out[q] = v;
    }
  }
  for (int round = 0; round < 3; ++round)
    for (size_t q = 0; q < bs.size(); ++q) {
      if (!T[q].ok || long_sample[q]) continue;
      const double v = sample(q);
      if (v < 0) { T[q].ok = false; out[q] = -1.0; continue; }
      out[q] = out[q] < 0 ? v : std::min(out[q], v);
    }
  cudaGetLastError();
  for (Timed& t : T) {
    if (t.d_cnt) cudaFree(t.d_cnt);
    if (t.d_slots) cudaFree(t.d_slots);
    if (t.d_tier) cudaFree(t.d_tier);
    if (t.lib) cudaLibraryUnload(t.lib);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  return out;
}

Built Planner::build(const Cand& c) {
  Built b;
  std::vector<int> cp;
  order_with(c.base, b.rp, cp);
  b.tasks = geometry(c.K, b.sp, c.bcap);
  b.colp = colp_of(cp, elim_of_base.at(c.base * 32 + c.ev), c.K, c.var, b.sp.B, nullptr, b.sp.U);
  b.o = permute_ccs(p->ccs, b.rp, b.colp);
  b.xo = make_x0(b.o);
  b.sp.cc = c.cc;
  b.sp.i01_asm_mul = getenv("PERM_ASM_MUL") && atoi(getenv("PERM_ASM_MUL")) == 1;
  if (smem_ro_rung && getenv("PERM_SMEM_RO_FORCE") && atoi(getenv("PERM_SMEM_RO_FORCE")) == 1)
    b.sp.smem_ro = smem_ro_uses;  // tests: the rung's placement from the first attempt
  set_hybrid(b.sp, b.o);
  if (n == 1 || p->singular) { b.ok = true; return b; }
  // start at <= 255 registers (2 blocks/SM: the FP64 pipe is already ~95 %
  // busy there); 3 blocks only for clearly small kernels
  {
    KernelSpec se = b.sp;
    se.w_only = true;
    const int est = generate_kernel(b.o, b.xo, se).est_regs;
    b.sp.min_blocks = p->opts.min_blocks > 0 ? p->opts.min_blocks : std::min(2, bps_of(est + 16, b.sp.threads));
    // the estimate misses the composite-evaluation temporaries of
    // eliminated columns: measured, every K > 0 kernel with est >= 100
    // spilled hundreds of bytes at the 168-register cap, while K = 0
    // kernels up to est 102 fit (n = 24-44, ER / band)
    if (p->opts.min_blocks <= 0 && est + 16 <= 152 && (c.K == 0 || est <= 90)) b.sp.min_blocks = 3;
  }
  // escalation ladder on a spill: a larger register cap (only steps that
  // really raise the __launch_bounds__ cap), then a shorter unrolled block,
  // then fewer chunk bits
  auto reg_cap = [](int mb, int threads) { return std::min(255, 65536 / (threads * std::max(mb, 1)) / 8 * 8); };
  auto escalate = [&](KernelSpec& sp, uint64_t& tasks) -> bool {
    const int cap0 = reg_cap(sp.min_blocks, sp.threads);
    while (sp.min_blocks > 1) {
      --sp.min_blocks;
      if (reg_cap(sp.min_blocks, sp.threads) > cap0) return true;
    }
    // real FP64: body-read-only values with few body uses into volatile
    // shared memory (DESIGN 3.13(f)) before giving up unrolled steps
    if (smem_ro_rung && sp.smem_ro == 0 && sp.U >= 3) { sp.smem_ro = smem_ro_uses; return true; }
    if (sp.U > 2) { --sp.U; sp.smem_ro = 0; return true; }
    if (sp.B > 2 && p->opts.chunk_log2 == 0) {
      sp.smem_ro = 0;
      const int keepU = sp.U;  // geometry() keeps min_blocks
      tasks = geometry(c.K, sp, sp.B - 2);
      set_hybrid(sp, b.o);
      sp.U = std::min(keepU, sp.B);
      return true;
    }
    return false;
  };
  struct Att {
    KernelSpec sp;
    uint64_t tasks = 0;
    KernelCode kc;
    std::vector<char> cubin;
    std::string log, err;
    int status = PERM_OK, regs = -1, stack = 0, spill = 0;
    double ms = 0;
    bool cached = false;
  };
  auto attempt = [&](const KernelSpec& sp, uint64_t tasks) {
    Att t;
    t.sp = sp;
    t.tasks = tasks;
    CpuSlot slot;
    t.kc = generate_kernel(b.o, b.xo, sp);
    t.status = nvrtc_compile(t.kc.source, t.cubin, t.log, p->is_u128, t.cached, t.ms);
    if (t.status != PERM_OK) { t.err = g_err; return t; }
    parse_ptxas(t.log, t.regs, t.stack, t.spill);
    int cr = -1, cf = -1;  // authoritative: the cubin's own attributes (the log may be empty, see cubin_attrs)
    if (cubin_attrs(t.cubin, cr, cf)) {
      t.regs = cr;
      t.stack = std::max(t.stack, cf);
      if (cf > 0) t.spill = std::max(t.spill, cf);
    }
    if (getenv("PERM_DEBUG_PLAN"))
      fprintf(stderr, "[plan]   attempt K %d B %d U %d minb %d cc %d ro %d: regs %d stack %d spill %d w %.5f est %d\n",
              c.K, sp.B, sp.U, sp.min_blocks, (int)sp.cc, sp.smem_ro, t.regs, t.stack, t.spill, t.kc.w_plan,
              t.kc.est_regs);
    return t;
  };
  auto take_into = [](Built& d, Att& t) {
    d.spill = std::max(t.stack, t.spill);
    d.sp = t.sp;
    d.tasks = t.tasks;
    d.kc = std::move(t.kc);
    d.cubin = std::move(t.cubin);
    d.log = std::move(t.log);
    d.regs = t.regs;
    d.cached = t.cached;
  };
  auto take = [&](Att& t) { take_into(b, t); };
  // a small spill is accepted (real FP64: spill_ok bytes per thread, an
  // L1-resident local frame; measured on B200, DESIGN 3.13(f)), scored
  // with spill_pen below
  auto clean = [&](const Att& t) {
    return (t.stack <= spill_ok && t.spill <= spill_ok) || getenv("PERM_ALLOW_SPILL");
  };
  // the first rungs compile concurrently (speculatively); the first
  // accepted rung in ladder order wins -- the same choice as compiling
  // them one after another, in one compile latency.  Real FP64 speculates
  // four (U, U + smem_ro, U-1, U-1 + smem_ro: the n=40 bench plan is taken
  // at the fourth), other modes two (the first spill-free rung was the
  // first or second in every measured plan)
  std::vector<std::pair<KernelSpec, uint64_t>> ladder = {{b.sp, b.tasks}};
  const size_t spec_rungs = getenv("PERM_LADDER_RUNGS") ? (size_t)std::max(1, atoi(getenv("PERM_LADDER_RUNGS")))
                                                        : (smem_ro_rung ? 4 : 2);
  while (ladder.size() < spec_rungs) {
    auto nx = ladder.back();
    if (!escalate(nx.first, nx.second)) break;
    ladder.push_back(nx);
  }
  std::vector<std::future<Att>> fa;
  for (auto& rung : ladder) fa.push_back(std::async(std::launch::async, attempt, rung.first, rung.second));
  std::vector<Att> done;
  for (auto& f : fa) done.push_back(f.get());
  for (Att& t : done) {
    b.nvrtc_ms += t.ms;
    if (t.status != PERM_OK) { b.status = t.status; b.err = t.err; return b; }
  }
  for (size_t q = 0; q < done.size(); ++q)
    if (clean(done[q])) {
      // a tolerated spill: with autotune, the first spill-free rung
      // compiled speculatively is measured beside it
      if (will_autotune && std::max(done[q].stack, done[q].spill) > 0)
        for (size_t r = q + 1; r < done.size(); ++r)
          if (done[r].stack <= 0 && done[r].spill <= 0) {
            b.alt = std::make_shared<Built>();
            b.alt->rp = b.rp; b.alt->colp = b.colp; b.alt->o = b.o; b.alt->xo = b.xo;
            take_into(*b.alt, done[r]);
            b.alt->ok = true;
            break;
          }
      take(done[q]);
      b.ok = true;
      return b;
    }
  KernelSpec sp = ladder.back().first;
  uint64_t tasks = ladder.back().second;
  for (int more = 0; more < 24 && escalate(sp, tasks); ++more) {
    Att t = attempt(sp, tasks);
    b.nvrtc_ms += t.ms;
    if (t.status != PERM_OK) { b.status = t.status; b.err = t.err; return b; }
    if (clean(t)) { take(t); b.ok = true; return b; }
  }
  take(done.back());  // every rung spilled: b.ok stays false
  return b;
}

void Planner::search() {
  const bool fp64 = mode == PERM_MODE_REG || mode == PERM_MODE_HYBRID;
  // ev = scoring (ev % 3) x search (ev / 3: greedy, beam of width elim_beam)
  // FP64 also repeats every search with larger composite bounds (160 and 256
  // leaf evaluations): larger composites win on some matrices and lose on others
  const bool tiers = !getenv("PERM_ELIM_MAXSIZE");  // every mode: FP64, INT01, complex
  const int nev = getenv("PERM_ELIM_VARIANTS") ? std::max(1, atoi(getenv("PERM_ELIM_VARIANTS")))
                                                : (tiers ? (elim_tier4 ? 24 : 18) : 6);
  {
    Nvtx r_search("perm_plan/search");
    std::vector<std::pair<int, std::future<std::vector<int>>>> runs;  // greedy runs, concurrently
    for (int base : bases)
      for (int ev = 0; ev < nev; ++ev) {
        if (ev % 3 == 1 && !fp64) continue;
        if ((ev / 3) % 2 == 1 && elim_beam == 1) continue;  // greedy only: the beam run would repeat it
        // the giant composite tier (ev 18-23) only as beam searches with
        // scorings 0 and 1 (ev 21, 22): every measured winner of that tier
        // came from them, and its searches are the most expensive
        if (ev >= 18 && ev != 21 && ev != 22 && !(getenv("PERM_ELIM_TIER4_ALL") && atoi(getenv("PERM_ELIM_TIER4_ALL")) == 1))
          continue;
        runs.emplace_back(base * 32 + ev, std::async(std::launch::async, [&, base, ev] {
                            std::vector<int> rp, cp;
                            order_with(base, rp, cp);
                            return elimination_search(base, rp, cp, ev);
                          }));
      }
    for (auto& r : runs) elim_of_base[r.first] = r.second.get();
  }
  if (getenv("PERM_DEBUG_TIMING"))
    fprintf(stderr, "[timing] elimination searches %.3f ms (%zu; %d evaluations, %d memo hits)\n", now_ms() - tc,
            elim_of_base.size(), memo_evals.load(), memo_hits.load());
}

void Planner::rank_candidates() {
  // candidates per distinct sequence, generated concurrently and merged in
  // sequence order (deterministic)
  std::vector<std::future<std::vector<Cand>>> cjobs;
  for (auto& be : elim_of_base) {
    const int base = be.first / 32, ev = be.first % 32;
    const std::vector<int>& picks = be.second;
    bool dup = false;  // the same sequence found under another scoring
    for (auto& o2 : elim_of_base)
      if (o2.first < be.first && o2.first / 32 == base && o2.second == picks) dup = true;
    if (dup) continue;
    cjobs.push_back(std::async(std::launch::async, [&, base, ev]() {  // picks: map element, stable
    std::vector<Cand> cands;
    std::vector<int> rp, cp;
    order_with(base, rp, cp);
    const int kmax = (int)picks.size();
    const int kmin = p->opts.factor_cols > 0 ? kmax : std::max(0, kmax - 2);
    // K in [kmax-2, kmax], plus the plain sweep K = 0 from the first search
    // (intermediate K never ranks near the top: W falls steeply with K)
    std::vector<int> Ks;
    if (ev == 0 && kmin > 0) Ks.push_back(0);
    for (int K = kmin; K <= kmax; ++K) Ks.push_back(K);
    for (int K : Ks)
      for (int var = 0; var < nvar + (mode == PERM_MODE_INT01 && p->opts.zero_skip >= 0 ? 2 : 0); ++var) {
        const int vv = var < nvar ? var : 2 + (var - nvar);
        Csx o = permute_ccs(p->ccs, rp, colp_of(cp, picks, K, vv));
        std::vector<double> xo = make_x0(o);
        std::set<int> seenB;
        for (int bc : bcaps) {
          KernelSpec sp;
          geometry(K, sp, bc);
          set_hybrid(sp, o);
          if (!seenB.insert(sp.B).second) continue;  // cap not binding: duplicate
          double pskip = 0;
          if (vv >= 2) {  // the placement depends on B (and U)
            o = permute_ccs(p->ccs, rp, colp_of(cp, picks, K, vv, sp.B, &pskip, sp.U));
            xo = make_x0(o);
            if (pskip <= 0) continue;
          }
          for (int ccv = 0; ccv < (K > 0 && cc_allowed ? 2 : 1); ++ccv) {
            sp.cc = ccv == 1;
            sp.w_only = true;
            KernelCode kc;
            {
              CpuSlot slot;
              kc = generate_kernel(o, xo, sp);
            }
            // estimates above the 255-register cap are optimistic-capped: ptxas
            // usually fits them (2 blocks of 128); the spill gate escalates if not
            const double score =
                kc.w_plan * (1.0 - pskip) / eff(bps_of(std::min(kc.est_regs, 255), sp.threads));
            cands.push_back({score, kc.w_plan, base, K, vv, bc, kc.est_regs, sp.cc, ev, pskip});
          }
        }
      }
    return cands;
    }));
  }
  for (auto& j : cjobs) {
    std::vector<Cand> part = j.get();
    cands.insert(cands.end(), part.begin(), part.end());
  }
  std::stable_sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) { return a.score < b.score; });
  if (getenv("PERM_DEBUG_TIMING")) fprintf(stderr, "[timing] candidates %.3f ms (%zu)\n", now_ms() - tc, cands.size());
  if (dbg_plan)
    for (const Cand& c : cands)
      fprintf(stderr, "[plan] cand score %.5f w %.5f base %d K %d var %d bcap %d est %d cc %d pskip %.3f ev %d\n", c.score, c.w,
              c.base, c.K, c.var, c.bcap, c.est, (int)c.cc, c.pskip, c.ev);
  {  // the top ncomp by model score, plus the best of every swept-order
     // variant not among them (the model's skip / occupancy estimates are
     // rough; autotune compares the variants on the device)
    const size_t ncomp = getenv("PERM_PLAN_COMPILES") ? (size_t)atoi(getenv("PERM_PLAN_COMPILES")) : 3;
    std::vector<Cand> keep;
    std::set<int> vars;
    for (size_t q = 0; q < cands.size(); ++q)
      if (q < ncomp) {
        keep.push_back(cands[q]);
        vars.insert(cands[q].var);
      }
    for (size_t q = ncomp; q < cands.size() && keep.size() < ncomp + 3; ++q)
      if (vars.insert(cands[q].var).second) keep.push_back(cands[q]);
    // one fewer eliminated column than the favourite: bigger composites need
    // more registers than the estimate says, and when the favourite has to
    // drop to a small U, K-1 at a larger U can be faster (autotune decides)
    if (!keep.empty() && keep[0].K > 0) {
      bool have_km1 = false;
      for (const Cand& k2 : keep) have_km1 |= k2.K == keep[0].K - 1;
      for (size_t q = ncomp; q < cands.size() && !have_km1; ++q)
        if (cands[q].K == keep[0].K - 1) {
          keep.push_back(cands[q]);
          have_km1 = true;
        }
    }
    // zero-aware placements (INT01): the skip model is the roughest, so the
    // two best of each such variant (B changes the placed columns) get measured
    for (int zv = 2; zv <= 3; ++zv) {
      int have_v = 0;
      for (const Cand& c : keep) have_v += c.var == zv;
      for (size_t q = 0; q < cands.size() && have_v < 2 && keep.size() < ncomp + 5; ++q) {
        const Cand& c = cands[q];
        if (c.var != zv) continue;
        bool dup = false;
        for (const Cand& k2 : keep)
          dup |= k2.var == c.var && k2.K == c.K && k2.bcap == c.bcap && k2.base == c.base && k2.ev == c.ev &&
                 k2.cc == c.cc;
        if (dup) continue;
        bool same_geo = false;  // prefer a different B (a different placement) for the second
        for (const Cand& k2 : keep) same_geo |= k2.var == zv && k2.bcap == c.bcap;
        if (same_geo && have_v > 0) continue;
        keep.push_back(c);
        ++have_v;
      }
    }
    cands.swap(keep);
  }
  if (p->singular || n == 1) cands.resize(std::min<size_t>(cands.size(), 1));
}

int Planner::compile() {
  const double t_compile0 = now_ms();
  I.codegen_ms = t_compile0 - tc;
  auto nvrtc_range = std::make_unique<Nvtx>("perm_plan/nvrtc");  // popped below or on an early return
  std::vector<std::future<Built>> fut;  // candidates compiled concurrently (NVRTC is thread-safe)
  for (const Cand& c : cands) fut.push_back(std::async(std::launch::async, [this](const Cand& cc) { return build(cc); }, c));
  for (size_t ci = 0; ci < cands.size(); ++ci) {
    if (ci + 1 == cands.size() && oks.empty() && cands[ci].K > 0 && fut.size() == cands.size()) {
      // every elimination candidate spilled: fall back to the plain sweep (K = 0)
      Cand plain = cands[ci];
      plain.K = 0;
      plain.var = 0;
      plain.pskip = 0;
      cands.push_back(plain);
      fut.push_back(std::async(std::launch::async, [this](const Cand& cc) { return build(cc); }, plain));
    }
    Built b = fut[ci].get();
    const Cand& c = cands[ci];
    if (b.status != PERM_OK) {
      for (size_t cj = ci + 1; cj < cands.size(); ++cj) fut[cj].wait();
      g_err = b.err;
      return (b.status);
    }
    I.nvrtc_cpu_ms += b.nvrtc_ms;
    if (!b.ok) continue;
    const double score = (n == 1 || p->singular)
                             ? 0.0
                             : b.kc.w_plan * (1.0 - c.pskip) / eff(bps_of(b.regs, b.sp.threads)) *
                                   ((b.spill > 0 || b.sp.smem_ro > 0) ? spill_pen : 1.0);
    if (dbg_plan)
      fprintf(stderr, "[plan] built K %d B %d U %d minb %d regs %d spill %d ro %d w %.5f score %.5f ok %d\n", c.K,
              b.sp.B, b.sp.U, b.sp.min_blocks, b.regs, b.spill, b.sp.smem_ro, b.kc.w_plan, score, (int)b.ok);
    std::shared_ptr<Built> alt = std::move(b.alt);
    oks.push_back({score, ci, std::move(b)});
    if (alt) {
      const double sa = alt->kc.w_plan * (1.0 - c.pskip) / eff(bps_of(alt->regs, alt->sp.threads));
      if (dbg_plan)
        fprintf(stderr, "[plan] built (spill-free alternative) K %d B %d U %d regs %d w %.5f score %.5f\n", c.K,
                alt->sp.B, alt->sp.U, alt->regs, alt->kc.w_plan, sa);
      oks.push_back({sa, ci, std::move(*alt)});
    }
  }
  I.nvrtc_ms = now_ms() - t_compile0;
  nvrtc_range.reset();
  if (getenv("PERM_DEBUG_TIMING")) fprintf(stderr, "[timing] compiles %.3f ms (%zu)\n", now_ms() - tc, oks.size());
  return PERM_OK;
}

int Planner::choose() {
  bool have = false;
  // model choice; then, with a device, measured choice (autotune): each
  // compiled candidate sweeps a few spread samples of its task range, and
  // replaces the model's pick only when it is clearly faster per Gray step
  // (> 4 %), so near-ties stay deterministic across ranks
  size_t pick = 0;
  for (size_t q = 1; q < oks.size(); ++q)
    if (oks[q].score < oks[pick].score) pick = q;
  const bool measured = !p->opts.no_device && p->opts.autotune >= 0 &&
                        !(getenv("PERM_NO_AUTOTUNE") && atoi(getenv("PERM_NO_AUTOTUNE")));
  // INT01 with on-device autotune: the model's pick also with the
  // hand-scheduled int x u128 multiply (DESIGN 3.9) -- same spec, one more
  // compile.  It wins on some kernels (0/1 ER n=40: 14.6 -> 12.8 ms) and
  // loses on others (0/1 band n=44: 1.22 -> 1.31 ms), which only a
  // measurement tells apart; the model pick alone keeps nvcc's multiply.
  if (mode == PERM_MODE_INT01 && measured && !oks.empty() && !oks[pick].b.sp.i01_asm_mul &&
      !getenv("PERM_NO_ASM_MUL")) {
    Ok alt{oks[pick].score, oks[pick].ci, oks[pick].b};
    Built& b = alt.b;
    b.sp.i01_asm_mul = true;
    {
      CpuSlot slot;
      b.kc = generate_kernel(b.o, b.xo, b.sp);
    }
    double ms = 0;
    bool cached = false;
    b.cubin.clear();
    if (nvrtc_compile(b.kc.source, b.cubin, b.log, p->is_u128, cached, ms) == PERM_OK) {
      int regs = -1, stack = 0, spill = 0, cr = -1, cf = -1;
      parse_ptxas(b.log, regs, stack, spill);
      if (cubin_attrs(b.cubin, cr, cf)) {
        regs = cr;
        stack = std::max(stack, cf);
        spill = std::max(spill, cf);
      }
      I.nvrtc_cpu_ms += ms;
      if (stack <= 0 && spill <= 0) {
        b.regs = regs;
        b.cached = cached;
        oks.push_back(std::move(alt));
      }
    }
  }
  if (oks.size() > 1 && measured) {
    std::vector<const Built*> bs;
    std::vector<double> pskips;
    for (const Ok& o : oks) {
      bs.push_back(&o.b);
      pskips.push_back(cands[o.ci].pskip);
    }
    if (ctx_ready.valid()) ctx_ready.wait();
    const double t_at0 = now_ms();
    const std::vector<double> t = time_candidates(bs, pskips, p->opts.device, p->is_u128 || p->is_c128);
    I.autotune_ms = now_ms() - t_at0;
    if (t[pick] > 0) {
      size_t best = pick;
      for (size_t q = 0; q < oks.size(); ++q)
        if (t[q] > 0 && t[q] < t[best]) best = q;
      if (best != pick && t[best] < 0.96 * t[pick]) pick = best;
    }
    if (dbg_plan)
      for (size_t q = 0; q < oks.size(); ++q)
        fprintf(stderr, "[plan] autotune cand %zu: %.4g s per 2^30 Gray steps%s\n", q, t[q] * 1073741824.0,
                q == pick ? " <- pick" : "");
  }
  if (!oks.empty()) {
    const Built& b = oks[pick].b;
    const Cand& c = cands[oks[pick].ci];
    have = true;

    p->rowp = b.rp; p->colp = b.colp; p->occs = b.o; p->spec = b.sp;
    p->code = b.kc; p->cubin = b.cubin; p->ptxas_log = b.log;
    I.ordering = c.base; I.tasks = b.tasks; I.K = c.K; I.swept_order = c.var;
    I.regs_per_thread = b.regs;
    I.local_bytes = b.spill;
    I.cubin_cached = b.cached;
  }
  if (!have) {
    g_err = "every candidate kernel spills to local memory; reduce chunk_log2 or n";
    return (PERM_ESPILL);
  }
  I.B = p->spec.B;
  I.U = p->spec.U;
  I.M = p->spec.M;
  for (int i = 0; i < n; ++i) { I.row_perm[i] = p->rowp[i]; I.col_perm[i] = p->colp[i]; }
  {  // Alg. 4 partition reported for the base ordering (paper's (k, c))
    std::vector<int> rp, cp;
    order_with(I.ordering, rp, cp);
    Csx ob = permute_ccs(p->ccs, rp, cp);
    partition_alg4(ob, gr, 148, I.k, I.c);
  }
  if (n == 1) p->trivial1 = true;
  I.candidates_compiled = (int)oks.size();
  I.w_alg1 = w_alg1(p->occs);
  if (p->is_c128)  // complex Alg. 1: an update is 2 DP ops, a product step 4, the accumulate 2
    I.w_alg1 = 2.0 * (I.w_alg1 - n) + 4.0 * (n - 1) + 2.0;
  if (!p->singular && !p->trivial1) {
    I.w_plan = p->code.w_plan;
    I.reg_rows = p->code.live_rows;
    I.tier_rows = p->code.tier_rows;
    I.seed_rows = p->code.seed_rows;
    I.levels = p->code.levels;
    I.smem_bytes = p->code.smem_bytes;
    I.block = p->spec.threads;
  }
  return PERM_OK;
}


}  // namespace

int plan_kernel(perm_plan_s* p, perm_ordering ord, double gr, const std::shared_future<void>& ctx_ready) {
  Planner pl(p, ord, gr, ctx_ready);
  return pl.run();
}

}  // namespace perm
