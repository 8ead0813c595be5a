// perm_internal.h -- internal types of libperm (not part of the C ABI).
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "perm.h"

namespace perm {

// Compressed sparse matrix (CCS or CRS), Sec. II.
struct Csx {
  int n = 0;
  std::vector<int32_t> ptr, idx;
  std::vector<double> val;
  std::vector<double> vim;  // imaginary parts (complex matrices); empty = real
  int nnz() const { return ptr.empty() ? 0 : ptr[n]; }
  bool complex() const { return !vim.empty(); }
  double im(int p) const { return vim.empty() ? 0.0 : vim[p]; }
};

constexpr int PERM_MODE_COMPLEX_INTERNAL = 4;  // complex FP64 sweep (perm_plan_complex)

// ---- matrix.cpp ----------------------------------------------------------
// Validate a CCS/CRS input (boundary rules of perm.h); on success fill both
// layouts.  Returns a perm_status; err gets a message.
int validate_and_convert(int n, perm_format fmt, const int32_t* ptr, const int32_t* idx,
                         const double* val, Csx& ccs, Csx& crs, std::string& err);
// complex variant: val2 = interleaved (re, im) pairs, nnz of them
int validate_and_convert_c(int n, perm_format fmt, const int32_t* ptr, const int32_t* idx,
                           const double* val2, Csx& ccs, Csx& crs, std::string& err);
Csx transpose(const Csx& a);
int structural_rank(const Csx& ccs);  // Hopcroft-Karp
void order_permanent(const Csx& ccs, const Csx& crs, std::vector<int>& rowp, std::vector<int>& colp);
void order_degree(const Csx& ccs, std::vector<int>& rowp, std::vector<int>& colp);
// ordered(i, j) = a(rowp[i], colp[j]); returns CCS of the ordered matrix
Csx permute_ccs(const Csx& ccs, const std::vector<int>& rowp, const std::vector<int>& colp);
// column order with the first K picks moved to the front (pick order), the
// other columns in base order (the base's last column stays last).
std::vector<int> factored_columns(const std::vector<int>& base_colp, const std::vector<int>& picks, int K);
// largest elimination-tree evaluation size after eliminating colp[0..K)
// (leaf 1, node 2 x sum of children)
int elim_eval_size(const Csx& ccs, const std::vector<int>& colp, int K);
// swept columns (positions K..n-2) stably sorted by flip cost
// nnz(c) + sum over touched factored groups g of dcost(|g|) (0, 2, 3|g|-1)
std::vector<int> costsort_swept(const Csx& ccs, const std::vector<int>& colp, int K);
uint64_t b200_threads(int nregisters, int sms);  // CalculateNoThreads model
void partition_alg4(const Csx& ordered_ccs, double gr_ratio, int sms, int& k, int& c);
int alg2_launch_parameters(uint64_t tau, int n, uint64_t* out, int cap);

// ---- codegen.cpp -----------------------------------------------------------
struct KernelSpec {
  int n = 0;
  int K = 0;                   // factored (pairwise row-disjoint) leading columns
  int B = 0, U = 0, M = 1;     // chunk log2, unrolled block log2, chunks per lane per task
  int mode = PERM_MODE_REG;    // REG / HYBRID / INT01
  int hybrid_c = 0;            // HYBRID: factors of levels >= hybrid_c live in the global tier
  int threads = 128;           // threads per block
  bool zero_skip = false;      // INT01: warp-uniform skip of blocks whose product above them is 0
  bool cc = false;             // composite caches (level/suffix products inside composite roots)
  int min_blocks = 1;          // __launch_bounds__ second argument
  uint64_t nchunks_total = 0;  // 2^(n-1-B)
  bool w_only = false;         // planner scoring: skip source steps that change neither W nor registers
  bool i01_asm_mul = false;    // INT01: int x u128 products through the hand-scheduled mul_s32_u128
  int smem_ro = 0;             // > 0: body-read-only loop-carried values with <= smem_ro body uses
                               // also go to (volatile) shared-memory slots (spill escalation rung)
  // INT01 (internal to generate_kernel): raised register bounds for a regeneration
  const std::map<std::string, double>* reg_lb_extra = nullptr;
};

struct KernelCode {
  std::string source;
  std::string name = "perm_sweep";
  int live_rows = 0, tier_rows = 0, seed_rows = 0, levels = 0;
  int tier_bytes = 0;       // bytes of global tier storage per thread (HYBRID)
  int smem_bytes = 0;       // dynamic shared memory per block (loop-carried values off the body)
  double ops_seed = 0, ops_block = 0, ops_chunk_total = 0;
  double w_plan = 0;        // arithmetic ops per Gray step
  int est_regs = 0;         // rough register estimate (for __launch_bounds__)
};

// Generate the matrix-specific sweep kernel for the ORDERED matrix (CCS) with
// x0 given per ordered row (double; INT01: 2*x0 exactly integral).
KernelCode generate_kernel(const Csx& occs, const std::vector<double>& x0, const KernelSpec& spec);

// cumulative generate_kernel wall time (all threads), post-pass share, calls
void codegen_timing(double& gen_ms, double& post_ms, long long& calls);

// Work per Gray step of Alg. 1 as written on this ordered matrix.
double w_alg1(const Csx& occs);

}  // namespace perm
