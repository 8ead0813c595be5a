// oracle/oracle.cpp -- CPU ORACLE for the sparse-permanent hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
// It shares no code, header, table or helper with the CUDA path
// (paper_2501_15126_b200/); it takes dense row-major matrices, not CCS/CRS.
//
// Citation key: P:n = /root/reference/PAPER.md line n (arXiv 2501.15126).
// Every function states the passage it follows.  Precision: long double
// (x87 80-bit, u = 2^-64) for floating point; exact (wrapping) __int128 for
// integer inputs.  The paper fixes FP64 for its own kernels;
// the oracle is more precise than the method on purpose.
//
// Parity pins (tests/test_oracle.py): closed forms n!, D_n, Fibonacci,
// identity, triangular, block-diagonal rank-1; brute-force Eq. 1 on tiny
// inputs; cross-mode equality (naive == Ryser Eq. 2 == NW Alg. 1 == band DP).
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <algorithm>
#include <omp.h>

typedef __int128 i128;
typedef unsigned __int128 u128;

extern "C" {

// ---------------------------------------------------------------------------
// Eq. 1: perm(A) = sum over permutations sigma of prod_i a_{i,sigma(i)}.
// Written out as a row-by-row depth-first enumeration of sigma with a bitmask
// of used columns; a zero factor makes the whole term zero, so such branches
// are not expanded (this drops only terms that are exactly 0).
// ---------------------------------------------------------------------------
static long double naive_ld_rec(int n, const long double* A, int i, uint64_t used) {
    if (i == n) return 1.0L;
    long double s = 0.0L;
    for (int c = 0; c < n; ++c) {
        if (used >> c & 1) continue;
        long double a = A[(size_t)i * n + c];
        if (a == 0.0L) continue;
        s += a * naive_ld_rec(n, A, i + 1, used | (1ull << c));
    }
    return s;
}

long double oracle_perm_naive_ld(int n, const double* A) {
    if (n <= 0) return 1.0L;  // empty product / empty permutation set
    std::vector<long double> L((size_t)n * n);
    for (size_t k = 0; k < L.size(); ++k) L[k] = A[k];
    return naive_ld_rec(n, L.data(), 0, 0);
}

static i128 naive_i_rec(int n, const int64_t* A, int i, uint64_t used) {
    if (i == n) return 1;
    i128 s = 0;
    for (int c = 0; c < n; ++c) {
        if (used >> c & 1) continue;
        int64_t a = A[(size_t)i * n + c];
        if (a == 0) continue;
        s += (i128)a * naive_i_rec(n, A, i + 1, used | (1ull << c));
    }
    return s;
}

// Eq. 1 in exact integers (inputs must be integers; result exact while
// |perm| < 2^127, which the caller certifies).
void oracle_perm_naive_i128(int n, const int64_t* A, uint64_t* lo, uint64_t* hi) {
    i128 r = n <= 0 ? 1 : naive_i_rec(n, A, 0, 0);
    u128 u = (u128)r;
    *lo = (uint64_t)u;
    *hi = (uint64_t)(u >> 64);
}

// ---------------------------------------------------------------------------
// Eq. 2, Ryser: perm(A) = (-1)^n sum_{S subset [n]} (-1)^{|S|}
//   prod_i sum_{j in S} a_ij.   Literal subset enumeration, exact integers.
// ---------------------------------------------------------------------------
void oracle_perm_ryser_i128(int n, const int64_t* A, int threads, uint64_t* lo, uint64_t* hi) {
    const uint64_t nsub = 1ull << n;
    u128 total = 0;
#pragma omp parallel num_threads(threads > 0 ? threads : omp_get_max_threads())
    {
        u128 local = 0;
#pragma omp for schedule(static)
        for (long long S = 0; S < (long long)nsub; ++S) {
            u128 prod = 1;
            for (int i = 0; i < n; ++i) {
                i128 rs = 0;
                for (int j = 0; j < n; ++j)
                    if ((uint64_t)S >> j & 1) rs += A[(size_t)i * n + j];
                prod *= (u128)rs;  // wrapping product = exact mod 2^128
            }
            int card = __builtin_popcountll((uint64_t)S);
            if (card & 1) local -= prod; else local += prod;
        }
#pragma omp critical
        total += local;
    }
    if (n & 1) total = (u128)0 - total;  // (-1)^n
    *lo = (uint64_t)total;
    *hi = (uint64_t)(total >> 64);
}

// ---------------------------------------------------------------------------
// Alg. 1 SparsePerman with the chunked parallelisation of Sec. II-A
// (P:131-132), in long double.
//
//   x_i  = a_{i,n-1} - (1/2) sum_j a_ij             (lines 1-5; DESIGN reading R1:
//                                                    the true a_{i,n-1}, 0 if absent)
//   for g: j = log2(Gray_g XOR Gray_{g-1})         (line 9)
//          s = 2*Gray_g[j] - 1                      (line 10)
//          x[row] += s * a_{row,j} over column j    (lines 12-15)
//          prod = prod_i x_i                        (lines 17-19)
//          p += (-1)^g prod                          (line 21)
//   perm = p * (4 (n mod 2) - 2)                    (line 23)
//
// Chunking (Sec. II-A): the g range is split into chunks of DELTA = 2^12
// consecutive iterations; a chunk starting at g_start seeds its private x
// from x (lines 1-5) plus the columns of the set bits of Gray_{g_start}
// (the paper writes Gray_{g_start - 1} because its chunk begins with a flip;
// here a chunk begins with the product at g_start -- DESIGN reading R3).
// Chunk partials are folded pairwise in chunk-index order (deterministic,
// thread-count independent).
// ---------------------------------------------------------------------------
static const int ORACLE_CHUNK_LOG2 = 12;

struct NWMatrix {
    int n;
    std::vector<long double> a;          // dense row-major
    std::vector<long double> x0;         // lines 1-5
    std::vector<std::vector<int>> colrows;  // rows with a_ij != 0, per column j
};

static void nw_prepare(NWMatrix& M, int n, const double* A) {
    M.n = n;
    M.a.assign((size_t)n * n, 0.0L);
    for (size_t k = 0; k < M.a.size(); ++k) M.a[k] = A[k];
    M.x0.assign(n, 0.0L);
    for (int i = 0; i < n; ++i) {
        long double sum = 0.0L;
        for (int j = 0; j < n; ++j) sum += M.a[(size_t)i * n + j];
        M.x0[i] = M.a[(size_t)i * n + (n - 1)] - sum / 2;
    }
    M.colrows.assign(n, {});
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i)
            if (M.a[(size_t)i * n + j] != 0.0L) M.colrows[j].push_back(i);
}

static inline uint64_t gray(uint64_t g) { return g ^ (g >> 1); }

// Sum over g in [gb, ge) of (-1)^g prod_i x_i(Gray_g); also sum of |terms|.
// R = long double (the oracle proper) or double (the FP64 CPU-SparsePerman
// analogue timed as a CPU baseline; same steps, same order).
extern "C++" {
template <class R>
static void nw_chunk(const NWMatrix& M, uint64_t gb, uint64_t ge, R* out, R* out_abs) {
    const int n = M.n;
    R x[64];
    for (int i = 0; i < n; ++i) x[i] = (R)M.x0[i];
    uint64_t G = gray(gb);
    for (int j = 0; j + 1 < n; ++j)
        if (G >> j & 1)
            for (int i : M.colrows[j]) x[i] += M.a[(size_t)i * n + j];
    R p = 0, pa = 0;
    for (uint64_t g = gb; g < ge; ++g) {
        if (g != gb) {
            uint64_t d = gray(g) ^ gray(g - 1);
            int j = 63 - __builtin_clzll(d);                    // log2 of a power of two
            R s = (R)2 * (R)(gray(g) >> j & 1) - (R)1;
            for (int i : M.colrows[j]) x[i] += s * M.a[(size_t)i * n + j];
        }
        R prod = 1;
        for (int i = 0; i < n; ++i) prod *= x[i];
        if (g & 1) p -= prod; else p += prod;
        pa += prod < 0 ? -prod : prod;
    }
    *out = p;
    *out_abs = pa;
}

// pairwise (perfect binary tree on power-of-two lengths) sum in index order
template <class R>
static R pairwise(const R* v, size_t len) {
    if (len == 0) return 0;
    if (len == 1) return v[0];
    size_t h = 1;
    while (h * 2 < len) h *= 2;
    return pairwise(v, h) + pairwise(v + h, len - h);
}

// Unscaled NW sum over the Gray range [gb, ge):  sum (-1)^g prod_i x_i(Gray_g).
// Chunks are the 2^12-aligned pieces of the range.  threads <= 0: all cores.
template <class R>
static void nw_range(int n, const double* A, uint64_t gb, uint64_t ge, int threads, R* out_sum, R* out_abs) {
    NWMatrix M;
    nw_prepare(M, n, A);
    const uint64_t CH = 1ull << ORACLE_CHUNK_LOG2;
    // chunk boundaries: aligned multiples of CH inside [gb, ge)
    uint64_t first = (gb + CH - 1) / CH * CH;
    std::vector<std::pair<uint64_t, uint64_t>> pieces;
    // leading partial piece
    if (gb < std::min(first, ge)) pieces.push_back({gb, std::min(first, ge)});
    const uint64_t nfull = ge > first ? (ge - first) / CH : 0;
    const uint64_t tail_start = first + nfull * CH;
    // Full chunks are processed in batches of 2^16 chunks; each batch is a
    // perfect pairwise tree over its chunks, batches are folded pairwise.
    const uint64_t BATCH = 1ull << 16;
    std::vector<R> batch_sum, batch_abs;
    int nt = threads > 0 ? threads : omp_get_max_threads();
    std::vector<R> cs, ca;
    for (uint64_t b0 = 0; b0 < nfull; b0 += BATCH) {
        uint64_t bn = std::min(BATCH, nfull - b0);
        cs.assign(bn, 0.0L);
        ca.assign(bn, 0.0L);
#pragma omp parallel for schedule(dynamic, 16) num_threads(nt)
        for (long long c = 0; c < (long long)bn; ++c) {
            uint64_t s = first + (b0 + (uint64_t)c) * CH;
            nw_chunk(M, s, s + CH, &cs[c], &ca[c]);
        }
        batch_sum.push_back(pairwise(cs.data(), bn));
        batch_abs.push_back(pairwise(ca.data(), bn));
    }
    std::vector<R> parts, parts_abs;
    if (!pieces.empty()) {
        R s, a;
        nw_chunk(M, pieces[0].first, pieces[0].second, &s, &a);
        parts.push_back(s);
        parts_abs.push_back(a);
    }
    if (!batch_sum.empty()) {
        parts.push_back(pairwise(batch_sum.data(), batch_sum.size()));
        parts_abs.push_back(pairwise(batch_abs.data(), batch_abs.size()));
    }
    if (tail_start < ge && tail_start >= first) {
        R s, a;
        nw_chunk(M, tail_start, ge, &s, &a);
        parts.push_back(s);
        parts_abs.push_back(a);
    }
    R S = 0, SA = 0;
    for (size_t k = 0; k < parts.size(); ++k) { S += parts[k]; SA += parts_abs[k]; }
    *out_sum = S;
    *out_abs = SA;
}

}  // extern "C++"

void oracle_nw_range_ld(int n, const double* A, uint64_t gb, uint64_t ge, int threads,
                        long double* out_sum, long double* out_abs) {
    nw_range<long double>(n, A, gb, ge, threads, out_sum, out_abs);
}

// The same sweep in IEEE double (x, products and sums): the FP64 analogue of
// the paper's CPU-SparsePerman, a CPU baseline only.
void oracle_nw_range_d(int n, const double* A, uint64_t gb, uint64_t ge, int threads,
                       double* out_sum, double* out_abs) {
    nw_range<double>(n, A, gb, ge, threads, out_sum, out_abs);
}

// perm(A) via Alg. 1 over the full range g in [0, 2^(n-1)), times the
// line-23 factor 4(n mod 2) - 2.   Returns the result; *kappa_num = sum|terms|*2.
long double oracle_perm_nw_ld(int n, const double* A, int threads, long double* sum_abs) {
    if (n == 1) { if (sum_abs) *sum_abs = A[0] < 0 ? -A[0] : A[0]; return A[0]; }
    long double s, a;
    oracle_nw_range_ld(n, A, 0, 1ull << (n - 1), threads, &s, &a);
    long double f = 4.0L * (long double)(n % 2) - 2.0L;   // line 23
    if (sum_abs) *sum_abs = 2.0L * a;
    return s * f;
}

// ---------------------------------------------------------------------------
// Alg. 1 in exact integers for integer-valued A (the "doubled" form):
// with x'_i = 2 x_i = 2 a_{i,n-1} - sum_j a_ij (an integer), the accumulated
//   T' = sum_g (-1)^g prod_i x'_i(Gray_g) = 2^n * p   (p of Alg. 1),
// so perm = p * (4(n mod 2) - 2) = (-1)^(n-1) * T' / 2^(n-1).
// Wrapping u128 arithmetic: exact while |perm| * 2^(n-1) < 2^127.
// Returns T' (mod 2^128).  Gray steps as in Alg. 1 lines 9-15.
// ---------------------------------------------------------------------------
void oracle_nw2_range_i128(int n, const int64_t* A, uint64_t gb, uint64_t ge, int threads,
                           uint64_t* lo, uint64_t* hi, uint64_t* nzero_terms) {
    std::vector<int64_t> x0(n);
    std::vector<std::vector<int>> colrows(n);
    for (int i = 0; i < n; ++i) {
        int64_t sum = 0;
        for (int j = 0; j < n; ++j) sum += A[(size_t)i * n + j];
        x0[i] = 2 * A[(size_t)i * n + (n - 1)] - sum;
    }
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i)
            if (A[(size_t)i * n + j] != 0) colrows[j].push_back(i);
    const uint64_t CH = 1ull << ORACLE_CHUNK_LOG2;
    const uint64_t len = ge > gb ? ge - gb : 0;
    const uint64_t nch = (len + CH - 1) / CH;
    u128 total = 0;
    uint64_t zeros = 0;
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel num_threads(nt)
    {
        u128 local = 0;
        uint64_t lz = 0;
        int64_t x[64];
#pragma omp for schedule(dynamic, 16)
        for (long long c = 0; c < (long long)nch; ++c) {
            uint64_t s0 = gb + (uint64_t)c * CH, s1 = std::min(ge, s0 + CH);
            for (int i = 0; i < n; ++i) x[i] = x0[i];
            uint64_t G = gray(s0);
            for (int j = 0; j + 1 < n; ++j)
                if (G >> j & 1)
                    for (int i : colrows[j]) x[i] += 2 * A[(size_t)i * n + j];
            for (uint64_t g = s0; g < s1; ++g) {
                if (g != s0) {
                    uint64_t d = gray(g) ^ gray(g - 1);
                    int j = 63 - __builtin_clzll(d);
                    int64_t s = 2 * (int64_t)(gray(g) >> j & 1) - 1;
                    for (int i : colrows[j]) x[i] += s * 2 * A[(size_t)i * n + j];
                }
                u128 prod = 1;
                bool z = false;
                for (int i = 0; i < n; ++i) { prod *= (u128)(i128)x[i]; z |= x[i] == 0; }
                lz += z;
                if (g & 1) local -= prod; else local += prod;
            }
        }
#pragma omp critical
        { total += local; zeros += lz; }
    }
    *lo = (uint64_t)total;
    *hi = (uint64_t)(total >> 64);
    if (nzero_terms) *nzero_terms = zeros;
}

// ---------------------------------------------------------------------------
// Band DP: exact textbook evaluation of Eq. 1 for matrices with a_ij = 0
// whenever |i - j| > w.  Rows are assigned in order; the state is the set of
// used columns inside the window [i-w, i+w]; a column leaving the window must
// already be used (no later row can reach it).  Cost O(n 2^(2w+1) (2w+1)).
// ---------------------------------------------------------------------------
}  // extern "C"

template <class T, class GetA>
static T band_dp(int n, int w, GetA geta) {
    const int W = 2 * w + 1;
    const size_t NS = (size_t)1 << W;
    // state bit b <-> column (i - w + b) for current row i
    std::vector<T> cur(NS, T(0)), nxt(NS, T(0));
    // columns outside [0, n) do not exist: pre-set their bits as "used"
    uint64_t init = 0;
    for (int b = 0; b < W; ++b) if (0 - w + b < 0 || 0 - w + b >= n) init |= 1ull << b;
    cur[init] = T(1);
    for (int i = 0; i < n; ++i) {
        std::fill(nxt.begin(), nxt.end(), T(0));
        for (size_t st = 0; st < NS; ++st) {
            if (cur[st] == T(0)) continue;
            for (int b = 0; b < W; ++b) {
                int c = i - w + b;
                if (c < 0 || c >= n) continue;
                if (st >> b & 1) continue;
                T a = geta(i, c);
                if (a == T(0)) continue;
                uint64_t ns = st | (1ull << b);
                // shift window for row i+1: bit 0 (column i-w) leaves; must be used
                if (!(ns & 1)) continue;
                uint64_t sh = ns >> 1;
                // new top bit: column i+1+w; mark used if it does not exist
                if (i + 1 + w >= n) sh |= 1ull << (W - 1);
                nxt[sh] += cur[st] * a;
            }
        }
        std::swap(cur, nxt);
    }
    return cur[NS - 1];
}

extern "C" {

long double oracle_perm_band_ld(int n, const double* A, int w) {
    return band_dp<long double>(n, w, [&](int i, int j) { return (long double)A[(size_t)i * n + j]; });
}

void oracle_perm_band_i128(int n, const int64_t* A, int w, uint64_t* lo, uint64_t* hi) {
    i128 r = band_dp<i128>(n, w, [&](int i, int j) { return (i128)A[(size_t)i * n + j]; });
    u128 u = (u128)r;
    *lo = (uint64_t)u;
    *hi = (uint64_t)(u >> 64);
}

// ---------------------------------------------------------------------------
// Structural rank ("rejected structurally rank-deficient matrices"):
// size of a maximum bipartite matching of the nonzero pattern, by simple
// augmenting paths (Kuhn).  Textbook; O(n * nnz).
// ---------------------------------------------------------------------------
static bool kuhn(int i, int n, const double* A, std::vector<int>& mcol, std::vector<char>& seen) {
    for (int j = 0; j < n; ++j) {
        if (A[(size_t)i * n + j] == 0.0 || seen[j]) continue;
        seen[j] = 1;
        if (mcol[j] < 0 || kuhn(mcol[j], n, A, mcol, seen)) { mcol[j] = i; return true; }
    }
    return false;
}

int oracle_structural_rank(int n, const double* A) {
    std::vector<int> mcol(n, -1);
    int r = 0;
    for (int i = 0; i < n; ++i) {
        std::vector<char> seen(n, 0);
        if (kuhn(i, n, A, mcol, seen)) ++r;
    }
    return r;
}

int oracle_max_threads(void) { return omp_get_max_threads(); }

}  // extern "C"

// ---------------------------------------------------------------------------
// Complex permanents (boson sampling).  Same
// definitions as above over C: Eq. 1 and Alg. 1 in std::complex<long double>.
// Matrices are dense row-major interleaved (re, im) pairs.
// ---------------------------------------------------------------------------
#include <complex>
typedef std::complex<long double> cld;

static cld naive_c_rec(int n, const cld* A, int i, uint64_t used) {
  if (i == n) return cld(1.0L);
  cld s(0.0L);
  for (int c = 0; c < n; ++c) {
    if (used >> c & 1) continue;
    const cld a = A[(size_t)i * n + c];
    if (a == cld(0.0L)) continue;
    s += a * naive_c_rec(n, A, i + 1, used | (1ull << c));
  }
  return s;
}

// Alg. 1 lines 9-21 over a chunk of the Gray range in complex long double
static void nw_chunk_c(int n, const std::vector<cld>& a, const std::vector<cld>& x0,
                       const std::vector<std::vector<int>>& colrows, uint64_t gb, uint64_t ge, cld* out,
                       long double* out_abs) {
  cld x[64];
  for (int i = 0; i < n; ++i) x[i] = x0[i];
  const uint64_t G = gray(gb);
  for (int j = 0; j + 1 < n; ++j)
    if (G >> j & 1)
      for (int i : colrows[j]) x[i] += a[(size_t)i * n + j];
  cld p(0.0L);
  long double pa = 0.0L;
  for (uint64_t g = gb; g < ge; ++g) {
    if (g != gb) {
      const uint64_t d = gray(g) ^ gray(g - 1);
      const int j = 63 - __builtin_clzll(d);
      const long double s = 2.0L * (long double)(gray(g) >> j & 1) - 1.0L;
      for (int i : colrows[j]) x[i] += s * a[(size_t)i * n + j];
    }
    cld prod(1.0L);
    for (int i = 0; i < n; ++i) prod *= x[i];
    if (g & 1) p -= prod; else p += prod;
    pa += std::abs(prod);
  }
  *out = p;
  *out_abs = pa;
}

extern "C" {

void oracle_perm_naive_c(int n, const double* A, long double* re, long double* im) {
  std::vector<cld> L((size_t)n * n);
  for (size_t k = 0; k < L.size(); ++k) L[k] = cld(A[2 * k], A[2 * k + 1]);
  const cld r = n <= 0 ? cld(1.0L) : naive_c_rec(n, L.data(), 0, 0);
  *re = r.real();
  *im = r.imag();
}

// band DP of Eq. 1 over C (same textbook DP as oracle_perm_band_ld)
void oracle_perm_band_c(int n, const double* A, int w, long double* re, long double* im) {
  const cld r = band_dp<cld>(n, w, [&](int i, int j) {
    const size_t k = (size_t)i * n + j;
    return cld(A[2 * k], A[2 * k + 1]);
  });
  *re = r.real();
  *im = r.imag();
}

// Unscaled complex Alg. 1 sum over [gb, ge) (chunks of 2^12, pairwise fold)
void oracle_nw_range_c(int n, const double* A, uint64_t gb, uint64_t ge, int threads, long double* re,
                       long double* im, long double* sum_abs) {
  std::vector<cld> a((size_t)n * n);
  for (size_t k = 0; k < a.size(); ++k) a[k] = cld(A[2 * k], A[2 * k + 1]);
  std::vector<cld> x0(n);
  for (int i = 0; i < n; ++i) {
    cld sum(0.0L);
    for (int j = 0; j < n; ++j) sum += a[(size_t)i * n + j];
    x0[i] = a[(size_t)i * n + (n - 1)] - sum / 2.0L;  // Alg. 1 lines 1-5 (reading R1)
  }
  std::vector<std::vector<int>> colrows(n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (a[(size_t)i * n + j] != cld(0.0L)) colrows[j].push_back(i);
  const uint64_t CH = 1ull << ORACLE_CHUNK_LOG2;
  const uint64_t len = ge > gb ? ge - gb : 0, nch = (len + CH - 1) / CH;
  std::vector<cld> part(nch);
  std::vector<long double> pabs(nch);
  const int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(nt)
  for (long long c = 0; c < (long long)nch; ++c) {
    const uint64_t s0 = gb + (uint64_t)c * CH, s1 = std::min(ge, s0 + CH);
    nw_chunk_c(n, a, x0, colrows, s0, s1, &part[c], &pabs[c]);
  }
  // pairwise fold in chunk order
  for (uint64_t h = 1; h < nch; h <<= 1)
    for (uint64_t i = 0; i + h < nch; i += 2 * h) { part[i] += part[i + h]; pabs[i] += pabs[i + h]; }
  const cld r = nch ? part[0] : cld(0.0L);
  *re = r.real();
  *im = r.imag();
  *sum_abs = nch ? pabs[0] : 0.0L;
}

}  // extern "C"

extern "C" {

}  // extern "C"
