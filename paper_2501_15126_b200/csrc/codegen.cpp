// codegen.cpp -- matrix-specific sm_100a sweep-kernel generator.
//
// Paper design (prior art): one inclusion and one exclusion __device__
// function per column with the matrix values as literals, x in registers, and
// a full product of the register rows per Gray step (Listings 2-5,
// P:224-262); hybrid mode keeps the rows of columns >= c in global
// memory with a cached global product (Sec. V).
//
// B200 design generated here:
//  * Each lane sweeps aligned chunks of 2^B products (Lemma 1), so
//    the flipped column j = ctz(g) is warp-uniform; the sign (Theorem 1,
//    + iff bit j+1 of g is 0) is warp-uniform except for column
//    B-1, handled branch-free with an FMA by a +-1 register.
//  * The low U Gray bits are unrolled into a straight-line block of 2^U steps
//    where column and sign are compile-time constants (no dispatch at all);
//    the flips of columns U..B-1 between blocks go through one warp-uniform
//    switch (a BRX).
//  * Rows are grouped into levels by the lowest in-chunk column touching them
//    (m(r) = min{j < B : a_rj != 0}).  Level products Q_l and suffix products
//    S_l = Q_l * S_(next level) are cached, so a flip of column j recomputes
//    only the touched levels and the suffix chain below j (Lemma 2, P:382-401:
//    column j flips in 2^-(j+1) of the steps, so the chain is short on average).
//    Rows untouched by columns < B never change inside a chunk; their product
//    F is computed once per chunk at seed time (the B200 counterpart of the
//    paper's cold "global" rows: they need no storage at all during the sweep).
//  * Column 0 flips on every odd step; the two products of a pair differ only
//    in Q_0, so a pair contributes (Q_0(even) - Q_0(odd)) * S_(above 0).
//  * Each chunk is seeded exactly from x0 + the columns of Gray(g0)
//    (Sec. II-A), which bounds incremental x drift to 2^B steps.
//  * Lane partials: pairwise inside a block, sequential over blocks and chunks,
//    then a fixed xor-shuffle tree per warp-task (deterministic slot).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <set>
#include <sstream>

#include "perm_internal.h"

namespace perm {

namespace {

std::string lit(double v) {  // exact hexadecimal floating literal
  char b[64];
  snprintf(b, sizeof b, "%a", v);
  return std::string("(") + b + ")";
}

struct Gen {
  const Csx& A;
  const KernelSpec& S;
  const std::vector<double>& x0;
  const bool i01;
  int n, B, U;
  std::vector<int> minc;                 // per row: level, -1 = frozen (seed-only)
  std::vector<std::vector<int>> G;       // rows per level
  std::vector<int> nonempty;             // ascending
  bool has_frozen = false;
  std::ostringstream o;
  double ops = 0;                        // arithmetic ops emitted in the current region
  int tmp = 0;
  std::string ind = "";

  Gen(const Csx& a, const std::vector<double>& x, const KernelSpec& s)
      : A(a), S(s), x0(x), i01(s.mode == PERM_MODE_INT01), n(a.n), B(s.B), U(s.U) {
    minc.assign(n, -1);
    for (int j = B - 1; j >= 0; --j)
      for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) minc[A.idx[p]] = j;
    G.assign(std::max(B, 1), {});
    for (int r = 0; r < n; ++r) {
      if (minc[r] >= 0) G[minc[r]].push_back(r);
      else has_frozen = true;
    }
    for (int l = 0; l < B; ++l)
      if (!G[l].empty()) nonempty.push_back(l);
  }

  const char* PT() const { return i01 ? "u128" : "double"; }
  const char* VT() const { return i01 ? "int" : "double"; }
  std::string xv(int r) const { return "x" + std::to_string(r); }
  std::string pt(int r) const { return i01 ? "((u128)(i128)" + xv(r) + ")" : xv(r); }

  void line(const std::string& s) { o << ind << s << "\n"; }

  std::string mul(const std::string& a, const std::string& b) {
    if (b.empty()) return a;
    if (a.empty()) return b;
    ops += 1;
    return "(" + a + " * " + b + ")";
  }
  std::string tree(std::vector<std::string> v) {
    if (v.empty()) return "";
    while (v.size() > 1) {
      std::vector<std::string> w;
      for (size_t i = 0; i + 1 < v.size(); i += 2) w.push_back(mul(v[i], v[i + 1]));
      if (v.size() & 1) w.push_back(v.back());
      v.swap(w);
    }
    return v[0];
  }

  bool qreg(int l) const { return G[l].size() >= 2; }
  std::string qexpr(int l) const { return qreg(l) ? "Q" + std::to_string(l) : pt(G[l][0]); }
  int next_level(int l) const {
    for (int m : nonempty)
      if (m > l) return m;
    return -1;
  }
  bool sreg(int l) const { return next_level(l) >= 0 || has_frozen; }
  std::string sexpr(int l) const { return sreg(l) ? "S" + std::to_string(l) : qexpr(l); }
  std::string above(int l) const {
    int m = next_level(l);
    if (m >= 0) return sexpr(m);
    return has_frozen ? "F" : "";
  }

  void recompute_q(int l) {
    if (!qreg(l)) return;
    std::vector<std::string> v;
    for (int r : G[l]) v.push_back(pt(r));
    line("Q" + std::to_string(l) + " = " + tree(v) + ";");
  }
  void recompute_s(int l) {  // l >= 1
    if (!sreg(l)) return;
    line("S" + std::to_string(l) + " = " + mul(qexpr(l), above(l)) + ";");
  }

  // one update x_r +-= a_rj.  sign: "+", "-" (static) or a runtime +-1 name
  void update(int r, double a, const std::string& sign) {
    ops += 1;
    if (i01) {
      if (sign == "+") line(xv(r) + " += 2;");
      else if (sign == "-") line(xv(r) + " -= 2;");
      else line(xv(r) + " += " + sign + ";");  // runtime sign register holds +-2
    } else {
      if (sign == "+") line(xv(r) + " += " + lit(a) + ";");
      else if (sign == "-") line(xv(r) + " -= " + lit(a) + ";");
      else line(xv(r) + " = fma(" + sign + ", " + lit(a) + ", " + xv(r) + ");");
    }
  }

  // flip of column j >= 1 (affects levels <= j); S chain recomputed down to level 1
  void flip(int j, const std::string& sign) {
    std::set<int> aff;
    for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) {
      update(A.idx[p], A.val[p], sign);
      aff.insert(minc[A.idx[p]]);
    }
    for (int l : aff) recompute_q(l);
    int h = aff.empty() ? -1 : *aff.rbegin();
    for (auto it = nonempty.rbegin(); it != nonempty.rend(); ++it)
      if (*it >= 1 && *it <= h) recompute_s(*it);
  }

  // ---- the block body: 2^U steps, pairs (2k, 2k+1) --------------------------
  void block_body() {
    std::vector<std::string> stack(U + 1);
    const int npairs = 1 << (U - 1);
    for (int k = 0; k < npairs; ++k) {
      const int u = 2 * k;
      if (u > 0) {
        int j = __builtin_ctz(u);
        std::string sg = (j == U - 1) ? "sU" : (((u >> (j + 1)) & 1) ? "-" : "+");
        flip(j, sg);
      }
      // pair: product at even step u (current state), flip column 0, product at u+1
      std::string sg0 = (U >= 2) ? ((((u + 1) >> 1) & 1) ? "-" : "+") : "sU";
      std::string e = "e" + std::to_string(tmp++);
      line(std::string("const ") + PT() + " " + e + " = " + qexpr(0) + ";");
      for (int p = A.ptr[0]; p < A.ptr[1]; ++p) update(A.idx[p], A.val[p], sg0);
      recompute_q(0);
      ops += 1;  // e - Q0
      std::string d = "(" + e + " - " + qexpr(0) + ")";
      std::string t = "t" + std::to_string(tmp++);
      line(std::string("const ") + PT() + " " + t + " = " + mul(d, above(0)) + ";");
      // pairwise (binary-counter) accumulation of the pair terms
      std::string v = t;
      int lvl = 0;
      unsigned kk = (unsigned)k;
      while (kk & 1u) {
        std::string w = "v" + std::to_string(tmp++);
        ops += 1;
        line(std::string("const ") + PT() + " " + w + " = " + stack[lvl] + " + " + v + ";");
        v = w;
        kk >>= 1;
        ++lvl;
      }
      stack[lvl] = v;
    }
    ops += 1;
    line("cacc += " + stack[U - 1] + ";");
  }

  void seed() {
    // x = x0 + columns of Gray(g0); only columns >= B-1 can be set (g0 = chunk << B)
    line("const u64 gr = g0 ^ (g0 >> 1);");
    for (int r = 0; r < n; ++r) {
      if (i01) line(std::string(VT()) + " " + xv(r) + " = " + std::to_string((long long)std::llround(x0[r])) + ";");
      else line(std::string(VT()) + " " + xv(r) + " = " + lit(x0[r]) + ";");
    }
    for (int j = std::max(B - 1, 0); j <= n - 2; ++j) {
      if (A.ptr[j + 1] == A.ptr[j]) continue;
      std::string b = "b" + std::to_string(j);
      if (i01) {
        line("const int " + b + " = (int)((gr >> " + std::to_string(j) + ") & 1ull) << 1;");
        for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) { ops += 1; line(xv(A.idx[p]) + " += " + b + ";"); }
      } else {
        line("const double " + b + " = __longlong_as_double((long long)(((gr >> " + std::to_string(j) +
             ") & 1ull) * 0x3FF0000000000000ull));");
        for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) {
          ops += 1;
          line(xv(A.idx[p]) + " = fma(" + b + ", " + lit(A.val[p]) + ", " + xv(A.idx[p]) + ");");
        }
      }
    }
    if (has_frozen) {
      std::vector<std::string> v;
      for (int r = 0; r < n; ++r)
        if (minc[r] < 0) v.push_back(pt(r));
      line(std::string("const ") + PT() + " F = " + tree(v) + ";");
    }
    for (int l : nonempty)
      if (qreg(l)) line(std::string(PT()) + " Q" + std::to_string(l) + ";");
    for (int l : nonempty)
      if (l >= 1 && sreg(l)) line(std::string(PT()) + " S" + std::to_string(l) + ";");
    for (int l : nonempty) recompute_q(l);
    for (auto it = nonempty.rbegin(); it != nonempty.rend(); ++it)
      if (*it >= 1) recompute_s(*it);
  }
};

}  // namespace

double w_alg1(const Csx& A) {
  const int n = A.n;
  if (n < 2) return 0;
  const double denom = std::ldexp(1.0, n - 1) - 1.0;
  double w = 0;
  for (int j = 0; j + 1 < n; ++j) w += std::ldexp(1.0, n - j - 2) / denom * (A.ptr[j + 1] - A.ptr[j]);
  return w + (n - 1) + 1;
}

KernelCode generate_kernel(const Csx& A, const std::vector<double>& x0, const KernelSpec& S) {
  Gen g(A, x0, S);
  KernelCode kc;
  const int B = S.B, U = S.U;
  const uint64_t nblk = 1ull << (B - U);
  const bool masked = S.nchunks_total < 32;
  std::ostringstream& o = g.o;

  o << "// generated by libperm codegen (arXiv 2501.15126 sweep, B200 design)\n"
    << "// n=" << A.n << " nnz=" << A.nnz() << " B=" << B << " U=" << U << " M=" << S.M
    << " mode=" << S.mode << "\n";
  o << "typedef unsigned long long u64;\n";
  if (g.i01) o << "typedef unsigned __int128 u128;\ntypedef __int128 i128;\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << S.threads << ", " << S.min_blocks << ")\n"
    << kc.name << "(const u64 task_begin, const unsigned task_count, unsigned* __restrict__ counter, "
    << g.PT() << "* __restrict__ slots)\n{\n";
  g.ind = "  ";
  g.line("const unsigned lane = threadIdx.x & 31u;");
  g.line("for (;;) {");
  g.ind = "    ";
  g.line("unsigned t = 0;");
  g.line("if (lane == 0) t = atomicAdd(counter, 1u);");
  g.line("t = __shfl_sync(0xffffffffu, t, 0);");
  g.line("if (t >= task_count) break;");
  g.line("const u64 task = task_begin + t;");
  g.line(std::string(g.PT()) + " lacc = 0;");
  g.line("#pragma unroll 1");
  g.line("for (unsigned m = 0; m < " + std::to_string(S.M) + "u; ++m) {");
  g.ind = "      ";
  g.line("const u64 chunk = ((task * " + std::to_string(S.M) + "ull + m) << 5) | lane;");
  g.line("const u64 g0 = chunk << " + std::to_string(B) + ";");
  g.ops = 0;
  g.seed();
  kc.ops_seed = g.ops;
  g.line(std::string(g.PT()) + " cacc = 0;");
  double ops_body = 0, ops_switch = 0;
  if (U == 0) {
    // B == 0: one product per chunk (g = chunk), everything frozen; sign (-1)^g
    g.ops = 0;
    const std::string P = g.has_frozen ? std::string("F") : std::string("1");
    g.line("cacc = (chunk & 1ull) ? (" + std::string(g.PT()) + ")(0 - " + P + ") : " + P + ";");
    ops_body = 0;
  } else {
    if (nblk > 1) {
      g.line("#pragma unroll 1");
      g.line("for (unsigned blk = 0; blk < " + std::to_string(nblk) + "u; ++blk) {");
      g.ind = "        ";
      g.line("const u64 g = g0 | ((u64)blk << " + std::to_string(U) + ");");
      g.line("if (blk != 0) {");
      g.ind = "          ";
      g.line("const int j = " + std::to_string(U - 1) + " + __ffs(blk);");
      if (g.i01) g.line("const int s = ((g >> (j + 1)) & 1ull) ? -2 : 2;");
      else g.line("const double s = ((g >> (j + 1)) & 1ull) ? -1.0 : 1.0;");
      g.line("switch (j) {");
      for (int j = U; j < B; ++j) {
        g.line("case " + std::to_string(j) + ": {");
        std::string save = g.ind;
        g.ind += "  ";
        g.ops = 0;
        g.flip(j, "s");
        ops_switch += g.ops * (double)(1ull << (B - 1 - j));  // flips of j per chunk
        g.line("break; }");
        g.ind = save;
      }
      g.line("default: break;");
      g.line("}");
      g.ind = "        ";
      g.line("}");
    } else {
      g.line("{");
      g.ind = "        ";
      g.line("const u64 g = g0;");
    }
    if (g.i01) g.line("const int sU = ((g >> " + std::to_string(U) + ") & 1ull) ? -2 : 2;");
    else g.line("const double sU = ((g >> " + std::to_string(U) + ") & 1ull) ? -1.0 : 1.0;");
    g.ops = 0;
    g.block_body();
    ops_body = g.ops;
    g.ind = "      ";
    g.line("}");
  }
  if (masked) g.line("if (chunk < " + std::to_string(S.nchunks_total) + "ull) lacc += cacc;");
  else g.line("lacc += cacc;");
  g.ind = "    ";
  g.line("}");
  // fixed-order warp tree (deterministic task slot)
  if (g.i01) {
    g.line("#pragma unroll");
    g.line("for (int o = 16; o > 0; o >>= 1) {");
    g.line("  const u64 lo = __shfl_xor_sync(0xffffffffu, (u64)lacc, o);");
    g.line("  const u64 hi = __shfl_xor_sync(0xffffffffu, (u64)(lacc >> 64), o);");
    g.line("  lacc += ((u128)hi << 64) | lo;");
    g.line("}");
  } else {
    g.line("#pragma unroll");
    g.line("for (int o = 16; o > 0; o >>= 1) lacc += __shfl_xor_sync(0xffffffffu, lacc, o);");
  }
  g.line("if (lane == 0) slots[t] = lacc;");
  g.ind = "  ";
  g.line("}");
  o << "}\n";

  kc.source = o.str();
  kc.ops_block = ops_body;
  const double chunk_ops = kc.ops_seed + (double)nblk * ops_body + ops_switch + 1.0;  // + lacc
  kc.ops_chunk_total = chunk_ops;
  kc.w_plan = chunk_ops / std::ldexp(1.0, B);
  int live = 0;
  for (int r = 0; r < A.n; ++r) live += g.minc[r] >= 0;
  kc.live_rows = live;
  kc.seed_rows = A.n - live;
  kc.tier_rows = 0;
  kc.levels = (int)g.nonempty.size();
  int qs = 0;
  for (int l : g.nonempty) qs += g.qreg(l) + (l >= 1 && g.sreg(l));
  const int wpv = g.i01 ? 1 : 2;   // 32-bit registers per x value
  const int wpp = g.i01 ? 4 : 2;   // per product value
  kc.est_regs = live * wpv + qs * wpp + (U + 2) * wpp + 28;
  return kc;
}

}  // namespace perm
