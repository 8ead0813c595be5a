// codegen.cpp -- matrix-specific sm_100a sweep-kernel generator.
//
// Paper design (prior art): one inclusion and one exclusion __device__
// function per column with the matrix values as literals, x in registers, and
// a full product of the register rows per Gray step (Listings 2-5,
// P:224-262); hybrid mode keeps the rows of columns >= c in global
// memory with a cached global product (Sec. V).
//
// B200 design generated here:
//  * Factored columns 0..K-1 (pairwise row-disjoint, chosen by the planner):
//    for fixed states of all other columns, the sum over the 2^K states of
//    these columns of (-1)^|S| prod_i y_i factorises exactly into
//    (-1)^K prod_k D_k * (product of the other rows), with
//    D_k = prod_{r in col k}(y_r + a_rk) - prod_{r in col k} y_r.
//    So the Gray sweep runs over the remaining "swept" columns K..n-2 only
//    (h-space, 2^(n-1-K) states) and each state's product carries the D_k.
//    K = 0 is Alg. 1 exactly.
//  * Each lane sweeps aligned chunks of 2^B h-states (Lemma 1):
//    the flipped column j = K + ctz(h) is warp-uniform; its sign (Theorem 1,
//    + iff bit ctz(h)+1 of h is 0) is warp-uniform except for the
//    top chunk bit, handled branch-free with an FMA by a +-1 register.
//  * The low U bits are unrolled into a straight-line block of 2^U h-steps in
//    which column and sign are compile-time constants; the flips of bits
//    U..B-1 between blocks go through one warp-uniform switch (BRX).
//  * Factors (plain rows and D_k groups) are grouped into levels by the lowest
//    in-chunk swept bit touching them.  Level products Q_l and suffix products
//    S_l = Q_l * S_(next level) are cached, so a flip recomputes only the
//    touched factors, their levels and the suffix chain below (Lemma 2,
//    bit b flips in 2^-(b+1) of the steps).  Factors untouched by
//    any in-chunk bit never change inside a chunk; their product F is formed
//    once per chunk at seed time (the B200 counterpart of the paper's cold
//    "global" rows: they need no storage at all during the sweep).
//  * Bit 0 flips on every odd h-step; the two products of a pair differ only
//    in Q_0, so a pair contributes (Q_0(even) - Q_0(odd)) * S_(above 0).
//  * Each chunk is seeded exactly from x0 + the swept columns of Gray(h0)
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

struct Factor {
  bool group = false;          // D_k group of factored column `col`
  int col = -1;                // factored column (group)
  std::vector<int> rows;       // 1 row for a plain factor
  std::vector<double> a;       // group: a_rk per row
  int level = -1;              // -1: frozen (no in-chunk bit touches it)
  bool constant() const { return group && rows.size() == 1; }
};

struct Gen {
  const Csx& A;
  const KernelSpec& S;
  const std::vector<double>& x0;
  const bool i01;
  int n, K, B, U;
  std::vector<Factor> fac;
  std::vector<int> fac_of_row;
  std::vector<std::vector<int>> G;       // factor ids per level
  std::vector<int> nonempty;             // ascending levels
  bool has_frozen = false;
  std::ostringstream o;
  double ops = 0;                        // arithmetic ops emitted in the current region
  int tmp = 0;
  std::string ind = "";

  Gen(const Csx& a, const std::vector<double>& x, const KernelSpec& s)
      : A(a), S(s), x0(x), i01(s.mode == PERM_MODE_INT01), n(a.n), K(s.K), B(s.B), U(s.U) {
    fac_of_row.assign(n, -1);
    for (int k = 0; k < K; ++k) {
      Factor f;
      f.group = true;
      f.col = k;
      for (int p = A.ptr[k]; p < A.ptr[k + 1]; ++p) {
        f.rows.push_back(A.idx[p]);
        f.a.push_back(A.val[p]);
        fac_of_row[A.idx[p]] = (int)fac.size();
      }
      fac.push_back(f);
    }
    for (int r = 0; r < n; ++r)
      if (fac_of_row[r] < 0) {
        Factor f;
        f.rows.push_back(r);
        fac_of_row[r] = (int)fac.size();
        fac.push_back(f);
      }
    // level = lowest in-chunk swept bit whose column touches the factor
    for (int b = B - 1; b >= 0; --b) {
      const int j = K + b;
      for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) fac[fac_of_row[A.idx[p]]].level = b;
    }
    G.assign(std::max(B, 1), {});
    for (int f = 0; f < (int)fac.size(); ++f) {
      if (fac[f].constant()) fac[f].level = -1;
      if (fac[f].level >= 0) G[fac[f].level].push_back(f);
      else has_frozen = true;
    }
    for (int l = 0; l < B; ++l)
      if (!G[l].empty()) nonempty.push_back(l);
  }

  const char* PT() const { return i01 ? "u128" : "double"; }
  const char* VT() const { return i01 ? "int" : "double"; }
  std::string xv(int r) const { return "x" + std::to_string(r); }
  std::string pt(int r) const { return i01 ? "((u128)(i128)" + xv(r) + ")" : xv(r); }
  std::string dv(int f) const { return "D" + std::to_string(fac[f].col); }

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

  // value expression of factor f (after recompute_factor for groups)
  std::string fexpr(int f) const {
    const Factor& F = fac[f];
    if (!F.group) return pt(F.rows[0]);
    if (F.constant()) return i01 ? std::string("((u128)2)") : lit(F.a[0]);
    return dv(f);
  }
  // D_k = prod(y + a) - prod(y); emitted inline (returns expression)
  std::string dexpr(int f) {
    const Factor& F = fac[f];
    const size_t k = F.rows.size();
    if (i01) {
      if (k == 2) {  // (x1+2)(x2+2) - x1 x2 = 2 x1 + 2 x2 + 4 (x doubled, a = 1)
        ops += 3;
        return "((u128)(i128)(2 * " + xv(F.rows[0]) + " + 2 * " + xv(F.rows[1]) + " + 4))";
      }
      std::vector<std::string> in, out;
      for (int r : F.rows) {
        ops += 1;
        in.push_back("((u128)(i128)(" + xv(r) + " + 2))");
        out.push_back(pt(r));
      }
      std::string a = tree(in), b = tree(out);
      ops += 1;
      return "(" + a + " - " + b + ")";
    }
    if (k == 2) {  // a1 y2 + a2 y1 + a1 a2: two FMAs, no cancellation
      ops += 2;
      return "fma(" + lit(F.a[0]) + ", " + xv(F.rows[1]) + ", fma(" + lit(F.a[1]) + ", " + xv(F.rows[0]) + ", " +
             lit(F.a[0] * F.a[1]) + "))";
    }
    std::vector<std::string> in, out;
    for (size_t q = 0; q < k; ++q) {
      ops += 1;
      in.push_back("(" + xv(F.rows[q]) + " + " + lit(F.a[q]) + ")");
      out.push_back(xv(F.rows[q]));
    }
    std::string a = tree(in), b = tree(out);
    ops += 1;
    return "(" + a + " - " + b + ")";
  }
  void recompute_factor(int f) {
    const Factor& F = fac[f];
    if (!F.group || F.constant()) return;
    line(dv(f) + " = " + dexpr(f) + ";");
  }

  bool qreg(int l) const { return G[l].size() >= 2; }
  std::string qexpr(int l) const { return qreg(l) ? "Q" + std::to_string(l) : fexpr(G[l][0]); }
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
    for (int f : G[l]) v.push_back(fexpr(f));
    line("Q" + std::to_string(l) + " = " + tree(v) + ";");
  }
  void recompute_s(int l) {  // l >= 1
    if (!sreg(l)) return;
    line("S" + std::to_string(l) + " = " + mul(qexpr(l), above(l)) + ";");
  }

  // a row of a single-row factored column only enters through D_k = a_rk:
  // its y value is never needed (no register, no updates)
  bool dead_row(int r) const { return fac[fac_of_row[r]].constant(); }

  // one update y_r +-= a_rj.  sign: "+", "-" (static) or a runtime +-1 name
  void update(int r, double a, const std::string& sign) {
    if (dead_row(r)) return;
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

  // flip of swept bit b (column K+b); recompute touched factors, their levels
  // and the suffix chain down to level `lowest_s` (1 inside pairs, else 1)
  void flip(int b, const std::string& sign) {
    const int j = K + b;
    std::set<int> facs, levels;
    for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) {
      update(A.idx[p], A.val[p], sign);
      facs.insert(fac_of_row[A.idx[p]]);
    }
    for (int f : facs) recompute_factor(f);
    for (int f : facs)
      if (fac[f].level >= 0) levels.insert(fac[f].level);  // constant D_k: unchanged
    for (int l : levels) recompute_q(l);
    int h = levels.empty() ? -1 : *levels.rbegin();
    for (auto it = nonempty.rbegin(); it != nonempty.rend(); ++it)
      if (*it >= 1 && *it <= h) recompute_s(*it);
  }

  // ---- the block body: 2^U h-steps, pairs (2k, 2k+1) -------------------------
  void block_body() {
    std::vector<std::string> stack(U + 1);
    const int npairs = 1 << (U - 1);
    for (int k = 0; k < npairs; ++k) {
      const int u = 2 * k;
      if (u > 0) {
        int b = __builtin_ctz(u);
        std::string sg = (b == U - 1) ? "sU" : (((u >> (b + 1)) & 1) ? "-" : "+");
        flip(b, sg);
      }
      // pair: product at even step u (current state), flip bit 0, product at u+1
      std::string sg0 = (U >= 2) ? ((((u + 1) >> 1) & 1) ? "-" : "+") : "sU";
      std::string e = "e" + std::to_string(tmp++);
      line(std::string("const ") + PT() + " " + e + " = " + qexpr(0) + ";");
      {
        const int j = K;
        std::set<int> facs;
        for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) {
          update(A.idx[p], A.val[p], sg0);
          facs.insert(fac_of_row[A.idx[p]]);
        }
        for (int f : facs) recompute_factor(f);
        recompute_q(0);
      }
      ops += 1;  // e - Q0
      std::string d = "(" + e + " - " + qexpr(0) + ")";
      std::string t = "t" + std::to_string(tmp++);
      std::string v;
      int lvl = 0;
      unsigned kk = (unsigned)k;
      const std::string ab = above(0);
      if ((kk & 1u) && !ab.empty() && !i01) {
        // first merge of the pairwise tree fused with the pair product:
        // t = fma(d, S_above, stack[0]) -- one DFMA (the kernel is compiled
        // with --fmad=false, so every emitted op is exactly one instruction)
        ops += 1;
        line(std::string("const ") + PT() + " " + t + " = fma(" + d + ", " + ab + ", " + stack[0] + ");");
        v = t;
        kk >>= 1;
        ++lvl;
      } else {
        line(std::string("const ") + PT() + " " + t + " = " + mul(d, ab) + ";");
        v = t;
      }
      // pairwise (binary-counter) accumulation of the pair terms
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
    // y = x0 + swept columns of Gray(h0); only bits >= B-1 can be set (h0 = chunk << B)
    const int nbits = n - 1 - K;
    line("const u64 gr = h0 ^ (h0 >> 1);");
    for (int r = 0; r < n; ++r) {
      if (dead_row(r)) continue;
      if (i01) line(std::string(VT()) + " " + xv(r) + " = " + std::to_string((long long)std::llround(x0[r])) + ";");
      else line(std::string(VT()) + " " + xv(r) + " = " + lit(x0[r]) + ";");
    }
    for (int b = std::max(B - 1, 0); b < nbits; ++b) {
      const int j = K + b;
      bool any = false;
      for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) any |= !dead_row(A.idx[p]);
      if (!any) continue;
      std::string bn = "b" + std::to_string(b);
      if (i01) {
        line("const int " + bn + " = (int)((gr >> " + std::to_string(b) + ") & 1ull) << 1;");
        for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) {
          if (dead_row(A.idx[p])) continue;
          ops += 1;
          line(xv(A.idx[p]) + " += " + bn + ";");
        }
      } else {
        line("const double " + bn + " = __longlong_as_double((long long)(((gr >> " + std::to_string(b) +
             ") & 1ull) * 0x3FF0000000000000ull));");
        for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) {
          if (dead_row(A.idx[p])) continue;
          ops += 1;
          line(xv(A.idx[p]) + " = fma(" + bn + ", " + lit(A.val[p]) + ", " + xv(A.idx[p]) + ");");
        }
      }
    }
    for (int f = 0; f < (int)fac.size(); ++f)
      if (fac[f].group && !fac[f].constant() && fac[f].level >= 0) line(std::string(PT()) + " " + dv(f) + ";");
    if (has_frozen) {
      std::vector<std::string> v;
      for (int f = 0; f < (int)fac.size(); ++f)
        if (fac[f].level < 0) v.push_back(fac[f].group && !fac[f].constant() ? dexpr(f) : fexpr(f));
      line(std::string("const ") + PT() + " F = " + tree(v) + ";");
    }
    for (int f = 0; f < (int)fac.size(); ++f)
      if (fac[f].level >= 0) recompute_factor(f);
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
    << "// n=" << A.n << " nnz=" << A.nnz() << " K=" << S.K << " B=" << B << " U=" << U << " M=" << S.M
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
  g.line("const u64 h0 = chunk << " + std::to_string(B) + ";");
  g.ops = 0;
  g.seed();
  kc.ops_seed = g.ops;
  g.line(std::string(g.PT()) + " cacc = 0;");
  double ops_body = 0, ops_switch = 0;
  if (U == 0) {
    // B == 0: one product per chunk (h = chunk), everything frozen; sign (-1)^h
    g.ops = 0;
    const std::string P = g.has_frozen ? std::string("F") : std::string("1");
    g.line("cacc = (chunk & 1ull) ? (" + std::string(g.PT()) + ")(0 - " + P + ") : " + P + ";");
  } else {
    if (nblk > 1) {
      g.line("#pragma unroll 1");
      g.line("for (unsigned blk = 0; blk < " + std::to_string(nblk) + "u; ++blk) {");
      g.ind = "        ";
      g.line("const u64 h = h0 | ((u64)blk << " + std::to_string(U) + ");");
      g.line("if (blk != 0) {");
      g.ind = "          ";
      g.line("const int j = " + std::to_string(U - 1) + " + __ffs(blk);");
      if (g.i01) g.line("const int s = ((h >> (j + 1)) & 1ull) ? -2 : 2;");
      else g.line("const double s = ((h >> (j + 1)) & 1ull) ? -1.0 : 1.0;");
      g.line("switch (j) {");
      for (int b = U; b < B; ++b) {
        g.line("case " + std::to_string(b) + ": {");
        std::string save = g.ind;
        g.ind += "  ";
        g.ops = 0;
        g.flip(b, "s");
        ops_switch += g.ops * (double)(1ull << (B - 1 - b));  // flips of bit b per chunk
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
      g.line("const u64 h = h0;");
    }
    if (g.i01) g.line("const int sU = ((h >> " + std::to_string(U) + ") & 1ull) ? -2 : 2;");
    else g.line("const double sU = ((h >> " + std::to_string(U) + ") & 1ull) ? -1.0 : 1.0;");
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
  kc.w_plan = chunk_ops / std::ldexp(1.0, B + S.K);  // per Gray step of the full range
  int live = 0, frozen_rows = 0;
  for (const Factor& f : g.fac) {
    if (f.level >= 0) live += (int)f.rows.size();
    else if (!f.constant()) frozen_rows += (int)f.rows.size();
  }
  kc.live_rows = live;
  kc.seed_rows = frozen_rows;
  kc.tier_rows = 0;
  kc.levels = (int)g.nonempty.size();
  int qs = 0, ds = 0;
  for (int l : g.nonempty) qs += g.qreg(l) + (l >= 1 && g.sreg(l));
  for (const Factor& f : g.fac) ds += f.group && !f.constant() && f.level >= 0;
  const int wpv = g.i01 ? 1 : 2;   // 32-bit registers per x value
  const int wpp = g.i01 ? 4 : 2;   // per product value
  kc.est_regs = live * wpv + (qs + ds) * wpp + (U + 2) * wpp + 28;
  return kc;
}

}  // namespace perm
