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
//  * Value numbering: every straight-line region (seed, block body, each
//    switch case) is emitted in SSA form with hash-consed subexpressions, so
//    unchanged sub-products are reused instead of recomputed and every
//    emitted arithmetic op is exactly one executed instruction (the kernel is
//    compiled with --fmad=false; fusions are explicit).  W_plan therefore
//    counts executed DADD/DMUL/DFMA.
//  * Each chunk is seeded exactly from x0 + the swept columns of Gray(h0)
//    (Sec. II-A), which bounds incremental x drift to 2^B steps.
//  * Lane partials: pairwise inside a block, sequential over blocks and chunks,
//    then a fixed xor-shuffle tree per warp-task (deterministic slot).
//  * A whole-kernel post-pass (post_pass) removes dead code, contracts
//    single-use products into explicit FMAs, recounts the executed DP
//    instructions per region and moves loop-carried values the block body
//    never references into per-thread shared-memory slots.
//  * INT01 values are typed int / i64 / wrapping u128 by magnitude bounds; the
//    chunk loop skips a chunk when its frozen product is 0 on all 32 lanes.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cctype>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <deque>
#include <string_view>
#include <map>
#include <set>
#include <sstream>
#include <complex>
#include <functional>
#include <tuple>
#include <unordered_map>

#include "perm_internal.h"

namespace perm {

namespace {

std::string hexlit(double v) {  // exact hexadecimal floating literal
  char b[64];
  snprintf(b, sizeof b, "%a", v);
  return std::string("(") + b + ")";
}

// Elimination tree: eliminating column c merges the factors it touches (T(c))
// into one node E_c = prod_{f in T(c)} f(y + a_c) - prod_{f in T(c)} f(y).
struct Node {
  bool leaf = true;
  int row = -1;                // leaf
  int col = -1;                // internal: eliminated (ordered) column
  std::vector<int> ch;         // internal: children node ids
};

struct Factor {                // a top-level factor (root of an elimination tree)
  bool group = false;          // internal root (composite) vs plain row
  int col = -1;                // group: its eliminated column (names the register)
  int node = -1;
  std::vector<int> rows;       // every row under the root
  bool is_const = false;       // single-leaf elimination: value a_rc, y unused
  int level = -1;              // -1: frozen (no in-chunk bit touches it)
  bool constant() const { return is_const; }
};

struct Gen {
  const Csx& A;
  const KernelSpec& S;
  const std::vector<double>& x0;
  const bool i01;
  bool asm_mul = false;                  // INT01: int x u128 products via mul_s32_u128
  int n, K, B, U;
  std::vector<Factor> fac;
  std::vector<int> fac_of_row;
  std::vector<std::vector<int>> G;       // factor ids per level
  std::vector<int> nonempty;             // ascending register levels (< cT)
  std::vector<int> tier_levels;          // HYBRID: nonempty levels >= cT (global tier)
  int cT = 0;                            // first tier level (B: no tier)
  std::vector<int> tier_slot;            // row -> tier slot or -1
  std::map<std::string, int> tier_of;    // register name -> tier slot
  bool has_frozen = false;
  std::ostringstream o;
  double ops = 0;                        // arithmetic ops emitted in the current region
  std::string ind = "";

  // ---- value numbering (SSA within one straight-line region) ----------------
  struct Val {
    char op;
    int a, b, c;
    char ty;
    std::string name;
    bool real_lit = false;  // complex literal with zero imaginary part
    double re = 0;          // its real part
    double lb = 1e9;        // INT01: log2 of a bound on |value| (1e9: unbounded / wrapping u128)
  };
  std::vector<Val> vals;
  std::map<std::tuple<char, int, int, int>, int> memo;
  std::map<std::string, int> leafs;      // leaf text -> id (literals, region-start registers)
  std::map<std::string, int> cur;        // register -> current value id
  std::set<std::string> dirty;
  int tmp = 0;
  std::map<std::string, double> wt;      // temporary -> executed DP instructions

  std::vector<Node> nodes;
  typedef std::complex<double> zd;
  std::vector<std::map<int, zd>> colval;  // ordered column -> (row -> a) (imag 0 for real)
  bool cx = false;                        // complex FP64 sweep

  Gen(const Csx& a, const std::vector<double>& x, const KernelSpec& s)
      : A(a), S(s), x0(x), i01(s.mode == PERM_MODE_INT01), n(a.n), K(s.K), B(s.B), U(s.U) {
    asm_mul = i01 && s.i01_asm_mul;
    cx = S.mode == PERM_MODE_COMPLEX_INTERNAL;
    colval.assign(n, {});
    for (int j = 0; j < n; ++j)
      for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) colval[j][A.idx[p]] = zd(A.val[p], A.im(p));
    // replay the elimination of ordered columns 0..K-1
    std::vector<int> root_of(n);          // row -> current root node
    for (int r = 0; r < n; ++r) {
      Node nd;
      nd.row = r;
      nodes.push_back(nd);
      root_of[r] = r;
    }
    for (int c = 0; c < K; ++c) {
      std::set<int> T;
      for (auto& kv : colval[c]) T.insert(root_of[kv.first]);
      Node nd;
      nd.leaf = false;
      nd.col = c;
      nd.ch.assign(T.begin(), T.end());
      nodes.push_back(nd);
      const int id = (int)nodes.size() - 1;
      for (int r = 0; r < n; ++r)
        if (T.count(root_of[r])) root_of[r] = id;
    }
    dead.assign(n, 0);  // the only child leaf of an elimination: value a_rc, y never read
    for (const Node& nd : nodes)
      if (!nd.leaf && nd.ch.size() == 1 && nodes[nd.ch[0]].leaf) dead[nodes[nd.ch[0]].row] = 1;
    fac_of_row.assign(n, -1);
    std::map<int, int> fac_of_root;
    for (int r = 0; r < n; ++r) {
      const int rt = root_of[r];
      auto it = fac_of_root.find(rt);
      if (it == fac_of_root.end()) {
        Factor f;
        f.node = rt;
        f.group = !nodes[rt].leaf;
        f.col = nodes[rt].col;
        f.is_const = f.group && nodes[rt].ch.size() == 1 && nodes[nodes[rt].ch[0]].leaf;
        it = fac_of_root.emplace(rt, (int)fac.size()).first;
        fac.push_back(f);
      }
      fac[it->second].rows.push_back(r);
      fac_of_row[r] = it->second;
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
    // HYBRID (Sec. V): factors first flipped by bits >= cT keep their
    // rows in a per-thread global tier; cT >= U so the tier is touched only by
    // the block-boundary flips
    cT = (S.mode == PERM_MODE_HYBRID && S.hybrid_c > 0) ? std::max(std::min(S.hybrid_c, B), std::min(U, B)) : B;
    for (int l = 0; l < B; ++l)
      if (!G[l].empty()) (l < cT ? nonempty : tier_levels).push_back(l);
    zs = i01 && S.zero_skip && U >= 2;
    build_cc();
    if (i01) {
      std::vector<int> rn(n, 0);
      for (int q = 0; q < A.nnz(); ++q) ++rn[A.idx[q]];
      row_lb.assign(n, 0.0);
      for (int r = 0; r < n; ++r) row_lb[r] = std::log2((double)std::max(rn[r], 1));
      init_reg_bounds();
      if (S.reg_lb_extra) for (auto& kv : *S.reg_lb_extra) reg_lb[kv.first] = std::max(reg_lb[kv.first], kv.second);
    }
    tier_slot.assign(n, -1);
    int slots = 0;
    for (int l : tier_levels)
      for (int f : G[l])
        for (int r : fac[f].rows) {
          tier_slot[r] = slots++;
          tier_of[xv(r)] = tier_slot[r];
          tier_row.push_back(r);
        }
  }
  // HYBRID tier vectorisation: slots 2p and 2p+1 of a thread are adjacent
  // (double2 / int2 per thread, coalesced across the warp: one 16-byte or
  // 8-byte access moves a row pair); complex rows are 16 bytes already
  std::vector<int> tier_row;             // slot -> row
  bool tier_pairs() const { return !cx; }
  int tier_partner(int r) const {
    if (!tier_pairs() || tier_slot[r] < 0) return -1;
    const int q = tier_slot[r] ^ 1;
    return q < (int)tier_row.size() ? tier_row[q] : -1;
  }
  const char* VT2() const { return i01 ? "int2" : "double2"; }
  // store the tier rows in `rows` (value ids from `val`), pairing partners
  void tier_store(const std::vector<int>& rows, const std::function<int(int)>& val) {
    std::set<int> done;
    for (int r : rows) {
      if (done.count(r)) continue;
      const int q = tier_partner(r);
      if (q >= 0 && std::find(rows.begin(), rows.end(), q) != rows.end()) {
        const int lo = tier_slot[r] < tier_slot[q] ? r : q, hi = lo == r ? q : r;
        line(std::string("TIER2(") + std::to_string(tier_slot[lo] >> 1) + ") = make_" + VT2() + "(" + nm(val(lo)) +
             ", " + nm(val(hi)) + ");");
        done.insert(q);
      } else {
        line("TIER(" + std::to_string(tier_slot[r]) + ") = " + nm(val(r)) + ";");
      }
      done.insert(r);
    }
  }
  bool has_tier() const { return !tier_levels.empty(); }
  bool tierf(int f) const { return fac[f].level >= cT; }

  const char* PT() const { return i01 ? "u128" : (cx ? "cplx" : "double"); }
  const char* VT() const { return i01 ? "int" : (cx ? "cplx" : "double"); }
  const char* tyname(char t) const {
    return t == 'i' ? "int" : (t == 'l' ? "i64" : (t == 'u' ? "u128" : (t == 'z' ? "cplx" : "double")));
  }
  char pty() const { return i01 ? 'u' : (cx ? 'z' : 'd'); }
  char xty() const { return i01 ? 'i' : (cx ? 'z' : 'd'); }
  std::string zero() const { return cx ? "cplx{0.0, 0.0}" : "0"; }
  std::string xv(int r) const { return "x" + std::to_string(r); }
  std::string dv(int f) const { return "D" + std::to_string(fac[f].col); }
  std::vector<char> dead;
  bool dead_row(int r) const { return dead[r]; }

  void line(const std::string& s) { o << ind << s << "\n"; }

  // ---- VN primitives -----------------------------------------------------------
  int leaf(const std::string& text, char ty) {
    auto it = leafs.find(text);
    if (it != leafs.end()) return it->second;
    vals.push_back({'L', -1, -1, -1, ty, text});
    return leafs[text] = (int)vals.size() - 1;
  }
  int lit(double v) { return leaf(hexlit(v), 'd'); }
  int zlit(zd v) {
    const int id = leaf("cplx{" + hexlit(v.real()) + ", " + hexlit(v.imag()) + "}", 'z');
    if (v.imag() == 0.0) { vals[id].real_lit = true; vals[id].re = v.real(); }
    return id;
  }
  int vlit(zd v) { return cx ? zlit(v) : lit(v.real()); }  // value literal of the sweep's type
  int ilit(long long v) {
    const int id = leaf(std::to_string(v), 'i');
    vals[id].lb = v == 0 ? -100.0 : std::log2(std::fabs((double)v));
    return id;
  }
  const std::string& nm(int id) const { return vals[id].name; }

  // ---- INT01 bound-typed integers ------------------------------------------------
  // Doubled row values are tiny (|x'_r| <= r_r, the row's nonzero count), so
  // most products fit 32 or 64 bits.  Every value carries log2 of a bound on
  // its magnitude; an op runs in the narrowest of int / long long / wrapping
  // u128 that holds its bound (never narrower than its operands).  Exact
  // while no int/long long overflows; u128 is the ring Z/2^128 the result is
  // recovered from.  Loop-carried product registers get their type from the
  // largest bound ever assigned to them (reg_lb, fixed point over
  // generations: generate_kernel reruns when an assignment exceeds it).
  std::map<std::string, double> reg_lb;   // input: register -> assumed bound
  std::map<std::string, double> reg_seen; // output: register -> largest assigned bound
  std::vector<double> row_lb;             // row -> log2(max(nnz in row, 1))
  static char ity(double lb) { return lb <= 30.9 ? 'i' : (lb <= 62.9 ? 'l' : 'u'); }
  static int irank(char t) { return t == 'i' ? 0 : (t == 'l' ? 1 : 2); }
  static double lsum(double a, double b) {  // log2(2^a + 2^b)
    const double m = std::max(a, b);
    return m >= 1e8 ? 1e9 : m + std::log2(1.0 + std::exp2(std::min(a, b) - m));
  }
  std::string icast(int v, char rt) const {
    const char t = vals[v].ty;
    if (t == rt) return nm(v);
    if (rt == 'l') return "(i64)" + nm(v);
    return "(u128)(i128)" + nm(v);
  }
  double reg_bound(const std::string& r) const {
    auto it = reg_lb.find(r);
    return it == reg_lb.end() ? 1e9 : it->second;
  }
  char reg_ty(const std::string& r) const { return r == "cacc" ? 'u' : ity(reg_bound(r)); }
  std::string rty(const std::string& r) const { return i01 ? tyname(reg_ty(r)) : std::string(PT()); }

  int reg(const std::string& r, char ty) {
    auto it = cur.find(r);
    if (it != cur.end()) return it->second;
    if (i01 && ty == 'u') {  // product register: typed by its bound
      const int id = leaf(r, reg_ty(r));
      vals[id].lb = r == "cacc" ? 1e9 : reg_bound(r);
      return cur[r] = id;
    }
    const int id = leaf(r, ty);
    if (i01 && ty == 'i' && r.size() > 1 && r[0] == 'x') vals[id].lb = row_lb[std::atoi(r.c_str() + 1)];
    return cur[r] = id;
  }
  void set(const std::string& r, int id) {
    cur[r] = id;
    dirty.insert(r);
    if (i01 && r[0] != 'x' && r != "cacc") {  // product registers: record the assigned bound
      auto it = reg_seen.find(r);
      if (it == reg_seen.end()) reg_seen[r] = vals[id].lb;
      else it->second = std::max(it->second, vals[id].lb);
    }
  }
  // semantic bounds of the loop-carried product registers (mirror the
  // expressions node_value / recompute_* emit; set() records any excess and
  // generate_kernel then regenerates with the larger bound)
  double node_lb(int id, const std::map<int, zd>& sh) const {
    const Node& N = nodes[id];
    if (N.leaf) return row_lb[N.row];
    if (N.ch.size() == 1 && nodes[N.ch[0]].leaf) return 1.0;  // the constant 2
    auto shift = [&](int r) { auto it = sh.find(r); return it == sh.end() ? 0.0 : it->second.real(); };
    if (N.ch.size() == 2 && nodes[N.ch[0]].leaf && nodes[N.ch[1]].leaf) {
      const int r1 = nodes[N.ch[0]].row, r2 = nodes[N.ch[1]].row;
      const double c = std::fabs(std::llround(2 * shift(r1) + 2 * shift(r2) + 4));
      return lsum(1.0 + lsum(row_lb[r1], row_lb[r2]), c == 0 ? -100.0 : std::log2(c));
    }
    std::map<int, zd> shin = sh;
    for (auto& kv : colval[N.col]) shin[kv.first] += zd(2.0);
    double in = 0, out = 0;
    for (int c : N.ch) {
      in += node_lb(c, shin);
      out += node_lb(c, sh);
    }
    return lsum(in, out);
  }
  void init_reg_bounds() {
    auto fb = [&](int f) {
      const Factor& F = fac[f];
      if (!F.group) return row_lb[F.rows[0]];
      if (F.constant()) return 1.0;
      return node_lb(F.node, {});
    };
    for (int f = 0; f < (int)fac.size(); ++f) {
      if (!fac[f].group || fac[f].constant()) continue;
      reg_lb[dv(f)] = fb(f);
      const int m = (int)cc[f].lev.size();
      std::vector<double> qi(m, 0), qo(m, 0);
      const std::map<int, zd> shin = cc_shift(f);
      for (int i = 0; i < m; ++i)
        for (int c : cc[f].ch[i]) {
          qi[i] += node_lb(c, shin);
          qo[i] += node_lb(c, {});
        }
      double si = 0, so = 0;
      for (int i = m - 1; i >= 0; --i) {
        si += qi[i];
        so += qo[i];
        reg_lb[ccn("qI", f, i)] = qi[i];
        reg_lb[ccn("qO", f, i)] = qo[i];
        reg_lb[ccn("sI", f, i)] = si;
        reg_lb[ccn("sO", f, i)] = so;
      }
    }
    double frozen = 0;
    for (int f = 0; f < (int)fac.size(); ++f)
      if (fac[f].level < 0) frozen += fb(f);
    reg_lb["F"] = frozen;
    double above_lb = has_frozen ? frozen : 0.0;
    for (auto it = nonempty.rbegin(); it != nonempty.rend(); ++it) {
      double q = 0;
      for (int f : G[*it]) q += fb(f);
      reg_lb["Q" + std::to_string(*it)] = q;
      above_lb += q;
      reg_lb["S" + std::to_string(*it)] = above_lb;
    }
  }
  int mk(char op, int a, int b, int c = -1) {
    if ((op == '+' || op == '*') && a > b) std::swap(a, b);
    auto key = std::make_tuple(op, a, b, c);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    char ty = vals[a].ty;
    const bool z = vals[a].ty == 'z' || (b >= 0 && vals[b].ty == 'z') || (c >= 0 && vals[c].ty == 'z');
    std::string expr;
    double w = 1;  // executed DP instructions
    if (z) {  // complex: cplx helpers of the generated prelude (1, 2 or 4 DP instructions)
      ty = 'z';
      // a literal with zero imaginary part multiplies / adds as a real number
      auto rl = [&](int v) { return vals[v].real_lit; };
      auto rs = [&](int v) { return hexlit(vals[v].re); };
      switch (op) {
        case '+':
          if (rl(b)) { expr = "caddr(" + nm(a) + ", " + rs(b) + ")"; w = 1; }
          else if (rl(a)) { expr = "caddr(" + nm(b) + ", " + rs(a) + ")"; w = 1; }
          else { expr = "cadd(" + nm(a) + ", " + nm(b) + ")"; w = 2; }
          break;
        case '-':
          if (rl(b)) { expr = "caddr(" + nm(a) + ", -" + rs(b) + ")"; w = 1; }
          else { expr = "csub(" + nm(a) + ", " + nm(b) + ")"; w = 2; }
          break;
        case '*':
          if (vals[a].ty == 'd') { expr = "cscale(" + nm(a) + ", " + nm(b) + ")"; w = 2; }
          else if (vals[b].ty == 'd') { expr = "cscale(" + nm(b) + ", " + nm(a) + ")"; w = 2; }
          else if (rl(a)) { expr = "cscale(" + rs(a) + ", " + nm(b) + ")"; w = 2; }
          else if (rl(b)) { expr = "cscale(" + rs(b) + ", " + nm(a) + ")"; w = 2; }
          else { expr = "cmul(" + nm(a) + ", " + nm(b) + ")"; w = 4; }
          break;
        case 'f':
          if (vals[a].ty == 'd' && rl(b)) {  // s * (real a) + x: only the real part moves
            expr = "cfmar(" + nm(a) + ", " + rs(b) + ", " + nm(c) + ")"; w = 1;
          } else if (vals[a].ty == 'd') {
            expr = "cfma_s(" + nm(a) + ", " + nm(b) + ", " + nm(c) + ")"; w = 2;
          } else if (rl(a)) {
            expr = "cfma_s(" + rs(a) + ", " + nm(b) + ", " + nm(c) + ")"; w = 2;
          } else {
            expr = "cfma(" + nm(a) + ", " + nm(b) + ", " + nm(c) + ")"; w = 4;
          }
          break;
      }
    } else if (i01) {
      const double la = vals[a].lb, lbv = b >= 0 ? vals[b].lb : -100.0;
      double lr = op == '*' ? la + lbv : (op == 'h' ? la + 1.0 : lsum(la, lbv));
      char rt = ity(lr);
      if (irank(vals[a].ty) > irank(rt)) rt = vals[a].ty;
      if (b >= 0 && irank(vals[b].ty) > irank(rt)) rt = vals[b].ty;
      if (rt == 'u') lr = std::min(lr, 1e9);
      ty = rt;
      switch (op) {
        case '+': expr = icast(a, rt) + " + " + icast(b, rt); break;
        case '-': expr = icast(a, rt) + " - " + icast(b, rt); break;
        case '*':
          if (rt == 'u' && asm_mul && ((vals[a].ty == 'i' && vals[b].ty == 'u') || (vals[b].ty == 'i' && vals[a].ty == 'u')))
            expr = vals[a].ty == 'i' ? "mul_s32_u128(" + nm(a) + ", " + nm(b) + ")"
                                     : "mul_s32_u128(" + nm(b) + ", " + nm(a) + ")";
          else
            expr = icast(a, rt) + " * " + icast(b, rt);
          break;
        case 'h': expr = "2 * " + icast(a, rt); break;
      }
      ops += w;
      std::string name = "t" + std::to_string(tmp++);
      wt[name] = w;
      line(std::string("const ") + tyname(ty) + " " + name + " = " + expr + ";");
      Val v{op, a, b, c, ty, name};
      v.lb = lr;
      vals.push_back(v);
      return memo[key] = (int)vals.size() - 1;
    } else {
      switch (op) {
        case '+': expr = nm(a) + " + " + nm(b); break;
        case '-': expr = nm(a) + " - " + nm(b); break;
        case '*': expr = nm(a) + " * " + nm(b); break;
        case 'f': expr = "fma(" + nm(a) + ", " + nm(b) + ", " + nm(c) + ")"; break;
      }
    }
    ops += w;
    std::string name = "t" + std::to_string(tmp++);
    wt[name] = w;
    line(std::string("const ") + tyname(ty) + " " + name + " = " + expr + ";");
    vals.push_back({op, a, b, c, ty, name});
    return memo[key] = (int)vals.size() - 1;
  }
  int add(int a, int b) { return mk('+', a, b); }
  int sub(int a, int b) { return mk('-', a, b); }
  int mul(int a, int b) {
    if (a < 0) return b;
    if (b < 0) return a;
    return mk('*', a, b);
  }
  int prod(std::vector<int> v) {  // balanced tree in fixed (list) order
    if (v.empty()) return -1;
    while (v.size() > 1) {
      std::vector<int> w;
      for (size_t i = 0; i + 1 < v.size(); i += 2) w.push_back(mul(v[i], v[i + 1]));
      if (v.size() & 1) w.push_back(v.back());
      v.swap(w);
    }
    return v[0];
  }
  void begin_region() {
    memo.clear();
    leafs.clear();
    cur.clear();
    dirty.clear();
  }
  // region marker for the post-pass: ops of region k execute `weight` times per chunk
  std::vector<double> region_weight;
  void mark_region(double weight) {
    o << "//@R" << region_weight.size() << "\n";
    region_weight.push_back(weight);
  }

  void end_region() {  // write loop-carried registers (and tier rows) back
    std::vector<int> tier_dirty;
    for (const std::string& r : dirty) {
      const int id = cur[r];
      auto t = tier_of.find(r);
      if (t != tier_of.end()) {
        tier_dirty.push_back(tier_row[t->second]);
        continue;
      }
      if (vals[id].op == 'L' && vals[id].name == r) continue;
      line(r + " = " + nm(id) + ";");
    }
    tier_store(tier_dirty, [&](int row) { return cur[xv(row)]; });
    dirty.clear();
  }

  // ---- factors, levels, products -------------------------------------------------
  int xval(int r) {
    if (tier_slot[r] < 0) return reg(xv(r), xty());
    auto it = cur.find(xv(r));
    if (it != cur.end()) return it->second;
    const int q = tier_partner(r);
    if (q >= 0 && !cur.count(xv(q))) {  // one vector load for the row pair
      const int lo = tier_slot[r] < tier_slot[q] ? r : q, hi = lo == r ? q : r;
      const std::string v = "tv" + std::to_string(tmp++);
      line(std::string("const ") + VT2() + " " + v + " = TIER2(" + std::to_string(tier_slot[lo] >> 1) + ");");
      for (int k = 0; k < 2; ++k) {
        const std::string name = "t" + std::to_string(tmp++);
        line(std::string("const ") + VT() + " " + name + " = " + v + (k ? ".y;" : ".x;"));
        vals.push_back({'M', -1, -1, -1, xty(), name});
        cur[xv(k ? hi : lo)] = (int)vals.size() - 1;
      }
      return cur[xv(r)];
    }
    std::string name = "t" + std::to_string(tmp++);  // tier load (coalesced across lanes)
    line(std::string("const ") + VT() + " " + name + " = TIER(" + std::to_string(tier_slot[r]) + ");");
    vals.push_back({'M', -1, -1, -1, xty(), name});
    return cur[xv(r)] = (int)vals.size() - 1;
  }
  int pval(int r) { return xval(r); }  // row value (INT01: widened by the ops that use it)
  // value of elimination-tree node `id` with row shifts `sh` (ancestors'
  // eliminated columns switched in; INT01 shifts in doubled units)
  int node_value(int id, const std::map<int, zd>& sh) {
    const Node& N = nodes[id];
    auto shift = [&](int r) { auto it = sh.find(r); return it == sh.end() ? zd(0.0) : it->second; };
    if (N.leaf) {
      const zd s = shift(N.row);
      if (i01) {
        if (s == zd(0.0)) return pval(N.row);
        const int v = add(xval(N.row), ilit(std::llround(s.real())));
        vals[v].lb = std::min(vals[v].lb, row_lb[N.row]);  // another state of row N.row: |.| <= r
        return v;
      }
      return s == zd(0.0) ? xval(N.row) : add(xval(N.row), vlit(s));
    }
    const std::map<int, zd>& cv = colval[N.col];
    if (N.ch.size() == 1 && nodes[N.ch[0]].leaf)  // (y + s + a) - (y + s) = a exactly
      return i01 ? ilit(2) : vlit(cv.at(nodes[N.ch[0]].row));
    if (N.ch.size() == 2 && nodes[N.ch[0]].leaf && nodes[N.ch[1]].leaf) {
      const int r1 = nodes[N.ch[0]].row, r2 = nodes[N.ch[1]].row;
      const zd s1 = shift(r1), s2 = shift(r2);
      if (i01) {  // (x1+s1+2)(x2+s2+2) - (x1+s1)(x2+s2) = 2 (x1 + x2) + (2 s1 + 2 s2 + 4)
        int t = mk('h', add(xval(r1), xval(r2)), -1);
        return add(t, ilit(std::llround(2 * s1.real() + 2 * s2.real() + 4)));
      }
      // a1 (y2 + s2) + a2 (y1 + s1) + a1 a2: two FMAs, no cancellation
      const zd a1 = cv.at(r1), a2 = cv.at(r2);
      return mk('f', vlit(a1), xval(r2), mk('f', vlit(a2), xval(r1), vlit(a1 * a2 + a1 * s2 + a2 * s1)));
    }
    std::map<int, zd> shin = sh;
    for (auto& kv : cv) shin[kv.first] += i01 ? zd(2.0) : kv.second;
    std::vector<int> in, out;
    for (int c : N.ch) {
      in.push_back(node_value(c, shin));
      out.push_back(node_value(c, sh));
    }
    return sub(prod(in), prod(out));
  }
  int group_value(int f) { return node_value(fac[f].node, {}); }
  int fval(int f) {  // current value of factor f
    const Factor& F = fac[f];
    if (!F.group) return pval(F.rows[0]);
    if (F.constant()) return group_value(f);  // literal a_rc
    if (tierf(f) || zs0(f)) return group_value(f);  // tier / zero-skip level-0 groups: no register
    return reg(dv(f), pty());
  }
  bool zs = false;  // INT01 block-level zero skip (block_zero_skip_body)
  bool zs0(int) const { return false; }
  bool qreg(int l) const { return G[l].size() >= 2; }
  int qval(int l) { return qreg(l) ? reg("Q" + std::to_string(l), pty()) : fval(G[l][0]); }
  int next_level(int l) const {
    for (int m : nonempty)
      if (m > l) return m;
    return -1;
  }
  bool sreg(int l) const { return next_level(l) >= 0 || has_frozen || has_tier(); }
  int sval(int l) { return sreg(l) ? reg("S" + std::to_string(l), pty()) : qval(l); }
  int above(int l) {  // -1 = the empty product
    int m = next_level(l);
    if (m >= 0) return sval(m);
    if (has_tier()) return reg("SG", pty());  // the paper's globalProduct (tier x frozen)
    return has_frozen ? reg("F", pty()) : -1;
  }
  void recompute_sg() {  // product of every tier factor (rows loaded from the tier) and F
    std::vector<int> v;
    for (int l : tier_levels)
      for (int f : G[l]) v.push_back(fval(f));
    if (has_frozen) v.push_back(reg("F", pty()));
    set("SG", prod(v));
  }
  void recompute_q(int l) {
    if (!qreg(l)) return;
    std::vector<int> v;
    for (int f : G[l]) v.push_back(fval(f));
    set("Q" + std::to_string(l), prod(v));
  }
  void recompute_s(int l) {  // l >= 1
    if (!sreg(l)) return;
    set("S" + std::to_string(l), mul(qval(l), above(l)));
  }
  void recompute_factor(int f) {
    const Factor& F = fac[f];
    if (!F.group || F.constant() || tierf(f) || zs0(f)) return;
    if (ccon(f)) { cc_update(f, {}, true); return; }
    set(dv(f), group_value(f));
  }

  // ---- composite caches (DESIGN 3.12): for a register-resident composite root
  // E = prod_c c(in) - prod_c c(out), its direct children are grouped by the
  // lowest in-chunk swept bit touching them; level products (in/out) and
  // suffix products over child levels are cached, so a flip re-evaluates only
  // the touched children and the suffix chain below them.
  struct CCache {
    std::vector<int> lev;                // distinct child levels, ascending (B = never in-chunk)
    std::vector<std::vector<int>> ch;    // children per level
    std::map<int, int> idx_of_child;     // child node -> level index
  };
  std::vector<CCache> cc;
  std::vector<int> cc_child_of_row;      // row -> direct child (of its root) containing it
  bool ccon(int f) const {
    if (!S.cc || !fac[f].group || fac[f].constant() || fac[f].level < 0 || tierf(f) || cc[f].lev.size() < 2)
      return false;
    const Node& N = nodes[fac[f].node];  // two-leaf roots keep their 2-FMA closed form
    return !(N.ch.size() == 2 && nodes[N.ch[0]].leaf && nodes[N.ch[1]].leaf);
  }
  // rows changed by a flip -> composite-cache updates (touched level indices)
  void update_factors(const std::map<int, std::vector<int>>& rows_by_fac) {
    for (auto& kv : rows_by_fac) {
      const int f = kv.first;
      if (!ccon(f)) { recompute_factor(f); continue; }
      std::set<int> touched;
      for (int r : kv.second) touched.insert(cc[f].idx_of_child.at(cc_child_of_row[r]));
      cc_update(f, touched, false);
    }
  }
  std::string ccn(const char* t, int f, int i) const {
    return std::string(t) + std::to_string(fac[f].col) + "_" + std::to_string(i);
  }
  bool cc_qreg(int f, int i) const {  // cache the level product unless it is a single leaf
    return cc[f].ch[i].size() > 1 || !nodes[cc[f].ch[i][0]].leaf;
  }
  std::map<int, zd> cc_shift(int f) {  // the root's column switched in
    std::map<int, zd> s;
    for (auto& kv : colval[fac[f].col]) s[kv.first] = i01 ? zd(2.0) : kv.second;
    return s;
  }
  int cc_levprod(int f, int i, bool in) {  // product of the children at level index i, fresh
    std::vector<int> v;
    const std::map<int, zd> sh = in ? cc_shift(f) : std::map<int, zd>();
    for (int c : cc[f].ch[i]) v.push_back(node_value(c, sh));
    return prod(v);
  }
  int cc_q(int f, int i, bool in) {
    if (cc_qreg(f, i)) return reg(ccn(in ? "qI" : "qO", f, i), pty());
    return cc_levprod(f, i, in);
  }
  int cc_s(int f, int i, bool in) {  // suffix product over levels >= i
    if (i + 1 >= (int)cc[f].lev.size()) return cc_q(f, i, in);
    return reg(ccn(in ? "sI" : "sO", f, i), pty());
  }
  // touched: level indices whose children changed; all = recompute every level
  void cc_update(int f, const std::set<int>& touched, bool all) {
    const int m = (int)cc[f].lev.size();
    int h = -1;
    for (int i = 0; i < m; ++i) {
      if (!all && !touched.count(i)) continue;
      h = std::max(h, i);
      if (cc_qreg(f, i)) {
        set(ccn("qI", f, i), cc_levprod(f, i, true));
        set(ccn("qO", f, i), cc_levprod(f, i, false));
      }
    }
    for (int i = std::min(h, m - 2); i >= 0; --i) {
      set(ccn("sI", f, i), mul(cc_q(f, i, true), cc_s(f, i + 1, true)));
      set(ccn("sO", f, i), mul(cc_q(f, i, false), cc_s(f, i + 1, false)));
    }
    set(dv(f), sub(cc_s(f, 0, true), cc_s(f, 0, false)));
  }
  void build_cc() {
    cc.assign(fac.size(), {});
    cc_child_of_row.assign(n, -1);
    std::vector<int> rowlev(n, B);
    for (int b = B - 1; b >= 0; --b)
      for (auto& kv : colval[K + b]) rowlev[kv.first] = b;
    std::function<void(int, int, int&)> scan = [&](int nd, int top, int& lv) {
      if (nodes[nd].leaf) {
        lv = std::min(lv, rowlev[nodes[nd].row]);
        cc_child_of_row[nodes[nd].row] = top;
        return;
      }
      for (int c : nodes[nd].ch) scan(c, top, lv);
    };
    for (int f = 0; f < (int)fac.size(); ++f) {
      if (!fac[f].group || fac[f].constant()) continue;
      std::map<int, std::vector<int>> bylev;
      for (int c : nodes[fac[f].node].ch) {
        int lv = B;
        scan(c, c, lv);
        bylev[lv].push_back(c);
      }
      for (auto& kv : bylev) {
        for (int c : kv.second) cc[f].idx_of_child[c] = (int)cc[f].lev.size();
        cc[f].lev.push_back(kv.first);
        cc[f].ch.push_back(kv.second);
      }
    }
  }

  // one update y_r +-= a_rj.  sign: "+", "-" (static) or a runtime +-1 register
  void update(int r, int pos, const std::string& sign) {  // pos: CCS position of a_rj
    if (dead_row(r)) return;  // only enters through the constant D_k = a_rk
    const zd a(A.val[pos], A.im(pos));
    int x = xval(r), y;
    if (i01) {
      if (sign == "+") y = add(x, ilit(2));
      else if (sign == "-") y = sub(x, ilit(2));
      else y = add(x, reg(sign, 'i'));  // runtime sign register holds +-2
    } else {
      if (sign == "+") y = add(x, vlit(a));
      else if (sign == "-") y = sub(x, vlit(a));
      else y = mk('f', reg(sign, 'd'), vlit(a), x);
    }
    set(xv(r), y);
  }

  // flip of swept bit b (column K+b): touched factors, their levels, suffix chain
  void flip(int b, const std::string& sign) {
    const int j = K + b;
    std::set<int> facs, levels;
    std::map<int, std::vector<int>> rows_by_fac;
    for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) {
      update(A.idx[p], p, sign);
      facs.insert(fac_of_row[A.idx[p]]);
      if (!dead_row(A.idx[p])) rows_by_fac[fac_of_row[A.idx[p]]].push_back(A.idx[p]);
    }
    update_factors(rows_by_fac);
    bool tier_touched = false;
    for (int f : facs) {
      if (fac[f].level < 0) continue;  // constant D_k: unchanged
      if (tierf(f)) tier_touched = true;
      else levels.insert(fac[f].level);
    }
    for (int l : levels) recompute_q(l);
    int h = levels.empty() ? -1 : *levels.rbegin();
    if (tier_touched) {
      recompute_sg();
      h = nonempty.empty() ? -1 : nonempty.back();
    }
    for (auto it = nonempty.rbegin(); it != nonempty.rend(); ++it)
      if (*it >= 1 && *it <= h) recompute_s(*it);
  }

  // ---- the block body: 2^U h-steps, pairs (2k, 2k+1) -------------------------
  // INT01 zero tracking (Sec. VI-B: "In the presence of a zero, all the
  // expensive multiplications and the update on the result ... are skipped"),
  // at block granularity: every term of the block carries the cached product
  // of the factors above the in-block levels (S_U); when it is zero on all 32
  // lanes (warp vote) the block contributes 0 and is replaced by its net
  // effect on y -- over a full reflected Gray block only column U-1 changes
  // state (the lower columns flip an even number of times with alternating
  // signs; exact in integers).  An executed block first refreshes the in-block
  // levels (they may be stale after skipped blocks).
  void block_zero_skip_body() {
    const int su = above(U - 1);
    if (su < 0) { block_body(); return; }
    line("if (__any_sync(0xffffffffu, " + nm(su) + " != 0)) {");
    auto save_memo = memo;
    auto save_cur = cur;
    auto save_leafs = leafs;
    const std::string save_ind = ind;
    ind += "  ";
    // refresh levels < U from y: groups, level products, suffix chain
    for (int l : nonempty) {
      if (l >= U) continue;
      for (int f : G[l]) recompute_factor(f);
      recompute_q(l);
    }
    for (auto it = nonempty.rbegin(); it != nonempty.rend(); ++it)
      if (*it >= 1 && *it < U) recompute_s(*it);
    block_body();
    end_region();
    ind = save_ind;
    memo = save_memo;
    cur = save_cur;
    leafs = save_leafs;
    line("} else {");
    ind += "  ";
    for (int p = A.ptr[K + U - 1]; p < A.ptr[K + U]; ++p) update(A.idx[p], p, "sU");
    end_region();
    ind = save_ind;
    memo = save_memo;
    cur = save_cur;
    leafs = save_leafs;
    line("}");
  }

  void block_body() {
    std::vector<int> stack(U + 1, -1);
    const int npairs = 1 << (U - 1);
    const bool dbg = getenv("PERM_DEBUG_OPS") != nullptr;
    for (int k = 0; k < npairs; ++k) {
      const int u = 2 * k;
      const double ops0 = ops;
      if (u > 0) {
        int b = __builtin_ctz(u);
        std::string sg = (b == U - 1) ? "sU" : (((u >> (b + 1)) & 1) ? "-" : "+");
        flip(b, sg);
        if (dbg) fprintf(stderr, "[ops] pair %d flip bit %d: %.0f\n", k, b, ops - ops0);
      }
      // pair: product at even step u (current state), flip bit 0, product at u+1
      std::string sg0 = (U >= 2) ? ((((u + 1) >> 1) & 1) ? "-" : "+") : "sU";
      const int e = qval(0);
      {
        const int j = K;
        std::map<int, std::vector<int>> rows_by_fac;
        for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) {
          update(A.idx[p], p, sg0);
          if (!dead_row(A.idx[p])) rows_by_fac[fac_of_row[A.idx[p]]].push_back(A.idx[p]);
        }
        update_factors(rows_by_fac);
        recompute_q(0);
      }
      const int d = sub(e, qval(0));
      const int ab = above(0);
      int v;
      int lvl = 0;
      unsigned kk = (unsigned)k;
      if ((kk & 1u) && ab >= 0 && !i01) {
        // first merge of the pairwise tree fused with the pair product (one DFMA)
        v = mk('f', d, ab, stack[0]);
        kk >>= 1;
        ++lvl;
      } else {
        v = mul(d, ab);
      }
      while (kk & 1u) {  // pairwise (binary-counter) accumulation of the pair terms
        v = add(stack[lvl], v);
        kk >>= 1;
        ++lvl;
      }
      stack[lvl] = v;
      if (dbg) fprintf(stderr, "[ops] pair %d total %.0f\n", k, ops - ops0);
    }
    set("cacc", add(reg("cacc", pty()), stack[U - 1]));
  }

  // seed: y = x0 + swept columns of Gray(h0); only bits >= B-1 can be set
  void seed() {
    const int nbits = n - 1 - K;
    line("const u64 gr = h0 ^ (h0 >> 1);");
    mark_region(1.0);
    begin_region();
    for (int r = 0; r < n; ++r) {
      if (dead_row(r)) continue;
      // x0 per row; complex sweeps pass (re, im) pairs
      cur[xv(r)] = i01 ? ilit(std::llround(x0[r])) : (cx ? zlit(zd(x0[2 * r], x0[2 * r + 1])) : lit(x0[r]));
    }
    for (int b = std::max(B - 1, 0); b < nbits; ++b) {
      const int j = K + b;
      bool any = false;
      for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p) any |= !dead_row(A.idx[p]);
      if (!any) continue;
      std::string bn = "b" + std::to_string(b);
      if (i01) {
        line("const int " + bn + " = (int)((gr >> " + std::to_string(b) + ") & 1ull) << 1;");
        vals[leaf(bn, 'i')].lb = 1.0;
        for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p)
          if (!dead_row(A.idx[p])) set(xv(A.idx[p]), add(xval(A.idx[p]), leaf(bn, 'i')));
      } else {
        line("const double " + bn + " = __longlong_as_double((long long)(((gr >> " + std::to_string(b) +
             ") & 1ull) * 0x3FF0000000000000ull));");
        for (int p = A.ptr[j]; p < A.ptr[j + 1]; ++p)
          if (!dead_row(A.idx[p]))
            set(xv(A.idx[p]), mk('f', leaf(bn, 'd'), vlit(zd(A.val[p], A.im(p))), xval(A.idx[p])));
      }
    }
    // frozen product
    int F = -1;
    if (has_frozen) {
      std::vector<int> v;
      for (int f = 0; f < (int)fac.size(); ++f)
        if (fac[f].level < 0) v.push_back(fac[f].group && !fac[f].constant() ? group_value(f) : fval(f));
      F = prod(v);
      line(std::string("const ") + rty("F") + " F = " + nm(F) + ";");
      cur.erase("F");
      reg("F", pty());
    }
    // live groups, level products, suffix chain
    for (int f = 0; f < (int)fac.size(); ++f)
      if (fac[f].group && !fac[f].constant() && fac[f].level >= 0 && !tierf(f) && !zs0(f)) {
        if (ccon(f)) cc_update(f, {}, true);
        else cur[dv(f)] = group_value(f);
      }
    if (has_tier()) recompute_sg();
    for (int l : nonempty)
      if (qreg(l)) {
        std::vector<int> v;
        for (int f : G[l]) v.push_back(fval(f));
        cur["Q" + std::to_string(l)] = prod(v);
      }
    for (auto it = nonempty.rbegin(); it != nonempty.rend(); ++it)
      if (*it >= 1 && sreg(*it)) cur["S" + std::to_string(*it)] = mul(qval(*it), above(*it));
    // declare the loop-carried registers
    std::vector<int> seed_tier;
    for (int r = 0; r < n; ++r) {
      if (dead_row(r) || fac[fac_of_row[r]].level < 0) continue;
      if (tier_slot[r] >= 0) seed_tier.push_back(r);
      else line(std::string(VT()) + " " + xv(r) + " = " + nm(cur[xv(r)]) + ";");
    }
    tier_store(seed_tier, [&](int row) { return cur[xv(row)]; });
    for (int f = 0; f < (int)fac.size(); ++f)
      if (fac[f].group && !fac[f].constant() && fac[f].level >= 0 && !tierf(f) && !zs0(f)) {
        line(rty(dv(f)) + " " + dv(f) + " = " + nm(cur[dv(f)]) + ";");
        if (!ccon(f)) continue;
        const int m = (int)cc[f].lev.size();
        for (int i = 0; i < m; ++i) {
          if (cc_qreg(f, i))
            for (const char* t : {"qI", "qO"})
              line(rty(ccn(t, f, i)) + " " + ccn(t, f, i) + " = " + nm(cur[ccn(t, f, i)]) + ";");
          if (i + 1 < m)
            for (const char* t : {"sI", "sO"})
              line(rty(ccn(t, f, i)) + " " + ccn(t, f, i) + " = " + nm(cur[ccn(t, f, i)]) + ";");
        }
      }
    if (has_tier()) line(std::string(PT()) + " SG = " + nm(cur["SG"]) + ";");
    for (int l : nonempty)
      if (qreg(l)) line(rty("Q" + std::to_string(l)) + " Q" + std::to_string(l) + " = " + nm(cur["Q" + std::to_string(l)]) + ";");
    for (int l : nonempty)
      if (l >= 1 && sreg(l)) line(rty("S" + std::to_string(l)) + " S" + std::to_string(l) + " = " + nm(cur["S" + std::to_string(l)]) + ";");
    (void)F;
    dirty.clear();
  }
};

// ---- whole-kernel post-pass ----------------------------------------------------
// 1. Dead-code elimination.  Composite caches and level registers can end up
//    written but never read (e.g. a composite whose value only enters through
//    its cached in/out suffixes); nvcc would drop them, so W_plan would count
//    instructions that never execute.  Registers with no read and temporaries
//    with no use are removed to a fixpoint.
// 2. FMA contraction (real FP64 only).  With --fmad=false nothing is
//    contracted behind our back, so the generator contracts itself: a product
//    tA = X * Y used exactly once, by tC = tA +- tB (or tB +- tA) in the same
//    straight-line segment (no brace between them), becomes
//    tC = fma(X, Y, +-tB) (or fma(-X, Y, tB)): one DP instruction and one
//    rounding fewer.
// 3. The surviving temporaries' instruction weights give the executed DP
//    instructions per region (W_plan stays equal to ncu's executed count) and
//    the surviving loop-carried registers give the register estimate.
std::atomic<long long> g_pp_ns[4];  // post-pass phases: parse, DCE, FMA contraction, placement + output
struct PostStats {
  std::vector<double> region_ops;
  int reg_words = 0;   // 32-bit words of surviving loop-carried registers
  int fused = 0, removed = 0;
  int smem_bytes = 0;  // per block: loop-carried values moved to shared memory
  int moved = 0;
  int hoisted = 0;     // literals moved to the __constant__ table
  int vol = 0;         // of the moved values: volatile (really in shared memory)
};

// 4. Shared-memory placement.  A loop-carried value (row, composite cache,
//    level/suffix product) that the block body never references is only read
//    and written by the switch cases (once per block at most), yet it would
//    hold registers through the whole body.  Such values live in shared memory
//    instead, one 8/16-byte slot per thread (`SM_name`, conflict-free
//    [slot][thread] layout), which frees the registers the unrolled body
//    needs (at n=40 29 of 68 loop-carried doubles qualify).
PostStats post_pass(std::string& src, const std::map<std::string, double>& wt, size_t nregions, bool fuse,
                    int body_region = -1, int threads = 128, bool hoist_lits = false,
                    const std::vector<double>* region_weight = nullptr, double vol_frac_default = 0.5,
                    bool w_only = false, int smem_ro = 0) {
  PostStats ps;
  ps.region_ops.assign(nregions, 0.0);
  auto tp = [](){ return std::chrono::steady_clock::now(); };
  auto ns = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return (long long)std::chrono::duration_cast<std::chrono::nanoseconds>(b - a).count(); };
  const auto T0 = tp();
  struct Ln {
    std::string_view text;      // the line: a view into src, or into own once rewritten
    std::string own;
    int region = -1, kind = 0;  // 1 const def, 2 register decl, 3 register assign
    int name = -1;              // defined / assigned identifier
    std::vector<int> toks;      // identifier ids on the line (all occurrences)
    bool alive = true;
  };
  // identifiers interned by view (no allocation per token); the names live in
  // a deque, whose elements never move, so the views stay valid
  std::unordered_map<std::string_view, int> ids;
  std::deque<std::string> idname;
  auto intern = [&](std::string_view s) {
    auto it = ids.find(s);
    if (it != ids.end()) return it->second;
    idname.emplace_back(s);
    ids.emplace(std::string_view(idname.back()), (int)idname.size() - 1);
    return (int)idname.size() - 1;
  };
  auto isid0 = [](char c) { return std::isalpha((unsigned char)c) || c == '_'; };
  auto isid = [](char c) { return std::isalnum((unsigned char)c) || c == '_'; };
  std::vector<Ln> L;
  {
    int region = -1;
    L.reserve(std::count(src.begin(), src.end(), '\n') + 1);
    for (size_t b = 0; b < src.size();) {
      size_t e = src.find('\n', b);
      if (e == std::string::npos) e = src.size();
      const std::string_view s(src.data() + b, e - b);
      b = e + 1;
      if (s.compare(0, 3, "//@") == 0) {
        region = std::atoi(std::string(s.substr(4)).c_str());
        continue;
      }
      Ln l;
      l.text = s;
      l.region = region;
      for (size_t i = 0; i < s.size();) {
        if (isid0(s[i]) && (i == 0 || !isid(s[i - 1]))) {
          size_t j = i;
          while (j < s.size() && isid(s[j])) ++j;
          l.toks.push_back(intern(s.substr(i, j - i)));
          i = j;
        } else if (std::isdigit((unsigned char)s[i])) {
          while (i < s.size() && (isid(s[i]) || s[i] == '.')) ++i;
        } else {
          ++i;
        }
      }
      L.push_back(std::move(l));
    }
  }
  const auto T1 = tp();
  g_pp_ns[0] += ns(T0, T1);
  std::vector<int> occ(idname.size(), 0), ndef(idname.size(), 0);
  std::vector<char> is_reg(idname.size(), 0);
  const int id_const = ids.count("const") ? ids.find("const")->second : -2;
  auto tyword = [&](int id) {
    const std::string& w = idname[id];
    return w == "double" || w == "u128" || w == "cplx" || w == "int" || w == "i64";
  };
  for (Ln& l : L) {
    for (int t : l.toks) ++occ[t];
    if (l.region < 0 || l.toks.empty() || l.text.empty() || l.text.back() != ';') continue;
    const size_t eq = l.text.find(" = ");
    if (eq == std::string::npos) continue;
    if (l.toks.size() >= 3 && l.toks[0] == id_const && tyword(l.toks[1])) {
      l.kind = 1;
      l.name = l.toks[2];
    } else if (l.toks.size() >= 2 && tyword(l.toks[0]) && l.region == 0) {
      const std::string& nmv = idname[l.toks[1]];
      if (nmv != "cacc" && nmv != "lacc") {
        l.kind = 2;
        l.name = l.toks[1];
        is_reg[l.name] = 1;
      }
    }
  }
  for (Ln& l : L)
    if (l.kind == 0 && l.region >= 0 && !l.toks.empty() && is_reg[l.toks[0]] && l.text.back() == ';' &&
        l.text.find(" = ") != std::string::npos &&
        l.text.find_first_not_of(' ') == l.text.find(idname[l.toks[0]])) {
      l.kind = 3;
      l.name = l.toks[0];
    }
  for (const Ln& l : L)
    if (l.kind == 2 || l.kind == 3) ++ndef[l.name];
  auto kill = [&](Ln& l) {
    l.alive = false;
    for (int t : l.toks) --occ[t];
    if (l.kind == 2 || l.kind == 3) --ndef[l.name];
    ++ps.removed;
  };
  if (!getenv("PERM_NO_DCE")) {
    for (bool changed = true; changed;) {
      changed = false;
      for (Ln& l : L)  // registers never read
        if (l.alive && (l.kind == 2 || l.kind == 3) && occ[l.name] == ndef[l.name]) {
          kill(l);
          changed = true;
        }
      for (size_t k = L.size(); k-- > 0;) {  // unused temporaries (uses follow definitions)
        Ln& l = L[k];
        if (l.alive && l.kind == 1 && occ[l.name] == 1) {
          kill(l);
          changed = true;
        }
      }
    }
  }
  const auto T2 = tp();
  g_pp_ns[1] += ns(T1, T2);
  if (fuse) {
    std::unordered_map<int, int> def_line;
    std::vector<int> seg(L.size(), 0);
    int sg = 0;
    for (size_t k = 0; k < L.size(); ++k) {
      if (!L[k].alive) continue;
      if (L[k].text.find_first_of("{}") != std::string::npos) ++sg;
      seg[k] = sg;
      if (L[k].kind == 1) def_line[L[k].name] = (int)k;
    }
    const std::string pre = "const double ";
    // "<indent>const double NAME = A op B;" with op one of * + - (views into the line)
    struct Bin { std::string_view a, op, b, indent; };
    auto parse = [&](const Ln& l, Bin& b) {
      const std::string_view t(l.text);
      const size_t p = t.find_first_not_of(' ');
      if (p == std::string_view::npos || t.compare(p, pre.size(), pre) != 0) return false;
      const size_t eq = t.find(" = ", p);
      if (eq == std::string_view::npos || t.size() < eq + 4) return false;
      const std::string_view e = t.substr(eq + 3, t.size() - eq - 4);
      std::string_view tok[4];
      int nt = 0;
      for (size_t i = 0; i < e.size();) {
        if (e[i] == ' ' || e[i] == '\t') { ++i; continue; }
        size_t j = i;
        while (j < e.size() && e[j] != ' ' && e[j] != '\t') ++j;
        if (nt == 3) return false;
        tok[nt++] = e.substr(i, j - i);
        i = j;
      }
      if (nt != 3 || tok[1].size() != 1 || !std::strchr("*+-", tok[1][0])) return false;
      b = {tok[0], tok[1], tok[2], t.substr(0, p)};
      return true;
    };
    auto single_mul = [&](std::string_view v, int sgu, Bin& m) -> int {
      auto it = ids.find(v);
      if (it == ids.end() || occ[it->second] != 2) return -1;
      auto d = def_line.find(it->second);
      if (d == def_line.end() || !L[d->second].alive || seg[d->second] != sgu) return -1;
      if (!parse(L[d->second], m) || m.op != "*") return -1;
      return d->second;
    };
    for (size_t k = 0; k < L.size(); ++k) {
      Ln& l = L[k];
      Bin c, m;
      if (!l.alive || l.kind != 1 || !parse(l, c) || c.op == "*") continue;
      const std::string& name = idname[l.name];
      const char* neg = c.op == "-" ? "-" : "";
      int d = single_mul(c.a, seg[k], m);
      std::string text;
      auto cat = [&text](std::initializer_list<std::string_view> parts) {
        for (std::string_view v : parts) text.append(v.data(), v.size());
      };
      if (d >= 0) {
        cat({c.indent, pre, name, " = fma(", m.a, ", ", m.b, ", ", neg, c.b, ");"});
      } else if ((d = single_mul(c.b, seg[k], m)) >= 0) {
        cat({c.indent, pre, name, " = fma(", neg, m.a, ", ", m.b, ", ", c.a, ");"});
      } else {
        continue;
      }
      // the consumer now reads X, Y instead of tA; the product line goes
      const int ta = L[d].name;
      kill(L[d]);
      --ps.removed;
      for (size_t q = 0; q < l.toks.size(); ++q)
        if (l.toks[q] == ta) {
          l.toks.erase(l.toks.begin() + q);
          --occ[ta];
          break;
        }
      for (std::string_view v : {m.a, m.b})
        if (!v.empty() && isid0(v[0])) {
          const int id = intern(v);
          if (id >= (int)occ.size()) occ.resize(id + 1, 0);
          l.toks.push_back(id);
          ++occ[id];
        }
      ++ps.fused;
      l.own = std::move(text);  // the views in c and m are not used past this point
      l.text = l.own;
    }
  }
  const auto T3 = tp();
  g_pp_ns[2] += ns(T2, T3);
  // ---- 4. shared-memory placement of values the body never references
  std::set<int> moved;
  std::string smem_decl;
  if (body_region >= 0 && !getenv("PERM_NO_SMEM")) {
    std::set<int> in_body;
    for (const Ln& l : L)
      if (l.alive && l.region == body_region) in_body.insert(l.toks.begin(), l.toks.end());
    struct Mv { int id, size; std::string ty; };
    std::vector<Mv> mv;
    const bool all = getenv("PERM_SMEM_ALL") != nullptr;
    // smem_ro (spill escalation): values the body reads but never writes, with
    // at most smem_ro uses in the body, also move -- always volatile, so every
    // body use is an LDS and the value holds no register across the body
    std::set<int> ro_moved;
    if (smem_ro > 0) {
      std::unordered_map<int, int> body_uses;
      std::set<int> body_written;
      for (const Ln& l : L)
        if (l.alive && l.region == body_region) {
          for (int t : l.toks) ++body_uses[t];
          if (l.kind == 3) body_written.insert(l.name);
        }
      for (const Ln& l : L)
        if (l.alive && l.kind == 2 && in_body.count(l.name) && !body_written.count(l.name) &&
            idname[l.name] != "cacc" && idname[l.toks[0]] == "double" && body_uses[l.name] <= smem_ro)
          ro_moved.insert(l.name);
    }
    for (const Ln& l : L)
      if (l.alive && l.kind == 2 && (all || !in_body.count(l.name) || ro_moved.count(l.name)) &&
          idname[l.name] != "cacc") {
        const std::string& ty = idname[l.toks[0]];
        mv.push_back({l.name, ty == "int" ? 4 : ((ty == "double" || ty == "i64") ? 8 : 16), ty});
      }
    std::stable_sort(mv.begin(), mv.end(), [](const Mv& a, const Mv& b) { return a.size > b.size; });
    int off = 0;
    std::ostringstream d;
    d << "extern __shared__ __align__(16) unsigned char sm_[];  // loop-carried values the block body never touches\n";
    // volatile: without it ptxas forwards every slot store to the slot's
    // loads and keeps the value in a register anyway (0 LDS in the SASS), so
    // the placement frees nothing.  A volatile slot really lives in shared
    // memory: an LDS at every read, on the block-boundary path.  So only the
    // cold slots are volatile: those whose switch-case accesses happen in at
    // most a fraction vol_frac of the blocks (case j runs in 2^-(j-U+1) of
    // them); the hot ones stay plain and ptxas keeps them in registers.
    // cplx slots go through a proxy of two volatile doubles (a volatile
    // struct has no assignment operator).
    const double vol_frac = getenv("PERM_SMEM_VOL_FRAC") ? atof(getenv("PERM_SMEM_VOL_FRAC")) : vol_frac_default;
    std::map<int, double> acc_w;  // value -> executions per chunk of the regions touching it (seed excluded)
    if (region_weight && !w_only)  // only the volatile split reads it (not W or the registers)
      for (const Ln& l : L)
        if (l.alive && l.region > 0 && l.region != body_region && l.region < (int)region_weight->size())
          for (int t : std::set<int>(l.toks.begin(), l.toks.end())) acc_w[t] += (*region_weight)[l.region];
    const double body_w =
        (region_weight && body_region >= 0 && body_region < (int)region_weight->size()) ? (*region_weight)[body_region]
                                                                                         : 0.0;
    auto is_vol = [&](int id) {
      if (ro_moved.count(id)) return true;
      if (vol_frac <= 0 || body_w <= 0) return false;
      auto it = acc_w.find(id);
      return (it == acc_w.end() ? 0.0 : it->second) <= vol_frac * body_w * (1 + 1e-9);
    };
    bool any_cx = false;
    for (const Mv& m : mv) any_cx |= m.ty == "cplx" && is_vol(m.id);
    if (any_cx)
      d << "struct vcref { volatile double* p;\n"
           "  __device__ __forceinline__ operator cplx() const { return cplx{p[0], p[1]}; }\n"
           "  __device__ __forceinline__ void operator=(cplx v) const { p[0] = v.re; p[1] = v.im; } };\n";
    for (const Mv& m : mv) {
      const bool vol = is_vol(m.id);
      ps.vol += vol;
      if (vol && m.ty == "cplx")
        d << "#define SM_" << idname[m.id] << " (vcref{((volatile double*)(sm_ + " << off << ")) + 2 * threadIdx.x})\n";
      else
        d << "#define SM_" << idname[m.id] << " (((" << (vol ? "volatile " : "") << m.ty << "*)(sm_ + " << off
          << "))[threadIdx.x])\n";
      off += m.size * threads;
      moved.insert(m.id);
    }
    if (!mv.empty()) {
      smem_decl = d.str();
      ps.smem_bytes = off;
      ps.moved = (int)mv.size();
    }
  }
  auto rename = [&](Ln& l) {  // moved names -> SM_name (declarations become stores)
    std::string t;
    const std::string_view s0 = l.text;
    size_t i = 0;
    if (l.kind == 2 && moved.count(l.name)) {  // "  TYPE name = expr;" -> "  SM_name = expr;"
      const size_t p0 = s0.find_first_not_of(' ');
      const size_t p1 = s0.find(idname[l.name], p0);
      t = std::string(s0.substr(0, p0));
      i = p1;
    }
    while (i < s0.size()) {
      if (isid0(s0[i]) && (i == 0 || !isid(s0[i - 1]))) {
        size_t j = i;
        while (j < s0.size() && isid(s0[j])) ++j;
        const std::string w(s0.substr(i, j - i));
        auto it = ids.find(w);
        if (it != ids.end() && moved.count(it->second)) t += "SM_";
        t += w;
        i = j;
      } else {
        t += s0[i++];
      }
    }
    l.own = std::move(t);
    l.text = l.own;
  };
  // ---- 5. hot literals -> __constant__ table.  sm_100a FP64 instructions
  // take no constant-bank operand: a literal becomes a uniform register
  // built by two UMOVs at every use (31 % of the executed instructions of the
  // n=40 bench kernel).  Literals the block body uses at least twice per
  // iteration go to a __constant__ table instead; ptxas loads those with
  // LDCU and keeps them in uniform registers across the block loop.  The
  // table is capped (the 63 uniform registers hold ~31 doubles, and the
  // UMOV temporaries need some): beyond ~24 entries ptxas spills uniform
  // registers into the register file.
  std::string kc_decl;
  std::unordered_map<std::string, int> kc_index;
  if (hoist_lits && body_region >= 0 && !getenv("PERM_NO_KC")) {
    auto lit_at = [](std::string_view t, size_t i, size_t& a, size_t& e) {  // "(0x..p..)" / "(-0x..p..)"
      if (t[i] != '(') return false;
      size_t j = i + 1;
      if (j < t.size() && t[j] == '-') ++j;
      if (t.compare(j, 2, "0x") != 0) return false;
      a = j;
      size_t k = j + 2;
      while (k < t.size() && (std::isxdigit((unsigned char)t[k]) || t[k] == '.')) ++k;
      if (k >= t.size() || t[k] != 'p') return false;
      ++k;
      if (k < t.size() && (t[k] == '+' || t[k] == '-')) ++k;
      while (k < t.size() && std::isdigit((unsigned char)t[k])) ++k;
      if (k >= t.size() || t[k] != ')') return false;
      e = k;
      return true;
    };
    std::map<std::string, int> cnt;
    for (const Ln& l : L)
      if (l.alive && l.region == body_region)
        for (size_t i = 0, a, e; i < l.text.size(); ++i)
          if (lit_at(l.text, i, a, e)) {
            ++cnt[std::string(l.text.substr(a, e - a))];
            i = e;
          }
    std::vector<std::pair<int, std::string>> hot;
    for (auto& kv : cnt)
      if (kv.second >= 2) hot.push_back({-kv.second, kv.first});
    std::stable_sort(hot.begin(), hot.end());
    const int cap = getenv("PERM_KC_CAP") ? atoi(getenv("PERM_KC_CAP")) : 24;
    if ((int)hot.size() > cap) hot.resize(cap);
    if (!hot.empty()) {
      std::ostringstream d;
      d << "__constant__ double kc_[" << hot.size() << "] = {";
      for (size_t q = 0; q < hot.size(); ++q) {
        kc_index[hot[q].second] = (int)q;
        d << (q ? ", " : "") << hot[q].second;
      }
      d << "};  // body literals used >= 2 times per block (LDCU + uniform registers instead of UMOV pairs)\n";
      kc_decl = d.str();
      for (Ln& l : L) {
        if (!l.alive || l.region < 0) continue;
        std::string t;
        bool any = false;
        for (size_t i = 0, a, e; i < l.text.size(); ++i) {
          if (lit_at(l.text, i, a, e)) {
            auto it = kc_index.find(std::string(l.text.substr(a, e - a)));
            if (it != kc_index.end()) {
              t += '(';
              t.append(l.text.data() + i + 1, a - i - 1);  // sign
              t += "kc_[" + std::to_string(it->second) + "])";
              i = e;
              any = true;
              continue;
            }
          }
          t += l.text[i];
        }
        if (any) {
          l.own = std::move(t);
          l.text = l.own;
        }
      }
      ps.hoisted = (int)hot.size();
    }
  }
  if (w_only) {  // planner scoring: the per-region counts and registers, no source text
    for (const Ln& l : L) {
      if (!l.alive) continue;
      if (l.kind == 1 && l.region >= 0 && l.region < (int)nregions) {
        auto it = wt.find(idname[l.name]);
        if (it != wt.end()) ps.region_ops[l.region] += it->second;
      }
      if (l.kind == 2 && !moved.count(l.name)) {
        const std::string& ty = idname[l.toks[0]];
        ps.reg_words += ty == "int" ? 1 : ((ty == "double" || ty == "i64") ? 2 : 4);
      }
    }
    g_pp_ns[3] += ns(T3, tp());
    return ps;
  }
  std::string out;
  out.reserve(src.size() + smem_decl.size() + kc_decl.size());
  for (Ln& l : L) {
    if (!l.alive) continue;
    if (!moved.empty()) {
      bool hit = false;
      for (int tk : l.toks) hit |= moved.count(tk) > 0;
      if (hit) rename(l);
    }
    if (l.text.compare(0, 10, "extern \"C\"") == 0) {
      out += smem_decl;
      out += kc_decl;
    }
    out += l.text;
    out += '\n';
    if (l.kind == 1 && l.region >= 0 && l.region < (int)nregions) {
      auto it = wt.find(idname[l.name]);
      if (it != wt.end()) ps.region_ops[l.region] += it->second;
    }
    if (l.kind == 2 && !moved.count(l.name)) {
      const std::string& ty = idname[l.toks[0]];
      ps.reg_words += ty == "int" ? 1 : ((ty == "double" || ty == "i64") ? 2 : 4);
    }
  }
  src.swap(out);
  g_pp_ns[3] += ns(T3, tp());
  if (getenv("PERM_DEBUG_POST"))
    fprintf(stderr, "[post] lines %zu regions %zu removed %d fused %d regwords %d smem %d B (%d values)\n",
            L.size(), nregions, ps.removed, ps.fused, ps.reg_words, ps.smem_bytes, ps.moved);
  return ps;
}

}  // namespace

double w_alg1(const Csx& A) {
  const int n = A.n;
  if (n < 2) return 0;
  const double denom = std::ldexp(1.0, n - 1) - 1.0;
  double w = 0;
  for (int j = 0; j + 1 < n; ++j) w += std::ldexp(1.0, n - j - 2) / denom * (A.ptr[j + 1] - A.ptr[j]);
  return w + (n - 1) + 1;
}

KernelCode generate_kernel_once(const Csx& A, const std::vector<double>& x0, const KernelSpec& S,
                                std::map<std::string, double>& excess);

KernelCode generate_kernel(const Csx& A, const std::vector<double>& x0, const KernelSpec& S0) {
  // INT01: regenerate while an assignment exceeds a register's semantic bound
  // (never expected; the bounds mirror the emitted expressions)
  std::map<std::string, double> extra;
  KernelSpec S = S0;
  for (int iter = 0;; ++iter) {
    std::map<std::string, double> excess;
    S.reg_lb_extra = &extra;
    KernelCode kc = generate_kernel_once(A, x0, S, excess);
    if (excess.empty() || iter >= 6) return kc;
    for (auto& kv : excess) extra[kv.first] = std::max(extra[kv.first], kv.second);
  }
}

std::atomic<long long> g_gen_ns{0}, g_post_ns{0}, g_gen_calls{0};
void codegen_timing(double& gen_ms, double& post_ms, long long& calls) {
  if (getenv("PERM_DEBUG_TIMING"))
    fprintf(stderr, "[timing] post-pass phases ms: parse %.1f dce %.1f fuse %.1f place+out %.1f\n", g_pp_ns[0] * 1e-6,
            g_pp_ns[1] * 1e-6, g_pp_ns[2] * 1e-6, g_pp_ns[3] * 1e-6);
  gen_ms = g_gen_ns.load() * 1e-6;
  post_ms = g_post_ns.load() * 1e-6;
  calls = g_gen_calls.load();
}

KernelCode generate_kernel_once(const Csx& A, const std::vector<double>& x0, const KernelSpec& S,
                                std::map<std::string, double>& excess) {
  const auto t_gen0 = std::chrono::steady_clock::now();
  struct GenTimer {
    std::chrono::steady_clock::time_point t0;
    ~GenTimer() {
      g_gen_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
      ++g_gen_calls;
    }
  } gen_timer{t_gen0};
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
  if (g.cx)  // complex sweep helpers: each op is 2 or 4 DP instructions (counted as such)
    o << "struct cplx { double re, im; };\n"
         "__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }\n"
         "__device__ __forceinline__ cplx csub(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }\n"
         "__device__ __forceinline__ cplx cneg(cplx a) { return cplx{-a.re, -a.im}; }\n"
         "__device__ __forceinline__ cplx caddr(cplx a, double r) { return cplx{a.re + r, a.im}; }\n"
         "__device__ __forceinline__ cplx cfmar(double s, double r, cplx x) { return cplx{fma(s, r, x.re), x.im}; }\n"
         "__device__ __forceinline__ cplx cmul(cplx a, cplx b) {\n"
         "  return cplx{fma(a.re, b.re, -(a.im * b.im)), fma(a.re, b.im, a.im * b.re)}; }\n"
         "__device__ __forceinline__ cplx cscale(double s, cplx a) { return cplx{s * a.re, s * a.im}; }\n"
         "__device__ __forceinline__ cplx cfma_s(double s, cplx a, cplx x) {\n"
         "  return cplx{fma(s, a.re, x.re), fma(s, a.im, x.im)}; }\n"
         "__device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx c) {\n"
         "  return cplx{fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))}; }\n";
  if (g.i01) o << "typedef unsigned __int128 u128;\ntypedef __int128 i128;\ntypedef long long i64;\n";
  if (g.i01 && S.i01_asm_mul)
    // a * b mod 2^128 for a signed 32-bit b: a * (uint32)b as four 32x32
    // partial products chained through the carry flag, minus (a << 32) when
    // b < 0 (~12 integer instructions; nvcc's generic sign-extended 128-bit
    // multiply is ~17)
    o << "__device__ __forceinline__ u128 mul_s32_u128(int b, u128 a) {\n"
         "  unsigned a0 = (unsigned)a, a1 = (unsigned)(a >> 32), a2 = (unsigned)(a >> 64), a3 = (unsigned)(a >> 96);\n"
         "  unsigned r0, r1, r2, r3;\n"
         "  const unsigned ub = (unsigned)b, m = (unsigned)(b >> 31);\n"
         "  asm(\"mul.lo.u32 %0, %4, %8;\\n\\tmul.hi.u32 %1, %4, %8;\\n\\tmad.lo.cc.u32 %1, %5, %8, %1;\\n\\t\"\n"
         "      \"madc.hi.u32 %2, %5, %8, 0;\\n\\tmad.lo.cc.u32 %2, %6, %8, %2;\\n\\tmadc.hi.u32 %3, %6, %8, 0;\\n\\t\"\n"
         "      \"mad.lo.u32 %3, %7, %8, %3;\\n\\tand.b32 %4, %4, %9;\\n\\tand.b32 %5, %5, %9;\\n\\tand.b32 %6, %6, %9;\\n\\t\"\n"
         "      \"sub.cc.u32 %1, %1, %4;\\n\\tsubc.cc.u32 %2, %2, %5;\\n\\tsubc.u32 %3, %3, %6;\"\n"
         "      : \"=&r\"(r0), \"=&r\"(r1), \"=&r\"(r2), \"=&r\"(r3), \"+r\"(a0), \"+r\"(a1), \"+r\"(a2) : \"r\"(a3), \"r\"(ub), \"r\"(m));\n"
         "  return ((u128)(((unsigned long long)r3 << 32) | r2) << 64) | (((unsigned long long)r1 << 32) | r0);\n"
         "}\n";
  // HYBRID tier: the paper's coalesced x[nthreads * row + tid] layout (Listing 4,
  // P:543-550), vectorised: row slots 2p, 2p+1 of a thread form one double2
  // (int2) at pair index p * (all threads) + thread; complex rows: one cplx each
  if (g.tier_pairs()) {
    o << "#define TIER(s) tier[((((size_t)((s) >> 1)) * nt_ + gt_) << 1) | ((s) & 1)]\n";
    o << "#define TIER2(p) (reinterpret_cast<" << g.VT2() << "*>(tier)[(size_t)(p) * nt_ + gt_])\n";
  } else {
    o << "#define TIER(s) tier[(size_t)(s) * nt_ + gt_]\n";
  }
  o << "extern \"C\" __global__ void __launch_bounds__(" << S.threads << ", " << S.min_blocks << ")\n"
    << kc.name << "(const u64 task_begin, const unsigned task_count, const u64 task_stride, "
    << "unsigned* __restrict__ counter, "
    << g.PT() << "* __restrict__ slots, " << g.VT() << "* __restrict__ tier)\n{\n";
  g.ind = "  ";
  g.line("const unsigned lane = threadIdx.x & 31u;");
  if (g.has_tier()) {
    g.line("const unsigned gt_ = blockIdx.x * blockDim.x + threadIdx.x;");
    g.line("const unsigned nt_ = gridDim.x * blockDim.x;");
  }
  g.line("for (;;) {");
  g.ind = "    ";
  g.line("unsigned t = 0;");
  g.line("if (lane == 0) t = atomicAdd(counter, 1u);");
  g.line("t = __shfl_sync(0xffffffffu, t, 0);");
  g.line("if (t >= task_count) break;");
  g.line("const u64 task = task_begin + (u64)t * task_stride;  // stride 1 except planner samples");
  g.line(std::string(g.PT()) + " lacc = " + g.zero() + ";");
  g.line("#pragma unroll 1");
  g.line("for (unsigned m = 0; m < " + std::to_string(S.M) + "u; ++m) {");
  g.ind = "      ";
  g.line("const u64 chunk = ((task * " + std::to_string(S.M) + "ull + m) << 5) | lane;");
  g.line("const u64 h0 = chunk << " + std::to_string(B) + ";");
  g.ops = 0;
  g.seed();
  kc.ops_seed = g.ops;
  g.line(std::string(g.PT()) + " cacc = " + g.zero() + ";");
  double ops_body = 0, ops_switch = 0;
  if (U == 0) {
    // B == 0: one product per chunk (h = chunk), everything frozen; sign (-1)^h
    const std::string P = g.has_frozen ? std::string("F") : std::string("1");
    if (g.cx) g.line("cacc = (chunk & 1ull) ? cneg(" + (g.has_frozen ? P : std::string("cplx{1.0, 0.0}")) +
                     ") : " + (g.has_frozen ? P : std::string("cplx{1.0, 0.0}")) + ";");
    else g.line("cacc = (chunk & 1ull) ? (" + std::string(g.PT()) + ")(0 - " + P + ") : " + P + ";");
  } else {
    // INT01 zero tracking at chunk level: the frozen product F is constant over
    // the chunk, so a warp whose 32 lanes all have F == 0 skips the chunk
    const bool chunk_skip = g.i01 && S.zero_skip && g.has_frozen;
    if (chunk_skip) g.line("if (!__all_sync(0xffffffffu, F == 0)) {");
    // the signs need only bits U..B of h = (chunk << B) | (blk << U): bits
    // U..B-1 are blk, bit B is chunk bit 0 (= lane bit 0); a 32-bit hu keeps
    // the 64-bit h0 out of the loop (registers)
    const std::string hu_init = "const unsigned cb = ((unsigned)lane & 1u) << " + std::to_string(B - U) + ";";
    // software-pipelined dispatch (complex sweeps): the next block's flip j
    // and sign (BREV/FLO/shifts, MIO latency) are computed before this
    // block's body, and the most frequent flip (bit U, every other block) is
    // a direct uniform branch instead of the switch's BRX.  Measured
    // (profiles/r2_xform_variants_dispatch.jsonl): complex band n=44 +1.6 %;
    // the real kernels gain nothing or spill, so they keep the plain switch.
    const char* pd_env = getenv("PERM_PIPE_DISPATCH");
    const bool pipe_dispatch = pd_env ? atoi(pd_env) == 1 : g.cx;
    const std::string sty = g.i01 ? "int" : "double";
    const std::string splus = g.i01 ? "2" : "1.0", sminus = g.i01 ? "-2" : "-1.0";
    if (nblk > 1) {
      g.line(hu_init);
      if (pipe_dispatch) {
        g.line("unsigned jn_ = " + std::to_string(U) + ";");
        g.line("unsigned sb_ = ((cb | 1u) >> 1) & 1u;  // sign bit of the next block's flip");
      }
      g.line("#pragma unroll 1");
      g.line("for (unsigned blk = 0; blk < " + std::to_string(nblk) + "u; ++blk) {");
      g.ind = "        ";
      g.line("const unsigned hu = cb | blk;");
      g.line("if (blk != 0) {");
      g.ind = "          ";
      if (pipe_dispatch) {
        g.line("const int j = (int)jn_;");
        g.line("const " + sty + " s = sb_ ? " + sminus + " : " + splus + ";");
      } else {
        g.line("const int j = " + std::to_string(U - 1) + " + __ffs(blk);");
        g.line("const " + sty + " s = ((hu >> (j + " + std::to_string(1 - U) + ")) & 1u) ? " + sminus + " : " + splus + ";");
      }
      if (!pipe_dispatch) g.line("switch (j) {");
      for (int b = U; b < B; ++b) {
        if (pipe_dispatch && b == U) g.line("if (blk & 1u) {  // bit U: every other block");
        else if (pipe_dispatch && b == U + 1) g.line("} else switch (j) {");
        if (!(pipe_dispatch && b == U)) g.line("case " + std::to_string(b) + ": {");
        std::string save = g.ind;
        g.ind += "  ";
        g.ops = 0;
        g.mark_region((double)(1ull << (B - 1 - b)));
        g.begin_region();
        g.flip(b, "s");
        g.end_region();
        ops_switch += g.ops * (double)(1ull << (B - 1 - b));  // flips of bit b per chunk
        if (!(pipe_dispatch && b == U)) g.line("break; }");
        g.ind = save;
      }
      if (pipe_dispatch && B == U + 1) {
        g.line("}");  // bit U is the only block bit: no switch
      } else {
        g.line("default: break;");
        g.line("}");
      }
      g.ind = "        ";
      g.line("}");
      if (pipe_dispatch) {
        g.line("{");
        g.line("  const unsigned b1_ = blk + 1u;");
        g.line("  jn_ = " + std::to_string(U - 1) + " + __ffs(b1_ | (1u << 30));");
        g.line("  sb_ = ((cb | b1_) >> (jn_ + " + std::to_string(1 - U) + ")) & 1u;");
        g.line("}");
      }
    } else {
      g.line(hu_init);
      g.line("{");
      g.ind = "        ";
      g.line("const unsigned hu = cb;");
    }
    if (g.i01) g.line("const int sU = (hu & 1u) ? -2 : 2;");
    else g.line("const double sU = (hu & 1u) ? -1.0 : 1.0;");
    g.ops = 0;
    g.mark_region((double)nblk);
    g.begin_region();
    if (g.zs) g.block_zero_skip_body();
    else g.block_body();
    g.end_region();
    ops_body = g.ops;
    g.ind = "      ";
    g.line("}");
    if (chunk_skip) g.line("}");
  }
  const std::string acc_stmt = g.cx ? "lacc = cadd(lacc, cacc);" : "lacc += cacc;";
  if (masked) g.line("if (chunk < " + std::to_string(S.nchunks_total) + "ull) " + acc_stmt);
  else g.line(acc_stmt);
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
    if (g.cx) {
      g.line("for (int o = 16; o > 0; o >>= 1) {");
      g.line("  lacc.re += __shfl_xor_sync(0xffffffffu, lacc.re, o);");
      g.line("  lacc.im += __shfl_xor_sync(0xffffffffu, lacc.im, o);");
      g.line("}");
    } else {
      g.line("for (int o = 16; o > 0; o >>= 1) lacc += __shfl_xor_sync(0xffffffffu, lacc, o);");
    }
  }
  g.line("if (lane == 0) slots[t] = lacc;");
  g.ind = "  ";
  g.line("}");
  o << "}\n";

  if (g.i01)
    for (auto& kv : g.reg_seen)
      if (kv.second > g.reg_bound(kv.first) + 1e-9) excess[kv.first] = kv.second;
  kc.source = o.str();
  (void)ops_body;
  (void)ops_switch;
  const bool fuse = !g.i01 && !g.cx && !getenv("PERM_NO_FUSE");
  const int body_region = (U > 0 && nblk > 1) ? (int)g.region_weight.size() - 1 : -1;
  const auto t_post0 = std::chrono::steady_clock::now();
  const PostStats ps = post_pass(kc.source, g.wt, g.region_weight.size(), fuse, body_region, S.threads,
                                   !g.i01 && !S.w_only, &g.region_weight,
                                   // measured on B200 (profiles/r2_smem_vol_ab.txt): real FP64 0.5,
                                   // INT01 0.125, complex 0 (its 3-block volatile kernels run slower)
                                   g.cx ? 0.0 : (g.i01 ? 0.125 : 0.5), S.w_only, S.smem_ro);
  g_post_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_post0).count();
  kc.smem_bytes = ps.smem_bytes;
  double chunk_ops = 1.0;  // + lacc
  for (size_t k = 0; k < ps.region_ops.size(); ++k) chunk_ops += ps.region_ops[k] * g.region_weight[k];
  kc.ops_seed = ps.region_ops.empty() ? 0.0 : ps.region_ops[0];
  kc.ops_block = (U > 0 && ps.region_ops.size() > 1) ? ps.region_ops.back() : 0.0;
  kc.ops_chunk_total = chunk_ops;
  kc.w_plan = chunk_ops / std::ldexp(1.0, B + S.K);  // per Gray step of the full range
  int live = 0, frozen_rows = 0;
  for (const Factor& f : g.fac) {
    if (f.level >= 0) live += (int)f.rows.size();
    else if (!f.constant()) frozen_rows += (int)f.rows.size();
  }
  kc.live_rows = live;
  kc.seed_rows = frozen_rows;
  int tier_rows = 0;
  for (int r = 0; r < A.n; ++r) tier_rows += g.tier_slot[r] >= 0;
  kc.tier_rows = tier_rows;
  kc.tier_bytes = (g.tier_pairs() ? (tier_rows + 1) / 2 * 2 : tier_rows) * (g.i01 ? 4 : (g.cx ? 16 : 8));
  kc.live_rows = live - tier_rows;
  kc.levels = (int)g.nonempty.size();
  int qs = 0, ds = 0;
  for (int l : g.nonempty) qs += g.qreg(l) + (l >= 1 && g.sreg(l));
  for (const Factor& f : g.fac) ds += f.group && !f.constant() && f.level >= 0;
  const int wpv = g.i01 ? 1 : (g.cx ? 4 : 2);   // 32-bit registers per x value
  const int wpp = g.i01 ? 4 : (g.cx ? 4 : 2);   // per product value
  (void)wpv;
  (void)qs;
  (void)ds;
  // surviving loop-carried registers (rows, level / suffix products, composite
  // values and caches) + the pairwise-accumulation stack + addressing
  kc.est_regs = ps.reg_words + (U + 2) * wpp + 28;
  return kc;
}

}  // namespace perm
