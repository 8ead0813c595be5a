// matrix.cpp -- host planner of libperm: input validation, CCS/CRS conversion,
// structural rank, orderings (Alg. 3, degree sort), Alg. 4 partitioning with a
// B200 register model, Alg. 2 launch parameters (reference planner).
// P:n = /root/reference/PAPER.md line n.
#include <algorithm>
#include <climits>
#include <functional>
#include <cmath>
#include <map>
#include <queue>
#include <set>

#include "perm_internal.h"

namespace perm {

Csx transpose(const Csx& a) {
  Csx t;
  t.n = a.n;
  const int n = a.n, nnz = a.nnz();
  t.ptr.assign(n + 1, 0);
  t.idx.resize(nnz);
  t.val.resize(nnz);
  for (int p = 0; p < nnz; ++p) t.ptr[a.idx[p] + 1]++;
  for (int i = 0; i < n; ++i) t.ptr[i + 1] += t.ptr[i];
  if (a.complex()) t.vim.resize(nnz);
  std::vector<int32_t> pos(t.ptr.begin(), t.ptr.end() - 1);
  for (int j = 0; j < n; ++j)  // ascending outer index => ascending inner index in t
    for (int p = a.ptr[j]; p < a.ptr[j + 1]; ++p) {
      int q = pos[a.idx[p]]++;
      t.idx[q] = j;
      t.val[q] = a.val[p];
      if (a.complex()) t.vim[q] = a.vim[p];
    }
  return t;
}

int validate_and_convert_c(int n, perm_format fmt, const int32_t* ptr, const int32_t* idx, const double* val2,
                           Csx& ccs, Csx& crs, std::string& err) {
  if (n < 1 || n > 64 || !ptr) return validate_and_convert(n, fmt, ptr, idx, nullptr, ccs, crs, err);
  const int nnz = ptr[n] > 0 ? ptr[n] : 0;
  if (nnz > 0 && !val2) { err = "val is NULL"; return PERM_EINVAL; }
  std::vector<double> mag(nnz, 1.0);  // structural check with |a| as the value
  for (int p = 0; p < nnz; ++p) {
    const double re = val2[2 * p], im = val2[2 * p + 1];
    if (!std::isfinite(re) || !std::isfinite(im)) { err = "non-finite value"; return PERM_EINVAL; }
    if (re == 0.0 && im == 0.0) { err = "explicit zero value (formats store nonzeros only)"; return PERM_EINVAL; }
  }
  int st = validate_and_convert(n, fmt, ptr, idx, mag.data(), ccs, crs, err);
  if (st != PERM_OK) return st;
  Csx in;
  in.n = n;
  in.ptr.assign(ptr, ptr + n + 1);
  in.idx.assign(idx, idx + nnz);
  in.val.resize(nnz);
  in.vim.resize(nnz);
  for (int p = 0; p < nnz; ++p) { in.val[p] = val2[2 * p]; in.vim[p] = val2[2 * p + 1]; }
  if (fmt == PERM_CCS) { ccs = in; crs = transpose(in); }
  else { crs = in; ccs = transpose(in); }
  return PERM_OK;
}

int validate_and_convert(int n, perm_format fmt, const int32_t* ptr, const int32_t* idx,
                         const double* val, Csx& ccs, Csx& crs, std::string& err) {
  if (n < 1 || n > 64) {
    err = "n must be in [1, 64] (Gray indices are 64-bit)";
    return PERM_ERANGE;
  }
  if (fmt != PERM_CCS && fmt != PERM_CRS) { err = "unknown format"; return PERM_EINVAL; }
  if (!ptr) { err = "ptr is NULL"; return PERM_EINVAL; }
  if (ptr[0] != 0) { err = "ptr[0] must be 0"; return PERM_EINVAL; }
  for (int j = 0; j < n; ++j)
    if (ptr[j + 1] < ptr[j]) { err = "ptr must be nondecreasing"; return PERM_EINVAL; }
  const int nnz = ptr[n];
  if (nnz > 0 && (!idx || !val)) { err = "idx/val is NULL"; return PERM_EINVAL; }
  for (int j = 0; j < n; ++j)
    for (int p = ptr[j]; p < ptr[j + 1]; ++p) {
      if (idx[p] < 0 || idx[p] >= n) { err = "index out of range"; return PERM_EINVAL; }
      if (p > ptr[j] && idx[p] <= idx[p - 1]) {
        err = "indices must be strictly increasing within each column/row (duplicate or unsorted)";
        return PERM_EINVAL;
      }
      if (!std::isfinite(val[p])) { err = "non-finite value"; return PERM_EINVAL; }
      if (val[p] == 0.0) { err = "explicit zero value (formats store nonzeros only)"; return PERM_EINVAL; }
    }
  Csx in;
  in.n = n;
  in.ptr.assign(ptr, ptr + n + 1);
  in.idx.assign(idx, idx + nnz);
  in.val.assign(val, val + nnz);
  if (fmt == PERM_CCS) { ccs = in; crs = transpose(in); }
  else { crs = in; ccs = transpose(in); }
  return PERM_OK;
}

// Hopcroft-Karp maximum matching of the bipartite graph rows x columns.
int structural_rank(const Csx& ccs) {
  const int n = ccs.n;
  Csx crs = transpose(ccs);  // row -> columns
  std::vector<int> mrow(n, -1), mcol(n, -1), dist(n);
  const int INF = INT_MAX;
  auto bfs = [&]() {
    std::queue<int> q;
    bool found = false;
    for (int r = 0; r < n; ++r) {
      if (mrow[r] < 0) { dist[r] = 0; q.push(r); } else dist[r] = INF;
    }
    while (!q.empty()) {
      int r = q.front(); q.pop();
      for (int p = crs.ptr[r]; p < crs.ptr[r + 1]; ++p) {
        int c = crs.idx[p], r2 = mcol[c];
        if (r2 < 0) found = true;
        else if (dist[r2] == INF) { dist[r2] = dist[r] + 1; q.push(r2); }
      }
    }
    return found;
  };
  std::vector<int> it(n);
  // iterative-free recursion depth <= n <= 64
  std::function<bool(int)> dfs = [&](int r) -> bool {
    for (int& p = it[r]; p < crs.ptr[r + 1]; ++p) {
      int c = crs.idx[p], r2 = mcol[c];
      if (r2 < 0 || (dist[r2] == dist[r] + 1 && dfs(r2))) {
        mrow[r] = c; mcol[c] = r;
        return true;
      }
    }
    dist[r] = INF;
    return false;
  };
  int match = 0;
  while (bfs()) {
    for (int r = 0; r < n; ++r) it[r] = crs.ptr[r];
    for (int r = 0; r < n; ++r)
      if (mrow[r] < 0 && dfs(r)) ++match;
  }
  return match;
}

// Alg. 3 PermanentOrdering.  Readings (DESIGN R11): argmin ties go
// to the lowest column index; rows of the chosen column are visited in CCS
// (ascending row) order; rows never reached are appended in original order.
void order_permanent(const Csx& ccs, const Csx& crs, std::vector<int>& rowp, std::vector<int>& colp) {
  const int n = ccs.n;
  std::vector<long long> cdeg(n);
  std::vector<char> chosen(n, 0), rmark(n, 0);
  for (int j = 0; j < n; ++j) cdeg[j] = ccs.ptr[j + 1] - ccs.ptr[j];   // lines 1-3
  rowp.clear();
  colp.clear();
  for (int cidx = 0; cidx < n; ++cidx) {                               // line 8
    int col = -1;
    for (int j = 0; j < n; ++j)                                        // line 10: argmin
      if (!chosen[j] && (col < 0 || cdeg[j] < cdeg[col])) col = j;
    colp.push_back(col);                                               // line 11
    chosen[col] = 1;                                                   // line 12: cdeg = inf
    for (int p = ccs.ptr[col]; p < ccs.ptr[col + 1]; ++p) {            // line 13
      int row = ccs.idx[p];
      if (!rmark[row]) {                                               // line 15
        rmark[row] = 1;
        rowp.push_back(row);                                           // line 17
        for (int q = crs.ptr[row]; q < crs.ptr[row + 1]; ++q)          // line 20
          if (!chosen[crs.idx[q]]) cdeg[crs.idx[q]]--;                 // line 21 (inf - 1 = inf)
      }
    }
  }
  for (int r = 0; r < n; ++r)
    if (!rmark[r]) rowp.push_back(r);
}

// Degree sort ascending (Sec. VI-B): columns by (degree, index); rows unchanged.
void order_degree(const Csx& ccs, std::vector<int>& rowp, std::vector<int>& colp) {
  const int n = ccs.n;
  colp.resize(n);
  rowp.resize(n);
  for (int j = 0; j < n; ++j) { colp[j] = j; rowp[j] = j; }
  std::stable_sort(colp.begin(), colp.end(), [&](int a, int b) {
    return ccs.ptr[a + 1] - ccs.ptr[a] < ccs.ptr[b + 1] - ccs.ptr[b];
  });
}

Csx permute_ccs(const Csx& ccs, const std::vector<int>& rowp, const std::vector<int>& colp) {
  const int n = ccs.n;
  std::vector<int> rinv(n);
  for (int i = 0; i < n; ++i) rinv[rowp[i]] = i;
  Csx o;
  o.n = n;
  o.ptr.assign(1, 0);
  for (int j = 0; j < n; ++j) {
    int oc = colp[j];
    std::vector<std::pair<int, int>> e;  // (ordered row, source position)
    for (int p = ccs.ptr[oc]; p < ccs.ptr[oc + 1]; ++p) e.push_back({rinv[ccs.idx[p]], p});
    std::sort(e.begin(), e.end());
    for (auto& q : e) {
      o.idx.push_back(q.first);
      o.val.push_back(ccs.val[q.second]);
      if (ccs.complex()) o.vim.push_back(ccs.vim[q.second]);
    }
    o.ptr.push_back((int)o.idx.size());
  }
  return o;
}

std::vector<int> factored_columns(const std::vector<int>& base_colp, const std::vector<int>& picks, int K) {
  std::vector<int> out(picks.begin(), picks.begin() + K);
  for (int c : base_colp)
    if (std::find(picks.begin(), picks.begin() + K, c) == picks.begin() + K) out.push_back(c);
  return out;
}

int elim_eval_size(const Csx& ccs, const std::vector<int>& colp, int K) {
  // leaf = 1; elimination node = 2 x sum(children) (evaluated at the in and
  // out states); returns the largest root -- bounds generated code size
  const int n = ccs.n;
  std::vector<int> root(n);
  std::map<int, long long> size;
  for (int r = 0; r < n; ++r) { root[r] = r; size[r] = 1; }
  long long worst = 1;
  int next = n;
  for (int k = 0; k < K; ++k) {
    const int c = colp[k];
    std::set<int> T;
    for (int p = ccs.ptr[c]; p < ccs.ptr[c + 1]; ++p) T.insert(root[ccs.idx[p]]);
    long long s = 0;
    for (int t : T) s += size[t];
    const int id = next++;
    size[id] = std::min<long long>(2 * s, 1ll << 40);
    worst = std::max(worst, size[id]);
    for (int r = 0; r < n; ++r)
      if (T.count(root[r])) root[r] = id;
  }
  return (int)std::min<long long>(worst, 1 << 30);
}

std::vector<int> costsort_swept(const Csx& ccs, const std::vector<int>& colp, int K) {
  const int n = ccs.n;
  // replay the eliminations of colp[0..K): root per row, dead rows (the only
  // row of an elimination), live rows under each composite root
  std::vector<int> root(n);
  for (int r = 0; r < n; ++r) root[r] = r;
  std::vector<char> dead(n, 0), composite(2 * n + K + 1, 0);
  int next = n;
  for (int k = 0; k < K; ++k) {
    const int c = colp[k];
    std::set<int> T;
    for (int p = ccs.ptr[c]; p < ccs.ptr[c + 1]; ++p) T.insert(root[ccs.idx[p]]);
    if (T.size() == 1 && *T.begin() < n && ccs.ptr[c + 1] - ccs.ptr[c] == 1) dead[*T.begin()] = 1;
    const int id = next++;
    composite[id] = 1;
    for (int r = 0; r < n; ++r)
      if (T.count(root[r])) root[r] = id;
  }
  std::map<int, int> live;
  for (int r = 0; r < n; ++r)
    if (!dead[r]) live[root[r]]++;
  auto cost = [&](int c) {  // live rows updated + rough recompute cost of touched composites
    int w = 0;
    std::set<int> seen;
    for (int p = ccs.ptr[c]; p < ccs.ptr[c + 1]; ++p) {
      const int r = ccs.idx[p];
      if (dead[r]) continue;
      ++w;
      if (composite[root[r]] && seen.insert(root[r]).second) w += 2 * live[root[r]];
    }
    return w;
  };
  std::vector<int> out(colp.begin(), colp.end());
  if (n - 1 > K) {
    std::vector<int> cst(n);
    for (int q = K; q < n - 1; ++q) cst[colp[q]] = cost(colp[q]);
    std::stable_sort(out.begin() + K, out.end() - 1, [&](int a, int b) { return cst[a] < cst[b]; });
  }
  return out;
}

// CalculateNoThreads (Alg. 4 line 12; undefined in the paper): resident
// threads when each thread needs nregisters + 32 registers, on `sms` SMs of
// 65536 registers / 2048 threads, 255 registers per thread max.
uint64_t b200_threads(int nregisters, int sms) {
  const int per = nregisters + 32;
  if (per > 255) return 0;
  long long t = (65536 / per) / 32 * 32;
  if (t > 2048) t = 2048;
  return (uint64_t)sms * (uint64_t)t;
}

// Alg. 4 Partitioning, verbatim on the ordered CCS.
void partition_alg4(const Csx& o, double gr, int sms, int& k, int& c) {
  const int n = o.n;
  k = 0;
  c = 0;
  double best = 0.0;
  int nrows = 0;
  for (int j = 0; j < n; ++j) {                                             // line 5
    if (o.ptr[j + 1] > o.ptr[j]) nrows = std::max(nrows, o.idx[o.ptr[j + 1] - 1] + 1);  // line 7
    const int nreg = nrows * 2;                                             // line 8
    const double reg_cost = nreg * (1.0 - std::ldexp(1.0, -(j + 1)));       // line 9
    const double glob_cost = (n - nrows) * std::ldexp(1.0, -(j + 1)) * gr;  // line 10
    const double tau = (double)b200_threads(nreg, sms);                     // line 12
    const double denom = reg_cost + glob_cost;
    const double score = denom > 0 ? tau / denom : 0.0;                     // line 13
    if (score > best || nrows == k) { best = score; k = nrows; c = j + 1; } // line 14
  }
}

// Alg. 2 GenerateLaunchParameters, verbatim.
int alg2_launch_parameters(uint64_t tau, int n, uint64_t* out, int cap) {
  if (tau < 1 || n < 2 || n > 64) return -1;
  int cnt = 0;
  uint64_t start = 1, end = 1ull << (n - 1);
  while (end - start > 0) {
    uint64_t delta = 1024;
    while (delta * tau <= end - start) delta *= 2;
    delta /= 2;
    if (delta == 512) {
      if (cnt < cap) { out[3 * cnt] = start; out[3 * cnt + 1] = 1024; out[3 * cnt + 2] = end; }
      ++cnt;
      break;
    }
    if (cnt < cap) { out[3 * cnt] = start; out[3 * cnt + 1] = delta; out[3 * cnt + 2] = end; }
    ++cnt;
    start += tau * delta;
  }
  return cnt;
}

}  // namespace perm
