// plan_io.cpp -- binary (de)serialisation of a plan's planning output: the
// on-disk plan cache (PERM_CACHE_DIR / perm_opts.cache_dir) and the rank-0
// plan broadcast of multi-GPU runs (perm_plan_export / perm_plan_import).
//
// Layout: "PERMPLN2" | u32 format version (4) | build id | key | fields in the
// order of write_plan below.  Every length-prefixed field is bounds-checked
// on read; a blob from another libperm build (different generator) or with a
// different key is rejected, never half-applied.
#include <cstring>
#include <string>
#include <vector>

#include "plan_state.h"

namespace perm {

namespace {

constexpr char kMagic[8] = {'P', 'E', 'R', 'M', 'P', 'L', 'N', '2'};
constexpr uint32_t kFormat = 4;

struct W {
  std::string out;
  template <class T>
  void pod(const T& v) {
    out.append(reinterpret_cast<const char*>(&v), sizeof(T));
  }
  void bytes(const void* d, size_t n) {
    pod<uint64_t>(n);
    out.append(reinterpret_cast<const char*>(d), n);
  }
  void str(const std::string& s) { bytes(s.data(), s.size()); }
  template <class T>
  void vec(const std::vector<T>& v) {
    bytes(v.data(), v.size() * sizeof(T));
  }
  void csx(const Csx& a) {
    pod(a.n);
    vec(a.ptr);
    vec(a.idx);
    vec(a.val);
    vec(a.vim);
  }
};

struct R {
  const char* p;
  size_t left;
  bool ok = true;
  template <class T>
  void pod(T& v) {
    if (!ok || left < sizeof(T)) { ok = false; return; }
    std::memcpy(&v, p, sizeof(T));
    p += sizeof(T);
    left -= sizeof(T);
  }
  bool take(uint64_t& n) {
    pod(n);
    if (!ok || n > left) { ok = false; return false; }
    return true;
  }
  void str(std::string& s) {
    uint64_t n = 0;
    if (!take(n)) return;
    s.assign(p, n);
    p += n;
    left -= n;
  }
  template <class T>
  void vec(std::vector<T>& v) {
    uint64_t n = 0;
    if (!take(n) || n % sizeof(T)) { ok = false; return; }
    v.resize(n / sizeof(T));
    if (n) std::memcpy(v.data(), p, n);
    p += n;
    left -= n;
  }
  void csx(Csx& a) {
    pod(a.n);
    vec(a.ptr);
    vec(a.idx);
    vec(a.val);
    vec(a.vim);
    if (ok && (a.n < 0 || a.n > 64 || (!a.ptr.empty() && (int)a.ptr.size() != a.n + 1))) ok = false;
  }
};

void spec_io(W& w, const KernelSpec& s) {
  w.pod(s.n); w.pod(s.K); w.pod(s.B); w.pod(s.U); w.pod(s.M); w.pod(s.mode); w.pod(s.hybrid_c);
  w.pod(s.threads); w.pod(s.zero_skip); w.pod(s.cc); w.pod(s.min_blocks); w.pod(s.nchunks_total);
  w.pod(s.i01_asm_mul); w.pod(s.smem_ro);
}
void spec_io(R& r, KernelSpec& s) {
  r.pod(s.n); r.pod(s.K); r.pod(s.B); r.pod(s.U); r.pod(s.M); r.pod(s.mode); r.pod(s.hybrid_c);
  r.pod(s.threads); r.pod(s.zero_skip); r.pod(s.cc); r.pod(s.min_blocks); r.pod(s.nchunks_total);
  r.pod(s.i01_asm_mul); r.pod(s.smem_ro);
  s.reg_lb_extra = nullptr;
}
void code_io(W& w, const KernelCode& c) {
  w.str(c.source); w.str(c.name);
  w.pod(c.live_rows); w.pod(c.tier_rows); w.pod(c.seed_rows); w.pod(c.levels); w.pod(c.tier_bytes);
  w.pod(c.smem_bytes); w.pod(c.ops_seed); w.pod(c.ops_block); w.pod(c.ops_chunk_total); w.pod(c.w_plan);
  w.pod(c.est_regs);
}
void code_io(R& r, KernelCode& c) {
  r.str(c.source); r.str(c.name);
  r.pod(c.live_rows); r.pod(c.tier_rows); r.pod(c.seed_rows); r.pod(c.levels); r.pod(c.tier_bytes);
  r.pod(c.smem_bytes); r.pod(c.ops_seed); r.pod(c.ops_block); r.pod(c.ops_chunk_total); r.pod(c.w_plan);
  r.pod(c.est_regs);
}

}  // namespace

const char* build_id() { return "libperm-r2 " __DATE__ " " __TIME__; }

uint64_t fnv1a64(const std::string& s, uint64_t h) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

std::string plan_serialize(const perm_plan_s& p, const std::string& key) {
  W w;
  w.out.append(kMagic, 8);
  w.pod(kFormat);
  w.str(build_id());
  w.str(key);
  w.pod(p.n);
  w.csx(p.ccs);
  w.csx(p.crs);
  w.csx(p.occs);
  w.vec(p.rowp);
  w.vec(p.colp);
  w.pod(p.singular);
  w.pod(p.trivial1);
  spec_io(w, p.spec);
  code_io(w, p.code);
  w.vec(p.cubin);
  w.str(p.ptxas_log);
  w.pod(p.info);
  w.pod(p.is_u128);
  w.pod(p.is_c128);
  return w.out;
}

bool plan_deserialize(const void* blob, size_t size, perm_plan_s& out, std::string* key_out) {
  if (!blob || size < 12 || std::memcmp(blob, kMagic, 8) != 0) return false;
  R r{static_cast<const char*>(blob) + 8, size - 8};
  uint32_t fmt = 0;
  r.pod(fmt);
  std::string bid, key;
  r.str(bid);
  r.str(key);
  if (!r.ok || fmt != kFormat || bid != build_id()) return false;
  perm_plan_s p;
  r.pod(p.n);
  r.csx(p.ccs);
  r.csx(p.crs);
  r.csx(p.occs);
  r.vec(p.rowp);
  r.vec(p.colp);
  r.pod(p.singular);
  r.pod(p.trivial1);
  spec_io(r, p.spec);
  code_io(r, p.code);
  r.vec(p.cubin);
  r.str(p.ptxas_log);
  r.pod(p.info);
  r.pod(p.is_u128);
  r.pod(p.is_c128);
  if (!r.ok || r.left != 0 || p.n < 1 || p.n > 64 || (int)p.rowp.size() != p.n || (int)p.colp.size() != p.n)
    return false;
  if (key_out) *key_out = key;
  // planning fields only; device state stays empty
  out.n = p.n;
  out.ccs = std::move(p.ccs);
  out.crs = std::move(p.crs);
  out.occs = std::move(p.occs);
  out.rowp = std::move(p.rowp);
  out.colp = std::move(p.colp);
  out.singular = p.singular;
  out.trivial1 = p.trivial1;
  out.spec = p.spec;
  out.code = std::move(p.code);
  out.cubin = std::move(p.cubin);
  out.ptxas_log = std::move(p.ptxas_log);
  out.info = p.info;
  out.is_u128 = p.is_u128;
  out.is_c128 = p.is_c128;
  return true;
}

}  // namespace perm
