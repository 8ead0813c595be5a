"""Experiment harness: time source-level variants of a plan's generated sweep
kernel on the GPU, outside libperm (nvcc -cubin + the CUDA driver API), with
the plan's own launch geometry.  Used to evaluate codegen changes before they
go into the generator; every variant's per-task slots must equal the
baseline's bit for bit.

    python tools/kernel_xform.py [--dim 40 --p 0.2 --seed 1] [--variants base,kc]
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

LIT = re.compile(r"\((-?0x[0-9a-f.]+p[+-]\d+)\)")


def xf_kc(src):
    """double literals -> a __constant__ array (LDCU.64 instead of 2 x UMOV)."""
    i = src.index('extern "C"')
    lits = {}

    def rep(m):
        t = m.group(1)
        if t not in lits:
            lits[t] = len(lits)
        return f"kc_[{lits[t]}]"
    body = LIT.sub(rep, src[i:])
    decl = "__constant__ double kc_[%d] = {%s};\n" % (max(1, len(lits)), ", ".join(lits) or "0")
    return src[:i] + decl + body


def xf_hot(src, thr=2, cap=1000):
    """Body literals used >= thr times per block iteration (at most cap of
    them, most used first) -> a __constant__ table; ptxas keeps those in
    uniform registers across the block loop instead of re-materialising each
    with two UMOVs per use."""
    import collections
    L = src.split("\n")
    bi = max(i for i, l in enumerate(L) if "default: break;" in l) + 2
    be = max(i for i, l in enumerate(L) if "lacc += cacc" in l)
    cnt = collections.Counter(m.group(1).lstrip("-") for l in L[bi:be] for m in LIT.finditer(l))
    hot = [k for k, v in cnt.most_common() if v >= thr][:cap]
    idx = {k: i for i, k in enumerate(hot)}

    def rep(m):
        t = m.group(1)
        a = t.lstrip("-")
        return f"({'-' if t.startswith('-') else ''}kc_[{idx[a]}])" if a in idx else m.group(0)
    i = src.index('extern "C"')
    decl = "__constant__ double kc_[%d] = {%s};\n" % (max(1, len(hot)), ", ".join(hot) or "0")
    return src[:i] + decl + LIT.sub(rep, src[i:])


def xf_vol(src):
    """shared-memory slots as volatile: ptxas otherwise forwards every SM_
    store to its loads and keeps the values in registers (0 LDS in SASS)."""
    return re.sub(r"\(\(\((\w+)\*\)\(sm_ \+ (\d+)\)\)\[threadIdx.x\]\)",
                  r"(((volatile \1*)(sm_ + \2))[threadIdx.x])", src)


def xf_ro(src, vol=True):
    """loop-carried doubles the block body reads but never writes -> more
    per-thread shared-memory slots (read with LDS at each body use)."""
    L = src.split("\n")
    li = next(i for i, l in enumerate(L) if "for (unsigned blk" in l)
    bi = max(i for i, l in enumerate(L) if "default: break;" in l) + 2
    be = max(i for i, l in enumerate(L) if "lacc += cacc" in l)
    decl = {}
    for i in range(li - 1, 0, -1):
        m = re.match(r"\s+double (\w+) = (t\d+|0);$", L[i])
        if m:
            decl[m.group(1)] = i
        elif "const double" in L[i]:
            break
    body = "\n".join(L[bi:be])
    written = set(re.findall(r"^\s+(\w+) = ", body, re.M))
    used = set(re.findall(r"\b(\w+)\b", body))
    ro = [v for v in decl if v in used and v not in written and v != "cacc"]
    offs = [int(x) for x in re.findall(r"\(sm_ \+ (\d+)\)", src)]
    off = (max(offs) + 1024) if offs else 0
    thr = int(re.search(r"__launch_bounds__\((\d+)", src).group(1))
    defs = ""
    for v in ro:
        defs += "#define SM_%s (((double*)(sm_ + %d))[threadIdx.x])\n" % (v, off)
        off += 8 * thr
    for v in ro:
        L[decl[v]] = L[decl[v]].replace("double %s =" % v, "SM_%s =" % v)
    out = "\n".join(L)
    for v in ro:
        out = re.sub(r"(?<![\w])%s(?![\w])" % v, "SM_" + v, out)
        out = out.replace("SM_SM_" + v, "SM_" + v)
    if "extern __shared__" not in out:
        out = out.replace('extern "C"', "extern __shared__ __align__(16) unsigned char sm_[];\n" + 'extern "C"', 1)
    out = out.replace('extern "C"', defs + 'extern "C"', 1)
    out = out.replace("#define SM_" + ro[0] if ro else "@@", "#define SM_" + ro[0]) if ro else out
    return (xf_vol(out) if vol else out), off


def xf_br1(src):
    """the most frequent block-boundary flip (bit U, every other block) as a
    direct uniform branch instead of a BRX through the switch's jump table"""
    m = re.search(r"( +)switch \(j\) \{\n +case (\d+): \{\n", src)
    if not m:
        return src
    ind = m.group(1)
    head = m.group(0)
    i = m.start()
    k = src.index("break; }\n", m.end())
    k2 = k + len("break; }\n")
    case_body = src[m.end():k]
    rest_start = src[k2:]
    new = (ind + "if (blk & 1u) {  // case %s\n" % m.group(2) + case_body + ind + "} else switch (j) {\n")
    return src[:i] + new + rest_start


def xf_un2(src):
    """block loop unrolled by 2 (ptxas then sees case U inline on odd blocks)"""
    return re.sub(r"#pragma unroll 1\n(\s+)for \(unsigned blk", r"#pragma unroll 2\n\1for (unsigned blk", src)


def xf_kcase(src, scope="cases"):
    """switch-case literals -> a second __constant__ table indexed with a
    loop-variant zero (blk & (task_stride >> 40)), so ptxas cannot hoist the
    LDCU loads out of the block loop (uniform-register pressure) and loads
    them inside the case instead of building each literal with two UMOVs."""
    L = src.split("\n")
    si = next(i for i, l in enumerate(L) if "switch (j) {" in l)
    bi = max(i for i, l in enumerate(L) if "default: break;" in l)
    be = max(i for i, l in enumerate(L) if "lacc += cacc" in l)
    lo, hi = (si, bi) if scope == "cases" else (si, be)
    lits = {}

    def rep(m):
        t = m.group(1)
        a = t.lstrip("-")
        if a not in lits:
            lits[a] = len(lits)
        return f"({'-' if t.startswith('-') else ''}kcs_[{lits[a]} + zb_])"
    for i in range(lo, hi):
        L[i] = LIT.sub(rep, L[i])
    li = next(i for i, l in enumerate(L) if "for (unsigned blk" in l)
    L.insert(li + 1, "        const unsigned zb_ = blk & (unsigned)(task_stride >> 40);")
    out = "\n".join(L)
    decl = "__constant__ double kcs_[%d] = {%s};\n" % (max(1, len(lits)), ", ".join(lits) or "0")
    return out.replace('extern "C"', decl + 'extern "C"', 1)


def xf_kseed(src):
    """seed-region literals (executed once per chunk) -> a __constant__ table
    indexed with a loop-variant zero (m & (task_stride >> 40)): an LDC.64 per
    literal instead of two UMOVs, and a shorter seed for the instruction cache."""
    L = src.split("\n")
    mi = next(i for i, l in enumerate(L) if "for (unsigned m = 0;" in l)
    li = next(i for i, l in enumerate(L) if "for (unsigned blk" in l)
    lits = {}

    def rep(m):
        t = m.group(1)
        a = t.lstrip("-")
        if a not in lits:
            lits[a] = len(lits)
        return f"({'-' if t.startswith('-') else ''}kss_[{lits[a]} + zs_])"
    for i in range(mi + 1, li):
        L[i] = LIT.sub(rep, L[i])
    L.insert(mi + 1, "      const unsigned zs_ = m & (unsigned)(task_stride >> 40);")
    out = "\n".join(L)
    decl = "__constant__ double kss_[%d] = {%s};\n" % (max(1, len(lits)), ", ".join(lits) or "0")
    return out.replace('extern "C"', decl + 'extern "C"', 1)


def xf_pipej(src):
    """software-pipelined block dispatch: j and s of the NEXT block (BREV/FLO,
    shifts: MIO latency) are computed before the current block's body, so the
    dispatch at the loop top only branches; plus the direct branch for the
    most frequent flip (xf_br1)"""
    m = re.search(r"( +)#pragma unroll 1\n( +)for \(unsigned blk = 0; blk < (\d+)u; \+\+blk\) \{\n"
                  r"( +)const unsigned hu = cb \| blk;\n( +)if \(blk != 0\) \{\n"
                  r"( +)const int j = (\d+) \+ __ffs\(blk\);\n( +)const double s = \(\(hu >> \(j \+ (-?\d+)\)\) & 1u\) \? -1\.0 : 1\.0;\n", src)
    if not m:
        return src
    i0, nb, jb, sh = m.group(1), m.group(3), m.group(7), m.group(9)
    ind = m.group(4)
    pre = (f"{i0}unsigned jn_ = {jb} + __ffs(1u);\n{i0}double sn_ = (((cb | 1u) >> (jn_ + {sh})) & 1u) ? -1.0 : 1.0;\n"
           f"{i0}#pragma unroll 1\n{m.group(2)}for (unsigned blk = 0; blk < {nb}u; ++blk) {{\n"
           f"{ind}const unsigned hu = cb | blk;\n{m.group(5)}if (blk != 0) {{\n"
           f"{m.group(6)}const int j = (int)jn_;\n{m.group(8)}const double s = sn_;\n")
    out = src[:m.start()] + pre + src[m.end():]
    # next block's dispatch right after the switch (before the body)
    k = out.index("default: break;")
    k = out.index("\n", out.index("}", k)) + 1  # end of switch
    k = out.index("\n", out.index("}", k)) + 1  # end of if (blk != 0)
    nxt = (f"{ind}{{ const unsigned b1_ = blk + 1u; jn_ = {jb} + __ffs(b1_ | (1u << 30));"
           f" sn_ = (((cb | b1_) >> (jn_ + {sh})) & 1u) ? -1.0 : 1.0; }}\n")
    out = out[:k] + nxt + out[k:]
    return xf_br1(out)


def xf_order(src, how="asap", seed=0):
    """re-emit the block body's SSA temporaries in another topological order
    (asap: by dependency depth; alap: as late as possible; rand: random
    topological order) -- the loop-carried write-backs keep their place at
    the end; tests how much the source order steers ptxas's schedule"""
    import random
    L = src.split("\n")
    bi = max(i for i, l in enumerate(L) if "default: break;" in l) + 1
    while L[bi].strip() == "}":
        bi += 1
    be = max(i for i, l in enumerate(L) if "lacc += cacc" in l)
    body = L[bi:be]
    defs, rest = [], []
    for l in body:
        (defs if re.match(r"\s+const (double|int|u128|i64|cplx) t\d+ = ", l) else rest).append(l)
    # the block's sign line etc. (non-SSA) stay in front, write-backs after
    head = [l for l in rest if "sU" in l and "const" in l]
    tailr = [l for l in rest if l not in head]
    name = [re.match(r"\s+const \w+ (t\d+) = ", l).group(1) for l in defs]
    idx = {v: k for k, v in enumerate(name)}
    deps = [[idx[t] for t in re.findall(r"\b(t\d+)\b", l.split(" = ", 1)[1]) if t in idx] for l in defs]
    users = [[] for _ in defs]
    for k, ds in enumerate(deps):
        for d in ds:
            users[d].append(k)
    n = len(defs)
    if how == "asap":
        depth = [0] * n
        for k in range(n):
            depth[k] = 1 + max([depth[d] for d in deps[k]], default=0)
        order = sorted(range(n), key=lambda k: (depth[k], k))
    elif how == "alap":
        h = [0] * n
        for k in reversed(range(n)):
            h[k] = 1 + max([h[u] for u in users[k]], default=0)
        order = sorted(range(n), key=lambda k: (-h[k], k))
    elif how == "dfs":  # Sethi-Ullman-like: each sink's operand trees depth first, deepest operand first
        need = [0] * n
        for k in range(n):
            ds = sorted({need[d] for d in deps[k]}, reverse=True)
            need[k] = max([v + i for i, v in enumerate(ds)] + [1])
        done, order = [False] * n, []

        def emit(k):
            stack = [(k, False)]
            while stack:
                v, exp = stack.pop()
                if done[v]:
                    continue
                if exp:
                    done[v] = True
                    order.append(v)
                    continue
                stack.append((v, True))
                for d in sorted(set(deps[v]), key=lambda d: need[d]):
                    if not done[d]:
                        stack.append((d, False))
        for k in range(n):
            if not users[k]:
                emit(k)
        for k in range(n):
            emit(k)
    elif how == "greedy":  # list schedule minimising the live set, ties in source order
        import heapq
        remaining = [len(set(u)) for u in users]
        indeg = [len(set(d)) for d in deps]
        emitted = [False] * n
        order = []

        def score(k):
            kills = sum(1 for d in set(deps[k]) if remaining[d] == 1)
            return (1 if users[k] else 0) - kills
        ready = set(k for k in range(n) if indeg[k] == 0)
        while ready:
            k = min(ready, key=lambda k: (score(k), k))
            ready.discard(k)
            emitted[k] = True
            order.append(k)
            for d in set(deps[k]):
                remaining[d] -= 1
            for u in set(users[k]):
                indeg[u] -= 1
                if indeg[u] == 0:
                    ready.add(u)
    else:
        rnd = random.Random(seed)
        indeg = [len(set(d)) for d in deps]
        ready = [k for k in range(n) if indeg[k] == 0]
        order = []
        while ready:
            k = ready.pop(rnd.randrange(len(ready)))
            order.append(k)
            for u in set(users[k]):
                indeg[u] -= 1
                if indeg[u] == 0:
                    ready.append(u)
    return "\n".join(L[:bi] + head + [defs[k] for k in order] + tailr + L[be:])


MUL_S32_U128 = r"""
__device__ __forceinline__ u128 mul_s32_u128(int b, u128 a) {
  unsigned a0 = (unsigned)a, a1 = (unsigned)(a >> 32), a2 = (unsigned)(a >> 64), a3 = (unsigned)(a >> 96);
  unsigned r0, r1, r2, r3;
  const unsigned ub = (unsigned)b, m = (unsigned)(b >> 31);
  asm("mul.lo.u32 %0, %4, %8;\n\tmul.hi.u32 %1, %4, %8;\n\tmad.lo.cc.u32 %1, %5, %8, %1;\n\t"
      "madc.hi.u32 %2, %5, %8, 0;\n\tmad.lo.cc.u32 %2, %6, %8, %2;\n\tmadc.hi.u32 %3, %6, %8, 0;\n\t"
      "mad.lo.u32 %3, %7, %8, %3;\n\tand.b32 %4, %4, %9;\n\tand.b32 %5, %5, %9;\n\tand.b32 %6, %6, %9;\n\t"
      "sub.cc.u32 %1, %1, %4;\n\tsubc.cc.u32 %2, %2, %5;\n\tsubc.u32 %3, %3, %6;"
      : "=&r"(r0), "=&r"(r1), "=&r"(r2), "=&r"(r3), "+r"(a0), "+r"(a1), "+r"(a2) : "r"(a3), "r"(ub), "r"(m));
  return ((u128)(((unsigned long long)r3 << 32) | r2) << 64) | (((unsigned long long)r1 << 32) | r0);
}
"""


MUL_S32_U128_C = r"""
__device__ __forceinline__ u128 mul_s32_u128(int b, u128 a) {
  typedef unsigned long long u64_;
  const unsigned ub = (unsigned)b, m = (unsigned)(b >> 31);
  const unsigned a0 = (unsigned)a, a1 = (unsigned)(a >> 32), a2 = (unsigned)(a >> 64), a3 = (unsigned)(a >> 96);
  const u64_ p0 = (u64_)a0 * ub;
  const u64_ p1 = (u64_)a1 * ub + (p0 >> 32);
  const u64_ p2 = (u64_)a2 * ub + (p1 >> 32);
  const unsigned r3 = a3 * ub + (unsigned)(p2 >> 32);
  const u128 r = ((u128)(((u64_)r3 << 32) | (unsigned)p2) << 64) | ((p1 << 32) | (unsigned)p0);
  return r - ((u128)((((u64_)(a1 & m)) << 32) | (a0 & m)) << 32 | ((u128)(a2 & m) << 96));
}
"""


MUL_U128 = r"""
__device__ __forceinline__ u128 mul_u128(u128 a, u128 b) {
  const unsigned a0 = (unsigned)a, a1 = (unsigned)(a >> 32), a2 = (unsigned)(a >> 64), a3 = (unsigned)(a >> 96);
  const unsigned b0 = (unsigned)b, b1 = (unsigned)(b >> 32), b2 = (unsigned)(b >> 64), b3 = (unsigned)(b >> 96);
  unsigned r0, r1, r2, r3;
  asm("mul.lo.u32 %0, %4, %8;\n\t"
      "mul.hi.u32 %1, %4, %8;\n\t"
      "mad.lo.cc.u32 %1, %4, %9, %1;\n\t"
      "madc.hi.u32 %2, %4, %9, 0;\n\t"
      "mad.lo.cc.u32 %1, %5, %8, %1;\n\t"
      "madc.hi.cc.u32 %2, %5, %8, %2;\n\t"
      "addc.u32 %3, 0, 0;\n\t"
      "mad.lo.cc.u32 %2, %4, %10, %2;\n\t"
      "madc.hi.u32 %3, %4, %10, %3;\n\t"
      "mad.lo.cc.u32 %2, %5, %9, %2;\n\t"
      "madc.hi.u32 %3, %5, %9, %3;\n\t"
      "mad.lo.cc.u32 %2, %6, %8, %2;\n\t"
      "madc.hi.u32 %3, %6, %8, %3;\n\t"
      "mad.lo.u32 %3, %4, %11, %3;\n\t"
      "mad.lo.u32 %3, %5, %10, %3;\n\t"
      "mad.lo.u32 %3, %6, %9, %3;\n\t"
      "mad.lo.u32 %3, %7, %8, %3;"
      : "=&r"(r0), "=&r"(r1), "=&r"(r2), "=&r"(r3)
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(b2), "r"(b3));
  return ((u128)(((unsigned long long)r3 << 32) | r2) << 64) | (((unsigned long long)r1 << 32) | r0);
}
"""


def xf_m128u(src):
    """INT01: u128 x u128 products through a hand-scheduled schoolbook
    multiply (mod 2^128), on top of xf_m128"""
    out = xf_m128(src)
    ty = {m.group(2): m.group(1) for m in re.finditer(r"(?:const )?(int|i64|u128) (\w+) = ", src)}

    def rep(m):
        a, b = m.group(1), m.group(2)
        if ty.get(a) == "u128" and ty.get(b) == "u128":
            return f"mul_u128({a}, {b})"
        return m.group(0)
    out = re.sub(r"\b(\w+) \* (\w+)\b(?!\()", rep, out)
    return out.replace("__device__ __forceinline__ u128 mul_s32_u128", MUL_U128 + "__device__ __forceinline__ u128 mul_s32_u128", 1)


def xf_m128(src, helper=None):
    """INT01: (u128)(i128)int * u128 through a hand-scheduled 32 x 128-bit
    multiply (4 wide multiplies + masked correction for a negative int)"""
    ty = {m.group(2): m.group(1) for m in re.finditer(r"(?:const )?(int|i64|u128) (\w+) = ", src)}
    pat = re.compile(r"\(u128\)\(i128\)(\w+) \* (\w+)|(\w+) \* \(u128\)\(i128\)(\w+)")

    def rep(m):
        if m.group(1):
            nar, wide = m.group(1), m.group(2)
        else:
            wide, nar = m.group(3), m.group(4)
        if ty.get(nar) == "int" and ty.get(wide) == "u128":
            return f"mul_s32_u128({nar}, {wide})"
        return m.group(0)
    out = pat.sub(rep, src)
    return out.replace('extern "C"', (helper or MUL_S32_U128) + 'extern "C"', 1)


def xf_rw_le(src, maxuses, maxrw):
    """xf_ro_le plus the body-WRITTEN loop-carried doubles with <= maxrw uses
    (an STS per write, an LDS per read)."""
    import collections
    L = src.split("\n")
    li = next(i for i, l in enumerate(L) if "for (unsigned blk" in l)
    bi = max(i for i, l in enumerate(L) if "default: break;" in l) + 2
    be = max(i for i, l in enumerate(L) if "lacc += cacc" in l)
    decl = {}
    for i in range(li - 1, 0, -1):
        m = re.match(r"\s+double (\w+) = (t\d+|0);$", L[i])
        if m:
            decl[m.group(1)] = i
        elif "const double" in L[i]:
            break
    body = "\n".join(L[bi:be])
    written = set(re.findall(r"^\s+(\w+) = ", body, re.M))
    uses = collections.Counter(re.findall(r"\b(\w+)\b", body))
    mv = [v for v in decl if v != "cacc" and uses[v] > 0 and uses[v] <= (maxrw if v in written else maxuses)]
    return _ro_subset(src, mv, decl)


def xf_ro_le(src, maxuses):
    """only the body-read-only loop-carried doubles with <= maxuses uses in the
    block body -> volatile shared-memory slots (an LDS per use; frees their
    registers for a larger unrolled block)."""
    import collections
    L = src.split("\n")
    li = next(i for i, l in enumerate(L) if "for (unsigned blk" in l)
    bi = max(i for i, l in enumerate(L) if "default: break;" in l) + 2
    be = max(i for i, l in enumerate(L) if "lacc += cacc" in l)
    decl = {}
    for i in range(li - 1, 0, -1):
        m = re.match(r"\s+double (\w+) = (t\d+|0);$", L[i])
        if m:
            decl[m.group(1)] = i
        elif "const double" in L[i]:
            break
    body = "\n".join(L[bi:be])
    written = set(re.findall(r"^\s+(\w+) = ", body, re.M))
    uses = collections.Counter(re.findall(r"\b(\w+)\b", body))
    keep = {v for v in decl if v in written or v == "cacc" or uses[v] > maxuses}
    # reuse xf_ro on a copy where the kept names are hidden from it
    for v in keep:
        L[decl[v]] = L[decl[v]].replace("double %s =" % v, "double %s  =" % v)
    return xf_ro("\n".join(L).replace("  =", " ="), vol=True) if False else _ro_subset(src, [v for v in decl if v not in keep], decl)


def _ro_subset(src, ro, decl):
    L = src.split("\n")
    offs = [int(x) for x in re.findall(r"\(sm_ \+ (\d+)\)", src)]
    thr = int(re.search(r"__launch_bounds__\((\d+)", src).group(1))
    off = (max(offs) + 8 * thr) if offs else 0
    defs = ""
    for v in ro:
        defs += "#define SM_%s (((double*)(sm_ + %d))[threadIdx.x])\n" % (v, off)
        off += 8 * thr
    for v in ro:
        L[decl[v]] = L[decl[v]].replace("double %s =" % v, "SM_%s =" % v)
    out = "\n".join(L)
    for v in ro:
        out = re.sub(r"(?<![\w])%s(?![\w])" % v, "SM_" + v, out)
        out = out.replace("SM_SM_" + v, "SM_" + v)
    if "extern __shared__" not in out:
        out = out.replace('extern "C"', "extern __shared__ __align__(16) unsigned char sm_[];\n" + 'extern "C"', 1)
    out = out.replace('extern "C"', defs + 'extern "C"', 1)
    return xf_vol(out), off


def xf_lb(src, mb):
    return re.sub(r"__launch_bounds__\((\d+), (\d+)\)", r"__launch_bounds__(\1, %d)" % mb, src)


def xf_b64(src):
    return re.sub(r"__launch_bounds__\(128, (\d+)\)", r"__launch_bounds__(64, \1)", src)


VARIANTS = {"base": (lambda s: s, 128), "hot2": (xf_hot, 128), "hot2c16": (lambda s: xf_hot(s, 2, 16), 128),
            "hot3": (lambda s: xf_hot(s, 3), 128),
            "vol": (xf_vol, 128), "br1": (xf_br1, 128), "m128": (xf_m128, 128), "m128u": (xf_m128u, 128), "m128c": (lambda s: xf_m128(s, MUL_S32_U128_C), 128), "asap": (lambda s: xf_order(s, "asap"), 128),
            "alap": (lambda s: xf_order(s, "alap"), 128), "dfs": (lambda s: xf_order(s, "dfs"), 128),
            "greedy": (lambda s: xf_order(s, "greedy"), 128), "rand1": (lambda s: xf_order(s, "rand", 1), 128),
            "rand2": (lambda s: xf_order(s, "rand", 2), 128), "rand3": (lambda s: xf_order(s, "rand", 3), 128), "pipej": (xf_pipej, 128), "kcase": (xf_kcase, 128), "kall": (lambda s: xf_kcase(s, "all"), 128), "un2": (xf_un2, 128), "ro": (xf_ro, 128), "ro_hot2": (lambda s: xf_ro(xf_hot(s)), 128),
            "ro_lb3": (lambda s: xf_ro(xf_lb(s, 3)), 128), "vol_hot2": (lambda s: xf_vol(xf_hot(s)), 128), "kc": (xf_kc, 128), "b64": (xf_b64, 64), "kc_b64": (lambda s: xf_b64(xf_kc(s)), 64), "kseed": (xf_kseed, 128),
            **{"ro%d" % k: (lambda s, k=k: xf_ro_le(s, k), 128) for k in (0, 3, 5, 6, 10, 12, 35)}}


def variant(name):
    """'a+b+lb3' composes transforms left to right (lbN: __launch_bounds__ min blocks N)."""
    fs, threads = [], 128
    for part in name.split("+"):
        if part.startswith("lb"):
            fs.append(lambda s, mb=int(part[2:]): xf_lb(s, mb))
        elif re.fullmatch(r"rw\d+_\d+", part):  # rwA_B: xf_rw_le(A, B)
            a_, b_ = map(int, part[2:].split("_"))
            fs.append(lambda s, a_=a_, b_=b_: xf_rw_le(s, a_, b_))
        else:
            f, t = VARIANTS[part]
            fs.append(f)
            threads = min(threads, t)

    def run(src):
        smem = None
        for f in fs:
            r = f(src)
            src, smem = r if isinstance(r, tuple) else (r, smem)
        return (src, smem) if smem is not None else src
    return run, threads


def compile_cubin(src, extra=()):
    d = tempfile.mkdtemp()
    cu, cub = os.path.join(d, "k.cu"), os.path.join(d, "k.cubin")
    open(cu, "w").write(src)
    r = subprocess.run(["nvcc", "-arch=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo", "-cubin", "-Xptxas", "-v",
                        *extra, "-o", cub, cu], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr[-2000:])
    regs = re.search(r"Used (\d+) registers", r.stderr)
    spill = re.search(r"(\d+) bytes spill stores", r.stderr)
    return open(cub, "rb").read(), int(regs.group(1)) if regs else -1, int(spill.group(1)) if spill else 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=40)
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--variants", default="base,kc")
    ap.add_argument("--workload", default="", help="a tools/kernel_probe.py workload name instead of ER(--dim, --p)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--plan-kw", default="{}", help="JSON dict of extra Plan options")
    ap.add_argument("--static", action="store_true", help="compile only: print regs/spills per variant (no GPU)")
    a = ap.parse_args()
    import numpy as np
    import torch
    import cuda.bindings.driver as drv
    import synth
    import paper_2501_15126_b200 as pb
    A = synth.erdos_renyi(a.dim, a.p, a.seed)
    pkw = dict(mode="reg")
    if a.workload:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from kernel_probe import WORKLOADS
        make, pkw = WORKLOADS[a.workload]
        A = make()
    pkw = {**pkw, **json.loads(a.plan_kw)}
    if a.static:
        P = pb.Plan.from_dense(A, no_device=True, **pkw)
        for name in a.variants.split(","):
            s = variant(name)[0](P.source)
            s, smem = s if isinstance(s, tuple) else (s, P.info["smem_bytes"])
            cub, regs, spill = compile_cubin(s)
            with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
                f.write(cub)
                f.flush()
                sass = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout
            print(json.dumps({"variant": name, "regs": regs, "spill": spill, "smem": smem, "U": P.info["U"],
                              "umov": sass.count("UMOV "), "lds": sass.count("LDS"), "sts": sass.count("STS")}))
        return
    torch.cuda.init()
    P = pb.Plan.from_dense(A, device=0, autotune=-1, **pkw)
    info = P.info
    src = P.source
    base_ms = None
    base_slots = None
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream(device=dev)
    tasks = info["tasks"]
    slots = torch.zeros(tasks * 2, dtype=torch.float64, device=dev)  # complex slots: 2 doubles
    counter = torch.zeros(64, dtype=torch.int32, device=dev)
    tier = torch.zeros(1 << 20, dtype=torch.float64, device=dev)
    for name in a.variants.split(","):
        xf, threads = variant(name)
        s = xf(src)
        smem = info["smem_bytes"]
        if isinstance(s, tuple):
            s, smem = s
        cub, regs, spill = compile_cubin(s)
        err, mod = drv.cuModuleLoadData(cub)
        assert err == drv.CUresult.CUDA_SUCCESS, err
        err, fn = drv.cuModuleGetFunction(mod, b"perm_sweep")
        if smem:
            drv.cuFuncSetAttribute(fn, drv.CUfunction_attribute.CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem)
        err, bps = drv.cuOccupancyMaxActiveBlocksPerMultiprocessor(fn, threads, smem)
        grid = bps * info["sms"]
        args = (np.array([0], np.uint64), np.array([tasks], np.uint32), np.array([1], np.uint64),
                np.array([counter.data_ptr()], np.uint64), np.array([slots.data_ptr()], np.uint64),
                np.array([tier.data_ptr()], np.uint64))
        arg_ptrs = np.array([x.ctypes.data for x in args], dtype=np.uint64)
        times = []
        for r in range(a.reps + 1):
            counter.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            err, = drv.cuLaunchKernel(fn, grid, 1, 1, threads, 1, 1, smem, stream.cuda_stream, arg_ptrs.ctypes.data, 0)
            assert err == drv.CUresult.CUDA_SUCCESS, err
            e1.record(stream)
            torch.cuda.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        out = slots.cpu().numpy().copy()
        if base_slots is None:
            base_slots, base_ms = out, min(times)
        same = bool(np.array_equal(out.view(np.uint64), base_slots.view(np.uint64)))
        umov = None
        try:
            with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
                f.write(cub)
                f.flush()
                umov = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout.count("UMOV")
        except Exception:
            pass
        print(json.dumps({"variant": name, "regs": regs, "spill": spill, "blocks_per_sm": bps, "ms_min": min(times),
                          "ms_med": sorted(times)[len(times) // 2], "speedup_vs_base": base_ms / min(times), "threads": threads,
                          "slots_bitwise_equal": same, "umov_static": umov, "K": info["K"], "B": info["B"],
                          "U": info["U"], "w_plan": info["w_plan"]}), flush=True)
        drv.cuModuleUnload(mod)


if __name__ == "__main__":
    main()
