"""CPU-side tests of the product: the C-ABI library loads and exports every
symbol include/perm.h declares; host planner entry points match the planner
oracle bit for bit; codegen + NVRTC (sm_100a) run without a GPU and produce
spill-free kernels.  No compute call is made (no GPU here)."""
import json
import os
import re
import shutil
import subprocess
import tempfile

import numpy as np
import pytest

import paper_2501_15126_b200 as pb
from paper_2501_15126_b200 import _abi
from oracle import planner as OP
from conftest import ROOT
import synth
from conftest import ROOT


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "perm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(perm_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _abi.lib()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_abi.EXPORTS)
    assert "sm_100a" in pb.perm_version()


def test_nm_exports():
    out = subprocess.run(["nm", "-D", _abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (perm_\w+)", out))
    assert set(header_symbols()) <= exported


def ccs_crs(A):
    cp, ri, cv = synth.to_ccs(A)
    rp, ci, rv = synth.to_crs(A)
    return (cp, ri, cv), (rp, ci, rv)


@pytest.mark.parametrize("n,p,seed", [(10, 0.3, 1), (20, 0.2, 2), (40, 0.2, 3), (40, 0.1, 4), (44, 0.3, 5)])
def test_alg3_matches_oracle(n, p, seed):
    A = synth.erdos_renyi(n, p, seed)
    (cp, ri, cv), (rp, ci, rv) = ccs_crs(A)
    rowp, colp = pb.perm_order(n, pb.PERM_CCS, cp, ri, cv, "permanent")
    orow, ocol = OP.permanent_ordering(n, cp, ri, rp, ci)
    assert rowp == orow and colp == ocol
    # CRS input gives the same ordering
    rowp2, colp2 = pb.perm_order(n, pb.PERM_CRS, rp, ci, rv, "permanent")
    assert rowp2 == orow and colp2 == ocol
    d_row, d_col = pb.perm_order(n, pb.PERM_CCS, cp, ri, cv, "degree")
    assert d_col == OP.degree_sort_ascending(n, cp) and d_row == list(range(n))


@pytest.mark.parametrize("n,p,seed", [(12, 0.3, 1), (40, 0.2, 2), (40, 0.3, 3), (36, 0.2, 4)])
def test_alg4_matches_oracle(n, p, seed):
    A = synth.erdos_renyi(n, p, seed)
    (cp, ri, cv), (rp, ci, rv) = ccs_crs(A)
    orow, ocol = OP.permanent_ordering(n, cp, ri, rp, ci)
    B = A[np.ix_(orow, ocol)]
    bcp, bri, _ = synth.to_ccs(B)
    for sms in (108, 148):
        k, c = pb.perm_partition(n, bcp, bri, 16.0, sms)
        assert (k, c) == OP.partitioning(n, bcp, bri, 16.0, lambda r: OP.calculate_no_threads(r, sms=sms))


def test_alg4_fig3b_fixture_a100_model():
    from test_planner_oracle import read_golden
    lines = read_golden("fig3b_ordered.txt")
    n = int(lines[0])
    A = np.zeros((n, n))
    for l in lines[1:]:
        r, c, v = l.split()
        A[int(r), int(c)] = float(v)
    cp, ri, _ = synth.to_ccs(A)
    assert pb.perm_partition(n, cp, ri, 16.0, 108) == (4, 3)


def test_alg2_matches_oracle():
    for tau in (4, 32, 1024, 55296):
        for n in (12, 16, 22, 40):
            assert pb.perm_alg2_launch_parameters(tau, n) == OP.generate_launch_parameters(tau, n)


def test_structural_rank_matches_oracle():
    import oracle
    rng = np.random.default_rng(0)
    for t in range(20):
        n = 3 + t % 10
        A = (rng.uniform(size=(n, n)) < 0.25) * rng.uniform(0.5, 1, (n, n))
        cp, ri, cv = synth.to_ccs(A)
        assert pb.perm_structural_rank(n, pb.PERM_CCS, cp, ri, cv) == oracle.structural_rank(A)


@pytest.mark.parametrize("bad", ["dup", "range", "zero", "nan", "ptr0", "n0", "n65"])
def test_validation_errors(bad):
    A = synth.erdos_renyi(6, 0.5, 1)
    cp, ri, cv = [x.copy() for x in synth.to_ccs(A)]
    n = 6
    if bad == "dup":
        j = next(j for j in range(n) if cp[j + 1] - cp[j] >= 2)
        ri[cp[j] + 1] = ri[cp[j]]
    elif bad == "range":
        ri[0] = 17
    elif bad == "zero":
        cv[0] = 0.0
    elif bad == "nan":
        cv[0] = np.nan
    elif bad == "ptr0":
        cp = cp + 1
    elif bad == "n0":
        n = 0
    elif bad == "n65":
        n = 65
    with pytest.raises(pb.PermError) as e:
        pb.perm_plan(n, pb.PERM_CCS, cp, ri, cv, "auto", pb.make_opts(no_device=True))
    assert e.value.status in (1, 2)


def test_no_device_plan_then_compute_fails_loudly():
    A = synth.erdos_renyi(12, 0.3, 1)
    P = pb.Plan.from_dense(A, no_device=True)
    with pytest.raises(pb.PermError):
        P.compute()


@pytest.mark.parametrize("n,p,seed,mode", [(10, 0.3, 1, "auto"), (30, 0.3, 1, "reg"), (36, 0.2, 1, "reg"),
                                           (40, 0.2, 1, "reg"), (40, 0.2, 2, "reg"), (12, 0.3, 3, "int01")])
def test_codegen_compiles_within_spill_tolerance(n, p, seed, mode):
    """Real FP64 accepts a local frame of <= 96 bytes per thread (DESIGN
    3.13(f)); INT01 (without autotune) and complex kernels stay spill-free."""
    A = synth.erdos_renyi(n, p, seed, binary=(mode == "int01"))
    P = pb.Plan.from_dense(A, ordering="auto", mode=mode, no_device=True)
    i = P.info
    assert i["local_bytes"] <= (0 if i["mode"] == 3 else 96)
    assert 0 < i["regs_per_thread"] <= 255
    assert i["w_plan"] > 0
    assert "perm_sweep" in P.source
    cub = P.cubin()
    assert len(cub) > 1000
    if shutil.which("cuobjdump"):
        with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
            f.write(cub)
            f.flush()
            sass = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout
        assert "sm_100a" in sass
        if i["local_bytes"] == 0:
            assert not re.search(r"\b(LDL|STL)\b", sass), "local memory in generated kernel"
        with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
            f.write(cub)
            f.flush()
            elf = subprocess.run(["cuobjdump", "-elf", f.name], capture_output=True, text=True).stdout
        # the planner reads registers / frame from the cubin's .nv.info (not the ptxas log)
        m = re.search(r"register count: (\d+)", elf)
        assert m and int(m.group(1)) == i["regs_per_thread"]
        fr = re.search(r"frame size: (0x[0-9a-f]+)", elf)
        assert (0 if fr is None else int(fr.group(1), 16)) <= i["local_bytes"]
        if mode != "int01":
            assert re.search(r"\bD(ADD|MUL|FMA)\b", sass)


def test_hybrid_codegen_uses_coalesced_tier(monkeypatch):
    A = synth.erdos_renyi(36, 0.2, 1)
    P = pb.Plan.from_dense(A, mode="hybrid", factor_cols=-1, no_device=True)
    i = P.info
    assert i["mode"] == 2 and i["tier_rows"] > 0 and i["local_bytes"] == 0
    src = P.source
    # x[nthreads*row + tid] (Listing 4), vectorised: row pairs as one double2 per thread
    assert "#define TIER2(p) (reinterpret_cast<double2*>(tier)[(size_t)(p) * nt_ + gt_])" in src
    assert "= TIER2(" in src and "TIER2(0) = make_double2(" in src
    assert "SG" in src                                              # cached tier product (globalProduct)
    # same geometry and ordering: the tier takes rows out of the register file
    geo = dict(factor_cols=-1, chunk_log2=i["B"], block_log2=i["U"], ordering=["none", "degree", "permanent"][i["ordering"]])
    H = pb.Plan.from_dense(A, mode="hybrid", no_device=True, **geo)
    R = pb.Plan.from_dense(A, mode="reg", no_device=True, **geo)
    assert H.info["tier_rows"] > 0 and H.info["reg_rows"] < R.info["reg_rows"]
    # against x kept wholly in registers (no shared-memory placement) the
    # global tier frees registers; the B200 shared-memory placement of the same
    # block-boundary state frees more (DESIGN 3.5)
    monkeypatch.setenv("PERM_NO_SMEM", "1")
    R0 = pb.Plan.from_dense(A, mode="reg", no_device=True, **geo)
    monkeypatch.delenv("PERM_NO_SMEM")
    assert R0.info["smem_bytes"] == 0 and R.info["smem_bytes"] > 0
    assert H.info["regs_per_thread"] < R0.info["regs_per_thread"]
    assert R.info["regs_per_thread"] <= H.info["regs_per_thread"]
    # the row pairs move as 128-bit global accesses (LDG.E.128 / STG.E.128)
    if shutil.which("cuobjdump"):
        with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
            f.write(P.cubin())
            f.flush()
            sass = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout
        assert "LDG.E.128" in sass and "STG.E.128" in sass


def test_codegen_literals_are_exact_hex():
    # Listing 2 analogue: the column-0 values appear as exact literals
    A = np.zeros((6, 6))
    for r, v in [(0, 11.6), (2, 2.6), (3, 1.8), (5, 9.9)]:
        A[r, 0] = v
    for i in range(6):
        A[i, (i + 1) % 6 if i != 5 else 1] = 1.0
    P = pb.Plan.from_dense(A, ordering="none", mode="reg", no_device=True, factor_cols=-1)
    src = P.source
    for v in (11.6, 2.6, 1.8, 9.9):
        assert v.hex() in src


@pytest.mark.parametrize("n,p,seed", [(12, 0.3, 1), (30, 0.3, 1), (36, 0.2, 1), (40, 0.2, 1), (40, 0.2, 2)])
@pytest.mark.parametrize("fc", [0, 2, -1])
def test_factored_ordering_matches_oracle(n, p, seed, fc):
    """The base ordering (Alg. 3 / degree sort) is the oracle's bit for bit; the
    eliminated columns (W-driven greedy, DESIGN 3.6) come first, the base's
    last column stays last, and with no elimination the swept order is the
    base order or its documented cost sort."""
    A = synth.erdos_renyi(n, p, seed)
    P = pb.Plan.from_dense(A, ordering="auto", mode="reg", factor_cols=fc, no_device=True)
    i = P.info
    cp, ri, _ = synth.to_ccs(A)
    rp, ci, _ = synth.to_crs(A)
    if i["ordering"] == 2:
        rowp, colp = OP.permanent_ordering(n, cp, ri, rp, ci)
    else:
        rowp, colp = list(range(n)), OP.degree_sort_ascending(n, cp)
    assert i["row_perm"] == rowp
    got = i["col_perm"]
    assert sorted(got) == list(range(n))
    assert got[-1] == colp[-1]                       # the eliminated NW column is the base's last
    K = i["K"]
    if fc == -1:
        assert K == 0
    if fc > 0:
        assert K <= fc
    rest = [c for c in colp if c not in got[:K]]
    assert got[K:] == rest or sorted(got[K:-1]) == sorted(rest[:-1])


def test_plan_geometry_and_work_model():
    A = synth.erdos_renyi(40, 0.2, 1)
    P = pb.Plan.from_dense(A, ordering="auto", no_device=True)
    i = P.info
    n = 40
    L = 32 * i["M"] * (1 << i["B"]) << i["K"]
    assert i["tasks"] * L == 1 << (n - 1)          # exact cover of the Gray range
    assert i["tasks"] & (i["tasks"] - 1) == 0       # power of two (sharding)
    assert i["w_plan"] < i["w_alg1"]
    assert sorted(i["row_perm"]) == list(range(n)) and sorted(i["col_perm"]) == list(range(n))


def _sass_dp_count(cubin: bytes) -> int:
    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(cubin)
        f.flush()
        sass = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout
    return len(re.findall(r"\bD(ADD|MUL|FMA)\b", sass))


@pytest.mark.parametrize("n,p,seed", [(30, 0.3, 1), (40, 0.2, 1)])
def test_post_pass_removes_dead_registers_and_contracts(n, p, seed):
    """DESIGN 3.13: every loop-carried register the generated kernel declares is
    read somewhere; single-use products feeding an add/sub become DFMAs; the
    contraction lowers W_plan and the static DP instruction count."""
    A = synth.erdos_renyi(n, p, seed)
    P = pb.Plan.from_dense(A, mode="reg", no_device=True)
    src = P.source
    decls = re.findall(r"^\s*double (\w+) = ", src, re.M)
    for r in decls:
        if r in ("cacc", "lacc"):
            continue
        uses = len(re.findall(rf"\b{r}\b", src))
        defs = 1 + len(re.findall(rf"^\s*{r} = ", src, re.M))
        assert uses > defs, f"register {r} is never read"
    assert re.search(r"= fma\(-?[\w(][^,]*, [^,]+, -", src), "no contracted a*b - c"
    os.environ["PERM_NO_FUSE"] = "1"
    try:
        Q = pb.Plan.from_dense(A, mode="reg", no_device=True, factor_cols=P.info["K"] or -1,
                               chunk_log2=P.info["B"], block_log2=P.info["U"])
    finally:
        del os.environ["PERM_NO_FUSE"]
    if Q.info["K"] == P.info["K"] and Q.info["col_perm"] == P.info["col_perm"]:
        assert P.info["w_plan"] < Q.info["w_plan"]
        if shutil.which("cuobjdump"):
            assert _sass_dp_count(P.cubin()) < _sass_dp_count(Q.cubin())


def test_int01_codegen_uses_narrow_integer_types():
    """DESIGN 3.9: INT01 products run in int / i64 where a magnitude bound
    allows; only the accumulation path needs wrapping u128."""
    B = synth.erdos_renyi(30, 0.25, 2, binary=True)
    P = pb.Plan.from_dense(B, mode="int01", no_device=True)
    src = P.source
    assert P.info["local_bytes"] == 0
    muls = re.findall(r"const (int|i64|u128) t\d+ = .*\*", src)
    narrow = sum(1 for t in muls if t != "u128")
    assert narrow > 0.3 * len(muls), (narrow, len(muls))


def test_int01_zero_aware_placement_is_chosen_for_binary_er():
    """0/1 ER n=40 p=0.2: the planner puts even-degree rows' columns on
    lane-uniform bits (swept order 2) and the kernel skips chunks whose frozen
    product is 0 on all 32 lanes."""
    B = synth.erdos_renyi(40, 0.2, 1, binary=True)
    P = pb.Plan.from_dense(B, mode="int01", no_device=True)
    i = P.info
    assert i["swept_order"] in (2, 3) and i["seed_rows"] > 0
    assert "__all_sync(0xffffffffu, F == 0)" in P.source
    assert sorted(i["col_perm"]) == list(range(40))


def test_maximum_size_n64_plans_full_gray_range():
    """n = 64 (the u64 Gray-index limit): the plan covers exactly 2^63 Gray
    steps with a power-of-two task grid and no local memory."""
    A = synth.givens_brickwork(64, 4, 1)
    P = pb.Plan.from_dense(A, mode="reg", no_device=True)
    i = P.info
    assert i["local_bytes"] <= 96 and i["w_plan"] > 0
    assert i["tasks"] & (i["tasks"] - 1) == 0
    steps = i["tasks"] * 32 * i["M"] * (1 << i["B"]) * (1 << i["K"])
    assert steps == 2 ** 63
    r = P.shard_range(0, 1)
    assert r[-1] == 2 ** 63


def test_smem_placement_of_values_the_body_never_touches(monkeypatch):
    """DESIGN 3.13(d): loop-carried values absent from the block body live in
    per-thread shared-memory slots; none of them appears in the body.
    DESIGN 3.13(f): the spill-escalation rung (the n=40 bench plan takes it)
    also places values the body only reads, at most 6 times, in volatile
    slots: those appear in the body as reads only (at a 64-byte tolerance the
    n=40 plan takes that rung; at the default 96 a plain 88-byte frame wins)."""
    monkeypatch.setenv("PERM_SPILL_OK", "64")
    A = synth.erdos_renyi(40, 0.2, 1)
    P = pb.Plan.from_dense(A, mode="reg", no_device=True, autotune=-1)
    src, i = P.source, P.info
    names = re.findall(r"#define SM_(\w+) ", src)
    assert names and i["smem_bytes"] >= 128 * 8 * len(names) // 2
    body = src[src.index("const double sU"):src.index("lacc += cacc")]
    read_in_body = 0
    for nm_ in names:
        assert not re.search(rf"(?<!SM_)\b{nm_}\b", body)
        uses = len(re.findall(rf"\bSM_{nm_}\b", body))
        if uses:
            read_in_body += 1
            assert uses <= 6
            assert re.search(rf"#define SM_{nm_} \(\(\(volatile double\*\)", src)
            assert not re.search(rf"^\s*SM_{nm_} = ", body, re.M)
    assert read_in_body > 0 and i["local_bytes"] <= 64
    assert "extern __shared__" in src


# ---- round 2: plan transport (disk cache, rank-0 broadcast), knobs in the key ----

def test_plan_export_import_roundtrip_no_device():
    A = synth.erdos_renyi(24, 0.3, 2)
    P = pb.Plan.from_dense(A, mode="reg", no_device=True, autotune=-1)
    blob = P.export()
    Q = pb.Plan.from_blob(blob, no_device=True)
    assert Q.source == P.source and Q.cubin() == P.cubin()
    a, b = P.info, Q.info
    for k in ("n", "nnz", "K", "B", "U", "M", "tasks", "w_plan", "row_perm", "col_perm", "mode"):
        assert a[k] == b[k], k
    assert b["disk_cached"] == 1
    with pytest.raises(pb.PermError):
        pb.Plan.from_blob(blob[:-7], no_device=True)          # truncated
    with pytest.raises(pb.PermError):
        pb.Plan.from_blob(b"X" + blob[1:], no_device=True)    # foreign magic


def test_plan_export_import_keeps_spilling_smem_ro_kernel(monkeypatch):
    """Plan format 4 (DESIGN 3.13(f)): a plan whose kernel keeps a local frame
    and reads body values from volatile shared-memory slots travels through
    export / import (rank-0 broadcast, disk cache) unchanged, and reports its
    frame in local_bytes."""
    monkeypatch.setenv("PERM_SMEM_RO_FORCE", "1")
    monkeypatch.setenv("PERM_SPILL_OK", "4096")
    monkeypatch.setenv("PERM_ELIM_TIER4", "0")  # the plan this fixture was chosen on
    A = synth.erdos_renyi(22, 0.3, 2)
    P = pb.Plan.from_dense(A, mode="reg", block_log2=5, no_device=True, autotune=-1)
    assert P.info["local_bytes"] > 0 and "volatile double" in P.source
    Q = pb.Plan.from_blob(P.export(), no_device=True)
    assert Q.source == P.source and Q.cubin() == P.cubin()
    for k in ("K", "B", "U", "M", "tasks", "w_plan", "smem_bytes", "local_bytes", "regs_per_thread"):
        assert Q.info[k] == P.info[k], k


def test_disk_plan_cache(tmp_path):
    A = synth.erdos_renyi(22, 0.3, 5)
    d = str(tmp_path)
    P = pb.Plan.from_dense(A, mode="reg", no_device=True, autotune=-1, cache_dir=d)
    assert P.info["disk_cached"] == 0
    files = os.listdir(d)
    assert len(files) == 1 and files[0].endswith(".plan")
    # a new process would miss the in-process cache; a different option set is a
    # different key (the in-process cache is keyed identically, so force the disk
    # path by planning through a fresh library state: load the blob directly)
    Q = pb.Plan.from_dense(A, mode="reg", no_device=True, autotune=-1, cache_dir=d)
    assert Q.source == P.source
    R = pb.Plan.from_dense(A * 0.5, mode="reg", no_device=True, autotune=-1, cache_dir=d)
    assert len(os.listdir(d)) == 2 and R.source != P.source


def test_disk_plan_cache_in_fresh_process(tmp_path):
    """A second process plans the same matrix from the disk cache: no search,
    no NVRTC, identical kernel."""
    import subprocess
    import sys
    code = ("import sys, json; sys.path.insert(0, %r); import synth, paper_2501_15126_b200 as pb; "
            "P = pb.Plan.from_dense(synth.erdos_renyi(26, 0.25, 3), mode='reg', no_device=True, autotune=-1, "
            "cache_dir=%r); i = P.info; print(json.dumps([i['disk_cached'], i['plan_ms'], len(P.source)]))"
            % (ROOT, str(tmp_path)))
    out1 = json.loads(subprocess.check_output([sys.executable, "-c", code]).decode().strip().splitlines()[-1])
    out2 = json.loads(subprocess.check_output([sys.executable, "-c", code]).decode().strip().splitlines()[-1])
    assert out1[0] == 0 and out2[0] == 1 and out1[2] == out2[2]
    assert out2[1] < 0.5 * out1[1]


def test_env_knobs_are_part_of_the_plan_key(monkeypatch):
    A = synth.erdos_renyi(20, 0.3, 8)
    P = pb.Plan.from_dense(A, mode="reg", no_device=True, autotune=-1)
    monkeypatch.setenv("PERM_NO_CC", "1")
    Q = pb.Plan.from_dense(A, mode="reg", no_device=True, autotune=-1)
    assert Q.info["plan_cached"] == 0


def test_opts_world_validation_and_result_fields():
    A = synth.erdos_renyi(12, 0.4, 1)
    with pytest.raises(pb.PermError):
        pb.Plan.from_dense(A, no_device=True, world=3, rank=0)
    with pytest.raises(pb.PermError):
        pb.Plan.from_dense(A, no_device=True, world=4, rank=4)
    P = pb.Plan.from_dense(A, no_device=True, reseed_log2=4)
    assert P.info["B"] <= 4
    with pytest.raises(pb.PermError):   # no device: compute fails loudly (no CPU fallback)
        P.compute_ex()


def test_empty_column_is_singular_without_planning():
    """An all-zero column (or row) is structural rank < n: perm = 0 with no
    ordering, codegen or kernel (this used to reach the generator)."""
    A = synth.erdos_renyi(18, 0.3, 1)
    for k in range(2):
        S = A.copy()
        if k == 0:
            S[:, 5] = 0
        else:
            S[5, :] = 0
        P = pb.Plan.from_dense(S, no_device=True)
        assert P.info["singular"] == 1 and P.info["struct_rank"] == 17
        assert P.info["row_perm"] == list(range(18)) and P.info["K"] == 0
        P.close()


def test_checkpoint_auto_pieces_keep_many_waves():
    """checkpoint.auto_pieces: power-of-two pieces of >= 2^14 warp-tasks each
    (~14 waves of a B200's resident warps), at most 128, at least 1."""
    from paper_2501_15126_b200.checkpoint import auto_pieces, MIN_TASKS_PER_PIECE
    big = pb.Plan.from_dense(synth.erdos_renyi(40, 0.2, 1), mode="reg", no_device=True, autotune=-1)
    small = pb.Plan.from_dense(synth.erdos_renyi(20, 0.3, 1), mode="reg", no_device=True, autotune=-1)
    for P in (big, small):
        k = auto_pieces(P)
        t = P.info["tasks"]
        assert k & (k - 1) == 0 and 1 <= k <= 128
        assert k == 1 or t // k >= MIN_TASKS_PER_PIECE
        assert k == 128 or t // (2 * k) < MIN_TASKS_PER_PIECE
    assert auto_pieces(big) == 8 and auto_pieces(small) == 1
