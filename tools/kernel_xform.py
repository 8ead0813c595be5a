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


def xf_b64(src):
    return re.sub(r"__launch_bounds__\(128, (\d+)\)", r"__launch_bounds__(64, \1)", src)


VARIANTS = {"base": (lambda s: s, 128), "kc": (xf_kc, 128), "b64": (xf_b64, 64), "kc_b64": (lambda s: xf_b64(xf_kc(s)), 64)}


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
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--plan-kw", default="{}", help="JSON dict of extra Plan options")
    a = ap.parse_args()
    import numpy as np
    import torch
    import cuda.bindings.driver as drv
    import synth
    import paper_2501_15126_b200 as pb
    torch.cuda.init()
    A = synth.erdos_renyi(a.dim, a.p, a.seed)
    P = pb.Plan.from_dense(A, mode="reg", device=0, autotune=-1, **json.loads(a.plan_kw))
    info = P.info
    src = P.source
    base_ms = None
    base_slots = None
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream(device=dev)
    tasks = info["tasks"]
    slots = torch.zeros(tasks, dtype=torch.float64, device=dev)
    counter = torch.zeros(64, dtype=torch.int32, device=dev)
    tier = torch.zeros(1 << 20, dtype=torch.float64, device=dev)
    for name in a.variants.split(","):
        xf, threads = VARIANTS[name]
        s = xf(src)
        cub, regs, spill = compile_cubin(s)
        err, mod = drv.cuModuleLoadData(cub)
        assert err == drv.CUresult.CUDA_SUCCESS, err
        err, fn = drv.cuModuleGetFunction(mod, b"perm_sweep")
        smem = info["smem_bytes"]
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
