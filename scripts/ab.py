"""A/B of library builds on one box (developer tool).

    python scripts/ab.py build NAME [-DFLAG ...]    # here: builds scripts/ab/libpsigpu_NAME.so
    python scripts/ab.py run NAME1 LIB@LABEL ... [--n 256,512] [--reps 3] [--opt LIB@LABEL:method=value]
"""
import json
import os
import statistics
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
ABDIR = os.path.join(HERE, "ab")


def build(name, flags):
    os.makedirs(ABDIR, exist_ok=True)
    src = os.path.join(ROOT, "paper_0904_0939_b200", "csrc", "psigpu.cu")
    for f in list(flags):
        if f.startswith("--src="):
            src = f[len("--src="):]
            flags.remove(f)
    out = os.path.join(ABDIR, f"libpsigpu_{name}.so")
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
           "-lineinfo", "--fmad=false", "-std=c++17", *flags, "-Xcompiler", "-fPIC", "-shared",
           "-cudart", "static", "-I", os.path.join(ROOT, "include"),
           # a --src= copy finds its own headers first, then the tree's
           "-I", os.path.join(ROOT, "paper_0904_0939_b200", "csrc"), "-o", out, src]
    subprocess.run(cmd, check=True)
    print(out)


CHILD = r'''
import sys, json
sys.path.insert(0, ROOTDIR)
from paper_0904_0939_b200 import _lib
_lib.LIB_PATH = LIBPATH
import torch
from scripts.quick_bench import make
torch.cuda.init()
res = {}
opts = dict(OPTS)
ne = opts.pop("norm_every", 0)   # pseudo-option: renormalise every ne sweeps
for n in NS:
    s = make(n)
    for k, v in opts.items():
        getattr(s, k)(v)
    st = torch.cuda.ExternalStream(s.stream)
    steps = STEPS[n]
    s.run(20, 0, ne); s.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); s.run(steps, 0, ne); e1.record(st); e1.synchronize()
    res[n] = e0.elapsed_time(e1) * 1e3 / steps
    s.close()
print(json.dumps(res))
'''


def run(names, ns, reps, opts):
    steps = {n: max(40, min(4000, int(2.5e10 / n ** 3))) for n in ns}
    table = {nm: {n: [] for n in ns} for nm in names}
    for r in range(reps):
        for nm in names:
            libname = nm.split("@")[0]
            lib = os.path.join(ABDIR, f"libpsigpu_{libname}.so") if libname != "tree" else \
                os.path.join(ROOT, "paper_0904_0939_b200", "libpsigpu.so")
            code = CHILD.replace("ROOTDIR", repr(ROOT)).replace("LIBPATH", repr(lib)) \
                .replace("NS", repr(ns)).replace("STEPS", repr(steps)).replace("OPTS", repr(opts.get(nm, {})))
            out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
            if out.returncode:
                print(nm, "FAILED", out.stderr[-2000:])
                continue
            res = json.loads(out.stdout.strip().splitlines()[-1])
            for n in ns:
                table[nm][n].append(res[str(n)])
            print(f"rep {r} {nm:12s} " + "  ".join(f"N={n}: {res[str(n)]:8.2f} us" for n in ns), flush=True)
    print("median us/step (frac of 6541.8 GB/s):")
    for nm in names:
        cells = []
        for n in ns:
            v = statistics.median(table[nm][n]) if table[nm][n] else float("nan")
            cells.append(f"N={n}: {v:8.2f} ({24 * n ** 3 / v / 1e3 / 6541.8:.3f})")
        print(f"  {nm:12s} " + "  ".join(cells))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3:])
    else:
        args = sys.argv[2:]
        ns, reps, names, opts = [256, 512], 3, [], {}
        i = 0
        while i < len(args):
            if args[i] == "--n":
                ns = [int(x) for x in args[i + 1].split(",")]
                i += 2
            elif args[i] == "--reps":
                reps = int(args[i + 1])
                i += 2
            elif args[i] == "--opt":  # NAME:method=value
                nm, kv = args[i + 1].split(":")
                k, v = kv.split("=")
                opts.setdefault(nm, {})[k] = int(v)
                i += 2
            else:
                names.append(args[i])
                i += 1
        run(names, ns, reps, opts)
