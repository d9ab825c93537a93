"""Micro-benchmark of the engine primitives (developer tool)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0904_0939_b200.device import F_MEASURE, F_NORM, F_WRITE
from scripts.quick_bench import make


def clocks():
    try:
        return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu",
                               "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    except Exception:
        return "?"


def bench(s, n, label, body, reps=100):
    st = torch.cuda.ExternalStream(s.stream)
    for _ in range(5):
        body()
    s.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        body()
    e1.record(st)
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    glups = n ** 3 / (us * 1e-6) / 1e9
    print(f"N={n} {label:34s} {us:8.2f} us  {glups:6.1f} GLUPS  frac={24 * glups / 6541.8:.3f}  [{clocks()}]", flush=True)


if __name__ == "__main__":
    torch.cuda.init()
    for n in [int(x) for x in (sys.argv[1:] or ["256", "512"])]:
        s = make(n)
        w = s.w

        def sweep(flags, renorm):
            def f():
                s.sweep(1, w, flags)
                s.swap(renorm)
            return f

        s.reduce(1, w, F_NORM, combine=True)  # valid factor in scal
        for rep in range(2):
            bench(s, n, "W", sweep(F_WRITE, False))
            bench(s, n, "W+scale", sweep(F_WRITE, True))
            bench(s, n, "W+N", sweep(F_WRITE | F_NORM, False))
            bench(s, n, "W+N+scale", sweep(F_WRITE | F_NORM, True))
            bench(s, n, "W+N+M+scale", sweep(F_WRITE | F_NORM | F_MEASURE, True))
            bench(s, n, "M only", lambda: s.measure())
            bench(s, n, "reduce N (no combine)", lambda: s.reduce(1, w, F_NORM, combine=False))
            bench(s, n, "reduce N + combine", lambda: s.reduce(1, w, F_NORM, combine=True))
            bench(s, n, "reduce NM + combine", lambda: s.reduce(1, w, F_NORM | F_MEASURE, combine=True))
            bench(s, n, "norm_partials", lambda: s.norm_partials())
        s.close()
