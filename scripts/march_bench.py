"""march vs per-step launches (developer tool).  set_march(v): 0 off, 1 on,
2|3 diagnostic variants (bit0 of v>>1: per-thread fence, bit1: no waits)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from scripts.quick_bench import make


def t(s, n, steps, mode, label, zc=0):
    s._lib.psg_set_march(s.handle, mode)
    s.tune(0, zc, 0)
    st = torch.cuda.ExternalStream(s.stream)
    s.run(20, 0, 0)
    s.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.run(steps, 0, 0)
    e1.record(st)
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / steps
    g = n ** 3 / us / 1e3
    print(f"N={n} {label:28s} zc={zc:3d} {us:8.2f} us/step {g:6.1f} GLUPS frac={24 * g / 6541.8:.3f}", flush=True)


if __name__ == "__main__":
    torch.cuda.init()
    for n in [int(x) for x in (sys.argv[1:] or ["256", "512"])]:
        s = make(n)
        steps = 1000 if n <= 256 else 300
        for rep in range(2):
            for zc in (0, 8, 16, 32):
                s.set_temporal(False)
                t(s, n, steps, 0, "single-step launches", zc)
                s.set_temporal(True)
                t(s, n, steps, 0, "two steps per pass", zc)
        s.close()
