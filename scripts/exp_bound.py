"""Is the sweep memory- or compute-bound? Compare the real library with an
experimental build without the IEEE divisions (developer tool)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
variant = sys.argv[1]
from paper_0904_0939_b200 import _lib  # noqa: E402

if variant == "nodiv":
    _lib.LIB_PATH = os.path.join(HERE, "libpsigpu_nodiv.so")
import torch  # noqa: E402

from paper_0904_0939_b200.device import F_WRITE  # noqa: E402
from scripts.quick_bench import make  # noqa: E402


def clk():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                          capture_output=True, text=True).stdout.strip()


torch.cuda.init()
for n in (256, 512):
    s = make(n)
    st = torch.cuda.ExternalStream(s.stream)
    for steps in (200, 2000 if n == 256 else 400):
        s.run(20, 0, 0)
        s.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.run(steps, 0, 0)
        e1.record(st)
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / steps
        print(f"{variant:6s} N={n} steps={steps} {us:8.2f} us/step frac={24 * n ** 3 / us / 1e3 / 6541.8:.3f} [{clk()}]", flush=True)
    s.close()
