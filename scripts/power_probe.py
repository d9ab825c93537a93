"""Board power at full HBM streaming vs the sweep (developer tool): a device
copy loop (1 read + 1 write per byte) for ~8 s with nvidia-smi sampling, then
plain two-sweep passes at 1024^3 for ~8 s.  Prints median power, SM clock and
achieved rates."""
import os
import subprocess
import sys
import tempfile
import time
import statistics

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

Q = "clocks.sm,power.draw"


def sample(fn):
    fd, path = tempfile.mkstemp(suffix=".csv")
    os.close(fd)
    p = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={Q}", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=open(path, "w"))
    time.sleep(0.3)
    res = fn()
    p.terminate()
    p.wait()
    rows = [l.split(",") for l in open(path) if l.strip()]
    sm = [float(r[0]) for r in rows[len(rows) // 3:]]
    pw = [float(r[1]) for r in rows[len(rows) // 3:]]
    return res, statistics.median(sm), statistics.median(pw)


def copy_loop():
    a = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < 8.0:
        for _ in range(10):
            b.copy_(a)
        torch.cuda.synchronize()
        n += 10
    dt = time.perf_counter() - t0
    return 2 * a.numel() * n / dt / 1e9


def sweep_loop():
    from paper_0904_0939_b200 import workloads
    from paper_0904_0939_b200.device import Slab
    w = workloads.scaled(workloads.CONFIGS["C5"], 1024)
    with Slab(w.spec) as s:
        workloads.fill_slab(s, w)
        s.run(20, 0, 0)
        s.sync()
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < 8.0:
            s.run(20, 0, 0)
            s.sync()
            n += 20
        dt = time.perf_counter() - t0
    return 1024 ** 3 * n / dt / 1e9


def idle():
    time.sleep(3)
    return 0.0


for name, fn in (("idle", idle), ("copy GB/s", copy_loop), ("sweep GLUPS 1024^3", sweep_loop)):
    r, sm, pw = sample(fn)
    print(f"{name}: {r:.1f}  sm_mhz {sm:.0f}  power_w {pw:.0f}", flush=True)
