"""Two-sweep pass time at large N vs chunk / z-chunk / work split (developer tool).

    python scripts/large_tune.py [N] [--chunks 0,128,256,512] [--zcs 0,32,64,128] [--segs 0,1,2] [--lib PATH]

Compare settings in SEPARATE processes, alternating: the first setting timed in a process
runs before the board reaches its power cap and looks 1-3 % faster than it is.

Single-buffer slab with device-generated C5 inputs; prints one JSON line per
setting: mean pass time over `reps` back-to-back passes and the GB/s of the
algorithmic 24 B/site.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_0904_0939_b200 import _lib, workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", type=int, nargs="?", default=2048)
    ap.add_argument("--chunks", default="0")
    ap.add_argument("--zcs", default="0")
    ap.add_argument("--segs", default="0")
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--single", type=int, default=1)
    ap.add_argument("--set", default="", help="Slab setters to call first: method=value[,method=value]")
    ap.add_argument("--reserve", type=int, default=-1, help="time psg_pass with this many SMs left idle instead of psg_run")
    ap.add_argument("--lib", default="", help="library to load instead of the tree's (scripts/ab builds)")
    a = ap.parse_args()
    if a.lib:
        _lib.LIB_PATH = a.lib
    w = workloads.scaled(workloads.CONFIGS["C5"], a.n)
    n = w.spec.N
    for chunk in [int(x) for x in a.chunks.split(",")]:
        _lib.load().psg_trim_memory(0)
        s = Slab(w.spec, single_buffer=bool(a.single), chunk=chunk)
        workloads.fill_slab(s, w)
        for kv in filter(None, a.set.split(",")):
            k, v = kv.split("=")
            getattr(s, k)(int(v))
        st = torch.cuda.ExternalStream(s.stream)
        for zc in [int(x) for x in a.zcs.split(",")]:
            for seg in [int(x) for x in a.segs.split(",")]:
                s.tune(0, zc, 0)
                s.set_t2_seg(seg)
                s.run(4, 0, 0)
                s.sync()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                l0 = s.launches()
                e0.record(st)
                if a.reserve >= 0:
                    for _ in range(a.reps):
                        s.pass2(a.reserve)
                else:
                    s.run(2 * a.reps, 0, 0)
                e1.record(st)
                e1.synchronize()
                t = e0.elapsed_time(e1) * 1e-3 / a.reps
                print(json.dumps({"n": n, "lib": os.path.basename(a.lib) or "tree", "set": a.set, "reserve": a.reserve, "chunk": chunk, "zc": zc, "seg": seg,
                                  "pass_ms": t * 1e3, "GBps": 24 * n ** 3 / t / 1e9,
                                  "launches_per_pass": (s.launches() - l0) / a.reps}), flush=True)
        s.close()


if __name__ == "__main__":
    main()
