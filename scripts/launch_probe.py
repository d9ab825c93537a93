"""Short runs for ncu launch lists (developer tool).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \\
        python scripts/launch_probe.py linear 256
modes: linear (renormalising pairs), exact (per-step norm), plain (plain
pairs), c1 (64^3 BASELINE
cadence through the persistent small-lattice kernel).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0904_0939_b200 import workloads
from paper_0904_0939_b200.device import Slab


def main():
    mode = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    w = workloads.scaled(workloads.CONFIGS["C2"], n) if mode != "c1" else workloads.CONFIGS["C1"]
    with Slab(w.spec) as s:
        workloads.fill_slab(s, w)
        if mode == "c1":
            s.run(300, measure_every=100, norm_every=100)
        elif mode == "plain":
            s.run(12, 0, 0)
        else:
            s.run(12, 0, 1, linear_norm=(mode == "linear"))
        s.sync()
    print("ok", flush=True)


if __name__ == "__main__":
    main()
