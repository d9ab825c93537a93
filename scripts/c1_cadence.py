"""One BASELINE C1 run (64^3 harmonic, 2000 sweeps, norm + observables every
100) through psg_run on one slab: the target of an ncu capture of k_small2
(option 15 on: the checks inside the persistent launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0904_0939_b200 import workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab  # noqa: E402

w = workloads.CONFIGS["C1"]
chk = int(sys.argv[1]) if len(sys.argv) > 1 else 1
with Slab(w.spec) as s:
    workloads.fill_slab(s, w)
    s.set_option(15, chk)
    idx, sums, st = s.run(2000, 100, 100)
    s.sync()
    print("checks", len(idx), "status", int(st.max()) if len(st) else 0)
