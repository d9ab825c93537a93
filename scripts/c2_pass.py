"""A few two-sweep passes of a 256^3 Coulomb lattice (the C2 shape) through
psg_run: the target of an ncu capture of k_sweep2b (developer tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0904_0939_b200 import workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
w = workloads.scaled(workloads.CONFIGS["C2"], n)
with Slab(w.spec) as s:
    workloads.fill_slab(s, w)
    s.run(8, 0, 0)
    s.sync()
    print("ok", n)
