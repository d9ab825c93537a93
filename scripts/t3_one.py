import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0904_0939_b200 import workloads
from paper_0904_0939_b200.device import Slab
n = int(sys.argv[1]); t3 = int(sys.argv[2])
w = workloads.scaled(workloads.CONFIGS["C5"], n)
with Slab(w.spec) as s:
    workloads.fill_slab(s, w)
    s.set_option(12, 0); s.set_option(14, t3)
    s.run(12, 0, 0); s.sync()
print("ok")
