import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0904_0939_b200 import workloads
from paper_0904_0939_b200.device import Slab
w = workloads.CONFIGS["C1"]
for opt in [(12, 0, 0), (12, 1, 0)]:
    with Slab(w.spec) as s:
        workloads.fill_slab(s, w)
        s.set_option(12, opt[1])
        st = torch.cuda.ExternalStream(s.stream)
        s.run(98, 0, 0); s.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); s.run(980, 0, 0); e1.record(st); e1.synchronize()
        print(opt, "us/step", e0.elapsed_time(e1) * 1e3 / 980, flush=True)
