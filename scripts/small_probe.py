"""Per-sweep time of the fused loop at small lattices (developer tool): two-sweep
passes on / off, renormalisation every 100 sweeps (BASELINE) or every sweep
(psibox's evolve_to_convergence).  (A CUDA-graph capture option was measured
here and removed: DESIGN.md section 8.)

    python scripts/small_probe.py [--sizes 32,64,96,128,256] [--t2 0,1]
        [--norm 100,1] [--steps 2000] [--segment 0]

--segment k: issue the steps as run() calls of k sweeps (the convergence
loop's check_freq segments), timed over all of them.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_0904_0939_b200 import workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="32,64,96,128")
    ap.add_argument("--t2", default="0,1")
    ap.add_argument("--norm", default="100")
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--segment", type=int, default=0)
    a = ap.parse_args()
    for n in [int(x) for x in a.sizes.split(",")]:
        w = workloads.scaled(workloads.CONFIGS["C1"], n)
        for ne in [int(x) for x in a.norm.split(",")]:
            for t2 in [int(x) for x in a.t2.split(",")]:
                for g in (0,):
                    s = Slab(w.spec)
                    workloads.fill_slab(s, w)
                    s.set_temporal(bool(t2))
                    st = torch.cuda.ExternalStream(s.stream)
                    seg = a.segment or a.steps
                    s.run(2 * seg, 0, ne)
                    s.sync()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    done = 0
                    while done < a.steps:
                        k = min(seg, a.steps - done)
                        s.run(k, 0, ne, step_offset=done)
                        done += k
                    e1.record(st)
                    e1.synchronize()
                    print(json.dumps({"n": n, "norm_every": ne, "t2": t2, "graph": g,
                                      "segment": seg,
                                      "us_per_step": e0.elapsed_time(e1) * 1e3 / a.steps}),
                          flush=True)
                    s.close()


if __name__ == "__main__":
    main()
