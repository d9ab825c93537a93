"""Cost of the fused-exchange two-sweep pass (k_sweep2b<..., PEER>) against the
plain pass on the same slab geometry (developer tool; run under ncu for
per-launch numbers).

    python scripts/fused_probe.py [--lattice 256] [--passes 6]

Runs two in-process slabs of W = N/2 through psg_run_multi (every pair of
plain sweeps is one fused pass per slab, storing its edge planes into the
other slab's halos), then the same passes on one W = N/2 slab with psg_pass
(plain kernel, no peer stores).  Prints CUDA-event times per pass of each.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_0904_0939_b200 import workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab, run_multi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", type=int, default=256)
    ap.add_argument("--passes", type=int, default=6)
    a = ap.parse_args()
    w = workloads.scaled(workloads.CONFIGS["C2"], a.lattice)
    spec = w.spec
    n = spec.N
    half = n // 2
    slabs = []
    for lo in (1, half + 1):
        s = Slab(spec, w=half, x_lo=lo, single_buffer=False)
        s.fill_uniform(1)
        s.fill_potential(1)
        s.set_temporal(True)
        slabs.append(s)
    run_multi(slabs, 2 * a.passes, measure_every=0, norm_every=0)
    fused = [s.fused_passes() for s in slabs]
    for s in slabs:
        s.sync()
    st = torch.cuda.ExternalStream(slabs[0].stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    run_multi(slabs, 2 * a.passes, measure_every=0, norm_every=0)
    e1.record(st)
    e1.synchronize()
    t_multi = e0.elapsed_time(e1) * 1e3 / a.passes
    for s in slabs:
        s.close()
    s = Slab(spec, w=half, x_lo=1, single_buffer=False)   # slab 0's geometry
    s.fill_uniform(1)
    s.fill_potential(1)
    s.set_temporal(True)
    st = torch.cuda.ExternalStream(s.stream)
    for _ in range(a.passes):
        s.pass2(0)
    s.sync()
    e0.record(st)
    for _ in range(a.passes):
        s.pass2(0)
    e1.record(st)
    e1.synchronize()
    t_one = e0.elapsed_time(e1) * 1e3 / a.passes
    s.close()
    print(json.dumps({"n": n, "w": half, "fused_passes": fused,
                      "two_fused_slabs_us_per_pass": t_multi, "one_plain_slab_us_per_pass": t_one}))


if __name__ == "__main__":
    main()
