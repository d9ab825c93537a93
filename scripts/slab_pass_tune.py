"""Two-sweep pass time of one slab of a z-decomposed lattice on one GPU
(developer tool): the per-GPU cost of the weak-scaling bench's slabs.

    python scripts/slab_pass_tune.py [--cases 320:160,384:96,512:64,256:256]
        [--segs 0,1,2] [--rows 16,8] [--zcs 0] [--reserve 8]

Prints one JSON line per setting: mean pass time over back-to-back passes,
the ideal (the whole-lattice pass's time per site x the slab's sites) is not
computed here -- compare against the case N:N.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_0904_0939_b200 import workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="320:160,384:96,512:64,256:256")
    ap.add_argument("--segs", default="0,1,2")
    ap.add_argument("--rows", default="16")
    ap.add_argument("--zcs", default="0")
    ap.add_argument("--reserve", type=int, default=8)
    ap.add_argument("--reps", type=int, default=100)
    a = ap.parse_args()
    for case in a.cases.split(","):
        n, w = (int(x) for x in case.split(":"))
        spec = workloads.scaled(workloads.CONFIGS["C2"], n).spec
        lo = (n - w) // 2 + 1
        s = Slab(spec, w=w, x_lo=lo, single_buffer=False)
        s.fill_uniform(1)
        s.fill_potential(1)
        s.set_temporal(True)
        st = torch.cuda.ExternalStream(s.stream)
        reserve = a.reserve if w < n else 0
        for rows in [int(x) for x in a.rows.split(",")]:
            for seg in [int(x) for x in a.segs.split(",")]:
                for zc in [int(x) for x in a.zcs.split(",")]:
                    s.set_t2_rows(rows)
                    s.set_t2_seg(seg)
                    s.tune(0, zc, 0)
                    for _ in range(5):
                        s.pass2(reserve)
                    s.sync()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    for _ in range(a.reps):
                        s.pass2(reserve)
                    e1.record(st)
                    e1.synchronize()
                    t = e0.elapsed_time(e1) * 1e-3 / a.reps
                    print(json.dumps({"n": n, "w": w, "rows": rows, "seg": seg, "zc": zc,
                                      "reserve": reserve, "pass_us": t * 1e6,
                                      "ns_per_site_update": t * 1e9 / (2 * w * n * n)}),
                          flush=True)
        s.close()


if __name__ == "__main__":
    main()
