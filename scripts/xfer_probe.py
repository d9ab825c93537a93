"""Host <-> device transfer rate of a dense padded field through the staging
engine (pageable host array), for a given PSG_HOST_THREADS (developer tool).

    PSG_HOST_THREADS=8 python scripts/xfer_probe.py [--n 1024] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_0904_0939_b200.device import Slab  # noqa: E402
from paper_0904_0939_b200.lattice import LatticeSpec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
spec = LatticeSpec(N=a.n, a=0.1, m=1.0, dtau=0.0025)
host = np.ones((a.n + 2,) * 3)
out = np.empty_like(host)
out.fill(0.0)   # resident pages, like the e2e leg's out=psi0
up, down = [], []
with Slab(spec) as s:
    for _ in range(a.reps):
        t0 = time.perf_counter()
        s.set_field(host)
        s.sync()
        t1 = time.perf_counter()
        s.get_field(out=out)
        t2 = time.perf_counter()
        up.append(host.nbytes / (t1 - t0) / 1e9)
        down.append(host.nbytes / (t2 - t1) / 1e9)
print(json.dumps({"threads": os.environ.get("PSG_HOST_THREADS", "default"), "n": a.n,
                  "gb": host.nbytes / 1e9, "upload_gbs": up, "download_gbs": down}))
