"""Why the e2e leg's 2048^3 download runs below the link rate (developer tool):
the staged download into different host arrays, before and after a run."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_0904_0939_b200 import workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab  # noqa: E402

w = workloads.CONFIGS["C5"]
spec = w.spec
ext = spec.N + 2
psi0 = np.empty((ext,) * 3)
vhost = np.empty((ext,) * 3)
res = {}


def t(label, f):
    t0 = time.perf_counter()
    f()
    res[label] = round(psi0.nbytes / (time.perf_counter() - t0) / 1e9, 1)


with Slab(spec) as s:
    s.fill_uniform(workloads.PSI_SEED)
    t("get_field_fresh_psi0_GBs", lambda: s.get_field(out=psi0))
    t("get_field_again_psi0_GBs", lambda: s.get_field(out=psi0))
    t("get_potential_fresh_v_GBs", lambda: s.get_potential(out=vhost))
    t("set_field_GBs", lambda: (s.set_field(psi0), s.sync()))
    t("set_potential_GBs", lambda: (s.set_potential(vhost), s.sync()))
    t("get_field_after_uploads_GBs", lambda: s.get_field(out=psi0))
    s.run(4, 0, 0)
    s.sync()
    t("get_field_after_run_GBs", lambda: s.get_field(out=psi0))
print(json.dumps(res))
