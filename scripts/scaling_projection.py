"""Per-GPU work of the C5 strong-scaling run (2048^3, z-slabs over M GPUs)
measured on ONE B200 (developer tool; every box of this build has one GPU).

For M = 1 the whole lattice (single-buffer slab, psg_run); for M = 2, 4, 8 the
slab one GPU holds in the M-GPU run (W = 2048 / M planes of 2048^2, two psi
buffers with deep halos, an interior slab where one exists), its two-sweep
passes timed back to back for a few seconds so the board settles at its power
cap as in the real run; SM clock and power sampled by nvidia-smi meanwhile.

The M-GPU run does exactly this per GPU plus the halo exchange, which the
fused transport performs inside the same pass (edge items store their output
planes into the neighbours' halos as well: 4 of W output planes stored twice),
so projected aggregate = M x per-GPU rate and projected efficiency = per-GPU
rate(M) / rate(1) -- a projection from measured per-GPU work, NOT a multi-GPU
measurement.

    python scripts/scaling_projection.py [--seconds 4] [--ms 1,2,4,8] [--fused 256]

--fused N:M: the C5 recipe at N^3 in M slabs of N / M planes, all on this one
GPU, driven by psg_run_multi (the fused exchange: each two-sweep pass also
stores its edge output planes into the neighbours' halo planes), timed per
slab-pass against an interior slab's plain pass -- the cost of the fused
exchange inside the pass with W = 256 planes per slab as at M = 8 for 2048^3
(2048^3 in 8 two-buffer slabs does not fit one GPU; on one GPU the "peer"
stores are local stores, over NVLink they are remote writes of 4 of W planes).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_0904_0939_b200 import _lib, workloads  # noqa: E402
from paper_0904_0939_b200.device import Slab, run_multi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--ms", default="1,2,4,8")
    ap.add_argument("--fused", default="1024:4")
    a = ap.parse_args()
    w = workloads.CONFIGS["C5"]
    spec = w.spec
    n = spec.N
    base = None
    out = []
    for m in [int(x) for x in a.ms.split(",")]:
        wpl = n // m
        if m == 1:
            s = Slab(spec)   # single-buffer automatically (two buffers do not fit)
        else:
            lo = wpl + 1 if m > 2 else 1   # an interior slab (rank 1) where one exists
            s = Slab(spec, w=wpl, x_lo=lo, single_buffer=False)
        workloads.fill_slab(s, w)
        s.set_temporal(True)
        st = torch.cuda.ExternalStream(s.stream)

        def passes(k):
            if m == 1:
                s.run(2 * k, 0, 0)
            else:
                for _ in range(k):
                    s.pass2(0)

        passes(2)
        s.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        passes(2)
        e1.record(st)
        e1.synchronize()
        t1 = e0.elapsed_time(e1) * 1e-3 / 2
        k = max(4, int(a.seconds / t1))
        with ClockSampler(torch.cuda.current_device()) as clk:
            passes(max(2, k // 4))   # let the clock settle under the power cap
            e0.record(st)
            passes(k)
            e1.record(st)
            e1.synchronize()
        pass_s = e0.elapsed_time(e1) * 1e-3 / k
        glups = 2 * wpl * n * n / pass_s / 1e9
        if base is None and m == 1:
            base = glups
        rec = {"M": m, "planes_per_gpu": wpl, "passes": k, "pass_ms": pass_s * 1e3,
               "per_gpu_glups": glups, "clocks": clk.summary(),
               "projected_aggregate_glups": m * glups,
               "projected_efficiency": (glups / base) if base else None}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        s.close()
        del s
        _lib.load().psg_trim_memory(torch.cuda.current_device())   # return the pool's memory
    if a.fused:
        nf, mf = (int(x) for x in a.fused.split(":"))
        wf = workloads.scaled(w, nf)
        wpl = nf // mf
        sl = [Slab(wf.spec, w=wpl, x_lo=1 + r * wpl, single_buffer=False) for r in range(mf)]
        for sb in sl:
            workloads.fill_slab(sb, wf)
            sb.set_temporal(True)
        run_multi(sl, 8, 0, 0)
        torch.cuda.synchronize()
        k = 100
        t0 = time.perf_counter()
        run_multi(sl, 2 * k, 0, 0)
        torch.cuda.synchronize()
        fused_s = (time.perf_counter() - t0) / (mf * k)   # per slab-pass (the slabs share the GPU)
        fused = sl[1].fused_passes()
        for sb in sl[2:]:
            sb.close()
        sb = sl[1]
        st = torch.cuda.ExternalStream(sb.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(k):
            sb.pass2(0)
        e1.record(st)
        e1.synchronize()
        plain_s = e0.elapsed_time(e1) * 1e-3 / k
        rec = {"fused_exchange": {"N": nf, "slabs_on_one_gpu": mf, "planes_per_slab": wpl,
                                  "fused_passes_of_slab1": fused,
                                  "slab_pass_ms_fused": fused_s * 1e3, "slab_pass_ms_plain": plain_s * 1e3,
                                  "overhead": fused_s / plain_s - 1.0}}
        print(json.dumps(rec), flush=True)
        for sb in sl[:2]:
            sb.close()
    return out


if __name__ == "__main__":
    main()
