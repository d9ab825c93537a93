"""Benchmark of the imaginary-time FDTD hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Workload (BASELINE.json configs[1], "C2"): Coulomb V = -1/max(r, a/2) on a
256^3 fp64 lattice, a = 0.1, dtau = a*a/4, seeded U(-0.5, 0.5) start
(synthetic, workloads.py), observables + renormalisation every 500 sweeps.
A step is one sweep of the whole lattice.  Metric: lattice-site updates per
second (GLUPS), whole job.  psi (2 buffers) + V are 3 x 137 MB, larger than
the 126 MB L2, so no flush is needed between steps.

JSON fields beyond the base contract:
  roofline      dominant kernel vs measured HBM copy bandwidth.  For N >= 8
                the run's plain steps go in pairs through k_sweep2b (two
                sweeps per HBM pass): one launch reads psi and V and writes
                psi once for 2 N^3 site-updates, so achieved = 24 B/site x
                N^3 / mean launch duration (CUDA events on the slab's stream);
                with temporal blocking off the kernel is k_sweep (one sweep per
                launch, same 24 B/site).  traffic from the committed ncu capture
                (profiles/).
  cpu_baseline  the CPU oracle port (oracle/, C + OpenMP, all host threads) on
                a bounded sample of the same workload, rank 0, N=1.
  e2e           the same metric through the public API (evolve_fixed) from
                pinned host arrays: upload psi0 + V, K sweeps, download psi
                and the observable plane sums.
``--config C5`` (2048^3, harmonic + 8 wells): on one GPU a single-buffer slab
with device-generated inputs (run_large; two psi buffers would need 207 GB);
under torchrun the lattice itself is split into M slabs ("scaling": "strong",
the north star's 1/2/4/8-GPU run).  Neither has an e2e leg: at 69 GB per field
the inputs only ever exist in HBM.
``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port: the reference package is Python/numba and cannot be built into
oracle/_ref) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAK_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
BYTES_PER_SITE = 24     # psi read + V read + psi write, fp64


def cpu_model() -> str:
    """The host CPU's model name and logical CPU count (lscpu's "Model name")."""
    name = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    name = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return f"{name} ({os.cpu_count()} logical CPUs)"


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return PEAK_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx = float(f[2])
                except ValueError:
                    continue
                for nm, val in zip(names, f[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(nm)
        except Exception:
            pass
        finally:
            try:
                os.unlink(self.path)
            except Exception:
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_traffic(n, kernel="k_sweep"):
    """dram bytes per launch of `kernel` from the committed ncu capture (or None)."""
    p = os.path.join(ROOT, "profiles", "sweep_traffic.json" if kernel == "k_sweep"
                     else f"{kernel}_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        rec = d.get(str(n))
        return float(rec["dram_bytes_per_launch"]) if rec else None
    except Exception:
        return None


def workload(name="C2"):
    from paper_0904_0939_b200 import workloads

    return workloads.CONFIGS[name]


# ---------------------------------------------------------------------------
# CPU legs (oracle port) — only place the bench executes oracle/
# ---------------------------------------------------------------------------
def cpu_sample(w, target_s=10.0, max_steps=2000):
    """Time the oracle (C, OpenMP, all host threads) on the workload's fixed-step
    loop for a bounded number of sweeps; returns (GLUPS, threads, sample)."""
    from oracle import oracle as O
    from paper_0904_0939_b200 import workloads

    spec = w.spec
    n = spec.N
    psi = np.zeros((n + 2,) * 3)
    psi[1:-1] = workloads.uniform_start(spec)
    v = workloads.potential_planes(w, spec, 0, n + 2)
    out = psi.copy()
    t0 = time.perf_counter()
    O.stencil_update_v(psi, v, spec.dtau, spec.m, spec.a, out, 1, n)
    t1 = time.perf_counter() - t0
    steps = int(min(max(target_s / max(t1, 1e-6), 3), max_steps))
    t0 = time.perf_counter()
    _, checks = O.evolve_fixed(psi, v, n, spec.a, spec.m, spec.dtau, steps, w.measure_every,
                               norm_every=w.measure_every)
    dt = time.perf_counter() - t0
    return (n ** 3 * steps / dt / 1e9, O.threads(),
            f"{steps} sweeps of the {w.name} lattice ({n}^3), fixed-step loop with "
            f"norm/measure every {w.measure_every}, oracle/psi_oracle.c with "
            f"{O.threads()} OpenMP threads")


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation (oracle port)
    on the lattice our arm runs (weak-scaled for N > 1 GPUs, C5 strong), each step
    a bounded sample of it: the leading planes of the lattice, sized so the whole
    warmup + steps run stays within ~3 minutes.  Only those planes (plus their
    two neighbours) are generated on the host, so even 2048^3 fits in memory."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_0904_0939_b200 import workloads

    world = int(os.environ.get("WORLD_SIZE", "1"))
    w = workload(args.config)
    if args.size:
        w = workloads.scaled(w, args.size)
    if world > 1 and not strong_scaling(args):
        n_lat = weak_n(w.N, world)
        if n_lat != w.N:
            w = workloads.scaled(w, n_lat)
    spec = w.spec
    n = spec.N

    def window(planes):
        psi = np.zeros((planes + 2, n + 2, n + 2))
        psi[1:-1] = workloads.uniform_start(spec, first=1, count=planes)
        v = workloads.potential_planes(w, spec, 0, planes + 2)
        return psi, v

    # calibrate on a few planes, then size the sample
    probe = min(n, 32)
    psi, v = window(probe)
    out = psi.copy()
    O.stencil_update_v(psi, v, spec.dtau, spec.m, spec.a, out, 1, probe)   # threads up
    t0 = time.perf_counter()
    O.stencil_update_v(psi, v, spec.dtau, spec.m, spec.a, out, 1, probe)
    t1 = (time.perf_counter() - t0) / probe
    budget = 150.0
    mem_cap = 6e9   # bytes of host arrays (psi, out, V) for the sample
    max_planes = int(mem_cap / (3 * 8 * (n + 2) ** 2)) - 2
    planes = max(1, min(n, max_planes, int(budget / ((args.steps + args.warmup) * t1))))
    psi, v = window(planes)
    out = psi.copy()
    a3 = O.cell_volume(spec.a)

    def one(s):
        nonlocal psi, out
        O.stencil_update_v(psi, v, spec.dtau, spec.m, spec.a, out, 1, planes)
        psi, out = out, psi
        if s % w.measure_every == 0:
            n2 = O.np_sum(O.norm_plane_sums(psi, 1, planes)) * a3
            O.load().oracle_scale(O._p(psi), psi.size, 1.0 / math.sqrt(n2))

    for s in range(1, args.warmup + 1):
        one(s)
    t0 = time.perf_counter()
    for s in range(args.warmup + 1, args.warmup + args.steps + 1):
        one(s)
    dt = time.perf_counter() - t0
    sites = planes * n * n
    glups = sites * args.steps / dt / 1e9
    sample = (f"each step sweeps planes 1..{planes} of the {n}^3 {w.name} lattice "
              f"({sites} sites) with oracle/psi_oracle.c (C port of the reference kernels, "
              f"{O.threads()} OpenMP threads)")
    line = {
        "metric": "fp64 FDTD lattice-site updates/s (GLUPS)", "value": glups, "unit": "GLUPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if strong_scaling(args) and world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "N": n, "a": spec.a, "dtau": spec.dtau,
                   "measure_every": w.measure_every},
        "impl": "reference",
        "cpu_baseline": {"value": glups, "unit": "GLUPS", "cores": O.threads(), "kind": "port",
                         "cpu": cpu_model(),
                         "sample": sample},
        "e2e": {"value": glups, "unit": "GLUPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def _pinned(shape):
    import torch

    return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()


E2E_WARMUP = 2


def run_single(args):
    import torch

    from paper_0904_0939_b200 import Field3D, PotentialGrid, evolve_fixed, workloads
    from paper_0904_0939_b200.device import F_WRITE, Slab

    w = workload(args.config)
    spec = w.spec
    n = spec.N
    ext = n + 2
    dev = 0
    torch.cuda.set_device(dev)
    psi0 = _pinned((ext, ext, ext))
    psi0[...] = 0.0
    psi0[1:-1] = workloads.uniform_start(spec)
    vhost = _pinned((ext, ext, ext))
    vhost[...] = workloads.potential_planes(w, spec, 0, ext)

    slab = Slab(spec, device=dev)
    slab.set_field(psi0)
    slab.set_potential(vhost)
    st = torch.cuda.ExternalStream(slab.stream)
    m = w.measure_every
    slab.run(args.warmup, measure_every=m, norm_every=m)
    slab.sync()

    # ---- timed region: K sweeps, observables + renormalisation every m ----
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = slab.launches()
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        e0.record(st)
        idx, sums, status = slab.run(args.steps, measure_every=m, norm_every=m,
                                     step_offset=args.warmup)
        e1.record(st)
        e1.synchronize()
        torch.cuda.synchronize()
    launches = slab.launches() - l0
    ms = e0.elapsed_time(e1)
    clocks = clk.summary()
    value = n ** 3 * args.steps / (ms * 1e-3) / 1e9
    if status.any():
        raise SystemExit(f"device status {status} during the timed run")

    # ---- mean duration of the dominant kernel (same stream) ----
    # run(2) with no measure / norm is one two-sweep pass (k_sweep2b) when the
    # slab uses temporal blocking, else two k_sweep launches
    l_probe = slab.launches()
    slab.run(2, 0, 0)
    slab.sync()
    two_step = slab.launches() - l_probe == 1
    reps = 50
    if two_step:
        # back to back inside one run() as in the timed region (PDL overlaps a
        # launch's prologue with its predecessor's tail), as long as the timed
        # region so clocks / power settle the same way: the passes of the
        # timed-region schedule (npass), then 3 samples of 50 for the spread
        npass0, _ = t2_schedule(args.steps, args.warmup, m)
        durs = []
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(st)
        slab.run(2 * npass0, 0, 0)
        eb.record(st)
        eb.synchronize()
        long_s = ea.elapsed_time(eb) * 1e-3 / npass0
        for _ in range(3):
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record(st)
            slab.run(2 * reps, 0, 0)
            eb.record(st)
            eb.synchronize()
            durs.append(ea.elapsed_time(eb) * 1e-3 / reps)
    else:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        evs[0].record(st)
        for i in range(reps):
            slab.sweep(1, n, F_WRITE)
            slab.swap(False)
            evs[i + 1].record(st)
        evs[-1].synchronize()
        durs = [evs[i].elapsed_time(evs[i + 1]) * 1e-3 for i in range(reps)]
    kernel_s = statistics.mean(durs)
    short_s = kernel_s
    if two_step:
        kernel_s = long_s   # the steady-state duration under the timed region's load
    slab.close()

    peak, peak_kind = hbm_peak()
    achieved = BYTES_PER_SITE * n ** 3 / kernel_s / 1e9
    traffic = load_traffic(n, "k_sweep2b" if two_step else "k_sweep")
    kname = ("k_sweep2b (two fp64 7-point sweeps per HBM pass, TMA z-march)" if two_step
             else "k_sweep (fp64 7-point, TMA z-march)")
    npass, nsingle = t2_schedule(args.steps, args.warmup, m)
    share = ((npass if two_step else args.steps) * kernel_s) / (ms * 1e-3)

    # ---- e2e through the public API from pinned host buffers ----
    grid = PotentialGrid(spec=spec, v=vhost, v_inf=0.0, unbounded=False, name="custom")
    init = Field3D(spec, psi0)
    e2e_times = []
    # the user-facing call, from host arrays: two untimed warm-up calls (the
    # memory pool and the pinned result cache reach steady state: a caller
    # still holding the previous result makes the second call allocate one
    # more pinned block), then the median of five
    for i in range(E2E_WARMUP + 5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        state = evolve_fixed(init, grid, args.steps, m, norm_every=m)
        if i >= E2E_WARMUP:
            e2e_times.append(time.perf_counter() - t0)
    t_e2e = statistics.median(e2e_times)
    e2e = n ** 3 * args.steps / t_e2e / 1e9
    h2d = 2 * ext ** 3 * 8
    d2h = ext ** 3 * 8 + len(state.checks) * (3 * n + 2) * 8

    cpu = None
    if not args.no_cpu:
        g, cores, sample = cpu_sample(w)
        cpu = {"value": g, "unit": "GLUPS", "cores": cores, "kind": "port", "sample": sample,
               "cpu": cpu_model()}

    line = {
        "metric": "fp64 FDTD lattice-site updates/s (GLUPS)",
        "value": value, "unit": "GLUPS", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "N": n, "a": spec.a, "dtau": spec.dtau,
                   "potential": w.potential, "measure_every": m, "norm_every": m,
                   "l2": "inputs (3 x %.0f MB) larger than L2; no flush" % (ext ** 3 * 8 / 1e6),
                   "parallelism": "single GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": kname,
                     "kernel_us": kernel_s * 1e6, "kernel_us_short_runs": short_s * 1e6,
                     "peak_source": peak_kind,
                     "algorithmic_bytes_per_launch": BYTES_PER_SITE * n ** 3,
                     "site_updates_per_launch": (2 if two_step else 1) * n ** 3,
                     # launches of this kernel in the timed region x its mean duration, over
                     # the region's time (the committed ncu launch list gives its share too)
                     "share_of_timed_region": share},
        "clocks": clocks,
        "e2e": {"value": e2e, "unit": "GLUPS", "h2d_bytes_per_step": h2d / args.steps,
                "d2h_bytes_per_step": d2h / args.steps,
                "api": "paper_0904_0939_b200.evolve_fixed(Field3D, PotentialGrid) from pinned "
                       "host memory, psi0+V uploaded and psi downloaded inside the timed region",
                "calls_s": [round(t, 4) for t in e2e_times],
                "statistic": f"median of 5 calls after {E2E_WARMUP} untimed warm-up calls"},
        "gpu_launches": launches,
        "cpu_baseline": cpu,
        "observables": {"E_last": float(np.sum(sums[-1][0]) / np.sum(sums[-1][1]))
                        if len(sums) else None},
    }
    print(json.dumps(line), flush=True)


def run_large(args):
    """One GPU, lattices whose host arrays do not fit the bench's pinned
    buffers (C5: 2048^3, 69 GB per field).  Start field and potential are
    generated on the device (bitwise the host recipes, workloads.fill_slab) and
    the slab is single-buffer (psi 77.9 GB + V 69.1 GB at 2048^3; two psi
    buffers would need 207 GB).  Same timed region and roofline method as
    run_single; no e2e leg (the inputs never exist on the host)."""
    import torch

    from paper_0904_0939_b200 import workloads
    from paper_0904_0939_b200.device import Slab

    w = workload(args.config)
    if args.size:
        w = workloads.scaled(w, args.size)
    spec = w.spec
    n = spec.N
    dev = 0
    torch.cuda.set_device(dev)
    slab = Slab(spec, device=dev, single_buffer=True, chunk=args.chunk)
    t0 = time.perf_counter()
    workloads.fill_slab(slab, w)
    slab.sync()
    fill_s = time.perf_counter() - t0
    st = torch.cuda.ExternalStream(slab.stream)
    m = w.measure_every
    slab.run(args.warmup, measure_every=m, norm_every=m)
    slab.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = slab.launches()
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        e0.record(st)
        idx, sums, status = slab.run(args.steps, measure_every=m, norm_every=m,
                                     step_offset=args.warmup)
        e1.record(st)
        e1.synchronize()
        torch.cuda.synchronize()
    launches = slab.launches() - l0
    ms = e0.elapsed_time(e1)
    clocks = clk.summary()
    if status.any():
        raise SystemExit(f"device status {status} during the timed run")
    value = n ** 3 * args.steps / (ms * 1e-3) / 1e9
    # dominant kernel: plain pairs (one two-sweep pass over the lattice = its
    # chunk launches), timed back to back as in the timed region
    npass, nsingle = t2_schedule(args.steps, args.warmup, m)
    l_probe = slab.launches()
    slab.run(2, 0, 0)
    slab.sync()
    per_pass = slab.launches() - l_probe
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(4, min(npass, 40))
    ea.record(st)
    slab.run(2 * reps, 0, 0)
    eb.record(st)
    eb.synchronize()
    pass_s = ea.elapsed_time(eb) * 1e-3 / reps
    fbytes = slab.field_bytes
    slab.close()
    peak, peak_kind = hbm_peak()
    achieved = BYTES_PER_SITE * n ** 3 / pass_s / 1e9
    line = {
        "metric": "fp64 FDTD lattice-site updates/s (GLUPS)",
        "value": value, "unit": "GLUPS", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "N": n, "a": spec.a, "dtau": spec.dtau,
                   "potential": w.potential, "measure_every": m, "norm_every": m,
                   "l2": "fields (%.1f GB) larger than L2; no flush" % (fbytes / 1e9),
                   "parallelism": "single GPU, single-buffer slab",
                   "inputs": "device-generated (workloads.fill_slab), %.1f s" % fill_s,
                   "field_bytes": fbytes},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": "k_sweep2b (two fp64 7-point sweeps per HBM pass), "
                               f"{per_pass} chunk launches per pass",
                     "pass_us": pass_s * 1e6, "peak_source": peak_kind,
                     "algorithmic_bytes_per_pass": BYTES_PER_SITE * n ** 3,
                     "site_updates_per_pass": 2 * n ** 3,
                     "share_of_timed_region": npass * pass_s / (ms * 1e-3)},
        "clocks": clocks,
        "e2e": None,
        "e2e_note": "inputs generated in HBM (no host arrays at this size): no end-to-end number",
        "gpu_launches": launches,
        "cpu_baseline": None,
        "observables": {"E": [float(np.sum(sm[0]) / np.sum(sm[1])) for sm in sums]},
    }
    print(json.dumps(line), flush=True)


def t2_schedule(steps: int, offset: int, m: int):
    """(two-sweep passes, single sweeps) psg_run issues for a fixed run with
    measure / norm every m (the pairing rule of run_loop in csrc/psigpu.cu:
    runs of plain steps go in pairs; a step carrying a pending factor is single)."""
    def plain(t):
        sidx = offset + t
        meas = m > 0 and sidx - 1 > 0 and (sidx - 1) % m == 0
        norm = m > 0 and sidx % m == 0
        return not meas and not norm

    t, pending, passes, singles = 1, False, 0, 0
    while t <= steps:
        if not pending and plain(t):
            run = 1
            while t + run <= steps and plain(t + run):
                run += 1
            if run >= 2:
                passes += run // 2
                t += 2 * (run // 2)
                continue
        pending = m > 0 and (offset + t) % m == 0
        singles += 1
        t += 1
    return passes, singles


def weak_n(n1: int, m: int) -> int:
    """Lattice size with ~n1^3 sites per GPU on m GPUs: the multiple of
    lcm(64, m) nearest n1 * m^(1/3) (64-column tiles stay full; m equal slabs)."""
    if m == 1:
        return n1
    step = 64 * m // math.gcd(64, m)
    return max(step, int(round(n1 * m ** (1.0 / 3.0) / step)) * step)


def strong_scaling(args) -> bool:
    return args.config == "C5" or args.strong


def run_dist(args):
    import torch
    import torch.distributed as dist

    from paper_0904_0939_b200 import Field3D, PotentialGrid, evolve_parallel, workloads
    from paper_0904_0939_b200.device import Slab
    from paper_0904_0939_b200.parallel import (SlabEngine, _DistGroup, get_comm, partition,
                                               release_comms)

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    # one GPU per rank (the modulo only matters for protocol runs that share a GPU)
    local = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if args.transport == "auto":
        ndev = torch.cuda.device_count()
        peers = all(torch.cuda.can_device_access_peer(i, j)
                    for i in range(ndev) for j in range(ndev) if i != j)
        args.transport = "ipc" if (world > 1 and world <= ndev and peers) else "nccl"
    ipc = args.transport == "ipc"
    # the IPC transport needs torch.distributed only for the handshake and the
    # e2e leg's scatter / gather: NCCL when every rank has its own GPU, gloo
    # when ranks share one (protocol runs on a one-GPU box)
    shared = world > torch.cuda.device_count()
    if ipc and shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    coll_dev = "cpu" if (ipc and shared) else "cuda"
    base = workload(args.config)
    if args.size:
        base = workloads.scaled(base, args.size)
    # weak scaling: the same recipe (box side fixed) on N_lat ~ N_1 * M^(1/3),
    # a multiple of M, so every GPU holds ~N_1^3 sites (M=1: the config itself).
    # Strong scaling (C5, the north star's 2048^3 sharded run): the lattice
    # itself split into M slabs; inputs only ever exist in HBM (no e2e leg)
    strong = strong_scaling(args)
    n_lat = base.N if strong else weak_n(base.N, world)
    w = base if n_lat == base.N else workloads.scaled(base, n_lat)
    spec = w.spec
    n = spec.N
    part = partition(spec, world)
    lo, hi = part.x_range(rank)
    slab = Slab(spec, w=part.W, x_lo=lo, device=local, single_buffer=False, ipc=ipc)
    # start field and potential generated on the device (bitwise the host
    # recipes: Philox plane stream, Coulomb floor)
    workloads.fill_slab(slab, w)

    class _G:  # the grid object the engine needs (v only used on the host for checks)
        pass

    grid = _G()
    grid.spec = spec
    grid.unbounded = w.potential in ("cornell", "wells")
    grid.v_inf = 0.0
    if ipc:   # NCCL-free: halos stored by the sweep kernel through CUDA IPC mappings
        from paper_0904_0939_b200.device import IpcLink

        comm = IpcLink.from_process_group(slab)
    else:
        comm = get_comm(local)   # cached: the e2e calls below reuse it
    engine = SlabEngine(grid, part, [slab], [rank], _DistGroup(slab, rank, part, comm))
    m = w.measure_every
    kw = dict(tol=1e-300, check_freq=m, snap_freq=10 ** 12, reimpose_freq=10 ** 12,
              max_snapshots=0, constraints=(), norm_every=m, fixed=True, measure_every=m,
              gather=False)
    engine.run(max_steps=args.warmup, **kw)
    st = torch.cuda.ExternalStream(slab.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = slab.launches()
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(st)
        engine.run(max_steps=args.steps, **kw)
        e1.record(st)
        e1.synchronize()
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=coll_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    launches = torch.tensor([float(slab.launches() - l0)], dtype=torch.float64, device=coll_dev)
    dist.all_reduce(launches)
    ms = float(ms.item())
    value = n ** 3 * args.steps / (ms * 1e-3) / 1e9
    peak, peak_kind = hbm_peak()
    if ipc:
        dist.barrier()
        comm.close()
    slab.close()
    if strong:
        if rank == 0:
            print(json.dumps({
                "metric": "fp64 FDTD lattice-site updates/s (GLUPS)", "value": value,
                "unit": "GLUPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": w.name, "N": n, "measure_every": m, "norm_every": m,
                           "parallelism": f"z-slabs x{world} of {part.W} planes ("
                                          + ("IPC: halos stored by the sweep kernel"
                                             if ipc else "NCCL halos overlapped")
                                          + ", exact all-reduce of plane sums)",
                           "inputs": "device-generated per slab (workloads.fill_slab)",
                           "l2": "inputs larger than L2; no flush"},
                "roofline": {"bound": "hbm", "achieved": 12 * n ** 3 * args.steps /
                             (ms * 1e-3) / 1e9 / world, "peak": peak, "unit": "GB/s",
                             "frac": 12 * n ** 3 * args.steps / (ms * 1e-3) / 1e9 / world / peak,
                             "traffic": None, "per": "GPU, whole timed run, 12 B per site-update",
                             "peak_source": peak_kind},
                "clocks": clk.summary(), "e2e": None,
                "e2e_note": "inputs generated in HBM (no host arrays at this size)",
                "gpu_launches": int(launches.item()), "cpu_baseline": None}), flush=True)
        release_comms()
        dist.destroy_process_group()
        return

    # ---- e2e: the public multi-GPU API from host arrays (rank 0 holds psi0) ----
    ext = n + 2
    # the grid's V array is lattice-sized, but a rank only reads its own planes
    # (load_grid): fill those (untouched zero pages cost no host memory)
    vfull = np.zeros((ext, ext, ext))
    vfull[lo - 1:lo + part.W + 1] = workloads.potential_planes(w, spec, lo - 1, part.W + 2)
    pgrid = PotentialGrid(spec=spec, v=vfull, v_inf=0.0, unbounded=False, name="custom")
    init = None
    if rank == 0:
        psi0 = np.zeros((ext, ext, ext))
        psi0[1:-1] = workloads.uniform_start(spec)
        init = Field3D(spec, psi0)
    e2e_times = []
    for i in range(E2E_WARMUP + 3):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st_e = evolve_parallel(pgrid, workers=world, initial=init, transport=args.transport,
                               scatter_initial=True, check_freq=m, max_steps=args.steps,
                               max_snapshots=0, norm_every=m, fixed=True)
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        if i >= E2E_WARMUP:
            e2e_times.append(float(dt.item()))
    t_e2e = statistics.median(e2e_times)
    if rank == 0:
        line = {
            "metric": "fp64 FDTD lattice-site updates/s (GLUPS)", "value": value,
            "unit": "GLUPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "N": n, "measure_every": m, "norm_every": m,
                       "weak": f"{base.name} recipe (box side {base.N * base.a:g}) on N = the "
                               f"multiple of lcm(64, M) nearest {base.N}*M^(1/3): "
                               f"{n ** 3 / world / 1e6:.2f} M sites per GPU",
                       "transport": args.transport,
                       "parallelism": f"z-slabs x{world} (" + (
                           "IPC: two halo planes per face stored by each two-sweep pass into "
                           "the neighbours' buffers" if ipc else
                           "NCCL: two halo planes per face every other sweep, overlapped")
                       + "; exact all-reduce of plane sums)",
                       "l2": "inputs larger than L2; no flush"},
            # whole timed run per GPU: a two-sweep pass moves 24 B per site for two
            # updates (12 B per site-update); the few single sweeps around the
            # norm / measure steps move 24
            "roofline": {"bound": "hbm", "achieved": 12 * n ** 3 * args.steps /
                         (ms * 1e-3) / 1e9 / world, "peak": peak, "unit": "GB/s",
                         "frac": 12 * n ** 3 * args.steps / (ms * 1e-3) / 1e9 / world / peak,
                         "traffic": None, "per": "GPU, whole timed run, 12 B per site-update",
                         "peak_source": peak_kind},
            "clocks": clk.summary(),
            "e2e": {"value": n ** 3 * args.steps / t_e2e / 1e9, "unit": "GLUPS",
                    "h2d_bytes_per_step": 2 * ext ** 3 * 8 / args.steps,
                    "d2h_bytes_per_step": (ext ** 3 * 8 + len(st_e.checks) * (3 * n + 2) * 8)
                    / args.steps,
                    "api": f"paper_0904_0939_b200.evolve_parallel(transport='{args.transport}', "
                           "scatter_initial=True, fixed=True) from host arrays on rank 0 (psi0) "
                           "and every rank (V); psi gathered to rank 0 inside the timed region",
                    "calls_s": [round(t, 4) for t in e2e_times],
                    "statistic": f"median of 3 calls after {E2E_WARMUP} untimed warm-up "
                                 "calls, max over ranks"},
            "gpu_launches": int(launches.item()),
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    release_comms()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--single-buffer", action="store_true",
                    help="one GPU, single-buffer slab, device-generated inputs (default for C5)")
    ap.add_argument("--size", type=int, default=0, help="rescale the config's lattice (with --single-buffer)")
    ap.add_argument("--chunk", type=int, default=0, help="planes per chunk launch of a single-buffer slab")
    ap.add_argument("--transport", choices=["auto", "nccl", "ipc"], default="auto",
                    help="multi-GPU slab transport: NCCL (device-triggered exchange) or the "
                         "NCCL-free IPC transport (halos stored by the sweep kernel); auto = "
                         "IPC when every pair of local GPUs has peer access, else NCCL")
    ap.add_argument("--strong", action="store_true",
                    help="multi-GPU: split the config's lattice itself (default for C5)")
    ap.add_argument("--dist", action="store_true",
                    help="use the torch.distributed slab engine even for one rank (testing)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if (args.single_buffer or args.config == "C5") and world == 1 and not args.dist:
        return run_large(args)
    if world > 1 or args.dist:
        return run_dist(args)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main() or 0)
