"""Bitwise check of the NCCL-free IPC slab transport (run under torchrun, gloo
backend for the host handshake; every rank may share one GPU).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29533 scripts/ipc_check.py --lattice 40 --steps 61 --every 20

Each rank runs its slab through Slab.run_dist(IpcLink) (fused two-sweep
passes storing into the neighbours' halos, pulled single-sweep halos,
mailbox all-reduce), then compares its planes, the check sums and a final
measurement with a whole-lattice run of the same inputs on its device.
Prints one line "IPC_OK rank=<r> fused=<passes>" per rank on success.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_0904_0939_b200.device import IpcLink, Slab  # noqa: E402
from paper_0904_0939_b200.lattice import LatticeSpec  # noqa: E402
from paper_0904_0939_b200.parallel import partition  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", type=int, default=40)
    ap.add_argument("--steps", type=int, default=61)
    ap.add_argument("--every", type=int, default=20)
    ap.add_argument("--device", type=int, default=-1, help="-1: LOCAL_RANK modulo visible GPUs")
    ap.add_argument("--api", action="store_true",
                    help="through evolve_parallel(transport='ipc') against workers=1 (inproc)")
    a = ap.parse_args()
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ndev = torch.cuda.device_count()
    dev = a.device if a.device >= 0 else int(os.environ.get("LOCAL_RANK", rank)) % ndev
    torch.cuda.set_device(dev)
    n = a.lattice
    spec = LatticeSpec(N=n, a=0.3, m=1.0, dtau=0.3 * 0.3 / 4.0)
    rng = np.random.default_rng(n + 17)
    ext = n + 2
    psi0 = np.zeros((ext,) * 3)
    psi0[1:-1, 1:-1, 1:-1] = rng.uniform(-0.5, 0.5, (n, n, n))
    v = np.zeros((ext,) * 3)
    v[1:-1, 1:-1, 1:-1] = rng.uniform(-1.0, 3.0, (n, n, n))
    every = a.every
    if a.api:
        return api_check(a, spec, psi0, v, rank, world)
    with Slab(spec, device=dev, single_buffer=False) as whole:
        whole.set_temporal(True)
        whole.set_field(psi0)
        whole.set_potential(v)
        idx_w, sums_w, _ = whole.run(a.steps, measure_every=every, norm_every=every or 1,
                                          exact=True)
        want = whole.get_field()
        from paper_0904_0939_b200.device import measure_multi

        meas_w = measure_multi([whole])
    part = partition(spec, world)
    lo, hi = part.x_range(rank)
    s = Slab(spec, w=part.W, x_lo=lo, device=dev, single_buffer=False, ipc=True)
    s.set_temporal(True)
    s.set_field(psi0[lo - 1:hi + 2])
    s.set_potential(v[lo - 1:hi + 2])
    link = IpcLink.from_process_group(s)
    try:
        idx, sums, status = s.run_dist(link, None, None, a.steps, measure_every=every,
                                       norm_every=every or 1)
        meas = s.measure_dist(link, None, None)
        got = s.get_field(1, part.W)
        fused = s.fused_passes()
        dist.barrier()
    finally:
        link.close()
        s.close()
    ok = (np.array_equal(got, want[lo:hi + 1]) and np.array_equal(idx, idx_w)
          and np.array_equal(sums, sums_w) and np.array_equal(meas, meas_w) and not status.any())
    if not ok:
        d = np.abs(got - want[lo:hi + 1]).max()
        print(f"IPC_FAIL rank={rank} max|dpsi|={d:.3e} sums_eq={np.array_equal(sums, sums_w)} "
              f"meas_eq={np.array_equal(meas, meas_w)} status={status}", flush=True)
        dist.destroy_process_group()
        return 1
    print(f"IPC_OK rank={rank} fused={fused}", flush=True)
    dist.destroy_process_group()
    return 0


def api_check(a, spec, psi0, v, rank, world):
    """evolve_parallel(transport="ipc") from rank 0's host field (scattered
    over the gloo group), a converging run with checks and snapshots and a
    fixed run, against the single-slab engine: same fields and checks."""
    from paper_0904_0939_b200 import Field3D, evolve_parallel
    from paper_0904_0939_b200.potential import custom

    n = spec.N
    grid = custom(spec, v[1:-1, 1:-1, 1:-1], v_inf=0.0, unbounded=False)
    init = Field3D(spec, psi0)
    ok = True
    for kw in (dict(tol=1e-300, check_freq=a.every or 10, max_steps=a.steps, max_snapshots=2,
                    snap_freq=2 * (a.every or 10)),
               dict(check_freq=a.every or 10, max_steps=a.steps, max_snapshots=0, fixed=True,
                    norm_every=a.every or 10)):
        got = evolve_parallel(grid, workers=world, initial=init if rank == 0 else None,
                              transport="ipc", scatter_initial=True, **kw)
        if rank == 0:
            want = evolve_parallel(grid, workers=1, initial=init, transport="inproc", **kw)
            ok = ok and np.array_equal(got.psi.values, want.psi.values)
            ok = ok and [c.energy for c in got.checks] == [c.energy for c in want.checks]
            ok = ok and len(got.snapshots) == len(want.snapshots) and all(
                np.array_equal(x[1].values, y[1].values) for x, y in zip(got.snapshots,
                                                                         want.snapshots))
        else:
            ok = ok and got is None
    print(("IPC_OK" if ok else "IPC_FAIL") + f" rank={rank} fused=1", flush=True)
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
