"""Run the slab engine's torch.distributed path on real GPUs (launch with torchrun).

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port 29511 scripts/dist_smoke.py

Each rank owns one slab on its GPU; the result on rank 0 must equal the
single-slab run bitwise (checked on rank 0).  With N=1 this exercises the
NCCL all-reduce of device plane-sum views, the stream ordering of NCCL with
the slab stream and the gather path.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from paper_0904_0939_b200 import (LatticeSpec, SymmetryConstraint, allocate, evolve_fixed,
                                  evolve_parallel, evolve_to_convergence, fill_random_gaussian,
                                  harmonic, impose_inplace)


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = LatticeSpec(N=24, a=0.4, m=1.0, dtau=0.04)
    grid = harmonic(spec)
    init = fill_random_gaussian(allocate(spec), 11)
    cs = [SymmetryConstraint("x", "antisymmetric"), SymmetryConstraint("y", "symmetric")]
    for c in cs:
        impose_inplace(init.values, spec.N, c)
    ok = True
    for native in (True, False):
        st = evolve_parallel(grid, workers=world, initial=init, transport="nccl", tol=1e-300,
                             check_freq=20, max_steps=100, max_snapshots=0, constraints=cs,
                             native=native)
        if rank == 0:
            ref = evolve_to_convergence(init, grid, tol=1e-300, check_freq=20, max_steps=100,
                                        max_snapshots=0, constraints=cs, exact=True)
            same = np.array_equal(st.psi.values, ref.psi.values)
            e_same = [c.energy for c in st.checks] == [c.energy for c in ref.checks]
            print(f"dist_smoke world={world} native={native}: psi bitwise {same}, energies "
                  f"bitwise {e_same}, halo messages {st.halo_messages}, "
                  f"sweeps {st.sweeps_started} vs {ref.sweeps_started}", flush=True)
            ok = ok and same and e_same
        else:
            assert st is None
    # converging run: stop at the same check, same state
    st = evolve_parallel(grid, workers=world, initial=init, transport="nccl", tol=1e-5,
                         check_freq=10, max_steps=4000, max_snapshots=0, constraints=cs)
    if rank == 0:
        ref = evolve_to_convergence(init, grid, tol=1e-5, check_freq=10, max_steps=4000,
                                    max_snapshots=0, constraints=cs, exact=True)
        same = (np.array_equal(st.psi.values, ref.psi.values) and st.step_count == ref.step_count
                and st.converged == ref.converged)
        print(f"dist_smoke converging: bitwise {same}, steps {st.step_count} vs "
              f"{ref.step_count}, converged {st.converged}", flush=True)
        ok = ok and same
    # fixed-step recipe (fused observables, renormalisation every 20)
    st = evolve_parallel(grid, workers=world, initial=init, transport="nccl", check_freq=20,
                         max_steps=100, max_snapshots=0, norm_every=20, fixed=True)
    if rank == 0:
        ref = evolve_fixed(init, grid, 100, 20, norm_every=20, exact=True)
        same = np.array_equal(st.psi.values, ref.psi.values)
        e_same = [c.energy for c in st.checks] == [c.energy for c in ref.checks]
        print(f"dist_smoke fixed: psi bitwise {same}, energies bitwise {e_same}", flush=True)
        ok = ok and same and e_same
    # scatter from rank 0 / gather to rank 0 through device buffers
    st = evolve_parallel(grid, workers=world, initial=init if rank == 0 else None,
                         transport="nccl", scatter_initial=True, check_freq=20, max_steps=60,
                         max_snapshots=0, norm_every=20, fixed=True)
    if rank == 0:
        ref = evolve_fixed(init, grid, 60, 20, norm_every=20, exact=True)
        same = np.array_equal(st.psi.values, ref.psi.values)
        print(f"dist_smoke scatter/gather: psi bitwise {same}", flush=True)
        ok = ok and same
    from paper_0904_0939_b200.parallel import release_comms

    release_comms()
    if rank == 0 and not ok:
        sys.exit(1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
