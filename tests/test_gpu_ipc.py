"""The NCCL-free IPC slab transport across processes (scripts/ipc_check.py
under torchrun; the ranks share this box's GPU, which only exercises the
protocol: peer stores, pulled halos, mailbox all-reduce and counter waits in
the same order as across GPUs).  Every rank's planes, check sums and final
measurement must equal the whole-lattice run bitwise."""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("ranks,n,steps,every", [
    (2, 40, 61, 20),     # fused passes + measure / norm single sweeps
    (2, 130, 45, 0),     # norm every step: single sweeps only (pulled halos)
    (3, 96, 50, 10),
    (4, 128, 33, 16),
])
def test_ipc_transport_bitwise(gpu_lib, ranks, n, steps, every):
    port = 29600 + 10 * ranks + n % 10
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={ranks}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "scripts", "ipc_check.py"), "--lattice", str(n), "--steps",
           str(steps), "--every", str(every)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=ROOT)
    # the ranks' lines may interleave on the shared stdout
    ok = re.findall(r"IPC_OK rank=(\d+) fused=(\d+)", r.stdout)
    assert r.returncode == 0 and sorted(int(a) for a, _ in ok) == list(range(ranks)), \
        r.stdout[-2000:] + r.stderr[-3000:]
    if every:   # plain pairs ran as fused two-sweep passes
        assert all(int(f) > 0 for _, f in ok)


@pytest.mark.parametrize("ranks,n,steps,every", [(2, 40, 60, 10), (4, 64, 41, 10)])
def test_ipc_evolve_parallel_api(gpu_lib, ranks, n, steps, every):
    """evolve_parallel(transport="ipc"): scatter from rank 0, converging run
    with checks and snapshots, fixed run; equal to the one-slab engine."""
    port = 29700 + 10 * ranks + n % 10
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={ranks}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "scripts", "ipc_check.py"), "--lattice", str(n), "--steps",
           str(steps), "--every", str(every), "--api"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    ok = re.findall(r"IPC_OK rank=(\d+)", r.stdout)
    assert r.returncode == 0 and sorted(int(x) for x in ok) == list(range(ranks)), \
        r.stdout[-2000:] + r.stderr[-3000:]
