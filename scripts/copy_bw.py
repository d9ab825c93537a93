"""HBM copy bandwidth of this box (same method as MEASURED_PEAKS.json) + our sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch


def copy_bw(n_elems=1 << 30, dtype=torch.bfloat16, reps=10):
    a = torch.empty(n_elems, dtype=dtype, device="cuda").uniform_()
    b = torch.empty_like(a)
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return 2 * a.numel() * a.element_size() / best / 1e9


def read2_write1(n=1 << 27, reps=10):
    """2 reads + 1 write fp64 stream (the sweep's mix): c = a + b."""
    a = torch.empty(n, dtype=torch.float64, device="cuda").uniform_()
    b = torch.empty_like(a).uniform_()
    c = torch.empty_like(a)
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.add(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return 3 * n * 8 / best / 1e9


if __name__ == "__main__":
    torch.cuda.init()
    print(f"copy bf16 1Gi: {copy_bw():.1f} GB/s   a+b fp64 (2R+1W): {read2_write1():.1f} GB/s", flush=True)
