"""PCIe link on this box: 268 MB pinned H2D alone, D2H alone, and both at
once on two streams (CUDA events).  The bound of the e2e (host-buffer) path."""
import torch

n = 1 << 25
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        h2d()
    with torch.cuda.stream(s2):
        d2h()
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for name, fn in (("H2D", h2d), ("D2H", d2h), ("both", both)):
    ms = timed(fn)
    print(f"{name:5s} {ms:.2f} ms  ({n * 8 / ms / 1e6:.1f} GB/s per direction)")
