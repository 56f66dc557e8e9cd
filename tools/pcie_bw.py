"""Host<->device copy bandwidth with pinned buffers: H2D alone, D2H alone, both at once
(separate streams), for the e2e ceiling of mf_apply_host."""
import torch

n = 136 * 1024 * 1024 // 8 * 2
h_src = torch.empty(n, dtype=torch.float64).pin_memory()
h_dst = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
bytes_ = n * 8


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    t = timed(fn)
    print(name, f"{bytes_ / t / 1e9:.1f} GB/s per direction ({bytes_ / 1e6:.0f} MB, {t * 1e3:.2f} ms)")
