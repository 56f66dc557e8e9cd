"""Copies-only replica of mf_apply_host's pipeline (C chunks, H2D stream -> event -> D2H
stream) for a 16.97 M-DoF vector: the e2e ceiling without the apply."""
import time

import torch

n = 16974593
h_src = torch.empty(n, dtype=torch.float64).pin_memory()
h_dst = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def call(C):
    evs = []
    for r in range(C):
        a, b = n * r // C, n * (r + 1) // C
        with torch.cuda.stream(s1):
            d_a[a:b].copy_(h_src[a:b], non_blocking=True)
            e = torch.cuda.Event()
            e.record(s1)
        s2.wait_event(e)
        with torch.cuda.stream(s2):
            h_dst[a:b].copy_(d_a[a:b], non_blocking=True)
    s2.synchronize()


for C in (1, 2, 4, 8, 16):
    call(C)
    t0 = time.perf_counter()
    for _ in range(20):
        call(C)
    dt = (time.perf_counter() - t0) / 20
    print(C, f"{n / dt / 1e9:.2f} GDoF/s equivalent ({dt * 1e3:.2f} ms)")
