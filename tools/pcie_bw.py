"""Pinned host<->device copy bandwidth on this box (context for the e2e number): H2D alone,
D2H alone, and both directions at once on two streams, 512 MiB each, CUDA events."""
import json

import torch

N = 512 << 20
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_a = torch.empty(N, dtype=torch.uint8, device="cuda")
d_b = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def both():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t_h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
t_both = timed(both)
print(json.dumps({"h2d_GBps": round(N / t_h2d / 1e6, 1), "d2h_GBps": round(N / t_d2h / 1e6, 1),
                  "bidir_GBps_per_direction": round(N / t_both / 1e6, 1)}))
