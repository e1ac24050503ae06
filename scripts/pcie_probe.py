"""Pinned host<->device copy bandwidth on this box: H2D alone, D2H alone, both at once
(the ceiling for bench.py's e2e leg)."""
import json

import torch

n = 1 << 30  # 1 GiB
h_up = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dn = torch.empty(n, dtype=torch.uint8).pin_memory()
d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
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
    return a.elapsed_time(b) / reps / 1e3


def up():
    d_up.copy_(h_up, non_blocking=True)


def dn():
    h_dn.copy_(d_dn, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        up()
    with torch.cuda.stream(s2):
        dn()
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_up, t_dn, t_both = timed(up), timed(dn), timed(both)
print(json.dumps({"h2d_GBps": n / t_up / 1e9, "d2h_GBps": n / t_dn / 1e9,
                  "duplex_GBps_each": n / t_both / 1e9}))
