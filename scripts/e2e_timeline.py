"""Timeline of bench.py's pipelined e2e leg (cfg5): CUDA events on the upload, compute and
download streams per step, printed as start/end ms relative to the first upload."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2005_03246_b200 import _lib  # noqa: E402

_lib.load_library()
wl = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
mode = sys.argv[3] if len(sys.argv) > 3 else "full"  # full | noup | nodown
w = bench.make_workload(wl)
w.shard(0, 1)
w.to_device()
w.step()
torch.cuda.synchronize()
w.to_pinned()
evs = []
main = torch.cuda.current_stream()


def ev(tag, stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    evs.append((tag, e, time.perf_counter()))


orig_upload = w._upload


def upload(j):
    b = j % 2
    if w.ev_free[b] is not None:
        w.up_stream.wait_event(w.ev_free[b])
    ev(f"up{j}.start", w.up_stream)
    if mode == "noup":
        w.ev_up[b] = w.up_stream.record_event()
    else:
        orig_upload(j)
    ev(f"up{j}.end", w.up_stream)


w._upload = upload
if mode == "nodown":
    class _Null:
        def copy_(self, *a, **k):
            return self

        def __getitem__(self, k):
            return self
    w.out_pinned = _Null()
    if getattr(w, "out2_pinned", None) is not None:
        w.out2_pinned = _Null()
orig_ecdf, orig_kde = w._ecdf, w._kde


def ecdf(s):
    ev("ecdf.start", main)
    r = orig_ecdf(s)
    ev("ecdf.end", main)
    return r


def kde(s):
    ev("kde.start", main)
    r = orig_kde(s)
    ev("kde.end", main)
    return r


w._ecdf, w._kde = ecdf, kde
if mode == "noup":
    for b in range(2):
        w.xd[b].copy_(w.p_x)
        if getattr(w, "yd", None) is not None:
            w.yd[b].copy_(w.p_yv)
    torch.cuda.synchronize()
_lib.profile_enable(True)
_lib.profile_report()
w.e2e_begin()
ev("begin", main)
for i in range(steps):
    ev(f"step{i}.host", main)
    w.step_e2e(last=i == steps - 1)
    ev(f"comp{i}.end", main)
    ev(f"down{i}.end", w.down_stream)
w.e2e_end()
ev("end", main)
torch.cuda.synchronize()
prof = _lib.profile_report()
_lib.profile_enable(False)
for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:24s} {c:4d} launches {ms:9.3f} ms")
t0 = evs[0][1]
h0 = evs[0][2]
for tag, e, h in evs:
    print(f"{tag:14s} gpu {t0.elapsed_time(e):9.2f} ms   host {1e3 * (h - h0):9.2f} ms")
