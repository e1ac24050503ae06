"""Where the ~33 us of host time per launch-bound call goes (config 1 shape)."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2005_03246_b200 as fcb
import workloads as wl
from paper_2005_03246_b200 import _lib
from paper_2005_03246_b200.fastsum import _ecdf_grid_device

w = wl.cfg1()
x = torch.from_numpy(w.points).cuda()
s = fcb.Sample(x, torch.ones(1, device="cuda"), None, True)
g = fcb.RectilinearGrid.from_knots(w.knots)
dv = fcb.DeltaVector(w.delta)
kn = _lib.device_knots(g)
out = torch.empty(g.size, dtype=torch.float64, device="cuda")
lib = _lib.load_library()


def bench(name, fn, k=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:40s} {1e6 * (t1 - t0) / k:7.2f} us/call")


bench("ecdf_fastsum (public API)", lambda: fcb.ecdf_fastsum(s, g, dv))
bench("_ecdf_grid_device", lambda: _ecdf_grid_device(s, g, dv, False, True))
args = (_lib.ptr(x), x.shape[0], 2, _lib.ptr(None), _lib.ptr(kn), _lib.i64_array(g.shape),
        _lib.i32_array(dv.signs), 0, 1, 0, _lib.ptr(out))
bench("call_ws(prepared args)", lambda: _lib.call_ws("fcg_ecdf_grid", *args))
nb = C.c_size_t(0)
sh = C.c_void_p(torch.cuda.current_stream().cuda_stream)
bench("size query only", lambda: lib.fcg_ecdf_grid(*args, None, C.byref(nb), sh))
ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
wsp = C.c_void_p(ws.data_ptr())
bench("run call only (ctypes + launch)", lambda: lib.fcg_ecdf_grid(*args, wsp, C.byref(nb), sh))
bench("torch.empty(65536 f64)", lambda: torch.empty(65536, dtype=torch.float64, device="cuda"))
bench("current_stream()", lambda: torch.cuda.current_stream())
bench("to_device_f64(x)", lambda: _lib.to_device_f64(x))
bench("i64_array + i32_array", lambda: (_lib.i64_array(g.shape), _lib.i32_array(dv.signs)))
