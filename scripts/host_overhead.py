"""Host-side cost of one public-API call (device-resident inputs): wall time per call over a
burst without syncs vs device time, for the launch-bound configurations."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2005_03246_b200 as fcb
import workloads as wl

w = wl.cfg1()
x = torch.from_numpy(w.points).cuda()
s = fcb.Sample(x, torch.ones(1, device="cuda"), None, True)
g = fcb.RectilinearGrid.from_knots(w.knots)
dv = fcb.DeltaVector(w.delta)
for _ in range(20):
    fcb.ecdf_fastsum(s, g, dv)
torch.cuda.synchronize()
K = 500
t0 = time.perf_counter()
for _ in range(K):
    fcb.ecdf_fastsum(s, g, dv)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"cfg1 ecdf_fastsum: host {1e6 * (t1 - t0) / K:.1f} us/call, end-to-end {1e6 * (t2 - t0) / K:.1f} us/call")
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    fcb.ecdf_fastsum(s, g, dv)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
