"""Throughput of the drop-in path's staged copies (fcg_copy_h2d / fcg_copy_d2h) against a
pinned-buffer cudaMemcpy and torch's pageable copies."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2005_03246_b200 import _lib

n = 400_000_000  # 3.2 GB of fp64
a = np.random.default_rng(0).random(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in [
    ("staged h2d", lambda: _lib.to_device_f64(a)),
    ("torch pageable h2d", lambda: torch.from_numpy(a).to("cuda")),
]:
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{name}: {a.nbytes / dt / 1e9:.1f} GB/s")
p = torch.from_numpy(a).pin_memory()
t0 = time.perf_counter(); d.copy_(p, non_blocking=True); torch.cuda.synchronize()
print(f"pinned h2d: {a.nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
for name, fn in [("staged d2h", lambda: _lib.to_host(d)), ("torch pageable d2h", lambda: d.cpu().numpy())]:
    fn()
    t0 = time.perf_counter(); fn(); dt = time.perf_counter() - t0
    print(f"{name}: {a.nbytes / dt / 1e9:.1f} GB/s")
t0 = time.perf_counter(); p.copy_(d, non_blocking=True); torch.cuda.synchronize()
print(f"pinned d2h: {a.nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
import os
print("host cpus", os.cpu_count())
