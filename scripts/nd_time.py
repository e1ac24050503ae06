"""Timing of the d >= 3 at-points route (ecdf_dnc / kde_dnc on device-resident samples)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2005_03246_b200 as fcb
from paper_2005_03246_b200 import _lib

def timeit(f, reps=3):
    f(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

cases = [(3, 100_000), (3, 1_000_000), (3, 10_000_000), (4, 1_000_000), (5, 300_000)]
if len(sys.argv) > 1:
    cases = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]]
for d, n in cases:
    g = torch.Generator(device="cuda").manual_seed(d * 7 + 1)
    x = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g)
    w = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5
    dist = (True,) * d  # skip the distinct-coordinates pass (continuous data)
    s = fcb.Sample(x, w, distinct_by_dim=dist, unit_weights=False)
    su = fcb.Sample(x, torch.ones_like(w), distinct_by_dim=dist, unit_weights=True)
    bw = fcb.Bandwidth.diag([0.3] * d)
    t_u = timeit(lambda: fcb.ecdf_dnc(su, scaled=False))
    t_w = timeit(lambda: fcb.ecdf_dnc(s, scaled=False))
    t_k = timeit(lambda: fcb.kde_dnc(s, fcb.laplacian(), bw))
    print(f"d={d} n={n}: ecdf_dnc unit {t_u:.2f} ms, weighted {t_w:.2f} ms, kde_dnc {t_k:.2f} ms", flush=True)
    _lib.profile_enable(True)
    fcb.ecdf_dnc(su, scaled=False); fcb.kde_dnc(s, fcb.laplacian(), bw); torch.cuda.synchronize()
    rep = _lib.profile_report(); _lib.profile_enable(False)
    print("   ", {k: (v[0], round(v[1], 3)) for k, v in rep.items() if v[1] > 0.05}, flush=True)
    t_m = timeit(lambda: fcb.kde_dnc(s, fcb.matern32_additive(), bw)) if d <= 4 else float("nan")
    print(f"    matern32-additive kde_dnc {t_m:.2f} ms", flush=True)
