"""Generate golden fixtures by running the REFERENCE package itself (build container only).

    NUMBA_CACHE_DIR=/tmp/numba_golden PYTHONPATH=/root/reference/pkg/src \
        python -B tests/golden/make_golden.py [--small] [--nd] [--csv] [--configs cfg1,cfg2,...]

Writes small .npz fixtures next to this file; they are committed and travel to the GPU box
(the reference itself does not).  Inputs are stored with the outputs wherever they are small,
so tests never depend on re-generating random streams.  For the full-size configurations only
SHA-256 digests (of inputs and of the reference's outputs) and seeded subsets are stored.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

import fastcdf as fc  # noqa: E402  (the reference, via PYTHONPATH)
from fastcdf.histogram import flat_bin_indices  # noqa: E402

import workloads as wl  # noqa: E402

assert "reference" in fc.__file__, fc.__file__

THREE = [[0.2, 0.7], [0.5, 0.1], [0.9, 0.9]]


class Bag:
    def __init__(self):
        self.d = {}

    def put(self, key, value):
        assert key not in self.d, key
        self.d[key] = np.asarray(value)

    def put_knots(self, key, knots):
        self.put(key + ".knots", np.concatenate([np.asarray(z, float) for z in knots]))
        self.put(key + ".m", np.array([len(z) for z in knots], dtype=np.int64))

    def save(self, name):
        np.savez_compressed(HERE / name, **self.d)
        print(f"wrote {name}: {len(self.d)} arrays", flush=True)


def small():
    b = Bag()
    # ---- hand KATs (test_histogram.py:18-50, test_fastsum.py:15-135, test_dnc.py) ----
    s3 = fc.validate_sample(THREE)
    g = fc.RectilinearGrid.from_knots([np.array([0.5]), np.array([0.5])])
    b.put("kat.ls_pp", fc.local_sums_sorted(s3, g, fc.DeltaVector((1, 1))).data)
    b.put("kat.ls_mp", fc.local_sums_sorted(s3, g, fc.DeltaVector((-1, 1))).data)
    g2 = fc.RectilinearGrid.from_knots([np.array([0.5, 0.9]), np.array([0.5, 0.9])])
    b.put("kat.ecdf", fc.ecdf_fastsum(s3, g2).values)
    b.put("kat.ecdf_mm", fc.ecdf_fastsum(s3, g2, fc.DeltaVector((-1, -1))).values)
    b.put("kat.esf04", fc.esf_fastsum(s3, fc.RectilinearGrid.from_knots([[0.4], [0.4]])).values)
    b.put("kat.dnc", fc.ecdf_dnc(s3).values)
    b.put("kat.dnc_self", fc.ecdf_dnc(s3, include_self=True).values)

    # ---- local sums with knot hits, random delta (test_histogram.py:80-97 pattern) ----
    for seed in range(40):
        rng = np.random.default_rng(seed)
        d = int(rng.integers(1, 6))
        n = int(rng.integers(1, 120))
        lat = np.linspace(-1.0, 1.0, 9)
        pts = np.where(rng.random((n, d)) < 0.5, rng.choice(lat, (n, d)),
                       rng.uniform(-1, 1, (n, d)))
        w = rng.integers(1, 4, n).astype(float)
        knots = [np.linspace(-1.0, 1.0, int(rng.integers(2, 6))) for _ in range(d)]
        if seed % 3 == 0:  # non-uniform grid -> sorted path
            knots = [np.sort(rng.uniform(-1, 1, len(z))) for z in knots]
            knots = [np.unique(z) for z in knots]
        delta = tuple(int(v) for v in rng.choice([-1, 1], d))
        s = fc.validate_sample(pts, w)
        grid = fc.RectilinearGrid.from_knots(knots)
        key = f"ls.{seed}"
        b.put(key + ".x", pts)
        b.put(key + ".w", w)
        b.put_knots(key, knots)
        b.put(key + ".delta", np.array(delta))
        b.put(key + ".out", fc.local_sums(s, grid, fc.DeltaVector(delta)).data)
        b.put(key + ".flat", flat_bin_indices(s, grid, fc.DeltaVector(delta)))

    # ---- grid ECDF bit-exact, integer and float weights (test_fastsum.py:88-101) ----
    for d in range(1, 6):
        for seed in range(6):
            rng = np.random.default_rng(1000 * d + seed)
            n = int(rng.integers(2, 400))
            wint = rng.integers(1, 5, n).astype(float)
            pts = rng.standard_normal((n, d))
            s = fc.validate_sample(pts, wint)
            counts = [int(c) for c in rng.integers(2, 5, d)]
            grid = fc.build_grid_auto(s, counts)
            delta = tuple(int(v) for v in rng.choice([-1, 1], d))
            key = f"ecdf.{d}.{seed}"
            b.put(key + ".x", pts)
            b.put(key + ".w", wint)
            b.put_knots(key, grid.knots)
            b.put(key + ".delta", np.array(delta))
            b.put(key + ".out", fc.ecdf_fastsum(s, grid, fc.DeltaVector(delta), scaled=False).values)
            b.put(key + ".unit", fc.ecdf_fastsum(fc.validate_sample(pts), grid,
                                                fc.DeltaVector(delta), scaled=True).values)
            wf = rng.uniform(0.5, 2.0, n)
            b.put(key + ".wf", wf)
            b.put(key + ".outf", fc.ecdf_fastsum(fc.validate_sample(pts, wf), grid,
                                                fc.DeltaVector(delta)).values)
            b.put(key + ".esf", fc.esf_fastsum(fc.validate_sample(pts, wf), grid).values)

    # ---- directional sweep, every code (test_fastsum.py:15-49) ----
    for d in range(1, 5):
        rng = np.random.default_rng(70 + d)
        dims = tuple(int(v) for v in rng.integers(1, 6, d))
        t = rng.random(dims)
        b.put(f"sweep.{d}.in", t)
        for code in range(1 << d):
            delta = fc.DeltaVector.from_code(code, d)
            out = fc.directional_sweep(fc.LocalSumTensor(t.copy()), delta).data
            b.put(f"sweep.{d}.{code}", out)

    # ---- grid Laplacian KDE (test_fastsum.py:138-164) ----
    for d in (1, 2, 3):
        rng = np.random.default_rng(d * 31)
        n = 500
        pts = rng.standard_normal((n, d))
        w = rng.uniform(0.5, 2.0, n)
        s = fc.validate_sample(pts, w)
        grid = fc.build_grid_auto(s, [max(2, round(n ** (1 / d)))] * d)
        h = rng.uniform(0.2, 0.6, d)
        key = f"kde.{d}"
        b.put(key + ".x", pts)
        b.put(key + ".w", w)
        b.put_knots(key, grid.knots)
        b.put(key + ".h", h)
        b.put(key + ".fast", fc.kde_fastsum(s, grid, fc.laplacian(), fc.Bandwidth.diag(h)).values)
        b.put(key + ".naive", fc.kde_naive(s, grid.lattice(), fc.laplacian(),
                                           fc.Bandwidth.diag(h)).values)
        b.put(key + ".unif", fc.kde_fastsum(s, grid, fc.uniform(), fc.Bandwidth.diag(h)).values)
        b.put(key + ".dnc", fc.kde_dnc(s, fc.laplacian(), fc.Bandwidth.diag(h)).values)
        # matern32-additive through the same terms (fastsum.py:170-181)
        b.put(key + ".mat", fc.kde_fastsum(s, grid, fc.matern32_additive(),
                                           fc.Bandwidth.diag(h)).values)
        b.put(key + ".matnaive", fc.kde_naive(s, grid.lattice(), fc.matern32_additive(),
                                              fc.Bandwidth.diag(h)).values)
    rng = np.random.default_rng(8)  # points on knots (test_fastsum.py:152-164)
    lat = np.linspace(-1.0, 1.0, 11)
    pts = np.column_stack([rng.choice(lat, 300), rng.choice(lat, 300)])
    w = rng.uniform(0.5, 2.0, 300)
    knots = [lat[::2], lat[1::3]]
    s = fc.validate_sample(pts, w)
    g = fc.RectilinearGrid.from_knots(knots)
    b.put("kdeknots.x", pts)
    b.put("kdeknots.w", w)
    b.put_knots("kdeknots", knots)
    b.put("kdeknots.fast", fc.kde_fastsum(s, g, fc.laplacian(), fc.Bandwidth.diag([0.25, 0.4])).values)

    # ---- multilinear interpolation grid -> points (interp.py:24-75) ----
    for d in (1, 2, 3):
        rng = np.random.default_rng(900 + d)
        knots = [np.sort(rng.uniform(-1, 1, int(rng.integers(2, 9)))) for _ in range(d)]
        g = fc.RectilinearGrid.from_knots(knots)
        vals = rng.standard_normal(g.size)
        q = rng.uniform(-1.3, 1.3, (257, d))   # some outside the hull (clamped)
        q[:5] = g.lattice()[:5]                # nodes reproduce bitwise
        q[5, 0] = knots[0][-1]                 # on the last knot
        r = fc.multilinear_interp(g, fc.EvalResult(vals, "grid"), q)
        key = f"interp.{d}"
        b.put_knots(key, knots)
        b.put(key + ".vals", vals)
        b.put(key + ".q", q)
        b.put(key + ".out", r.values)
        b.put(key + ".clamp", np.array(r.metadata["clamp_count"]))
    rng = np.random.default_rng(77)  # interpolated grid ECDF at the sample points (crit. 5)
    pts = rng.standard_normal((400, 2))
    s = fc.validate_sample(pts)
    g = fc.build_grid_auto(s, [20, 20])
    b.put("interp.ecdf.x", pts)
    b.put_knots("interp.ecdf", g.knots)
    b.put("interp.ecdf.out", fc.multilinear_interp(g, fc.ecdf_fastsum(s, g), pts).values)

    # ---- naive oracles (naive.py) ----
    rng = np.random.default_rng(4)
    pts = rng.standard_normal((300, 2))
    w = rng.uniform(0.5, 2, 300)
    s = fc.validate_sample(pts, w)
    q = rng.standard_normal((50, 2))
    b.put("naive.x", pts)
    b.put("naive.w", w)
    b.put("naive.q", q)
    for code in range(4):
        b.put(f"naive.ecdf.{code}", fc.ecdf_naive(s, q, fc.DeltaVector.from_code(code, 2)).values)
    b.put("naive.esf", fc.esf_naive(s, q).values)
    b.put("naive.kde", fc.kde_naive(s, q, fc.laplacian(), fc.Bandwidth.diag([0.4, 0.6])).values)

    # ---- divide and conquer at the points (test_dnc.py:36-66,113-189) ----
    for d in (1, 2, 3):
        for seed in range(4):
            rng = np.random.default_rng(100 * d + seed)
            n = int(rng.integers(1, 900))
            pts = rng.standard_normal((n, d))
            wi = rng.integers(1, 5, n).astype(float)
            key = f"dnc.{d}.{seed}"
            b.put(key + ".x", pts)
            b.put(key + ".w", wi)
            s = fc.validate_sample(pts, wi)
            b.put(key + ".out", fc.ecdf_dnc(s, scaled=False).values)
            b.put(key + ".self", fc.ecdf_dnc(s, include_self=True).values)
    for d in (1, 2, 3):
        rng = np.random.default_rng(d * 13)
        pts = rng.standard_normal((400, d))
        w = rng.uniform(0.5, 2.0, 400)
        h = rng.uniform(0.2, 0.5, d)
        s = fc.validate_sample(pts, w)
        key = f"kdednc.{d}"
        b.put(key + ".x", pts)
        b.put(key + ".w", w)
        b.put(key + ".h", h)
        b.put(key + ".out", fc.kde_dnc(s, fc.laplacian(), fc.Bandwidth.diag(h)).values)
        b.put(key + ".naive", fc.kde_naive(s, pts, fc.laplacian(), fc.Bandwidth.diag(h)).values)
        b.put(key + ".mat", fc.kde_dnc(s, fc.matern32_additive(), fc.Bandwidth.diag(h)).values)
        b.put(key + ".matnaive", fc.kde_naive(s, pts, fc.matern32_additive(),
                                              fc.Bandwidth.diag(h)).values)
        if d == 2:
            tt = fc.kde_terms_dnc(s, fc.Bandwidth.diag(h))
            b.put(key + ".psi", tt.psi)
            b.put(key + ".table", tt.table)
    # signed-weight fingerprint (test_dnc.py:135-146)
    rng = np.random.default_rng(79)
    pts = rng.standard_normal((256, 2))
    w = rng.standard_normal(256)
    tt = fc.kde_terms_dnc(fc.validate_sample(pts, w), fc.Bandwidth.diag([5.0, 5.0]))
    b.put("finger.x", pts)
    b.put("finger.w", w)
    b.put("finger.psi", tt.psi)
    b.put("finger.table", tt.table)

    # ---- generalized ECDF at the points with heavy ties (Eq. 3, naive semantics) ----
    for d in (1, 2, 3):
        for seed in range(3):
            rng = np.random.default_rng(500 + 10 * d + seed)
            n = int(rng.integers(50, 600))
            pts = rng.integers(0, 12, (n, d)).astype(float) / 4.0
            w = rng.uniform(0.0, 1.0, n)
            s = fc.validate_sample(pts, w)
            key = f"pts.{d}.{seed}"
            b.put(key + ".x", pts)
            b.put(key + ".w", w)
            for code in range(1 << d):
                dv = fc.DeltaVector.from_code(code, d)
                b.put(f"{key}.ecdf.{code}", fc.ecdf_naive(s, pts, dv).values)
            b.put(key + ".esf", fc.esf_naive(s, pts).values)

    # ---- generator (core.py:311-347) ----
    b.put("gen.4x2s7", fc.generate_gaussian_sample(4, 2, 7).points)
    b.put("gen.1001x3s3", fc.generate_gaussian_sample(1001, 3, 3).points)
    b.save("small.npz")


def cfg_golden(which):
    meta = {}
    path = HERE / "configs.json"
    if path.exists():
        meta = json.loads(path.read_text())
    rng_sub = np.random.default_rng(12345)
    for name in which:
        t0 = time.perf_counter()
        entry = {}
        bag = Bag()
        if name == "cfg1":
            w = wl.cfg1()
            s = fc.validate_sample(w.points)
            g = fc.RectilinearGrid.from_knots(w.knots)
            v = fc.ecdf_fastsum(s, g, fc.DeltaVector(w.delta), scaled=False).values
            entry["input_sha"] = wl.digest(w.points)
            entry["out_sha_f64"] = wl.digest(v)
            bag.put("counts", v.astype(np.int32))
            q = rng_sub.integers(0, g.size, 512)
            lat = g.lattice()[q]
            bag.put("naive_idx", q)
            bag.put("naive", fc.ecdf_naive(s, lat, scaled=False).values)
        elif name == "cfg2":
            w = wl.cfg2()
            s = fc.validate_sample(w.points, w.weights)
            lat_knots = [np.arange(1024) / 1024.0] * 2
            g = fc.RectilinearGrid.from_knots(lat_knots)
            r = (w.points * 1024).astype(np.int64)
            flat = r[:, 0] * 1024 + r[:, 1]
            ecdf = fc.ecdf_fastsum(s, g, fc.DeltaVector((1, -1))).values[flat]
            esf = fc.esf_fastsum(s, g).values[flat]
            entry["input_sha"] = wl.digest(w.points)
            entry["weights_sha"] = wl.digest(w.weights)
            idx = rng_sub.integers(0, w.n, 4096)
            bag.put("idx", idx)
            bag.put("ecdf", ecdf[idx])
            bag.put("esf", esf[idx])
            sub = idx[:1000]
            bag.put("naive_ecdf", fc.ecdf_naive(s, w.points[sub], fc.DeltaVector((1, -1))).values)
            bag.put("naive_esf", fc.esf_naive(s, w.points[sub]).values)
        elif name == "cfg3":
            w = wl.cfg3()
            s = fc.validate_sample(w.points)
            g = fc.RectilinearGrid.from_knots(w.knots)
            v = fc.ecdf_fastsum(s, g, fc.DeltaVector(w.delta), scaled=False).values
            entry["input_sha"] = wl.digest(w.points)
            entry["out_sha_i64"] = wl.digest(v.astype(np.int64))
            idx = rng_sub.integers(0, v.size, 8192)
            bag.put("idx", idx)
            bag.put("vals", v[idx])
        elif name in ("cfg4", "cfg4_1e6"):
            n = 10_000_000 if name == "cfg4" else 1_000_000
            w = wl.cfg4(n)
            bw = fc.Bandwidth.diag(w.h)
            entry["input_sha"] = wl.digest(w.points)
            entry["y_sha"] = wl.digest(w.extra["y"])
            dens = fc.kde_dnc(fc.validate_sample(w.points), fc.laplacian(), bw).values
            reg = fc.kde_dnc(fc.validate_sample(w.points, w.extra["y"]), fc.laplacian(), bw).values
            absn = fc.kde_dnc(fc.validate_sample(w.points, np.abs(w.extra["y"])), fc.laplacian(),
                              bw).values
            idx = rng_sub.integers(0, n, 8192)
            bag.put("idx", idx)
            bag.put("density", dens[idx])
            bag.put("regression", reg[idx])
            bag.put("abs_regression", absn[idx])
            entry["density_sha"] = wl.digest(dens)
        elif name in ("cfg5a", "cfg5b"):
            w = wl.cfg5()
            g = fc.RectilinearGrid.from_knots(w.knots)
            entry["input_sha"] = wl.digest(w.points)
            entry["y_sha"] = wl.digest(w.extra["y"])
            idx = rng_sub.integers(0, g.size, 8192)
            bag.put("idx", idx)
            if name == "cfg5a":
                s = fc.validate_sample(w.points)
                v = fc.ecdf_fastsum(s, g, fc.DeltaVector(w.delta), scaled=False).values
                entry["out_sha_i64"] = wl.digest(v.astype(np.int64))
                bag.put("vals", v[idx])
            else:
                s = fc.Sample(w.points, w.extra["y"], (True,) * 4)
                v = fc.kde_fastsum(s, g, fc.laplacian(), fc.Bandwidth.diag(w.h)).values
                bag.put("vals", v[idx])
            del v
        entry["reference_seconds"] = time.perf_counter() - t0
        meta[name] = entry
        bag.save(f"{name}.npz")
        path.write_text(json.dumps(meta, indent=1, sort_keys=True))
        print(name, json.dumps(entry), flush=True)


def csv_golden():
    """Bytes of the reference's CSV writers (core.py:350-377) for the wire-format tests."""
    import tempfile

    rng = np.random.default_rng(11)
    out = {}
    with tempfile.TemporaryDirectory() as td:
        s = fc.validate_sample(rng.standard_normal((7, 3)), rng.uniform(0.5, 2.0, 7))
        fc.write_sample_csv(s, f"{td}/w.csv")
        fc.write_sample_csv(fc.validate_sample(rng.standard_normal((5, 2))), f"{td}/u.csv")
        g = fc.RectilinearGrid.from_knots([np.array([0.0, 0.5]), np.array([1.0, 2.0, 3.0])])
        fc.write_result_csv(g.lattice(), np.arange(6.0) / 7.0, f"{td}/r.csv")
        for k in "wur":
            out[k] = np.frombuffer(open(f"{td}/{k}.csv", "rb").read(), dtype=np.uint8)
    np.savez_compressed(HERE / "csv.npz", **out)
    print("wrote csv.npz", flush=True)


def nd_golden():
    """At-points dominance sums for d >= 3 at sizes that take the rank-space coarse-grid route
    (n >= 8192): the reference's MergeND recursion (dnc.py:65-135, 307-410) is the oracle."""
    bag = Bag()
    rng = np.random.default_rng(20240521)
    for d, n in [(3, 10_000), (4, 9_000), (5, 8_500)]:
        x = rng.standard_normal((n, d))
        w = rng.uniform(0.5, 2.0, n)
        h = rng.uniform(0.4, 0.8, d)
        key = f"nd{d}"
        bag.put(key + ".x", x)
        bag.put(key + ".w", w)
        bag.put(key + ".h", h)
        s = fc.validate_sample(x, w)
        su = fc.validate_sample(x)
        bag.put(key + ".ecdf_w", fc.ecdf_dnc(s, scaled=False).values)
        bag.put(key + ".ecdf_unit_self", fc.ecdf_dnc(su, include_self=True, scaled=False).values)
        bag.put(key + ".ecdf_scaled", fc.ecdf_dnc(su).values)
        bag.put(key + ".kde_w", fc.kde_dnc(s, fc.laplacian(), fc.Bandwidth.diag(h)).values)
        bag.put(key + ".kde_unit", fc.kde_dnc(su, fc.laplacian(), fc.Bandwidth.diag(h)).values)
        bag.put(key + ".mat_w", fc.kde_dnc(s, fc.matern32_additive(), fc.Bandwidth.diag(h)).values)
        if d <= 4:
            tt = fc.kde_terms_dnc(s, fc.Bandwidth.diag(h), (0, d - 1, 1, 1))
            rows = rng.integers(0, n, 400)
            bag.put(key + ".terms_rows", rows)
            bag.put(key + ".terms", tt.table[rows])
    bag.save("nd.npz")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--nd", action="store_true")
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--csv", action="store_true")
    ap.add_argument("--configs", default="")
    a = ap.parse_args()
    if a.nd:
        nd_golden()
    if a.small:
        small()
    if a.csv:
        csv_golden()
    if a.configs:
        cfg_golden([c for c in a.configs.split(",") if c])
