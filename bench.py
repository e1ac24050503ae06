#!/usr/bin/env python
"""Benchmark of the B200 generalized-ECDF / Laplacian-KDE hot path (BASELINE.json metric:
"ECDF/Laplacian-KDE points/sec at 1/2/4/8 B200; % of HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg5|cfg5a|cfg5b|cfg3|cfg1|cfg2|cfg4|nd3]

Default workload: BASELINE config 5 (the largest configuration that fits one GPU): N = 1e8
points iid U[0,1]^4 on a 128^4 grid; one step = the 4-D grid ECDF (y == 1) followed by the
Laplacian KDE (y ~ Exp(1), h = 0.05) on the same resident points.  Prints ONE JSON line on
rank 0.  `value` is device throughput (points/s, inputs resident in HBM, CUDA events, max over
ranks); `e2e` is the same metric through the public API from pinned host buffers with the H2D
input copies and the D2H of the full result grids inside the timed region.

--impl reference times the unmodified reference package (baseline/_ref, installed with pip
--target; numba, single-threaded by design) through its public API on a bounded sample of the
same workload, rank 0 only; without baseline/_ref it falls back to the C restatement (oracle/).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import workloads as wl  # noqa: E402

METRIC = "ECDF/Laplacian-KDE points/sec at 1/2/4/8 B200; % of HBM roofline"
UNIT = "points/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="cfg5")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--numpy-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--slab", action="store_true",
                    help="run the grid configs through the multi-GPU slab path even on one GPU "
                         "(exercises the NCCL routing / carry exchange with world size 1)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------------------
# clocks during the timed region
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names[1:], parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        med = float(np.median(sm)) if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# workloads: algorithmic bytes per kernel launch (pass-structured)

def grid_ecdf_bytes(n, d, m, unit=True):
    L = int(np.prod(m))  # dead layers elided: lattice = output extents
    e = 4 if unit else 8
    return {
        # atomic path (sparse lattices)
        "lattice_zero": e * L,
        "bin_scatter_count" if unit else "bin_scatter_w": 8 * n * d + (0 if unit else 8 * n) + 2 * e * n,
        "scan_chunk_carry": e * L,  # chunk totals of a long axis (one read of the lattice)
        "scan_rows": 2 * e * L,
        "scan_lines": 2 * e * L,
        "scan_plane2d": 2 * e * L,  # both in-plane axes in one read + write
        "scan_lines_final": e * L + 8 * L,
        # plane-partitioned path: bucket keys + payloads (u32 each), one 8-bit radix pass each
        "part_bin": 8 * n * d + 8 * n,
        "radix_hist": 4 * n,
        "radix_scatter": 16 * n,
        "plane_count": 4 * n + e * L,
    }


def grid_kde_bytes(n, d, m, unit_w):
    """Algorithmic bytes per launch of the partitioned Laplacian KDE (d >= 3) and of the
    per-term pipeline (smaller problems)."""
    L = int(np.prod(m))
    terms = 1 << d
    wb = 0 if unit_w else 8 * n
    per0 = max(1, (1 << max(d - 2, 1)) // 2)  # group lattices per final axis-0 pass
    return {
        "lattice_zero": 8 * L,
        "bin_scatter_psi": 8 * n * d + wb + 16 * n,
        "scan_rows": 16 * L,
        "scan_lines": 16 * L,
        # first term only writes the accumulator; the other 2^d - 1 read and write it
        "scan_lines_final": 8 * L + (8 * L + 16 * L * (terms - 1)) // terms,
        "kde_zfac": 16 * int(np.sum(m)),
        "minmax": 8 * n * d,
        # keys + slots of every point from its coordinates
        "part_bin": 8 * n * d + 8 * n,
        "part_hist": 4 * n,
        # records built from x, w (coalesced) and written grouped by the key's top 8 bits
        "part_emit": 4 * n + 8 * n * d + wb + 8 * n * (d + 1) + 8 * n,
        "radix_hist": 4 * n,
        "radix_scatter": 16 * n,
        # last segmented sort pass: (key, slot) in, key out, and each slot's record gathered
        # from its coarse segment (L2-resident window) and written field-major
        "kde_materialize": 12 * n + 16 * n * (d + 1),
        # all term groups in one launch (d = 3, 4): two passes over the records (keys, A, the
        # leading q's, q_col; q_row in the second), and per group lattice the first row-sign
        # pass writes it and the second reads and rewrites it
        "plane_kde": 8 * n + 8 * n * (2 * (d + 1) - 1) + (1 << (d - 2)) * 24 * L,
        # one axis-0 pass over the group lattices sharing delta_0; accumulator written by the
        # first pass, read + written by the second
        "kde_final_group": per0 * 8 * L + (8 * L + 16 * L) // 2,
    }


def traffic_lookup(workload, kernel):
    """DRAM bytes per launch of `kernel` from a committed ncu --set full capture
    (profiles/traffic.json, written from dram__bytes_read.sum + dram__bytes_write.sum)."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    try:
        tab = json.loads(p.read_text())
    except ValueError:
        return None
    for wl_name in (workload, workload + "b", workload + "a"):  # cfg5 = cfg5a + cfg5b
        v = tab.get(wl_name, {}).get(kernel)
        if v is not None:
            return v
    return None


class GridWorkload:
    """Grid configs (1, 3, 5a, 5b, 5): device-resident sample + public API calls."""

    scaling = "strong"  # the configuration's total work is fixed; N > 1 shards it

    @staticmethod
    def parallelism(world):
        if world == 1:
            return "single GPU"
        return (f"slab x{world}: lattice split along axis 1, points routed with one NCCL "
                f"all-to-all, slab carry planes exchanged with an NCCL all-gather")

    def __init__(self, name):
        import paper_2005_03246_b200 as fcb

        self.fcb = fcb
        self.name = name
        base = name[:4]
        gen = {"cfg1": wl.cfg1, "cfg3": wl.cfg3, "cfg5": wl.cfg5}[base]
        self.w = gen()
        self.do_ecdf = name in ("cfg1", "cfg3", "cfg5", "cfg5a")
        self.do_kde = name in ("cfg5", "cfg5b")
        self.grid = fcb.RectilinearGrid.from_knots(self.w.knots)
        self.n, self.d = self.w.n, self.w.d
        self.m = self.grid.shape
        self.delta = fcb.DeltaVector(self.w.delta)
        self.bw = fcb.Bandwidth.diag(self.w.h) if self.w.h is not None else None
        self.y = self.w.extra.get("y")

    def describe(self):
        parts = []
        if self.do_ecdf:
            parts.append(f"{self.d}-D grid ECDF y==1 delta={self.w.delta}")
        if self.do_kde:
            parts.append(f"{self.d}-D grid Laplacian KDE y~Exp(1) h={float(self.w.h[0])}")
        return {
            "workload": self.name,
            "what": " + ".join(parts),
            "n_points": self.n, "dims": self.d, "grid": "x".join(str(v) for v in self.m),
            "lattice_cells": int(np.prod(self.m)),
            "l2": f"inputs larger than L2 ({self.n * self.d * 8 / 1e9:.2f} GB points)"
            if self.n * self.d * 8 > 126e6 else "L2-resident (launch-bound config)",
        }

    slab = False

    def shard(self, rank, world):
        """Strong scaling over the fixed config: rank r holds points r::world."""
        self.rank, self.world = rank, world
        self.n_total = self.n
        if world > 1:
            self.pts = np.ascontiguousarray(self.w.points[rank::world])
            self.yv = None if self.y is None else np.ascontiguousarray(self.y[rank::world])
        else:
            self.pts, self.yv = self.w.points, self.y

    def to_device(self):
        import torch

        fcb = self.fcb
        x = torch.from_numpy(self.pts).cuda()
        self.s_unit = fcb.Sample(x, torch.ones(x.shape[0], dtype=torch.float64, device=x.device),
                                 None, True)
        if self.do_kde:
            y = torch.from_numpy(self.yv).cuda()
            self.s_y = fcb.Sample(x, y, None, False)

    def to_pinned(self):
        import torch

        fcb = self.fcb
        xp = torch.from_numpy(self.pts).pin_memory()
        self.p_x = xp
        self.up_stream = torch.cuda.Stream()
        self.down_stream = torch.cuda.Stream()
        self.xd = [torch.empty_like(xp, device="cuda") for _ in range(2)]
        self.ones_dev = torch.ones(1, device="cuda")
        self.p_unit = fcb.Sample(xp, torch.ones(1), None, True)
        nloc = int(np.prod(self.m))
        self.out_pinned = torch.empty(nloc, dtype=torch.float64).pin_memory()
        if self.do_kde:
            yp = torch.from_numpy(self.yv).pin_memory()
            self.p_yv = yp
            self.yd = [torch.empty_like(yp, device="cuda") for _ in range(2)]
            self.p_y = fcb.Sample(xp, yp, None, False)
            self.out2_pinned = torch.empty(nloc, dtype=torch.float64).pin_memory()
        self.h2d_bytes = self.pts.nbytes + (self.yv.nbytes if self.do_kde else 0)
        self.d2h_bytes = nloc * 8 * (int(self.do_ecdf) + int(self.do_kde)) // self.world
        self.pipelined = self.h2d_bytes + self.d2h_bytes >= 64e6
        if not self.pipelined:
            self.e2e_mode = "serial: upload, compute, download (one stream)"


    def _ecdf(self, s):
        if self.world > 1 or self.slab:
            from paper_2005_03246_b200 import distributed as fdist

            return fdist.ecdf_fastsum_slab(s, self.grid, self.delta).values
        return self.fcb.ecdf_fastsum(s, self.grid, self.delta).values

    def _kde(self, s):
        if self.world > 1 or self.slab:
            from paper_2005_03246_b200 import distributed as fdist

            return fdist.kde_fastsum_slab(s, self.grid, self.fcb.laplacian(), self.bw).values
        return self.fcb.kde_fastsum(s, self.grid, self.fcb.laplacian(), self.bw).values

    def step(self):
        if self.do_ecdf:
            self._ecdf(self.s_unit)
        if self.do_kde:
            self._kde(self.s_y)

    def _upload(self, j):
        """H2D of step j's inputs on the upload stream into buffer j % 2, once the compute
        that last read that buffer (step j - 2) is done."""
        import torch

        b = j % 2
        up = self.up_stream
        if self.ev_free[b] is not None:
            up.wait_event(self.ev_free[b])
        with torch.cuda.stream(up):
            self.xd[b].copy_(self.p_x, non_blocking=True)
            if self.do_kde:
                self.yd[b].copy_(self.p_yv, non_blocking=True)
        self.ev_up[b] = up.record_event()

    e2e_mode = ("pipelined: step k+1's upload and step k's downloads overlap step k's compute "
                "(copy engines on two side streams)")

    def e2e_begin(self):
        if not self.pipelined:
            return
        main = __import__("torch").cuda.current_stream()
        self.ev_free = [main.record_event(), main.record_event()]
        self.ev_up = [None, None]
        self.e2e_k = 0
        self._upload(0)

    def e2e_end(self):
        if not self.pipelined:
            return
        main = __import__("torch").cuda.current_stream()
        main.wait_stream(self.up_stream)
        main.wait_stream(self.down_stream)

    def step_e2e(self, last=True):
        """Host-resident inputs -> public API -> host-resident results, two steps in flight:
        step k+1's upload (upload stream) and step k's downloads (download stream) run on the
        copy engines while step k computes, so a step costs max(H2D, D2H, compute) rather than
        their sum.  Every step still uploads its own points and weights and downloads its
        densities (h2d/d2h_bytes_per_step); the timed region starts before step 0's upload and
        ends after the last download."""
        import torch

        if not self.pipelined:  # small configs: cross-stream hand-offs cost more than they hide
            main = torch.cuda.current_stream()
            xd = self.p_x.to("cuda", non_blocking=True)
            if self.do_ecdf:
                v = self._ecdf(self.fcb.Sample(xd, self.ones_dev, None, True))
                self.out_pinned[: v.numel()].copy_(v, non_blocking=True)
            if self.do_kde:
                yd = self.p_yv.to("cuda", non_blocking=True)
                v = self._kde(self.fcb.Sample(xd, yd, None, False))
                self.out2_pinned[: v.numel()].copy_(v, non_blocking=True)
            return
        k = self.e2e_k
        self.e2e_k += 1
        if not last:
            self._upload(k + 1)
        main = torch.cuda.current_stream()
        down = self.down_stream
        b = k % 2
        main.wait_event(self.ev_up[b])
        xd = self.xd[b]
        if self.do_ecdf:
            v = self._ecdf(self.fcb.Sample(xd, self.ones_dev, None, True))
            down.wait_stream(main)
            with torch.cuda.stream(down):
                self.out_pinned[: v.numel()].copy_(v, non_blocking=True)
            v.record_stream(down)
        if self.do_kde:
            v = self._kde(self.fcb.Sample(xd, self.yd[b], None, False))
            down.wait_stream(main)
            with torch.cuda.stream(down):
                self.out2_pinned[: v.numel()].copy_(v, non_blocking=True)
            v.record_stream(down)
        self.ev_free[b] = main.record_event()

    def numpy_prepare(self):
        """Host numpy samples as a reference user builds them (validate_sample, outside the
        timing); the drop-in call then takes numpy in and returns numpy out."""
        fcb = self.fcb
        self.np_unit = fcb.validate_sample(self.pts)
        self.np_y = fcb.validate_sample(self.pts, self.yv) if self.do_kde else None
        nloc = int(np.prod(self.m))
        return (self.pts.nbytes * (int(self.do_ecdf) + int(self.do_kde))
                + (self.yv.nbytes if self.do_kde else 0),
                nloc * 8 * (int(self.do_ecdf) + int(self.do_kde)))

    def step_numpy(self):
        fcb = self.fcb
        if self.do_ecdf:
            fcb.ecdf_fastsum(self.np_unit, self.grid, self.delta).values
        if self.do_kde:
            fcb.kde_fastsum(self.np_y, self.grid, fcb.laplacian(), self.bw).values

    def bytes_per_launch(self):
        # per rank: ~1/world of the points and of the lattice (axis-1 slab) when sharded
        n = self.n // self.world
        m = list(self.m)
        if self.world > 1:
            m[1] = max(1, m[1] // self.world)
        b = {}
        if self.do_kde:
            b.update(grid_kde_bytes(n, self.d, m, False))
        if self.do_ecdf:
            e = grid_ecdf_bytes(n, self.d, m, True)
            for k, v in e.items():
                if k in b:  # shared label between ECDF and KDE: keep them apart
                    b[k + "@ecdf"] = v
                else:
                    b[k] = v
        return b

    # ---- CPU baseline / reference arm: the reference package itself on a bounded sample ----
    def ref_prepare(self, fc):
        """Build (outside any timing) the reference inputs for one bounded sample of this
        workload and return (n_points, description, call).  Configs with >= 5e7 points use the
        1/64 block made of the first 1/8 of the knots of axes 0 AND 1 (full axes 2, 3) and the
        points falling in it: the grid ECDF there is exactly the full configuration's ECDF
        restricted to those cells (forward sums only reach lower knots), and the KDE is the same
        reference algorithm (bincount + 2^d directional sweeps) over that block.  Smaller
        configurations run in full."""
        knots = [np.asarray(z) for z in self.w.knots]
        pts, y = self.w.points, self.y
        desc = "full configuration"
        if self.n >= 50_000_000:
            k = len(knots[0]) // 8
            knots[0], knots[1] = knots[0][:k], knots[1][:k]
            sel = (pts[:, 0] <= knots[0][-1]) & (pts[:, 1] <= knots[1][-1])
            pts = np.ascontiguousarray(pts[sel])
            y = None if y is None else np.ascontiguousarray(y[sel])
            desc = (f"{pts.shape[0]} points in the 1/64 block of the grid (first {k} knots of "
                    f"axes 0 and 1, full axes 2..{self.d - 1}: a "
                    f"{'x'.join(str(len(z)) for z in knots)} sub-grid)")
        grid = fc.RectilinearGrid.from_knots(knots)
        calls, what = [], []
        if self.do_ecdf:
            s1 = fc.validate_sample(pts)
            dv = fc.DeltaVector(tuple(self.w.delta))
            calls.append(lambda: fc.ecdf_fastsum(s1, grid, dv))
            what.append("fastcdf.ecdf_fastsum")
        if self.do_kde:
            s2 = fc.validate_sample(pts, y)
            bw = fc.Bandwidth.diag(self.w.h)
            lap = fc.laplacian()
            calls.append(lambda: fc.kde_fastsum(s2, grid, lap, bw))
            what.append("fastcdf.kde_fastsum(laplacian)")

        def call():
            for c in calls:
                c()
        return pts.shape[0], f"{desc}; {' + '.join(what)}", call

    def ref_warm(self, fc):
        """Compile the reference's numba kernels on a tiny instance of the same calls."""
        rng = np.random.default_rng(0)
        x = rng.random((256, self.d))
        g = fc.RectilinearGrid.from_knots([np.linspace(0, 1, 5)] * self.d)
        if self.do_ecdf:
            fc.ecdf_fastsum(fc.validate_sample(x), g, fc.DeltaVector(tuple(self.w.delta)))
        if self.do_kde:
            fc.kde_fastsum(fc.validate_sample(x, rng.random(256)), g, fc.laplacian(),
                           fc.Bandwidth.diag(np.full(self.d, 0.5)))

    # ---- fallback when baseline/_ref is absent: the C restatement (oracle/) ----------------
    def cpu_sample(self, threads):
        """Time the oracle port on the same bounded sample as ref_prepare (no scaling)."""
        import oracle

        used = oracle.set_threads(threads)
        knots = [np.asarray(z) for z in self.w.knots]
        pts, y = self.w.points, self.y
        if self.n >= 50_000_000:
            k = len(knots[0]) // 8
            knots[0], knots[1] = knots[0][:k], knots[1][:k]
            sel = (pts[:, 0] <= knots[0][-1]) & (pts[:, 1] <= knots[1][-1])
            pts = np.ascontiguousarray(pts[sel])
            y = None if y is None else np.ascontiguousarray(y[sel])
        n_s = pts.shape[0]
        t0 = time.perf_counter()
        if self.do_ecdf:
            oracle.ecdf_fastsum(pts, None, knots, self.w.delta, scaled=True)
        if self.do_kde:
            oracle.kde_fastsum_laplacian(pts, y, knots, self.w.h)
        dt = time.perf_counter() - t0
        return n_s / dt, used, f"{n_s} points (1/64 block when N >= 5e7); oracle port", dt


def dominant(prof: dict, bytes_map: dict):
    """Kernel label with the largest device time; its algorithmic bytes per launch."""
    best = None
    for name, (cnt, ms) in prof.items():
        if name == "lattice_zero":
            continue
        if best is None or ms > best[2]:
            best = (name, cnt, ms)
    if best is None:
        return None
    name, cnt, ms = best
    return name, cnt, ms, bytes_map.get(name)


def radix_bytes(n):
    # per radix pass: histogram reads 8-byte keys; scatter reads and writes key + int32 payload
    return {"radix_hist": 8 * n, "radix_scatter": 24 * n, "radix_init": 8 * n + 12 * n}


class PointsWorkload:
    """At-points configs: cfg2 (ECDF delta=(1,-1) + ESF with ties, N = 1e6) and cfg4 (Laplacian
    KDE density + regression numerators, N = 1e7, one device pass)."""

    scaling = "strong"  # the configuration's work is fixed; N > 1 splits cfg4's queries

    def parallelism(self, world):
        if world == 1:
            return "single GPU"
        if self.name == "cfg4":
            return (f"query shards x{world}: sources ranked on every GPU (replicated), queries "
                    f"split by dimension-1 rank chunks, one NCCL SUM all-reduce gathers the "
                    f"numerators")
        return (f"replicas x{world}: this route (rank lattice / d >= 3 rank grid) is not sharded, "
                f"every GPU computes the whole problem (counted once)")

    def __init__(self, name):
        import paper_2005_03246_b200 as fcb

        self.fcb = fcb
        self.name = name
        self.w = wl.cfg2() if name == "cfg2" else (wl.nd3() if name == "nd3" else wl.cfg4())
        self.n, self.d = self.w.n, self.w.d

    def describe(self):
        if self.name == "cfg2":
            what = "2-D ECDF at the points, ties (1024 levels), y~U(0,1), delta=(1,-1) + ESF"
        elif self.name == "nd3":
            what = ("3-D Laplacian KDE density + kernel-regression numerators at the points, "
                    "h=0.2 (not a BASELINE config: the SURVEY 8f #3 widening)")
        else:
            what = "2-D Laplacian KDE density + kernel-regression numerators at the points, h=0.1"
        return {"workload": self.name, "what": what, "n_points": self.n, "dims": self.d,
                "l2": "inputs fit in L2 (launch/latency-bound config)" if self.n * 16 < 126e6
                else f"inputs larger than L2 ({self.n * 16 / 1e9:.2f} GB points)"}

    def shard(self, rank, world):
        """cfg4: query shards (strong scaling); cfg2: replicas, the problem counted once."""
        self.rank, self.world = rank, world
        self.n_total = self.n

    def _sample(self, x, y):
        fcb = self.fcb
        if self.name == "cfg2":
            return fcb.Sample(x, y, None, False)
        return fcb.Sample(x, None, (True,) * self.d, True)

    def to_device(self):
        import torch

        x = torch.from_numpy(self.w.points).cuda()
        yv = self.w.weights if self.name == "cfg2" else self.w.extra["y"]
        self.y_dev = torch.from_numpy(yv).cuda()
        self.s_dev = self._sample(x, self.y_dev)

    def to_pinned(self):
        import torch

        xp = torch.from_numpy(self.w.points).pin_memory()
        yv = self.w.weights if self.name == "cfg2" else self.w.extra["y"]
        self.y_pin = torch.from_numpy(yv).pin_memory()
        self.s_pin = self._sample(xp, self.y_pin)
        nout = 2 * self.n
        self.out_pinned = torch.empty(nout, dtype=torch.float64).pin_memory()
        self.h2d_bytes = self.w.points.nbytes + yv.nbytes
        self.d2h_bytes = nout * 8

    def _run(self, s, y):
        fcb = self.fcb
        if self.name == "cfg2":  # both outputs from one ranking of the points
            a, b = fcb.ecdf_esf_at_points(s, fcb.DeltaVector(self.w.delta))
            return a.values, b.values
        if self.world > 1 and self.name == "cfg4":
            from paper_2005_03246_b200 import distributed as fdist

            num = fdist.kde_numerators_sharded(s, [None, y], fcb.Bandwidth.diag(self.w.h))
        else:
            num = fcb.kde_numerators(s, [None, y], fcb.Bandwidth.diag(self.w.h))
        return num[0], num[1]

    def step(self):
        self._run(self.s_dev, self.y_dev)

    e2e_mode = "serial: upload, compute, download"

    def e2e_begin(self):
        pass

    def e2e_end(self):
        pass

    def step_e2e(self, last=True):
        a, b = self._run(self.s_pin, self.y_pin)
        self.out_pinned[: self.n].copy_(a, non_blocking=True)
        self.out_pinned[self.n:].copy_(b, non_blocking=True)

    def numpy_prepare(self):
        fcb = self.fcb
        x = self.w.points
        if self.name == "cfg2":
            self.np_s = fcb.validate_sample(x, self.w.weights)
            return x.nbytes + self.w.weights.nbytes, 2 * self.n * 8
        self.np_s = fcb.validate_sample(x)
        return x.nbytes + self.w.extra["y"].nbytes, 2 * self.n * 8

    def step_numpy(self):
        fcb = self.fcb
        if self.name == "cfg2":
            fcb.ecdf_at_points(self.np_s, fcb.DeltaVector(self.w.delta)).values
            fcb.esf_at_points(self.np_s).values
        else:
            fcb.kde_numerators(self.np_s, [None, self.w.extra["y"]], fcb.Bandwidth.diag(self.w.h))

    def bytes_per_launch(self):
        n = self.n
        b = radix_bytes(n)
        if self.name == "cfg2":
            b.update({"pts_rank_scatter": (8 + 8 + 8) * n, "pts_gather": (8 + 8 + 8) * n})
        elif self.name == "nd3":
            pass  # pair-test kernels: issue-bound, no byte model
        else:
            # level-2 solvers: per source (id + 2 positions + 2 psi) and per query (threshold
            # pair + list entry + 2-channel output read-modify-write)
            # group-ordered self dominance, per launch and per point: slot + rank positions,
            # 2-channel psi, the z factor, and two read-modify-writes of the 2-channel
            # accumulator (slot-order pass, rank-order pass)
            # level-2 solvers, all four sign codes per launch: slot + rank position once, the
            # point and its two weights re-read per code, one 2-channel store per point
            b.update({"pts_level2_chunk": (4 + 4 + 4 * (16 + 16) + 16) * n,
                      "pts_level2_block": (4 + 4 + 4 * (16 + 16) + 16) * n,
                      "pts_group_gather": (4 + 8 + 16 + 16) * n + (4 + 4 + 16 + 16 + 4) * n,
                      "pts_psi": (16 + 16 + 16 + 8) * n})
        return b

    def ref_prepare(self, fc):
        """Reference inputs for one bounded sample (built outside the timing).
        cfg2: the reference's own route for ties at the points: the grid ECDF / ESF on
        the 1024-level lattice (fastsum.py:69-111) gathered at the points, full configuration.
        cfg4: fastcdf.kde_dnc (dnc.py:635-690) for both weight vectors on the first 1e6 points
        (the full N = 1e7 takes ~130 s per step on one core)."""
        x = self.w.points
        if self.name == "cfg2":
            lev = 1024
            g = fc.RectilinearGrid.from_knots([np.arange(lev) / lev] * 2)
            s = fc.validate_sample(x, self.w.weights)
            idx = (x * lev).astype(np.int64)
            flat = idx[:, 0] * lev + idx[:, 1]
            dv = fc.DeltaVector(tuple(self.w.delta))

            def call():
                fc.ecdf_fastsum(s, g, dv).values[flat]
                fc.esf_fastsum(s, g).values[flat]
            return self.n, ("full configuration; fastcdf.ecdf_fastsum + esf_fastsum on the "
                            "1024-level lattice, gathered at the points"), call
        m = 200_000 if self.name == "nd3" else 1_000_000
        s1 = fc.validate_sample(x[:m])
        s2 = fc.validate_sample(x[:m], self.w.extra["y"][:m])
        bw = fc.Bandwidth.diag(self.w.h)
        lap = fc.laplacian()

        def call():
            fc.kde_dnc(s1, lap, bw)
            fc.kde_dnc(s2, lap, bw)
        return m, f"first {m} points; fastcdf.kde_dnc(laplacian) for w == 1 and w = y", call

    def ref_warm(self, fc):
        rng = np.random.default_rng(0)
        x = rng.random((256, 2))
        if self.name == "cfg2":
            g = fc.RectilinearGrid.from_knots([np.arange(8) / 8] * 2)
            s = fc.validate_sample(x, rng.random(256))
            fc.ecdf_fastsum(s, g, fc.DeltaVector((1, -1)))
            fc.esf_fastsum(s, g)
        else:
            if self.name == "nd3":
                x = rng.random((256, 3))
            fc.kde_dnc(fc.validate_sample(x, rng.random(256)), fc.laplacian(),
                       fc.Bandwidth.diag(np.full(x.shape[1], 0.1)))

    def cpu_sample(self, threads):
        import oracle

        used = oracle.set_threads(threads)
        if self.name == "cfg2":
            t0 = time.perf_counter()
            oracle.ecdf_at_points(self.w.points, self.w.weights, self.w.delta)
            oracle.esf_at_points(self.w.points, self.w.weights)
            dt = time.perf_counter() - t0
            return self.n / dt, used, "full config (ECDF + ESF via the exact rank lattice)", dt
        if self.name == "nd3":  # the oracle has direct sums only for d = 3: a query subset
            m, nq = 200_000, 2_000
            used = oracle.set_threads(threads)
            t0 = time.perf_counter()
            oracle.kde_naive_laplacian(self.w.points[:m], None, self.w.points[:nq], self.w.h)
            oracle.kde_naive_laplacian(self.w.points[:m], self.w.extra["y"][:m],
                                       self.w.points[:nq], self.w.h)
            dt = time.perf_counter() - t0
            return nq / dt, used, f"direct sums of {nq} queries over the first {m} points", dt
        m = 1_000_000
        t0 = time.perf_counter()
        oracle.kde_dnc_laplacian(self.w.points[:m], None, self.w.h)
        oracle.kde_dnc_laplacian(self.w.points[:m], self.w.extra["y"][:m], self.w.h)
        dt = time.perf_counter() - t0
        return m / dt, 1, f"first {m} points, both numerators (the C recursion is single-threaded)", dt


def make_workload(name):
    if name in ("cfg1", "cfg3", "cfg5", "cfg5a", "cfg5b"):
        return GridWorkload(name)
    if name in ("cfg2", "cfg4", "nd3"):
        return PointsWorkload(name)
    raise SystemExit(f"unknown workload {name!r}")


# ------------------------------------------------------------------------------------------
def load_fastcdf():
    """The unmodified reference package installed under baseline/_ref (pip --target, see
    DESIGN.md), or None when it is absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "fastcdf" / "__init__.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fcg_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import fastcdf

    return fastcdf


def reference_timing(w, steps, warm=True):
    """Time `steps` runs of the reference's public API on the workload's bounded sample.
    Returns (points/s, seconds per step, cores, kind, sample description)."""
    fc = load_fastcdf()
    if fc is None:  # fallback: the C restatement of the same algorithm (oracle/)
        vals, secs, sample, used = [], [], "", 1
        for _ in range(steps):
            v, used, sample, dt = w.cpu_sample(0)
            vals.append(v)
            secs.append(dt)
        return float(np.sum([v * t for v, t in zip(vals, secs)]) / np.sum(secs)), \
            float(np.mean(secs)), used, "port", sample + " (baseline/_ref absent)"
    if warm:
        w.ref_warm(fc)
    n_s, sample, call = w.ref_prepare(fc)
    secs = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        secs.append(time.perf_counter() - t0)
    tot = float(np.sum(secs))
    return n_s * steps / tot, tot / steps, 1, "reference", sample


def run_reference(args, rank, world):
    """--impl reference: the unmodified reference package (baseline/_ref, numba, single-threaded
    by design: cli.py:265-268) through its public API on the host, rank 0 only."""
    if rank != 0:
        return
    w = make_workload(args.workload)
    fc = load_fastcdf()
    if fc is not None:
        for _ in range(max(args.warmup, 1)):  # warm-up = jit compile on a tiny instance
            w.ref_warm(fc)
    value, sec, cores, kind, sample = reference_timing(w, args.steps, warm=False)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": w.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded numpy, SURVEY §8d)",
        "config": w.describe(), "parallelism": "host CPU, rank 0 only",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample, "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("each step is one timed call sequence of the reference's public API on the "
                 "bounded sample named in cpu_baseline.sample (value = sample points / measured "
                 "seconds, no extrapolation); warm-up steps jit-compile on a tiny instance"),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1 or args.slab:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    from paper_2005_03246_b200 import _lib

    _lib.load_library()
    w = make_workload(args.workload)
    if args.slab and hasattr(w, "slab"):
        w.slab = True
    w.shard(rank, world)
    w.to_device()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        w.step()
    barrier()

    # ---- timed region: device-resident inputs (launch profiler off) ----------------------
    clocks = ClockSampler(local)
    clocks.start()
    stream = torch.cuda.current_stream()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        w.step()
    ev1.record(stream)
    barrier()
    ms_total = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    # ---- per-kernel shares: the same K steps again with the library's launch profiler (CUDA
    # events around every launch, on the launching stream); reported beside the timing, which
    # stays free of the profiler's per-launch event records
    _lib.profile_enable(True)
    _lib.profile_report()  # clear
    barrier()
    for _ in range(args.steps):
        w.step()
    barrier()
    prof = _lib.profile_report()
    _lib.profile_enable(False)
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = w.n_total / (ms_step / 1e3)

    launches = sum(c for k, (c, _) in prof.items() if k != "lattice_zero")
    peak, peak_src = peaks()
    dom = dominant(prof, w.bytes_per_launch())
    roof = None
    if dom is not None:
        name, cnt, ms, nbytes = dom
        avg_s = ms / cnt / 1e3
        ach = (nbytes / avg_s / 1e9) if nbytes else None
        roof = {"bound": "hbm", "kernel": name, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": (ach / peak) if ach else None,
                "traffic": traffic_lookup(w.name, name),
                "bytes_per_launch": nbytes, "avg_launch_ms": avg_s * 1e3,
                "share_of_step": ms / ms_total, "peak_source": peak_src}
    breakdown = {k: {"launches": c, "ms_total": round(ms, 4),
                     "share": round(ms / ms_total, 4)} for k, (c, ms) in prof.items()}

    # ---- e2e: public API from pinned host buffers, H2D + D2H inside the timed region ------
    e2e = None
    if not args.no_e2e:
        w.to_pinned()
        w.e2e_begin()
        w.step_e2e()
        w.e2e_end()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        w.e2e_begin()
        for i in range(args.e2e_steps):
            w.step_e2e(last=i == args.e2e_steps - 1)
        w.e2e_end()
        e1.record(stream)
        barrier()
        wall = (time.perf_counter() - t0) * 1e3
        ems = torch.tensor([max(e0.elapsed_time(e1), wall)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e_step = float(ems.item()) / args.e2e_steps
        e2e = {"value": w.n_total / (e_step / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": w.h2d_bytes, "d2h_bytes_per_step": w.d2h_bytes,
               "ms_per_step": e_step, "steps": args.e2e_steps, "mode": w.e2e_mode}

    # ---- e2e_numpy: the drop-in call exactly as a reference user makes it (numpy in, numpy
    # out, the library's own pageable copies inside the call), serial, wall clock ----------
    e2e_np = None
    if not args.no_e2e and world == 1 and hasattr(w, "step_numpy"):
        hb, db = w.numpy_prepare()
        w.step_numpy()
        torch.cuda.synchronize()
        k = max(1, args.numpy_steps)
        t0 = time.perf_counter()
        for _ in range(k):
            w.step_numpy()
        torch.cuda.synchronize()
        nsec = (time.perf_counter() - t0) / k
        e2e_np = {"value": w.n_total / nsec, "unit": UNIT, "ms_per_step": nsec * 1e3,
                  "steps": k, "h2d_bytes_per_step": hb, "d2h_bytes_per_step": db,
                  "mode": "drop-in call: numpy arrays in, numpy arrays out, one call after "
                          "another (wall clock)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, secs, used, kind, sample = reference_timing(w, 1)
        cpu = {"value": v, "unit": UNIT, "cores": used, "kind": kind, "sample": sample,
               "seconds": secs, "host_cpus": os.cpu_count()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": w.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded numpy, SURVEY §8d shapes)",
            "config": w.describe(), "parallelism": w.parallelism(world),
            "e2e": e2e, "e2e_numpy": e2e_np, "gpu_launches": int(launches), "roofline": roof,
            "cpu_baseline": cpu, "clocks": clk, "kernels": breakdown,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
    try:
        import torch.distributed as _dist

        if _dist.is_available() and _dist.is_initialized():
            _dist.destroy_process_group()
    except ImportError:
        pass
