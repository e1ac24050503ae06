"""Condense an `ncu --page raw --csv` export into one line per captured launch (the metrics the
roofline and DESIGN.md cite) and optionally merge per-kernel DRAM traffic into
profiles/traffic.json.  Usage: python scripts/ncu_summary.py WL raw.csv [--traffic out.json]"""
import csv
import json
import re
import sys
from collections import defaultdict

COLS = [("gpu__time_duration.sum", "ms"), ("dram__bytes_read.sum", "GB"),
        ("dram__bytes_write.sum", "GB"), ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"), ("launch__registers_per_thread", ""),
        ("launch__grid_size", ""), ("launch__block_size", "")]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12,
         "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}


# ncu kernel name -> the launch profiler's scope name (what bench.py's roofline reports)
SCOPES = [(r"^ecdf_final2d", "scan_lines_final"), (r"^final2d", "kde_final_group"),
          (r"^group_gather_packed|^pack_points", "pts_group_gather"), (r"^plane_kde", "plane_kde"), (r"^kde_gather", "kde_materialize"),
          (r"digit_stage", "part_emit"), (r"digit_hist", "part_hist"), (r"^kde_materialize", "kde_materialize"),
          (r"^kde_final_multi", "kde_final_group"), (r"^lines_kernel<\w+, \d, 1>", "scan_lines_final"),
          (r"^lines_kernel", "scan_lines"), (r"^rows_kernel", "scan_rows"),
          (r"^radix_scatter_kernel<.*SegMap, [1-9]", "kde_materialize"),
          (r"^radix_scatter", "radix_scatter"), (r"^radix_hist", "radix_hist"),
          (r"^part_bin", "part_bin"), (r"^plane_count", "plane_count"),
          (r"^bin_scatter_kernel", "bin_scatter_count"), (r"^level2_(self|codes)<0", "pts_level2_block"),
          (r"^level2_(self|codes)<1", "pts_level2_chunk"), (r"^group_gather", "pts_group_gather"),
          (r"^group_psi", "pts_psi"), (r"^scan_(lookback|single)", "scan_i32"),
          (r"^minmax", "minmax")]


def scope(kernel):
    for pat, sc in SCOPES:
        if re.search(pat, kernel):
            return sc
    return kernel


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"(fcg::)?(<unnamed>|\(anonymous namespace\)|unnamed>)::", "", name)
    return name.replace("void ", "").strip()


def main():
    wl = sys.argv[1]
    paths = [a for a in sys.argv[2:] if a.endswith(".csv") and not a.endswith(".json")]
    if "--traffic" in sys.argv:
        paths = [a for a in paths if a != sys.argv[sys.argv.index("--traffic") + 1]]
    out = []
    for path in paths:
        out.extend(read_raw(path))
    emit(wl, out)


def read_raw(path):
    rows = list(csv.reader(open(path)))
    head, units = rows[0], rows[1]
    idx = {c: i for i, c in enumerate(head)}
    out = []
    for r in rows[2:]:
        rec = {"kernel": short(r[idx["Kernel Name"]])}
        for col, want in COLS:
            i = idx.get(col)
            if i is None:
                continue
            v = float(r[i].replace(",", ""))
            u = units[i]
            if want == "ms":
                v = v * SCALE.get(u, 1.0) * 1e3
            elif want == "GB":
                v = v * SCALE.get(u, 1.0) / 1e9
            rec[col] = v
        out.append(rec)
    return out


def emit(wl, out):
    print(f"# {wl}: ncu --set full --clock-control none (per captured launch)")
    print("kernel,ms,dram_read_GB,dram_write_GB,mem_pct,sm_pct,occupancy_pct,regs,grid,block")
    for o in out:
        print(",".join([o["kernel"]] + [f"{o.get(c, float('nan')):.4g}" for c, _ in COLS]))
    if "--traffic" in sys.argv:
        tp = sys.argv[sys.argv.index("--traffic") + 1]
        try:
            tr = json.load(open(tp))
        except FileNotFoundError:
            tr = {}
        acc = defaultdict(list)
        for o in out:
            acc[scope(o["kernel"])].append((o["dram__bytes_read.sum"] + o["dram__bytes_write.sum"]) * 1e9)
        tr[wl] = {k: sum(v) / len(v) for k, v in acc.items()}
        json.dump(tr, open(tp, "w"), indent=1, sort_keys=True)


main()
