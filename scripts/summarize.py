"""Print one summary line per bench JSON log (used on gpurun_out/ results)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        print(f, "ERR", open(f).read()[-400:])
        continue
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    frac = r.get("frac")
    print(f"{f}: {d['ms_per_step']:.3f} ms/step {d['value']:.3e} pts/s e2e {e.get('value', 0):.3e} "
          f"dom={r.get('kernel')} frac={frac if frac is None else round(frac, 3)} launches={d.get('gpu_launches')}")
    ks = sorted(d["kernels"].items(), key=lambda kv: -kv[1]["ms_total"])
    print("    ", ", ".join(f"{k}:{v['share']:.2f}" for k, v in ks[:9]))
