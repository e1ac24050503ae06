# A/B of library variants built into _ab/*.so: alternating bench runs of one workload.
# usage: WL=cfg5b ROUNDS=3 bash scripts/ab_bench.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
WL=${WL:-cfg5b}
for i in $(seq ${ROUNDS:-3}); do
  for so in _ab/*.so; do
    FCG_LIB_PATH=$PWD/$so python bench.py --workload $WL --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.log 2>&1
    python - "$so" <<'PY'
import json, sys
line = [l for l in open("gpurun_out/ab.log") if l.startswith("{")][-1]
d = json.loads(line)
k = d["kernels"]
top = sorted(k.items(), key=lambda kv: -kv[1]["ms_total"])[:4]
print(f"{sys.argv[1]:14s} {d['ms_per_step']:8.3f} ms  frac={d['roofline']['frac']:.3f}  " +
      " ".join(f"{n}={v['ms_total'] / v['launches']:.3f}" for n, v in top))
PY
  done
done
