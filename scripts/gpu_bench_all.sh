# all bench workloads, short runs (logs into gpurun_out/)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for wl in cfg1 cfg2 cfg3 cfg4 cfg5a cfg5b; do
  timeout 600 python bench.py --workload $wl --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$wl.log 2>&1; echo "$wl rc=$?"
done
