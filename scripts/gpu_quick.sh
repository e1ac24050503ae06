# quick loop: selected tests + selected bench workloads
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests} -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for wl in ${WLS:-cfg5a cfg5b}; do
  timeout 600 python bench.py --workload $wl --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$wl.log 2>&1; echo "$wl rc=$?"
done
python scripts/summarize.py gpurun_out/bench_*.log
