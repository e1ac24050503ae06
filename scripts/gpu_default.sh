# round-end rehearsal: smoke, full gpu tests, default bench line (with cpu_baseline), reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
[ -n "$SKIP_TESTS" ] || { timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; }
T0=$SECONDS; timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo "bench rc=$? wall=$((SECONDS-T0))s"
T0=$SECONDS; timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo "ref rc=$? wall=$((SECONDS-T0))s"
tail -c 1500 gpurun_out/bench_default.log; echo; tail -c 800 gpurun_out/bench_ref.log
