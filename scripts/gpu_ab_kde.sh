# A/B of the one-write sparse plane kernel against the dense two-pass kernel + KDE parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_grid_gpu.py -m gpu -q -x -k "kde" > gpurun_out/pytest_kde.log 2>&1; echo "pytest sparse rc=$?"; tail -1 gpurun_out/pytest_kde.log
for R in ${ROWS:-3}; do
FCG_SPARSE_ROWS=$R timeout 600 python bench.py --workload cfg5b --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_sparse_$R.log 2>&1; echo "sparse $R rc=$?"
done
[ -n "$DENSE" ] && FCG_KDE_DENSE=1 FCG_SPARSE_ROWS=6 timeout 600 python bench.py --workload cfg5b --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_dense.log 2>&1
python scripts/summarize.py gpurun_out/ab_*.log
