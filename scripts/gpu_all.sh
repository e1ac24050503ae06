cd $GRAFT_REPO_ROOT
bash scripts/gpu_tests.sh
bash scripts/gpu_bench_all.sh
