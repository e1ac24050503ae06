cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for e in 0 1 2 3; do FCG_KDE_EXP=$e python bench.py --workload cfg5b --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/exp_$e.log 2>&1; echo "exp $e rc=$?"; done
python scripts/summarize.py gpurun_out/exp_*.log
