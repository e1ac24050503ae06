# ncu evidence for one workload: plain run, launch list, then full capture of selected kernels.
# usage: WL=cfg5b KREGEX='plane_kde|radix_scatter' bash scripts/gpu_ncu.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
WL=${WL:-cfg5b}
CMD="python bench.py --workload $WL --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_$WL.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$WL.csv $CMD > gpurun_out/ncu_launch_$WL.log 2>&1; echo "launch-list rc=$?"
if [ -n "$KREGEX" ]; then
  ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -c ${NCU_COUNT:-4} -o gpurun_out/prof_$WL -f $CMD > gpurun_out/ncu_full_$WL.log 2>&1; echo "full rc=$?"
fi
