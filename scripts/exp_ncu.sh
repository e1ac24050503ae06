cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for e in ${EXPS:-1 2}; do
  FCG_KDE_EXP=$e ncu --set full --clock-control none --import-source on -k "regex:plane_kde_group" -c 1 -o gpurun_out/exp$e -f python bench.py --workload cfg5b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/expncu_$e.log 2>&1; echo "ncu $e rc=$?"
  ncu -i gpurun_out/exp$e.ncu-rep --page details --csv > gpurun_out/exp_details_$e.csv 2>/dev/null
  ncu -i gpurun_out/exp$e.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/exp_source_$e.csv 2>/dev/null
  ncu -i gpurun_out/exp$e.ncu-rep --page raw --csv > gpurun_out/exp_raw_$e.csv 2>/dev/null
  rm -f gpurun_out/exp$e.ncu-rep
done
