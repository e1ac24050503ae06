# Round-end evidence: default bench line (e2e + cpu baseline), every workload's bench line,
# launch lists and ncu --set full captures of the top kernels (exported to CSV on the box).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
nvidia-smi > gpurun_out/prof/nvsmi.txt 2>&1
timeout 900 python bench.py > gpurun_out/prof/bench_default.log 2> gpurun_out/prof/bench_default.err; echo "default rc=$?"
for wl in cfg1 cfg2 cfg3 cfg4 cfg5a cfg5b; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_$wl.log 2>&1; echo "bench $wl rc=$?"
done
for spec in ${SPECS:-"cfg5a:part_bin|radix_scatter|plane_count|ecdf_final2d|radix_hist:8" "cfg5b:plane_kde_all|final2d|digit_stage|radix_scatter|part_bin|share_bounds:9" "cfg3:lines_kernel|bin_scatter|rows_kernel|plane2d:5" "cfg4:level2_codes|group_self_kernel|coarse_rows_codes:6" "cfg1:small2d:2" "cfg2:radix_scatter|scan_lookback|rank_:4"}; do
  IFS=: read wl rx cnt <<< "$spec"
  CMD="python bench.py --workload $wl --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$wl.csv $CMD > /dev/null 2>&1; echo "launches $wl rc=$?"
  ncu --set full --clock-control none -k "regex:$rx" -c $cnt -o gpurun_out/prof/full_$wl -f $CMD > gpurun_out/prof/full_$wl.log 2>&1; echo "full $wl rc=$?"
  ncu -i gpurun_out/prof/full_$wl.ncu-rep --page raw --csv > gpurun_out/prof/raw_$wl.csv 2>/dev/null
  rm -f gpurun_out/prof/full_$wl.ncu-rep
done
ls -la gpurun_out/prof
