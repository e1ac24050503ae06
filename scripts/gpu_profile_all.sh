# ncu evidence for every workload's top kernels: launch list + one full capture, exported on
# the box to compact CSVs (raw/details pages) so the copy-back stays small.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # $1 workload, $2 kernel regex, $3 count
  WL=$1 KREGEX="$2" NCU_COUNT=$3 bash scripts/gpu_ncu.sh
  if [ -f gpurun_out/prof_$1.ncu-rep ]; then
    ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$1.csv 2>/dev/null
    ncu -i gpurun_out/prof_$1.ncu-rep --page details --csv > gpurun_out/ncu_details_$1.csv 2>/dev/null
    [ -n "$KEEP_REP" ] || rm -f gpurun_out/prof_$1.ncu-rep
  fi
}
for spec in ${SPECS:-"cfg5a:radix_scatter|part_bin|plane_count|lines_kernel:6" "cfg5b:plane_kde|kde_final_multi|kde_materialize|lines_kernel:6" "cfg3:lines_kernel|bin_scatter|rows_kernel:5" "cfg4:level2_self|group_gather|radix_scatter:5" "cfg1:lines_kernel|bin_scatter|rows_kernel:4" "cfg2:radix_scatter|scan_|rank_:4"}; do
  IFS=: read wl rx cnt <<< "$spec"
  run "$wl" "$rx" "$cnt"
done
ls -la gpurun_out
