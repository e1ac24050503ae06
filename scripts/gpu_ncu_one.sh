# one full ncu capture of a kernel + csv exports (raw, details, source with SASS/line mapping)
# usage: WL=cfg5b KREGEX=plane_kde_group bash scripts/gpu_ncu_one.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --workload $WL --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/one_plain_$WL.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -c ${NCU_COUNT:-1} -o gpurun_out/one_$WL -f $CMD > gpurun_out/one_full_$WL.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/one_$WL.ncu-rep --page raw --csv > gpurun_out/one_raw_$WL.csv 2>/dev/null
ncu -i gpurun_out/one_$WL.ncu-rep --page details --csv > gpurun_out/one_details_$WL.csv 2>/dev/null
ncu -i gpurun_out/one_$WL.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/one_source_$WL.csv 2>/dev/null
ls -la gpurun_out/one_*
[ -n "$KEEP_REP" ] || rm -f gpurun_out/one_$WL.ncu-rep
