timeout 900 python -m pytest tests/test_points_gpu.py tests/test_distributed_gpu.py -m gpu -q -x 2>&1 | tail -2
python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4.log 2>&1; python scripts/summarize.py gpurun_out/b4.log
for pt in 1 4 16; do
  FCG_SMALL_PER_THREAD=$pt python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b1_$pt.log 2>&1 && \
  FCG_SMALL_PER_THREAD=$pt ncu --metrics gpu__time_duration.sum --clock-control none -k regex:small2d -c 5 --csv python bench.py --workload cfg1 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep small2d | awk -F'","' '{print $NF}' | tr '\n' ' '; echo " <- per_thread $pt"
done
python scripts/summarize.py gpurun_out/b1_*.log
