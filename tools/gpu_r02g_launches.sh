set -x
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 16000 --csv --log-file gpurun_out/r02g_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02g_ncu_bench.log 2>&1
echo "exit $?"
python tools/launch_summary.py gpurun_out/r02g_launches_bench.csv 2>&1 | head -30 > gpurun_out/r02g_launches_bench_summary.txt; cat gpurun_out/r02g_launches_bench_summary.txt
gzip -f gpurun_out/r02g_launches_bench.csv
