set -x
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 16000 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ncu_bench.log 2>&1
echo "exit $?"
wc -l gpurun_out/r02_launches_bench.csv
python tools/launch_summary.py gpurun_out/r02_launches_bench.csv 2>&1 | head -30
