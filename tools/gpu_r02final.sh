set -x
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02e_gpu.txt 2>&1; tail -3 gpurun_out/r02e_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02e_bench.txt 2> gpurun_out/r02e_bench.err; tail -c 700 gpurun_out/r02e_bench.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02e_bench_reference.txt 2> gpurun_out/r02e_bench_reference.err; tail -c 600 gpurun_out/r02e_bench_reference.txt
timeout 300 python tools/timeline.py 1024 1e-6 > gpurun_out/r02e_timeline.txt 2>&1; sed -n 3,12p gpurun_out/r02e_timeline.txt; tail -3 gpurun_out/r02e_timeline.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 16000 --csv --log-file gpurun_out/r02e_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02e_ncu_bench.log 2>&1
echo "exit $?"
wc -l gpurun_out/r02e_launches_bench.csv
python tools/launch_summary.py gpurun_out/r02e_launches_bench.csv 2>&1 | head -30 > gpurun_out/r02e_launches_bench_summary.txt; cat gpurun_out/r02e_launches_bench_summary.txt
gzip -f gpurun_out/r02e_launches_bench.csv
