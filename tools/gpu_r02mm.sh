set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02mm_gpu.txt 2>&1; tail -3 gpurun_out/r02mm_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02mm_bench.txt 2>gpurun_out/r02mm_bench.err; tail -c 1500 gpurun_out/r02mm_bench.txt
timeout 300 python tools/timeline.py 1024 1e-6 > gpurun_out/r02mm_timeline.txt 2>&1; head -60 gpurun_out/r02mm_timeline.txt
