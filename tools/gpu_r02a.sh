set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/c4_trace.py 1e-6 1024 --twice > gpurun_out/r02a_c4_1e6.txt 2>&1
FC_GEMM_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02a_bench.txt 2> gpurun_out/r02a_gemm_trace.txt
FC_TRACE=1 timeout 600 python tools/c4_trace.py 1e-8 1024 > gpurun_out/r02a_c4_1e8.txt 2> gpurun_out/r02a_c4_1e8_trace.txt
timeout 300 python tools/c4_trace.py 1e-7 1024 > gpurun_out/r02a_c4_1e7.txt 2>&1
tail -3 gpurun_out/*.txt
