python -m pytest tests/test_gpu_determinism.py tests/test_gpu_apply.py -q -x 2>&1 | tail -3
FC_GEMM_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/r02d_bench.txt 2> gpurun_out/r02d_gemm_trace.txt
FC_GEMM_MAX_SPLIT=64 FC_GEMM_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/r02d_bench64.txt 2> gpurun_out/r02d_gemm_trace64.txt
head -c 400 gpurun_out/r02d_bench.txt; echo; head -c 400 gpurun_out/r02d_bench64.txt
