python -m pytest tests/test_gpu_determinism.py -q -x 2>&1 | tail -15
python -m pytest tests/test_gpu_determinism.py -q 2>&1 | tail -15
FC_GEMM_TRACE=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02c_bench.txt 2> gpurun_out/r02c_gemm_trace.txt
head -c 600 gpurun_out/r02c_bench.txt
