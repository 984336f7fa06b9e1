python -m pytest tests/test_gpu_apply.py -q -x -k splitk 2>&1 | tail -2
FC_GEMM_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/r02e_bench.txt 2> gpurun_out/r02e_gemm_trace.txt
head -c 300 gpurun_out/r02e_bench.txt; echo
timeout 900 python tools/diag_trunc_err.py 1024 > gpurun_out/r02e_trunc_err.txt 2>&1
cat gpurun_out/r02e_trunc_err.txt
