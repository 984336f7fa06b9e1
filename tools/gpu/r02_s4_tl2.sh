mkdir -p gpurun_out
timeout 600 python tools/timeline.py 1024 1e-6 > gpurun_out/s4_timeline.txt 2>&1; echo "tl exit $?"
head -50 gpurun_out/s4_timeline.txt
FC_GEMM_TRACE=1 timeout 300 python tools/gemm_trace.py > gpurun_out/s4_gemm_trace.txt 2>&1; echo "gt exit $?"
head -45 gpurun_out/s4_gemm_trace.txt
