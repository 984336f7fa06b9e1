# real-run timeline of one warm C4 solve (CUPTI via torch.profiler) + per-truncation trace
mkdir -p gpurun_out
timeout 600 python tools/timeline.py 1024 1e-6 > gpurun_out/s4_timeline.txt 2>&1; echo "tl exit $?"
cat gpurun_out/s4_timeline.txt | head -70
FC_TRACE=1 timeout 300 python tools/one_solve.py 1024 > gpurun_out/s4_trace.txt 2>&1; echo "trace exit $?"
grep -c . gpurun_out/s4_trace.txt
