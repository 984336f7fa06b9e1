set -x
FC_TRACE=1 timeout 600 python tools/c4_trace.py 1e-6 > gpurun_out/r02nn_trace.out 2> gpurun_out/r02nn_trace.err
grep -c . gpurun_out/r02nn_trace.err
grep "fc trunc\|fc svd" gpurun_out/r02nn_trace.err | head -400 > gpurun_out/r02nn_trace_basis.txt
timeout 300 python tools/bench_syev.py 100,150,200,250,300,400,500 > gpurun_out/r02nn_syev.txt 2>&1
cat gpurun_out/r02nn_syev.txt
