# sketched structured basis: trace, timing, parity
mkdir -p gpurun_out
FC_TRACE=1 timeout 300 python tools/one_solve.py 1024 > gpurun_out/sk_trace.txt 2>&1; echo "trace exit $?"
grep "fc sketch" gpurun_out/sk_trace.txt | tail -12; tail -4 gpurun_out/sk_trace.txt
for tm in 1 0.1; do
FC_SKETCH_TAU=$tm FC_TRACE=1 timeout 300 python tools/one_solve.py 1024 2>&1 | grep "fc sketch" | tail -3
done
timeout 600 python tools/timeline.py 1024 1e-6 > gpurun_out/sk_timeline.txt 2>&1; echo "tl exit $?"
head -40 gpurun_out/sk_timeline.txt
FC_SKETCH=0 timeout 600 python tools/timeline.py 1024 1e-6 2>&1 | head -3
timeout 1200 python -m pytest tests -m gpu -x -q -k "truncate or parity or determinism or fullsize or apply" > gpurun_out/sk_tests.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/sk_tests.log
