mkdir -p gpurun_out
FC_TRACE=1 timeout 300 python tools/one_solve.py 1024 > gpurun_out/pr_trace.txt 2>&1; echo "trace exit $?"
grep "bcgs\]\|^rc" gpurun_out/pr_trace.txt | tail -5
timeout 300 python tools/solve_time.py 1024 1e-6 3
FC_BCGS_PRUNE=0 timeout 300 python tools/solve_time.py 1024 1e-6 3
FC_PHASES=1 timeout 300 python tools/solve_time.py 1024 1e-6 1 2>&1 | grep "fc phases" | head -8
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pr_tests.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pr_tests.log
