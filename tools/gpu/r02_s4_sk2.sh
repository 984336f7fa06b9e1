mkdir -p gpurun_out
for tm in 3 10 30 100; do
FC_SKETCH_TAU=$tm FC_TRACE=1 timeout 300 python tools/one_solve.py 1024 2>&1 | grep "fc sketch" | tail -4
FC_SKETCH_TAU=$tm timeout 300 python tools/solve_time.py 1024 1e-6 3
done
FC_SKETCH=0 timeout 300 python tools/solve_time.py 1024 1e-6 3
