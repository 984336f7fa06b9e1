mkdir -p gpurun_out
timeout 300 python tools/one_eps.py 1e-7 > gpurun_out/one_eps.log 2>&1 || { tail -3 gpurun_out/one_eps.log; exit 1; }
cat gpurun_out/one_eps.log
