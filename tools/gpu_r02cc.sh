set -x
ncu --set full --import-source on --clock-control none -k regex:dgemm_dmma_kernel --launch-skip 400 --launch-count 6 -o gpurun_out/r02cc_small python tools/one_solve.py 1024 > gpurun_out/r02cc_ncu.log 2>&1; tail -2 gpurun_out/r02cc_ncu.log
