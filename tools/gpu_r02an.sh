set -x
cap() { # name regex skip count
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 --launch-count $4 -o gpurun_out/r02f_$1 python tools/one_solve.py 1024 > gpurun_out/r02f_ncu_$1.log 2>&1; tail -1 gpurun_out/r02f_ncu_$1.log
}
cap gemm dgemm_dmma_kernel 1500 6
cap slice slice_svd_qrj_kernel 45 1
cap tridiag tridiag_cluster_kernel 25 1
cap bcgs bcgs_block_cluster_kernel 120 1
ls -la gpurun_out/*.ncu-rep
