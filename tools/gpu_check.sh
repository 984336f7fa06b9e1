mkdir -p gpurun_out
python tools/one_solve.py > gpurun_out/plain.log 2>&1 || exit 1
for spec in "bcgs_block_kernel 300 1" "tridiag_kernel 20 1" "slice_svd_kernel 60 1" "dgemm_big_kernel 150 2" "dgemm_dmma_kernel 1500 2" "tridiag_packed_kernel 40 1"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 -o gpurun_out/r01_$1 python tools/one_solve.py > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
done
