mkdir -p gpurun_out
timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 || exit 1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r01b.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
python tools/one_solve.py > gpurun_out/plain3.log 2>&1 || exit 1
for spec in "bcgs_block_cluster_kernel 300 1" "tridiag_cluster_kernel 10 1" "slice_svd_kernel 50 1" "dgemm_dmma_kernel 1500 2" "tri_invit_kernel 40 1"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 -o gpurun_out/r01b_$1 python tools/one_solve.py > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
done
