set -x
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dgemm_dmma_kernel -c 6000 --csv --log-file gpurun_out/r02c_gemm_traffic.csv python tools/one_solve.py 1024 > gpurun_out/r02c_gemm_traffic.log 2>&1
echo "exit $?"; tail -2 gpurun_out/r02c_gemm_traffic.log
python tools/gemm_traffic_summary.py gpurun_out/r02c_gemm_traffic.csv > gpurun_out/r02c_gemm_class_traffic.json; cat gpurun_out/r02c_gemm_class_traffic.json
gzip -f gpurun_out/r02c_gemm_traffic.csv
FC_GEMM_TRACE=1 timeout 300 python tools/gemm_trace.py > gpurun_out/r02c_gemm_trace.txt 2>&1; grep -c "fc gemm" gpurun_out/r02c_gemm_trace.txt
