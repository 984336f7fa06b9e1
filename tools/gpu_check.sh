mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_truncate_pcg.py tests/test_gpu_setup.py -q -m gpu -x 2>&1 | tail -2
python tools/one_solve.py > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/l_solve_warm.csv python tools/one_solve.py > /dev/null 2>&1
echo done
