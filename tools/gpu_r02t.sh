set -x
timeout 1500 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_truncate_pcg.py tests/test_gpu_caseA.py -q -s --durations=15 > gpurun_out/r02t_parity.txt 2>&1
grep -E "rank history|reldiff|passed|failed|Error|assert|apply-trunc|cp_truncate|fused|C4 eps|cap " gpurun_out/r02t_parity.txt | head -80
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02t_bench.txt 2> gpurun_out/r02t_bench.err
head -c 5000 gpurun_out/r02t_bench.txt; tail -5 gpurun_out/r02t_bench.err
