set -x
timeout 1500 python -m pytest tests -m gpu -q -x -s --durations=25 > gpurun_out/r02v_gpu.txt 2>&1
grep -E "rank history|reldiff|passed|failed|Error|assert|apply-trunc|cp_truncate|fused|C4 eps|S0|Z0|s call|cap " gpurun_out/r02v_gpu.txt | head -80
FC_GEMM_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02v_bench.txt 2> gpurun_out/r02v_gemm_trace.txt
grep "fc gemm" gpurun_out/r02v_gemm_trace.txt | head -40
python -c "import json;d=json.loads(open('gpurun_out/r02v_bench.txt').read().splitlines()[-1]);print(d['value'],d['roofline_hbm'])"
