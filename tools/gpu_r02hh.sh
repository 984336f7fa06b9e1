set -x
python -m pytest tests/test_gpu_apply.py -q -x 2>&1 | tail -1
timeout 300 python tools/bench_gemm_shapes.py > gpurun_out/r02hh_gemm_shapes.txt 2>&1; cat gpurun_out/r02hh_gemm_shapes.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02hh_bench.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02hh_bench.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['roofline_apply']['kr_product']['frac'], d['roofline_hbm']['kr_basis']['frac'])"
