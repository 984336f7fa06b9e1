set -x
python -m pytest tests/test_gpu_apply.py tests/test_gpu_truncate_pcg.py tests/test_gpu_determinism.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02gg_bench.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02gg_bench.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['roofline_apply']['kr_product'], d['roofline_hbm']['kr_basis'])"
