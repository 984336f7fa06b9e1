set -x
python -m pytest tests/test_gpu_apply.py tests/test_gpu_determinism.py -q -x 2>&1 | tail -1
for v in "X=0" "FC_GEMM_NO_AUTO_SPLIT=1"; do echo "== $v"; env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ii_bench.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02ii_bench.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['roofline']['frac'], d['roofline']['gemm_ms_per_step'], d['roofline']['launches_per_step'], d['iters_per_solve'], d['final_rel_res'])"; done
