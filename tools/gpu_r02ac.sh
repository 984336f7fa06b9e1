set -x
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ac_bench.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02ac_bench.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'], d['roofline']['frac'], d['roofline']['gemm_ms_per_step'])"
timeout 1500 python -m pytest tests/test_gpu_apply.py tests/test_gpu_parity_fullsize.py tests/test_gpu_truncate_pcg.py tests/test_gpu_determinism.py -q -x > gpurun_out/r02ac_gpu.txt 2>&1; tail -3 gpurun_out/r02ac_gpu.txt
