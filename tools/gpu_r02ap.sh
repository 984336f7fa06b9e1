set -x
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ap_bench.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02ap_bench.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'])"
FC_TRACE=1 timeout 600 python tools/c4_trace.py 1e-6 2>&1 | grep "fc svd" | tail -4
timeout 1500 python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_lr2d.py tests/test_gpu_parity_fullsize.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02ap_gpu.txt 2>&1; tail -3 gpurun_out/r02ap_gpu.txt
