set -x
for v in 1 0; do
FC_STREAMK=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ak_bench_$v.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02ak_bench_$v.txt').read().splitlines()[-1]); print('streamk=$v', d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'], d['roofline']['frac'])"
done
timeout 1500 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_determinism.py tests/test_gpu_truncate_pcg.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02ak_gpu.txt 2>&1; tail -3 gpurun_out/r02ak_gpu.txt
