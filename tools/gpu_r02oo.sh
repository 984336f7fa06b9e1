set -x
for v in 1 0; do
FC_BASIS_WEIGHT=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02oo_bench_w$v.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02oo_bench_w$v.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'])"
done
FC_PHASES=1 timeout 300 python tools/c4_trace.py 1e-6 > gpurun_out/r02oo_phases.txt 2>&1; cat gpurun_out/r02oo_phases.txt | cut -c1-400
FC_TRACE=1 timeout 600 python tools/c4_trace.py 1e-6 2>&1 | grep "fc trunc" | tail -60 > gpurun_out/r02oo_basis.txt; tail -24 gpurun_out/r02oo_basis.txt
timeout 1500 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_truncate_pcg.py tests/test_gpu_apply.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02oo_gpu.txt 2>&1; tail -30 gpurun_out/r02oo_gpu.txt
