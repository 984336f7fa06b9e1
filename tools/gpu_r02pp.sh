set -x
for tol in 1e-11 1e-12 1e-13; do
echo "== tol $tol"
FC_WBASIS_TOL=$tol timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02pp_bench_$tol.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02pp_bench_$tol.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'])"
FC_WBASIS_TOL=$tol timeout 900 python -m pytest tests/test_gpu_parity_fullsize.py -q -x -s -k "apply_truncate_c4_iterate or fused_vs_plain" 2>&1 | grep "apply-trunc\|passed\|failed\|fused\|plain" | head
done
timeout 1500 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_truncate_pcg.py tests/test_gpu_apply.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02pp_gpu.txt 2>&1; tail -30 gpurun_out/r02pp_gpu.txt
