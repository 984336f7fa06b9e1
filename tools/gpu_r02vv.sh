set -x
run() { # name, env...
  name=$1; shift
  env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02vv_bench_$name.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02vv_bench_$name.txt').read().splitlines()[-1]); print('$name', d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'])"
}
run rot1 FC_JACOBI_ROT=1
run rot0 FC_JACOBI_ROT=0
for g in 1 0; do
FC_JACOBI_ROT=$g FC_TRACE=1 timeout 600 python tools/c4_trace.py 1e-6 2>&1 | grep "fc svd" | tail -30 > gpurun_out/r02vv_svd_cycles_rot$g.txt; tail -6 gpurun_out/r02vv_svd_cycles_rot$g.txt
done
FC_GEMM_TRACE=1 timeout 300 python tools/gemm_trace.py > gpurun_out/r02vv_gemm_trace.txt 2>&1; tail -60 gpurun_out/r02vv_gemm_trace.txt
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_truncate_pcg.py tests/test_gpu_lr2d.py tests/test_gpu_determinism.py -q -x > gpurun_out/r02vv_gpu.txt 2>&1; tail -3 gpurun_out/r02vv_gpu.txt
