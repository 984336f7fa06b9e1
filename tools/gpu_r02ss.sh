set -x
run() { # name, env...
  name=$1; shift
  env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ss_bench_$name.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02ss_bench_$name.txt').read().splitlines()[-1]); print('$name', d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'])"
}
run f0_q0 FC_TRI_FUSED=0 FC_JACOBI_QUAD=0
run f0_q8 FC_TRI_FUSED=0
run f0_q7 FC_TRI_FUSED=0 FC_JACOBI_QUAD=1e-7
run f96_q8 FC_TRI_FUSED_MAX=96
run f128_q8 FC_TRI_FUSED_MAX=128
run f160_q8 FC_TRI_FUSED_MAX=160
FC_TRI_FUSED=0 FC_TRACE=1 timeout 600 python tools/c4_trace.py 1e-6 2>&1 | grep "fc svd" | grep -o "sweeps [0-9]*" | sort | uniq -c
FC_TRI_FUSED=0 timeout 1500 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_truncate_pcg.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py tests/test_gpu_lr2d.py -q -x > gpurun_out/r02ss_gpu.txt 2>&1; tail -5 gpurun_out/r02ss_gpu.txt
