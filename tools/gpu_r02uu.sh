set -x
run() { # name, env...
  name=$1; shift
  env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02uu_bench_$name.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02uu_bench_$name.txt').read().splitlines()[-1]); print('$name', d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'])"
}
run g8 FC_SLICE_G=8
run g4 FC_SLICE_G=4
run g16 FC_SLICE_G=16
run g8_t384 FC_SLICE_G=8 FC_SLICE_THREADS=384
run g8_t256 FC_SLICE_G=8 FC_SLICE_THREADS=256
for g in 8 4; do
FC_SLICE_G=$g FC_TRACE=1 timeout 600 python tools/c4_trace.py 1e-6 2>&1 | grep "fc svd" | tail -30 > gpurun_out/r02uu_svd_cycles_g$g.txt; tail -6 gpurun_out/r02uu_svd_cycles_g$g.txt
done
timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_truncate_pcg.py tests/test_gpu_lr2d.py tests/test_gpu_determinism.py -q -x > gpurun_out/r02uu_gpu.txt 2>&1; tail -3 gpurun_out/r02uu_gpu.txt
