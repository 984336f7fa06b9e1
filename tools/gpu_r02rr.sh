set -x
timeout 600 python -m pytest tests/test_gpu_linalg.py -q -x > gpurun_out/r02rr_linalg.txt 2>&1; tail -5 gpurun_out/r02rr_linalg.txt
for v in 1 0; do
FC_TRI_FUSED=$v timeout 300 python tools/bench_syev.py 50,100,150,200,216 > gpurun_out/r02rr_syev_$v.txt 2>&1; cat gpurun_out/r02rr_syev_$v.txt
FC_TRI_FUSED=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02rr_bench_$v.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02rr_bench_$v.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'])"
done
timeout 300 python tools/timeline.py 1024 1e-6 > gpurun_out/r02rr_timeline.txt 2>&1; head -30 gpurun_out/r02rr_timeline.txt
timeout 1500 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_truncate_pcg.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02rr_gpu.txt 2>&1; tail -5 gpurun_out/r02rr_gpu.txt
