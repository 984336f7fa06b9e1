set -x
for v in 16 8 4; do
echo "== FC_TRI_CS $v"
FC_TRI_CS=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02qq_bench_$v.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02qq_bench_$v.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'])"
done
timeout 300 python tools/timeline.py 1024 1e-6 > gpurun_out/r02qq_timeline.txt 2>&1; head -40 gpurun_out/r02qq_timeline.txt
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02qq_gpu.txt 2>&1; tail -30 gpurun_out/r02qq_gpu.txt
