for v in 512 640 768 896 1024; do
FC_SLICE_THREADS=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ao_bench_$v.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02ao_bench_$v.txt').read().splitlines()[-1]); print('slice_threads=$v', d['value'], d['time_to_eps_ms'], d['final_rel_res'])"
done
