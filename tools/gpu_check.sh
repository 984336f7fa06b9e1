mkdir -p gpurun_out
for i in 1 2 3; do
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_v$i.jsonl 2> gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_v$i.jsonl').read().strip().splitlines()[-1])
print(round(d['value'],2), d['step_ms'], round(d['e2e']['value'],2)); print('slow', d['slowest_step_iter_ms'])"
done
