mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
for i in 1 2 3; do
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench.jsonl').read().strip().splitlines()[-1])
print(round(d['value'],2), d['step_ms'], round(d['e2e']['value'],2), d['iters_per_solve'], d['ranks_last_iter'], d['final_rel_res'])"
done
