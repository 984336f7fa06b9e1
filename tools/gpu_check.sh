mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_caseA.py -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
FC_TRACE=1 python tools/one_solve.py > gpurun_out/trace.log 2>&1
grep "fc t2c" gpurun_out/trace.log | sort | uniq -c | sort -rn | head -4
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench.jsonl').read().strip().splitlines()[-1])
print(round(d['value'],2), d['step_ms'], round(d['e2e']['value'],2), d['iters_per_solve'])"
