mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_caseA.py -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench.jsonl').read().strip().splitlines()[-1])
print(round(d['value'],2), d['step_ms'], round(d['e2e']['value'],2), d['iters_per_solve'])"
python tools/one_solve.py > gpurun_out/plain3.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_solve.csv python tools/one_solve.py > /dev/null 2>&1
