mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_linalg.py -q --tb=short -x > gpurun_out/pytest_linalg.log 2>&1
echo "linalg rc=$?"; tail -1 gpurun_out/pytest_linalg.log
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_caseA.py -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
for w in 128 64; do
FC_BCGS_W=$w timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_w$w.jsonl 2> gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_w$w.jsonl').read().strip().splitlines()[-1])
print('W=$w', round(d['value'],2), d['step_ms'], round(d['e2e']['value'],2), d['gpu_launches'], round(d['roofline']['achieved'],2), round(d['roofline']['share_of_step'],3))"
done
