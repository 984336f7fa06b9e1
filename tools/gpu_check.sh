mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_linalg.py -q --tb=short -x > gpurun_out/pytest_linalg.log 2>&1
echo "linalg rc=$?"; tail -1 gpurun_out/pytest_linalg.log
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench.jsonl').read().strip().splitlines()[-1])
print(round(d['value'],2), d['step_ms'], round(d['e2e']['value'],2), d['iters_per_solve'], d['gpu_launches'])"
FC_GEMM_TRACE=1 timeout 600 python tools/gemm_trace.py > gpurun_out/gemm_trace.log 2>&1
grep "fc gemm" gpurun_out/gemm_trace.log | head -16; tail -1 gpurun_out/gemm_trace.log
