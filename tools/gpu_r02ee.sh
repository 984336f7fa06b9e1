set -x
python -m pytest tests/test_gpu_apply.py tests/test_gpu_truncate_pcg.py tests/test_gpu_determinism.py tests/test_gpu_linalg.py -q -x 2>&1 | tail -2
for e in 1e-6 1e-7 1e-8; do FC_PHASES=1 timeout 300 python tools/c4_trace.py $e 1024 > gpurun_out/r02ee_phases_$e.txt 2>&1; done
grep -h "fc phases\|\"rc\"" gpurun_out/r02ee_phases_*.txt | cut -c1-120 | grep -E "rc|total|dd factor|basis|side Gram|core"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02ee_bench.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02ee_bench.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['roofline']['frac'], d['roofline']['gemm_ms_per_step'], d['roofline_apply']['frac'])"
