set -x
timeout 900 python -m pytest tests/test_gpu_apply.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02zz_apply_tests.txt 2>&1; tail -3 gpurun_out/r02zz_apply_tests.txt
timeout 1800 python tools/bench_apply.py > gpurun_out/r02zz_c5_sweep.jsonl 2>&1; cut -c1-330 gpurun_out/r02zz_c5_sweep.jsonl
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02zz_bench.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02zz_bench.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['ranks_last_iter'], d['gpu_launches']); print(json.dumps(d['roofline_apply'])[:900])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_big_streamk --launch-skip 2 --launch-count 1 -o gpurun_out/r02zz_streamk python tools/profile_apply.py > gpurun_out/r02zz_ncu.log 2>&1; tail -3 gpurun_out/r02zz_ncu.log
