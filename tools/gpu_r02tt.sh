set -x
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02tt_bench.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02tt_bench.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'])"
FC_BCGS_PREPASS=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02tt_bench_pre1.txt 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02tt_bench_pre1.txt').read().splitlines()[-1]); print('prepass1', d['value'], d['time_to_eps_ms'], d['iters_per_solve'], d['final_rel_res'], d['ranks_last_iter'], d['gpu_launches'])"
FC_TRACE=1 timeout 600 python tools/c4_trace.py 1e-6 2>&1 | grep "fc svd" | tail -30 > gpurun_out/r02tt_svd_cycles.txt; tail -12 gpurun_out/r02tt_svd_cycles.txt
timeout 600 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_truncate_pcg.py tests/test_gpu_lr2d.py -q -x > gpurun_out/r02tt_gpu.txt 2>&1; tail -3 gpurun_out/r02tt_gpu.txt
timeout 1200 python tools/sweep_apply_splitk.py > gpurun_out/r02tt_apply_splitk.jsonl 2> gpurun_out/r02tt_apply_splitk.err; wc -l gpurun_out/r02tt_apply_splitk.jsonl
