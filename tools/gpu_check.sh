mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_caseA.py tests/test_gpu_state.py tests/test_gpu_apply.py tests/test_gpu_als.py -q -m gpu -x > gpurun_out/pt.log 2>&1 || { echo "pytest failed/timeout"; tail -15 gpurun_out/pt.log; exit 1; }
tail -1 gpurun_out/pt.log
for i in 1 2 3; do timeout 120 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['final_rel_res'])" || exit 1; done
