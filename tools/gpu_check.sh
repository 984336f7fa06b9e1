mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_truncate_pcg.py tests/test_gpu_caseA.py tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/pt.log 2>&1 || { echo "pytest failed/timeout"; tail -15 gpurun_out/pt.log; exit 1; }
tail -1 gpurun_out/pt.log
FC_TRACE=1 timeout 120 python tools/one_solve.py > gpurun_out/trace3.log 2>&1; grep -a "in-block Mcycles" gpurun_out/trace3.log
for i in 1 2; do timeout 120 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['final_rel_res'])" || exit 1; done
