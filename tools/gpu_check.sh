mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lr2d.py tests/test_gpu_truncate_pcg.py tests/test_gpu_als.py -q -m gpu -x -s > gpurun_out/pt.log 2>&1 || { echo "pytest failed/timeout"; tail -15 gpurun_out/pt.log; exit 1; }
grep "2D n=1024" gpurun_out/pt.log; tail -1 gpurun_out/pt.log
for i in 1 2; do timeout 120 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['final_rel_res'])" || exit 1; done
