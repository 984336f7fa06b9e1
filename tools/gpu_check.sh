mkdir -p gpurun_out
FC_INVIT_SOLVES=2 timeout 1200 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_truncate_pcg.py tests/test_gpu_caseA.py tests/test_gpu_fullsize.py -q -m gpu > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
for v in 2 3 2 3; do FC_INVIT_SOLVES=$v timeout 300 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('solves$v', d['value'], d['ms_per_step'], d['final_rel_res'])"; done
