mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_caseA.py tests/test_gpu_fullsize.py tests/test_gpu_state.py -q -m gpu -x 2>&1 | tail -3
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['final_rel_res'], d['iters_per_solve'])"; done
FC_NO_CORE_DOT=1 timeout 300 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('nocore', d['value'], d['ms_per_step'], d['final_rel_res'])"
