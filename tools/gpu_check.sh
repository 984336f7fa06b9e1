mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['final_rel_res'], d['ranks_last_iter'])"; done
FC_NO_ORTH_PREFIX=1 timeout 300 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('noprefix', d['value'], d['ms_per_step'], d['final_rel_res'])"
