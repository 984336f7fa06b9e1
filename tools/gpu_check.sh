mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1 || { tail -30 gpurun_out/pytest_gpu.log; exit 1; }
tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 2>gpurun_out/bench.err | tee -a gpurun_out/bench.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'])"; done
FC_ORTH_CGS2=1 timeout 300 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('cgs2', d['value'], d['ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_solve.csv python tools/one_solve.py > /dev/null 2>&1
