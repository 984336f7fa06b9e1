mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_caseA.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1 || { tail -30 gpurun_out/pytest_gpu.log; exit 1; }
tail -2 gpurun_out/pytest_gpu.log
FC_TRACE=1 timeout 300 python tools/one_solve.py > gpurun_out/trace.log 2>&1 || { tail -20 gpurun_out/trace.log; exit 1; }
grep -a "\[bcgs\]\|^rc" gpurun_out/trace.log
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 2>gpurun_out/bench.err | tee -a gpurun_out/bench.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'])"; done
FC_BCGS_SEQ=1 timeout 300 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('seq', d['value'], d['ms_per_step'])"
