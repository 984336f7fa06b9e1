mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py -q -m gpu -x > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['final_rel_res'])"; done
FC_TRACE=1 timeout 300 python tools/one_solve.py > gpurun_out/trace2.log 2>&1
grep -a "fc svd" gpurun_out/trace2.log | awk '{print $(NF)}' | sort -n | uniq -c
grep -a "fc svd" gpurun_out/trace2.log | head -3
