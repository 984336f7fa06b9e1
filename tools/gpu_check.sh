mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_full.log 2>&1; tail -2 gpurun_out/pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
rm -f gpurun_out/bench_r01g.jsonl
for i in 1 2 3; do timeout 120 python bench.py --steps 5 --warmup 3 2>gpurun_out/bench.err | tee -a gpurun_out/bench_r01g.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || exit 1; done
