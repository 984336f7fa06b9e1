set -x
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ad_bench.txt 2>gpurun_out/r02ad_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r02ad_bench.txt').read().splitlines()[-1]); print(d['value'], d['time_to_eps_ms']); print(json.dumps(d['roofline_apply_large'])[:1500])"
tail -3 gpurun_out/r02ad_bench.err
