set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02jj_gpu.txt 2>&1; tail -3 gpurun_out/r02jj_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for e in 1e-5 1e-6 1e-7 1e-8; do timeout 300 python tools/c4_trace.py $e 1024 --twice > gpurun_out/r02jj_c4_$e.txt 2>&1; done
for e in 1e-5 1e-6 1e-7 1e-8; do python -c "
import json
ls=[json.loads(l) for l in open('gpurun_out/r02jj_c4_$e.txt') if l.startswith('{')]
print('$e', [(d.get('rc'), d.get('iters'), round(d['time_ms'],1)) for d in ls if 'time_ms' in d], ls[-1])"; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02jj_bench.txt 2> gpurun_out/r02jj_bench.err; tail -c 400 gpurun_out/r02jj_bench.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02jj_ref.txt 2>&1; tail -c 600 gpurun_out/r02jj_ref.txt
