set -x
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r02aa_gpu.txt 2>&1; tail -15 gpurun_out/r02aa_gpu.txt
timeout 600 python tools/bench_apply.py > gpurun_out/r02aa_c5.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/r02aa_c5.jsonl'):
    d=json.loads(l); print(d['n'],d['R'],d['r'],round(d['inv_kernel_ms'],4),round(d['inv_frac_dmma'],3), d.get('trunc_ms'), d.get('trunc_tucker'), d.get('trunc_rank'), str(d.get('trunc',''))[:60])"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02aa_bench.txt 2> gpurun_out/r02aa_bench.err; tail -c 3000 gpurun_out/r02aa_bench.txt
ncu --set full --import-source on --clock-control none -k regex:dgemm_big --launch-count 1 -o gpurun_out/r02aa_inv python tools/profile_apply.py > gpurun_out/r02aa_ncu.log 2>&1; tail -2 gpurun_out/r02aa_ncu.log
