set -x
python -m pytest tests/test_gpu_linalg.py tests/test_gpu_determinism.py tests/test_gpu_apply.py -q -x -s 2>&1 | grep -E "C5 n=|passed|failed|Error" | tail -8
for e in 1e-5 1e-6 1e-7 1e-8; do timeout 300 python tools/c4_trace.py $e 1024 --twice > gpurun_out/r02bb_c4_$e.txt 2>&1; done
for e in 1e-5 1e-6 1e-7 1e-8; do python -c "
import json
ls=[json.loads(l) for l in open('gpurun_out/r02bb_c4_$e.txt') if l.startswith('{')]
print('$e', [(d.get('rc'), d.get('iters'), round(d['time_ms'],1)) for d in ls if 'time_ms' in d], ls[-1])" | cut -c1-200; done
FC_PHASES=1 timeout 300 python tools/c4_trace.py 1e-8 1024 > gpurun_out/r02bb_phases_1e-8.txt 2>&1
grep -h "fc phases" gpurun_out/r02bb_phases_1e-8.txt | head -8
