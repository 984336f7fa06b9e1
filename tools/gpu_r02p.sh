timeout 120 python tools/diag_bcgs_dump.py scratch/kdump.npy
python -m pytest tests/test_gpu_linalg.py -q -x 2>&1 | tail -2
for e in 1e-5 1e-6 1e-7 1e-8; do timeout 600 python tools/c4_trace.py $e 1024 | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['eps'], d['rc'], d['iters'], round(d['time_ms'],1), d['rel_res'][-1], d['rank_R'][-1])"; done
