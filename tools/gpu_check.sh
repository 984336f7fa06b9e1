mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_linalg.py -x -q -m gpu -k syev 2>&1 | tail -1
FC_TRI_CS=16 timeout 300 python -m pytest tests/test_gpu_linalg.py -x -q -m gpu -k syev 2>&1 | tail -1
FC_TRI_CS=4 timeout 300 python -m pytest tests/test_gpu_linalg.py -x -q -m gpu -k syev 2>&1 | tail -1
for cs in 8 16 8 16; do FC_TRI_CS=$cs timeout 300 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('cs$cs', d['value'], d['ms_per_step'])"; done
