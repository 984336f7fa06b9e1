mkdir -p gpurun_out
for t in 1024 256 512 1024 256 512; do FC_TRI_PACKED_THREADS=$t timeout 300 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('pthr$t', d['value'], d['ms_per_step'])"; done
FC_TRI_PACKED_THREADS=256 timeout 300 python -m pytest tests/test_gpu_linalg.py -q -m gpu -k syev 2>&1 | tail -1
