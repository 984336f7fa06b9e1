mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_apply.py tests/test_gpu_truncate_pcg.py -q --tb=short > gpurun_out/pytest_apply.log 2>&1
tail -2 gpurun_out/pytest_apply.log
timeout 600 python tools/bench_apply.py > gpurun_out/bench_apply.jsonl 2>&1
python bench.py --steps 3 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
