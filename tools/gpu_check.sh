mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_apply.py -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
tail -c 300 gpurun_out/bench.err
