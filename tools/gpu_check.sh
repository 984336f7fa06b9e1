mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_linalg.py -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for c in "C1 32" "C2 128" "C4 1024" "C3a 512" "C3b 512"; do timeout 600 python tools/diag_setup.py $c >> gpurun_out/diag_all.jsonl 2>&1; done
