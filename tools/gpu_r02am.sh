timeout 900 python -m pytest tests/test_gpu_determinism.py -q -x -k streamk 2>&1 | tail -5
