timeout 300 python tools/timeline.py 1024 1e-8 > gpurun_out/r02ai_timeline_1e-8.txt 2>&1; sed -n 3,6p gpurun_out/r02ai_timeline_1e-8.txt; grep "struct_" gpurun_out/r02ai_timeline_1e-8.txt
timeout 900 python -m pytest tests/test_gpu_parity_fullsize.py -q -x 2>&1 | tail -2
