timeout 300 python tools/timeline.py 1024 1e-8 > gpurun_out/r02ah_timeline_1e-8.txt 2>&1; sed -n 3,16p gpurun_out/r02ah_timeline_1e-8.txt; grep "struct_" gpurun_out/r02ah_timeline_1e-8.txt
