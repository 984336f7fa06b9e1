set -x
for e in 1e-7 1e-8; do FC_PHASES=1 timeout 300 python tools/c4_trace.py $e 1024 > gpurun_out/r02ae_phases_$e.txt 2>&1; grep "fc phases" gpurun_out/r02ae_phases_$e.txt | head -24; done
timeout 300 python tools/timeline.py 1024 1e-8 > gpurun_out/r02ae_timeline_1e-8.txt 2>&1; sed -n 3,30p gpurun_out/r02ae_timeline_1e-8.txt
