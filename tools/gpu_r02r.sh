set -x
nproc; free -g | head -2
timeout 900 python tools/oracle_c4.py C4 1024 2 > gpurun_out/r02r_oracle_c4.txt 2>&1
timeout 600 python tools/oracle_c4.py C2 128 100 > gpurun_out/r02r_oracle_c2.txt 2>&1
timeout 900 python tools/oracle_c4.py C3a 512 3 > gpurun_out/r02r_oracle_c3a.txt 2>&1
FC_PHASES=1 timeout 300 python tools/c4_trace.py 1e-6 1024 > gpurun_out/r02r_phases_1e6.txt 2>&1
FC_PHASES=1 timeout 300 python tools/c4_trace.py 1e-7 1024 > gpurun_out/r02r_phases_1e7.txt 2>&1
FC_PHASES=1 timeout 300 python tools/c4_trace.py 1e-8 1024 > gpurun_out/r02r_phases_1e8.txt 2>&1
tail -n 25 gpurun_out/r02r_*.txt | cut -c1-400
