timeout 300 python tools/solve_time.py 1024 1e-6 3
FC_INVIT_GLOBAL=1 timeout 300 python tools/solve_time.py 1024 1e-6 3
timeout 300 python tools/solve_time.py 1024 1e-7 2
FC_INVIT_GLOBAL=1 timeout 300 python tools/solve_time.py 1024 1e-7 2
timeout 600 python tools/timeline.py 1024 1e-6 2>&1 | head -20
