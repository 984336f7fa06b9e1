mkdir -p gpurun_out
timeout 300 python tools/diag_setup.py C3b 2048 nosolve > gpurun_out/diag.jsonl 2>&1
timeout 300 python tools/diag_setup.py C1 32 >> gpurun_out/diag.jsonl 2>&1
timeout 300 python tools/diag_setup.py C2 128 >> gpurun_out/diag.jsonl 2>&1
timeout 600 python tools/diag_setup.py C4 1024 >> gpurun_out/diag.jsonl 2>&1
timeout 600 python tools/diag_setup.py C3a 512 >> gpurun_out/diag.jsonl 2>&1
