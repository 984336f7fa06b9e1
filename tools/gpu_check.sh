mkdir -p gpurun_out
FC_PRECISE_GRAM=1 FC_POOL_RESERVE_MB=60000 timeout 1500 python tools/eps_sweep.py > gpurun_out/eps_sweep_precise.jsonl 2>&1
cat gpurun_out/eps_sweep_precise.jsonl | tail -4
