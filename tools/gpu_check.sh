mkdir -p gpurun_out
timeout 900 python tools/diag_apply8.py > gpurun_out/diag_apply8.log 2>&1
FC_NO_OVERLAP=1 timeout 900 python tools/diag_apply8.py >> gpurun_out/diag_apply8.log 2>&1
grep -E "^which|^pcg|Error" gpurun_out/diag_apply8.log | cut -c1-300
