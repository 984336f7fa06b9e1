mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_linalg.py -q --tb=short > gpurun_out/pytest_linalg.log 2>&1
tail -1 gpurun_out/pytest_linalg.log
python - <<'PY' > gpurun_out/replay_dev.txt 2>&1
import numpy as np, torch, sys
sys.path.insert(0,'.')
from paper_2006_09314_b200.binding import Library
raw = open('gpurun_out/kdump.bin','rb').read()
n, q = np.frombuffer(raw[:8], dtype=np.int32)
K = np.frombuffer(raw[8:], dtype=np.float64).reshape(q, n).T.copy()
ctx = Library().context()
Q = ctx.orthonormalize(torch.tensor(np.ascontiguousarray(K.T), device='cuda'), 1e-13).cpu().numpy().T
print("device basis", Q.shape[1], "orth %.2e" % np.max(np.abs(Q.T@Q - np.eye(Q.shape[1]))), "capture %.2e" % (np.linalg.norm(K-Q@(Q.T@K))/np.linalg.norm(K)))
PY
FC_TRACE=1 timeout 300 python tools/diag_setup.py C4 1024 > gpurun_out/diag.jsonl 2> gpurun_out/trace_c4.txt
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 6000 --csv --log-file gpurun_out/launches_c4.csv python tools/diag_setup.py C4 1024 > /dev/null 2>&1
