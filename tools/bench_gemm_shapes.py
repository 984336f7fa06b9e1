"""Skinny-GEMM microbenchmark: the projection shapes of the blocked Gram-Schmidt (the DMMA GEMM
class's dominant launches in the C4 solve) timed through fc_dgemm_splitk with CUDA events over
many back-to-back launches (single batch entry; the solve batches 3 modes).
`python tools/bench_gemm_shapes.py`"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_09314_b200.binding import Library  # noqa: E402

L = Library()
ctx = L.context()
n = 1024
shapes = []
for k in (64, 256, 512, 1024):
    shapes.append((0, 0, n, 64, k))      # A -= Q P       (n x 64 x k)
    shapes.append((1, 0, k, 64, n))      # P = Q^T A      (k x 64 x n)
for tA, tB, M, N, K in shapes:
    A = torch.randn(max(M, K) * max(M, K) + 64, dtype=torch.float64, device="cuda")
    B = torch.randn(max(K, N) * max(K, N) + 64, dtype=torch.float64, device="cuda")
    Cm = torch.zeros(M * N + 64, dtype=torch.float64, device="cuda")
    lda = K if tA else M
    ldb = N if tB else K
    best = None
    for sk in (1, 2, 4, 8, 16):
        if K // sk < 32:
            continue
        for _ in range(3):
            ctx.dgemm(tA, tB, M, N, K, 1.0, A, lda, B, ldb, 0.0, Cm, M, splitk=sk)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        e0.record()
        for _ in range(reps):
            ctx.dgemm(tA, tB, M, N, K, 1.0, A, lda, B, ldb, 0.0, Cm, M, splitk=sk)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        tf = 2.0 * M * N * K / (us * 1e-6) / 1e12
        print(json.dumps({"tA": tA, "tB": tB, "M": M, "N": N, "K": K, "splitk": sk, "us": round(us, 2),
                          "tflops": round(tf, 3)}), flush=True)
