"""GPU unit tests of the dense building blocks behind the truncation: the rank-revealing
orthonormalisation (fc_orthonormalize) against NumPy's SVD rank and orthogonality."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p,rank", [(64, 40, 40), (1024, 272, 80), (1024, 300, 300), (200, 512, 200),
                                      (1024, 96, 33)])
def test_orthonormalize(lib, n, p, rank):
    import torch
    ctx = lib.context()
    rng = np.random.default_rng(n + p)
    K = rng.standard_normal((n, rank)) @ rng.standard_normal((rank, p))
    K *= np.logspace(0, -6, p)[None, :]          # widely varying column norms
    A = torch.tensor(np.ascontiguousarray(K.T), device="cuda")
    Q = ctx.orthonormalize(A, 1e-13).cpu().numpy().T
    assert Q.shape[1] == rank
    assert np.max(np.abs(Q.T @ Q - np.eye(Q.shape[1]))) < 1e-13
    R = Q.T @ K
    assert np.linalg.norm(K - Q @ R, axis=0).max() <= 1e-12 * np.linalg.norm(K, axis=0).max()
