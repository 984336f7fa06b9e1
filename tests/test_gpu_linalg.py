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


def _graded_psd(N, seed, decay=16.0):
    """Gram-like symmetric PSD matrix: eigenvalues 10^(-decay * i / N), random eigenbasis."""
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((N, N)))
    lam = 10.0 ** (-decay * np.arange(N) / N)
    M = (Q * lam) @ Q.T
    return 0.5 * (M + M.T)


@pytest.mark.parametrize("sizes", [[200, 400, 700], [231, 600, 601, 840], [1000], [17, 841], [96, 97, 440, 441],
                                   [1400, 900], [1500], [3, 4, 5, 31, 32, 33, 64, 65], [100, 150, 215, 216, 217]])
def test_syev_paths(lib, sizes):
    """fc_syev (the truncation's Gram eigensolver) on every tridiagonalisation path: packed
    shared memory (N <= 96), 16-CTA cluster (97..840; FC_TRI_CS=8 / 4: 8-CTA up to 600 / 4-CTA
    up to 440), 16-CTA cluster with the columns in L2 (841..2048), mixed in one batch; the eigenvectors through the polar
    orthonormalisation (host-known ranks).  Eigenvalues within 20 eps ||M|| of LAPACK; the leading 64 eigenvectors
    orthonormal with residual <= 1e-13 ||M||."""
    import torch
    ctx = lib.context()
    mats = [_graded_psd(N, N + i) if i % 2 == 0 else
            (lambda A: 0.5 * (A + A.T))(np.random.default_rng(N).standard_normal((N, N)))
            for i, N in enumerate(sizes)]
    rs = [min(64, N) for N in sizes]
    dev = [torch.tensor(M, device="cuda") for M in mats]
    out = ctx.syev(dev, rs)
    for M, (lam, Y), r in zip(mats, out, rs):
        ref = np.linalg.eigvalsh(M)[::-1]
        nrm = np.abs(ref).max()
        lam = lam.cpu().numpy()
        assert np.max(np.abs(lam - ref)) <= 20 * 2.2e-16 * nrm * np.sqrt(M.shape[0])
        Y = Y.cpu().numpy().T
        assert np.max(np.abs(Y.T @ Y - np.eye(r))) < 1e-12
        res = np.abs(M @ Y - Y * lam[None, :r]).max()
        assert res <= 1e-13 * nrm * np.sqrt(M.shape[0])
