import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built CUDA library")
    config.addinivalue_line("markers", "slow: oracle work of tens of seconds")


@pytest.fixture(scope="session")
def ora():
    import oracle
    oracle.build()
    return oracle


def rel_fro(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def qr_signed(X):
    """LAPACK Householder QR (numpy) normalised to diag(R) > 0: the unique thin QR."""
    Q, R = np.linalg.qr(np.asarray(X, np.float64))
    d = np.sign(np.diag(R)); d[d == 0] = 1.0
    return Q * d, R * d[:, None]


def orth_err(Q):
    """||Q^T Q - I||_F with 4096-row chunked BLAS Gram + pairwise chunk sum."""
    Q = np.asarray(Q, np.float64)
    m, n = Q.shape
    parts = [Q[i:i + 4096].T @ Q[i:i + 4096] for i in range(0, m, 4096)]
    while len(parts) > 1:
        parts = [parts[i] + parts[i + 1] if i + 1 < len(parts) else parts[i] for i in range(0, len(parts), 2)]
    return float(np.linalg.norm(parts[0] - np.eye(n)))


def rel_residual(Q, R, X):
    Q = np.asarray(Q, np.float64); X = np.asarray(X, np.float64)
    num = 0.0; den = 0.0
    for i in range(0, Q.shape[0], 65536):
        d = Q[i:i + 65536] @ R - X[i:i + 65536]
        num += float((d * d).sum()); den += float((X[i:i + 65536] ** 2).sum())
    return (num / den) ** 0.5
