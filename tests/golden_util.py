"""Digest and projection helpers shared by the golden generator and tests."""

import hashlib

import numpy as np


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def probe_vectors(n, count=3, seed=1234):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal(n) for _ in range(count)]


def operator_checksums(A):
    """u_k^T A v_k for seeded vectors: storage-independent operator pins."""
    n = A.shape[0]
    us = probe_vectors(n, 3, 1234)
    vs = probe_vectors(n, 3, 4321)
    return [float(u @ (A @ v)) for u, v in zip(us, vs)]


def vector_checksums(x):
    return [float(np.linalg.norm(x))] + [float(p @ x) for p in probe_vectors(len(x), 2, 99)]
