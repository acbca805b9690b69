"""Test-only helpers (no method arithmetic)."""
import numpy as np


def sin_angle(q1, q2):
    """sin of the largest principal angle between span(q1) and span(q2), both with
    orthonormal columns: ||(I - q2 q2^T) q1||_2 (accurate down to ~1e-16, unlike
    sqrt(1 - sigma_min^2))."""
    q1 = np.asarray(q1)
    q2 = np.asarray(q2)
    return float(np.linalg.norm(q1 - q2 @ (q2.T @ q1), 2))


def orth_err(q):
    n = q.shape[1]
    return float(np.linalg.norm(q.T @ q - np.eye(n)))
