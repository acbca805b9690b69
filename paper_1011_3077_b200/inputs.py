"""Seeded synthetic inputs for the split step (shared by the oracle tests and the CUDA path).

This module holds NO arithmetic of the method: it only draws random matrices with the
recipes of SURVEY.md §8(d) / DESIGN.md "Input recipe" (numpy PCG64 `default_rng(seed)`,
exact draw order below) and builds the Haar factors V that Alg. 1 lines 1-2 prescribe
("QR of an N(0,1) matrix"), which the ABI takes as inputs.

haar(G) = Q_G * diag(sign(diag R_G))   (reading Q15).

The dense linear algebra of input *preparation* (the Haar QR, A = U T U^T) runs through
numpy/LAPACK on the CPU, or through torch on a CUDA device for the large configs
(`device="cuda"`); it is never timed and never part of the product path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

STOP_FIXED, STOP_RTEST, STOP_E21 = 0, 1, 2


@dataclass
class Problem:
    name: str
    n: int
    A: object          # (n, n) float64, numpy (Fortran order) or torch (column-major view)
    B: object | None   # None => B = I (RNEP)
    V: object
    VL: object | None
    max_iters: int
    tol: float
    stop: int
    expected_k: int | None = None


# ---------------------------------------------------------------------------------------
# linear-algebra helpers for input prep (numpy or torch)
# ---------------------------------------------------------------------------------------
def _haar_np(G: np.ndarray) -> np.ndarray:
    q, r = np.linalg.qr(G)
    d = np.where(np.diag(r) < 0, -1.0, 1.0)
    return np.asfortranarray(q * d[None, :])


def _haar_torch(G, device):
    import torch
    g = torch.as_tensor(G, dtype=torch.float64, device=device)
    q, r = torch.linalg.qr(g)
    d = torch.where(torch.diagonal(r) < 0, -1.0, 1.0).to(q)
    return q * d[None, :]


def haar(G, device=None):
    if device is None or str(device) == "cpu":
        return _haar_np(np.asarray(G, dtype=np.float64))
    return _haar_torch(G, device)


def _finish(x, device):
    """-> Fortran-ordered numpy (cpu) or a column-major torch tensor on `device`
    (strides (1, n): the storage the C ABI expects, PAPER's A(i,j) at offset i + j*n)."""
    if device is None or str(device) == "cpu":
        if not isinstance(x, np.ndarray):
            x = x.cpu().numpy()
        return np.asfortranarray(x, dtype=np.float64)
    import torch
    t = torch.as_tensor(x, dtype=torch.float64, device=device)
    return t.t().contiguous().t()


# ---------------------------------------------------------------------------------------
# recipes (BASELINE.json configs[0..4])
# ---------------------------------------------------------------------------------------
def ginibre(n: int, seed: int, vseed: int, scale: float | None = None, device=None) -> tuple:
    """A_ij ~ N(0, 2/n) (configs 1 and 3): circular law of radius sqrt(2)."""
    s = math.sqrt(2.0 / n) if scale is None else scale
    A = np.random.default_rng(seed).standard_normal((n, n)) * s
    V = haar(np.random.default_rng(vseed).standard_normal((n, n)), device)
    return _finish(A, device), _finish(V, device)


def sym_known(n: int, seed: int, vseed: int, device=None) -> tuple:
    """Config 2: A = U diag(lam) U^T, lam: n/2 in U[0.1,0.9], n/2 in U[1.1,3.0]."""
    g = np.random.default_rng(seed)
    lam_in = g.uniform(0.1, 0.9, n // 2)
    lam_out = g.uniform(1.1, 3.0, n - n // 2)
    U = haar(g.standard_normal((n, n)), device)
    lam = np.concatenate([lam_in, lam_out])
    if device is None or str(device) == "cpu":
        A = (U * lam[None, :]) @ U.T
    else:
        import torch
        lt = torch.as_tensor(lam, device=device)
        A = (U * lt[None, :]) @ U.T
    V = haar(np.random.default_rng(vseed).standard_normal((n, n)), device)
    return _finish(A, device), _finish(V, device), lam


def pencil(n: int, seed_a: int, seed_b: int, vseed: int, vlseed: int, device=None) -> tuple:
    """Config 4: A, B ~ N(0,1) independent (spherical-ensemble pencil)."""
    A = np.random.default_rng(seed_a).standard_normal((n, n))
    B = np.random.default_rng(seed_b).standard_normal((n, n))
    V = haar(np.random.default_rng(vseed).standard_normal((n, n)), device)
    VL = haar(np.random.default_rng(vlseed).standard_normal((n, n)), device)
    return _finish(A, device), _finish(B, device), _finish(V, device), _finish(VL, device)


def schur_known(n: int, seed: int, vseed: int, device=None) -> tuple:
    """Config 5 (reading Q14): A = U T U^T, T real block upper triangular with
    n/2 2x2 blocks [[rho cos phi, rho sin phi], [-rho sin phi, rho cos phi]] on the diagonal
    (first n/4 pairs rho ~ U[0.2,0.8], last n/4 rho ~ U[1.25,5], phi ~ U[0,pi]) and
    strictly-upper entries outside the blocks ~ N(0, 1/n).  Draw order: rho_in, rho_out,
    phi, N, then the Gaussian for U."""
    assert n % 4 == 0
    g = np.random.default_rng(seed)
    rho_in = g.uniform(0.2, 0.8, n // 4)
    rho_out = g.uniform(1.25, 5.0, n // 4)
    phi = g.uniform(0.0, math.pi, n // 2)
    N = g.standard_normal((n, n))
    T = np.triu(N * math.sqrt(1.0 / n), 1)
    del N
    rho = np.concatenate([rho_in, rho_out])
    i = np.arange(n // 2)
    c, s = rho * np.cos(phi), rho * np.sin(phi)
    T[2 * i, 2 * i] = c
    T[2 * i + 1, 2 * i + 1] = c
    T[2 * i, 2 * i + 1] = s
    T[2 * i + 1, 2 * i] = -s
    U = haar(g.standard_normal((n, n)), device)
    if device is None or str(device) == "cpu":
        A = U @ T @ U.T
    else:
        import torch
        Tt = torch.as_tensor(T, device=device)
        A = U @ Tt @ U.T
        del Tt
    V = haar(np.random.default_rng(vseed).standard_normal((n, n)), device)
    eig = np.concatenate([rho_in, rho_in, rho_out, rho_out])
    return _finish(A, device), _finish(V, device), eig


CONFIG_DOC = {
    1: "n=64 Ginibre N(0,2/n) seed 1, B=I, V seed 1001, 12 passes",
    2: "n=1024 U diag(lam) U^T (seed 2), lam 512 in [.1,.9] + 512 in [1.1,3], V seed 1002, 20 passes, k=512",
    3: "n=4096 Ginibre N(0,2/n) seed 3, V seed 1003, stop when ||E21||_1/||A||_1 <= 1e-13 or 30 passes",
    4: "n=8192 pencil A,B ~ N(0,1) seeds 4,5, V_R seed 1004, V_L seed 2004, 30 passes",
    5: "n=16384 A = U T U^T (seed 6), |lam| in [.2,.8] (n/2) and [1.25,5] (n/2), V seed 1006, 30 passes, k=8192",
    6: "singular-value split (f3, PAPER.md:453): A 8192x8192 = U diag(s) W^T (seed 8), s in [.05,.8] (half) "
       "and [1.25,20], rho=1, RSEP step on the order-16384 embedding [[0,A],[A^T,0]], V seed 1008, 30 passes",
}
CONFIG_DOC[9] = ("config 4's pencil (n=8192, seeds 4,5, V_R seed 1004), 30 passes, with the cheaper left "
                 "basis Q_L = Q of QR(A Q_R) (SDC_FLAG_QL_ORTH, f3): no left IRS")
CONFIG_N = {1: 64, 2: 1024, 3: 4096, 4: 8192, 5: 16384, 6: 16384, 9: 8192}


def make_config(cfg: int, n: int | None = None, device=None) -> Problem:
    """BASELINE.json configs[cfg-1] (n overridable for downscaled twins: same recipe+seeds)."""
    n = CONFIG_N[cfg] if n is None else n
    if cfg == 1:
        A, V = ginibre(n, 1, 1001, device=device)
        return Problem("cfg1", n, A, None, V, None, 12, 0.0, STOP_FIXED)
    if cfg == 2:
        A, V, lam = sym_known(n, 2, 1002, device=device)
        return Problem("cfg2", n, A, None, V, None, 20, 0.0, STOP_FIXED,
                       expected_k=int(np.sum(np.abs(lam) < 1)))
    if cfg == 3:
        A, V = ginibre(n, 3, 1003, device=device)
        return Problem("cfg3", n, A, None, V, None, 30, 1e-13, STOP_E21)
    if cfg == 4:
        A, B, V, VL = pencil(n, 4, 5, 1004, 2004, device=device)
        return Problem("cfg4", n, A, B, V, VL, 30, 0.0, STOP_FIXED)
    if cfg == 5:
        A, V, eig = schur_known(n, 6, 1006, device=device)
        return Problem("cfg5", n, A, None, V, None, 30, 0.0, STOP_FIXED,
                       expected_k=int(np.sum(eig < 1)))
    raise ValueError(cfg)


# ---------------------------------------------------------------------------------------
# the paper's numerical experiments (Figures numexp_rand / numexp_hard):
# normal matrices with random eigenvalues under a random orthogonal similarity, split on
# the imaginary axis (half plane Re z < 0).  Real matrices: complex eigenvalues come in
# conjugate pairs, realised as 2x2 blocks [[x, y], [-y, x]] (eigenvalues x +- i y).
# ---------------------------------------------------------------------------------------
def _pairs_block(xs, ys):
    m = len(xs)
    D = np.zeros((2 * m, 2 * m))
    for t, (x, y) in enumerate(zip(xs, ys)):
        D[2 * t, 2 * t] = D[2 * t + 1, 2 * t + 1] = x
        D[2 * t, 2 * t + 1] = y
        D[2 * t + 1, 2 * t] = -y
    return D


def normal_random_eigs(n: int, seed: int, vseed: int, lo: float = -1.5, hi: float = 1.5):
    """E1/E2: Re, Im ~ U[lo, hi] (n//2 conjugate pairs, one real eigenvalue
    if n is odd), A = U D U^T with U Haar.  Returns (A, V, eigenvalues)."""
    g = np.random.default_rng(seed)
    m = n // 2
    xs, ys = g.uniform(lo, hi, m), g.uniform(lo, hi, m)
    D = np.zeros((n, n))
    D[:2 * m, :2 * m] = _pairs_block(xs, ys)
    eig = list(xs + 1j * ys) + list(xs - 1j * ys)
    if n % 2:
        x0 = g.uniform(lo, hi)
        D[n - 1, n - 1] = x0
        eig.append(x0)
    U = haar(g.standard_normal((n, n)))
    A = U @ D @ U.T
    V = haar(np.random.default_rng(vseed).standard_normal((n, n)))
    return _finish(A, None), _finish(V, None), np.array(eig)


def imag_axis_eigs(n: int, seed: int, vseed: int, eps: float = 1e-10):
    """E3: Re lambda = +-eps (random signs), Im ~ U[-1.5, 1.5], orthogonal
    eigenvectors."""
    g = np.random.default_rng(seed)
    m = n // 2
    xs = eps * np.where(g.uniform(size=m) < 0.5, -1.0, 1.0)
    ys = g.uniform(-1.5, 1.5, m)
    D = np.zeros((n, n))
    D[:2 * m, :2 * m] = _pairs_block(xs, ys)
    eig = list(xs + 1j * ys) + list(xs - 1j * ys)
    if n % 2:
        x0 = eps * (1.0 if g.uniform() < 0.5 else -1.0)
        D[n - 1, n - 1] = x0
        eig.append(x0)
    U = haar(g.standard_normal((n, n)))
    V = haar(np.random.default_rng(vseed).standard_normal((n, n)))
    return _finish(U @ D @ U.T, None), _finish(V, None), np.array(eig)


def jordan_case(n: int, seed: int, vseed: int, mu: float = 0.1):
    """E4: n/2 random eigenvalues with negative real part (Re ~ U[-1.5, 0),
    Im ~ U[-1.5, 1.5], conjugate pairs) and one n/2 x n/2 Jordan block at mu, under a random
    orthogonal similarity (non-normal; the imaginary axis meets its pseudospectrum)."""
    g = np.random.default_rng(seed)
    h = n // 2
    m = h // 2
    xs, ys = g.uniform(-1.5, 0.0, m), g.uniform(-1.5, 1.5, m)
    D = np.zeros((n, n))
    D[:2 * m, :2 * m] = _pairs_block(xs, ys)
    J = mu * np.eye(n - h) + np.diag(np.ones(n - h - 1), 1)
    D[h:, h:] = J
    U = haar(g.standard_normal((n, n)))
    V = haar(np.random.default_rng(vseed).standard_normal((n, n)))
    eig = np.array(list(xs + 1j * ys) + list(xs - 1j * ys) + [mu] * (n - h))
    return _finish(U @ D @ U.T, None), _finish(V, None), eig


EXPERIMENTS = {
    "E1": dict(fn=normal_random_eigs, n=100, seed=101, vseed=1101, passes=60),
    "E2": dict(fn=normal_random_eigs, n=1000, seed=102, vseed=1102, passes=60),
    "E3": dict(fn=imag_axis_eigs, n=25, seed=103, vseed=1103, passes=60),
    "E4": dict(fn=jordan_case, n=32, seed=104, vseed=1104, passes=60),
}


# ---------------------------------------------------------------------------------------
# singular-value split: A = U[:, :p] diag(s) W^T with
# Haar U (m x m), W (n x n), p = min(m, n); s log-uniform, half in [.05, .8], half in
# [1.25, 20] (bounded away from rho = 1, like configs[4]'s eigenvalue annuli).
# ---------------------------------------------------------------------------------------
def svd_known(m: int, n: int, seed: int, vseed: int, device=None):
    """-> (A m x n, V (m+n) x (m+n) Haar for the split, U, s, W) with A = U[:, :p] diag(s) W^T."""
    rng = np.random.default_rng(seed)
    p = min(m, n)
    lo = np.exp(rng.uniform(np.log(0.05), np.log(0.8), p // 2))
    hi = np.exp(rng.uniform(np.log(1.25), np.log(20.0), p - p // 2))
    s = rng.permutation(np.concatenate([lo, hi]))
    if device is None or str(device) == "cpu":
        U = haar(rng.standard_normal((m, m)))
        W = haar(rng.standard_normal((n, n)))
        A = (U[:, :p] * s[None, :]) @ W[:, :p].T
        V = haar(np.random.default_rng(vseed).standard_normal((m + n, m + n)))
        return _finish(A, None), _finish(V, None), U, s, W
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    U = haar(torch.randn((m, m), dtype=torch.float64, device=device, generator=g), device)
    W = haar(torch.randn((n, n), dtype=torch.float64, device=device, generator=g), device)
    st = torch.as_tensor(s, dtype=torch.float64, device=device)
    A = (U[:, :p] * st[None, :]) @ W[:, :p].T
    gv = torch.Generator(device=device).manual_seed(vseed)
    V = haar(torch.randn((m + n, m + n), dtype=torch.float64, device=device, generator=gv), device)
    return _finish(A, device), _finish(V, device), U, s, W


# ---------------------------------------------------------------------------------------
# TREVC input: real upper triangular T with
# distinct real eigenvalues T_ii ~ U[-2, 2] and strictly-upper entries ~ N(0, 1/n^2)
# (departure from normality ||N||_F ~ 0.7, so X stays far from overflow at n = 16384).
# ---------------------------------------------------------------------------------------
def tri_known(n: int, seed: int, device=None):
    """-> T (n x n upper triangular)."""
    g = np.random.default_rng(seed)
    d = g.uniform(-2.0, 2.0, n)
    if device is None or str(device) == "cpu":
        T = np.triu(g.standard_normal((n, n)) / n, 1)
        T[np.arange(n), np.arange(n)] = d
        return _finish(T, None)
    import torch
    gt = torch.Generator(device=device).manual_seed(seed)
    T = torch.triu(torch.randn((n, n), dtype=torch.float64, device=device, generator=gt) / n, 1)
    T += torch.diag(torch.as_tensor(d, dtype=torch.float64, device=device))
    return _finish(T, device)
