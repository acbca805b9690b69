"""Cached ORACLE results for the full-code-path twins (test infrastructure only).

The parity cases that exercise the code paths of the full-size configs (multi-cluster
panels, look-ahead, two pencil chains, the literal monitor protocol) need oracle runs of
minutes.  `tools/make_oracle_cache.py` runs the oracle (and nothing else: `oracle/` +
the seeded input generators) once per case and stores, under tests/golden/oracle_cache/:

  * the input identity: SHA-256 of every input matrix plus 512 sampled entries of each;
  * the oracle's outputs: r, k, metric, metric_fro, iters, converged, status, hist;
  * subspace sketches Z = Q(:,1:r) (Q(:,1:r)^T Omega) (and Z_L for Q_L) with a seeded
    Gaussian Omega of 10 columns (SURVEY §8(c) "ship subspace sketches, not Q").

`case(name)` regenerates the inputs and returns the cached result when the inputs are
bit-identical (digest), or equal to within 1e-13 relative on the stored samples (another
CPU's BLAS may round the input preparation differently: an O(eps) input change moves the
oracle's outputs far less than the parity tolerances); otherwise it runs the oracle live.
Nothing here ever reads the CUDA path.

sin(largest principal angle) from sketches: for the orthogonal projectors P, P' onto the
two r-dimensional subspaces, ||P - P'||_2 = sin of the largest angle, and for Gaussian
Omega with s columns ||E||_2 <= 10 sqrt(2/pi) max_i ||E omega_i|| with probability
>= 1 - 10^-s (Halko-Martinsson-Tropp 2011, Lemma 4.1), E = P - P'.
"""
from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE_DIR = os.path.join(HERE, "golden", "oracle_cache")
SKETCH_COLS = 10
SKETCH_FACTOR = 10.0 * np.sqrt(2.0 / np.pi)


@dataclass
class Case:
    name: str
    cfg: int
    n: int
    max_iters: int
    tol: float
    stop: int
    flags: int = 0
    doc: str = ""


# the twins (SURVEY §8(c) "downscaled twins ... with full oracle parity")
CASES = {
    "cfg5_n2304": Case("cfg5_n2304", 5, 2304, 30, 0.0, 0,
                       doc="configs[4] recipe at n=2304: 4608-row stacks -> multi-cluster panels, "
                           "look-ahead QR, 30 passes"),
    "cfg4_n1024": Case("cfg4_n1024", 4, 1024, 30, 0.0, 0,
                       doc="configs[3] pencil recipe at n=1024: Alg. 4, both chains, 30 + 30 passes"),
    "cfg3_n1024_tol13": Case("cfg3_n1024_tol13", 3, 1024, 30, 1e-13, 2,
                             doc="configs[2] literal protocol (E21 stop at 1e-13, cap 30) at n=1024"),
    "cfg2_n2048_p12": Case("cfg2_n2048_p12", 2, 2048, 12, 0.0, 0,
                           doc="configs[1] recipe at n=2048, 12 passes (forced multi-cluster panels)"),
}


def problem(c: Case):
    from paper_1011_3077_b200 import inputs
    p = inputs.make_config(c.cfg, n=c.n)
    p.max_iters, p.tol, p.stop = c.max_iters, c.tol, c.stop
    return p


def _inputs(p):
    return {k: v for k, v in (("A", p.A), ("B", p.B), ("V", p.V), ("VL", p.VL)) if v is not None}


def _digest(x):
    return hashlib.sha256(np.asfortranarray(x).tobytes(order="F")).hexdigest()


def _sample_idx(n, seed=12345, count=512):
    g = np.random.default_rng(seed)
    return g.integers(0, n, count), g.integers(0, n, count)


def omega(n, seed=777):
    return np.random.default_rng(seed).standard_normal((n, SKETCH_COLS))


def sketch(Q, r, om):
    q = np.asarray(Q)[:, :r]
    return q @ (q.T @ om)


def sketch_sin_bound(Z1, Z2):
    """Upper bound (probability >= 1 - 1e-10) on sin of the largest principal angle."""
    return float(SKETCH_FACTOR * np.max(np.linalg.norm(Z1 - Z2, axis=0)))


def run_oracle(c: Case, p=None):
    import oracle
    p = problem(c) if p is None else p
    o = oracle.split(p.A, p.B, p.V, p.VL, max_iters=c.max_iters, tol=c.tol, stop=c.stop, flags=c.flags)
    return p, o


def make(name: str) -> str:
    """Run the oracle for one case and write its cache file (tools/make_oracle_cache.py)."""
    c = CASES[name]
    p, o = run_oracle(c)
    om = omega(c.n)
    rows, cols = _sample_idx(c.n)
    rec = {"name": name, "n": c.n, "r": o.r, "k": o.k, "metric": o.metric,
           "metric_fro": o.metric_fro, "iters": o.iters, "converged": o.converged,
           "status": o.status, "hist": o.hist, "Z": sketch(o.Q, o.r, om)}
    if o.QL is not None:
        rec["ZL"] = sketch(o.QL, o.r, om)
    for k, v in _inputs(p).items():
        rec["digest_" + k] = _digest(v)
        rec["sample_" + k] = np.asarray(v)[rows, cols]
    os.makedirs(CACHE_DIR, exist_ok=True)
    path = os.path.join(CACHE_DIR, name + ".npz")
    np.savez_compressed(path, **rec)
    return path


@dataclass
class Ref:
    """The oracle's result for a case: from the cache ('exact' / 'eps') or a live run ('live')."""
    p: object
    r: int
    k: int
    metric: float
    metric_fro: float
    iters: int
    converged: int
    status: int
    hist: np.ndarray
    Z: np.ndarray
    ZL: np.ndarray | None
    source: str
    Q: np.ndarray | None = None
    QL: np.ndarray | None = None


def case(name: str) -> Ref:
    c = CASES[name]
    p = problem(c)
    path = os.path.join(CACHE_DIR, name + ".npz")
    source = None
    if os.path.exists(path):
        d = np.load(path)
        ins = _inputs(p)
        if all(d["digest_" + k] == _digest(v) for k, v in ins.items()):
            source = "exact"
        else:
            rows, cols = _sample_idx(c.n)
            ok = all(np.max(np.abs(np.asarray(v)[rows, cols] - d["sample_" + k]))
                     <= 1e-13 * max(1.0, np.max(np.abs(d["sample_" + k]))) for k, v in ins.items())
            source = "eps" if ok else None
        if source:
            return Ref(p, int(d["r"]), int(d["k"]), float(d["metric"]), float(d["metric_fro"]),
                       int(d["iters"]), int(d["converged"]), int(d["status"]), d["hist"], d["Z"],
                       d["ZL"] if "ZL" in d else None, source)
    p, o = run_oracle(c, p)
    om = omega(c.n)
    return Ref(p, o.r, o.k, o.metric, o.metric_fro, o.iters, o.converged, o.status, o.hist,
               sketch(o.Q, o.r, om), None if o.QL is None else sketch(o.QL, o.r, om), "live",
               o.Q, o.QL)
