"""GPU (-m gpu): the CholeskyQR2 panel with Householder reconstruction (csrc/cqr.cuh) --
the default panel path since round 2, with the Householder column loop as its fallback.

R with a non-negative diagonal is unique for a full-rank panel, so the blocked QR's R is
compared elementwise with the oracle's dgeqr2 R (whatever panel algorithm produced it);
Q from the reconstructed compact-WY factors must be orthogonal and reproduce the input.
Counters prove which path ran: sdc_schedule_counters panel_cqr_done / panel_cqr_fallback."""
import os

import numpy as np
import pytest
import torch

from _util import orth_err

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def sdc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1011_3077_b200 import api
    return api


def dev(x):
    return torch.as_tensor(np.asfortranarray(x), dtype=torch.float64).cuda().t().contiguous().t()


def handle(sdc, n_max, **env):
    env.setdefault("SDC_CQR", 2)   # CholeskyQR2 on every full-width panel
    old = {k: os.environ.get(k) for k in env}
    try:
        for k, v in env.items():
            os.environ[k] = str(v)
        return sdc.Handle(n_max)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def check_qr(orc, h, s, r_unique=True, r_cols=None):
    m, n = s.shape
    q, r = h.qr(dev(s))
    q, r = q.cpu().numpy(), r.cpu().numpy()
    assert np.all(np.diag(r) >= 0)
    assert orth_err(q) <= 64 * n * EPS
    assert np.linalg.norm(q @ r - s) <= 64 * n * EPS * np.linalg.norm(s)
    if r_unique:
        y, _ = orc.geqr2(s)
        d = np.where(np.diag(y)[:n] < 0, -1.0, 1.0)
        r_o = d[:, None] * np.triu(y[:n, :n])
        c = n if r_cols is None else r_cols      # R's forward error grows with kappa(S(:, :c))
        assert np.allclose(r[:c, :c], r_o[:c, :c], rtol=0, atol=1e-12 * np.abs(r_o).max() * np.sqrt(n))
    return h.schedule_counters(reset=True)


@pytest.mark.parametrize("m,n", [(128, 64), (1000, 300), (2048, 1024), (4096, 2048), (8192, 640),
                                 (12288, 320)])
def test_cqr_panels_r_unique(sdc, orc, m, n):
    # well-conditioned Gaussian panels: every full-width panel is factored by CholeskyQR2
    # (single cluster up to 4096 rows, several clusters above); R equals the oracle's
    h = handle(sdc, max(n, (m + 1) // 2))
    c = check_qr(orc, h, np.random.default_rng(m + 7 * n).standard_normal((m, n)))
    assert c["panel_cqr_tried"] > 0 and c["panel_cqr_done"] == c["panel_cqr_tried"], c
    assert c["panel_cqr_fallback"] == 0, c


def test_cqr_fallback_on_dependent_columns(sdc, orc):
    # column 70 = column 66 + 1e-9 noise: the second panel's Gram is numerically singular,
    # so that panel falls back to the Householder loop (uniformly on every CTA); R stays the
    # oracle's
    m, n = 2048, 256
    g = np.random.default_rng(3)
    s = g.standard_normal((m, n))
    s[:, 70] = s[:, 66] + 1e-9 * g.standard_normal(m)
    h = handle(sdc, 1024)
    c = check_qr(orc, h, s, r_cols=70)   # R beyond column 70 carries kappa ~ 1e9 amplification
    assert c["panel_cqr_fallback"] >= 1 and c["panel_cqr_done"] >= 1, c


def test_cqr_fallback_exact_rank_deficiency(sdc, orc):
    # exactly repeated columns (GRURV's rank-deficient operands look like this): Householder
    # fallback; R is not unique there, so only orthogonality and reconstruction are checked
    m, n = 1024, 192
    g = np.random.default_rng(4)
    s = g.standard_normal((m, n))
    s[:, 100:110] = s[:, 90:100]
    h = handle(sdc, 512)
    c = check_qr(orc, h, s, r_unique=False)
    assert c["panel_cqr_fallback"] >= 1, c


@pytest.mark.parametrize("cqr", [0, 2])
def test_cqr_vs_householder_step_invariants(sdc, orc, cqr):
    # the whole step with and without CholeskyQR2 panels: the oracle's invariants at n = 1024
    from paper_1011_3077_b200 import inputs
    p = inputs.make_config(2)
    h = handle(sdc, 1024, SDC_CQR=cqr)
    Q, _, _, info = h.split(dev(p.A), None, dev(p.V), max_iters=p.max_iters)
    o = orc.split(p.A, None, p.V, None, max_iters=p.max_iters)
    assert (info.r, info.k) == (o.r, o.k) and info.k == 512
    assert abs(info.metric - o.metric) <= 1e-12
    qh = Q.cpu().numpy()
    r = info.r
    assert np.linalg.norm(qh[:, :r] - o.Q[:, :r] @ (o.Q[:, :r].T @ qh[:, :r]), 2) <= 1e-9
    c = h.schedule_counters()
    assert (c["panel_cqr_done"] > 0) == bool(cqr), c


# ---- the same CholeskyQR2 panel as a chain of small kernels (csrc/cqr_split.cuh): the default
# for the tall stack panels that run next to the bulk trailing update at n > 4096; SDC_CQ_SPLIT=2
# forces it on every full-width panel of >= 128 rows so the oracle-sized cases run it ---------
@pytest.mark.parametrize("m,n", [(128, 64), (1000, 300), (2048, 1024), (4096, 2048), (8192, 640),
                                 (12288, 320), (32768, 128)])
def test_cq_split_panels_r_unique(sdc, orc, m, n):
    h = handle(sdc, max(n, (m + 1) // 2, 2049), SDC_CQ_SPLIT=2)
    c = check_qr(orc, h, np.random.default_rng(m + 11 * n).standard_normal((m, n)))
    assert c["panel_cq_split"] >= n // 64 and c["cq_split_breakdowns"] == 0, c


def test_cq_split_breakdown_falls_back(sdc, orc):
    # a numerically dependent column in the second panel: its first Cholesky breaks down, the
    # chain's later stages skip and the single-CTA Householder fallback factors the panel
    m, n = 2048, 256
    g = np.random.default_rng(3)
    s = g.standard_normal((m, n))
    s[:, 70] = s[:, 66] + 1e-9 * g.standard_normal(m)
    h = handle(sdc, 2049, SDC_CQ_SPLIT=2)
    c = check_qr(orc, h, s, r_cols=70)
    assert c["cq_split_breakdowns"] >= 1 and c["panel_cq_split"] == n // 64, c
    # exactly repeated columns: R not unique, orthogonality and reconstruction only
    s = g.standard_normal((1024, 192))
    s[:, 100:110] = s[:, 90:100]
    c = check_qr(orc, h, s, r_unique=False)
    assert c["cq_split_breakdowns"] >= 1, c


def test_cq_split_second_cholesky_breakdown(sdc, orc):
    # kappa(panel) ~ 1e7: chol(G1) passes its pivot test on some columns only barely and Q1 is
    # far from orthonormal, so the breakdown can also come from the second Cholesky (P must
    # still be intact for the fallback); whichever stage breaks, R is the oracle's
    m, n = 4096, 64
    g = np.random.default_rng(9)
    u, _ = np.linalg.qr(g.standard_normal((m, n)))
    w, _ = np.linalg.qr(g.standard_normal((n, n)))
    s = (u * np.logspace(0, -5, n)) @ w.T
    h = handle(sdc, 2049, SDC_CQ_SPLIT=2)
    q, r = h.qr(dev(s))
    q, r = q.cpu().numpy(), r.cpu().numpy()
    assert orth_err(q) <= 64 * n * EPS
    assert np.linalg.norm(q @ r - s) <= 64 * n * EPS * np.linalg.norm(s)


def test_cq_split_step_parity_and_determinism(sdc, orc):
    # config 2's recipe (n = 1024) with every IRS and GRURV panel on the split chain: the
    # oracle's invariants, twice bit-identical.  (GRURV's rank-deficient X = A_p V^T does not break
    # the Cholesky down here: k = 512 is a multiple of the panel width, and a panel of pure
    # rounding noise is well conditioned relative to its own scale.)
    from paper_1011_3077_b200 import inputs
    p = inputs.make_config(2)
    h = handle(sdc, 2049, SDC_CQ_SPLIT=2, SDC_CQR=1)
    outs = []
    for _ in range(2):
        Q, _, _, info = h.split(dev(p.A), None, dev(p.V), max_iters=p.max_iters)
        outs.append((Q.cpu().numpy().copy(), info))
    o = orc.split(p.A, None, p.V, None, max_iters=p.max_iters)
    qh, info = outs[0]
    assert (info.r, info.k) == (o.r, o.k) and info.k == 512
    assert abs(info.metric - o.metric) <= 1e-12
    r = info.r
    assert np.linalg.norm(qh[:, :r] - o.Q[:, :r] @ (o.Q[:, :r].T @ qh[:, :r]), 2) <= 1e-9
    assert orth_err(qh) <= 1e-13 * p.n
    assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1].metric == outs[1][1].metric
    c = h.schedule_counters()
    assert c["panel_cq_split"] > 0, c


def test_cq_split_default_on_tall_stack(sdc, orc):
    # default knobs: the IRS stack panels above 8192 rows of an n = 4352 step take the split chain
    # (look-ahead QR), everything else the cluster kernels; k from the construction, Q orthogonal
    from paper_1011_3077_b200 import inputs
    n = 4352
    p = inputs.make_config(5, n=n)
    h = handle(sdc, n, SDC_CQR=1)
    Q, _, _, info = h.split(dev(p.A), None, dev(p.V), max_iters=3)
    c = h.schedule_counters()
    assert c["panel_cq_split"] >= 3 * (2 * n - 8192) // 64 - 3 and c["cq_split_breakdowns"] == 0, c
    assert c["lookahead_forks"] > 0 and c["panel_mcluster"] > 0, c
    assert orth_err(Q.cpu().numpy()) <= 1e-13 * n
