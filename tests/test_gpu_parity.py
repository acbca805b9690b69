"""GPU parity tests (-m gpu): libsdc (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Criteria (north_star):
  k and r bit-exact; largest principal angle between span Q(:,1:r) <= 1e-9;
  |metric_gpu - metric_oracle| <= 1e-12; ||Q^T Q - I||_F <= 1e-13 n.
Elementwise Q / A_j / B_j are not unique between two correct implementations (DESIGN.md
"parity unpinned"), so only invariants are compared.
"""
import numpy as np
import pytest
import torch

from _util import orth_err, sin_angle
from paper_1011_3077_b200 import inputs

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def sdc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1011_3077_b200 import api
    return api


@pytest.fixture(scope="module")
def handle(sdc):
    return sdc.Handle(1024, pencil=True)


def dev(x):
    return torch.as_tensor(np.asfortranarray(x), dtype=torch.float64).cuda().t().contiguous().t()


def host(x):
    return x.cpu().numpy()


# ---------------------------------------------------------------------------------------
# building blocks
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1)])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (64, 64, 64), (65, 130, 33),
                                   (300, 257, 129), (129, 700, 64), (64, 515, 1000)])
def test_dgemm_vs_oracle(orc, handle, ta, tb, M, N, K):
    g = np.random.default_rng(M * 7 + N * 3 + K)
    a = g.standard_normal((K, M) if ta else (M, K))
    b = g.standard_normal((N, K) if tb else (K, N))
    c0 = g.standard_normal((M, N))
    ref = -0.5 * orc.gemm(a, b, bool(ta), bool(tb)) + 2.0 * c0
    c = dev(c0)
    handle.dgemm(dev(a), dev(b), bool(ta), bool(tb), alpha=-0.5, beta=2.0, C=c)
    # fp64 products summed in a different order: |err| <= K eps sum|a||b| (+ beta term)
    bound = (K + 2) * EPS * (0.5 * orc.gemm(np.abs(a), np.abs(b), bool(ta), bool(tb)) + 2 * np.abs(c0))
    assert np.all(np.abs(host(c) - ref) <= bound + 1e-300)


def test_dgemm_odd_leading_dims(orc, handle):
    # ld odd -> 8-byte cp.async path; submatrix views with ld > rows
    g = np.random.default_rng(9)
    big_a = dev(g.standard_normal((101, 77)))
    big_b = dev(g.standard_normal((91, 59)))
    a = big_a[:37, :29]
    b = big_b[:29, :41]
    c = handle.dgemm(a, b)
    ref = orc.gemm(host(a), host(b))
    assert np.allclose(host(c), ref, rtol=0, atol=64 * EPS * 29 * 8)


@pytest.mark.parametrize("m,n", [(2, 1), (16, 8), (130, 65), (400, 200), (600, 300), (2048, 1024)])
def test_blocked_qr_vs_oracle(orc, handle, m, n):
    # R with diag >= 0 is unique for full-rank input: compare to the oracle elementwise;
    # Q: reconstruction and orthogonality (SPEC.md:127-128 invariants)
    s = np.random.default_rng(m + n).standard_normal((m, n))
    q, r = handle.qr(dev(s))
    q, r = host(q), host(r)
    _, r_o = orc.qr_signed(s)
    assert np.allclose(r, r_o, rtol=0, atol=1e-12 * np.abs(r_o).max() * np.sqrt(n))
    assert np.linalg.norm(q @ r - s) <= 64 * n * EPS * np.linalg.norm(s)
    assert orth_err(q) <= 64 * n * EPS


@pytest.mark.parametrize("n", [3, 64, 100, 257])
def test_irs_pass_vs_oracle(orc, handle, n):
    # R_j unique (= chol); A_{j+1}^{-1} B_{j+1} = (A_j^{-1} B_j)^2 is basis-invariant
    g = np.random.default_rng(n)
    a = g.standard_normal((n, n)) + 3 * np.eye(n)
    b = g.standard_normal((n, n))
    ao, bo, r = (host(x) for x in handle.irs_pass(dev(a), dev(b)))
    ao_o, bo_o, r_o = orc.irs_pass(a, b)
    assert np.allclose(r, r_o, rtol=0, atol=1e-12 * np.abs(r_o).max())
    m_gpu = np.linalg.solve(ao, bo)
    m_ora = np.linalg.solve(ao_o, bo_o)
    # both equal (A^{-1}B)^2 up to rounding amplified by the conditioning of A_{j+1}
    kappa = np.linalg.cond(ao_o)
    assert np.linalg.norm(m_gpu - m_ora) <= 1e-14 * n * kappa * np.linalg.norm(m_ora)
    # Q12^T B_j = Q22^T A_j means the new pencil is left-equivalent:
    # [A_{j+1}; B_{j+1}] has orthonormal-complement structure -> same singular values
    sv = np.linalg.svd(np.vstack([ao, bo]), compute_uv=False)
    sv_o = np.linalg.svd(np.vstack([ao_o, bo_o]), compute_uv=False)
    assert np.allclose(sv, sv_o, rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("n", [2, 3, 31, 32, 33, 100, 777])
def test_split_select_vs_oracle(orc, handle, n):
    g = np.random.default_rng(100 + n)
    ah = g.standard_normal((n, n)) * np.exp(-np.abs(np.subtract.outer(np.arange(n), np.arange(n))) / 5)
    bh = g.standard_normal((n, n))
    r, met, mv = handle.split_select(dev(ah), 2.5)
    r_o, met_o, mv_o = orc.split_select(ah, 2.5)
    assert r == r_o
    assert abs(met - met_o) <= 1e-14 * max(1.0, abs(met_o))
    assert np.allclose(host(mv)[1:], mv_o, rtol=1e-13, atol=0)
    r, met, _ = handle.split_select(dev(ah), 2.5, dev(bh), 0.75)
    r_o, met_o, _ = orc.split_select(ah, 2.5, bh, 0.75)
    assert r == r_o and abs(met - met_o) <= 1e-13 * max(1.0, met_o)


def test_split_select_ties_smallest(handle):
    t = np.array([[1.0, 0, 0], [1, 1, 0], [0, 1, 1]])
    r, met, _ = handle.split_select(dev(t), 1.0)
    assert (r, met) == (1, 1.0)


# ---------------------------------------------------------------------------------------
# the whole step vs the oracle
# ---------------------------------------------------------------------------------------
def assert_parity(orc_res, Q, info, A, n, ahat=None, sin_tol=1e-9, met_tol=1e-12):
    assert info.r == orc_res.r, (info.r, orc_res.r)
    assert info.k == orc_res.k == n - info.r
    assert abs(info.metric - orc_res.metric) <= met_tol, (info.metric, orc_res.metric)
    Qh = host(Q)
    assert orth_err(Qh) <= 1e-13 * n
    r = info.r
    assert sin_angle(Qh[:, :r], orc_res.Q[:, :r]) <= sin_tol
    if ahat is not None:
        assert np.allclose(host(ahat), Qh.T @ A @ Qh, atol=1e-11 * np.abs(A).max() * np.sqrt(n))


def run_both(orc, handle, p, want_ahat=True):
    Bd = None if p.B is None else dev(p.B)
    VLd = None if p.VL is None else dev(p.VL)
    Q, QL, Ah, info = handle.split(dev(p.A), Bd, dev(p.V), VLd, max_iters=p.max_iters, tol=p.tol,
                                   stop={0: "fixed", 1: "rtest", 2: "e21"}[p.stop], want_ahat=want_ahat)
    o = orc.split(p.A, p.B, p.V, p.VL, max_iters=p.max_iters, tol=p.tol, stop=p.stop)
    return Q, QL, Ah, info, o


def test_config1_parity(orc, handle):
    p = inputs.make_config(1)
    Q, _, Ah, info, o = run_both(orc, handle, p)
    assert_parity(o, Q, info, p.A, p.n, Ah)
    assert info.status == 0 and info.iters == 12
    assert info.k == int(np.sum(np.abs(np.linalg.eigvals(p.A)) < 1))


@pytest.mark.parametrize("n", [2, 3, 5, 8, 25, 32, 100, 200])
def test_edge_sizes_parity(orc, handle, n):
    # ragged sizes (non-multiples of the 64-wide panels / 32-row select tiles)
    p = inputs.make_config(5, n=n) if n % 4 == 0 and n >= 8 else None
    if p is None:
        A, V = inputs.ginibre(n, 50 + n, 1050 + n)
        p = inputs.Problem("edge", n, A, None, V, None, 14, 0.0, 0)
    Q, _, Ah, info, o = run_both(orc, handle, p)
    if o.status == 0:
        assert_parity(o, Q, info, p.A, n, Ah)
    else:
        assert info.status == o.status


def test_config2_parity_full(orc, handle):
    # configs[1] at its full size n=1024: k = 512 exactly
    p = inputs.make_config(2)
    Q, _, Ah, info, o = run_both(orc, handle, p)
    assert_parity(o, Q, info, p.A, p.n, Ah)
    assert info.k == p.expected_k == 512


def test_config3_twin_monitor_parity(orc, handle):
    # configs[2] protocol (split after every pass, stop at metric <= tol) at n=256 with a
    # tolerance both sides can reach; equal pass count p
    p = inputs.make_config(3, n=256)
    p.tol = 1e-11
    Q, _, Ah, info, o = run_both(orc, handle, p)
    assert info.iters == o.iters and info.converged == o.converged
    assert_parity(o, Q, info, p.A, p.n, Ah)


def test_config4_twin_pencil_parity(orc, handle):
    # configs[3] recipe at n=200 (pencil, 30 + 30 passes)
    p = inputs.make_config(4, n=200)
    Q, QL, Ah, info, o = run_both(orc, handle, p)
    assert info.r == o.r and info.k == o.k
    assert abs(info.metric - o.metric) <= 1e-12
    r = info.r
    assert sin_angle(host(Q)[:, :r], o.Q[:, :r]) <= 1e-9
    assert sin_angle(host(QL)[:, :r], o.QL[:, :r]) <= 1e-9
    assert orth_err(host(QL)) <= 1e-13 * p.n


def test_config5_twin_parity(orc, handle):
    p = inputs.make_config(5, n=512)
    Q, _, Ah, info, o = run_both(orc, handle, p)
    assert_parity(o, Q, info, p.A, p.n, Ah)
    assert info.k == p.expected_k == 256


def test_rtest_mode_parity(orc, handle):
    p = inputs.make_config(1)
    p.stop, p.tol, p.max_iters = 1, 1e-6, 40
    Q, _, Ah, info, o = run_both(orc, handle, p)
    assert info.iters == o.iters and info.converged == 1
    assert np.allclose(info.hist[1:info.iters, 2], o.hist[1:o.iters, 2], rtol=1e-6)
    assert_parity(o, Q, info, p.A, p.n, Ah)


def test_explicit_identity_equals_null_b(handle):
    p = inputs.make_config(1)
    Q1, _, _, i1 = handle.split(dev(p.A), None, dev(p.V), max_iters=12)
    Q2, _, _, i2 = handle.split(dev(p.A), dev(np.eye(p.n)), dev(p.V), dev(p.V), max_iters=12)
    assert i1.r == i2.r
    assert sin_angle(host(Q1)[:, :i1.r], host(Q2)[:, :i2.r]) <= 1e-9


def test_nonfinite_input_status(handle):
    p = inputs.make_config(1)
    a = p.A.copy()
    a[3, 5] = np.nan
    _, _, _, info = handle.split(dev(a), None, dev(p.V), max_iters=3)
    assert info.status == 2


def test_no_split_orthogonal(handle):
    q = inputs.haar(np.random.default_rng(5).standard_normal((16, 16)))
    v = inputs.haar(np.random.default_rng(6).standard_normal((16, 16)))
    _, _, _, info = handle.split(dev(q), None, dev(v), max_iters=20)
    assert info.status == 1


def test_argument_errors(sdc, handle):
    p = inputs.make_config(1)
    with pytest.raises(sdc._lib.SdcError):
        handle.split(dev(p.A[:1, :1]), None, dev(p.V[:1, :1]))
    with pytest.raises(sdc._lib.SdcError):
        handle.split(dev(p.A), None, dev(p.V), max_iters=0)


def test_host_path_matches_device_path(handle):
    p = inputs.make_config(1)
    Qd, _, _, i1 = handle.split(dev(p.A), None, dev(p.V), max_iters=12)
    Qh, _, _, i2 = handle.split_host(p.A, None, p.V, max_iters=12)
    assert (i1.r, i1.metric) == (i2.r, i2.metric)
    assert np.array_equal(host(Qd), Qh)   # same kernels, same order: bit-identical


def test_deterministic(handle):
    p = inputs.make_config(1)
    Q1, _, _, i1 = handle.split(dev(p.A), None, dev(p.V), max_iters=12)
    Q2, _, _, i2 = handle.split(dev(p.A), None, dev(p.V), max_iters=12)
    assert i1.metric == i2.metric and torch.equal(Q1, Q2)


def _handle_with_env(sdc, n_max, pencil=False, **env):
    import os
    old = {k: os.environ.get(k) for k in env}
    try:
        for k, v in env.items():
            os.environ[k] = str(v)
        return sdc.Handle(n_max, pencil=pencil)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("nbo", [64, 128, 256])
def test_outer_block_widths_parity(orc, sdc, nbo):
    # two-level blocking (64-wide panels inside nbo-wide compact-WY blocks) at a ragged
    # size: every outer width gives the same invariants as the oracle
    h = _handle_with_env(sdc, 600, SDC_NBO=nbo)
    p = inputs.make_config(2, n=600)
    Q, _, Ah, info, o = run_both(orc, h, p)
    assert_parity(o, Q, info, p.A, p.n, Ah)
    assert info.k == p.expected_k


@pytest.mark.parametrize("la,xp", [(0, 0), (1, 0), (1, 1)])
def test_lookahead_schedule_parity(orc, sdc, la, xp):
    # look-ahead QR (panels on a high-priority stream, bulk trailing updates overlapped on
    # the caller's stream), with and without the cross-pass overlap (pass j+1's first panels
    # next to pass j's products), and the serial order give the oracle's invariants at a
    # ragged n with 4 outer blocks; the R of a 2n x n QR stays the unique diag >= 0 factor
    # SDC_NBO=128: the look-ahead schedule needs outer blocks wider than one panel (at n=900
    # the default width is 64, which runs the serial order) -- the counters prove the fork
    h = _handle_with_env(sdc, 900, SDC_LOOKAHEAD=la, SDC_XPASS=xp, SDC_NBO=128)
    p = inputs.make_config(2, n=900)
    Q, _, Ah, info, o = run_both(orc, h, p)
    c = h.schedule_counters()
    assert (c["lookahead_forks"] > 0) == bool(la), c
    assert (c["xpass_forks"] > 0) == bool(xp), c
    assert_parity(o, Q, info, p.A, p.n, Ah)
    assert info.k == p.expected_k
    s = np.random.default_rng(78).standard_normal((1800, 900))
    q, r = h.qr(dev(s))
    _, r_o = orc.qr_signed(s)
    assert np.allclose(host(r), r_o, rtol=0, atol=1e-12 * np.abs(r_o).max() * np.sqrt(900))
    assert orth_err(host(q)) <= 64 * 900 * EPS


def test_lookahead_graph_replay_matches_direct(sdc):
    # the two-stream look-ahead schedule captured into the step's CUDA graph (fork/join by
    # events) replays bit-identically to the directly launched sequence
    p = inputs.make_config(2, n=800)
    hg = _handle_with_env(sdc, 800, SDC_GRAPH_MAX_N=4096, SDC_LOOKAHEAD=1, SDC_NBO=128)
    hd = _handle_with_env(sdc, 800, SDC_GRAPH_MAX_N=0, SDC_LOOKAHEAD=1, SDC_NBO=128)
    A, V = dev(p.A), dev(p.V)
    Qg = sdc.empty_colmajor(800, 800, A.device)
    Qd = sdc.empty_colmajor(800, 800, A.device)
    _, _, _, ig1 = hg.split(A, None, V, max_iters=6, Q=Qg)
    q1 = Qg.clone()
    _, _, _, ig2 = hg.split(A, None, V, max_iters=6, Q=Qg)
    _, _, _, idd = hd.split(A, None, V, max_iters=6, Q=Qd)
    assert torch.equal(q1, Qg) and torch.equal(Qg, Qd)
    assert ig1.metric == ig2.metric == idd.metric and ig1.r == idd.r
    cg, cd = hg.schedule_counters(), hd.schedule_counters()
    assert cg["lookahead_forks"] > 0 and cg["graph_captures"] == 1 and cg["graph_replays"] == 1, cg
    assert cd["lookahead_forks"] > 0 and cd["graph_captures"] == 0, cd


@pytest.mark.parametrize("cfg,n", [(3, 700), (4, 300)])
def test_second_context_bit_identical(sdc, cfg, n):
    # monitor mode with GRURV(j) on the second context next to IRS pass j+1 (config 3), and
    # the pencil's left IRS / left GRURV concurrent with the right ones (config 4): same
    # kernels on the same inputs as the single-stream order -> bit-identical outputs
    p = inputs.make_config(cfg, n=n)
    outs = []
    for pipe in (0, 1):
        h = _handle_with_env(sdc, n, pencil=p.B is not None, SDC_PIPELINE=pipe)
        Bd = None if p.B is None else dev(p.B)
        VLd = None if p.VL is None else dev(p.VL)
        Q, QL, Ah, info = h.split(dev(p.A), Bd, dev(p.V), VLd, max_iters=p.max_iters, tol=p.tol,
                                  stop={0: "fixed", 1: "rtest", 2: "e21"}[p.stop], want_ahat=True)
        outs.append((Q, QL, Ah, info))
    (q0, l0, a0, i0), (q1, l1, a1, i1) = outs
    assert torch.equal(q0, q1) and torch.equal(a0, a1)
    assert (l0 is None) == (l1 is None) and (l0 is None or torch.equal(l0, l1))
    assert (i0.k, i0.r, i0.iters, i0.metric, i0.status) == (i1.k, i1.r, i1.iters, i1.metric, i1.status)


@pytest.mark.parametrize("rows", [64, 128, 256])
@pytest.mark.parametrize("m,n", [(2048, 1024), (1000, 997), (4096, 300), (129, 64), (70, 70)])
def test_panel_variants_r_unique(orc, sdc, rows, m, n):
    # panels at every rows-per-CTA tier (register variants RPT 8/16/32) give the unique
    # diag >= 0 R of the oracle and an orthogonal Q at ragged sizes
    h = _handle_with_env(sdc, max(m, n), SDC_PANEL_ROWS=rows)
    s = np.random.default_rng(m * 3 + n).standard_normal((m, n))
    q, r = h.qr(dev(s))
    _, r_o = orc.qr_signed(s)
    assert np.allclose(host(r), r_o, rtol=0, atol=1e-12 * np.abs(r_o).max() * np.sqrt(n))
    assert orth_err(host(q)) <= 64 * n * EPS
    assert np.linalg.norm(host(q) @ host(r) - s) <= 64 * n * EPS * np.linalg.norm(s)


def test_second_context_alloc_failure_falls_back(sdc):
    # when the second context does not fit next to the handle's workspace (simulated), the
    # pencil and monitor-mode paths run on the single context with bit-identical results
    p = inputs.make_config(4, n=300)
    outs = []
    for env in ({"SDC_PIPELINE": 0}, {"SDC_ALT_FAIL_ALLOC": 1}):
        h = _handle_with_env(sdc, 300, pencil=True, **env)
        Q, QL, Ah, info = h.split(dev(p.A), dev(p.B), dev(p.V), dev(p.VL), max_iters=12, want_ahat=True)
        Q2, _, _, info2 = h.split(dev(p.A), None, dev(p.V), max_iters=12, tol=1e-13, stop="e21")
        outs.append((Q, QL, info, Q2, info2))
    (a, b, i, c, j), (a2, b2, i2, c2, j2) = outs
    assert torch.equal(a, a2) and torch.equal(b, b2) and torch.equal(c, c2)
    assert (i.k, i.r, i.metric) == (i2.k, i2.r, i2.metric) and (j.k, j.iters) == (j2.k, j2.iters)


def test_blocked_qr_two_level_r_unique(orc, sdc):
    # R of the two-level QR equals the oracle's (unique with diag >= 0) at 2n x n, n = 700
    h = _handle_with_env(sdc, 700, SDC_NBO=256)
    s = np.random.default_rng(77).standard_normal((1400, 700))
    q, r = h.qr(dev(s))
    _, r_o = orc.qr_signed(s)
    assert np.allclose(host(r), r_o, rtol=0, atol=1e-12 * np.abs(r_o).max() * np.sqrt(700))
    assert orth_err(host(q)) <= 64 * 700 * EPS


def test_graph_replay_matches_direct(sdc):
    # the FIXED-mode step captured as one CUDA graph gives bit-identical results to the
    # directly launched sequence, and replays (same pointers) stay identical
    p = inputs.make_config(1)
    hg = _handle_with_env(sdc, 64, SDC_GRAPH_MAX_N=4096)
    hd = _handle_with_env(sdc, 64, SDC_GRAPH_MAX_N=0)
    A, V = dev(p.A), dev(p.V)
    Qg = sdc.empty_colmajor(64, 64, A.device)
    Qd = sdc.empty_colmajor(64, 64, A.device)
    _, _, _, ig1 = hg.split(A, None, V, max_iters=12, Q=Qg)
    q1 = Qg.clone()
    _, _, _, ig2 = hg.split(A, None, V, max_iters=12, Q=Qg)   # replay
    _, _, _, idd = hd.split(A, None, V, max_iters=12, Q=Qd)
    assert torch.equal(q1, Qg) and torch.equal(Qg, Qd)
    assert ig1.metric == ig2.metric == idd.metric and ig1.r == idd.r
    assert hg.launches > 0


@pytest.mark.parametrize("env", [{"SDC_NO_CLUSTER": 1}, {}, {"SDC_PANEL_ROWS": 64},
                                 {"SDC_PANEL_ROWS": 256}])
def test_panel_exchange_modes_parity(orc, sdc, env):
    # cluster/DSMEM panel (small panels) and cooperative-grid/L2 panel give the same
    # invariants on config 2's recipe at n = 600 (the multi-cluster exchange, which needs
    # stacks above 2048 rows, is covered in test_gpu_fullpath.py)
    h = _handle_with_env(sdc, 600, **env)
    p = inputs.make_config(2, n=600)
    Q, _, Ah, info, o = run_both(orc, h, p)
    c = h.schedule_counters()
    if "SDC_NO_CLUSTER" in env:
        assert c["panel_grid"] > 0 and c["panel_cluster"] == 0, c
    else:
        assert c["panel_cluster"] > 0 and c["panel_grid"] == 0, c
    assert_parity(o, Q, info, p.A, p.n, Ah)


# ---------------------------------------------------------------------------------------
# schedule / kernel-variant knobs (DESIGN.md §6 table): every non-default variant the
# library can run gives the oracle's results
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("persist", [0, 1, 2])
def test_forced_gemm_variants_vs_oracle(orc, sdc, variant, persist):
    # SDC_GEMM_VARIANT forces one TMA tile shape for every GEMM (0 128x128, 1 64x128,
    # 2 64x64, 3 128x64 two CTAs/SM, 4 128x128 with the C tile prefetched by TMA) and
    # SDC_PERSIST picks one-tile vs persistent grids; beta = 1 exercises the reduce-add epilogue
    h = _handle_with_env(sdc, 256, SDC_GEMM_VARIANT=variant, SDC_PERSIST=persist)
    for (M, N, K, beta) in [(256, 192, 64, 1.0), (300, 257, 129, 0.5), (128, 640, 512, 0.0)]:
        g = np.random.default_rng(M + N + K + variant)
        a, b, c0 = g.standard_normal((K, M)), g.standard_normal((K, N)), g.standard_normal((M, N))
        ref = orc.gemm(a, b, True, False) + beta * c0
        c = dev(c0)
        h.dgemm(dev(a), dev(b), True, False, alpha=1.0, beta=beta, C=c)
        bound = (K + 2) * EPS * (orc.gemm(np.abs(a), np.abs(b), True, False) + abs(beta) * np.abs(c0))
        assert np.all(np.abs(host(c) - ref) <= bound + 1e-300), (M, N, K)


@pytest.mark.parametrize("env", [{"SDC_PERSIST": 0}, {"SDC_PERSIST": 2}, {"SDC_RED": 0},
                                 {"SDC_SIDE_PERSIST": 1, "SDC_NBO": 128}, {"SDC_PANEL_SMEM": 1},
                                 {"SDC_GEMM_VARIANT": 4}, {"SDC_CQR": 2}, {"SDC_CQR": 0}])
def test_step_variants_parity(orc, sdc, env):
    # the whole step with each non-default kernel variant (persistent grids off / everywhere,
    # load-FMA-store instead of the bulk reduce-add epilogue, persistent side-stream updates,
    # shared-memory panel loop instead of registers) on config 2's recipe at n = 600
    h = _handle_with_env(sdc, 600, **env)
    p = inputs.make_config(2, n=600)
    Q, _, Ah, info, o = run_both(orc, h, p)
    assert_parity(o, Q, info, p.A, p.n, Ah)
    assert info.k == p.expected_k


@pytest.mark.parametrize("n", [777, 778])
def test_odd_n_keeps_tma_gemms(orc, sdc, n):
    # the n x n workspace has ld = n rounded up to even, so an odd-order step stages its GEMM
    # operands by TMA like an even one.  The exceptions: Q22^T B_j reads the complement at row
    # offset n, and the similarity / Q_L products read the caller's A and Q with their own
    # (here odd) leading dimension -- a few percent of the launches (round 1: all of them)
    h = sdc.Handle(n)
    A, V = inputs.ginibre(n, 90 + n, 1090 + n)
    p = inputs.Problem("odd", n, A, None, V, None, 6, 0.0, 0)
    Q, _, Ah, info, o = run_both(orc, h, p)
    c = h.schedule_counters()
    if n % 2:
        assert c["gemm_cpasync"] <= 0.05 * (c["gemm_cpasync"] + c["gemm_tma"]), c
    else:
        assert c["gemm_cpasync"] == 0, c
    if o.status == 0:
        assert_parity(o, Q, info, p.A, n, Ah)
    assert orth_err(host(Q)) <= 1e-13 * n
