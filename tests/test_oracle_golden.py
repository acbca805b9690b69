"""The oracle against the golden fixtures (tests/golden/*.txt): values the paper
and its companion spec print or fix for worked examples, each line citing its
passage.  CPU only (-m "not gpu").  Every fixture line must have a checker here."""
import os

import numpy as np
import pytest

from paper_1011_3077_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _cases(fname):
    out = {}
    for line in open(os.path.join(GOLDEN, fname)):
        line = line.split("#", 1)[0].strip() if line.lstrip().startswith("#") else line.strip()
        if not line:
            continue
        name, inp, exp, cite = (f.strip() for f in line.split("|", 3))
        out[name] = (inp, exp, cite)
    return out


SPEC = _cases("spec_worked_examples.txt")
EXPS = _cases("paper_experiments.txt")


def haar(n, seed):
    return inputs.haar(np.random.default_rng(seed).standard_normal((n, n)))


def check_qr_3_4(orc):
    _, r = orc.qr_signed(np.array([[3.0], [4.0]]))
    assert r[0, 0] == pytest.approx(5.0, rel=1e-15)


def check_qr_identity4(orc):
    q, r = orc.qr_signed(np.eye(4))
    assert np.array_equal(r, np.eye(4)) and np.allclose(np.abs(q), np.eye(4), atol=0)


def check_select_1_0_1_1(orc):
    r, met, _ = orc.split_select(np.array([[1.0, 0.0], [1.0, 1.0]]), 2.0)
    assert (r, met) == (1, 0.5)


def check_select_blocktri4(orc):
    a = np.arange(1.0, 17.0).reshape(4, 4)
    a[2:, :2] = 0.0
    r, met, _ = orc.split_select(a, np.abs(a).sum(axis=0).max())
    assert (r, met) == (2, 0.0)


def check_irs_diag_2_half(orc):
    a, b = np.diag([2.0, 0.5]), np.eye(2)
    for j in range(1, 5):
        a, b, _ = orc.irs_pass(a, b)
        lam = np.sort(np.linalg.eigvals(np.linalg.solve(a, b)).real)
        want = np.sort([2.0 ** (-(2 ** j)), 2.0 ** (2 ** j)])
        assert np.allclose(lam, want, rtol=1e-12, atol=0)


def check_irs_b_zero(orc):
    a, b = np.random.default_rng(5).standard_normal((6, 6)), np.zeros((6, 6))
    for _ in range(4):
        a, b, _ = orc.irs_pass(a, b)
        assert np.linalg.norm(b) == 0.0


def check_step_diag_4_qtr(orc):
    res = orc.split(np.diag([4.0, 0.25]), V=haar(2, 31), max_iters=10)
    assert res.r == 1 and abs(res.Ahat[0, 0]) == pytest.approx(4.0, rel=1e-12)


def check_step_diag_2_half(orc):
    res = orc.split(np.diag([2.0, 0.5]), V=haar(2, 32), max_iters=12)
    assert res.k == 1 and res.metric <= 1e-12


def check_step_identity_pen(orc):
    res = orc.split(np.eye(3), B=np.eye(3), V=haar(3, 33), VL=haar(3, 34), max_iters=20)
    assert res.status == orc.STATUS_NO_SPLIT


def _monitor(orc, name, passes):
    e = inputs.EXPERIMENTS[name]
    A, V, eig = e["fn"](e["n"], e["seed"], e["vseed"])
    res = orc.split(A, V=V, max_iters=passes, tol=0.0, stop=orc.STOP_E21,
                    region=orc.REGION_HALFPLANE, param=0.0)
    return res, res.hist[:, 1], eig


def _first_at_floor(hist):
    h = hist[~np.isnan(hist)]
    return 1 + int(np.argmax(h <= 100 * np.min(h)))


def check_E1(orc):
    res, h, eig = _monitor(orc, "E1", 16)
    assert res.k == int(np.sum(eig.real < 0)) and np.nanmin(h) <= 1e-11
    return _first_at_floor(h)


def check_E2(orc):
    # n = 1000 in the oracle: 16 full splits (~1 min on 8 cores) -- same-iteration landmark
    res, h, eig = _monitor(orc, "E2", 16)
    assert res.k == int(np.sum(eig.real < 0)) and np.nanmin(h) <= 1e-10
    assert abs(_first_at_floor(h) - check_E1(orc)) <= 6


def check_E3(orc):
    res, h, eig = _monitor(orc, "E3", 45)
    assert res.k == int(np.sum(eig.real < 0))
    assert _first_at_floor(h) <= 40 and np.nanmin(h) <= 1e-10
    assert np.all(h[:30] > 1e-3)     # much slower than E1 (eigenvalues 1e-10 from the line)


def check_E4(orc):
    res, h, _ = _monitor(orc, "E4", 60)
    assert res.status == orc.STATUS_NO_SPLIT and np.nanmin(h[20:]) > 1e-6


@pytest.mark.parametrize("name", sorted(SPEC))
def test_spec_worked_example(orc, name):
    globals()["check_" + name](orc)


@pytest.mark.parametrize("name", sorted(EXPS))
def test_paper_experiment_landmark(orc, name):
    globals()["check_" + name](orc)


def test_every_fixture_has_a_checker():
    for name in list(SPEC) + list(EXPS):
        assert "check_" + name in globals(), name
