"""GPU parity (-m gpu) of the singular-value split sdc_svd_split (SURVEY §8(f)
row f3) against the oracle's orc_svd_split: k, r exact; principal angle of span Q(:,1:r)
<= 1e-9; |metric difference| <= 1e-12; ||Q^T Q - I||_F <= 1e-13 N; Ahat symmetric.
Full size (m = n = 4096, N = 8192): properties that hold at any size (k against the
construction, the right singular subspace of the small singular values)."""
import numpy as np
import pytest
import torch

from _util import orth_err, sin_angle
from paper_1011_3077_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def handle():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1011_3077_b200 import api
    return api.Handle(1024)


def api_error():
    from paper_1011_3077_b200._lib import SdcError
    return SdcError


def dev(x):
    return torch.as_tensor(np.asfortranarray(x), dtype=torch.float64).cuda().t().contiguous().t()


@pytest.mark.parametrize("m,n,passes", [(40, 40, 30), (72, 50, 30), (50, 72, 30), (300, 261, 30)])
def test_svd_parity(orc, handle, m, n, passes):
    A, V, U, s, W = inputs.svd_known(m, n, 60 + m, 160 + n)
    Q, Ah, info = handle.svd_split(dev(A), 1.0, dev(V), max_iters=passes, want_ahat=True)
    o = orc.svd_split(A, 1.0, V, max_iters=passes)
    N = m + n
    assert (info.k, info.r) == (o.k, o.r) == (N - o.r, o.r)
    assert info.k == 2 * int(np.sum(s < 1)) + abs(m - n)
    assert abs(info.metric - o.metric) <= 1e-12
    q = Q.cpu().numpy()
    assert orth_err(q) <= 1e-13 * N
    assert sin_angle(q[:, :info.r], o.Q[:, :o.r]) <= 1e-9
    ah = Ah.cpu().numpy()
    assert np.array_equal(ah, ah.T)


def test_svd_edge_cases(orc, handle):
    # 1 x 1 and 1 x n: the smallest embeddings (N = 2, N = n + 1)
    for m, n in [(1, 1), (1, 7)]:
        A = np.full((m, n), 0.5)
        V = inputs.haar(np.random.default_rng(m + n).standard_normal((m + n, m + n)))
        Q, _, info = handle.svd_split(dev(A), 1.0, dev(V), max_iters=12)
        o = orc.svd_split(A, 1.0, V, max_iters=12)
        assert (info.k, info.r, info.status) == (o.k, o.r, o.status)


def test_svd_argument_errors(handle):
    A = torch.zeros((4, 4), dtype=torch.float64, device="cuda")
    V = torch.eye(8, dtype=torch.float64, device="cuda")
    with pytest.raises(api_error()):
        handle.svd_split(A, 0.0, V)          # rho must be > 0
    with pytest.raises(api_error()):
        handle.svd_split(torch.zeros((600, 600), dtype=torch.float64, device="cuda"), 1.0,
                         torch.eye(1200, dtype=torch.float64, device="cuda"))   # m + n > n_max


@pytest.mark.slow
def test_svd_fullsize_properties():
    from paper_1011_3077_b200 import api
    m = n = 4096
    h = api.Handle(m + n)
    A, V, U, s, W = inputs.svd_known(m, n, 7, 107, device="cuda")
    Q, _, info = h.svd_split(A, 1.0, V, max_iters=30)
    small = torch.as_tensor(s < 1, device="cuda")
    assert info.k == 2 * int(small.sum())
    assert info.status == 0 and info.metric <= 1e-10
    # rows m.. of the inside block span exactly the right singular vectors with s < 1
    inside_bottom = Q[m:, info.r:]
    Wsmall = W[:, small]
    resid = inside_bottom - Wsmall @ (Wsmall.T @ inside_bottom)
    assert float(torch.linalg.matrix_norm(resid, 2)) <= 1e-8
