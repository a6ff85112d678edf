"""Rank study on the device compression: measured per-level ranks of
T_{alpha,N} for N up to 2^17 stay below the paper's eps-qsrank bound B(N, eps/2) (Lemma 3.7,
P:577-582; oracle.compress.qsrank_bound_T), grow at most logarithmically in N (Table 1's
O(log N log 1/eps) shape), and equal the truncated-SVD ranks of the oracle where it can run."""
import numpy as np
import pytest
import torch

from oracle.compress import qsrank_bound_T, level_ranks

gpu = pytest.mark.gpu


def _ranks(n, alpha, tol, leaf=128):
    from paper_1804_05522_b200.hodlr import Hodlr, FDE_COMPRESS_ONLY
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    H = Hodlr(n, alpha, 1.0 / (n + 1), 1.0 / 32, ones, ones, tol, leaf, flags=FDE_COMPRESS_ONLY)
    r = H.ranks()
    H.close()
    return r


@gpu
@pytest.mark.parametrize("alpha,tol", [(1.1, 1e-8), (1.5, 1e-10), (1.9, 1e-12)])
def test_ranks_within_paper_bound_up_to_2e17(alpha, tol):
    prev = 0
    for e in range(9, 18):
        n = 1 << e
        r = _ranks(n, alpha, tol)
        assert max(r) <= qsrank_bound_T(n, tol), (n, r, qsrank_bound_T(n, tol))
        # top-level rank grows at most like log N: +<= 3 per doubling (bound grows ~ +1.8)
        assert r[0] >= prev - 1 and r[0] <= prev + 3 or prev == 0, (n, r[0], prev)
        prev = r[0]


@gpu
@pytest.mark.parametrize("n,alpha,tol", [(1024, 1.3, 1e-8), (2048, 1.7, 1e-12)])
def test_ranks_equal_oracle_svd_ranks(n, alpha, tol):
    assert _ranks(n, alpha, tol) == level_ranks(alpha, n, 128, tol)


@gpu
def test_compress_only_handle_refuses_factor():
    from paper_1804_05522_b200.hodlr import Hodlr, FDE_COMPRESS_ONLY
    from paper_1804_05522_b200._lib import FdeError
    ones = torch.ones(4096, dtype=torch.float64, device="cuda")
    H = Hodlr(4096, 1.5, 1.0 / 4097, 0.1, ones, ones, 1e-10, 128, flags=FDE_COMPRESS_ONLY)
    assert len(H.ranks()) == 5
    with pytest.raises(FdeError) as e:
        H.factor()
    assert e.value.code == 2                         # FDE_EDIM
    H.close()
