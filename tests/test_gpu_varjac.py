"""GPU parity on the conforming varying-Jacobian mesh (tests/varjac.py): J differs across every face, so
the kernels' per-side J^{-T} (T- record a-, T+ record a+) is exercised where the pinned oracle
(test_oracle_varjac.py) fixes the answer. Checks the CUDA path both against the oracle (random x, full
vector, c = 1 and c(x)) and directly against the closed forms (u = a.x -> 0, u = |x|^2 -> -6 |det J| w_J).
"""
import numpy as np
import pytest

import oracle
import synth
import varjac
from oracle import brute

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


def _op(w, **kw):
    from paper_1812_08075_b200 import Operator
    jac = varjac.jac_planes(w.N, -1, w.N[0] + 2)
    return Operator(w.N, w.k, geom_kind=1, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale, jac=jac, **kw)


# N1, N2 multiples of the k_gen tiles (2 x 4) so that the production kernel (not a fallback) runs
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("coeff", [0, 1])
def test_varjac_parity(k, coeff):
    N = (5, 4, 8) if k <= 4 else (3, 4, 4)
    w = synth.small(k, N, geom_kind=1, coeff_kind=coeff, seed=40 + k)
    op = _op(w)
    assert op.kernel_name == "k_gen"
    x = synth.x_torch(w, device="cuda")
    r = op.apply(x)
    torch.cuda.synchronize()
    ref = oracle.apply(w, x.cpu().numpy(), varjac.jac_cells(N, np.arange(w.ncells)))
    err = np.abs(r.cpu().numpy() - ref).max() / np.abs(ref).max()
    op.close()
    assert err <= TOL, err


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_varjac_consistency_gpu(k):
    N = (5, 6, 8) if k <= 3 else (5, 4, 8)
    w = synth.small(k, N, geom_kind=1, coeff_kind=0, seed=3)
    n = w.n
    xi, wq = brute.gl01(n)
    P = varjac.node_positions(N, n, xi)
    m = varjac.interior_mask(N, n)
    op = _op(w)
    x = torch.from_numpy((0.7 * P[..., 0] - 1.1 * P[..., 1] + 0.4 * P[..., 2]).reshape(-1)).cuda()
    r = op.apply(x).cpu().numpy()
    assert np.abs(r[m]).max() < 1e-11
    x = torch.from_numpy((P ** 2).sum(-1).reshape(-1)).cuda()
    r = op.apply(x).cpu().numpy()
    jac = varjac.jac_cells(N, np.arange(w.ncells))
    j = np.arange(n ** 3)
    wJ = wq[j % n] * wq[(j // n) % n] * wq[j // (n * n)]
    expect = (-6.0 * np.abs(np.linalg.det(jac.reshape(-1, 3, 3)))[:, None] * wJ[None, :]).reshape(-1)
    op.close()
    assert np.abs(r[m] - expect[m]).max() < 1e-11 * np.abs(expect[m]).max() + 1e-13
