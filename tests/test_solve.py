"""CPU test of the CG driver (paper_1812_08075_b200/solve.py) on a plain SPD matrix (no GPU)."""
import numpy as np
import torch

from paper_1812_08075_b200 import solve


def test_cg_on_spd_matrix():
    rng = np.random.default_rng(3)
    B = rng.standard_normal((40, 40))
    A = torch.from_numpy(B @ B.T + 40 * np.eye(40))
    xs = torch.from_numpy(rng.standard_normal(40))
    b = A @ xs
    res = solve.cg(lambda v: A @ v, b, rtol=1e-14, maxiter=200)
    assert res.converged and res.iterations <= 40
    assert torch.allclose(res.x, xs, rtol=0, atol=1e-10)


def test_solve_residual_affine_operator():
    """solve_residual: R(x) = A x - b -> CG on A x = -R(0) reaches the root of R."""
    rng = np.random.default_rng(4)
    B = rng.standard_normal((25, 25))
    A = torch.from_numpy(B @ B.T + 25 * np.eye(25))
    b = torch.from_numpy(rng.standard_normal(25))

    class Op:
        def apply(self, x, out=None):
            y = A @ x - b
            if out is not None:
                out.copy_(y)
                return out
            return y

    res = solve.solve_residual(Op(), 25, device="cpu", rtol=1e-14)
    assert res.converged
    assert torch.allclose(A @ res.x, b, rtol=0, atol=1e-10)
