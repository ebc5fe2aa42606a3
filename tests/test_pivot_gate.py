"""P9: pivot-free safety of the row-modified sweeps (D12).

The GPU factors M + diag(c) S along the stiffened axis without pivoting.  On the
materials of configs c3 (p=3, nested-ellipsoid phantom, +-5% noise), c4 (p=2,
tissue eps_r ~ U[30,70]) and the c5 recipe (eps_r ~ U[1,80] inside the scalp;
generated at n=64), every sampled fiber of all six row-modified families is
factored here without pivoting (plain numpy, independent of oracle/ and of the
CUDA path) and solved against LAPACK's partially pivoted banded solver.  Gate:
growth factor < 10 and solution difference < 1e-13 (relative).  The matrices
and per-test-function eps^ come from the oracle (pinned by P1/P1d).
"""
import numpy as np
import pytest
from scipy.linalg import solve_banded

import oracle
import workloads


def nopivot_lu_solve(A, f):
    """Dense-storage banded LU without pivoting; returns (x, growth = max|U| / max|A|)."""
    n = A.shape[0]
    U = A.copy()
    L = np.eye(n)
    for k in range(n - 1):
        piv = U[k, k]
        for i in range(k + 1, n):
            if U[i, k] != 0.0:
                L[i, k] = U[i, k] / piv
                U[i, k:] -= L[i, k] * U[k, k:]
    y = np.zeros(n)
    for i in range(n):
        y[i] = f[i] - L[i, :i] @ y[:i]
    x = np.zeros(n)
    for i in range(n - 1, -1, -1):
        x[i] = (y[i] - U[i, i + 1:] @ x[i + 1:]) / U[i, i]
    return x, np.abs(U).max() / np.abs(A).max()


def to_band(A, p):
    n = A.shape[0]
    ab = np.zeros((2 * p + 1, n))
    for i in range(n):
        for j in range(max(0, i - p), min(n, i + p + 1)):
            ab[p + i - j, j] = A[i, j]
    return ab


@pytest.mark.parametrize("name,n,p,material", [("c3", 64, 3, "phantom3"), ("c4", 128, 2, "phantom4"),
                                               ("c5@64", 64, 2, "phantom5")])
def test_P9_pivot_free_gate(name, n, p, material):
    tau = 1e-2
    O = oracle.Patch(n, p, tau)
    O.set_materials(workloads.element_eps(n, material))
    eps, mu = O.get_materials_tf()
    N = n + p
    c = (tau * tau / (4.0 * eps * mu)).reshape(N, N, N)  # [k, j, i]
    M, S, _ = O.matrices()
    rng = np.random.default_rng(0)
    worst_growth, worst_diff = 0.0, 0.0
    for s in (1, 2):
        for d in range(3):
            ax = (d + 1) % 3 if s == 1 else (d + 2) % 3  # stiffened axis (K1/K2)
            lo, hi = (0, N) if ax == d else (1, N - 1)  # PEC active rows (D1)
            for _ in range(40):
                a, b = rng.integers(1, N - 1, size=2)  # an active fiber position
                if ax == 0:
                    cf = c[b, a, lo:hi]
                elif ax == 1:
                    cf = c[b, lo:hi, a]
                else:
                    cf = c[lo:hi, b, a]
                A = M[lo:hi, lo:hi] + cf[:, None] * S[lo:hi, lo:hi]  # row k scaled by c_k
                f = rng.uniform(-1, 1, hi - lo)
                x0, g = nopivot_lu_solve(A, f)
                x1 = solve_banded((p, p), to_band(A, p), f)
                worst_growth = max(worst_growth, g)
                worst_diff = max(worst_diff, np.linalg.norm(x0 - x1) / np.linalg.norm(x1))
    print(f"{name}: max growth {worst_growth:.3f}, max rel diff {worst_diff:.2e}")
    assert worst_growth < 10.0
    assert worst_diff < 1e-13
