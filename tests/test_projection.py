"""NEXT-4: the test-function-weighted L2 projection of the Appendix
 in 3D,  diag(eps^) (M (x) M (x) M) u = f.

CPU pins of the oracle (``oracle.Patch.project_weighted``):
  P10a  the Appendix's own space (linear B-splines on [0 0 1 2 2]; matrix entries
        from tests/golden/linear_splines_0_0_1_2_2.txt): the weighted Kronecker system solved
        densely by numpy;
  P10b  the dense weak form assembled by 3D quadrature (tests/dense_ref.py, no 1D matrices,
        no Kronecker factoring) with each row scaled by its test function's eps, p = 1..3;
  P10c  closed form: eps = kappa constant and f = kappa (M (x) M (x) M) c reproduce c;
  P10d  a column-scaled system (eps on the trial index) is NOT what the oracle solves
        (negative control of the reading "the index of eps is the test function's").
GPU parity (``adi_project_weighted`` through the C ABI) against the oracle: tests marked gpu.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
import workloads
from tests.dense_ref import DenseMaxwell

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden_M():
    rows, cur = [], None
    for line in open(os.path.join(GOLD, "linear_splines_0_0_1_2_2.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line[0].isalpha():
            cur = line
            continue
        if cur == "M":
            rows.append([float(x) for x in line.split()])
    return np.array(rows)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


def test_P10a_appendix_linear_space():
    # the golden M is on unit elements [0, 2]; the oracle's patch is [0, 1] with n = 2: h = 1/2
    M = _golden_M() / 2.0
    K3 = np.kron(np.kron(M, M), M)  # flat index i + N (j + N k): x fastest
    rng = np.random.default_rng(100)
    eps = rng.uniform(1.0, 80.0, 27)
    f = rng.standard_normal(27)
    ref = np.linalg.solve(eps[:, None] * K3, f)
    u = oracle.Patch(2, 1, 0.1).project_weighted(f, eps)
    assert rel(u, ref) <= 1e-13


@pytest.mark.parametrize("p", [1, 2, 3])
def test_P10b_dense_weak_form(p):
    n = 3
    D = DenseMaxwell(n, p, 0.1, pec=False)
    Mq = D.form(D.Phi, D.Phi)  # rows: test functions
    rng = np.random.default_rng(200 + p)
    eps = rng.uniform(1.0, 80.0, D.U)
    f = rng.standard_normal(D.U)
    ref = np.linalg.solve(eps[:, None] * Mq, f)
    u = oracle.Patch(n, p, 0.1).project_weighted(f, eps)
    assert rel(u, ref) <= 1e-11


def test_P10c_reproduces_splines():
    n, p = 5, 2
    D = DenseMaxwell(n, p, 0.1, pec=False)
    c = np.random.default_rng(300).standard_normal(D.U)
    kappa = 7.5
    f = kappa * (D.form(D.Phi, D.Phi) @ c)
    u = oracle.Patch(n, p, 0.1).project_weighted(f, np.full(D.U, kappa))
    assert rel(u, c) <= 1e-12


def test_P10d_row_not_column_scaling():
    n, p = 3, 2
    D = DenseMaxwell(n, p, 0.1, pec=False)
    Mq = D.form(D.Phi, D.Phi)
    rng = np.random.default_rng(400)
    eps = rng.uniform(1.0, 80.0, D.U)
    f = rng.standard_normal(D.U)
    u = oracle.Patch(n, p, 0.1).project_weighted(f, eps)
    col = np.linalg.solve(Mq * eps[None, :], f)
    assert rel(u, col) > 1e-3
    with pytest.raises(oracle.OracleError):
        oracle.Patch(n, p, 0.1).project_weighted(f, np.where(np.arange(D.U) == 5, 0.0, eps))


# ---------------------------------------------------------------- GPU parity
TOL = 1e-10


def _gpu_case(n, p, seed, inplace=False):
    import torch
    import paper_2103_06998_b200 as adi
    N = n + p
    rng = np.random.default_rng(seed)
    eps = workloads.random_tf(N, seed, 1.0, 80.0)
    f = rng.standard_normal(N ** 3)
    ref = oracle.Patch(n, p, 0.1).project_weighted(f, eps)
    G = adi.Patch(n, p, 0.1)
    ft = torch.tensor(f, device="cuda")
    et = torch.tensor(eps, device="cuda")
    out = G.project_weighted(ft, et, out=ft if inplace else None)
    G.synchronize()
    u = out.cpu().numpy()
    return rel(u, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("n,p", [(1, 1), (1, 5), (2, 2), (7, 1), (37, 2), (40, 3), (21, 4), (13, 5)])
def test_project_weighted_parity(n, p):
    """Degenerate single-element patches, several 32-fiber tiles and sweep chunks, ragged tails
    (N odd/even), every degree."""
    assert _gpu_case(n, p, 10 + p) <= TOL


@pytest.mark.gpu
def test_project_weighted_inplace_and_larger():
    assert _gpu_case(96, 2, 77, inplace=True) <= TOL


@pytest.mark.gpu
def test_project_weighted_errors():
    import torch
    import paper_2103_06998_b200 as adi
    n, p = 6, 2
    N = n + p
    G = adi.Patch(n, p, 0.1)
    f = torch.ones(N ** 3, dtype=torch.float64, device="cuda")
    e = torch.ones_like(f)
    e[17] = -1.0
    out = torch.full_like(f, 3.0)
    with pytest.raises(adi.AdiError):
        G.project_weighted(f, e, out=out)
    assert bool((out == 3.0).all())  # untouched on error
