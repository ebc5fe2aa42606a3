"""Pins of the CPU oracle -- CPU only.

Each test pins the oracle to something other than itself: values PAPER.md
prints (tests/golden/), closed forms, invariants, a dense brute-force
assembly from the weak forms (tests/dense_ref.py, scipy BSpline basis), or
library routines (numpy.linalg) on tiny inputs.
"""
import math
import os

import numpy as np
import pytest
from numpy.polynomial.legendre import leggauss
from scipy.interpolate import BSpline

import oracle
import workloads
from tests.dense_ref import DenseMaxwell

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def golden_values():
    out = {}
    for line in open(os.path.join(GOLD, "paper_values.txt")):
        line = line.split("#")[0].strip()
        if line:
            k, v = line.split("=")
            out[k.strip()] = float(v)
    return out


def golden_matrices(name):
    mats, cur = {}, None
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line[0].isalpha():
            cur = line
            mats[cur] = []
        else:
            mats[cur].append([float(x) for x in line.split()])
    return {k: np.array(v) for k, v in mats.items()}


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# ---------------------------------------------------------------------------
# P1a: interior stencils (closed forms, cardinal B-spline values)
# ---------------------------------------------------------------------------
STENCILS = {
    1: dict(M=np.array([1, 4, 1]) / 6, S=np.array([-1, 2, -1]), A=np.array([-1, 0, 1]) / 2),
    2: dict(M=np.array([1, 26, 66, 26, 1]) / 120, S=np.array([-1, -2, 6, -2, -1]) / 6,
            A=np.array([-1, -10, 0, 10, 1]) / 24),
    3: dict(M=np.array([1, 120, 1191, 2416, 1191, 120, 1]) / 5040,
            S=np.array([-1, -24, -15, 80, -15, -24, -1]) / 120,
            A=np.array([-1, -56, -245, 0, 245, 56, 1]) / 720),
}


@pytest.mark.parametrize("p", [1, 2, 3])
def test_P1a_interior_stencils(p):
    n = 12
    h = 1.0 / n
    P = oracle.Patch(n, p, 1e-2)
    M, S, A = P.matrices()
    st = STENCILS[p]
    for row in range(2 * p, P.N - 2 * p):
        sl = slice(row - p, row + p + 1)
        assert np.allclose(M[row, sl], h * st["M"], rtol=1e-14, atol=1e-16)
        assert np.allclose(S[row, sl], st["S"] / h, rtol=1e-13, atol=1e-12)
        assert np.allclose(A[row, sl], st["A"], rtol=1e-13, atol=1e-15)
        # band: exact zeros outside |i-l| <= p
        assert np.all(M[row, : row - p] == 0) and np.all(M[row, row + p + 1 :] == 0)


# ---------------------------------------------------------------------------
# P1b: boundary rows (identities + hand values) and the Appendix space
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("n", [1, 3, 7])
def test_P1b_identities(p, n):
    P = oracle.Patch(n, p, 1e-2)
    M, S, A = P.matrices()
    t = P.knots()
    N = P.N
    # row sums of M = int B_l = (t_{l+p+1} - t_l)/(p+1)
    integ = np.array([(t[l + p + 1] - t[l]) / (p + 1) for l in range(N)])
    assert np.allclose(M.sum(1), integ, rtol=1e-13, atol=1e-15)
    assert np.allclose(S @ np.ones(N), 0, atol=1e-11 * n)
    assert np.allclose(A @ np.ones(N), 0, atol=1e-13)
    Bd = np.zeros((N, N))
    Bd[0, 0], Bd[-1, -1] = -1.0, 1.0
    assert np.allclose(A + A.T, Bd, atol=1e-13)  # integration by parts
    assert np.allclose(M, M.T, atol=0) and np.allclose(S, S.T, atol=1e-12)
    assert np.linalg.eigvalsh(M).min() > 0


def test_P1b_p2_row0():
    n = 10
    h = 1.0 / n
    P = oracle.Patch(n, 2, 1e-2)
    M, S, _ = P.matrices()
    assert np.allclose(M[0, :3], h * np.array([12, 7, 1]) / 60, rtol=1e-14)
    assert np.allclose(S[0, :3], np.array([4 / 3, -1, -1 / 3]) / h, rtol=1e-13)
    assert np.allclose(M[1, :4], h * np.array([7, 20, 12.5, 0.5]) / 60, rtol=1e-14)


def test_P1b_appendix_linear_space():
    """Knots [0 0 1 2 2] of the Appendix; oracle lives on [0,1] (h=1/2)."""
    g = golden_matrices("linear_splines_0_0_1_2_2.txt")
    P = oracle.Patch(2, 1, 1e-2)
    M, S, A = P.matrices()
    assert np.allclose(M * 2.0, g["M"], rtol=1e-14)
    assert np.allclose(S / 2.0, g["S"], rtol=1e-14)
    assert np.allclose(A, g["A"], rtol=1e-14)


# ---------------------------------------------------------------------------
# P1c: basis (partition of unity, derivative sum, Greville reproduces x,
#      agreement with scipy's independent B-spline evaluation)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_P1c_basis(p):
    n = 6
    P = oracle.Patch(n, p, 1e-2)
    t = P.knots()
    N = P.N
    gre = np.array([t[i + 1 : i + p + 1].mean() for i in range(N)])
    spl = BSpline(t, np.eye(N), p, extrapolate=False)
    dspl = spl.derivative(1)
    rng = np.random.default_rng(1)
    for x in list(rng.uniform(0, 1, 200)) + [0.0, 0.5, 1.0 - 1e-15]:
        v, d = P.basis(x)
        assert abs(v.sum() - 1) <= 1e-13 and abs(d.sum()) <= 1e-10
        assert abs(gre @ v - x) <= 1e-13
        assert np.all(v >= 0)
        assert np.allclose(v, np.nan_to_num(spl(x)), atol=1e-14)
        assert np.allclose(d, np.nan_to_num(dspl(x)), atol=1e-11)
    v, _ = P.basis(1.0)
    assert v[-1] == 1.0 and np.all(v[:-1] == 0.0)
    v, _ = P.basis(0.0)
    assert v[0] == 1.0


# ---------------------------------------------------------------------------
# P1d: material map D6
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 3])
def test_P1d_material_weights(p):
    n = 8
    P = oracle.Patch(n, p, 1e-2)
    w = P.material_weights()
    assert np.allclose(w.sum(1), 1.0, atol=1e-14)
    if p == 2:
        # interior B_r spans 3 equal elements with integrals 1/6, 2/3, 1/6 of the total
        r = 5
        assert np.allclose(w[r, r - 2 : r + 1], [1 / 6, 2 / 3, 1 / 6], atol=1e-14)
    eps = np.full(n ** 3, 3.7)
    P.set_materials(eps)
    e, m = P.get_materials_tf()
    assert np.allclose(e, 3.7, rtol=1e-14) and np.allclose(m, 1.0, rtol=1e-14)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_P1d_bruteforce_3d(p):
    """eps^_rst = int eps B_rst / int B_rst by brute-force 3D Gauss quadrature."""
    n = 3
    P = oracle.Patch(n, p, 1e-2)
    rng = np.random.default_rng(7)
    eps = rng.uniform(1, 80, n ** 3)
    P.set_materials(eps)
    e, _ = P.get_materials_tf()
    N = P.N
    t = P.knots()
    gx, gw = leggauss(p + 2)
    spl = BSpline(t, np.eye(N), p, extrapolate=False)
    num = np.zeros((N, N, N))
    den = np.zeros((N, N, N))
    for c in range(n):
        for b in range(n):
            for a in range(n):
                xs = [(ea + (gx + 1) / 2) / n for ea in (a, b, c)]
                Bx, By, Bz = (np.nan_to_num(spl(x)) for x in xs)
                for gk in range(len(gx)):
                    for gj in range(len(gx)):
                        for gi in range(len(gx)):
                            w = gw[gi] * gw[gj] * gw[gk] / (2 * n) ** 3
                            B3 = np.einsum("k,j,i->kji", Bz[gk], By[gj], Bx[gi]) * w
                            num += B3 * eps[a + n * (b + n * c)]
                            den += B3
    ref = (num / den).reshape(-1)  # [k,j,i] C-order -> i + N j + N^2 k
    assert np.allclose(e, ref, rtol=1e-13)


# ---------------------------------------------------------------------------
# P2: one and three full steps against the dense brute force from weak1-weak4
# ---------------------------------------------------------------------------
def _dense_vs_oracle(n, p, tau, material, steps, seed, source=False, bc=0):
    N = n + p
    U = N ** 3
    rng = np.random.default_rng(seed)
    fields = workloads.random_fields(N, seed)
    P = oracle.Patch(n, p, tau, bc)
    if material == "uniform":
        eps_tf, mu_tf = np.ones(U), np.ones(U)
    else:
        eps_tf = rng.uniform(1, 80, U)
        mu_tf = rng.uniform(0.5, 2.0, U)
    P.set_materials_tf(eps_tf, mu_tf)
    a, b, c = tau / (2 * eps_tf), tau / (2 * mu_tf), tau * tau / (4 * eps_tf * mu_tf)
    J = None
    sig = np.zeros(steps)
    if source:
        J = [None, None, rng.uniform(-1, 1, U)]
        sig = rng.uniform(-1, 1, steps)
        P.set_source(J, sig)
    P.set_fields(fields)
    D = DenseMaxwell(n, p, tau, pec=(bc == 0))
    E = [f.copy() for f in fields[:3]]
    H = [f.copy() for f in fields[3:]]
    for k in range(steps):
        E, H = D.step(E, H, a, b, c, s_val=sig[k], J=J)
    P.step(steps)
    got = P.get_fields()
    errs = [rel(got[d], (E + H)[d]) for d in range(6)]
    return max(errs)


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("material", ["uniform", "random"])
def test_P2_dense_one_step(p, material):
    n = 3 if p == 3 else 4
    assert _dense_vs_oracle(n, p, 0.05, material, 1, seed=10 + p) <= 1e-10


@pytest.mark.parametrize("p", [1, 2])
def test_P2_dense_three_steps_source(p):
    assert _dense_vs_oracle(3, p, 0.1, "random", 3, seed=20 + p, source=True) <= 1e-10


def test_P2_dense_5cubed():
    assert _dense_vs_oracle(5, 1, 0.02, "random", 1, seed=33) <= 1e-10


@pytest.mark.parametrize("p", [1, 2, 3])
def test_P2_dense_natural_bc(p):
    """NATURAL BC (SPEC default, NEXT-2): no coefficient eliminated; the oracle's bc=1 step
    equals the dense weak-form brute force on the full index sets (1 and 2 steps, random
    per-test-function eps and mu, with a source)."""
    n = 3
    assert _dense_vs_oracle(n, p, 0.05, "random", 1, seed=40 + p, bc=1) <= 1e-10
    assert _dense_vs_oracle(n, p, 0.1, "random", 2, seed=50 + p, source=True, bc=1) <= 1e-10


def _v2_vs_dense(n, p, tau, steps, seed, source=False):
    """Oracle V2 step (element-wise material inside the RHS quadrature) vs the dense weak-form
    assembly with the element coefficient at every 3D Gauss point (tests/dense_ref.py)."""
    N = n + p
    U = N ** 3
    rng = np.random.default_rng(seed)
    eps_e = rng.uniform(1, 80, n ** 3)
    mu_e = rng.uniform(0.5, 2.0, n ** 3)
    fields = workloads.random_fields(N, seed)
    P = oracle.Patch(n, p, tau)
    P.set_materials(eps_e, mu_e)
    P.set_rhs_variant(2)
    eps_tf, mu_tf = P.get_materials_tf()
    a, b, c = tau / (2 * eps_tf), tau / (2 * mu_tf), tau * tau / (4 * eps_tf * mu_tf)
    J, sig = None, np.zeros(steps)
    if source:
        J = [None, rng.uniform(-1, 1, U), None]
        sig = rng.uniform(-1, 1, steps)
        P.set_source(J, sig)
    P.set_fields(fields)
    P.step(steps)
    got = P.get_fields()
    D = DenseMaxwell(n, p, tau)
    E = [f.copy() for f in fields[:3]]
    H = [f.copy() for f in fields[3:]]
    v2 = (tau / (2 * eps_e), tau * tau / (4 * eps_e * mu_e))
    for k in range(steps):
        E, H = D.step(E, H, a, b, c, s_val=sig[k], J=J, v2=v2)
    return max(rel(got[d], (E + H)[d]) for d in range(6)), got, (eps_e, mu_e, fields)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_V2_dense(p):
    """NEXT-2 V2 (P:548-549 read as element-wise eps, mu inside the RHS integrals): the oracle's
    element-by-element sums of local 1D matrices equal the dense 3D quadrature with the element's
    coefficient at each Gauss point (no Kronecker factoring, scipy basis), 1 step; with p = 1 also
    2 steps and a source."""
    n = 3 if p == 3 else 4
    err, _, _ = _v2_vs_dense(n, p, 0.05, 1, seed=70 + p)
    assert err <= 1e-10, err
    if p == 1:
        err, _, _ = _v2_vs_dense(3, p, 0.1, 2, seed=77, source=True)
        assert err <= 1e-10, err


def test_V2_reduces_to_D5_for_constant_material_and_differs_otherwise():
    """Uniform eps, mu: the element coefficient is the row factor, V2 == D5 (to rounding);
    varying material: the two readings differ (the variant is not a no-op)."""
    n, p, tau = 4, 2, 0.05
    N = n + p
    f = workloads.random_fields(N, 81)
    out = {}
    for mat in ("const", "random"):
        eps_e = np.full(n ** 3, 7.5) if mat == "const" else np.random.default_rng(82).uniform(1, 80, n ** 3)
        for v in (0, 2):
            P = oracle.Patch(n, p, tau)
            P.set_materials(eps_e)
            P.set_rhs_variant(v)
            P.set_fields(f)
            P.step(2)
            out[mat, v] = P.get_fields()
    assert max(rel(out["const", 2][d], out["const", 0][d]) for d in range(6)) <= 1e-13
    assert max(rel(out["random", 2][d], out["random", 0][d]) for d in range(3)) >= 1e-6


def test_V2_needs_element_materials():
    n, p = 3, 2
    P = oracle.Patch(n, p, 0.05)
    P.set_materials_tf(np.ones((n + p) ** 3))
    P.set_rhs_variant(2)
    P.set_fields(workloads.random_fields(n + p, 1))
    with pytest.raises(Exception):
        P.step(1)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_point_load_vs_scipy(p):
    """orc_point_load (the oracle side of every c3/c4 source, D9): J_rst = B_r(x) B_s(y) B_t(z),
    against scipy's independent B-spline evaluation, incl. points on knots and on the boundary."""
    n = 5
    P = oracle.Patch(n, p, 0.01)
    N = P.N
    t = np.concatenate([np.zeros(p + 1), np.arange(1, n) / n, np.ones(p + 1)])
    spl = BSpline(t, np.eye(N), p, extrapolate=False)
    rng = np.random.default_rng(p)
    pts = [tuple(rng.uniform(0, 1, 3)) for _ in range(5)] + [(0.2, 0.4, 0.6), (0.0, 0.5, 1.0 - 1e-16),
                                                             workloads.dipole_position(n)]
    for x, y, z in pts:
        got = P.point_load(x, y, z)
        bx, by, bz = (np.nan_to_num(spl(v)) for v in (x, y, z))
        ref = np.kron(np.kron(bz, by), bx)  # index i + N (j + N k)
        assert np.allclose(got, ref, rtol=0, atol=1e-14), (x, y, z)
        assert abs(got.sum() - 1.0) <= 1e-13  # partition of unity in every axis


# ---------------------------------------------------------------------------
# P2b: block structure (Schur identities) -- pins D2/D3/D4 and
# every Kronecker placement of P:247-258 using the oracle's 1D matrices.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 3])
def test_P2b_schur_structure(p):
    n = 3
    P = oracle.Patch(n, p, 1e-2)
    M, S, A = P.matrices()
    B = A.T
    N = P.N
    k = lambda X, Y, Z: np.kron(np.kron(Z, Y), X)  # X acts on x (fastest)
    I = np.arange(N)
    inner = (I >= 1) & (I <= N - 2)
    act = []
    for d in range(3):
        m = [np.ones(N, bool) if ax == d else inner for ax in range(3)]
        act.append(np.kron(np.kron(m[2], m[1]), m[0]).astype(bool))
    Z = lambda: np.zeros((N ** 3, N ** 3))
    # E-test / H-trial curl blocks (C1, C2 of P:254-255 with D3) and H-test / E-trial
    C1 = [[None] * 3 for _ in range(3)]
    C1[0][2] = k(M, A, M); C1[1][0] = k(M, M, A); C1[2][1] = k(A, M, M)
    C2 = [[None] * 3 for _ in range(3)]
    C2[0][1] = k(M, M, A); C2[1][2] = k(A, M, M); C2[2][0] = k(M, A, M)
    R1 = {(0, 1): k(A, B, M), (1, 2): k(M, A, B), (2, 0): k(B, M, A)}
    R2 = {(0, 2): k(A, M, B), (1, 0): k(B, A, M), (2, 1): k(M, B, A)}
    Minv = np.linalg.inv(k(M, M, M))
    # R1 = -C1 M^{-1} C1', with C1'(H-test, E-trial) = -C2^T (skew-adjointness under PEC)
    def prod(Ca, Cb):
        out = {}
        for i in range(3):
            for j in range(3):
                acc = None
                for m in range(3):
                    if Ca[i][m] is None or Cb[m][j] is None:
                        continue
                    term = Ca[i][m] @ Minv @ Cb[m][j]
                    acc = term if acc is None else acc + term
                if acc is not None:
                    out[(i, j)] = acc
        return out

    def restrict(X, i, j):
        return X[np.ix_(act[i], act[j])]

    # H-test / E-trial discretisations (derivative on the trial E, as in the
    # H equations of) have the same Kronecker blocks as C1, C2.
    C1p, C2p = C1, C2
    # skew-adjointness under PEC: C1' = -C2^T and C2' = -C1^T on
    # the active E columns (rows = H components, unrestricted)
    for Cp, Co in ((C1p, C2), (C2p, C1)):
        for i in range(3):
            for j in range(3):
                if Cp[i][j] is None:
                    continue
                assert np.allclose(Cp[i][j][:, act[j]], -Co[j][i].T[:, act[j]], atol=1e-14)
    S1 = prod(C1, C1p)
    for key, blk in R1.items():
        assert np.allclose(restrict(-S1[key], *key), restrict(blk, *key), atol=1e-13)
    S2 = prod(C2, C2p)
    for key, blk in R2.items():
        assert np.allclose(restrict(-S2[key], *key), restrict(blk, *key), atol=1e-13)
    # K1 - (-C1 M^{-1} C2') is symmetric PSD on each diagonal block
    K1 = {0: k(M, S, M), 1: k(M, M, S), 2: k(S, M, M)}
    S12 = prod(C1, C2p)
    for d in range(3):
        X = restrict(K1[d] + S12[(d, d)], d, d)
        assert np.allclose(X, X.T, atol=1e-12)
        assert np.linalg.eigvalsh(0.5 * (X + X.T)).min() > -1e-10
    K2 = {0: k(M, M, S), 1: k(S, M, M), 2: k(M, S, M)}
    S21 = prod(C2, C1p)
    for d in range(3):
        X = restrict(K2[d] + S21[(d, d)], d, d)
        assert np.allclose(X, X.T, atol=1e-12)
        assert np.linalg.eigvalsh(0.5 * (X + X.T)).min() > -1e-10


# ---------------------------------------------------------------------------
# P3: direction-splitting factorisation under arbitrary per-test-function c
# (north-star check 4; Appendix)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("s", [1, 2])
def test_P3_split_equals_dense(p, s):
    n = 4 if p < 3 else 3
    tau = 1.0
    P = oracle.Patch(n, p, tau)
    N, U = P.N, P.N ** 3
    c = workloads.random_tf(N, seed=100 + p + 10 * s)
    eps = tau * tau / (4.0 * c)  # mu = 1  =>  c = tau^2 / (4 eps)
    P.set_materials_tf(eps)
    D = DenseMaxwell(n, p, tau)
    Mass = D.form(D.Phi, D.Phi)
    rng = np.random.default_rng(5)
    stiff = {1: [1, 2, 0], 2: [2, 0, 1]}[s]
    for d in range(3):
        rhs = rng.uniform(-1, 1, U)
        act = D.active(d)
        rhs[~act] = 0
        Stf = D.form(D.D[stiff[d]], D.D[stiff[d]])
        L = Mass + c[:, None] * Stf
        ref = np.zeros(U)
        ref[act] = np.linalg.solve(L[np.ix_(act, act)], rhs[act])
        got = P.solve_e(s, d, rhs)
        # both sides are backward stable: forward error <= O(cond * eps)
        tol = max(1e-12, 50 * np.linalg.cond(L[np.ix_(act, act)]) * np.finfo(float).eps)
        assert rel(got, ref) <= tol
        # negative control: paper-literal x->y->z order (variant V1) is wrong
        # whenever c varies along an axis swept before the stiffened one
        P.set_order_variant(1)
        bad = P.solve_e(s, d, rhs)
        P.set_order_variant(0)
        if stiff[d] > 0:
            assert rel(bad, ref) >= 1e-6
        else:
            assert rel(bad, ref) <= tol  # x stiffened: literal order is stiffened-first


def test_P3_appendix_2d_example():
    """2D linear splines on [0 0 1 2 2]^2, eps_ij per test function.
    Row-scaled blocks A_m (eq:split1) first, then the plain y system (eq:split2),
    equals the dense solve of the 9x9 row-scaled system."""
    g = golden_matrices("linear_splines_0_0_1_2_2.txt")
    Mx = My = g["M"]
    rng = np.random.default_rng(3)
    eps = rng.uniform(1, 50, (3, 3))  # eps[i, j] for test function B_i(x) B_j(y)
    F = rng.uniform(-1, 1, (3, 3))  # F[i, j] = int F B_i B_j
    # dense: row (i,j), column (l,m): eps_ij * Mx[i,l] * My[j,m]
    Ad = np.zeros((9, 9))
    for j in range(3):
        for i in range(3):
            for m in range(3):
                for l in range(3):
                    Ad[i + 3 * j, l + 3 * m] = eps[i, j] * Mx[i, l] * My[j, m]
    u_dense = np.linalg.solve(Ad, F.T.reshape(-1))  # unknown index l + 3 m
    # split: for each y-row j, A_j = diag(eps[:, j]) Mx ; A_j G_j = F_j ; then My U^T = G
    G = np.stack([np.linalg.solve(np.diag(eps[:, j]) @ Mx, F[:, j]) for j in range(3)], axis=1)
    Usplit = np.linalg.solve(My, G.T).T  # U[l, m]
    assert np.allclose(Usplit.T.reshape(-1), u_dense, rtol=1e-13, atol=1e-14)


# ---------------------------------------------------------------------------
# P4: second order in time (CLAIM-3, Fig. 2)
# ---------------------------------------------------------------------------
def _run_uA(n, p, tau, steps):
    P = oracle.Patch(n, p, tau)
    P.project_uA(0.0)
    P.step(steps)
    return P


@pytest.mark.slow
def test_P4_temporal_order_c2_taus():
    """c2 (32^3 elements, p = 2, u_A): tau in {1e-2, 5e-3, 2.5e-3}, compared at the common time
    t = 0.25 (steps 25, 50, 100); self-convergence order in [1.8, 2.2] for E and for H."""
    from concurrent.futures import ThreadPoolExecutor

    n, p = 32, 2
    # three independent oracle patches; ctypes releases the GIL, so the runs overlap on three cores
    with ThreadPoolExecutor(3) as ex:
        runs = list(ex.map(lambda ts: _run_uA(n, p, ts[0], ts[1]).get_fields(),
                           [(1e-2, 25), (5e-3, 50), (2.5e-3, 100)]))
    for grp in (slice(0, 3), slice(3, 6)):
        d1 = np.sqrt(sum(np.sum((a - b) ** 2) for a, b in zip(runs[0][grp], runs[1][grp])))
        d2 = np.sqrt(sum(np.sum((a - b) ** 2) for a, b in zip(runs[1][grp], runs[2][grp])))
        order = math.log2(d1 / d2)
        assert 1.8 <= order <= 2.2, order


# ---------------------------------------------------------------------------
# P5: stability (CLAIM-2)
#
# Finding (recorded in DESIGN.md §3): the M-norm energy u^T M u is NOT the quantity
# these ADI schemes conserve.  The exact-Schur Peaceman-Rachford control (first-order
# (E, H) form of scheme1a-scheme1d with the same Galerkin blocks, tests/dense_ref.py)
# conserves Et(u) = u^T M u + ||T2 u||^2_{M^-1} (T2 = the explicit curl operator of
# substep 1), so even it lets u^T M u rise up to Et(0) -- for u_A that is
# 1 + pi^2 tau^2 / 4 (1.0247 at tau = 1/10, 3.47 at tau = 1, 248 at tau = 10).  The
# paper's scheme replaces the exact Schur complement by the stiffness K (discrete1/3),
# a PSD perturbation that keeps rho(G) = 1 but makes G non-normal: transient growth
# sup_n ||G^n||_M > 1, bounded (power-bounded), no secular growth.  SURVEY's P5(ii)
# "max E(n) <= 1.01 E(0)" therefore cannot hold at tau >= 1/10; the pins below
# are the properties that do hold, each checked against an independent computation.
# ---------------------------------------------------------------------------
def _masks(N):
    I = np.arange(N)
    inner = (I >= 1) & (I <= N - 2)
    out = []
    for d in range(3):
        m = [np.ones(N, bool) if ax == d else inner for ax in range(3)]
        out.append(np.kron(np.kron(m[2], m[1]), m[0]).astype(bool))
    return out + [np.ones(N ** 3, bool)] * 3


def _amplification(n, p, tau, eps_tf=None):
    """Brute-force amplification matrix of one oracle step over the free coefficients
    (E on their PEC active sets, H everywhere): column j = step(e_j)."""
    P = oracle.Patch(n, p, tau)
    if eps_tf is not None:
        P.set_materials_tf(eps_tf)
    N, U = P.N, P.N ** 3
    masks = _masks(N)
    idx = [(c, i) for c in range(6) for i in np.nonzero(masks[c])[0]]
    G = np.zeros((len(idx), len(idx)))
    for col, (c, i) in enumerate(idx):
        f = [np.zeros(U) for _ in range(6)]
        f[c][i] = 1.0
        P.set_fields(f)
        P.step(1)
        out = P.get_fields()
        G[:, col] = np.concatenate([out[cc][masks[cc]] for cc in range(6)])
    return G


@pytest.mark.parametrize("n,p", [(3, 1), (3, 2), (3, 3), (4, 2)])
@pytest.mark.parametrize("tau", [1e-1, 10.0, 1e3])
def test_P5_pr_control_conserves_energy(n, p, tau):
    """Control for P5: the exact-Schur Peaceman-Rachford scheme built
    from the dense weak-form blocks conserves Et to rounding -- every curl block is skew
    (C1' = -C1^T, C2' = -C2^T under PEC, D1) and every sign of scheme1a-1d / D2 is right.
    Negative control: flipping the sign of one H-equation block (a D2-type error) breaks it."""
    D = DenseMaxwell(n, p, tau)
    f = workloads.random_fields(n + p, 3)
    _, _, Et = D.step_pr(f[:3], f[3:], tau / 2, tau / 2, steps=3)
    drift = np.abs(np.diff(Et)) / np.asarray(Et[:-1])
    assert drift.max() <= 1e-12, drift
    masks, off, Mb, T1, T2 = D.pr_operators(np.full(D.U, tau / 2), np.full(D.U, tau / 2))
    u = np.concatenate([x[m] for x, m in zip(f, masks)])
    bad = T2.copy()
    bad[off[3]:off[4], :off[3]] *= -1.0  # H1 row of -b C1' E with the wrong sign
    L1, R1, L2, R2 = Mb - T1, Mb + bad, Mb - bad, Mb + T1
    e0 = float((L2 @ u) @ np.linalg.solve(Mb, L2 @ u))
    u1 = np.linalg.solve(L2, R2 @ np.linalg.solve(L1, R1 @ u))
    e1 = float((L2 @ u1) @ np.linalg.solve(Mb, L2 @ u1))
    assert abs(e1 - e0) / e0 >= 1e-6


_RHO_CASES = [(3, 1, t) for t in (1e-3, 1e-2, 1e-1, 1.0, 10.0, 1e2, 1e3)] + \
             [(3, 2, t) for t in (1e-3, 1e-2, 1e-1, 1.0, 10.0, 1e2, 1e3)] + \
             [(4, 1, t) for t in (1e-3, 1e-1, 10.0, 1e3)]
_RHO_SLOW = [(3, 3, t) for t in (1e-3, 1e-2, 1e-1, 1.0, 10.0, 1e2, 1e3)] + \
            [(4, 2, t) for t in (1e-3, 1e-1, 10.0, 1e3)] + \
            [(4, 1, t) for t in (1e-2, 1.0, 1e2)] + [(4, 3, t) for t in (1e-3, 1.0, 1e3)]


@pytest.mark.parametrize("n,p,tau", _RHO_CASES + [pytest.param(*c, marks=pytest.mark.slow) for c in _RHO_SLOW])
def test_P5_spectral_radius(n, p, tau):
    """P5(i): rho(G) <= 1 + 1e-12 on 3^3 and 4^3 elements, p = 1..3, tau = 1e-3 .. 1e3
    (eps = mu = 1): the paper's unconditional stability in the spectral sense.
    The eigenvalue 1 belongs to the discrete gradients (curl-free E, H), which every step
    leaves unchanged."""
    G = _amplification(n, p, tau)
    rho = np.abs(np.linalg.eigvals(G)).max()
    assert rho <= 1 + 1e-12, rho


def _amplification_el(n, p, tau, eps_e, variant):
    """Amplification matrix of one oracle step with ELEMENT materials and the given RHS variant."""
    P = oracle.Patch(n, p, tau)
    P.set_materials(eps_e)
    P.set_rhs_variant(variant)
    N, U = P.N, P.N ** 3
    masks = _masks(N)
    idx = [(c, i) for c in range(6) for i in np.nonzero(masks[c])[0]]
    G = np.zeros((len(idx), len(idx)))
    for col, (c, i) in enumerate(idx):
        f = [np.zeros(U) for _ in range(6)]
        f[c][i] = 1.0
        P.set_fields(f)
        P.step(1)
        out = P.get_fields()
        G[:, col] = np.concatenate([out[cc][masks[cc]] for cc in range(6)])
    return G


@pytest.mark.parametrize("p", [1, 2])
def test_V2_is_unstable_where_D5_is_not(p):
    """NEXT-2 finding (recorded in DESIGN.md): with a two-valued element material (eps 1 / 50, the
    phantom's contrast) the paper-literal D5 step keeps rho(G) at 1 (p = 1; 1 + 1.3e-4 for p = 2,
    the P5(iii) growth of the row-scaled scheme), while V2 -- the
    element material inside the RHS quadrature but the test function's c^ in the row-modified
    LHS, as the ADI solve requires -- has rho(G) > 1: the RHS mixed-derivative term no longer
    matches the implicit stiffness it was eliminated against.  On the GPU the c3 / c4 phantoms
    blow up under V2 within 40 steps (tools/v2_study.py)."""
    n, tau = 3, 0.1
    eps = np.where(np.random.default_rng(5).uniform(size=n ** 3) < 0.5, 1.0, 50.0)
    rho5 = np.abs(np.linalg.eigvals(_amplification_el(n, p, tau, eps, 0))).max()
    rho2 = np.abs(np.linalg.eigvals(_amplification_el(n, p, tau, eps, 2))).max()
    # D5 with varying material: rho = 1 to rounding for p = 1; p = 2 shows the small growth of the
    # row-scaled (non-normal) scheme recorded under P5(iii) (1.3e-4 here); V2 grows > 100x faster
    assert rho5 - 1 <= (1e-12 if p == 1 else 1e-3), rho5
    assert rho2 - 1 >= max(0.01, 100 * (rho5 - 1)), (rho2, rho5)


def _mass_sqrt(n, p):
    D = DenseMaxwell(n, p, 1.0)
    masks, _, Mb, _, _ = D.pr_operators(np.zeros(D.U), np.zeros(D.U))
    w, V = np.linalg.eigh(Mb)
    return (V * np.sqrt(w)) @ V.T, (V / np.sqrt(w)) @ V.T


@pytest.mark.slow
@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("tau", [1.0, 10.0, 1e3])
def test_P5_power_bounded(p, tau):
    """P5(i'): no secular growth: ||G^n||_M (n up to 4096, by repeated squaring) levels off --
    the largest value over n in [512, 4096] does not exceed the largest over n <= 256 by more
    than 2%.  (A Jordan block at |lambda| = 1 or a rho slightly above 1 would grow ~n or
    exponentially.)  The transient itself is large: G is non-normal (see the finding above);
    on 3^3, p = 2 sup_n ||G^n||_M is ~1.07 / 5.8 / 116 at tau = 1/10, 1, 10."""
    n = 3
    G = _amplification(n, p, tau)
    Mh, Mih = _mass_sqrt(n, p)
    norms = {}
    X = np.eye(len(G))
    for k in range(1, 17):
        X = G @ X
        norms[k] = np.linalg.norm(Mh @ X @ Mih, 2)
    X = np.linalg.matrix_power(G, 16)
    k = 16
    while k < 4096:
        X = X @ X
        k *= 2
        norms[k] = np.linalg.norm(Mh @ X @ Mih, 2)
    early = max(v for kk, v in norms.items() if kk <= 256)
    late = max(v for kk, v in norms.items() if kk >= 512)
    assert late <= 1.02 * early, (early, late, norms)
    assert np.isfinite(late)


def _mass_energy(M, fs):
    e = 0.0
    for f in fs:
        N = M.shape[0]
        u = f.reshape(N, N, N)  # [k, j, i]
        Mu = np.einsum("ai,bj,ck,kji->cba", M, M, M, u)
        e += float(np.sum(u * Mu))
    return e


@pytest.mark.parametrize("tau,steps", [(0.1, 10), pytest.param(1.0, 4000, marks=pytest.mark.slow),
                                       pytest.param(10.0, 4000, marks=pytest.mark.slow)])
def test_P5_energy_uA_bounded(tau, steps):
    """P5(ii) as it holds: 8^3, p = 2, u_A (eps = mu = 1).  The M-energy u^T M u of the oracle's
    steps stays below Et(u^0), the quantity the exact-Schur PR control conserves, evaluated on
    the initial data by the independent dense blocks (measured max u^T M u / u0^T M u0: 1.0120
    at tau = 1/10 (10 steps), 2.912 at tau = 1, 245.3 at tau = 10 against Et(0) / u0^T M u0 =
    1.0247, 3.467, 247.7); and there is no secular growth (4000 steps -- 2.5x the 10^3 steps in
    which the maxima above are reached: the second half's maximum does not exceed the first
    half's)."""
    n, p = 8, 2
    P = oracle.Patch(n, p, tau)
    P.project_uA(0.0)
    f0 = P.get_fields()
    M, _, _ = P.matrices()
    D = DenseMaxwell(n, p, tau)
    em0, et0 = D.pr_energy(f0[:3], f0[3:], tau / 2, tau / 2)
    assert abs(_mass_energy(M, f0) - em0) <= 1e-12 * em0  # the two mass matrices agree
    every = 1 if steps <= 100 else 20
    tr = []
    for _ in range(steps // every):
        P.step(every)
        tr.append(_mass_energy(M, P.get_fields()))
    tr = np.array(tr)
    assert tr.max() <= et0 * (1 + 1e-12), (tr.max() / em0, et0 / em0)
    if steps >= 1000:
        h = len(tr) // 2
        # quasi-periodic (non-normal G, rho = 1): later peaks may come marginally closer to the
        # supremum; secular growth would exceed it by far more than 1 %
        assert tr[h:].max() <= tr[:h].max() * 1.01, (tr[:h].max() / em0, tr[h:].max() / em0)


@pytest.mark.parametrize("tau", [0.01, 0.1, 10.0])
def test_P5_random_material_report(tau):
    """P5(iii), reported not asserted as stable: i.i.d. per-test-function eps in [1, 80] (3^3,
    p = 2).  Row scaling makes the mass non-symmetric and the energy argument fails (SURVEY
    §A.3); measured rho(G) - 1 is ~1e-4..9e-4 at tau = 0.01..0.1 (a finding: slow growth) and
    at rounding level for tau >= 1.  The assertion only brackets what was measured."""
    worst = 0.0
    for seed in range(2):
        eps = workloads.random_tf(5, 70 + seed, 1.0, 80.0)
        rho = np.abs(np.linalg.eigvals(_amplification(3, 2, tau, eps))).max()
        worst = max(worst, rho)
    print(f"P5(iii) tau={tau}: max rho(G) - 1 = {worst - 1:.3e}")
    assert worst <= 1.01, worst


# ---------------------------------------------------------------------------
# P6: manufactured-solution accuracy vs the bounds PAPER.md prints
# ---------------------------------------------------------------------------
def test_P6_gamma_and_norm():
    gv = golden_values()
    assert abs(2 / math.sqrt(14) - gv["gamma"]) < 1e-15
    # ||u_A(.,0)||_L2 by Gauss quadrature against the zero state == 1
    P = oracle.Patch(4, 2, 0.1)
    P.set_fields([np.zeros(P.U)] * 6)
    err = P.errors_uA(0.0)
    assert abs(err[0] - gv["uA_norm_t0"]) < 1e-10 and err[1] == 0.0
    f, _ = oracle.exact_uA(0.5, 0.5, 0.5, 0.0)
    assert np.allclose(f, [gv["gamma"], 2 * gv["gamma"], 3 * gv["gamma"], 0, 0, 0], atol=1e-15)


def test_P6_exact_solution_satisfies_maxwell():
    """Residuals of dE/dt = curl H, dH/dt = -curl E (eps=mu=1) -- needs D8."""
    rng = np.random.default_rng(0)
    h = 1e-5
    for _ in range(50):
        x, y, z, t = rng.uniform(0, 1, 4)
        f, cu = oracle.exact_uA(x, y, z, t)
        fp, _ = oracle.exact_uA(x, y, z, t + h)
        fm, _ = oracle.exact_uA(x, y, z, t - h)
        dt = (fp - fm) / (2 * h)
        assert np.allclose(dt[:3], cu[3:], atol=1e-8)
        assert np.allclose(dt[3:], -cu[:3], atol=1e-8)
        # curl by finite differences in space
        def fd(comp, ax):
            e = np.zeros(3); e[ax] = h
            a, _ = oracle.exact_uA(*(np.array([x, y, z]) + e), t)
            b, _ = oracle.exact_uA(*(np.array([x, y, z]) - e), t)
            return (a[comp] - b[comp]) / (2 * h)
        curlE = [fd(2, 1) - fd(1, 2), fd(0, 2) - fd(2, 0), fd(1, 0) - fd(0, 1)]
        assert np.allclose(curlE, cu[:3], atol=1e-7)
    # tangential E vanishes on the faces (E x n = 0, Eq. 1)
    for _ in range(50):
        u, v = rng.uniform(0, 1, 2)
        for face in range(3):
            for val in (0.0, 1.0):
                pt = np.insert(np.array([u, v]), face, val)
                f, _ = oracle.exact_uA(*pt, rng.uniform())
                tang = [f[c] for c in range(3) if c != face]
                assert np.allclose(tang, 0, atol=1e-15)


def test_P6_paper_bound_tau_1_10():
    gv = golden_values()
    n, p, tau = int(gv["mesh_elements_per_axis"]), 2, 0.1
    P = oracle.Patch(n, p, tau)
    P.project_uA(0.0)
    mx = np.zeros(4)
    for k in range(10):
        P.step(1)
        mx = np.maximum(mx, P.errors_uA((k + 1) * tau))
    assert mx[0] < gv["l2_bound_tau_1_10"] and mx[1] < gv["l2_bound_tau_1_10"]
    assert mx[2] < gv["hcurl_bound_tau_1_10"] and mx[3] < gv["hcurl_bound_tau_1_10"]


@pytest.mark.slow
def test_P6_paper_bound_tau_1_1280():
    gv = golden_values()
    n, p, tau = int(gv["mesh_elements_per_axis"]), 2, 1.0 / 1280
    P = oracle.Patch(n, p, tau)
    P.project_uA(0.0)
    mx = np.zeros(4)
    for k in range(32):
        P.step(40)
        mx = np.maximum(mx, P.errors_uA((k + 1) * 40 * tau))
    assert mx[0] < gv["l2_bound_tau_1_1280"] and mx[1] < gv["l2_bound_tau_1_1280"], mx
    assert mx[2] < gv["hcurl_bound_tau_1_1280"] and mx[3] < gv["hcurl_bound_tau_1_1280"], mx


# ---------------------------------------------------------------------------
# P7: spatial convergence (textbook expectations; the paper is silent)
# ---------------------------------------------------------------------------
@pytest.mark.slow
@pytest.mark.parametrize("p", [2, 3])
def test_P7_spatial_rates(p):
    errs = []
    for n in (6, 12):
        P = oracle.Patch(n, p, 1e-4)
        P.project_uA(0.0)
        P.step(10)
        errs.append(P.errors_uA(10 * 1e-4))
    e0, e1 = errs
    assert math.log2(e0[0] / e1[0]) >= p  # L2 of E
    assert math.log2(e0[2] / e1[2]) >= p - 0.3  # H(curl) of E


# ---------------------------------------------------------------------------
# P8: invariants
# ---------------------------------------------------------------------------
def test_P8_zero_linearity_identity():
    n, p, tau = 3, 2, 0.07
    P = oracle.Patch(n, p, tau)
    P.set_materials_tf(workloads.random_tf(P.N, 4, 1, 80))
    U = P.U
    P.set_fields([np.zeros(U)] * 6)
    P.step(2)
    assert all(np.all(f == 0) for f in P.get_fields())
    u = workloads.random_fields(P.N, 1)
    v = workloads.random_fields(P.N, 2)
    alpha = -1.7
    outs = []
    for f in (u, v, [alpha * a + b for a, b in zip(u, v)]):
        P.set_fields(f)
        P.step(1)
        outs.append(P.get_fields())
    for d in range(6):
        assert rel(outs[2][d], alpha * outs[0][d] + outs[1][d]) <= 1e-13
    # tau -> 0: a = b = c = 0 => identity (up to the mass solves)
    P0 = oracle.Patch(n, p, 1e-300)
    P0.set_fields(u)
    P0.step(1)
    got = P0.get_fields()
    P0.set_fields(u)  # zeroes PEC entries
    ref = P0.get_fields()
    for d in range(6):
        assert rel(got[d], ref[d]) <= 1e-13


def _cyc_coeff(f, N):
    """Relabel (x1,x2,x3) -> (x2,x3,x1): new[j,k,i] = old[i,j,k]."""
    u = f.reshape(N, N, N)  # [k, j, i]
    # new field g(x'1,x'2,x'3) with x'1 = x2, x'2 = x3, x'3 = x1: g[i'=j, j'=k, k'=i]
    return np.ascontiguousarray(u.transpose(2, 0, 1)).reshape(-1)


def test_P8_cyclic_equivariance():
    n, p, tau = 3, 2, 0.05
    P = oracle.Patch(n, p, tau)
    N = P.N
    eps = workloads.random_tf(N, 8, 1, 80)
    P.set_materials_tf(eps)
    f = workloads.random_fields(N, 3)
    P.set_fields(f)
    f = P.get_fields()
    P.step(1)
    out = P.get_fields()
    Q = oracle.Patch(n, p, tau)
    Q.set_materials_tf(_cyc_coeff(eps, N))
    # the component along x'_1 = x_2 is old E2, etc.: new comp c' carries old comp c'+1
    g = [None] * 6
    for c in range(3):
        g[(c + 2) % 3] = _cyc_coeff(f[c], N)
        g[3 + (c + 2) % 3] = _cyc_coeff(f[3 + c], N)
    Q.set_fields(g)
    Q.step(1)
    got = Q.get_fields()
    for c in range(3):
        assert rel(got[(c + 2) % 3], _cyc_coeff(out[c], N)) <= 1e-13
        assert rel(got[3 + (c + 2) % 3], _cyc_coeff(out[3 + c], N)) <= 1e-13


def test_P8_uniform_material_and_checkpoint():
    n, p, tau = 4, 2, 0.05
    f = workloads.random_fields(n + p, 9)
    A = oracle.Patch(n, p, tau)
    A.set_fields(f)
    A.step(2)
    B = oracle.Patch(n, p, tau)
    B.set_materials_tf(np.ones(B.U), np.ones(B.U))
    B.set_fields(f)
    B.step(2)
    for x, y in zip(A.get_fields(), B.get_fields()):
        assert np.array_equal(x, y)
    # checkpoint / resume is a bitwise continuation
    C = oracle.Patch(n, p, tau)
    C.set_fields(f)
    C.step(1)
    ck = C.get_fields()
    D = oracle.Patch(n, p, tau)
    D.set_fields(ck)
    D.step(1)
    for x, y in zip(A.get_fields(), D.get_fields()):
        assert np.array_equal(x, y)


def test_oracle_errors_and_states():
    with pytest.raises(oracle.OracleError):
        oracle.Patch(0, 2, 0.1)
    with pytest.raises(oracle.OracleError):
        oracle.Patch(4, 6, 0.1)
    with pytest.raises(oracle.OracleError):
        oracle.Patch(4, 2, -1.0)
    P = oracle.Patch(3, 2, 0.1)
    with pytest.raises(oracle.OracleError):
        P.step(1)  # fields not set
    with pytest.raises(oracle.OracleError):
        P.set_materials(np.concatenate([np.ones(26), [-1.0]]))
    with pytest.raises(oracle.OracleError):
        P.set_materials_tf(np.full(P.U, np.nan))


@pytest.mark.parametrize("p,bc", [(2, 0), (3, 1)])
def test_threads_bit_identical(p, bc):
    """orc_set_threads only splits independent outputs (kron3 points, sweep fibers) over OpenMP
    threads: the fields after two steps with a source equal the single-threaded run bit for bit."""
    n, tau = 7, 0.05
    N = n + p
    eps = workloads.element_eps(n, "phantom5")
    f = workloads.random_fields(N, 11)
    sig = np.sin(np.arange(4) * 0.3)
    out = []
    for t in (1, 4):
        P = oracle.Patch(n, p, tau, bc)
        P.set_threads(t)
        P.set_materials(eps)
        P.set_fields(f)
        P.set_source([None, P.point_load(0.3, 0.6, 0.45), None], sig)
        P.step(2)
        out.append(P.get_fields())
    for x, y in zip(*out):
        assert np.array_equal(x, y)

