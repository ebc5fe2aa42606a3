"""Dense brute-force reference of one ADI step, straight from the weak forms.

Test code (pin P2 of SURVEY.md §8(c)).  It shares nothing with ``oracle/``:
the 1D basis comes from ``scipy.interpolate.BSpline`` and the Gauss rule from
``numpy.polynomial.legendre``; the 3D matrices are assembled by 3D quadrature
of the integrands printed in PAPER.md ``weak1``-``weak4`` -- no 1D
matrices and no Kronecker factoring of the operators -- then row-scaled by
the material of each test function (D5), restricted to the PEC active set
(D1) and solved densely with ``numpy.linalg.solve``.

Only tiny grids (<= 5^3 elements) are meant to go through here.
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial.legendre import leggauss
from scipy.interpolate import BSpline


class DenseMaxwell:
    def __init__(self, n: int, p: int, tau: float, pec: bool = True):
        self.n, self.p, self.tau, self.pec = n, p, tau, pec
        N = n + p
        self.N, self.U = N, N ** 3
        t = np.concatenate([np.zeros(p + 1), np.arange(1, n) / n, np.ones(p + 1)])
        q = p + 1  # exact for every integrand below (degree <= 2p per axis)
        gx, gw = leggauss(q)
        pts, wts = [], []
        for e in range(n):
            a, b = e / n, (e + 1) / n
            pts.append(a + (gx + 1) * (b - a) / 2)
            wts.append(gw * (b - a) / 2)
        x = np.concatenate(pts)
        w = np.concatenate(wts)
        spl = BSpline(t, np.eye(N), p, extrapolate=False)
        Bv = np.nan_to_num(spl(x))  # (nq, N)
        Bd = np.nan_to_num(spl.derivative(1)(x))
        # 3D basis at the 3D Gauss points: Phi[P, I] = B_i(x_P) B_j(y_P) B_k(z_P)
        # with I = i + N j + N^2 k and P = px + nq py + nq^2 pz (x fastest).
        K = lambda bz, by, bx: np.kron(np.kron(bz, by), bx)
        self.Phi = K(Bv, Bv, Bv)
        self.D = [K(Bv, Bv, Bd), K(Bv, Bd, Bv), K(Bd, Bv, Bv)]  # d/dx1, d/dx2, d/dx3
        self.W = np.kron(np.kron(w, w), w)

        # element of each 3D Gauss point (x fastest, q points per element per axis)
        ex = np.repeat(np.arange(n), q)
        self.elem_of_point = (ex[None, None, :] + n * (ex[None, :, None] + n * ex[:, None, None])).reshape(-1)

    # (f, g) with f = trial operator, g = test operator: rows = test functions
    def form(self, test, trial, weight=None):
        """weight: optional coefficient at every 3D Gauss point (V2: the element's material)."""
        W = self.W if weight is None else self.W * weight
        return test.T @ (W[:, None] * trial)

    def active(self, comp: int) -> np.ndarray:
        """Boolean mask of active coefficients (D1)."""
        N = self.N
        i, j, k = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
        ijk = [i, j, k]
        m = np.ones((N, N, N), dtype=bool)
        if self.pec and comp < 3:
            for ax in range(3):
                if ax != comp:
                    m &= (ijk[ax] >= 1) & (ijk[ax] <= N - 2)
        # back to x-fastest flat order
        return m.transpose(2, 1, 0).reshape(-1)

    def step(self, E, H, a, b, c, s_val=0.0, J=None, v2=None):
        """One full step (weak1 -> weak2 -> weak3 -> weak4).

        E, H: lists of 3 flat arrays; a, b, c: per-test-function row factors
        tau/(2 eps), tau/(2 mu), tau^2/(4 eps mu); J: list of 3 load vectors
        or None; s_val the signal value of this step (D9).
        v2: None (D5) or element arrays (a_e, c_e) = (tau/(2 eps_e), tau^2/(4 eps_e mu_e)): variant V2,
        the E right-hand sides' curl and mixed-derivative integrals with the element's coefficient
        inside the 3D quadrature (no row factor on those terms); LHS, H systems and source unchanged.
        """
        Phi, D = self.Phi, self.D
        Mass = self.form(Phi, Phi)
        # (d_a trial, V)
        Adv = [self.form(Phi, D[ax]) for ax in range(3)]
        # (d_a trial, d_b test)
        Mix = lambda ta, tb: self.form(D[tb], D[ta])
        if v2 is None:
            aAdv = [a[:, None] * X for X in Adv]
            cMix = lambda ta, tb: c[:, None] * Mix(ta, tb)
        else:
            wa, wc = (np.asarray(x, dtype=float)[self.elem_of_point] for x in v2)
            aAdv = [self.form(Phi, D[ax], wa) for ax in range(3)]
            cMix = lambda ta, tb: self.form(D[tb], D[ta], wc)
        Stf = [Mix(ax, ax) for ax in range(3)]
        E = [np.asarray(e, dtype=float).copy() for e in E]
        H = [np.asarray(h, dtype=float).copy() for h in H]
        for d in range(3):
            E[d][~self.active(d)] = 0.0

        def solve_E(lhs_stiff_axis, d, rhs):
            act = self.active(d)
            L = Mass + c[:, None] * Stf[lhs_stiff_axis]
            x = np.zeros(self.U)
            x[act] = np.linalg.solve(L[np.ix_(act, act)], rhs[act])
            return x

        def source(d):
            if J is None or J[d] is None:
                return 0.0
            return -a * s_val * J[d]

        # ---- weak1: substep-1 E systems -------------------------
        # LHS: (E1,V1)+c(d2 E1, d2 V1); (E2,V2)+c(d3 E2,d3 V2); (E3,V3)+c(d1 E3,d1 V3)
        # RHS: (E^n,V) + a[(-d3 H2 + d2 H3, V1) + (d3 H1 - d1 H3, V2) + (-d2 H1 + d1 H2, V3)]
        #      + c[(d1 E2, d2 V1) + (d2 E3, d3 V2) + (d3 E1, d1 V3)]
        R = [
            Mass @ E[0] + (-aAdv[2] @ H[1] + aAdv[1] @ H[2]) + cMix(0, 1) @ E[1] + source(0),
            Mass @ E[1] + (aAdv[2] @ H[0] - aAdv[0] @ H[2]) + cMix(1, 2) @ E[2] + source(1),
            Mass @ E[2] + (-aAdv[1] @ H[0] + aAdv[0] @ H[1]) + cMix(2, 0) @ E[0] + source(2),
        ]
        Eh = [solve_E(1, 0, R[0]), solve_E(2, 1, R[1]), solve_E(0, 2, R[2])]
        # ---- weak2: substep-1 H systems -------------------------
        # (H^{1/2},V) = (H^n,V) - b[(d2 E3^n,V1)+(d3 E1^n,V2)+(d1 E2^n,V3)]
        #                      + b[(d3 E2^h,V1)+(d1 E3^h,V2)+(d2 E1^h,V3)]
        Mi = np.linalg.inv(Mass)
        G = [
            Mass @ H[0] - b * (Adv[1] @ E[2]) + b * (Adv[2] @ Eh[1]),
            Mass @ H[1] - b * (Adv[2] @ E[0]) + b * (Adv[0] @ Eh[2]),
            Mass @ H[2] - b * (Adv[0] @ E[1]) + b * (Adv[1] @ Eh[0]),
        ]
        Hh = [np.linalg.solve(Mass, g) for g in G]
        del Mi
        # ---- weak3: substep-2 E systems -------------------------
        # LHS: (E1,V1)+c(d3 E1,d3 V1); (E2,V2)+c(d1 E2,d1 V2); (E3,V3)+c(d2 E3,d2 V3)
        # RHS: (E^h,V) + a[C-term with H^h] + c[(d1 E3,d3 V1)+(d2 E1,d1 V2)+(d3 E2,d2 V3)]
        R = [
            Mass @ Eh[0] + (-aAdv[2] @ Hh[1] + aAdv[1] @ Hh[2]) + cMix(0, 2) @ Eh[2] + source(0),
            Mass @ Eh[1] + (aAdv[2] @ Hh[0] - aAdv[0] @ Hh[2]) + cMix(1, 0) @ Eh[0] + source(1),
            Mass @ Eh[2] + (-aAdv[1] @ Hh[0] + aAdv[0] @ Hh[1]) + cMix(2, 1) @ Eh[1] + source(2),
        ]
        E1 = [solve_E(2, 0, R[0]), solve_E(0, 1, R[1]), solve_E(1, 2, R[2])]
        # ---- weak4: substep-2 H systems -------------------------
        # (H^{n+1},V) = (H^h,V) + b[(d3 E2^h,V1)+(d1 E3^h,V2)+(d2 E1^h,V3)]
        #                       - b[(d2 E3^{n+1},V1)+(d3 E1^{n+1},V2)+(d1 E2^{n+1},V3)]
        G = [
            Mass @ Hh[0] + b * (Adv[2] @ Eh[1]) - b * (Adv[1] @ E1[2]),
            Mass @ Hh[1] + b * (Adv[0] @ Eh[2]) - b * (Adv[2] @ E1[0]),
            Mass @ Hh[2] + b * (Adv[1] @ Eh[0]) - b * (Adv[0] @ E1[1]),
        ]
        H1 = [np.linalg.solve(Mass, g) for g in G]
        return E1, H1

    # ------------------------------------------------------------------------
    # Control scheme for pin P5: the first-order
    # Peaceman-Rachford ADI in (E, H) with the SAME Galerkin blocks, solved as
    # coupled block systems (no substitution, hence the exact Schur complement
    # -C1 M^-1 C2' where the paper's discrete1/discrete3 put the stiffness K).
    # Substep 1 is implicit in C1 H and C2 E, substep 2 in C2 H and C1 E
    # (scheme1a-scheme1d):
    #   M E^h - a C1 H^h = M E^n - a C2 H^n ,   M H^h - b C2' E^h = M H^n - b C1' E^n
    #   M E^1 + a C2 H^1 = M E^h + a C1 H^h ,   M H^1 + b C1' E^1 = M H^h + b C2' E^h
    # with (C1 H)_1 = d2 H3, (C1 H)_2 = d3 H1, (C1 H)_3 = d1 H2 and
    #      (C2 H)_1 = d3 H2, (C2 H)_2 = d1 H3, (C2 H)_3 = d2 H1; the primed
    # operators are the same derivatives with H test functions and E trial functions.
    # ------------------------------------------------------------------------
    def curl_blocks(self):
        """Dense Galerkin blocks of C1, C2 (E test / H trial) and C1', C2' (H test / E trial) as
        dicts {(row component, column component): matrix}, components 0..2 of E resp. H."""
        Adv = [self.form(self.Phi, self.D[ax]) for ax in range(3)]  # (d_ax trial, V)
        C1 = {(0, 2): Adv[1], (1, 0): Adv[2], (2, 1): Adv[0]}
        C2 = {(0, 1): Adv[2], (1, 2): Adv[0], (2, 0): Adv[1]}
        return C1, C2, dict(C1), dict(C2)

    def pr_operators(self, a, b):
        """Block matrices over the unknowns (E1, E2, E3 on their active sets, H1, H2, H3):
        Mb = blockdiag(M), and for substep s the implicit / explicit operators
        L1 = Mb - T1, R1 = Mb + T2 (substep 1) and L2 = Mb - T2, R2 = Mb + T1 (substep 2),
        T1 = [[0, a C1], [b C2', 0]], T2 = [[0, -a C2], [-b C1', 0]] (row-scaled by the
        test function's a = tau/(2 eps), b = tau/(2 mu), D5)."""
        U = self.U
        masks = [self.active(d) for d in range(3)] + [np.ones(U, bool)] * 3
        off = np.cumsum([0] + [int(m.sum()) for m in masks])
        n = off[-1]
        Mass = self.form(self.Phi, self.Phi)
        C1, C2, C1p, C2p = self.curl_blocks()
        Mb, T1, T2 = np.zeros((n, n)), np.zeros((n, n)), np.zeros((n, n))
        for c in range(6):
            m = masks[c]
            Mb[off[c]:off[c + 1], off[c]:off[c + 1]] = Mass[np.ix_(m, m)]

        def put(T, r, c, X, scale):
            mr, mc = masks[r], masks[c]
            T[off[r]:off[r + 1], off[c]:off[c + 1]] += scale[mr][:, None] * X[np.ix_(mr, mc)]

        for (i, j), X in C1.items():
            put(T1, i, 3 + j, X, a)
        for (i, j), X in C2p.items():
            put(T1, 3 + i, j, X, b)
        for (i, j), X in C2.items():
            put(T2, i, 3 + j, X, -a)
        for (i, j), X in C1p.items():
            put(T2, 3 + i, j, X, -b)
        return masks, off, Mb, T1, T2

    def pr_energy(self, E, H, a, b):
        """Et(u) = u^T Mb u + ||T2 u||^2_{Mb^-1} = ||(Mb - T2) u||^2_{Mb^-1} (T2 skew for
        eps = mu = 1), evaluated block by block without forming the block matrices."""
        Mass = self.form(self.Phi, self.Phi)
        C1, C2, C1p, _ = self.curl_blocks()
        a = np.broadcast_to(a, self.U)
        b = np.broadcast_to(b, self.U)
        masks = [self.active(d) for d in range(3)] + [np.ones(self.U, bool)] * 3
        f = [np.where(m, np.asarray(x, dtype=float), 0.0) for x, m in zip(list(E) + list(H), masks)]
        em = sum(float(x @ Mass @ x) for x in f)
        t2 = [np.zeros(self.U) for _ in range(6)]
        for (i, j), X in C2.items():  # E rows: -a C2 H
            t2[i] -= a * (X @ f[3 + j])
        for (i, j), X in C1p.items():  # H rows: -b C1' E
            t2[3 + i] -= b * (X @ f[j])
        extra = 0.0
        for c in range(6):
            m = masks[c]
            extra += float(t2[c][m] @ np.linalg.solve(Mass[np.ix_(m, m)], t2[c][m]))
        return em, em + extra

    def step_pr(self, E, H, a, b, steps=1):
        """`steps` steps of the exact-Schur Peaceman-Rachford control; returns (E, H, Et) where
        Et[k] = ||(Mb - T2) u^k||^2_{Mb^-1}, the quadratic form the scheme conserves for
        eps = mu = 1 (each half step is a Cayley transform of a skew operator)."""
        masks, off, Mb, T1, T2 = self.pr_operators(np.broadcast_to(a, self.U), np.broadcast_to(b, self.U))
        u = np.concatenate([np.asarray(f, dtype=float)[m] for f, m in zip(list(E) + list(H), masks)])
        L1, R1, L2, R2 = Mb - T1, Mb + T2, Mb - T2, Mb + T1

        def energy(v):
            w = L2 @ v
            return float(w @ np.linalg.solve(Mb, w))

        Et = [energy(u)]
        for _ in range(steps):
            u = np.linalg.solve(L1, R1 @ u)
            u = np.linalg.solve(L2, R2 @ u)
            Et.append(energy(u))
        out = []
        for c in range(6):
            f = np.zeros(self.U)
            f[masks[c]] = u[off[c]:off[c + 1]]
            out.append(f)
        return out[:3], out[3:], Et
