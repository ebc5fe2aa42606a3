"""CPU test double of the library's box-level kernels (adi_box_*), for the gloo
tests of the slab-decomposed schedule (paper_2103_06998_b200.dist).

Test infrastructure only: dense 1D matrices from the oracle, torch/numpy
arithmetic on CPU tensors.  It restates the per-box operations from the paper
(Kronecker terms of discrete1-discrete4 with the readings
D1-D9, banded sweeps, the uniform-mu derivative projection) so that the
orchestration -- which slab, which halo, which transpose, in which order -- can
be checked against the oracle's single-domain step on CPU.
"""
import numpy as np
import torch

import oracle

OP_M, OP_A, OP_B = 0, 1, 2


def _v(t, dims):
    """(z, y, x) numpy view of a flat/contiguous tensor holding a box of dims (x, y, z)."""
    return t.numpy().reshape(int(dims[2]), int(dims[1]), int(dims[0]))


class CpuBoxBackend:
    def __init__(self, n, p, tau, bc=0):
        self.O = oracle.Patch(n, p, tau, bc)
        self.n, self.p, self.tau, self.bc = n, p, tau, bc
        self.N = n + p
        M, S, A = self.O.matrices()
        self.M, self.S, self.A = M, S, A
        self.ops = {OP_M: M, OP_A: A, OP_B: A.T.copy()}

    def active(self, comp, axis):
        if self.bc == 0 and comp < 3 and axis != comp:
            return 1, self.N - 1
        return 0, self.N

    # -- data movement -------------------------------------------------------------
    def box_copy(self, dst, ddims, doff, src, sdims, soff, ext):
        d, s_ = _v(dst, ddims), _v(src, sdims)
        d[doff[2]:doff[2] + ext[2], doff[1]:doff[1] + ext[1], doff[0]:doff[0] + ext[0]] = \
            s_[soff[2]:soff[2] + ext[2], soff[1]:soff[1] + ext[1], soff[0]:soff[0] + ext[0]]

    def box_abc(self, eps, mu, count, a, b, c):
        e, m = eps.reshape(-1)[:count], mu.reshape(-1)[:count]
        a.view(-1)[:count] = self.tau / (2.0 * e)
        b.view(-1)[:count] = self.tau / (2.0 * m)
        c.view(-1)[:count] = self.tau * self.tau / (4.0 * e * m)

    def box_pec(self, comp, u, dims, off):
        if comp >= 3 or self.bc != 0:
            return
        v = _v(u, dims)
        for ax in range(3):
            lo, hi = self.active(comp, ax)
            idx = np.arange(dims[ax]) + off[ax]
            bad = (idx < lo) | (idx >= hi)
            sl = [slice(None)] * 3
            sl[2 - ax] = bad
            v[tuple(sl)] = 0.0

    def box_materials_tf(self, eps_elem, mu_elem, eps_tf, mu_tf):
        self.O.set_materials(np.asarray(eps_elem, dtype=np.float64), None if mu_elem is None else np.asarray(mu_elem))
        e, m = self.O.get_materials_tf()
        eps_tf.copy_(torch.from_numpy(e))
        mu_tf.copy_(torch.from_numpy(m))

    def box_factor(self, comp, axis, dims, c, iu):
        pass  # the double solves each fiber directly

    # -- sweeps -----------------------------------------------------------------------
    def box_sweep(self, mode, jobs):
        for j in jobs:
            dims, ax = j["dims"], j["axis"]
            lo, hi = self.active(j["comp"], ax)
            u = np.moveaxis(_v(j["in"], dims), 2 - ax, -1).copy()  # fibers on the last axis
            shp = u.shape
            u = u.reshape(-1, shp[-1])
            if mode == 0:
                x = np.linalg.solve(self.M[lo:hi, lo:hi], u[:, lo:hi].T).T
                res = u.copy()
                res[:, lo:hi] = x
            elif mode == 1:
                cc = np.moveaxis(_v(j["c"], dims), 2 - ax, -1).reshape(-1, shp[-1])
                res = u.copy()
                for f in range(u.shape[0]):
                    Af = self.M[lo:hi, lo:hi] + cc[f, lo:hi, None] * self.S[lo:hi, lo:hi]  # row scaling
                    res[f, lo:hi] = np.linalg.solve(Af, u[f, lo:hi])
            else:
                base = np.moveaxis(_v(j["base"], dims), 2 - ax, -1).reshape(-1, shp[-1])
                res = base + j["coef"] * np.linalg.solve(self.M, self.A @ u.T).T
            out = _v(j["out"], dims)
            out[...] = np.moveaxis(res.reshape(shp), -1, 2 - ax)

    # -- right-hand sides -------------------------------------------------------------
    def _program(self, kind, s, d):
        """[(input index, ops per axis (x, y, z), scale name, sign)] of SURVEY §8(a) a1/a3/a5/a7."""
        sig = (d + 1) % 3 if s == 1 else (d + 2) % 3
        def ops(**kw):
            o = [OP_M, OP_M, OP_M]
            for ax, op in kw.items():
                o[int(ax[1])] = op
            return o
        if kind == 0:
            t3 = [OP_M, OP_M, OP_M]
            t3[d] = OP_A
            t3[sig] = OP_B
            return [(0, [OP_M] * 3, "one", 1.0), (1, ops(**{f"a{(d + 1) % 3}": OP_A}), "a", 1.0),
                    (2, ops(**{f"a{(d + 2) % 3}": OP_A}), "a", -1.0), (3, t3, "c", 1.0)]
        if s == 1:
            return [(0, [OP_M] * 3, "one", 1.0), (1, ops(**{f"a{(d + 1) % 3}": OP_A}), "b", -1.0),
                    (2, ops(**{f"a{(d + 2) % 3}": OP_A}), "b", 1.0)]
        return [(0, [OP_M] * 3, "one", 1.0), (1, ops(**{f"a{(d + 2) % 3}": OP_A}), "b", 1.0),
                (2, ops(**{f"a{(d + 1) % 3}": OP_A}), "b", -1.0)]

    def box_rhs(self, kind, s, d, ins, nzin, zoff, kg0, nzout, a, b, c, load, sval, out):
        N = self.N
        zwin = np.arange(nzin) + kg0 - zoff  # global planes held by the inputs
        ok = (zwin >= 0) & (zwin < N)
        acc = {"one": 0.0, "a": 0.0, "b": 0.0, "c": 0.0}
        for t, opx, sc, sign in self._program(kind, s, d):
            u = ins[t].numpy().reshape(nzin, N, N)
            X, Y, Z = self.ops[opx[0]], self.ops[opx[1]], self.ops[opx[2]]
            Zr = np.zeros((nzout, nzin))
            Zr[:, ok] = Z[kg0:kg0 + nzout][:, zwin[ok]]
            v = np.einsum("kz,zyx->kyx", Zr, u)
            v = np.einsum("jy,kyx->kjx", Y, v)
            v = np.einsum("ix,kjx->kji", X, v)
            acc[sc] = acc[sc] + sign * v
        sh = (nzout, N, N)
        res = acc["one"]
        if kind == 0:
            av, cv = a.numpy().reshape(sh), c.numpy().reshape(sh)
            res = res + av * acc["a"] + cv * acc["c"]
            if load is not None and sval != 0.0:
                res = res - av * sval * load.numpy().reshape(sh)
            comp = d
        else:
            res = res + b.numpy().reshape(sh) * acc["b"]
            comp = 3 + d
        o = out.numpy().reshape(sh)
        o[...] = res
        self.box_pec(comp, out, (N, N, nzout), (0, 0, kg0))

    # -- NEXT-1: partitioned z-solve (restated from spike.cuh / adi_zsolve_tables) ------------
    def _w(self, mode, j, T, k0):
        """Right-hand side rows of the rank's active z-segment: f, or A u along z (halo'd u)."""
        g0l, m, P = T["g0"] - k0, T["m"], self.p
        if mode != 2:  # mass
            return j["in"].numpy()[g0l:g0l + m].reshape(m, -1)
        uh = j["in_h"].numpy().reshape(j["in_h"].shape[0], -1)  # planes -P .. nz+P-1
        A = self.A
        w = np.zeros((m, uh.shape[1]))
        for k in range(m):
            g = T["g0"] + k
            for q in range(-P, P + 1):
                if 0 <= g + q < self.N:
                    w[k] += A[g, g + q] * uh[g0l + k + q + P]
        return w

    def spike_tips(self, mode, jobs, tabs, k0):
        out = []
        for j in jobs:
            T = tabs[j["v"]]
            out.append(T["tw"] @ self._w(mode, j, T, k0))
        return torch.from_numpy(np.stack(out))  # [job, 2p, N*N]

    def spike_solve(self, mode, jobs, tabs, k0, gath):
        P = self.p
        G = gath.numpy()  # [R, job, 2p, N*N]
        for q, j in enumerate(jobs):
            T = tabs[j["v"]]
            g0l, m = T["g0"] - k0, T["m"]
            tb = T["q"] @ G[:, q].reshape(-1, G.shape[-1])  # rows: t_{r+1} (P), b_{r-1} (P)
            w = self._w(mode, j, T, k0).copy()
            w[:P] -= T["C"] @ tb[P:]
            w[m - P:] -= T["B"] @ tb[:P]
            fac = T["fac"]
            g = np.zeros_like(w)
            for k in range(m):  # forward elimination (l_{k,k-1-q} = fac[k, q])
                g[k] = w[k] - sum(fac[k, qq] * g[k - 1 - qq] for qq in range(P) if k - 1 - qq >= 0)
            x = np.zeros_like(w)
            for k in range(m - 1, -1, -1):  # back substitution (1/u_kk = fac[k, P], u_{k,k+1+q} = fac[k, P+1+q])
                x[k] = (g[k] - sum(fac[k, P + 1 + qq] * x[k + 1 + qq] for qq in range(P) if k + 1 + qq < m)) * fac[k, P]
            out = j["out"].numpy().reshape(j["out"].shape[0], -1)
            if mode == 2:
                base = j["base"].numpy().reshape(out.shape)[g0l:g0l + m].copy()
                out[g0l:g0l + m] = base + j["coef"] * x
            else:
                out[g0l:g0l + m] = x
            out[:g0l] = 0.0
            out[g0l + m:] = 0.0

    # -- NEXT-1 for the row-modified z sweep (restated from spike.cuh with dense per-fiber blocks) ---
    def _mod_blocks(self, T, k0, c, R, r):
        """Per fiber: A_r (m x m), C_r (p x p), B_r (p x p) of M + diag(c) S on the rank's block."""
        g0, m, P = T["g0"], T["m"], self.p
        g1 = g0 + m
        cl = c.numpy().reshape(c.shape[0], -1)[g0 - k0:g1 - k0].T  # (nf, m): c of the block rows
        M, S = self.M, self.S
        A = M[g0:g1, g0:g1][None] + cl[:, :, None] * S[g0:g1, g0:g1][None]
        C = np.zeros((cl.shape[0], P, P))
        B = np.zeros((cl.shape[0], P, P))
        if r > 0:
            C = M[g0:g0 + P, g0 - P:g0][None] + cl[:, :P, None] * S[g0:g0 + P, g0 - P:g0][None]
        if r < R - 1:
            B = M[g1 - P:g1, g1:g1 + P][None] + cl[:, m - P:, None] * S[g1 - P:g1, g1:g1 + P][None]
        return A, C, B

    def spike_mod_tips(self, j, T, k0, c, R, r):
        P, m, g0l = self.p, T["m"], T["g0"] - k0
        A, C, B = self._mod_blocks(T, k0, c, R, r)
        w = j["in"].numpy().reshape(j["in"].shape[0], -1)[g0l:g0l + m].T  # (nf, m)
        X = np.zeros((A.shape[0], m, 1 + 2 * P))
        X[:, :, 0] = w
        X[:, :P, 1:1 + P] = C
        X[:, m - P:, 1 + P:] = B
        Y = np.linalg.solve(A, X)
        tips = np.concatenate([Y[:, :P, 0], Y[:, m - P:, 0], Y[:, :P, 1:1 + P].reshape(-1, P * P),
                               Y[:, m - P:, 1:1 + P].reshape(-1, P * P), Y[:, :P, 1 + P:].reshape(-1, P * P),
                               Y[:, m - P:, 1 + P:].reshape(-1, P * P)], axis=1)
        return torch.from_numpy(np.ascontiguousarray(tips.T))  # [2P + 4P^2, nf]

    def spike_mod_solve(self, j, T, k0, c, R, r, gath):
        P, m, g0l = self.p, T["m"], T["g0"] - k0
        A, C, B = self._mod_blocks(T, k0, c, R, r)
        G = gath.numpy()  # [R, 2P + 4P^2, nf]
        nf = G.shape[2]
        nK = 2 * P * R
        K = np.tile(np.eye(nK), (nf, 1, 1))
        rhs = np.zeros((nf, nK))
        for s in range(R):
            t = G[s].T  # (nf, 2P + 4P^2)
            yt, yb = t[:, :P], t[:, P:2 * P]
            Wt, Wb, Vt, Vb = (t[:, 2 * P + q * P * P:2 * P + (q + 1) * P * P].reshape(nf, P, P) for q in range(4))
            rhs[:, 2 * P * s:2 * P * s + P] = yt
            rhs[:, 2 * P * s + P:2 * P * (s + 1)] = yb
            for rows, Vx, Wx in ((slice(2 * P * s, 2 * P * s + P), Vt, Wt), (slice(2 * P * s + P, 2 * P * (s + 1)), Vb, Wb)):
                if s + 1 < R:
                    K[:, rows, 2 * P * (s + 1):2 * P * (s + 1) + P] += Vx
                if s > 0:
                    K[:, rows, 2 * P * (s - 1) + P:2 * P * s] += Wx
        xi = np.linalg.solve(K, rhs[:, :, None])[:, :, 0]
        tn = xi[:, 2 * P * (r + 1):2 * P * (r + 1) + P] if r + 1 < R else np.zeros((nf, P))
        bp = xi[:, 2 * P * (r - 1) + P:2 * P * r] if r > 0 else np.zeros((nf, P))
        out = j["out"].numpy().reshape(j["out"].shape[0], -1)
        w = j["in"].numpy().reshape(j["in"].shape[0], -1)[g0l:g0l + m].T.copy()
        w[:, :P] -= np.einsum("fij,fj->fi", C, bp)
        w[:, m - P:] -= np.einsum("fij,fj->fi", B, tn)
        x = np.linalg.solve(A, w[:, :, None])[:, :, 0]
        out[g0l:g0l + m] = x.T
        out[:g0l] = 0.0
        out[g0l + m:] = 0.0
