"""Slab-decomposed path on one B200 with the CUDA box kernels (adi_box_*).

R = 1 through DistPatch (halo'd slab RHS, z-sweeps on the y-slab layout) and
R = 2 / 3 as threads of one process sharing cuda:0: each thread owns a box-mode
library patch (rank r of R) and its slab buffers; the exchanges go through an
in-process stand-in of torch.distributed (ThreadComm: device copies between the
threads' tensors after a host barrier -- no kernel ever waits on another
rank's kernel).  Results must match the oracle to 1e-10 and the R = 1 run bit for
bit (per-fiber arithmetic is independent of the decomposition).
"""
import threading

import numpy as np
import pytest
import torch

import oracle
import workloads
from paper_2103_06998_b200.dist import DistPatch, SlabPlan

pytestmark = pytest.mark.gpu


class ThreadComm:
    """halo_exchange / z2y / y2z of rank `rank` among threads sharing `shared`."""

    def __init__(self, plan: SlabPlan, rank: int, shared):
        self.plan, self.rank, self.sh = plan, rank, shared

    def _post(self, obj):
        torch.cuda.synchronize()
        self.sh["post"][self.rank] = obj
        self.sh["bar"].wait()

    def _done(self):
        torch.cuda.synchronize()
        self.sh["bar"].wait()

    def halo_exchange(self, fields):
        pl, r, P = self.plan, self.rank, self.plan.p
        nz = pl.nz(r)
        self._post(fields)
        if r > 0:
            nb = self.sh["post"][r - 1]
            nzb = pl.nz(r - 1)
            for f, g in zip(fields, nb):
                f[0:P].copy_(g[nzb:nzb + P])
        if r < pl.R - 1:
            nb = self.sh["post"][r + 1]
            for f, g in zip(fields, nb):
                f[nz + P:nz + 2 * P].copy_(g[P:2 * P])
        self._done()

    def z2y(self, src, dst, sendbuf):
        pl, r = self.plan, self.rank
        j0, j1 = pl.j[r]
        self._post(src)
        for q in range(pl.R):
            k0, k1 = pl.k[q]
            dst[k0:k1].copy_(self.sh["post"][q][:, j0:j1, :])
        self._done()

    def y2z(self, src, dst, recvbuf):
        pl, r = self.plan, self.rank
        k0, k1 = pl.k[r]
        self._post(src)
        for q in range(pl.R):
            j0, j1 = pl.j[q]
            dst[:, j0:j1, :].copy_(self.sh["post"][q][k0:k1])
        self._done()


def run_ranks(R, n, p, tau, steps, mu_kind="uniform", source=False):
    N = n + p
    shared = {"bar": threading.Barrier(R), "post": [None] * R}
    out = [None] * R
    err = []
    eps = workloads.element_eps(n, "phantom4" if n >= 8 else "random", seed=4)
    mu = None if mu_kind == "uniform" else workloads.element_eps(n, "random", seed=6) / 40.0
    f = [x.reshape(N, N, N) for x in workloads.random_fields(N, 17)]

    def work(r):
        try:
            torch.cuda.set_device(0)
            plan = SlabPlan(N, p, R)
            D = DistPatch(n, p, tau, rank=r, nranks=R, comm=ThreadComm(plan, r, shared) if R > 1 else None)
            D.set_materials(eps, mu)
            D.set_fields([torch.from_numpy(np.ascontiguousarray(x[D.k0:D.k1])) for x in f])
            if source:
                O = oracle.Patch(n, p, tau)
                D.set_source([None, None, O.point_load(*workloads.dipole_position(n))],
                             workloads.signal("modsine", tau, steps))
            D.step(steps)
            torch.cuda.synchronize()
            out[r] = np.stack([x.cpu().numpy() for x in D.get_fields()])
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            shared["bar"].abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return np.concatenate(out, axis=1), eps, mu, f


def oracle_ref(n, p, tau, steps, eps, mu, f, source=False):
    O = oracle.Patch(n, p, tau)
    O.set_materials(eps, mu)
    O.set_fields([x.reshape(-1) for x in f])
    if source:
        O.set_source([None, None, O.point_load(*workloads.dipole_position(n))], workloads.signal("modsine", tau, steps))
    O.step(steps)
    return [x.reshape(n + p, n + p, n + p) for x in O.get_fields()]


@pytest.mark.parametrize("R,n,p,mu_kind,source", [(1, 10, 2, "uniform", False), (2, 10, 2, "uniform", True),
                                                  (3, 9, 3, "uniform", False), (2, 8, 2, "random", False)])
def test_dist_threads_match_oracle(R, n, p, mu_kind, source):
    tau, steps = 0.02, 2
    got, eps, mu, f = run_ranks(R, n, p, tau, steps, mu_kind, source)
    ref = oracle_ref(n, p, tau, steps, eps, mu, f, source)
    for c in range(6):
        e = np.linalg.norm(got[c] - ref[c]) / np.linalg.norm(ref[c])
        assert e <= 1e-10, (c, e)


def test_dist_decomposition_invariance_bitwise():
    """R = 1, 2, 4 slab decompositions give bit-identical fields."""
    outs = [run_ranks(R, 14, 2, 0.01, 2)[0] for R in (1, 2, 4)]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_box_mode_abi_contract():
    """Box-mode patch (nranks > 1): layout = balanced z-slab; whole-patch calls are
    ADI_ERR_STATE; box calls validate their arguments (ADI_ERR_ARG)."""
    import paper_2103_06998_b200 as adi

    n, p = 10, 2
    N = n + p
    for r in range(3):
        B = adi.Patch(n, p, 0.01, rank=r, nranks=3)
        assert B.layout() == (N, r * N // 3, (r + 1) * N // 3)
    B = adi.Patch(n, p, 0.01, rank=1, nranks=3)
    with pytest.raises(adi.AdiError) as e:
        B.step(1)
    assert e.value.status == adi.ADI_ERR_STATE
    with pytest.raises(adi.AdiError) as e:
        B.set_fields([np.zeros(B.local_count)] * 6)
    assert e.value.status == adi.ADI_ERR_STATE
    t = torch.zeros(N, N, 4, dtype=torch.float64, device="cuda")
    with pytest.raises(adi.AdiError) as e:  # dims[axis] must equal N
        B.box_sweep(0, [dict(dims=(N, N, 4), axis=2, comp=3, **{"in": t}, out=t)])
    assert e.value.status == adi.ADI_ERR_ARG
    with pytest.raises(adi.AdiError) as e:  # box outside the array
        B.box_copy(t, (N, N, 4), (0, 0, 1), t, (N, N, 4), (0, 0, 0), (N, N, 4))
    assert e.value.status == adi.ADI_ERR_ARG
    with pytest.raises(adi.AdiError) as e:
        B.box_rhs(0, 3, 0, [t] * 4, 4, 0, 0, 4, t, t, t, None, 0.0, t)
    assert e.value.status == adi.ADI_ERR_ARG
    with pytest.raises(adi.AdiError):
        adi.Patch(n, p, 0.01, rank=3, nranks=3)


# ---------------------------------------------------------------------------
# The library's own distributed schedule (adi_step with nranks > 1) over the in-process
# loopback transport: R host threads, one patch each, on cuda:0.
# ---------------------------------------------------------------------------
def run_loopback(R, n, p, tau, steps, mu_kind="uniform", source=False, eps_kind="phantom4", seed=17, zsolve=0,
                 active=None):
    import paper_2103_06998_b200 as adi

    N = n + p
    eps = workloads.element_eps(n, eps_kind, seed=4)
    mu = None if mu_kind == "uniform" else workloads.element_eps(n, "random", seed=6) / 40.0
    f = [x.reshape(N, N, N) for x in workloads.random_fields(N, seed)]
    sig = workloads.signal("modsine", tau, steps) if source else None
    pos = workloads.dipole_position(n)
    if R == 1:
        G = adi.Patch(n, p, tau)
        G.set_materials(eps, mu)
        G.set_fields([x.reshape(-1) for x in f])
        if source:
            G.set_point_source(2, pos, sig)
        G.step(steps)
        return np.stack([x.reshape(N, N, N) for x in G.get_fields()]), eps, mu, f, [None]
    grp = adi.Loopback(R)
    out, err, launches = [None] * R, [], [None] * R

    def work(r):
        try:
            P = adi.Patch(n, p, tau, device=0, rank=r, nranks=R, loopback=grp)
            act = P.set_zsolve(zsolve)
            if active is not None:
                active[r] = act
            Nn, k0, k1 = P.layout()
            P.set_materials(eps, mu)
            P.set_fields([np.ascontiguousarray(x[k0:k1]).reshape(-1) for x in f])
            if source:
                P.set_point_source(2, pos, sig)
            P.step(steps)
            out[r] = np.stack([x.reshape(k1 - k0, N, N) for x in P.get_fields()])
            launches[r] = P.launches_per_step
            P.close()
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    grp.close()
    if err:
        raise err[0]
    return np.concatenate(out, axis=1), eps, mu, f, launches


@pytest.mark.parametrize("R,n,p,mu_kind,source", [(2, 10, 2, "uniform", True), (3, 9, 3, "uniform", False),
                                                  (2, 8, 2, "random", False), (4, 14, 2, "uniform", False)])
def test_library_distributed_step_matches_oracle(R, n, p, mu_kind, source):
    """adi_step of R slab patches (the library's distributed schedule: halo exchange, z sweeps on
    y-slabs between batched transposes; loopback transport) == the oracle's single-domain step."""
    tau, steps = 0.02, 2
    got, eps, mu, f, _ = run_loopback(R, n, p, tau, steps, mu_kind, source)
    ref = oracle_ref(n, p, tau, steps, eps, mu, f, source)
    for c in range(6):
        e = np.linalg.norm(got[c] - ref[c]) / np.linalg.norm(ref[c])
        assert e <= 1e-10, (c, e)


@pytest.mark.parametrize("R,n,p,mu_kind,source", [(2, 10, 2, "uniform", True), (3, 22, 3, "uniform", False),
                                                  (2, 12, 2, "random", False), (4, 30, 2, "uniform", True),
                                                  (3, 13, 1, "uniform", False)])
def test_library_partitioned_zsolve_matches_oracle(R, n, p, mu_kind, source):
    """NEXT-1: the mass sweeps and derivative projections along the partitioned axis
    solved in place by the SPIKE z-solve (tips, all-gather of 2p values per fiber, corrected segment
    solve; no transposes for them) == the oracle's single-domain step (D16, <= 1e-10 per field), and
    == the whole patch to 1e-12 (the partitioned solve reorders the rounding only)."""
    tau, steps = 0.02, 3
    act = [None] * R
    got, eps, mu, f, _ = run_loopback(R, n, p, tau, steps, mu_kind, source, zsolve=1, active=act)
    assert all(act), act
    ref = oracle_ref(n, p, tau, steps, eps, mu, f, source)
    whole = run_loopback(1, n, p, tau, steps, mu_kind, source)[0]
    for c in range(6):
        e = np.linalg.norm(got[c] - ref[c]) / np.linalg.norm(ref[c])
        w = np.linalg.norm(got[c] - whole[c]) / np.linalg.norm(whole[c])
        assert e <= 1e-10 and w <= 1e-12, (c, e, w)


def test_partitioned_zsolve_falls_back_when_slabs_are_thin():
    """A rank with fewer than 2p active rows cannot host the p-row interface blocks: mode 1 reports
    inactive and the step keeps the transposes (still == the oracle)."""
    act = [None] * 3
    tau, steps = 0.02, 1
    got, eps, mu, f, _ = run_loopback(3, 9, 3, tau, steps, zsolve=1, active=act)
    assert not any(act)
    ref = oracle_ref(9, 3, tau, steps, eps, mu, f)
    for c in range(6):
        assert np.linalg.norm(got[c] - ref[c]) <= 1e-10 * np.linalg.norm(ref[c])


def test_library_distributed_bitwise_vs_whole_patch():
    """R = 2, 3, 4 slab decompositions through adi_step are bit-identical to the
    whole-patch step (per-fiber arithmetic does not depend on the decomposition); even N = 36 so
    the TMA-staged sweeps run on both layouts, with a source."""
    outs = [run_loopback(R, 34, 2, 0.01, 3, source=True)[0] for R in (1, 2, 3, 4)]
    for R, o in zip((2, 3, 4), outs[1:]):
        assert np.array_equal(o, outs[0]), R


def test_library_distributed_contract():
    """Distributed-mode contract: layout = balanced z-slab; set/get_fields take the local slab;
    both transports at once is ADI_ERR_ARG; a loopback group of the wrong size is ADI_ERR_ARG."""
    import paper_2103_06998_b200 as adi

    n, p = 10, 2
    N = n + p
    grp = adi.Loopback(2)
    with pytest.raises(adi.AdiError) as e:
        adi.Patch(n, p, 0.01, rank=0, nranks=3, loopback=grp)
    assert e.value.status == adi.ADI_ERR_ARG
    with pytest.raises(adi.AdiError) as e:
        adi.Patch(n, p, 0.01, rank=0, nranks=2, loopback=grp, nccl_id=bytes(128))
    assert e.value.status == adi.ADI_ERR_ARG
    P = adi.Patch(n, p, 0.01, rank=1, nranks=2, loopback=grp)
    assert P.layout() == (N, N // 2, N)
    assert P.local_count == N * N * (N - N // 2)
    with pytest.raises(ValueError):
        P.set_fields([np.zeros(N ** 3)] * 6)
    with pytest.raises(adi.AdiError) as e:
        P.step(1)
    assert e.value.status == adi.ADI_ERR_STATE
    P.close()
    grp.close()
