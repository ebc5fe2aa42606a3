"""Multi-rank path on CPU: world_size 2 and 3 with the gloo backend.

* SlabPlan matches the library's z-slab formula (adi_layout) and covers the grid.
* Comm: halo exchange and the all-to-all z<->y transposes move exactly the right
  planes (checked against the global array).
* DistPatch: the full slab-decomposed schedule (halo exchange before the RHS
  stencils, batched local x/y sweeps, z-sweeps on y-slabs between transposes,
  uniform-mu derivative projections or the general H path, sources) driven over
  gloo with a CPU test double of the box kernels (tests/dist_backend.py) matches
  the oracle's single-domain step; the GPU path runs the same schedule with the
  CUDA box kernels over NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_06998_b200.dist import Comm, DistPatch, SlabPlan, split


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(fn, world, *args):
    port = _port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def torch_copy_box(dst, ddims, doff, src, sdims, soff, ext):
    d = dst.view(-1).view(int(ddims[2]), int(ddims[1]), int(ddims[0]))
    s = src.reshape(-1).view(int(sdims[2]), int(sdims[1]), int(sdims[0]))
    d[doff[2]:doff[2] + ext[2], doff[1]:doff[1] + ext[1], doff[0]:doff[0] + ext[0]] = \
        s[soff[2]:soff[2] + ext[2], soff[1]:soff[1] + ext[1], soff[0]:soff[0] + ext[0]]


@pytest.mark.parametrize("N,R", [(10, 1), (10, 2), (11, 3), (514, 8), (130, 8)])
def test_slab_plan(N, R):
    pl = SlabPlan(N, 2, R)
    ks = [k for r in range(R) for k in range(*pl.k[r])]
    assert ks == list(range(N))
    assert all(pl.k[r] == (r * N // R, (r + 1) * N // R) == split(N, R, r) for r in range(R))
    assert max(pl.nz(r) for r in range(R)) - min(pl.nz(r) for r in range(R)) <= 1


def _comm_worker(rank, world, N, P):
    pl = SlabPlan(N, P, world)
    g = torch.arange(N ** 3, dtype=torch.float64).view(N, N, N)  # [k, j, i]
    k0, k1 = pl.k[rank]
    nz = k1 - k0
    f = torch.zeros(nz + 2 * P, N, N, dtype=torch.float64)
    f[P:P + nz] = g[k0:k1]
    comm = Comm(pl, rank, torch_copy_box)
    comm.halo_exchange([f])
    for q in range(P):
        kb, kt = k0 - P + q, k1 + q
        assert torch.equal(f[q], g[kb] if kb >= 0 else torch.zeros(N, N))
        assert torch.equal(f[P + nz + q], g[kt] if kt < N else torch.zeros(N, N))
    j0, j1 = pl.j[rank]
    ybuf = torch.empty(N, j1 - j0, N, dtype=torch.float64)
    send = torch.empty(nz * N * N, dtype=torch.float64)
    comm.z2y(f[P:P + nz], ybuf, send)
    assert torch.equal(ybuf, g[:, j0:j1, :])
    back = torch.zeros(nz, N, N, dtype=torch.float64)
    comm.y2z(ybuf, back, send)
    assert torch.equal(back, g[k0:k1])


@pytest.mark.parametrize("world,N,P", [(2, 9, 2), (3, 11, 3)])
def test_comm_gloo(world, N, P):
    _run(_comm_worker, world, N, P)


def _step_worker(rank, world, n, p, tau, steps, mu_kind, source, outdir, zsolve=False):
    from tests.dist_backend import CpuBoxBackend

    import workloads

    N = n + p
    be = CpuBoxBackend(n, p, tau)
    D = DistPatch(n, p, tau, backend=be, rank=rank, nranks=world, zsolve=zsolve)
    eps = workloads.element_eps(n, "random", seed=5)
    mu = None if mu_kind == "uniform" else workloads.element_eps(n, "random", seed=6) / 40.0
    D.set_materials(eps, mu)
    f = [x.reshape(N, N, N) for x in workloads.random_fields(N, 13)]
    k0, k1 = D.k0, D.k1
    D.set_fields([x[k0:k1] for x in f])
    if source:
        sig = workloads.signal("pulse", tau, steps)
        D.set_source([None, None, be.O.point_load(*workloads.dipole_position(n))], sig)
    D.step(steps)
    np.save(os.path.join(outdir, f"r{rank}.npy"), np.stack([x.numpy() for x in D.get_fields()]))


@pytest.mark.parametrize("world,n,p,mu_kind,source,zsolve",
                         [(2, 6, 2, "uniform", False, False), (2, 5, 3, "random", False, False),
                          (3, 7, 2, "uniform", True, False),
                          (2, 10, 2, "uniform", True, True), (3, 13, 2, "uniform", False, True),
                          (2, 11, 3, "uniform", False, True)])
def test_dist_step_gloo(tmp_path, world, n, p, mu_kind, source, zsolve):
    """Slab-decomposed step (world ranks, gloo) == oracle single-domain step, <= 1e-10.
    zsolve: NEXT-1 partitioned z-solve of the mass sweeps / derivative projections (tables from the
    library's adi_zsolve_tables, tips all-gathered over gloo) instead of their transposes."""
    import oracle
    import workloads

    tau, steps = 0.02, 2
    _run(_step_worker, world, n, p, tau, steps, mu_kind, source, str(tmp_path), zsolve)
    N = n + p
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(world)], axis=1)  # [c, k, j, i]
    O = oracle.Patch(n, p, tau)
    O.set_materials(workloads.element_eps(n, "random", seed=5),
                    None if mu_kind == "uniform" else workloads.element_eps(n, "random", seed=6) / 40.0)
    O.set_fields(workloads.random_fields(N, 13))
    if source:
        O.set_source([None, None, O.point_load(*workloads.dipole_position(n))], workloads.signal("pulse", tau, steps))
    O.step(steps)
    ref = O.get_fields()
    for c in range(6):
        r = ref[c].reshape(N, N, N)
        err = np.linalg.norm(got[c] - r) / np.linalg.norm(r)
        assert err <= 1e-10, (c, err)


def _zsolve_worker(rank, world, n, p, lo, hi):
    """NEXT-1 host logic over gloo: each rank solves its diagonal block with the library's tables,
    all-gathers 2p tips per fiber, corrects and finishes -- equal to the global banded solve."""
    import paper_2103_06998_b200 as adi
    import oracle

    N = n + p
    M = oracle.Patch(n, p, 0.01).matrices()[0]
    rng = np.random.default_rng(7)
    F = rng.uniform(-1, 1, size=(N, 40))  # 40 fibers, rows along the partitioned axis
    T = adi.zsolve_tables(n, p, world, rank, lo, hi)
    g0, m = T["g0"], T["m"]
    assert (g0, g0 + m) == (max(rank * N // world, lo), min((rank + 1) * N // world, hi))
    # tips of y = A_r^{-1} f: the tip weights are rows of the inverse of the diagonal block
    Ar = M[g0:g0 + m, g0:g0 + m]
    Ainv = np.linalg.inv(Ar)
    assert np.allclose(T["tw"], np.concatenate([Ainv[:p], Ainv[m - p:]]), rtol=0, atol=1e-12 * abs(Ainv).max())
    w = F[g0:g0 + m]
    tips = torch.from_numpy(T["tw"] @ w)
    out = [torch.empty_like(tips) for _ in range(world)]
    dist.all_gather(out, tips)
    tb = T["q"] @ torch.stack(out).numpy().reshape(-1, F.shape[1])
    w = w.copy()
    w[:p] -= T["C"] @ tb[p:]
    w[m - p:] -= T["B"] @ tb[:p]
    x = np.linalg.solve(Ar, w)
    ref = np.linalg.solve(M[lo:hi, lo:hi], F[lo:hi])[g0 - lo:g0 - lo + m]
    assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()
    # the banded LU factors of the block (no pivoting) reproduce A_r
    fac = T["fac"]
    L, U = np.eye(m), np.zeros((m, m))
    for k in range(m):
        for q in range(p):
            if k - 1 - q >= 0:
                L[k, k - 1 - q] = fac[k, q]
        U[k, k] = 1.0 / fac[k, p]
        for q in range(p):
            if k + 1 + q < m:
                U[k, k + 1 + q] = fac[k, p + 1 + q]
    assert np.abs(L @ U - Ar).max() <= 1e-13 * np.abs(Ar).max()


@pytest.mark.parametrize("world,n,p,lo_off", [(2, 10, 2, 0), (2, 10, 2, 1), (3, 13, 2, 1), (3, 16, 3, 0), (2, 11, 1, 1)])
def test_zsolve_tables_gloo(world, n, p, lo_off):
    N = n + p
    _run(_zsolve_worker, world, n, p, lo_off, N - lo_off)


def test_zsolve_tables_reject_thin_slabs():
    import paper_2103_06998_b200 as adi

    with pytest.raises(adi.AdiError) as e:  # N = 12, 4 ranks: 3 rows each < 2p = 4
        adi.zsolve_tables(10, 2, 4, 0, 0, 12)
    assert e.value.status == adi.ADI_ERR_ARG
