"""Slab-decomposed ADI step across GPUs.

The product path is the library's own distributed schedule (``adi_step`` on a patch created
with ``nranks > 1`` and an NCCL unique id, include/adi_maxwell.h): ``create_patch`` below only
broadcasts the id over ``torch.distributed`` and creates this rank's patch.

``DistPatch`` is the same schedule written out in Python over the library's box-level calls
(``adi_box_*``); it drives the gloo CPU tests (tests/test_dist_cpu.py, with a CPU test double
of the box kernels) and documents the orchestration step by step:

One process per GPU.  Rank r of R owns the z-planes [r N / R, (r+1) N / R) of the
global N^3 coefficient grid (``adi_layout``).  Per substep:

  * halo exchange: p planes of each E/H field from both z-neighbours
    (``batch_isend_irecv``), before the RHS stencil (a1/a5; a3/a7 on the
    general-mu path) -- the only coupling of the stencils;
  * x- and y-sweeps are local (fibers lie in a z-plane);
  * every z-sweep runs on a y-slab: an all-to-all transpose (z-slab -> y-slab,
    rank s receives rows [s N / R, (s+1) N / R) of y for all z), the sweep, and
    the transpose back.  Per-fiber arithmetic is unchanged, so the result is
    independent of R bit for bit except for the order of nothing: each fiber is
    solved by the same kernel with the same inputs.

All arithmetic runs in the library's kernels through the box-level C ABI
(``adi_box_*``: RHS on a slab with halos, batched sweeps on arbitrary boxes,
pivot caches, strided box copies for packing); this module is orchestration and
``torch.distributed`` plumbing.  The collectives are device-agnostic: NCCL on
CUDA tensors in production; the CPU tests drive the same schedule with gloo and
a test double of the kernels (tests/test_dist_cpu.py).
"""
from __future__ import annotations

import torch

try:
    import torch.distributed as tdist
except Exception:  # pragma: no cover
    tdist = None


def create_patch(n: int, p: int, tau: float, bc: int = 0, device: int | None = None, group=None):
    """This rank's patch of a distributed run: rank 0 creates the NCCL unique id
    (adi_nccl_unique_id), every rank receives it over torch.distributed and creates its z-slab
    patch; the library then owns the NCCL communicator and runs every exchange itself."""
    import paper_2103_06998_b200 as adi

    rank, R = tdist.get_rank(group), tdist.get_world_size(group)
    obj = [adi.nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(obj, src=0, group=group)
    if device is None:
        device = torch.cuda.current_device()
    return adi.Patch(n, p, tau, bc, device=device, rank=rank, nranks=R, nccl_id=obj[0])


def split(N: int, R: int, r: int):
    """Balanced partition of [0, N) into R parts: part r = [r N / R, (r+1) N / R)."""
    return r * N // R, (r + 1) * N // R


class SlabPlan:
    """z-slabs (the resident layout) and y-slabs (the layout of z-sweeps)."""

    def __init__(self, N: int, p: int, R: int):
        if R > N:
            raise ValueError(f"{R} ranks for {N} planes")
        self.N, self.p, self.R = N, p, R
        self.k = [split(N, R, r) for r in range(R)]
        self.j = [split(N, R, r) for r in range(R)]

    def nz(self, r):
        return self.k[r][1] - self.k[r][0]

    def ny(self, r):
        return self.j[r][1] - self.j[r][0]


class Comm:
    """Halo exchange and z<->y transposes of one rank.

    copy_box(dst, ddims, doff, src, sdims, soff, ext) performs the strided packing
    (the library's ``adi_box_copy`` kernel on GPUs).  Tensors are flat-contiguous
    with x fastest; a z-slab field with halos has shape (nz + 2p, N, N)."""

    def __init__(self, plan: SlabPlan, rank: int, copy_box, group=None):
        self.plan, self.rank, self.copy_box, self.group = plan, rank, copy_box, group
        self.R = plan.R

    # -- halo exchange ------------------------------------------------------------
    def halo_exchange(self, fields):
        """fields: tensors (nz + 2p, N, N); planes [p, p + nz) are the rank's own.
        Planes [0, p) receive the last p planes of rank - 1, [nz + p, nz + 2p) the
        first p planes of rank + 1; at the patch ends they stay zero."""
        P, r, R = self.plan.p, self.rank, self.R
        nz = self.plan.nz(r)
        if R == 1 or P == 0:
            return
        ops = []
        for f in fields:
            if r > 0:
                ops.append(tdist.P2POp(tdist.isend, f[P:2 * P], r - 1, self.group))
                ops.append(tdist.P2POp(tdist.irecv, f[0:P], r - 1, self.group))
            if r < R - 1:
                ops.append(tdist.P2POp(tdist.isend, f[nz:nz + P], r + 1, self.group))
                ops.append(tdist.P2POp(tdist.irecv, f[nz + P:nz + 2 * P], r + 1, self.group))
        for req in tdist.batch_isend_irecv(ops):
            req.wait()

    # -- NEXT-1: interface tips of the partitioned z-solve ---------------------------
    def allgather(self, t):
        """[R, *t.shape]: every rank's t (the 2p tips per fiber of the partitioned z-solve)."""
        if self.R == 1:
            return t.unsqueeze(0).clone()
        out = [torch.empty_like(t) for _ in range(self.R)]
        tdist.all_gather(out, t.contiguous(), group=self.group)
        return torch.stack(out)

    # -- transposes ---------------------------------------------------------------
    def z2y(self, src, dst, sendbuf):
        """src: own z-slab (nz, N, N) -> dst: own y-slab (N, ny, N)."""
        pl, r = self.plan, self.rank
        N, nz = pl.N, pl.nz(r)
        if self.R == 1:
            self.copy_box(dst, (N, N, N), (0, 0, 0), src, (N, N, nz), (0, 0, 0), (N, N, N))
            return
        off = 0
        for s in range(self.R):
            ny_s = pl.ny(s)
            blk = sendbuf.view(-1)[off:off + nz * ny_s * N]
            self.copy_box(blk, (N, ny_s, nz), (0, 0, 0), src, (N, N, nz), (0, pl.j[s][0], 0), (N, ny_s, nz))
            off += nz * ny_s * N
        ny = pl.ny(r)
        tdist.all_to_all_single(dst.view(-1), sendbuf.view(-1)[:off],
                                output_split_sizes=[pl.nz(q) * ny * N for q in range(self.R)],
                                input_split_sizes=[nz * pl.ny(s) * N for s in range(self.R)], group=self.group)

    def y2z(self, src, dst, recvbuf):
        """src: own y-slab (N, ny, N) -> dst: own z-slab (nz, N, N)."""
        pl, r = self.plan, self.rank
        N, nz, ny = pl.N, pl.nz(r), pl.ny(r)
        if self.R == 1:
            self.copy_box(dst, (N, N, nz), (0, 0, 0), src, (N, N, N), (0, 0, 0), (N, N, N))
            return
        total = nz * N * N
        tdist.all_to_all_single(recvbuf.view(-1)[:total], src.view(-1),
                                output_split_sizes=[nz * pl.ny(s) * N for s in range(self.R)],
                                input_split_sizes=[pl.nz(q) * ny * N for q in range(self.R)], group=self.group)
        off = 0
        for s in range(self.R):
            ny_s = pl.ny(s)
            blk = recvbuf.view(-1)[off:off + nz * ny_s * N]
            self.copy_box(dst, (N, N, nz), (0, pl.j[s][0], 0), blk, (N, ny_s, nz), (0, 0, 0), (N, ny_s, nz))
            off += nz * ny_s * N


def stiff_axis(s: int, d: int) -> int:
    """Stiffened axis of E component d in substep s: K1 E1->y, E2->z, E3->x;
    K2 E1->z, E2->x, E3->y."""
    return (d + 1) % 3 if s == 1 else (d + 2) % 3


MASS, MOD, DER = 0, 1, 2


class DistPatch:
    """One rank's z-slab of an n x n x n patch; the step runs on all ranks together.

    backend: an object with the box-level methods of ``paper_2103_06998_b200.Patch``
    (box_rhs, box_sweep, box_factor, box_copy, box_abc, box_pec, box_materials_tf);
    by default the library patch of this rank (CUDA; no other backend in the product)."""

    def __init__(self, n: int, p: int, tau: float, bc: int = 0, group=None, backend=None, device=None,
                 rank: int | None = None, nranks: int | None = None, comm=None, zsolve: bool = False):
        if rank is None:
            if tdist is not None and tdist.is_available() and tdist.is_initialized():
                rank, nranks = tdist.get_rank(group), tdist.get_world_size(group)
            else:
                rank, nranks = 0, 1
        self.rank, self.R = rank, nranks
        self.n, self.p, self.tau, self.bc = n, p, tau, bc
        self.N = N = n + p
        self.plan = SlabPlan(N, p, nranks)
        self.stream = None
        if backend is None:
            import paper_2103_06998_b200 as adi
            if device is None:
                device = torch.cuda.current_device()
            # one CUDA stream for everything of this rank: the library's kernels, torch's
            # copies and the NCCL collectives (which order themselves after the current stream)
            self.stream = torch.cuda.Stream(device)
            backend = adi.Patch(n, p, tau, bc, device=device, rank=rank, nranks=nranks, stream=self.stream.cuda_stream)
            self.device = torch.device("cuda", device)
        else:
            self.device = torch.device("cpu")
        self.B = backend
        # comm: the exchange layer (torch.distributed by default; tests may inject another
        # object with halo_exchange / z2y / y2z)
        self.comm = comm if comm is not None else Comm(self.plan, rank, backend.box_copy, group)
        self.k0, self.k1 = self.plan.k[rank]
        self.nz, self.ny = self.plan.nz(rank), self.plan.ny(rank)
        nz, ny, P = self.nz, self.ny, p
        z = lambda *shape: torch.zeros(shape, dtype=torch.float64, device=self.device)  # noqa: E731
        self.F = [z(nz + 2 * P, N, N) for _ in range(6)]   # E1 E2 E3 H1 H2 H3 with z-halos
        self.Rb = [z(nz + 2 * P, N, N) for _ in range(3)]  # new E
        self.Gb = [z(nz + 2 * P, N, N) for _ in range(3)]  # new H
        self.Y = [z(N, ny, N) for _ in range(4)]           # y-slab work buffers
        self.sendbuf = z(nz * N * N)
        self.a, self.b, self.c = z(nz, N, N), z(nz, N, N), z(nz, N, N)
        self.cy = z(N, ny, N)
        self.iu = {}
        self.mu_uniform, self.b_scalar = True, tau / 2.0
        self.loads = [None, None, None]
        self.signal = None
        self.step_index = 0
        if self.stream is not None:
            # the buffers above were allocated and zero-filled on the current stream; every later
            # use is on self.stream, so order it after those fills
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
        # NEXT-1 (opt-in here; the library's own distributed step defaults to it): mass sweeps and
        # derivative projections along z by the partitioned solve (tables from adi_zsolve_tables;
        # the backend provides spike_tips / spike_solve), no transposes for them
        self.ztab = None
        if zsolve:
            import paper_2103_06998_b200 as adi
            self.ztab = {0: adi.zsolve_tables(n, p, nranks, rank, 0, N)}
            if bc == 0:
                self.ztab[1] = adi.zsolve_tables(n, p, nranks, rank, 1, N - 1)
        self.set_materials_tf(torch.ones(N ** 3, dtype=torch.float64, device=self.device), None)

    def _on_stream(self):
        import contextlib
        return torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext()

    # -- layout helpers -------------------------------------------------------------
    def inner(self, t):
        return t[self.p:self.p + self.nz]

    @property
    def zdims(self):
        return (self.N, self.N, self.nz)

    @property
    def ydims(self):
        return (self.N, self.ny, self.N)

    # -- setup ----------------------------------------------------------------------
    def set_materials(self, eps_elem, mu_elem=None):
        with self._on_stream():
            return self._set_materials(eps_elem, mu_elem)

    def _set_materials(self, eps_elem, mu_elem=None):
        """Element-wise eps, mu (global n^3 arrays, given on every rank) -> eps^, mu^ (D6)."""
        N = self.N
        eps_tf = torch.empty(N ** 3, dtype=torch.float64, device=self.device)
        mu_tf = torch.empty(N ** 3, dtype=torch.float64, device=self.device)
        self.B.box_materials_tf(eps_elem, mu_elem, eps_tf, mu_tf)
        self._set_materials_tf(eps_tf, mu_tf)

    def set_materials_tf(self, eps_tf, mu_tf=None):
        with self._on_stream():
            return self._set_materials_tf(eps_tf, mu_tf)

    def _set_materials_tf(self, eps_tf, mu_tf=None):
        """Per-test-function eps^, mu^ (global N^3 arrays on every rank)."""
        N, nz, ny = self.N, self.nz, self.ny
        eps_tf = torch.as_tensor(eps_tf, dtype=torch.float64).to(self.device).reshape(-1)
        mu_tf = (torch.ones_like(eps_tf) if mu_tf is None else
                 torch.as_tensor(mu_tf, dtype=torch.float64).to(self.device).reshape(-1))
        if not bool((eps_tf > 0).all()) or not bool((mu_tf > 0).all()):
            raise ValueError("eps, mu must be > 0 (P:81)")
        ez, mz = (torch.empty(nz, N, N, dtype=torch.float64, device=self.device) for _ in range(2))
        self.B.box_copy(ez, self.zdims, (0, 0, 0), eps_tf, (N, N, N), (0, 0, self.k0), self.zdims)
        self.B.box_copy(mz, self.zdims, (0, 0, 0), mu_tf, (N, N, N), (0, 0, self.k0), self.zdims)
        self.B.box_abc(ez, mz, nz * N * N, self.a, self.b, self.c)
        ey, my = (torch.empty(N, ny, N, dtype=torch.float64, device=self.device) for _ in range(2))
        j0 = self.plan.j[self.rank][0]
        self.B.box_copy(ey, self.ydims, (0, 0, 0), eps_tf, (N, N, N), (0, j0, 0), self.ydims)
        self.B.box_copy(my, self.ydims, (0, 0, 0), mu_tf, (N, N, N), (0, j0, 0), self.ydims)
        scratch_a, scratch_b = torch.empty_like(ey), torch.empty_like(ey)
        self.B.box_abc(ey, my, ny * N * N, scratch_a, scratch_b, self.cy)
        mu_min, mu_max = float(mu_tf.min()), float(mu_tf.max())
        self.mu_uniform = mu_min == mu_max
        self.b_scalar = self.tau / (2.0 * mu_min)
        # pivot caches of the six row-modified families, in the layout their sweep runs in
        self.iu = {}
        for s in (1, 2):
            for d in range(3):
                ax = stiff_axis(s, d)
                if ax == 2:
                    iu = torch.empty(N, ny, N, dtype=torch.float64, device=self.device)
                    self.B.box_factor(d, ax, self.ydims, self.cy, iu)
                else:
                    iu = torch.empty(nz, N, N, dtype=torch.float64, device=self.device)
                    self.B.box_factor(d, ax, self.zdims, self.c, iu)
                self.iu[(s, d)] = iu

    def set_fields(self, fields):
        with self._on_stream():
            return self._set_fields(fields)

    def _set_fields(self, fields):
        """Six local z-slabs (nz, N, N) (or flat), E1..H3; PEC entries forced to 0 (D1)."""
        for c in range(6):
            src = torch.as_tensor(fields[c], dtype=torch.float64).to(self.device).reshape(self.nz, self.N, self.N)
            self.inner(self.F[c]).copy_(src)
            self.B.box_pec(c, self.inner(self.F[c]), self.zdims, (0, 0, self.k0))

    def get_fields(self):
        with self._on_stream():
            out = [self.inner(f).clone() for f in self.F]
        if self.stream is not None:
            self.stream.synchronize()
        return out

    def set_source(self, loads, signal):
        with self._on_stream():
            return self._set_source(loads, signal)

    def _set_source(self, loads, signal):
        """loads: three global N^3 load vectors or None (D9); signal[m] = s((m+1/2) tau)."""
        N = self.N
        self.loads = [None, None, None]
        for d in range(3):
            if loads[d] is None:
                continue
            g = torch.as_tensor(loads[d], dtype=torch.float64).to(self.device).reshape(-1)
            loc = torch.empty(self.nz, N, N, dtype=torch.float64, device=self.device)
            self.B.box_copy(loc, self.zdims, (0, 0, 0), g, (N, N, N), (0, 0, self.k0), self.zdims)
            self.loads[d] = loc
        self.signal = None if signal is None else [float(x) for x in signal]

    # -- the step -------------------------------------------------------------------
    def _zsweep(self, mode, jobs_z):
        """Sweeps along z: transpose in, one batched launch on the y-slab, transpose back.
        jobs_z: dicts with 'comp', 'in' (z-slab), 'out' (z-slab) [, 'iu', 'base', 'coef']."""
        if not jobs_z:
            return
        if self.ztab is not None and mode == MOD:
            # per-fiber matrix: tips of y, W and V from the rank's block, all-gathered, the interface
            # system solved per fiber (NEXT-1 for the row-modified z sweep)
            for j in jobs_z:
                j["v"] = 1 if (self.bc == 0 and j["comp"] < 2) else 0
                tips = self.B.spike_mod_tips(j, self.ztab[j["v"]], self.k0, self.c, self.R, self.rank)
                self.B.spike_mod_solve(j, self.ztab[j["v"]], self.k0, self.c, self.R, self.rank,
                                       self.comm.allgather(tips))
            return
        if self.ztab is not None and mode != MOD:
            if mode == DER:  # A u along z reads p planes beyond the slab
                self.comm.halo_exchange([j["in_h"] for j in jobs_z])
            for j in jobs_z:
                j["v"] = 1 if (self.bc == 0 and j["comp"] < 2) else 0
            tips = self.B.spike_tips(mode, jobs_z, self.ztab, self.k0)
            self.B.spike_solve(mode, jobs_z, self.ztab, self.k0, self.comm.allgather(tips))
            return
        jobs = []
        for q, j in enumerate(jobs_z):
            self.comm.z2y(j["in"], self.Y[q], self.sendbuf)
            job = dict(dims=self.ydims, axis=2, comp=j["comp"])
            job["in"] = self.Y[q]
            job["out"] = self.Y[q]
            if mode == MOD:
                job["c"], job["iu"] = self.cy, j["iu"]
            if mode == DER:
                self.comm.z2y(j["base"], self.Y[3], self.sendbuf)
                job["base"], job["coef"], job["out"] = self.Y[3], j["coef"], self.Y[3]
                self.B.box_sweep(mode, [job])
                self.comm.y2z(self.Y[3], j["out"], self.sendbuf)
                continue
            jobs.append((job, j["out"]))
        if jobs:
            self.B.box_sweep(mode, [jb for jb, _ in jobs])
            for q, (jb, out) in enumerate(jobs):
                self.comm.y2z(jb["out"], out, self.sendbuf)

    def _sweeps(self, mode, jobs):
        """jobs: dicts with 'axis', 'comp', 'in', 'out' (z-slab views) [, 'iu', 'base', 'coef']."""
        local = []
        for j in jobs:
            if j["axis"] != 2:
                job = dict(j, dims=self.zdims)
                if mode == MOD:
                    job["c"] = self.c
                local.append(job)
        if local:
            self.B.box_sweep(mode, local)
        self._zsweep(mode, [j for j in jobs if j["axis"] == 2])

    def substep(self, s: int):
        P, nz = self.p, self.nz
        F, Rb, Gb = self.F, self.Rb, self.Gb
        self.comm.halo_exchange(F)
        sval = 0.0
        if self.signal is not None and self.step_index < len(self.signal):
            sval = self.signal[self.step_index]
        # a1 / a5: RHS of the three E systems (halo'd inputs, program order E_d, H_{d+2}, H_{d+1}, E_sigma)
        for d in range(3):
            ins = [F[d], F[3 + (d + 2) % 3], F[3 + (d + 1) % 3], F[stiff_axis(s, d)]]
            self.B.box_rhs(0, s, d, ins, nz + 2 * P, P, self.k0, nz, self.a, self.b, self.c, self.loads[d], sval,
                           self.inner(Rb[d]))
        # a2 / a6: stiffened (row-modified) sweep first, then the mass sweeps in ascending axis order (D7)
        E_new = [self.inner(Rb[d]) for d in range(3)]
        self._sweeps(MOD, [dict(axis=stiff_axis(s, d), comp=d, **{"in": E_new[d]}, out=E_new[d],
                                iu=self.iu[(s, d)]) for d in range(3)])
        for stage in range(2):
            jobs = []
            for d in range(3):
                axes = [a for a in range(3) if a != stiff_axis(s, d)]
                jobs.append(dict(axis=axes[stage], comp=d, **{"in": E_new[d]}, out=E_new[d]))
            self._sweeps(MASS, jobs)
        Eo = [self.inner(F[d]) for d in range(3)]
        if self.mu_uniform:
            # a3+a4 / a7+a8 for uniform mu: H_D' = H_D -+ b D_a1 Eo_X +- b D_a2 En_Y (exact identity)
            b = self.b_scalar
            jobs = []
            for d in range(3):
                a1 = (d + 1) % 3 if s == 1 else (d + 2) % 3
                x1 = (d + 2) % 3 if s == 1 else (d + 1) % 3
                jobs.append(dict(axis=a1, comp=3 + d, **{"in": Eo[x1]}, out=self.inner(Gb[d]),
                                 base=self.inner(F[3 + d]), coef=-b if s == 1 else b, in_h=F[x1]))
            self._sweeps(DER, jobs)
            jobs = []
            for d in range(3):
                a2 = (d + 2) % 3 if s == 1 else (d + 1) % 3
                x2 = (d + 1) % 3 if s == 1 else (d + 2) % 3
                jobs.append(dict(axis=a2, comp=3 + d, **{"in": E_new[x2]}, out=self.inner(Gb[d]),
                                 base=self.inner(Gb[d]), coef=b if s == 1 else -b, in_h=Rb[x2]))
            self._sweeps(DER, jobs)
        else:
            # general mu: G from discrete2/discrete4 (needs halos of the new E), then M^-3
            self.comm.halo_exchange(Rb)
            for d in range(3):
                if s == 1:
                    ins = [F[3 + d], F[(d + 2) % 3], Rb[(d + 1) % 3]]
                else:
                    ins = [F[3 + d], F[(d + 1) % 3], Rb[(d + 2) % 3]]
                self.B.box_rhs(1, s, d, ins, nz + 2 * P, P, self.k0, nz, self.a, self.b, self.c, None, 0.0,
                               self.inner(Gb[d]))
            for ax in range(3):
                self._sweeps(MASS, [dict(axis=ax, comp=3 + d, **{"in": self.inner(Gb[d])}, out=self.inner(Gb[d]))
                                    for d in range(3)])
        for d in range(3):
            F[d], Rb[d] = Rb[d], F[d]
            F[3 + d], Gb[d] = Gb[d], F[3 + d]
        # the halo planes of the swapped-in buffers are refreshed by the next exchange

    def step(self, k: int = 1):
        with self._on_stream():
            self._step(k)

    def _step(self, k: int):
        for _ in range(int(k)):
            self.substep(1)
            self.substep(2)
            self.step_index += 1
