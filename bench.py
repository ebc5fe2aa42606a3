#!/usr/bin/env python
"""Benchmark of the ADI-IGA Maxwell time step (arXiv 2103.06998) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Prints ONE JSON line (rank 0).  Metric (BASELINE.json): field DOF-updates/s per
time step (fp64) and the HBM roofline fraction of the dominant kernel class.

Workload: BASELINE config c5 (512^3 elements, p=2, seeded ellipsoid phantom with
per-voxel eps_r ~ U[1,80], mu_r=1, tau=1e-2) -- the configuration the metric's
"1/2/4/8 B200" is quoted on; it fits one B200 (~23 GB).  Inputs: seeded
synthetic (workloads/), every field 1.09 GB >> 126 MB L2 (no L2 flush needed).

Timed region: W untimed warm-up steps, then EXACTLY K steps bracketed by
barrier + cudaDeviceSynchronize, timed with CUDA events on the library's
stream; each kernel launch is bracketed by CUDA events on the same stream
(adi_set_timing) for the per-kernel roofline.  nvidia-smi clocks are sampled
during the timed region.

--impl reference runs the CPU oracle (oracle/, plain C, one core) on a bounded
sample of the same workload (this tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")
METRIC = "field DOF-updates/sec per time step (fp64) at 1/2/4/8 B200 and % of HBM roofline"
UNIT = "DOF-updates/s"
FALLBACK_HBM = 6650.0


def dof_count(n: int, p: int) -> int:
    """Free coefficients of the six fields under PEC (D1): 3 N (N-2)^2 + 3 N^3."""
    N = n + p
    return 3 * N * (N - 2) ** 2 + 3 * N ** 3


def step_class_bytes(n: int, p: int, mu_uniform: bool = True, fused_h: bool = True):
    """Algorithmic HBM bytes of one time step per kernel class, in SURVEY.md §8(a)/§8(d)'s
    counting (compulsory traffic of each hot-path step, independent of how many launches the
    schedule spends on it).  U = N^3 stored coefficients; Ue = N (N-2)^2 active rows of an E
    component (PEC, D1).  Per substep:
      rhs_e      (a1/a5): read E1..E3, H1..H3, a, c; write R1..R3            -> 11 U words
      sweep_mod  (a2/a6 first sweep): 24 B per active row (read f, c; write x), 3 components -> 9 Ue
      sweep_mass (a2/a6 other two sweeps): 16 B per active row, 2 x 3 components       -> 12 Ue
      sweep_der  (a3+a4 / a7+a8, uniform mu: the exact derivative-projection identity of
                  SURVEY §8(a)'s note): 24 B per row (read u, base; write out), 2 x 3 -> 18 U;
                  fused schedule (fused_h, the library's default for whole patches): the second
                  projection of a substep and the first of the next apply the same operator to
                  the same field, one pass writes both (read u, Q; write H, Q'): 32 B per row,
                  3 components -> 12 U
      rhs_h      (general mu only, a3/a7): read H_d, Eo, En, b; write G_d, 3 components -> 15 U
                  (then 9 mass sweeps over H: 18 U, counted under sweep_mass)
    Uniform mu: 29 U + 21 Ue words per substep, i.e. (58 U + 42 Ue) * 8 B per step."""
    N = n + p
    U = N ** 3
    Ue = N * (N - 2) ** 2
    w = 8.0
    out = {"rhs_e": 2 * 11 * U * w, "sweep_mod": 2 * 9 * Ue * w, "sweep_mass": 2 * 12 * Ue * w}
    if mu_uniform:
        out["sweep_der"] = 2 * (12 if fused_h else 18) * U * w
    else:
        out["rhs_h"] = 2 * 15 * U * w
        out["sweep_mass"] += 2 * 18 * U * w
    return out


def step_bytes(n: int, p: int, fused_h: bool = True) -> float:
    """Compulsory HBM bytes of one step of the schedule run (uniform mu): (58 U + 42 Ue) * 8 B, or
    (46 U + 42 Ue) * 8 B with the fused H projections."""
    return sum(step_class_bytes(n, p, fused_h=fused_h).values())


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = f"/tmp/adi_clocks_{os.getpid()}.csv"

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        # median over the samples taken under load (top half of the clock samples)
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm)}


def make_inputs(cfg, seed=12345, pinned=False):
    import torch

    n, p = cfg["n"], cfg["p"]
    N = n + p
    eps = workloads.element_eps(n, cfg["material"])
    # seeded random coefficient fields, generated in chunks into (pinned) host tensors
    rng = np.random.default_rng(seed)
    U = N ** 3
    fields = []
    for _ in range(6):
        t = torch.empty(U, dtype=torch.float64, pin_memory=pinned)
        a = t.numpy()
        step = 1 << 24
        for o in range(0, U, step):
            a[o:o + step] = rng.uniform(-1.0, 1.0, size=min(step, U - o))
        fields.append(t)
    return eps, fields


def host_info():
    """Host CPU facts reported next to the one-core oracle number."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"host_cores": os.cpu_count(), "cpu_model": model}


def pin_one_core():
    """Pin this process to one core (the oracle is single-threaded by definition); returns the
    previous affinity mask so it can be restored."""
    try:
        old = os.sched_getaffinity(0)
        core = min(old)
        os.sched_setaffinity(0, {core})
        return old, core
    except (AttributeError, OSError):
        return None, None


def cpu_oracle_rate(cfg, steps: int, sample_n: int, repeats: int = 5):
    """The oracle as it stands (oracle/, one core, pinned) on a bounded sample of the workload:
    the same recipe at n = sample_n, `repeats` timed regions of `steps` steps each (median).
    Returns (DOF-updates/s, seconds per region, description, extra facts)."""
    import oracle

    n, p = sample_n, cfg["p"]
    N = n + p
    old, core = pin_one_core()
    try:
        P = oracle.Patch(n, p, cfg["tau"])
        P.set_materials(workloads.element_eps(n, cfg["material"]))
        P.set_fields(workloads.random_fields(N, 1))
        times = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            P.step(steps)
            times.append(time.perf_counter() - t0)
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    dt = float(np.median(times))
    rate = dof_count(n, p) * steps / dt
    desc = (f"{cfg['name']} recipe at n={n} (N={N}, {dof_count(n, p)} DOF), median of {repeats} timed regions "
            f"of {steps} step(s), single-threaded C oracle pinned to core {core}, setup excluded")
    extra = dict(host_info(), pinned_core=core, seconds_per_region=times)
    return rate, dt, desc, extra


def parity_probe(cfg, n_small: int = 16, steps: int = 2):
    """A small in-run parity number: the bench recipe at n = n_small, `steps` steps, library vs
    oracle on identical seeded inputs (relative L2 per field, D16)."""
    import oracle
    import paper_2103_06998_b200 as adi

    n, p, tau = n_small, cfg["p"], cfg["tau"]
    N = n + p
    eps = workloads.element_eps(n, cfg["material"])
    f = workloads.random_fields(N, 77)
    outs = []
    for P in (adi.Patch(n, p, tau), oracle.Patch(n, p, tau)):
        P.set_materials(eps)
        P.set_fields(f)
        P.step(steps)
        outs.append(P.get_fields())
    errs = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(*outs)]
    return {"max_rel_l2": max(errs), "case": f"{cfg['name']} recipe at n={n}, {steps} steps, GPU vs oracle"}


def dist_init():
    """torch.distributed over NCCL when launched by torchrun with N > 1 (plumbing only: the id
    broadcast and the barriers / max-over-ranks of the timing; the step's exchanges are the
    library's own NCCL communicator)."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch.distributed as dist

        import torch

        local = int(os.environ.get("LOCAL_RANK", "0"))
        dist.init_process_group(backend="nccl", device_id=torch.device("cuda", local))
        return dist, dist.get_rank(), ws
    return None, 0, 1


def run_reference(args, cfg):
    # rank 0 alone runs the CPU oracle; the other ranks exit without work (no collective)
    if int(os.environ.get("RANK", "0")) != 0:
        return
    sample_n = args.oracle_n
    rates = []
    # warm-up steps are untimed; then K timed oracle steps of the bounded sample
    import oracle

    n, p = sample_n, cfg["p"]
    N = n + p
    old_aff, core = pin_one_core()
    P = oracle.Patch(n, p, cfg["tau"])
    P.set_materials(workloads.element_eps(n, cfg["material"]))
    P.set_fields(workloads.random_fields(N, 1))
    P.step(args.warmup)
    t0 = time.perf_counter()
    P.step(args.steps)
    dt = time.perf_counter() - t0
    if old_aff is not None:
        os.sched_setaffinity(0, old_aff)
    rate = dof_count(n, p) * args.steps / dt
    desc = (f"{cfg['name']} recipe at n={n} (N={N}), {args.steps} timed steps after {args.warmup} warm-up, "
            f"single-threaded C oracle pinned to core {core}")
    out = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(cfg, args),
        "cpu_baseline": dict({"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
                             **host_info()),
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(out)


def parallelism_label(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws == 1:
        return "single GPU, whole patch, CUDA graph per step"
    return (f"z-slab decomposition over {ws} GPUs (one process per GPU), the library's distributed adi_step: "
            "NCCL halo exchange before the RHS stencils; every z sweep by the partitioned (SPIKE) solve in "
            "place (NEXT-1: 2p interface values per fiber all-gathered for the mass sweeps and derivative "
            "projections, 2p + 4p^2 spike tips for the row-modified sweep), no transposes; one CUDA graph per step")


def config_dict(cfg, args):
    n, p = cfg["n"], cfg["p"]
    return {
        "workload": (f"{cfg['name']}: {n}^3 elements, p={p} (C^{p - 1}), N={n + p}, PEC, tau={cfg['tau']}, "
                     f"material={cfg['material']}, seeded random fields"),
        "n": n, "p": p, "N": n + p, "tau": cfg["tau"], "dof_per_step": dof_count(n, p),
        "l2_policy": "inputs larger than L2 (each field %.2f GB > 126 MB)" % ((n + p) ** 3 * 8 / 1e9),
        "parallelism": parallelism_label(args),
    }


class _Whole:
    """Single GPU: the whole patch in one library handle, one CUDA graph per step."""

    def __init__(self, cfg, local, seed):
        import paper_2103_06998_b200 as adi

        n, p, tau = cfg["n"], cfg["p"], cfg["tau"]
        self.N = n + p
        eps, self.fields = make_inputs(cfg, seed=seed, pinned=True)
        self.G = adi.Patch(n, p, tau, device=local)
        self.G.set_materials(eps)
        self.G.set_fields(self.fields)
        self.stream_handle = self.G.stream
        self.local_bytes = 6 * self.N ** 3 * 8

    def step(self, k):
        self.G.step(k)

    def timing(self, on):
        self.G.set_timing(on)

    def report(self):
        return self.G.timing_report()

    def e2e(self, out_host):
        self.G.set_fields(self.fields)  # pinned host -> device
        self.G.step(self.k_e2e)
        self.G.get_fields(out_host)     # device -> pinned host (synchronises)

    def launches_per_step(self):
        return self.G.launches_per_step

    def close(self):
        self.G.close()


class _Dist:
    """N > 1 GPUs: this rank's z-slab patch; the library runs the distributed schedule itself
    (adi_step over NCCL: halo exchanges and the partitioned z-solve of every z sweep; one CUDA
    graph per step)."""

    def __init__(self, cfg, local, seed):
        import torch

        from paper_2103_06998_b200.dist import create_patch

        n, p, tau = cfg["n"], cfg["p"], cfg["tau"]
        self.N = N = n + p
        self.G = create_patch(n, p, tau, device=local)
        self.zsolve_active = self.G.set_zsolve(1)
        _, k0, k1 = self.G.layout()
        self.nz = k1 - k0
        self.G.set_materials(workloads.element_eps(n, cfg["material"]))
        rng = np.random.default_rng(seed)
        self.fields = [torch.from_numpy(rng.uniform(-1.0, 1.0, size=self.nz * N * N)).pin_memory() for _ in range(6)]
        self.G.set_fields(self.fields)
        self.stream_handle = self.G.stream
        self.local_bytes = 6 * self.nz * N * N * 8

    def step(self, k):
        self.G.step(k)

    def timing(self, on):
        self.G.set_timing(on)

    def report(self):
        return self.G.timing_report()

    def e2e(self, out_host):
        self.G.set_fields(self.fields)
        self.G.step(self.k_e2e)
        self.G.get_fields(out_host)

    def launches_per_step(self):
        return self.G.launches_per_step

    def close(self):
        self.G.close()


def run_ours(args, cfg):
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist, rank, ws = dist_init()
    import paper_2103_06998_b200 as adi

    adi.build()
    n, p, tau = cfg["n"], cfg["p"], cfg["tau"]
    N = n + p
    U = N ** 3
    S = (_Whole if ws == 1 else _Dist)(cfg, local, 1000 + rank)
    S.step(args.warmup)
    torch.cuda.synchronize()
    # ---------------- timed region (device-resident state) ----------------
    stream = torch.cuda.ExternalStream(S.stream_handle, device=local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        S.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clocks = clk.summary()
    # ---------------- per-kernel breakdown (same steps, each launch bracketed by events) ----
    S.timing(True)
    S.timed_steps = max(1, min(args.steps, 3))
    S.step(S.timed_steps)
    rep = S.report()
    S.timing(False)
    lps = S.launches_per_step()
    # ---------------- end-to-end through the public API, host buffers ---------
    out_host = [torch.empty(S.local_bytes // 48, dtype=torch.float64, pin_memory=True) for _ in range(6)]
    S.k_e2e = args.steps
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    S.e2e(out_host)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    h2d = S.local_bytes * ws / args.steps
    d2h = S.local_bytes * ws / args.steps
    launches = args.steps * lps  # kernels of this library in the timed region (per rank)
    ms_t = torch.tensor([ms, e2e_s * 1e3], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(ms_t[0]), float(ms_t[1])
    if rank != 0:
        S.close()
        dist.destroy_process_group()
        return
    dofs = dof_count(n, p)
    value = dofs * args.steps / (ms * 1e-3)  # the whole patch (all ranks together)
    e2e_value = dofs * args.steps / (e2e_ms * 1e-3)
    # roofline of the dominant kernel class: survey bytes of the class per step, divided over
    # the class's launches per step (rep covers `timed_steps` steps)
    peak, peak_src = hbm_peak()
    cls_bytes = step_class_bytes(n, p, fused_h=(ws == 1))  # the slab path keeps two projections
    algo = {k: v * S.timed_steps / rep[k][1] for k, v in cls_bytes.items() if rep.get(k, (0, 0))[1] > 0}
    cls = max(algo, key=lambda k: rep[k][0])
    t_cls, n_cls = rep[cls]
    achieved = algo[cls] / (t_cls * 1e-3 / n_cls) / 1e9
    traffic = None
    traffic_src = None
    try:
        with open(TRAFFIC_PATH) as f:
            tr = json.load(f)
        if tr.get("config") == cfg["name"] and cls in tr.get("bytes_per_launch", {}):
            traffic = tr["bytes_per_launch"][cls]
            traffic_src = tr.get("source")
    except Exception:
        pass
    kernels = {}
    for k, (t, cnt) in rep.items():
        if cnt == 0:
            continue
        kd = {"ms_total": t, "launches": cnt, "share": t / sum(v[0] for v in rep.values())}
        if k in algo:
            kd["algorithmic_bytes_per_launch"] = algo[k]
            kd["achieved_gbs"] = algo[k] / (t * 1e-3 / cnt) / 1e9
            kd["frac"] = kd["achieved_gbs"] / peak
        kernels[k] = kd
    # end-to-end HBM fraction of the step (algorithmic bytes of the schedule run)
    sbytes = step_bytes(n, p, fused_h=(ws == 1))
    cpu = None
    if not args.no_cpu_baseline and ws == 1:  # the CPU oracle baseline: rank 0 at N = 1 only
        rate, dt, desc, extra = cpu_oracle_rate(cfg, args.oracle_steps, args.oracle_n)
        cpu = dict({"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc, "seconds": dt},
                   **extra)
    parity = parity_probe(cfg) if ws == 1 else None
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config_dict(cfg, args),
        "roofline": {"bound": "hbm", "kernel": cls, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": algo[cls],
                     "bytes_basis": "SURVEY §8(a)/(d) compulsory bytes of the class per step / launches per step"},
        "step_hbm_frac": (sbytes / (ms * 1e-3 / args.steps) / 1e9) / peak,
        "step_algorithmic_bytes": sbytes,
        "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms": e2e_ms, "note": "set_fields(pinned host) + step(K) via CUDA graph + get_fields(pinned host)"},
        "gpu_launches": launches,
        "clocks": clocks,
        "parity": parity,
    }
    emit(out)
    S.close()
    if dist is not None:
        dist.destroy_process_group()


_JSON_FD = None


def emit(out):
    """The one JSON line, to the process's original stdout (everything else -- NCCL's banner
    included, which it writes to fd 1 -- goes to stderr; see main())."""
    line = json.dumps(out) + "\n"
    if _JSON_FD is None:
        sys.stdout.write(line)
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, line.encode())


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)  # C-level writes to stdout (NCCL, CUDA libraries) land on stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--oracle-n", type=int, default=64,
                    help="n of the bounded CPU-oracle sample (c5 recipe at n=64: ~2 s per oracle step)")
    ap.add_argument("--oracle-steps", type=int, default=2,
                    help="steps per timed oracle region (5 regions, median)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = dict(workloads.CONFIGS[args.config])
    cfg["name"] = args.config
    if args.warmup < 3:
        print("warning: warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
