"""Cost of the library's distributed schedule on ONE B200 (loopback transport).

    python tools/dist_timing.py --config c5 --ranks 1,2,4 --steps 4

R = 1 is the whole patch.  R > 1 runs R slab patches of the same c5 patch through adi_step with
the loopback group (adi_loopback_create): one host thread per rank, all on cuda:0, exchanges as
device copies after a host barrier -- so the R ranks' kernels share one GPU and the wall time
per step is (sum of the ranks' work) + exchange + synchronisation.  What this measures is the
distributed algorithm's overhead (halo'd slab RHS, partitioned z-solve with its tips / all-gathers,
slab-local x/y sweeps, R-times more launches) against the whole patch, not multi-GPU scaling
(which needs R GPUs: bench.py --gpus R under torchrun).  Prints one JSON line.
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2103_06998_b200 as adi  # noqa: E402
import workloads  # noqa: E402


def run(R, n, p, tau, eps, fields, warm, steps, timing=False):
    N = n + p
    if R == 1:
        G = adi.Patch(n, p, tau)
        G.set_materials(eps)
        G.set_fields(fields)
        G.step(warm)
        G.synchronize()
        t0 = time.perf_counter()
        G.step(steps)
        G.synchronize()
        dt = time.perf_counter() - t0
        lp = G.launches_per_step
        rep = None
        if timing:
            G.set_timing(True)
            G.step(steps)
            G.synchronize()
            rep = [{k: round(v[0] / steps, 3) for k, v in G.timing_report().items() if v[1]}]
        G.close()
        return dt / steps, [lp], [True], rep
    grp = adi.Loopback(R)
    bar = threading.Barrier(R)
    res, err = [None] * R, []

    def work(r):
        try:
            P = adi.Patch(n, p, tau, device=0, rank=r, nranks=R, loopback=grp)
            act = P.set_zsolve(1)
            _, k0, k1 = P.layout()
            P.set_materials(eps)
            P.set_fields([np.ascontiguousarray(x.reshape(N, N, N)[k0:k1]).reshape(-1) for x in fields])
            P.step(warm)
            P.synchronize()
            if timing:
                P.set_timing(True)
            bar.wait()
            t0 = time.perf_counter()
            P.step(steps)
            P.synchronize()
            bar.wait()
            rep = {k: round(v[0] / steps, 3) for k, v in P.timing_report().items() if v[1]} if timing else None
            res[r] = (time.perf_counter() - t0, P.launches_per_step, act, rep)
            P.close()
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            bar.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    grp.close()
    if err:
        raise err[0]
    return max(x[0] for x in res) / steps, [x[1] for x in res], [x[2] for x in res], [x[3] for x in res]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--ranks", default="1,2,4")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--timing", action="store_true", help="per-class ms per step of every rank (library events; ranks overlap on the GPU)")
    a = ap.parse_args()
    cfg = workloads.CONFIGS[a.config]
    n = a.n or cfg["n"]
    p, tau = cfg["p"], cfg["tau"]
    N = n + p
    eps = workloads.element_eps(n, cfg["material"])
    fields = workloads.random_fields(N, 0)
    out = {"config": a.config, "n": n, "p": p, "steps": a.steps, "transport": "loopback (one GPU)", "runs": []}
    for R in [int(x) for x in a.ranks.split(",")]:
        ms, launches, act, rep = run(R, n, p, tau, eps, fields, a.warmup, a.steps, a.timing)
        out["runs"].append({"ranks": R, "ms_per_step": ms * 1e3, "dof_updates_per_s": 6 * N ** 3 / ms,
                            "launches_per_step_per_rank": launches, "partitioned_zsolve": act})
        if a.timing:
            out["runs"][-1]["class_ms_per_step"] = rep
    base = out["runs"][0]["ms_per_step"]
    for r in out["runs"]:
        r["overhead_vs_first"] = r["ms_per_step"] / base
    print(json.dumps(out))


if __name__ == "__main__":
    main()
