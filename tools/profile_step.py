"""Run a few ADI steps of a BASELINE config on cuda:0 (for ncu / compute-sanitizer).

    python tools/profile_step.py --config c4 --steps 2 [--timing]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2103_06998_b200 as adi  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--timing", action="store_true")
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
n = a.n or cfg["n"]
p, tau = cfg["p"], cfg["tau"]
N = n + p
G = adi.Patch(n, p, tau)
G.set_materials(workloads.element_eps(n, cfg["material"]))
G.set_fields(workloads.random_fields(N, 0))
if a.timing:
    G.set_timing(True)
t0 = time.perf_counter()
G.step(a.steps)
G.synchronize()
dt = time.perf_counter() - t0
print(f"{a.config} n={n} p={p}: {a.steps} steps in {dt*1e3:.1f} ms")
if a.timing:
    for k, (ms, cnt) in G.timing_report().items():
        if cnt:
            print(f"  {k:11s} {ms:9.3f} ms  {cnt:4d} launches  {ms/cnt:8.4f} ms/launch")
